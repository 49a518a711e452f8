cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "chain or cfg5 or interleave" > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 300 python scripts/cfg5_breakdown.py > gpurun_out/cfg5.log 2>&1

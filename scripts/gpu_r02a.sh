# round 2 first call: state check (gpu tests), geometry A/B, role isolation
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/a_tests.log
timeout 300 python scripts/tc05_geom.py 30 > gpurun_out/a_geom.log 2>&1; echo "rc=$?" >> gpurun_out/a_geom.log

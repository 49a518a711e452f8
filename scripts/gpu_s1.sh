# session re-entry check: smoke, gpu tests, bench (driver protocol), reference arm
cd $GRAFT_REPO_ROOT
timeout 300 python __graft_entry__.py --smoke > gpurun_out/s1_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s1_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/s1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s1_tests.log
timeout 900 python bench.py > gpurun_out/s1_bench.log 2>&1; echo "rc=$?" >> gpurun_out/s1_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s1_ref.log 2>&1; echo "rc=$?" >> gpurun_out/s1_ref.log

# ncu source-level capture of the w=48 (4-plane) fused kernel
cd $GRAFT_REPO_ROOT
timeout 120 python scripts/tc05_one.py --w48 > gpurun_out/b_one.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc05 -s 1 -c 1 \
    -o gpurun_out/b_prof_w48 python scripts/tc05_one.py --w48 > gpurun_out/b_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/b_ncu.log
timeout 900 python -m pytest tests/test_gpu_api.py -q -m gpu -x -p no:cacheprovider > gpurun_out/b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/b_tests.log

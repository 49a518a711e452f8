cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_imma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_imma.log
timeout 300 python scripts/imma_probe.py > gpurun_out/imma_probe.log 2>&1; echo "rc=$?" >> gpurun_out/imma_probe.log
CMD="python scripts/imma_probe.py 2"
$CMD > gpurun_out/imma_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:conv_imma -s 2 -c 1 -o gpurun_out/prof_imma $CMD > gpurun_out/ncu_imma.log 2>&1
echo "ncu rc=$?" >> gpurun_out/imma_plain.log

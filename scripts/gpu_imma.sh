cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_imma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_imma.log
timeout 300 python scripts/imma_probe.py > gpurun_out/imma_probe.log 2>&1; echo "rc=$?" >> gpurun_out/imma_probe.log

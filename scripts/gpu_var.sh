cd $GRAFT_REPO_ROOT
timeout 60 python scripts/tc05_debug.py 0 > gpurun_out/var.log 2>&1 || { echo "main rc=$?" >> gpurun_out/var.log; exit 1; }
for v in "$@"; do echo "== $v" >> gpurun_out/var.log; timeout 60 python scripts/tc05_variant.py libnent_b200_$v.so 0 >> gpurun_out/var.log 2>&1 || echo "rc=$?" >> gpurun_out/var.log; done
NENT_TIMERS_LIB=libnent_b200_timers.so timeout 60 python scripts/tc05_timers.py 0 2>&1 | tail -n 2 >> gpurun_out/var.log
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -x -k "tcgen05 or fused or chain" 2>&1 | tail -n 2 >> gpurun_out/var.log

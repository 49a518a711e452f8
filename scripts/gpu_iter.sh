# one iteration: role timings first (bounded), then tcgen05 parity tests and a short bench line
cd $GRAFT_REPO_ROOT
for d in 0 29760 4 256 17413; do timeout 60 python scripts/tc05_debug.py $d >> gpurun_out/it_dbg.log 2>&1 || { echo "debug $d rc=$?" >> gpurun_out/it_dbg.log; exit 1; }; done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -x -k "tcgen05 or fused or chain" > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/it_bench.log 2>&1; echo "rc=$?" >> gpurun_out/it_bench.log

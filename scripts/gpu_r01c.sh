# round-1 (third session) check: full gpu suite, default bench, reference arm, smoke
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r01c_smi.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r01c_smoke.log
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r01c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01c_pytest.log
timeout 600 python bench.py > gpurun_out/r01c_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01c_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01c_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r01c_bench_ref.log

# bench (default args, as the driver runs it), reference arm, then the ncu passes
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
bash scripts/profile.sh

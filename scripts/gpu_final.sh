# round-1 final evidence: smoke, full gpu tests, default bench, reference arm, launch list, ncu full capture
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/z_smoke.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/z_pytest.log
timeout 600 python bench.py > gpurun_out/z_bench.log 2>&1; echo "rc=$?" >> gpurun_out/z_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/z_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/z_bench_ref.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/z_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/z_launches.csv $CMD > gpurun_out/z_ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/z_plain.log
timeout 120 python scripts/tc05_one.py > gpurun_out/z_one.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc05 -s 1 -c 1 \
    -o gpurun_out/z_prof_tc05 python scripts/tc05_one.py > gpurun_out/z_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/z_one.log

# Evidence run of the committed build: smoke, GPU tests, bench (driver
# protocol), reference arm, then the ncu passes (each after its own command
# exited 0 without ncu).  Usage: gpurun -- 'bash scripts/gpu_round.sh TAG'
TAG=${1:-r02}
cd $GRAFT_REPO_ROOT
timeout 300 python __graft_entry__.py --smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/${TAG}_clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
kill $SMI
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ref.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_plain.log
CMD2="python scripts/m3_time.py 2"
$CMD2 > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:conv_tc05_m3 -s 2 -c 1 \
    -o gpurun_out/${TAG}_prof_m3 $CMD2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_plain2.log
# the cfg3 kernel: one full capture as well
CMD3="python scripts/m4_time.py 2"
$CMD3 > gpurun_out/${TAG}_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc05_m4 -s 2 -c 1 \
    -o gpurun_out/${TAG}_prof_m4 $CMD3 > gpurun_out/${TAG}_ncu_full_m4.log 2>&1
echo "full m4 rc=$?" >> gpurun_out/${TAG}_plain3.log
# per-CTA timelines (stamps builds, scripts/build_variant.py), the old-vs-new A/B when the
# previous build's library is there, and the NVML power / clock probe
if [ -f scripts/_bin/libnent_b200_stamps.so ]; then
  timeout 120 python scripts/with_variant.py libnent_b200_stamps.so scripts/m3_time.py 50 --dump > gpurun_out/${TAG}_timeline_m3.log 2>&1
fi
if [ -f scripts/_bin/libnent_b200_stamps4.so ]; then
  timeout 120 python scripts/with_variant.py libnent_b200_stamps4.so scripts/m4_time.py 50 --dump > gpurun_out/${TAG}_timeline_m4.log 2>&1
fi
if [ -f scripts/_bin/libnent_b200_old.so ]; then
  for i in 1 2; do
    echo "previous build (r02e)"; timeout 120 python scripts/with_variant.py libnent_b200_old.so scripts/m3_time.py 200
    echo "this build"; timeout 120 python scripts/m3_time.py 200
  done > gpurun_out/${TAG}_ab_m3.log 2>&1
fi
timeout 120 python scripts/m4_time.py 200 > gpurun_out/${TAG}_time_m4_m8.log 2>&1
timeout 120 python scripts/m8_time.py 100 >> gpurun_out/${TAG}_time_m4_m8.log 2>&1
timeout 120 python scripts/power_probe.py 4 > gpurun_out/${TAG}_power.log 2>&1

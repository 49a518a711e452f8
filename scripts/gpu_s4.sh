cd $GRAFT_REPO_ROOT
timeout 120 python scripts/m3_time.py 20 > gpurun_out/s4_main.log 2>&1
for v in nostage nosts noepi nomma; do
timeout 120 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 20 > gpurun_out/s4_$v.log 2>&1
done
for v in timers nostage_t nosts_t noepi_t; do
timeout 120 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 1 > gpurun_out/s4_$v.log 2>&1
done

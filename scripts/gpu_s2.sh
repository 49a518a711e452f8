cd $GRAFT_REPO_ROOT
timeout 120 python scripts/m3_time.py 20 > gpurun_out/s2_main.log 2>&1
for v in nomma noepi nostore; do
timeout 120 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 20 > gpurun_out/s2_$v.log 2>&1
done
for v in timers noepi_t nomma_t; do
timeout 120 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 1 > gpurun_out/s2_$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc05_m3 -s 2 -c 1 \
    -o gpurun_out/s2_prof_m3 python scripts/m3_time.py 2 > gpurun_out/s2_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/s2_ncu.log

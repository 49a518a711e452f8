cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 120 python scripts/m3_time.py 20 >> gpurun_out/x_main.log 2>&1
timeout 120 python scripts/with_variant.py libnent_b200_susp.so scripts/m3_time.py 20 >> gpurun_out/x_susp.log 2>&1
timeout 120 python scripts/with_variant.py libnent_b200_spin.so scripts/m3_time.py 20 >> gpurun_out/x_spin.log 2>&1
done

cd $GRAFT_REPO_ROOT
./scripts/_bin/mma_n_probe > gpurun_out/s7_probe.log 2>&1
timeout 120 python scripts/m3_time.py 20 > gpurun_out/s7_main.log 2>&1
for v in nstage2 sleep32 sleep256 nomma nomma_nostore nomma_noepi nomma_nostage; do
timeout 120 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 20 > gpurun_out/s7_$v.log 2>&1
done
timeout 120 python scripts/with_variant.py libnent_b200_nomma_t.so scripts/m3_time.py 1 > gpurun_out/s7_nomma_t.log 2>&1

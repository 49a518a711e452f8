# A/B of variant builds (scripts/_bin) on the full fused cfg2 kernel, 4 alternations, + exactness of each variant
cd $GRAFT_REPO_ROOT
for v in "$@"; do timeout 300 python scripts/with_variant.py libnent_b200_$v.so scripts/tc05_check.py > gpurun_out/ab2_check_$v.log 2>&1; echo "rc=$?" >> gpurun_out/ab2_check_$v.log; done
for rep in 1 2 3 4; do
timeout 60 python scripts/tc05_debug.py 0 0 2>&1 | sed 's/^/main /' >> gpurun_out/ab2.log
for v in "$@"; do timeout 60 python scripts/tc05_variant.py libnent_b200_$v.so 0 0 2>&1 | sed "s/^/$v /" >> gpurun_out/ab2.log; done
done

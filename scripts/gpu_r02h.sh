cd $GRAFT_REPO_ROOT
echo main >> gpurun_out/h.log; timeout 120 python scripts/m3_debug.py 1000000 256 >> gpurun_out/h.log 2>&1
for v in NOTMA NOMMA NOLD NOSTORE; do echo "variant $v" >> gpurun_out/h.log; timeout 120 python scripts/with_variant.py libnent_b200_m3$v.so scripts/m3_debug.py 1000000 256 >> gpurun_out/h.log 2>&1; done

# role-isolation timings of the tcgen05 fused conv (each mode in its own process, bounded)
cd $GRAFT_REPO_ROOT
for d in "$@"; do timeout 60 python scripts/tc05_debug.py $d >> gpurun_out/dbg.log 2>&1 || echo "debug $d rc=$?" >> gpurun_out/dbg.log; done

cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 60 python scripts/tc05_debug.py 0 17413 >> gpurun_out/pad.log 2>&1
NENT_PAD=1 timeout 60 python scripts/tc05_debug.py 0 17413 | sed 's/^/pad /' >> gpurun_out/pad.log 2>&1
done

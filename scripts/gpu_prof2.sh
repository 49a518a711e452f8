cd $GRAFT_REPO_ROOT

timeout 300 python scripts/tc05_one.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc05 -s 1 -c 1 \
    -o gpurun_out/prof_tc05_v3 python scripts/tc05_one.py > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log

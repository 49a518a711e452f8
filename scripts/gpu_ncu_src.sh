cd $GRAFT_REPO_ROOT
timeout 120 python scripts/tc05_one.py > gpurun_out/one.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc05 -s 1 -c 1 \
    -o gpurun_out/prof_src python scripts/tc05_one.py > gpurun_out/ncu_src.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_src.log

cd $GRAFT_REPO_ROOT
timeout 120 python scripts/m3_time.py 2 > gpurun_out/u_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc05_m3 -s 2 -c 1 \
    -o gpurun_out/u_prof_m3 python scripts/m3_time.py 2 > gpurun_out/u_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/u_ncu.log

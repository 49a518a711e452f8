cd $GRAFT_REPO_ROOT
timeout 120 python scripts/m3_time.py 2 > gpurun_out/s5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:conv_tc05_m3 -s 2 -c 1 \
    -o gpurun_out/s5_prof_m3 python scripts/m3_time.py 2 > gpurun_out/s5_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/s5_ncu.log

#!/bin/bash
# ncu evidence for the bench: launch list (cold, serialised) + one full capture
# of the headline kernel (tcgen05 fused conv).  Each ncu pass runs only after
# the same command exited 0 without ncu (B200_PROFILING.md).
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/plain.log
CMD2="python scripts/tc05_one.py"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc05 -s 1 -c 1 \
    -o gpurun_out/prof_tc05 $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/plain2.log

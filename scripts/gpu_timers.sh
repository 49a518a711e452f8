cd $GRAFT_REPO_ROOT
for lib in libnent_b200_timers.so libnent_b200_timers8.so; do
for d in 0 17413 29760; do echo "$lib $d" >> gpurun_out/tm.log; NENT_TIMERS_LIB=$lib timeout 60 python scripts/tc05_timers.py $d >> gpurun_out/tm.log 2>&1 || { echo "rc=$?" >> gpurun_out/tm.log; exit 1; }; done; done

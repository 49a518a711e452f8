cd $GRAFT_REPO_ROOT
export CUDA_LAUNCH_BLOCKING=1
echo check >> gpurun_out/i.log; timeout 120 python scripts/with_variant.py libnent_b200_m3CHECK.so scripts/m3_debug.py 1000000 256 >> gpurun_out/i.log 2>&1
echo check_small >> gpurun_out/i.log; timeout 120 python scripts/with_variant.py libnent_b200_m3CHECK.so scripts/m3_debug.py 909312 256 >> gpurun_out/i.log 2>&1

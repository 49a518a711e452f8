cd $GRAFT_REPO_ROOT
for n in 1000000 16777216; do
echo "prefix n=$n" >> gpurun_out/j.log; timeout 120 python scripts/with_variant.py libnent_b200_prefix.so scripts/m3_debug.py $n 256 >> gpurun_out/j.log 2>&1
echo "prefix blocking n=$n" >> gpurun_out/j.log; CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/with_variant.py libnent_b200_prefix.so scripts/m3_debug.py $n 256 >> gpurun_out/j.log 2>&1
echo "fixed n=$n" >> gpurun_out/j.log; timeout 120 python scripts/m3_debug.py $n 256 >> gpurun_out/j.log 2>&1
echo "fixed K=64 n=$n" >> gpurun_out/j.log; timeout 120 python scripts/m3_debug.py $n 64 >> gpurun_out/j.log 2>&1
done

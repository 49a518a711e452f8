cd $GRAFT_REPO_ROOT
export CUDA_LAUNCH_BLOCKING=1
for n in 18508 18509 100000; do for K in 1 256; do
echo "n=$n K=$K" >> gpurun_out/z.log
timeout 60 python scripts/with_variant.py libnent_b200_check.so scripts/m3_debug.py $n $K >> gpurun_out/z.log 2>&1
done; done

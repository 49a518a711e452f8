cd $GRAFT_REPO_ROOT
for n in 909312 909313 1000000 1048576 4194304 16777216; do
  echo "n=$n" >> gpurun_out/g_scale.log
  timeout 120 python scripts/m3_debug.py $n 256 >> gpurun_out/g_scale.log 2>&1; echo "rc=$?" >> gpurun_out/g_scale.log
done

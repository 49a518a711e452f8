# A/B: main library vs variant builds (scripts/_bin), same debug modes, alternated twice
cd $GRAFT_REPO_ROOT
M="$1"; shift
for rep in 1 2; do
timeout 60 python scripts/tc05_debug.py $M 2>&1 | sed 's/^/main /' >> gpurun_out/ab.log || { echo "main rc=$?" >> gpurun_out/ab.log; exit 1; }
for v in "$@"; do timeout 60 python scripts/tc05_variant.py libnent_b200_$v.so $M 2>&1 | sed "s/^/$v /" >> gpurun_out/ab.log || echo "$v rc=$?" >> gpurun_out/ab.log; done
done
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -n 2 >> gpurun_out/ab.log

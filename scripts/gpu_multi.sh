# N>1 bench paths on a one-GPU box: ranks share the device, exchanges over gloo (host)
cd $GRAFT_REPO_ROOT
NENT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/m_bench2.log 2>&1; echo "rc=$?" >> gpurun_out/m_bench2.log
NENT_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --config 3 --steps 4 --warmup 3 > gpurun_out/m_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/m_cfg3.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/m_ref2.log 2>&1; echo "rc=$?" >> gpurun_out/m_ref2.log
NENT_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 8 --config 5 --steps 3 --warmup 3 > gpurun_out/m_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/m_cfg5.log

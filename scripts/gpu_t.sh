cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -m gpu -x -p no:cacheprovider -k "outer" > gpurun_out/t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t_tests.log
timeout 600 python - > gpurun_out/t_outer.log 2>&1 <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1509_03838_b200 import fused, workloads
from bench import timed_ms
wl = workloads.make(4)
c = torch.from_numpy(wl.c[:, :16]).cuda().to(torch.int32).contiguous()
n4 = wl.c.shape[2]
out = torch.empty((3, 16, n4, n4), dtype=torch.int32, device='cuda')
st = torch.cuda.current_stream()
ms = timed_ms(lambda: fused.entangled_outer(wl.params, c, wl.g, out=out), st, 3)
ref = wl.c[:, :2, :, None] * wl.g[None, None, None, :]
print('ms', ms, 'GB/s', out.numel()*4/ms/1e6, 'exact', bool(np.array_equal(out[:, :2].to(torch.int64).cpu().numpy(), ref)))
PY

"""Single-process emulation of bench.py's halo-split shards on one GPU,
compared slice by slice with one fused launch over the whole signal."""
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _device as D, fused  # noqa: E402
from bench import make_inputs  # noqa: E402

n, K, world = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20, 256, 2
H = K - 1
dev = torch.device("cuda", 0)
params, _, g = make_inputs(0, n, K)
cs = [make_inputs(p, n, K)[1] for p in range(world)]
full = np.concatenate(cs, axis=1)
for flavor in (fused.conv_flavor(2048 * ((1 << params.l) + 1), g, n_out=1 << 30),
               fused.conv_flavor(2048 * ((1 << params.l) + 1), g, allow_imma=False)):
    gd = D.taps_tensor(g, flavor)
    L = full.shape[1] + H
    ref = D.fused_conv(torch.from_numpy(full).to(dev).to(torch.int32), gd, K, params.l, flavor, None,
                       True, L, n_in=full.shape[1], out_dtype=torch.int64).cpu().numpy()
    for p in range(world):
        c = torch.from_numpy(cs[p]).to(dev).to(torch.int32)
        halo = torch.zeros((3, H), dtype=torch.int32, device=dev)
        if p > 0:
            halo = torch.from_numpy(cs[p - 1][:, n - H:]).to(dev).to(torch.int32)
        x = torch.cat([halo, c], dim=1).contiguous()
        n_out = n + (H if p == world - 1 else 0)
        d = D.fused_conv(x, gd, K, params.l, flavor, None, True, H + n + H, n_in=H + n, y_begin=H,
                         n_out=n_out, out_dtype=torch.int64).cpu().numpy()
        want = ref[:, p * n:p * n + n_out]
        bad = np.argwhere(d != want)
        print(hex(flavor), "rank", p, "equal", np.array_equal(d, want), "nbad", len(bad),
              "first", bad[:3].tolist())

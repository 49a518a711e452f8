"""The five BASELINE configs at FULL size on the B200, bit-exact against the
reference's known answers (tests/golden/digests.json, produced by running the
reference API on the canonical seeded inputs), for every single-stream failure.
cfg4's outer products (3.3e12 values) are checked by the exact closed-form
sums over the whole batch plus elementwise on sampled vectors."""

import hashlib

import numpy as np
import pytest
import torch

import paper_1509_03838_b200 as nent
from paper_1509_03838_b200 import fused, workloads

pytestmark = pytest.mark.gpu


def sha(a):
    if isinstance(a, torch.Tensor):
        a = a.to(torch.int64).cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def wls():
    return {}


def get(wls, cfg):
    if cfg not in wls:
        wls[cfg] = workloads.make(cfg)
    return wls[cfg]


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_fused_conv_digest_every_failure(digests, wls, cfg):
    wl = get(wls, cfg)
    dev = nent.StreamBlock(wl.params, torch.from_numpy(wl.c).cuda().to(torch.int32))
    want = digests[f"cfg{cfg}"]["d"]
    for r in [None] + list(range(wl.m)):
        res = fused.entangled_conv(dev, wl.g, failed=r)
        assert sha(res.outputs.data) == want, (cfg, r, res.flavor)
        if r is None:
            assert res.mismatches == 0


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_plain_conv_digest(digests, wls, cfg):
    wl = get(wls, cfg)
    dev = nent.StreamBlock(wl.params, torch.from_numpy(wl.c).cuda().to(torch.int32))
    res = fused.plain_conv(dev, wl.g)
    assert sha(res.outputs.data) == digests[f"cfg{cfg}"]["d"]


@pytest.mark.parametrize("cfg", [1, 2])
def test_staged_reference_api_digests(digests, wls, cfg):
    """entangle -> apply_entangled(conv) -> poison -> disentangle through the
    reference-shaped API on device blocks, checking eps and delta digests too."""
    wl = get(wls, cfg)
    p = wl.params
    L = wl.n + wl.K - 1
    pad = torch.zeros((wl.m, L), dtype=torch.int64, device="cuda")
    pad[:, : wl.n] = torch.from_numpy(wl.c).cuda()
    ent = nent.entangle(nent.StreamBlock(p, pad))
    assert sha(ent.data) == digests[f"cfg{cfg}"]["eps"]
    op = nent.LsbOp(nent.OpKind.CIRCULAR_CONVOLUTION, nent.Kernel.of_vector(wl.g))
    delta = nent.apply_entangled(op, ent)
    assert sha(delta.data) == digests[f"cfg{cfg}"]["delta"]
    for r in [None] + list(range(wl.m)):
        d = delta.copy()
        if r is not None:
            from paper_1509_03838_b200 import _device as D
            D.poison(d.data[r], p.w)
        rec = nent.disentangle(d, failed=r)
        assert sha(rec.data) == digests[f"cfg{cfg}"]["d"], r


def test_cfg5_chain_digest_every_failure(digests, wls):
    wl = get(wls, 5)
    for r in [None] + list(range(8)):
        res = fused.entangled_chain_conv(nent.StreamBlock(wl.params, wl.c), wl.scale, wl.add,
                                         wl.perm, wl.g, failed=r)
        assert sha(res.outputs.data) == digests["cfg5"]["d"], r


def test_cfg4_inner_digest_every_failure(digests):
    wl = workloads.make(4)
    c = torch.from_numpy(wl.c).cuda().to(torch.int32)
    for r in [None, 0, 1, 2]:
        res = fused.entangled_inner(wl.params, c, wl.g, failed=r)
        assert sha(res.outputs.data) == digests["cfg4_inner"]["d"], r
        if r is None:
            assert res.mismatches == 0


def test_cfg4_outer_closed_form_and_samples():
    wl = workloads.make(4)
    m, B, n = wl.c.shape
    c = torch.from_numpy(wl.c).cuda().to(torch.int32)
    # whole batch, nothing materialised: per-(stream, vector) sums of d
    sums = torch.zeros((m, B), dtype=torch.int64, device="cuda")
    chunk = 8192
    for b0 in range(0, B, chunk):
        part = torch.zeros((m, chunk), dtype=torch.int64, device="cuda")
        fused.entangled_outer(wl.params, c[:, b0:b0 + chunk], wl.g, failed=1, out=None, sums=part)
        sums[:, b0:b0 + chunk] = part
    expect = wl.c.sum(axis=2) * int(wl.g.sum())
    assert np.array_equal(sums.cpu().numpy(), expect)
    # elementwise on sampled vectors, every failure index
    for b in (0, 1, 4095, 65535):
        for r in (None, 0, 1, 2):
            out = torch.empty((m, 1, n, n), dtype=torch.int32, device="cuda")
            fused.entangled_outer(wl.params, c[:, b:b + 1].contiguous(), wl.g, failed=r, out=out,
                                  sums=None)
            ref = wl.c[:, b, :, None] * wl.g[None, None, :]
            assert np.array_equal(out[:, 0].to(torch.int64).cpu().numpy(), ref), (b, r)

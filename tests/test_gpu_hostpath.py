"""The host-buffer pipeline (ChunkedEntangledConv: pinned host in, pinned
host out, three streams) against the CPU oracle: ramped chunk schedules,
host rows at every 4-byte offset from the 256-byte DMA boundary, every
failure index, eager and CUDA-graph replay."""

import numpy as np
import pytest
import torch

import paper_1509_03838_b200 as nent
from paper_1509_03838_b200 import fused
from paper_1509_03838_b200.hostpath import ChunkedEntangledConv

pytestmark = pytest.mark.gpu


def pinned_view(rows, cols, off, dtype=torch.int32):
    """(rows, cols) pinned view whose row starts sit `off` words past alignment
    and whose row stride (cols + 3) drifts the offset row by row."""
    flat = torch.zeros(rows * (cols + 3) + 64, dtype=dtype).pin_memory()
    return flat[off:off + rows * (cols + 3)].view(rows, cols + 3)[:, :cols]


@pytest.mark.parametrize("n,K,chunk,off", [(50000, 256, 1 << 13, 0), (70001, 255, 1 << 14, 1),
                                           (4096, 1, 1024, 3), (300, 64, 1 << 15, 2),
                                           (123457, 97, 1 << 15, 5)])
@pytest.mark.parametrize("w", [48, 64])
def test_chunked_pipeline_matches_oracle(oracle, n, K, chunk, off, w):
    # w = 48: the (3,48,16,16) geometry, whose chunks run on the fused m = 3
    # tcgen05 kernel (non-wrapping windows); w = 64: the generic tcgen05 kernel
    from paper_1509_03838_b200 import _device as D
    p = nent.derive_params(3, w)
    rng = np.random.default_rng(n + K)
    c = rng.integers(-2048, 2048, (3, n), dtype=np.int64)
    g = rng.integers(-2048, 2048, (K,), dtype=np.int64)
    ref = oracle.full_conv(c, g)
    fl = fused.conv_flavor(2048 * ((1 << p.l) + 1), g, n_out=1 << 30)
    c_host = pinned_view(3, n, off)
    c_host.copy_(torch.from_numpy(c).to(torch.int32))
    d_host = pinned_view(3, n + K - 1, (off * 7) % 64)
    assert c_host.is_pinned() and d_host.is_pinned()
    pipe = ChunkedEntangledConv(p, n, g, fl, chunk=chunk)
    for r in (None, 1):
        d_host.fill_(-1)
        pipe.run(c_host, d_host, failed=r)
        pipe.synchronize()
        assert np.array_equal(d_host.to(torch.int64).numpy(), ref), (n, K, chunk, off, r)
    if w == 48 and K >= 64:  # (short filters take a CUDA-core flavour)
        assert D.last_conv_kernel() == "tcgen05_m3"
    pipe.capture(c_host, d_host, failed=2)
    d_host.fill_(-1)
    pipe.replay()
    torch.cuda.synchronize()
    assert np.array_equal(d_host.to(torch.int64).numpy(), ref)


def test_chunked_pipeline_rejects_pageable_and_bad_shapes():
    p = nent.derive_params(3, 64)
    g = np.ones(8, dtype=np.int64)
    fl = fused.conv_flavor(2048 * ((1 << p.l) + 1), g, n_out=1 << 30)
    pipe = ChunkedEntangledConv(p, 1000, g, fl, chunk=1024)
    with pytest.raises(nent.ParameterError):
        pipe.run(torch.zeros((3, 1000), dtype=torch.int32), torch.zeros((3, 1007), dtype=torch.int32))
    with pytest.raises(nent.ParameterError):
        pipe.run(torch.zeros((3, 999), dtype=torch.int32).pin_memory(),
                 torch.zeros((3, 1007), dtype=torch.int32).pin_memory())


@pytest.mark.parametrize("jobs,chunk", [(3, 1 << 13), (4, 1 << 12)])
def test_run_many_streams_independent_jobs(oracle, jobs, chunk):
    """A stream of different batches through one continuous pipeline (the
    buffer ring and the output lag run across job boundaries), eager and as
    one captured graph: every job's output equals its own oracle result."""
    p = nent.derive_params(3, 64)
    n, K = 30001, 200
    rng = np.random.default_rng(jobs)
    g = rng.integers(-2048, 2048, (K,), dtype=np.int64)
    fl = fused.conv_flavor(2048 * ((1 << p.l) + 1), g, n_out=1 << 30)
    cs = [rng.integers(-2048, 2048, (3, n), dtype=np.int64) for _ in range(jobs)]
    refs = [oracle.full_conv(c, g) for c in cs]
    hosts = []
    for j, c in enumerate(cs):
        ch = pinned_view(3, n, j % 4)
        ch.copy_(torch.from_numpy(c).to(torch.int32))
        hosts.append((ch, pinned_view(3, n + K - 1, (5 * j) % 64)))
    pipe = ChunkedEntangledConv(p, n, g, fl, chunk=chunk)
    for _, dh in hosts:
        dh.fill_(-1)
    pipe.run_many(hosts, failed=0)
    pipe.synchronize()
    for (_, dh), ref in zip(hosts, refs):
        assert np.array_equal(dh.to(torch.int64).numpy(), ref)
    # the bench's form: the same buffers, `jobs` steps captured as one graph
    ch, dh = hosts[0]
    pipe.capture(ch, dh, jobs=jobs)
    dh.fill_(-1)
    pipe.replay()
    torch.cuda.synchronize()
    assert np.array_equal(dh.to(torch.int64).numpy(), refs[0])

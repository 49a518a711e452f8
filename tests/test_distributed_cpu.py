"""Multi-process (gloo, CPU) tests of the multi-GPU drivers' exchange logic:
ring shift, position-sharded all-to-all recovery with one rank dropped,
halo exchange and gathers.  Per-rank compute is injected as a CPU stand-in
built on the oracle (the product default is the sm_100a kernels)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleCompute:
    """CPU stand-in for DeviceCompute with identical semantics."""

    def __init__(self):
        from oracle import oracle as O
        self.O = O

    def chain_conv(self, c_prev, c_own, params, g, scale=1, add=None, perm=None, full=True):
        O = self.O
        pair = np.stack([c_prev.numpy(), c_own.numpy()])
        eps = O.entangle(pair, params.l)[1]  # row 1 = (c_prev << l) + c_own
        x = eps * scale
        if add is not None:
            x = x + O.self_entangle("add", add.numpy(), params.l)
        if perm is not None:
            x = x[perm.numpy()]
        y = O.full_conv(x.reshape(1, -1), g) if full else O.circ_conv(x.reshape(1, -1), g)
        return torch.from_numpy(y[0])

    def extract(self, rows, params, r):
        ref = next(t for t in rows if t is not None)
        delta = np.zeros((params.m, ref.shape[-1]), dtype=np.int64)
        for i, t in enumerate(rows):
            if t is not None:
                delta[i] = t.numpy()
        return torch.from_numpy(self.O.disentangle(delta, params.m, params.l, params.w, r))

    def fused_conv(self, x, params, g, period, n_in, y_begin, n_out, failed=None):
        O = self.O
        xv = np.zeros((x.shape[0], period), dtype=np.int64)
        xv[:, :n_in] = x.numpy()[:, :n_in]
        delta = O.circ_conv(O.entangle(xv, params.l), g)[:, y_begin:y_begin + n_out]
        if failed is not None:
            delta[failed] = O.poison_pattern(params.w, delta.shape[1])
        return torch.from_numpy(O.disentangle(delta, params.m, params.l, params.w, failed))


    def fused_inner(self, c, params, g, failed=None):
        O = self.O
        cn = c.numpy()
        m, B, n = cn.shape
        eps = O.entangle(cn.reshape(m, B * n), params.l).reshape(m, B, n)
        delta = (eps * np.asarray(g)[None, None, :]).sum(axis=2)
        if failed is not None:
            delta[failed] = O.poison_pattern(params.w, B)

        class R:
            outputs = None
            mismatches = 0
        r = R()
        r.outputs = torch.from_numpy(O.disentangle(delta, params.m, params.l, params.w, failed))
        return r


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _stream_worker(rank, world, port, cfg, failed_list, q):
    try:
        _init(rank, world, port)
        from paper_1509_03838_b200 import workloads
        from paper_1509_03838_b200.distributed import StreamPerGPU
        wl = workloads.make(cfg, n=700, K=33)
        drv = StreamPerGPU(wl.params, compute=OracleCompute())
        c_own = torch.from_numpy(wl.c[rank].copy())
        kw = {}
        if wl.scale is not None:
            kw = dict(scale=wl.scale, add=torch.from_numpy(wl.add), perm=torch.from_numpy(wl.perm))
        results = {}
        for failed in failed_list:
            out = drv.run(c_own, wl.g, failed=failed, **kw)
            if rank == 0:
                results[failed] = out.numpy()
        if rank == 0:
            from oracle import oracle as O
            x = wl.c if wl.scale is None else (wl.c * wl.scale + wl.add)[:, wl.perm]
            ref = O.full_conv(x, wl.g)
            q.put(all(np.array_equal(v, ref) for v in results.values()) and len(results) == len(failed_list))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        q.put(repr(exc))
        raise


def _subgroup_worker(rank, world, port, q):
    """StreamPerGPU and HaloSplit on a sub-group (global ranks 1..3 of 4):
    peers and gather destinations are group-local ranks."""
    try:
        _init(rank, world, port)
        from paper_1509_03838_b200 import workloads
        from paper_1509_03838_b200.distributed import HaloSplit, StreamPerGPU, shard_bounds
        sub = dist.new_group([1, 2, 3])
        ok = True
        if rank >= 1:
            me = dist.get_rank(sub)
            wl = workloads.make(1, n=500, K=17)
            drv = StreamPerGPU(wl.params, group=sub, compute=OracleCompute())
            c_own = torch.from_numpy(wl.c[me].copy())
            from oracle import oracle as O
            ref = O.full_conv(wl.c, wl.g)
            for failed in (None, 0, 2):
                out = drv.run(c_own, wl.g, failed=failed, dst=1)  # group rank 1 = global rank 2
                if me == 1:
                    ok = ok and np.array_equal(out.numpy(), ref)
                else:
                    ok = ok and out is None
            wl2 = workloads.make(2, n=900, K=40)
            b, e = shard_bounds(wl2.n, 3, me)
            halo = HaloSplit(wl2.params, wl2.K, group=sub, compute=OracleCompute())
            full = halo.gather(halo.run(torch.from_numpy(wl2.c[:, b:e].copy()), wl2.g, failed=1), dst=2)
            if me == 2:
                ok = ok and np.array_equal(full.numpy(), O.full_conv(wl2.c, wl2.g))
        oks = [None] * world
        dist.all_gather_object(oks, bool(ok))
        if rank == 0:
            q.put(all(oks))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        q.put(repr(exc))
        raise


def _halo_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from paper_1509_03838_b200 import workloads
        from paper_1509_03838_b200.distributed import HaloSplit, shard_bounds
        wl = workloads.make(2, n=2000, K=64)
        b, e = shard_bounds(wl.n, world, rank)
        drv = HaloSplit(wl.params, wl.K, compute=OracleCompute())
        ok = True
        for failed in (None, 0, 2):
            d_local = drv.run(torch.from_numpy(wl.c[:, b:e].copy()), wl.g, failed=failed)
            full = drv.gather(d_local)
            if rank == 0:
                from oracle import oracle as O
                ok = ok and np.array_equal(full.numpy(), O.full_conv(wl.c, wl.g))
        if rank == 0:
            q.put(ok)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        q.put(repr(exc))
        raise


def _batch_worker(rank, world, port, q):
    """cfg4's batch split: every rank's vectors are independent, no exchange."""
    try:
        _init(rank, world, port)
        from paper_1509_03838_b200 import workloads
        from paper_1509_03838_b200.distributed import BatchSplit
        wl = workloads.make(4, batch=37, n=129)
        drv = BatchSplit(wl.params, compute=OracleCompute())
        b, e = drv.bounds(wl.c.shape[1])
        ok = True
        want = (wl.c * wl.g[None, None, :]).sum(axis=2)
        for failed in (None, 0, 1, 2):
            res = drv.inner(torch.from_numpy(wl.c[:, b:e].copy()), wl.g, failed=failed)
            d = res.outputs if isinstance(res.outputs, torch.Tensor) else torch.from_numpy(res.outputs.data)
            full = drv.gather(d, wl.c.shape[1])
            if rank == 0:
                ok = ok and np.array_equal(full.numpy(), want)
        if rank == 0:
            q.put(ok)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        q.put(repr(exc))
        raise


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
    return res


@pytest.mark.parametrize("cfg,world", [(1, 3), (3, 4)])
def test_stream_per_gpu_every_failure(cfg, world):
    failed = [None] + list(range(world))
    assert _spawn(_stream_worker, world, cfg, failed) is True


def test_stream_per_gpu_chain_cfg5_shape():
    # cfg5's chain (scale, add, permutation, conv) with M = 8 ranks
    assert _spawn(_stream_worker, 8, 5, [None, 3, 7]) is True


def test_sub_group_peers_are_group_local():
    assert _spawn(_subgroup_worker, 4) is True


@pytest.mark.parametrize("world", [2, 3])
def test_halo_split(world):
    assert _spawn(_halo_worker, world) is True


@pytest.mark.parametrize("world", [2, 3])
def test_batch_split_cfg4(world):
    assert _spawn(_batch_worker, world) is True


def test_shard_bounds_cover():
    from paper_1509_03838_b200.distributed import shard_bounds
    for L in (1, 7, 100, 16777471):
        for parts in (1, 2, 3, 7):
            spans = [shard_bounds(L, parts, i) for i in range(parts)]
            assert spans[0][0] == 0 and spans[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))

"""Multi-GPU drivers: the method's unit of failure mapped onto real devices.

One process per GPU, ``torch.distributed`` (NCCL over NVLink/NVSwitch) for
the plumbing:

* ``StreamPerGPU`` -- M = world size; rank i owns stream c_i and is "worker i"
  of the reference's logical pipeline (pipeline.py:90-117).
    1. ring shift: rank i receives c_{i-1} from rank i-1 (one P2P exchange);
    2. worker: eps_i = (c_{i-1} << l) + c_i, the LSB chain and the
       convolution, fused in one kernel (nent_chain_conv) -> delta_i;
    3. fail-stop: rank r's delta is lost -- it is never sent or read;
    4. recovery, position-sharded: the M-1 survivors each own 1/(M-1) of the
       positions; one all-to-all among survivors (rank r sends and receives
       nothing) gives each survivor the surviving deltas of its slice, and K3
       recovers all M outputs there;
    5. optional gather of the recovered slices.
  ``recover_peer`` is the fused alternative for a single node: every
  surviving rank exports its delta buffer as a CUDA IPC handle (exchanged as
  a few bytes over the process group), and each survivor's K3 launch takes
  the other survivors' rows as peer pointers, so the extract kernel reads its
  1/(M-1) slice of every surviving delta straight out of peer HBM over NVLink
  (no staging copy, no collective on the data path; the failed rank exports
  nothing and nothing of it is read).

* ``HaloSplit`` -- a long signal cut into contiguous slices; rank p needs the
  K-1 samples left of its slice from rank p-1 (one P2P exchange), then runs the
  fused entangle -> conv -> extract kernel on [halo | slice].  Entangle and
  extract are position-local, so nothing else crosses ranks.

* ``BatchSplit`` -- cfg4's batch of independent vectors (inner / outer
  products against a shared vector, ops.py:205-227) cut into contiguous
  vector ranges, one per rank: every vector's entangle -> product -> extract
  is local, so the data path has no exchange at all (weak scaling); only the
  optional gather of the recovered dots crosses ranks.

Compute goes through a ``compute`` object (default ``DeviceCompute``: the
sm_100a kernels); the CPU tests inject a CPU stand-in to exercise the
exchange logic under gloo, and the GPU tests run ``DeviceCompute`` with
several ranks sharing one device (gloo exchanges through host memory).

Peers are given as group-local ranks (``group_peer`` / ``group_dst``), so any
sub-group of the world works, not only WORLD.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import ParameterError
from .params import CodecParams


class DeviceCompute:
    """The per-rank compute steps, each one sm_100a kernel via the C ABI."""

    def __init__(self, flavor: int | None = None):
        self.flavor = flavor

    def chain_conv(self, c_prev, c_own, params: CodecParams, g, scale=1, add=None, perm=None,
                   full=True):
        from . import _device as D
        from .fused import conv_flavor

        from .fused import chain_operands

        n = c_own.shape[-1]
        K = len(g)
        add, perm = chain_operands(add, perm, n)  # LsbOp.validate / Kernel.of_permutation
        flavor = self.flavor
        if flavor is None:
            mc = max(D.max_abs(c_own.reshape(1, -1)), D.max_abs(c_prev.reshape(1, -1)))
            xb = mc * ((1 << params.l) + 1) * abs(int(scale))
            if add is not None:
                xb += D.max_abs(add.reshape(1, -1))
            flavor = conv_flavor(xb, np.asarray(g), n_out=n + K - 1, gather=perm is not None)
        g_dev = D.taps_tensor(np.asarray(g, dtype=np.int64), flavor)
        period = n + K - 1 if full else n
        add_ent = D.shift_add(add, add, params.l) if add is not None else None
        return D.chain_conv(c_prev, c_own, g_dev, K, params.l, flavor, period, n_in=n,
                            scale=scale, add=add_ent, perm=perm)

    def extract(self, rows, params: CodecParams, r: int):
        from . import _device as D

        out, ovf = D.extract(rows, params.m, params.l, r, wide=params.w > 32)
        if ovf:
            raise OverflowError(f"{ovf} recovered values do not fit int64")
        return out

    def fused_conv(self, x, params: CodecParams, g, period, n_in, y_begin, n_out, failed=None):
        from . import _device as D
        from .fused import conv_flavor

        flavor = self.flavor
        if flavor is None:
            mc = D.max_abs(x)
            flavor = conv_flavor(mc * ((1 << params.l) + 1), np.asarray(g), n_out=n_out)
        g_dev = D.taps_tensor(np.asarray(g, dtype=np.int64), flavor)
        return D.fused_conv(x, g_dev, len(g), params.l, flavor, failed, params.w > 32, period,
                            n_in=n_in, y_begin=y_begin, n_out=n_out)


    def fused_inner(self, c, params: CodecParams, g, failed=None):
        from .fused import entangled_inner

        return entangled_inner(params, c, g, failed=failed)

    def fused_outer(self, c, params: CodecParams, g, failed=None, out=None, sums=None):
        from .fused import entangled_outer

        return entangled_outer(params, c, g, failed=failed, out=out, sums=sums)


def _host_exchange(group) -> bool:
    """gloo moves CPU tensors only: device data is staged through host memory."""
    return dist.get_backend(group) == "gloo"


def _to_x(t: torch.Tensor, group) -> torch.Tensor:
    return t.cpu() if (t.is_cuda and _host_exchange(group)) else t


def shard_bounds(L: int, parts: int, idx: int) -> tuple[int, int]:
    """[begin, end) of slice ``idx`` when L positions are cut into ``parts``
    near-equal contiguous slices (the first L % parts get one extra)."""
    base, rem = divmod(L, parts)
    begin = idx * base + min(idx, rem)
    return begin, begin + base + (1 if idx < rem else 0)


@dataclass
class StreamPerGPU:
    params: CodecParams
    group: object = None
    compute: object = None

    def __post_init__(self):
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        if self.world != self.params.m:
            raise ParameterError(f"stream-per-GPU needs world size == m ({self.params.m}), "
                                 f"got {self.world}")
        if self.compute is None:
            self.compute = DeviceCompute()

    # -- 1. ring shift ------------------------------------------------------
    def ring_shift(self, c_own: torch.Tensor) -> torch.Tensor:
        """Return c_{rank-1} (the stream entangled into this rank's word)."""
        m = self.world
        send = _to_x(c_own.contiguous(), self.group)
        prev = torch.empty_like(send)
        ops = [dist.P2POp(dist.isend, send, group=self.group, group_peer=(self.rank + 1) % m),
               dist.P2POp(dist.irecv, prev, group=self.group, group_peer=(self.rank - 1) % m)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        return prev.to(c_own.device)

    # -- 2. worker ------------------------------------------------------------
    def work(self, c_own: torch.Tensor, g, scale: int = 1, add=None, perm=None,
             full: bool = True) -> torch.Tensor:
        c_prev = self.ring_shift(c_own)
        return self.compute.chain_conv(c_prev, c_own, self.params, g, scale=scale, add=add,
                                       perm=perm, full=full)

    # -- 4. position-sharded recovery -----------------------------------------
    def survivors(self, failed: int | None) -> list[int]:
        return [i for i in range(self.world) if i != failed]

    def recover(self, delta_local: torch.Tensor, failed: int | None) -> tuple[torch.Tensor, int, int]:
        """All-to-all of surviving delta slices, then K3 on this rank's slice.

        Returns (d_slice (m, end-begin), begin, end); the failed rank returns
        an empty slice and contributes nothing."""
        m, L = self.world, int(delta_local.shape[-1])
        pivot_failed = failed
        surv = self.survivors(pivot_failed)
        nsurv = len(surv)
        me_alive = self.rank in surv
        my_idx = surv.index(self.rank) if me_alive else -1
        # send splits: survivor i sends slice k of its delta to survivor k
        send_sizes = [0] * m
        recv_sizes = [0] * m
        if me_alive:
            for k, dst in enumerate(surv):
                b, e = shard_bounds(L, nsurv, k)
                send_sizes[dst] = e - b
            mb, me = shard_bounds(L, nsurv, my_idx)
            for src in surv:
                recv_sizes[src] = me - mb
        else:
            mb = me = 0
        send = _to_x(delta_local.contiguous() if me_alive else delta_local.new_empty(0), self.group)
        recv = send.new_empty(sum(recv_sizes))
        dist.all_to_all_single(recv, send.reshape(-1), recv_sizes, send_sizes, group=self.group)
        recv = recv.to(delta_local.device)
        if not me_alive:  # (the recovered slices are int64 on every rank: gather() needs one dtype)
            return torch.empty((m, 0), dtype=torch.int64, device=delta_local.device), 0, 0
        width = me - mb
        rows = [None] * m
        off = 0
        for src in range(m):
            if recv_sizes[src]:
                rows[src] = recv[off:off + width]
                off += width
        r = 0 if failed is None else failed
        if failed is None:
            rows[0] = None  # pivot stream 0, as codec.disentangle does for failed=None
        d = self.compute.extract(rows, self.params, r)
        return d, mb, me

    # -- 5. gather ------------------------------------------------------------
    def gather(self, d_slice: torch.Tensor, L: int, failed: int | None, dst: int = 0):
        """Recovered (m, L) outputs assembled on ``dst`` (None elsewhere)."""
        m = self.world
        surv = self.survivors(failed)
        nsurv = len(surv)
        maxw = -(-L // nsurv)
        buf = d_slice.new_zeros((m, maxw))
        if d_slice.shape[-1]:
            buf[:, : d_slice.shape[-1]] = d_slice
        buf = _to_x(buf, self.group)
        parts = [torch.empty_like(buf) for _ in range(m)] if self.rank == dst else None
        dist.gather(buf, parts, group=self.group, group_dst=dst)
        if self.rank != dst:
            return None
        out = d_slice.new_empty((m, L))
        for k, src in enumerate(surv):
            b, e = shard_bounds(L, nsurv, k)
            out[:, b:e] = parts[src][:, : e - b].to(out.device)
        return out

    # -- 4'. fused peer-read recovery (one node, CUDA IPC over NVLink) ---------
    def recover_peer(self, delta_local: torch.Tensor, failed: int | None):
        """Position-sharded recovery reading the survivors' deltas in place.

        Every survivor exports its (L,) delta through CUDA IPC; the handles
        (a few bytes each) travel over the process group; survivor i opens the
        others' buffers and runs K3 (``nent_extract``) on positions
        [b_i, e_i) with row pointers straight into peer HBM -- the rows of
        ``codec.disentangle`` (codec.py:110-131, _kernels.py:33-67) are
        separate GPUs' memory here and the kernel never touches row ``failed``
        (the failed rank does not even export its buffer).  A barrier keeps
        every exported buffer alive until all reads are done.
        Returns (d_slice (m, e-b), b, e); the failed rank gets an empty slice."""
        rows = PeerRows(self, delta_local, exclude=failed)
        d, mb, me = rows.extract(failed)
        rows.close()
        return d, mb, me

    def run(self, c_own: torch.Tensor, g, failed: int | None = None, scale: int = 1, add=None,
            perm=None, full: bool = True, dst: int | None = 0):
        """The whole fail-stop pipeline; rank ``failed`` computes but its
        result is dropped (it is the worker that died)."""
        delta = self.work(c_own, g, scale, add, perm, full)
        d, b, e = self.recover(delta, failed)
        if dst is None:
            return d, b, e
        return self.gather(d, int(delta.shape[-1]), failed, dst)


class PeerRows:
    """The M ranks' delta buffers mapped into every rank (CUDA IPC), opened
    once for a persistent buffer so repeated recoveries cost one K3 launch.

    ``exclude`` (a failed rank) exports nothing.  ``extract(failed)`` runs K3
    on this rank's 1/(M-1) position slice with the survivors' rows as peer
    pointers; ``close()`` is collective (the owners may then free or rewrite
    their buffers).  Callers order the kernels across ranks: every owner's
    delta must be complete before any rank's extract reads it, and no owner
    rewrites its buffer before every extract of the step is done (bench.py
    uses one tiny NCCL all-reduce on each side; ``recover_peer`` host
    barriers)."""

    def __init__(self, drv: "StreamPerGPU", delta_local: torch.Tensor, exclude: int | None = None):
        from torch.multiprocessing.reductions import reduce_tensor

        from . import _device as D

        if not delta_local.is_cuda:
            raise ParameterError("peer-read recovery needs device-resident deltas")
        self.drv, self.local = drv, delta_local.reshape(-1)
        self.L = int(self.local.numel())
        torch.cuda.current_stream(delta_local.device).synchronize()  # the exported data is complete
        mine = reduce_tensor(self.local) if drv.rank != exclude else None
        shared = [None] * drv.world
        dist.all_gather_object(shared, mine, group=drv.group)
        self.rows = [None] * drv.world
        for j, h in enumerate(shared):
            if h is None:
                continue
            if j == drv.rank:
                self.rows[j] = self.local
                continue
            fn, args = h
            t = fn(*args)  # rank j's buffer, mapped from its GPU (NVLink) or the same device
            if t.device != delta_local.device:
                D.enable_peer_access(t.device.index)
            self.rows[j] = t.reshape(-1)

    def bounds(self, failed: int | None) -> tuple[int, int]:
        surv = self.drv.survivors(failed)
        if self.drv.rank not in surv:
            return 0, 0
        return shard_bounds(self.L, len(surv), surv.index(self.drv.rank))

    def extract(self, failed: int | None, out: torch.Tensor | None = None):
        from . import _device as D

        m = self.drv.world
        mb, me = self.bounds(failed)
        if me == mb:  # the failed rank: an empty slice of the dtype the survivors produce
            return torch.empty((m, 0), dtype=out.dtype if out is not None else torch.int64,
                               device=self.local.device), 0, 0
        r = 0 if failed is None else failed  # failed=None pivots on stream 0 (codec.py:49-51)
        rows = [None if (j == r or t is None) else t[mb:me] for j, t in enumerate(self.rows)]
        if out is None:
            out = torch.empty((m, me - mb), dtype=torch.int64, device=self.local.device)
        d, ovf = D.extract(rows, m, self.drv.params.l, r, wide=self.drv.params.w > 32, out=out,
                           check_overflow=out.dtype == torch.int64)
        if ovf:
            raise OverflowError(f"{ovf} recovered values do not fit int64")
        return d, mb, me

    def close(self):
        torch.cuda.current_stream(self.local.device).synchronize()
        dist.barrier(group=self.drv.group)  # every read of every rank is done
        self.rows = None


@dataclass
class HaloSplit:
    params: CodecParams
    K: int
    group: object = None
    compute: object = None

    def __post_init__(self):
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        if self.compute is None:
            self.compute = DeviceCompute()

    @property
    def halo_width(self) -> int:
        """K-1 rounded up to 4 samples, so the fused kernel's tiles start on
        16-byte boundaries of the [halo | slice] rows."""
        return (self.K - 1 + 3) // 4 * 4

    def exchange_halo(self, c_slice: torch.Tensor) -> torch.Tensor:
        """[halo | slice]: the halo_width samples left of this slice, from
        rank-1 (zeros on rank 0, the signal's left edge)."""
        H = self.halo_width
        m = c_slice.shape[0]
        if H > c_slice.shape[1]:
            raise ValueError(f"slice of {c_slice.shape[1]} samples is shorter than the halo ({H})")
        halo = c_slice.new_zeros((m, H))
        if H and self.world > 1:
            ops = []
            xh = _to_x(halo, self.group)
            if self.rank + 1 < self.world:
                ops.append(dist.P2POp(dist.isend, _to_x(c_slice[:, c_slice.shape[1] - H:].contiguous(), self.group),
                                      group=self.group, group_peer=self.rank + 1))
            if self.rank > 0:
                ops.append(dist.P2POp(dist.irecv, xh, group=self.group, group_peer=self.rank - 1))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            halo = xh.to(c_slice.device)
        return torch.cat([halo, c_slice], dim=1).contiguous()

    def window(self, n: int) -> dict:
        """The fused kernel's window over [halo | slice] for an n-sample slice:
        the full convolution of the zero-extended row (period), the halo_width
        lead-in skipped (y_begin), n outputs (+ the K-1 tail on the last rank)."""
        H, Hp = self.K - 1, self.halo_width
        last = self.rank == self.world - 1
        return {"period": Hp + n + H, "n_in": Hp + n, "y_begin": Hp, "n_out": n + (H if last else 0)}

    def run(self, c_slice: torch.Tensor, g, failed: int | None = None):
        """Recovered full-convolution outputs owned by this rank: positions
        [start, start + n_slice) of the global output (+ the K-1 tail on the
        last rank)."""
        x = self.exchange_halo(c_slice)
        return self.compute.fused_conv(x, self.params, g, failed=failed, **self.window(c_slice.shape[1]))

    def gather(self, d_local: torch.Tensor, dst: int = 0):
        xdev = torch.device("cpu") if _host_exchange(self.group) else d_local.device
        sizes = torch.tensor([d_local.shape[1]], dtype=torch.int64, device=xdev)
        all_sizes = [torch.zeros_like(sizes) for _ in range(self.world)]
        dist.all_gather(all_sizes, sizes, group=self.group)
        maxw = int(max(s.item() for s in all_sizes))
        buf = d_local.new_zeros((d_local.shape[0], maxw))
        buf[:, : d_local.shape[1]] = d_local
        buf = _to_x(buf, self.group)
        parts = [torch.empty_like(buf) for _ in range(self.world)] if self.rank == dst else None
        dist.gather(buf, parts, group=self.group, group_dst=dst)
        if self.rank != dst:
            return None
        return torch.cat([p[:, : int(s.item())] for p, s in zip(parts, all_sizes)], dim=1).to(d_local.device)


@dataclass
class BatchSplit:
    """cfg4: ``batch`` independent vectors per stream, rank p
    owns vectors shard_bounds(batch, world, p) of every stream.  Reference:
    INNER_PRODUCT / ROW_GEMM over a batch (ops.py:205-227); each vector is its
    own entangle -> op -> extract, so ranks never exchange data."""

    params: CodecParams
    group: object = None
    compute: object = None

    def __post_init__(self):
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        if self.compute is None:
            self.compute = DeviceCompute()

    def bounds(self, batch: int) -> tuple[int, int]:
        return shard_bounds(batch, self.world, self.rank)

    def inner(self, c_local: torch.Tensor, g, failed: int | None = None):
        """Recovered dots (m, local batch) of this rank's vectors c_local
        (m, local batch, n) against g; .mismatches is the redundant-stream check."""
        if c_local.dim() != 3 or c_local.shape[0] != self.params.m:
            raise ParameterError("BatchSplit.inner needs c of shape (m, local batch, n)")
        return self.compute.fused_inner(c_local, self.params, g, failed=failed)

    def outer(self, c_local: torch.Tensor, g, failed: int | None = None, out=None, sums=None):
        """Outer products of this rank's vectors with g: written to ``out``
        (m, local batch, n, p) and/or summed per (stream, vector) into ``sums``."""
        return self.compute.fused_outer(c_local, self.params, g, failed=failed, out=out, sums=sums)

    def gather(self, d_local: torch.Tensor, batch: int, dst: int = 0):
        """All ranks' (m, local batch) results concatenated along the batch on ``dst``."""
        m = d_local.shape[0]
        width = -(-batch // self.world)
        buf = d_local.new_zeros((m, width))
        buf[:, : d_local.shape[1]] = d_local
        buf = _to_x(buf, self.group)
        parts = [torch.empty_like(buf) for _ in range(self.world)] if self.rank == dst else None
        dist.gather(buf, parts, group=self.group, group_dst=dst)
        if self.rank != dst:
            return None
        spans = [shard_bounds(batch, self.world, r) for r in range(self.world)]
        return torch.cat([p[:, : e - b] for p, (b, e) in zip(parts, spans)], dim=1).to(d_local.device)

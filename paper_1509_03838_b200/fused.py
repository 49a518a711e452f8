"""Fused single-pass hot path: entangle -> LSB op -> extract in one kernel.

These are the B200 forms of the reference's composed calls
``disentangle(apply_entangled(op, entangle(block)), failed)``
(bench.py:103-106, pipeline.py:97-103) for the op kinds the BASELINE configs
use, producing bit-identical results:

* ``entangled_conv``       full or circular convolution (cfg1, cfg2, cfg3)
* ``entangled_chain_conv`` scale -> add -> permute -> full conv (cfg5)
* ``entangled_inner``      batched inner products (cfg4)
* ``entangled_outer``      outer products, streamed tile by tile (cfg4)
* ``plain_conv``           the non-entangled convolution the overhead is
                           measured against (apply_conventional, ops.py:241-247)

One CTA owns all m streams of an output tile, so entanglement happens while
the tile is staged into shared memory and extraction happens in registers:
the entangled words never touch HBM.  ``failed=r`` recovers from the m-1
other accumulators and never reads stream r's (the tcgen05 kernel does not
convolve stream r at all; the CUDA-core kernels compute it but the recovery
never reads it); ``failed=None`` pivots on stream 0 and, with
``verify=True``, checks the redundant stream against the recovered outputs
(a silent-data-corruption detector the entanglement gives for free).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import MAC_G64, MAC_NAMES, MAC_W64, MAC_X128, is_imma
from .blocks import StreamBlock
from .errors import DeviceError, ParameterError
from .params import CodecParams


@dataclass
class FusedResult:
    outputs: StreamBlock
    flavor: str
    mismatches: int | None = None  # redundant-stream inconsistencies (failed=None, verify)


def _eps_bound(max_c: int, p: CodecParams) -> int:
    return max_c * ((1 << p.l) + 1)


def conv_flavor(max_x: int, g: np.ndarray, allow_imma: bool = True, n_out: int | None = None,
                gather: bool = False) -> int:
    """Fastest exact MAC flavour for |x| <= max_x convolved with taps g."""
    g = np.asarray(g, dtype=np.int64)
    return D.pick_flavor(max_x, int(np.abs(g.astype(object)).sum()), D.host_max_abs(g),
                         K=len(g), allow_imma=allow_imma, n_out=n_out, gather=gather)


def _prep(block: StreamBlock, dtype=None) -> tuple[torch.Tensor, bool]:
    host = not block.on_device
    return D.as_device(block.data, dtype), host


def _finish(p, d: torch.Tensor, host: bool) -> StreamBlock:
    return StreamBlock(p, D.device_to_host(d) if host else d)


def entangled_conv(block: StreamBlock, g, failed: int | None = None, mode: str = "full",
                   verify: bool = True, flavor: int | None = None, out_dtype=torch.int64,
                   max_c: int | None = None, g_dev: torch.Tensor | None = None,
                   out: torch.Tensor | None = None, mismatch: torch.Tensor | None = None
                   ) -> FusedResult:
    """Recovered conv outputs of every stream in one fused kernel.

    mode="full": linear convolution, n + K - 1 outputs (the reference's
    circular convolution of the zero-padded stream);
    mode="circular": the reference's CIRCULAR_CONVOLUTION on n samples."""
    p = block.params
    if not 3 <= p.m <= 8:
        raise ParameterError("the fused kernel holds m in 3..8 streams per tile; "
                             "use entangle/apply_entangled/disentangle for larger m")
    c, host = _prep(block)
    m, n = c.shape
    g = np.asarray(g, dtype=np.int64) if not isinstance(g, torch.Tensor) else g
    K = int(g.shape[0])
    if not 1 <= K <= n and mode == "circular":
        raise ParameterError(f"kernel length {K} not in 1..{n}")
    period = n + K - 1 if mode == "full" else n
    g_np = g if not isinstance(g, torch.Tensor) else g.cpu().numpy()
    mc = None
    if flavor is None or host:
        # the bound of the data as it sits on the device (one reduction kernel;
        # a host pass over 2^24-sample streams would cost more than the upload)
        mc = max_c if max_c is not None else D.max_abs(c)
    if flavor is None:
        flavor = conv_flavor(_eps_bound(mc, p), g_np, n_out=period)
    if flavor in (MAC_G64, MAC_X128):
        raise ParameterError("operands too wide for the fused kernel; use the staged API")
    if g_dev is None:
        g_dev = D.taps_tensor(g_np, flavor)
    if verify and failed is None and mismatch is None:
        mismatch = torch.zeros(1, dtype=torch.int64, device=c.device)
    # Host (numpy int64) blocks: when the entangled words and the admitted output
    # bound (ops.py:163) fit 32 bits, the device works on int32 rows -- the
    # tensor-core kernels' operand width -- and widens the result before it
    # goes back, so the reference-shaped call runs the same kernels as a
    # device-resident int32 block.
    narrow = (host and out is None and out_dtype == torch.int64 and c.dtype == torch.int64
              and _eps_bound(mc, p) < 1 << 31 and mc * int(np.abs(g_np.astype(object)).sum()) < 1 << 31)
    if narrow:
        c = c.to(torch.int32)
    d = D.fused_conv(c, g_dev, K, p.l, flavor, failed, p.w > 32, period, n_in=n,
                     out_dtype=torch.int32 if narrow else out_dtype, out=out,
                     mismatch=mismatch if failed is None else None)
    if narrow:
        d = d.to(torch.int64)
    mm = int(mismatch.item()) if (verify and failed is None) else None
    return FusedResult(_finish(p, d, host), MAC_NAMES[flavor], mm)


def plain_conv(block: StreamBlock, g, mode: str = "full", flavor: int | None = None,
               out_dtype=torch.int64, max_c: int | None = None,
               g_dev: torch.Tensor | None = None, out: torch.Tensor | None = None) -> FusedResult:
    """The failure-intolerant convolution of the plain streams (same kernel family)."""
    p = block.params
    c, host = _prep(block)
    m, n = c.shape
    K = int(len(g))
    period = n + K - 1 if mode == "full" else n
    g = np.asarray(g, dtype=np.int64) if not isinstance(g, torch.Tensor) else g.cpu().numpy()
    if flavor is None:
        mc = max_c if max_c is not None else (D.host_max_abs(block.data) if host else D.max_abs(c))
        flavor = conv_flavor(mc, g, n_out=period)
    if g_dev is None:
        g_dev = D.taps_tensor(g, flavor)
    y, ovf = D.conv(c, g_dev, K, flavor, period=period, n_out=period, out_dtype=out_dtype, out=out)
    if ovf:
        raise OverflowError(f"{ovf} convolution outputs do not fit int64")
    return FusedResult(_finish(p, y, host), MAC_NAMES[flavor])


def chain_operands(add, perm, n: int):
    """The chain's ELEMENTWISE_ADD vector and PERMUTATION index map on the
    device (either may be None), validated as the reference's LsbOp.validate /
    Kernel.of_permutation do (ops.py:57-62, 84-112): the add vector has length
    n or 1 (a length-1 vector is broadcast, ops.py:90), the permutation is a
    bijection of [0, n) (checked by a device kernel) -- the chain kernels
    index add[q] and perm[p] for every position, so anything shorter would
    read out of bounds."""
    add_dev = perm_dev = None
    if add is not None:
        add_dev = D.as_device(np.asarray(add, dtype=np.int64) if not isinstance(add, torch.Tensor) else add)
        add_dev = add_dev.reshape(-1)
        if add_dev.numel() == 1:
            add_dev = add_dev.expand(n).contiguous()
        elif add_dev.numel() != n:
            raise ParameterError(f"kernel length {add_dev.numel()} != stream length {n}")
    if perm is not None:
        perm_dev = D.as_device(np.asarray(perm, dtype=np.int64) if not isinstance(perm, torch.Tensor) else perm)
        if perm_dev.dim() != 1 or perm_dev.numel() != n:
            raise ParameterError(f"permutation length {perm_dev.numel()} != stream length {n}")
        D.perm_check(perm_dev)
    return add_dev, perm_dev


def entangled_chain_conv(block: StreamBlock, scale: int, add, perm, g, failed: int | None = None,
                         verify: bool = True, flavor: int | None = None, out_dtype=torch.int64
                         ) -> FusedResult:
    """cfg5 chain SCALE s -> ELEMENTWISE_ADD a -> PERMUTATION -> full conv.

    The add kernel is self-entangled first (ops.py:250-262).  For m <= 8 the
    chain runs as interleave + one gather pass (each gathered position is one
    contiguous record of all m samples) and the chain output -- the permuted,
    scaled, shifted entangled words -- goes through the fused conv + extract
    kernel (pre_entangled); otherwise the gather happens inside the conv
    kernel's staging."""
    p = block.params
    c, host = _prep(block)
    m, n = c.shape
    add_dev, perm_dev = chain_operands(add, perm, n)
    if add_dev is None or perm_dev is None:
        raise ParameterError("the cfg5 chain needs an add vector and a permutation")
    add_ent = D.shift_add(add_dev, add_dev, p.l)
    g = np.asarray(g, dtype=np.int64)
    K = len(g)
    mc = D.host_max_abs(block.data) if host else D.max_abs(c)
    x_bound = _eps_bound(mc, p) * abs(int(scale)) + D.max_abs(add_ent.reshape(1, -1))
    mismatch = torch.zeros(1, dtype=torch.int64, device=c.device) if (verify and failed is None) else None
    two_pass = m <= 8 and x_bound < 1 << 31
    if flavor is None:
        flavor = conv_flavor(x_bound, g, n_out=n + K - 1, gather=not two_pass)
    g_dev = D.taps_tensor(g, flavor)
    L = n + K - 1
    if two_pass:
        # chain words computed in the coalesced interleave pass, then one random
        # record read per permuted position (int32 indices when they fit)
        perm_idx = perm_dev.to(torch.int32) if n < (1 << 31) else perm_dev
        x = D.gather_records(D.interleave_chain(c.to(torch.int32), p.l, scale, add_ent), perm_idx)
        sum_g = int(np.abs(g.astype(object)).sum())
        d_bound = (mc * abs(int(scale)) + D.max_abs(add_dev.reshape(1, -1))) * sum_g  # ops.py:163
        if (is_imma(flavor) and D.imma_kernel(flavor, K, m, True) == "tcgen05" and m > 3
                and d_bound < 1 << 31):
            # the fused tcgen05 kernels for m > 3 work on int32 rows (the
            # recovered outputs fit them: admitted bound < 2^31): conv + extract
            # in one pass, delta never reaches HBM
            d = D.fused_conv(x, g_dev, K, p.l, flavor, failed, p.w > 32, L, n_in=n,
                             out_dtype=torch.int32, mismatch=mismatch, pre_entangled=True)
            if out_dtype != torch.int32:
                d = d.to(out_dtype)
        elif (is_imma(flavor) and D.imma_kernel(flavor, K, m, True) != "tcgen05"
                and D.imma_kernel(flavor, K, m, False) == "tcgen05"):
            # m > 3: the fused tensor-core kernel would be the mma.sync one; the
            # tcgen05 kernel convolves the m chain rows (the workers' entangled
            # outputs) and a separate pass recovers them (+ the redundant check)
            wide_delta = x_bound * int(np.abs(g.astype(object)).sum()) >= 1 << 31
            delta, _ = D.conv(x, g_dev, K, flavor, period=L, n_out=L,
                              out_dtype=torch.int64 if wide_delta else torch.int32)
            if failed is None:
                d = D.extract_verify(delta, m, p.l, 0, p.w > 32, mismatch if mismatch is not None
                                     else torch.zeros(1, dtype=torch.int64, device=c.device),
                                     out_dtype=out_dtype)
            else:
                d, _ = D.extract(delta, m, p.l, failed, p.w > 32, out_dtype=out_dtype)
        else:
            d = D.fused_conv(x, g_dev, K, p.l, flavor, failed, p.w > 32, L, n_in=n,
                             out_dtype=out_dtype, mismatch=mismatch, pre_entangled=True)
    else:
        d = D.fused_conv(c, g_dev, K, p.l, flavor, failed, p.w > 32, n + K - 1, n_in=n,
                         scale=scale, add=add_ent, perm=perm_dev, out_dtype=out_dtype,
                         mismatch=mismatch)
    mm = int(mismatch.item()) if mismatch is not None else None
    return FusedResult(_finish(p, d, host), MAC_NAMES[flavor], mm)


def entangled_inner(params: CodecParams, c, g, failed: int | None = None, verify: bool = True,
                    out_dtype=torch.int64, max_c: int | None = None) -> FusedResult:
    """cfg4: c (m, batch, n) vectors, g (n,) -> recovered dots (m, batch)."""
    host = not isinstance(c, torch.Tensor)
    cd = D.as_device(c, None) if not host else torch.from_numpy(
        np.ascontiguousarray(c, dtype=np.int64)).to(D.device())
    if cd.dim() != 3 or cd.shape[0] != params.m:
        raise ParameterError("entangled_inner needs c of shape (m, batch, n)")
    g = np.asarray(g, dtype=np.int64)
    # The batched dot is HBM-bound: the generic 64-bit MAC (exact mod 2^64, so
    # exact whenever the admitted dot fits) keeps up with the 3.2 GB stream, so
    # no bound pass over the data is needed to pick a narrower flavour.
    flavor = MAC_G64
    if max_c is not None and _eps_bound(max_c, params) < 1 << 31 and D.host_max_abs(g) < 1 << 31:
        flavor = MAC_W64
    g_dev = D.taps_tensor(g, flavor)
    mismatch = torch.zeros(1, dtype=torch.int64, device=cd.device) if (verify and failed is None) else None
    d = D.fused_inner(cd, g_dev, params.l, failed, params.w > 32, flavor, out_dtype, mismatch)
    mm = int(mismatch.item()) if mismatch is not None else None
    return FusedResult(_finish(params, d, host), MAC_NAMES[flavor], mm)


def entangled_outer(params: CodecParams, c, g, failed: int | None = None,
                    out: torch.Tensor | None = None, sums: torch.Tensor | None = None):
    """cfg4 outer products: d[i, b, u, v] = c[i, b, u] * g[v] through the
    entangled domain.  Writes ``out`` (m, batch, n, p) when given and adds
    per-(stream, vector) sums into ``sums`` (m, batch) when given."""
    cd = c if isinstance(c, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(c, dtype=np.int64)).to(D.device())
    g_dev = D.taps_tensor(np.asarray(g, dtype=np.int64) if not isinstance(g, torch.Tensor) else g.cpu().numpy())
    D.fused_outer(cd, g_dev, params.l, failed, params.w > 32, out, sums)
    return out, sums


_ = DeviceError

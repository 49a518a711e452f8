"""Entangle / disentangle -- drop-in for /root/reference/pkg/src/nent/codec.py.

    entangle:     eps[i] = (c[(i-1) mod m] << l) + c[i]            (codec.py:57-72)
    disentangle:  all m results from the m-1 streams != failed     (codec.py:110-131)

Both run as sm_100a kernels (csrc/codec.cu, csrc/recover.cuh).  Host numpy
blocks are copied to the device and back; device blocks stay resident.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from .blocks import EntangledBlock, StreamBlock
from .counters import OpCounters
from .errors import ParameterError, RangeError
from .params import input_range

_WIDE_W = 32  # above this word width the recovery pivot needs > 64 bits (codec.py:31)


def _check_failed(failed, m: int) -> int:
    """codec.py:49-54: None pivots on stream 0."""
    if failed is None:
        return 0
    if not 0 <= failed < m:
        raise ParameterError(f"failed index {failed} out of range for m={m}")
    return int(failed)


def _wrap(block_like, params, tensor, host: bool, cls):
    return cls(params, tensor.cpu().numpy() if host else tensor)


def _raise_range(first: int, data_host_or_dev, n: int, bound: int):
    s, pos = divmod(int(first), n)
    if isinstance(data_host_or_dev, torch.Tensor):
        value = int(data_host_or_dev[s, pos].item())
    else:
        value = int(data_host_or_dev[s, pos])
    raise RangeError(f"stream {s} position {pos}: value {value} outside +/-{bound}",
                     stream=s, position=pos, value=value, bound=bound)


def entangle(block: StreamBlock, counters: OpCounters | None = None) -> EntangledBlock:
    """Entangled superposition of ``block`` (copying variant)."""
    p = block.params
    host = not block.on_device
    src = D.as_device(block.data, None)
    hi = input_range(p).hi
    eps, first = D.entangle(src, p.l, check_hi=hi, out_dtype=torch.int64)
    if first is not None:
        _raise_range(first, block.data, block.n, hi)
    m, n = src.shape
    if counters is not None:
        counters.encode_ops += m * n
        counters.shift_ops += m * n
    return _wrap(block, p, eps, host, EntangledBlock)


def _store_back(dst: torch.Tensor, src: torch.Tensor, what: str) -> None:
    """Copy ``src`` (int64) into the block's own device buffer.  An int32
    buffer cannot hold words that leave int32 (torch's copy_ would silently
    keep the low 32 bits; the reference's blocks are always int64), so that
    case raises instead."""
    if dst.dtype == torch.int32 and src.numel() and D.max_abs(src.reshape(src.shape[0], -1)) > (1 << 31) - 1:
        raise ParameterError(f"{what} words do not fit the block's int32 buffer; "
                             "use an int64 device block (or the copying variant)")
    dst.copy_(src)


def entangle_inplace(block: StreamBlock, counters: OpCounters | None = None) -> EntangledBlock:
    """Entangle overwriting ``block``'s buffer; the result shares it (codec.py:75-79)."""
    ent = entangle(block, counters)
    if block.on_device:
        _store_back(block.data, ent.data, "entangled")
    else:
        block.data[...] = ent.data
    return EntangledBlock(block.params, block.data)


def disentangle(block: EntangledBlock, failed: int | None = None,
                counters: OpCounters | None = None) -> StreamBlock:
    """Recover all m result streams, never reading stream ``failed``."""
    p = block.params
    r = _check_failed(failed, p.m)
    host = not block.on_device
    m, n = block.data.shape
    if host:
        # the failed row is never read: it is not even copied to the device
        rows = [None if i == r else D.as_device(block.data[i]) for i in range(m)]
    else:
        rows = [None if i == r else block.data[i] for i in range(m)]
    out, ovf = D.extract(rows, m, p.l, r, wide=p.w > _WIDE_W, out_dtype=torch.int64)
    if ovf:
        raise OverflowError(f"{ovf} recovered values do not fit int64 (Python int too large)")
    if counters is not None:
        counters.decode_ops += (2 * m - 3) * n
        counters.shift_ops += (2 * m - 2) * n
    return _wrap(block, p, out, host, StreamBlock)


def disentangle_inplace(block: EntangledBlock, failed: int | None = None,
                        counters: OpCounters | None = None) -> StreamBlock:
    rec = disentangle(block, failed, counters)
    if block.on_device:
        _store_back(block.data, rec.data, "recovered")
    else:
        block.data[...] = rec.data
    return StreamBlock(block.params, block.data)


def disentangle_m3(block: EntangledBlock, failed: int | None = None,
                   counters: OpCounters | None = None) -> StreamBlock:
    """Independent m=3 recovery recipe (codec.py:151-183), a cross-check oracle."""
    p = block.params
    if p.m != 3:
        raise ParameterError(f"m=3 oracle called with m={p.m}")
    r = _check_failed(failed, 3)
    host = not block.on_device
    dev = D.as_device(block.data, torch.int64)
    out = D.extract_m3(dev, p.l, p.w, r)
    if counters is not None:
        counters.decode_ops += 3 * block.n
        counters.shift_ops += 4 * block.n
    return _wrap(block, p, out, host, StreamBlock)


def _disentangle_reference(delta, p, r: int):
    """Name kept for reference-test compatibility (codec.py:89-107): the same
    recovery as ``disentangle`` on a raw (m, n) int64 array."""
    out = disentangle(EntangledBlock(p, np.asarray(delta, dtype=np.int64)), failed=r)
    return out.data

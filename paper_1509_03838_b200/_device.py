"""Device-level primitives over torch CUDA tensors, one per C-ABI entry point.

torch provides device memory, streams and the caching allocator only; every
arithmetic step is one of the sm_100a kernels in csrc/ reached through the C
ABI (``_lib.call``).  All functions are asynchronous on the current stream
except where a status word must be read back (range check, overflow count).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

from . import _lib
from ._lib import (MAC_F64, MAC_G64, MAC_I32, MAC_S64, MAC_W64, MAC_X128, bits, call, imma_flavor,
                   is_imma, ptr, row_ptrs)
from .errors import DeviceError, ParameterError

_I64_MIN = -(1 << 63)
UINT64_MAX_AS_I64 = -1


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the entanglement hot path runs only on B200 (sm_100a); "
                          "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


# ---- large host arrays: pinned staging + threaded host copies ---------------
# The reference API hands numpy int64 arrays in and expects them back.  A
# pageable cudaMemcpy of a 2^24-sample block runs at a few GB/s and the fresh
# result array is page-faulted in by one thread, which together cost far more
# than the kernels.  Blocks of STAGE_MIN bytes and more go through one cached
# pinned buffer per direction instead: the host-side copy into / out of it is
# split over a few threads (numpy releases the GIL for large copies) and the
# DMA runs at PCIe rate.
STAGE_MIN = 8 << 20
STAGE_MAX = 2 << 30
_stage = {}          # direction -> pinned uint8 tensor
_stage_pool = None
_stage_lock = {"in": threading.Lock(), "out": threading.Lock()}  # one user of a staging buffer at a time


def _pool():
    global _stage_pool
    if _stage_pool is None:
        from concurrent.futures import ThreadPoolExecutor
        _stage_pool = ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    return _stage_pool


def _staging(direction: str, nbytes: int) -> torch.Tensor:
    buf = _stage.get(direction)
    if buf is None or buf.numel() < nbytes:
        _stage[direction] = buf = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    return buf[:nbytes]


def _threaded_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[...] = src for two C-contiguous arrays of one dtype, in parallel slabs."""
    d, s = dst.reshape(-1), src.reshape(-1)
    n = d.size
    parts = min(8, max(1, n // (1 << 20)))
    step = -(-n // parts)
    list(_pool().map(lambda i: np.copyto(d[i * step:(i + 1) * step], s[i * step:(i + 1) * step]), range(parts)))


def host_to_device(arr: np.ndarray, dev) -> torch.Tensor:
    """C-contiguous int32/int64 numpy array -> device tensor."""
    if not STAGE_MIN <= arr.nbytes <= STAGE_MAX:
        return torch.from_numpy(arr).to(dev)
    tdt = torch.from_numpy(arr[:0]).dtype
    with _stage_lock["in"]:
        stage = _staging("in", arr.nbytes).view(tdt).reshape(arr.shape)  # pinned
        _threaded_copy(stage.numpy(), arr)
        t = torch.empty(arr.shape, dtype=tdt, device=dev)
        t.copy_(stage, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()  # the staging buffer may be refilled by the next call
    return t


def device_to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> a fresh numpy array (what ``t.cpu().numpy()`` returns)."""
    nbytes = t.numel() * t.element_size()
    if not t.is_cuda or not STAGE_MIN <= nbytes <= STAGE_MAX:
        return t.contiguous().cpu().numpy()  # (row-padded results are compacted first)
    with _stage_lock["out"]:
        stage = _staging("out", nbytes).view(t.dtype).reshape(t.shape)  # pinned
        stage.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        src = stage.numpy()
        out = np.empty(src.shape, dtype=src.dtype)
        _threaded_copy(out, src)
    return out


def as_device(data, dtype=torch.int64) -> torch.Tensor:
    """Host numpy / tensor -> CUDA tensor (2-D rows contiguous)."""
    dev = device()
    if isinstance(data, torch.Tensor):
        t = data.to(device=dev)
        if t.dtype not in (torch.int32, torch.int64):
            t = t.to(torch.int64)
        return t if dtype is None else t.to(dtype)
    arr = np.ascontiguousarray(data, dtype=np.int64)
    t = host_to_device(arr, dev)
    return t if dtype in (None, torch.int64) else t.to(dtype)


def alloc_rows(m: int, n: int, dtype, dev) -> torch.Tensor:
    """(m, n) device tensor whose rows start 128-byte aligned (a padded row pitch): the
    convolution kernels' warps then store whole 128-byte lines on every row.  The C ABI takes
    one pointer per row, so a row pitch is free."""
    q = 128 // torch.empty((), dtype=dtype).element_size()
    return torch.empty((m, -(-n // q) * q), dtype=dtype, device=dev)[:, :n]


def _status() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int64, device=device())


def _sh():
    return _lib.stream_handle()


# ----------------------------------------------------------------- bounds --

def max_abs(t: torch.Tensor) -> int:
    """Exact max |x| over a 2-D device tensor (reads back 8 bytes)."""
    if t.numel() == 0:
        return 0
    out = _status()
    call("nent_max_abs", row_ptrs(t), bits(t), t.shape[0], t.shape[1], ptr(out), _sh())
    return int(out.item()) & ((1 << 64) - 1)


def host_max_abs(a: np.ndarray) -> int:
    """Exact max |x| of a host int64 array (object path only for INT64_MIN)."""
    if a.size == 0:
        return 0
    lo, hi = int(a.min()), int(a.max())
    return max(abs(lo), abs(hi))


def signed_digits(maxabs: int) -> int:
    """Balanced base-256 int8 digits needed for every |v| <= maxabs."""
    p = 1
    while 127 * (256 ** p - 1) // 255 < maxabs:
        p += 1
    return p


# measured on B200 (bench.py microbenchmarks, MAC/s): the pipe peaks that
# decide which exact flavour is fastest for given operand widths
PIPE_PEAK = {MAC_I32: 16.9e12, MAC_F64: 13.0e12, MAC_W64: 8.2e12, MAC_S64: 5.35e12,
             MAC_G64: 3.4e12, "imma": 559e12}
IMMA_EFFICIENCY = 0.5  # fraction of the mma.sync peak the digit-sliced kernel reaches


def cuda_core_flavor(max_x: int, sum_g: int, max_g: int) -> int:
    """Narrowest CUDA-core MAC flavour exact for |x| <= max_x and the taps.

    bound = max_x * max(sum_g, 1) bounds every partial sum (ops.py:163)."""
    bound = max_x * max(sum_g, 1)
    if bound >= 1 << 62:
        return MAC_X128
    if bound < 1 << 31:
        return MAC_I32
    if bound < 1 << 53 and max_x < 1 << 53 and max_g < 1 << 53:
        return MAC_F64
    if max_x < 1 << 31 and max_g < 1 << 31:
        return MAC_W64
    if max_g < 1 << 31:
        return MAC_S64
    return MAC_G64


def pick_flavor(max_x: int, sum_g: int, max_g: int, K: int | None = None,
                allow_imma: bool = True, n_out: int | None = None, gather: bool = False) -> int:
    """Fastest exact flavour.  Every candidate is exact for these bounds; the
    IMMA digit-sliced tensor-core conv is chosen when its modelled rate
    (mma.sync peak x efficiency x K/KD / (np*ng)) beats the CUDA-core pipe.
    Small problems (fewer 1024-output tiles than ~2 waves) and gathered
    (permuted) inputs stay on the CUDA-core kernel, whose staging is cheaper."""
    core = cuda_core_flavor(max_x, sum_g, max_g)
    if not allow_imma or K is None or core == MAC_X128 or K + 15 >= 1 << 16 or gather:
        return core
    if n_out is not None and n_out < 2 * 148 * 1024:
        return core
    np_, ng = signed_digits(max_x), signed_digits(max_g)
    if np_ > 8 or ng > 4:
        return core
    KD = (K + 15 + 31) // 32 * 32
    imma_rate = PIPE_PEAK["imma"] * IMMA_EFFICIENCY * K / KD / (np_ * ng)
    return imma_flavor(np_, ng) if imma_rate > PIPE_PEAK[core] else core


def taps_tensor(g, flavor: int | None = None) -> torch.Tensor:
    """Filter taps on the device: int32 when every tap fits, else int64."""
    arr = np.asarray(g, dtype=np.int64)
    fits32 = arr.size == 0 or (int(arr.min()) >= -(1 << 31) and int(arr.max()) < (1 << 31))
    dtype = torch.int32 if fits32 and flavor not in (MAC_G64, MAC_X128) else torch.int64
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device=device(), dtype=dtype)


# ------------------------------------------------------------------- codec --

def entangle(c: torch.Tensor, l: int, check_hi: int | None = None, out_dtype=torch.int64,
             out: torch.Tensor | None = None):
    """K1: returns (eps, first_bad_linear_index or None)."""
    m, n = c.shape
    eps = torch.empty((m, n), dtype=out_dtype, device=c.device) if out is None else out
    bad = _status() if check_hi is not None else None
    call("nent_entangle", row_ptrs(c), bits(c), row_ptrs(eps), bits(eps), m, n, l,
         -1 if check_hi is None else int(check_hi), ptr(bad), _sh())
    first = None
    if bad is not None:
        v = int(bad.item())
        if v != UINT64_MAX_AS_I64:
            first = v
    return eps, first


def shift_add(a: torch.Tensor, b: torch.Tensor, l: int, out_dtype=torch.int64) -> torch.Tensor:
    if a.dtype != b.dtype:
        b = b.to(a.dtype)
    out = torch.empty(a.shape, dtype=out_dtype, device=a.device)
    call("nent_shift_add", ptr(a), ptr(b), bits(a), ptr(out), bits(out), a.numel(), l, _sh())
    return out


def extract(delta, m: int, l: int, r: int, wide: bool, out_dtype=torch.int64,
            out: torch.Tensor | None = None, check_overflow: bool = True):
    """K3: recover all m rows from the rows != r (row r is never read).

    ``delta`` is an (m, n) tensor or a list of m row tensors (entry r may be
    None or a peer buffer).  Returns (out, overflow_count)."""
    rows = list(delta) if not isinstance(delta, torch.Tensor) else [delta[i] for i in range(m)]
    ref = next(t for i, t in enumerate(rows) if i != r and t is not None)
    n = ref.shape[-1]
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=ref.device)
    ovf = _status() if (wide and check_overflow) else None
    rows = [None if i == r else t for i, t in enumerate(rows)]
    call("nent_extract", row_ptrs(rows), bits(ref), row_ptrs(out), bits(out), m, n, l, r,
         int(bool(wide)), ptr(ovf), _sh())
    return out, (int(ovf.item()) if ovf is not None else 0)


def extract_verify(delta: torch.Tensor, m: int, l: int, pivot: int, wide: bool, mismatch: torch.Tensor,
                   out_dtype=torch.int64, out: torch.Tensor | None = None):
    """K3 from the rows != pivot plus the redundant-stream check of row
    `pivot`; mismatches are added to the device counter ``mismatch``."""
    rows = [delta[i] for i in range(m)]
    n = rows[0].shape[-1]
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=delta.device)
    call("nent_extract_verify", row_ptrs(rows), bits(delta), row_ptrs(out), bits(out), m, n, l, pivot,
         int(bool(wide)), None, ptr(mismatch), _sh())
    return out


def extract_m3(delta: torch.Tensor, l: int, w: int, r: int, out_dtype=torch.int64):
    rows = [None if i == r else delta[i] for i in range(3)]
    out = torch.empty(delta.shape, dtype=out_dtype, device=delta.device)
    call("nent_extract_m3", row_ptrs(rows), bits(delta), row_ptrs(out), bits(out), delta.shape[1],
         l, w, r, _sh())
    return out


def poison(row: torch.Tensor, w: int) -> None:
    call("nent_poison", ptr(row), bits(row), row.numel(), w, _sh())


# --------------------------------------------------------------------- ops --

def imma_table(g_dev: torch.Tensor, K: int, flavor: int, y_begin: int = 0) -> torch.Tensor | None:
    """Prepared digit-split Toeplitz taps for an IMMA flavour (None otherwise):
    build once, pass as ``imma_table=`` to every launch with the same taps."""
    if not is_imma(flavor):
        return None
    nbytes = int(_lib.lib().nent_imma_table_bytes(K, flavor))
    tab = torch.empty(nbytes, dtype=torch.uint8, device=g_dev.device)
    call("nent_imma_table", ptr(g_dev), bits(g_dev), K, y_begin, flavor, ptr(tab), _sh())
    return tab


def conv(x: torch.Tensor, g_dev: torch.Tensor, K: int, flavor: int, period: int | None = None,
         y_begin: int = 0, n_out: int | None = None, out_dtype=torch.int64,
         out: torch.Tensor | None = None, imma_table: torch.Tensor | None = None):
    """K2 on every row: circular conv over `period` (default n) with zero-extension.
    Returns (y, overflow_count) -- overflow only counted for MAC_X128."""
    rows, n_in = x.shape
    period = n_in if period is None else period
    n_out = period if n_out is None else n_out
    if out is None:
        out = alloc_rows(rows, n_out, out_dtype, x.device)
    ovf = _status() if flavor == MAC_X128 else None
    if x.dtype == torch.int32 and flavor in (MAC_G64, MAC_X128):
        x = x.to(torch.int64)
    call("nent_conv", row_ptrs(x), bits(x), rows, n_in, period, ptr(g_dev), bits(g_dev), K,
         row_ptrs(out), bits(out), y_begin, n_out, flavor, ptr(ovf), ptr(imma_table), _sh())
    return out, (int(ovf.item()) if ovf is not None else 0)


def fused_conv(c, g_dev: torch.Tensor, K: int, l: int, flavor: int, r: int | None,
               wide: bool, period: int, n_in: int | None = None, y_begin: int = 0,
               n_out: int | None = None, scale: int = 1, add: torch.Tensor | None = None,
               perm: torch.Tensor | None = None, out_dtype=torch.int64,
               out: torch.Tensor | None = None, mismatch: torch.Tensor | None = None,
               pre_entangled: bool = False, imma_table: torch.Tensor | None = None):
    """K2f: entangle-on-load -> [scale, add, gather] -> conv -> extract.
    ``c`` is an (m, n) tensor or list of m row tensors; ``r=None`` = no failure
    (pivot 0, redundant-stream check into ``mismatch`` if given).  ``wide``
    (w > 32) is accepted for symmetry with ``extract``: the fused recovery is
    exact for any w <= 64 on the consistent words it produces."""
    rows = list(c) if not isinstance(c, torch.Tensor) else [c[i] for i in range(c.shape[0])]
    m = len(rows)
    n_in = rows[0].shape[-1] if n_in is None else n_in
    n_out = period if n_out is None else n_out
    if out is None:
        out = alloc_rows(m, n_out, out_dtype, rows[0].device)
    call("nent_fused_conv", row_ptrs(rows), bits(rows[0]), m, n_in, period, l, int(scale),
         ptr(add), bits(add) if add is not None else 64, ptr(perm), ptr(g_dev), bits(g_dev), K,
         -1 if r is None else int(r), int(bool(pre_entangled)), row_ptrs(out), bits(out), y_begin,
         n_out, flavor, ptr(mismatch), ptr(imma_table), _sh())
    return out


def chain_conv(a: torch.Tensor | None, b: torch.Tensor, g_dev: torch.Tensor, K: int, l: int,
               flavor: int, period: int, n_in: int | None = None, y_begin: int = 0,
               n_out: int | None = None, scale: int = 1, add: torch.Tensor | None = None,
               perm: torch.Tensor | None = None, out_dtype=torch.int64,
               out: torch.Tensor | None = None, imma_table: torch.Tensor | None = None) -> torch.Tensor:
    n_in = b.shape[-1] if n_in is None else n_in
    n_out = period if n_out is None else n_out
    if out is None:
        out = torch.empty((n_out,), dtype=out_dtype, device=b.device)
    call("nent_chain_conv", ptr(a), ptr(b), bits(b), n_in, period, l, int(scale), ptr(add),
         bits(add) if add is not None else 64, ptr(perm), ptr(g_dev), bits(g_dev), K, ptr(out),
         bits(out), y_begin, n_out, flavor, ptr(imma_table), _sh())
    return out


def imma_kernel(flavor: int, K: int, rows: int, extract: bool) -> str:
    """Which tensor-core kernel an IMMA flavour runs for this shape."""
    return {0: "cuda-core", 1: "mma.sync", 2: "tcgen05"}[
        _lib.lib().nent_imma_kernel(int(flavor), int(K), int(rows), int(bool(extract)))]


def last_conv_kernel() -> str:
    """The convolution kernel this host thread launched last."""
    return {0: "none", 1: "cuda-core", 2: "mma.sync", 3: "tcgen05", 4: "tcgen05_m3", 5: "tcgen05_m4", 6: "tcgen05_m8"}[
        _lib.lib().nent_last_conv_kernel()]


def copy_rows(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[:] = src for two (rows, width) views with contiguous rows and any
    row pitch, one on the device and one in pinned host memory (or both on
    the device), as one 2-D DMA on the current stream (nent_copy_rows)."""
    if dst.shape != src.shape or dst.dim() != 2 or dst.dtype != src.dtype:
        raise ParameterError("copy_rows needs two 2-D views of one shape and dtype")
    if (dst.shape[1] > 1 and (dst.stride(1) != 1 or src.stride(1) != 1)):
        raise ParameterError("copy_rows needs contiguous rows")
    if dst.is_cuda and src.is_cuda:
        direction = 3
    elif dst.is_cuda:
        direction = 1
    elif src.is_cuda:
        direction = 2
    else:
        raise ParameterError("copy_rows: one side must be on the device")
    es = dst.element_size()
    call("nent_copy_rows", dst.data_ptr(), dst.stride(0) * es, src.data_ptr(), src.stride(0) * es,
         dst.shape[1] * es, dst.shape[0], direction, _sh())


def interleave(x: torch.Tensor) -> torch.Tensor:
    """(m, n) rows -> (n, m) position-major copy (m <= 8)."""
    m, n = x.shape
    out = torch.empty((n, m), dtype=x.dtype, device=x.device)
    call("nent_interleave", row_ptrs(x), bits(x), m, n, ptr(out), _sh())
    return out


def gather_chain(ct: torch.Tensor, l: int, scale: int = 1, add: torch.Tensor | None = None,
                 perm: torch.Tensor | None = None, out_dtype=torch.int32,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """Entangle -> scale -> add -> permute from the interleaved (n, m) streams;
    returns the (m, n) chain output (entangled words, stream-major)."""
    n, m = ct.shape
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=ct.device)
    call("nent_gather_chain", ptr(ct), bits(ct), m, n, l, int(scale), ptr(add),
         bits(add) if add is not None else 64, ptr(perm), row_ptrs(out), bits(out), _sh())
    return out


def interleave_chain(x: torch.Tensor, l: int, scale: int = 1, add: torch.Tensor | None = None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """(m, n) rows -> (n, m) records of the chain words before the permutation:
    rec[p, s] = scale * ((x[s-1, p] << l) + x[s, p]) + add[p] (dtype of x; the
    caller's bound must fit it)."""
    m, n = x.shape
    if out is None:
        out = torch.empty((n, m), dtype=x.dtype, device=x.device)
    call("nent_interleave_chain", row_ptrs(x), bits(x), m, n, l, int(scale), ptr(add),
         bits(add) if add is not None else 64, ptr(out), bits(out), _sh())
    return out


def gather_records(rec: torch.Tensor, perm: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """x[s, p] = rec[perm[p], s]: the permutation of the chain records
    (perm int32 or int64)."""
    n, m = rec.shape
    if out is None:
        out = torch.empty((m, n), dtype=rec.dtype, device=rec.device)
    call("nent_gather_records", ptr(rec), bits(rec), m, n, ptr(perm), bits(perm), row_ptrs(out), _sh())
    return out


def enable_peer_access(peer: int) -> None:
    """Kernels on the current device may then read device ``peer``'s memory."""
    call("nent_enable_peer_access", int(peer))


def perm_check(perm: torch.Tensor) -> None:
    """Kernel.of_permutation's bijection test (ops.py:57-62) on the device;
    raises ParameterError unless ``perm`` is a permutation of [0, len)."""
    if perm.dim() != 1:
        raise ParameterError("permutation kernel is not a bijection")
    n = perm.numel()
    if n == 0:
        return
    if perm.dtype not in (torch.int32, torch.int64):
        perm = perm.to(torch.int64)
    bitmap = torch.zeros(((n + 31) // 32,), dtype=torch.int32, device=perm.device)
    bad = _status()
    call("nent_perm_check", ptr(perm), bits(perm), n, ptr(bitmap), ptr(bad), _sh())
    if int(bad.item()):
        raise ParameterError("permutation kernel is not a bijection")


def elementwise(x: torch.Tensor, g: torch.Tensor, op: int, check: bool, out_dtype=torch.int64):
    rows, n = x.shape
    out = torch.empty((rows, n), dtype=out_dtype, device=x.device)
    ovf = _status() if check else None
    call("nent_elementwise", row_ptrs(x), bits(x), rows, n, ptr(g), bits(g), g.numel(), op,
         row_ptrs(out), bits(out), int(check), ptr(ovf), _sh())
    return out, (int(ovf.item()) if ovf is not None else 0)


def scale(x: torch.Tensor, s: int, check: bool, out_dtype=torch.int64):
    rows, n = x.shape
    out = torch.empty((rows, n), dtype=out_dtype, device=x.device)
    ovf = _status() if check else None
    call("nent_scale", row_ptrs(x), bits(x), rows, n, int(s), row_ptrs(out), bits(out),
         int(check), ptr(ovf), _sh())
    return out, (int(ovf.item()) if ovf is not None else 0)


def permute(x: torch.Tensor, perm: torch.Tensor, out_dtype=torch.int64) -> torch.Tensor:
    rows, n = x.shape
    out = torch.empty((rows, n), dtype=out_dtype, device=x.device)
    call("nent_permute", row_ptrs(x), bits(x), rows, n, ptr(perm), row_ptrs(out), bits(out), _sh())
    return out


def reverse_circular(x: torch.Tensor) -> torch.Tensor:
    rows, n = x.shape
    out = torch.empty_like(x)
    call("nent_reverse_circular", row_ptrs(x), bits(x), rows, n, row_ptrs(out), bits(out), _sh())
    return out


def inner(x: torch.Tensor, g_dev: torch.Tensor, batch: int, n: int, flavor: int, check: bool):
    """Rows of `batch` vectors of length n -> (rows, batch) int64 dots."""
    rows = x.shape[0]
    out = torch.empty((rows, batch), dtype=torch.int64, device=x.device)
    ovf = _status() if check else None
    call("nent_inner", row_ptrs(x.reshape(rows, -1)), bits(x), rows, batch, n, ptr(g_dev),
         bits(g_dev), row_ptrs(out), flavor, int(check), ptr(ovf), _sh())
    return out, (int(ovf.item()) if ovf is not None else 0)


def fused_inner(c: torch.Tensor, g_dev: torch.Tensor, l: int, r: int | None, wide: bool,
                flavor: int, out_dtype=torch.int64, mismatch: torch.Tensor | None = None):
    """c: (m, batch, n) -> d: (m, batch) recovered dots."""
    m, batch, n = c.shape
    out = torch.empty((m, batch), dtype=out_dtype, device=c.device)
    call("nent_fused_inner", row_ptrs(c.reshape(m, -1)), bits(c), m, batch, n, l, ptr(g_dev),
         bits(g_dev), -1 if r is None else int(r), int(bool(wide)), row_ptrs(out), bits(out),
         flavor, ptr(mismatch), _sh())
    return out


def fused_outer(c: torch.Tensor, g_dev: torch.Tensor, l: int, r: int | None, wide: bool,
                out: torch.Tensor | None, sums: torch.Tensor | None):
    """c: (m, batch, n) -> out (m, batch, n, p) (optional) and sums (m, batch) added."""
    m, batch, n = c.shape
    p = g_dev.numel()
    d_rows = row_ptrs(out.reshape(m, -1)) if out is not None else None
    call("nent_fused_outer", row_ptrs(c.reshape(m, -1)), bits(c), m, batch, n, l, ptr(g_dev),
         bits(g_dev), p, -1 if r is None else int(r), int(bool(wide)),
         d_rows if d_rows is not None else ctypes.cast(None, ctypes.POINTER(ctypes.c_void_p)),
         bits(out) if out is not None else 64, ptr(sums), _sh())


def gemm(x: torch.Tensor, G: torch.Tensor, check: bool):
    rows, n = x.shape
    p = G.shape[1]
    out = torch.empty((rows, p), dtype=torch.int64, device=x.device)
    ovf = _status() if check else None
    call("nent_gemm", row_ptrs(x), bits(x), rows, n, ptr(G), p, row_ptrs(out), 64, int(check),
         ptr(ovf), _sh())
    return out, (int(ovf.item()) if ovf is not None else 0)


def first_out_of_range(x: torch.Tensor, hi: int):
    """Linear index of the first |x| > hi (row-major) or None."""
    bad = _status()
    call("nent_check_range", row_ptrs(x), bits(x), x.shape[0], x.shape[1], int(hi), ptr(bad), _sh())
    v = int(bad.item())
    return None if v == UINT64_MAX_AS_I64 else v


def checksum_encode(x: torch.Tensor) -> torch.Tensor:
    m, n = x.shape
    cs = torch.empty((n,), dtype=torch.int64, device=x.device)
    call("nent_checksum_encode", row_ptrs(x), bits(x), m, n, ptr(cs), 64, _sh())
    return cs


def checksum_recover(x: torch.Tensor, cs: torch.Tensor, failed: int) -> torch.Tensor:
    m, n = x.shape
    out = torch.empty((n,), dtype=torch.int64, device=x.device)
    rows = [None if i == failed else x[i] for i in range(m)]
    call("nent_checksum_recover", row_ptrs(rows), bits(x), ptr(cs), bits(cs), m, n, failed,
         ptr(out), 64, _sh())
    return out


def microbench(kind: int, blocks: int, threads: int, iters: int,
               stream: torch.cuda.Stream | None = None) -> float:
    """Launch the pipe microbenchmark; returns the MAC count it issues."""
    sink = torch.zeros(1024, dtype=torch.int64, device=device())
    macs = ctypes.c_double(0.0)
    call("nent_microbench", kind, blocks, threads, iters, ptr(sink), ctypes.byref(macs),
         _lib.stream_handle(stream))
    return macs.value


__all__ = [n for n in dir() if not n.startswith("__")]
_ = (MAC_F64, MAC_I32, MAC_S64, MAC_W64, ParameterError)

"""CPU oracle for the numerical-entanglement hot path -- TEST INFRASTRUCTURE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or
as the timed CPU baseline.  The product package never imports it.

The arithmetic lives in ``nent_oracle.c`` (a plain-C restatement of the
reference, each function citing /root/reference file:line); this module is the
numpy-level glue that mirrors the reference's block-level semantics:

* ``entangle``          -- pkg/src/nent/codec.py:57-72 (+ range check :34-46)
* ``disentangle``       -- pkg/src/nent/codec.py:110-131 (r=None -> 0, :49-54)
* ``disentangle_m3``    -- pkg/src/nent/codec.py:151-183
* ``apply_raw``         -- pkg/src/nent/ops.py:184-232 (all nine op kinds)
* ``self_entangle``     -- pkg/src/nent/ops.py:250-262
* ``poison_pattern``    -- pkg/src/nent/pipeline.py:65-70
* ``run_entangled``     -- pkg/src/nent/pipeline.py:97-103

Parity of this oracle against the reference is pinned by
tests/test_oracle.py using the reference's own golden vectors and the
fixtures in tests/golden/ (generated from the reference by
tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libnent_oracle.so"
_INT64_SAFE = 1 << 62  # pkg/src/nent/ops.py:25

_lib = None


def build(force: bool = False) -> Path:
    """Compile nent_oracle.c with the committed Makefile (gcc, OpenMP)."""
    src = _HERE / "nent_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int, ctypes.c_int64
        L.oracle_max_threads.restype = i32
        L.oracle_entangle.argtypes = [P, P, i32, i64, i32, i32]
        L.oracle_first_out_of_range.argtypes = [P, i64, i64]
        L.oracle_first_out_of_range.restype = i64
        L.oracle_disentangle.argtypes = [P, P, i32, i64, i32, i32, i32, i32]
        L.oracle_disentangle.restype = i64
        L.oracle_disentangle_m3.argtypes = [P, P, i64, i32, i32, i32]
        L.oracle_circ_conv.argtypes = [P, i32, i64, P, i32, P, i32, i32]
        L.oracle_circ_conv.restype = i64
        L.oracle_reverse_circular.argtypes = [P, i32, i64, P]
        L.oracle_elementwise.argtypes = [P, i32, i64, P, i64, i32, P, i32]
        L.oracle_elementwise.restype = i64
        L.oracle_permute.argtypes = [P, i32, i64, P, P]
        L.oracle_inner.argtypes = [P, i32, i64, P, P, i32]
        L.oracle_inner.restype = i64
        L.oracle_gemm.argtypes = [P, i32, i64, P, i64, P, i32]
        L.oracle_gemm.restype = i64
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _nt(threads: int, work: int) -> int:
    """OpenMP team size: one thread for small problems (fork/join would dominate)."""
    if threads:
        return threads
    return 1 if work < (1 << 18) else 0


class OracleOverflow(OverflowError):
    """The exact result does not fit int64 (the reference's object path raises)."""


# ---------------------------------------------------------------- geometry --

def output_range_hi(m: int, l: int, k: int) -> int:
    """pkg/src/nent/params.py:74-84."""
    return max((1 << ((m - 3) * l)) * ((1 << (l + k - 1)) - (1 << l)), 0)


def derive_lk(m: int, w: int) -> tuple[int, int]:
    """pkg/src/nent/params.py:52-71: maximise (m-2)l+k, smallest l on ties."""
    best = None
    for l in range(1, w + 1):
        k = min(l, w - (m - 1) * l)
        if k < 1:
            break
        bits = (m - 2) * l + k
        if best is None or bits > best[0]:
            best = (bits, l, k)
    if best is None:
        raise ValueError(f"no feasible (l, k) for m={m}, w={w}")
    return best[1], best[2]


# ------------------------------------------------------------------- codec --

def first_out_of_range(data, hi: int):
    """(stream, position, value) of the first |x| > hi in row-major order, or None."""
    d = _c64(data)
    idx = int(lib().oracle_first_out_of_range(_p(d), d.size, int(hi)))
    if idx < 0:
        return None
    s, pos = divmod(idx, d.shape[1])
    return s, pos, int(d[s, pos])


def entangle(data, l: int, threads: int = 0) -> np.ndarray:
    d = _c64(data)
    m, n = d.shape
    out = np.empty_like(d)
    lib().oracle_entangle(_p(d), _p(out), m, n, l, _nt(threads, d.size))
    return out


def disentangle(delta, m: int, l: int, w: int, r: int | None = None, threads: int = 0) -> np.ndarray:
    d = _c64(delta)
    rr = 0 if r is None else int(r)
    out = np.empty_like(d)
    ovf = lib().oracle_disentangle(_p(d), _p(out), m, d.shape[1], l, rr, int(w > 32),
                                   _nt(threads, d.size))
    if ovf:
        raise OracleOverflow(f"{ovf} recovered values do not fit int64")
    return out


def disentangle_m3(delta, l: int, w: int, r: int | None = None) -> np.ndarray:
    d = _c64(delta)
    out = np.empty_like(d)
    lib().oracle_disentangle_m3(_p(d), _p(out), d.shape[1], l, w, 0 if r is None else int(r))
    return out


# --------------------------------------------------------------------- ops --

def _max_abs(a: np.ndarray) -> int:
    """Exact max |x| (Python ints, so |INT64_MIN| = 2^63 as in the reference)."""
    a = np.asarray(a)
    return max(abs(int(a.min())), abs(int(a.max()))) if a.size else 0


def circ_conv(x, g, threads: int = 0, wide: bool | None = None) -> np.ndarray:
    x, g = _c64(x), _c64(g)
    if x.ndim == 1:
        x = x.reshape(1, -1)
    rows, n = x.shape
    if wide is None:
        wide = _max_abs(x) * max(sum(abs(int(v)) for v in g), 1) >= _INT64_SAFE
    y = np.empty_like(x)
    ovf = lib().oracle_circ_conv(_p(x), rows, n, _p(g), len(g), _p(y), int(bool(wide)),
                                 _nt(threads, x.size * len(g)))
    if ovf:
        raise OracleOverflow(f"{ovf} convolution outputs do not fit int64")
    return y


def full_conv(x, g, threads: int = 0) -> np.ndarray:
    """Linear convolution = circular convolution of the zero-padded stream."""
    x = _c64(x)
    K = len(g)
    xp = np.zeros((x.shape[0], x.shape[1] + K - 1), dtype=np.int64)
    xp[:, : x.shape[1]] = x
    return circ_conv(xp, g, threads)


def reverse_circular(x) -> np.ndarray:
    x = _c64(x)
    out = np.empty_like(x)
    lib().oracle_reverse_circular(_p(x), x.shape[0], x.shape[1], _p(out))
    return out


def apply_raw(kind: str, data, *, vector=None, scalar=None, perm=None, matrix=None, threads: int = 0):
    """Row-wise LSB op on an int64 (m, n) array; kind is the OpKind value string."""
    x = _c64(data)
    m, n = x.shape
    L = lib()
    if kind in ("add", "sub", "mul", "scale"):
        if kind == "scale":
            g = np.asarray([scalar], dtype=np.int64)
            code = 2
        else:
            g = _c64(vector)
            code = {"add": 0, "sub": 1, "mul": 2}[kind]
        wide = code == 2 and _max_abs(x) * max(_max_abs(g), 1) >= _INT64_SAFE
        y = np.empty_like(x)
        ovf = L.oracle_elementwise(_p(x), m, n, _p(g), len(g), code, _p(y), int(wide))
        if ovf:
            raise OracleOverflow(f"{ovf} products do not fit int64")
        return y
    if kind == "dot":
        g = _c64(vector)
        wide = _max_abs(x) * max(sum(abs(int(v)) for v in g), 1) >= _INT64_SAFE
        y = np.empty((m, 1), dtype=np.int64)
        if L.oracle_inner(_p(x), m, n, _p(g), _p(y), int(wide)):
            raise OracleOverflow("inner product does not fit int64")
        return y
    if kind == "conv":
        return circ_conv(x, vector, threads)
    if kind == "xcorr":
        return circ_conv(reverse_circular(x), vector, threads)
    if kind == "perm":
        p = _c64(perm)
        y = np.empty_like(x)
        L.oracle_permute(_p(x), m, n, _p(p), _p(y))
        return y
    if kind == "gemm":
        G = _c64(matrix)
        wide = _max_abs(x) * int(np.abs(G.astype(object)).sum(axis=0).max()) >= _INT64_SAFE
        y = np.empty((m, G.shape[1]), dtype=np.int64)
        if L.oracle_gemm(_p(x), m, n, _p(G), G.shape[1], _p(y), int(wide)):
            raise OracleOverflow("gemm output does not fit int64")
        return y
    raise ValueError(f"unknown op kind {kind!r}")


def self_entangle(kind: str, vector, l: int):
    """g <- (g << l) + g for add/sub only (pkg/src/nent/ops.py:250-262)."""
    if kind in ("add", "sub"):
        g = _c64(vector)
        return ((g.astype(np.uint64) << np.uint64(l)).astype(np.int64) + g)
    return vector


def poison_pattern(w: int, n: int) -> np.ndarray:
    """pkg/src/nent/pipeline.py:65-70."""
    pat = np.empty(n, dtype=np.int64)
    pat[0::2] = -(1 << (w - 1))
    pat[1::2] = (1 << (w - 1)) - 1
    return pat


def run_entangled(kind: str, data, m: int, w: int, l: int, failed: int | None = None,
                  threads: int = 0, **kernel) -> np.ndarray:
    """entangle -> op on entangled streams -> poison failed -> recover (pipeline.py:97-103)."""
    eps = entangle(data, l, threads)
    if kind in ("add", "sub"):
        kernel = dict(kernel, vector=self_entangle(kind, kernel["vector"], l))
    delta = apply_raw(kind, eps, threads=threads, **kernel)
    if failed is not None:
        delta = delta.copy()
        delta[failed] = poison_pattern(w, delta.shape[1])
    return disentangle(delta, m, l, w, failed, threads)


if __name__ == "__main__":  # pragma: no cover
    print(build(force=True))
    print("threads", max_threads(), os.cpu_count())

"""ctypes binding of libnent_b200.so (the C ABI declared in include/nent_b200.h).

There is no CPU fallback: if the library is missing, cannot be loaded, or no
sm_100 device is present, every call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import torch

from .errors import DeviceError, ParameterError, RangeError

LIB_PATH = Path(__file__).resolve().parent / "libnent_b200.so"

NENT_OK, NENT_ERR_PARAM, NENT_ERR_RANGE, NENT_ERR_CUDA, NENT_ERR_OVERFLOW = 0, 1, 2, 3, 4
MAC_I32, MAC_F64, MAC_W64, MAC_S64, MAC_G64, MAC_X128, MAC_IMMA = 1, 2, 3, 4, 5, 6, 7
BENCH_IMMA = 16
BENCH_TC05 = 17


IMMA_MMA_SYNC = 1 << 16  # NENT_IMMA_MMA_SYNC: force the mma.sync kernel


def imma_flavor(np_: int, ng: int, mma_sync: bool = False) -> int:
    """NENT_MAC_IMMA_DIGITS(np, ng): tensor-core digit slicing with np planes of x
    and ng digits of g (balanced base-256); tcgen05 where the shape fits it,
    mma.sync otherwise or when ``mma_sync``."""
    return MAC_IMMA | (np_ << 8) | (ng << 12) | (IMMA_MMA_SYNC if mma_sync else 0)


def is_imma(flavor: int) -> bool:
    return (flavor & 0xFF) == MAC_IMMA


class _FlavorNames(dict):
    def __missing__(self, key):
        if is_imma(key):
            return f"imma{(key >> 8) & 15}x{(key >> 12) & 15}" + ("-mma.sync" if key & IMMA_MMA_SYNC else "")
        raise KeyError(key)


MAC_NAMES = _FlavorNames({MAC_I32: "i32", MAC_F64: "f64", MAC_W64: "w64", MAC_S64: "s64",
                          MAC_G64: "g64", MAC_X128: "x128", BENCH_IMMA: "imma_s8_mma_sync", BENCH_TC05: "tcgen05_i8"})
EW_ADD, EW_SUB, EW_MUL = 0, 1, 2

_P = ctypes.c_void_p
_PP = ctypes.POINTER(ctypes.c_void_p)
_I = ctypes.c_int
_L = ctypes.c_int64

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "nent_last_error": [],
    "nent_abi_version": [],
    "nent_device_ok": [],
    "nent_enable_peer_access": [_I],
    "nent_entangle": [_PP, _I, _PP, _I, _I, _L, _I, _L, _P, _P],
    "nent_shift_add": [_P, _P, _I, _P, _I, _L, _I, _P],
    "nent_extract": [_PP, _I, _PP, _I, _I, _L, _I, _I, _I, _P, _P],
    "nent_extract_m3": [_PP, _I, _PP, _I, _L, _I, _I, _I, _P],
    "nent_conv": [_PP, _I, _I, _L, _L, _P, _I, _I, _PP, _I, _L, _L, _I, _P, _P, _P],
    "nent_imma_table_bytes": [_I, _I],
    "nent_imma_table": [_P, _I, _I, _L, _I, _P, _P],
    "nent_fused_conv": [_PP, _I, _I, _L, _L, _I, _L, _P, _I, _P, _P, _I, _I, _I, _I, _PP, _I,
                        _L, _L, _I, _P, _P, _P],
    "nent_chain_conv": [_P, _P, _I, _L, _L, _I, _L, _P, _I, _P, _P, _I, _I, _P, _I, _L, _L, _I,
                        _P, _P],
    "nent_interleave": [_PP, _I, _I, _L, _P, _P],
    "nent_gather_chain": [_P, _I, _I, _L, _I, _L, _P, _I, _P, _PP, _I, _P],
    "nent_interleave_chain": [_PP, _I, _I, _L, _I, _L, _P, _I, _P, _I, _P],
    "nent_gather_records": [_P, _I, _I, _L, _P, _I, _PP, _P],
    "nent_perm_check": [_P, _I, _L, _P, _P, _P],
    "nent_elementwise": [_PP, _I, _I, _L, _P, _I, _L, _I, _PP, _I, _I, _P, _P],
    "nent_scale": [_PP, _I, _I, _L, _L, _PP, _I, _I, _P, _P],
    "nent_permute": [_PP, _I, _I, _L, _P, _PP, _I, _P],
    "nent_reverse_circular": [_PP, _I, _I, _L, _PP, _I, _P],
    "nent_inner": [_PP, _I, _I, _L, _L, _P, _I, _PP, _I, _I, _P, _P],
    "nent_fused_inner": [_PP, _I, _I, _L, _L, _I, _P, _I, _I, _I, _PP, _I, _I, _P, _P],
    "nent_fused_outer": [_PP, _I, _I, _L, _L, _I, _P, _I, _L, _I, _I, _PP, _I, _P, _P],
    "nent_gemm": [_PP, _I, _I, _L, _P, _L, _PP, _I, _I, _P, _P],
    "nent_poison": [_P, _I, _L, _I, _P],
    "nent_max_abs": [_PP, _I, _I, _L, _P, _P],
    "nent_check_range": [_PP, _I, _I, _L, _L, _P, _P],
    "nent_checksum_encode": [_PP, _I, _I, _L, _P, _I, _P],
    "nent_checksum_recover": [_PP, _I, _P, _I, _I, _L, _I, _P, _I, _P],
    "nent_imma_kernel": [_I, _I, _I, _I],
    "nent_last_conv_kernel": [],
    "nent_extract_verify": [_PP, _I, _PP, _I, _I, _L, _I, _I, _I, _P, _P, _P],
    "nent_copy_rows": [_P, _L, _P, _L, _L, _I, _I, _P],
    "nent_microbench": [_I, _I, _I, _I, _P, ctypes.POINTER(ctypes.c_double), _P],
}
_RESTYPES = {"nent_last_error": ctypes.c_char_p, "nent_imma_table_bytes": ctypes.c_int64}

_lock = threading.Lock()
_lib = None
_device_checked: set[int] = set()


def load_library(path: Path = LIB_PATH):
    """Load the shared library and attach prototypes (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not path.exists():
                raise DeviceError(
                    f"{path} is missing: build it with paper_1509_03838_b200._build.build() "
                    "(there is no CPU fallback)")
            try:
                lib = ctypes.CDLL(str(path))
            except OSError as exc:
                raise DeviceError(f"cannot load {path}: {exc}") from exc
            for name, argtypes in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = lib
    return _lib


def lib():
    """The library, after checking that a usable sm_100 device is current."""
    L = load_library()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the entanglement hot path runs only on B200 (sm_100a); "
                          "there is no CPU fallback")
    dev = torch.cuda.current_device()
    if dev not in _device_checked:
        torch.cuda.init()
        if not L.nent_device_ok():
            raise DeviceError(L.nent_last_error().decode())
        _device_checked.add(dev)
    return L


def call(name: str, *args) -> None:
    """Invoke an entry point and map its status code onto the package errors."""
    st = getattr(lib(), name)(*args)
    if st == NENT_OK:
        return
    msg = _lib.nent_last_error().decode()
    if st == NENT_ERR_PARAM:
        raise ParameterError(f"{name}: {msg}")
    if st == NENT_ERR_RANGE:
        raise RangeError(f"{name}: {msg}")
    if st == NENT_ERR_OVERFLOW:
        raise OverflowError(f"{name}: {msg}")
    raise DeviceError(f"{name}: {msg}")


def stream_handle(stream: torch.cuda.Stream | None = None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def bits(t: torch.Tensor) -> int:
    if t.dtype == torch.int64:
        return 64
    if t.dtype == torch.int32:
        return 32
    raise ParameterError(f"device streams must be int32 or int64, got {t.dtype}")


def ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def row_ptrs(rows) -> ctypes.Array:
    """Host array of row pointers from a 2-D tensor (row stride honoured) or a
    sequence of 1-D tensors / None entries."""
    if isinstance(rows, torch.Tensor):
        if rows.dim() != 2 or rows.stride(1) != 1:
            raise ParameterError("row table needs a 2-D tensor with contiguous rows")
        base, step = rows.data_ptr(), rows.stride(0) * rows.element_size()
        vals = [base + i * step for i in range(rows.shape[0])]
    else:
        vals = [0 if r is None else r.data_ptr() for r in rows]
    arr = (ctypes.c_void_p * max(len(vals), 1))()
    for i, v in enumerate(vals):
        arr[i] = v
    return arr

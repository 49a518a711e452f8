"""Stream files: the reference's on-disk block format, read straight into HBM.

Format (/root/reference/pkg/src/nent/streamfile.py:1-7, byte-compatible): a
20-byte little-endian header -- magic ``NENT``, version u8 (= 1), word width
u8 (16 / 32 / 64), reserved u16, stream count u32, samples per stream u64 --
then the m streams back to back as w-bit two's-complement words.

``read_stream_file`` / ``write_stream_file`` keep the reference's signatures
and errors (streamfile.py:24-59: ``FormatError`` for a bad width, values that
do not fit, a 2-D shape violation, bad magic / version, empty geometry, a
truncated header or payload) and return int64 numpy like the reference.
``load_stream_file`` is the device path: the payload lands in a pinned host
buffer with one read and moves to the GPU with one asynchronous copy, in its
file word width (an int32 file stays int32 in HBM, which is what the fused
kernels consume), so the host never materialises the int64 widening.
``store_stream_file`` writes a device block back through a pinned buffer.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from .errors import FormatError

MAGIC = b"NENT"
VERSION = 1
HEADER = struct.Struct("<4sBBHIQ")  # magic, version, width, reserved, m, n
WIDTHS = {16: (np.dtype("<i2"), torch.int16), 32: (np.dtype("<i4"), torch.int32),
          64: (np.dtype("<i8"), torch.int64)}


def _check_width(w: int) -> None:
    if w not in WIDTHS:
        raise FormatError(f"unsupported word width {w} (use 16, 32 or 64)")


def _header(path, raw: bytes) -> tuple[int, int, int]:
    """(w, m, n) of a stream file whose bytes are ``raw``, validated."""
    if len(raw) < HEADER.size:
        raise FormatError(f"{path}: truncated header")
    magic, version, w, _reserved, m, n = HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    if w not in WIDTHS:
        raise FormatError(f"{path}: unsupported word width {w}")
    if m < 1 or n < 1:
        raise FormatError(f"{path}: empty stream geometry m={m}, n={n}")
    return w, m, n


def _payload_size(path, total: int, w: int, m: int, n: int) -> int:
    want = m * n * (w // 8)
    have = total - HEADER.size
    if have != want:
        raise FormatError(f"{path}: payload length {have} != {want}")
    return want


def write_stream_file(path, data, w: int) -> None:
    """Write an (m, n) integer array (numpy or tensor) as w-bit words
    (streamfile.py:24-38)."""
    _check_width(w)
    if isinstance(data, torch.Tensor):
        data = data.detach().cpu().numpy()
    data = np.asarray(data)
    if data.ndim != 2:
        raise FormatError("stream data must be 2-D (m x n)")
    m, n = data.shape
    lo, hi = -(1 << (w - 1)), (1 << (w - 1)) - 1
    if data.size and (int(data.min()) < lo or int(data.max()) > hi):
        raise FormatError(f"data does not fit in {w}-bit words")
    with open(path, "wb") as f:
        f.write(HEADER.pack(MAGIC, VERSION, w, 0, m, n))
        f.write(np.ascontiguousarray(data, dtype=WIDTHS[w][0]).tobytes())


def read_stream_file(path) -> tuple[np.ndarray, int]:
    """(m x n int64 array, word width) -- the reference's host reader
    (streamfile.py:41-59)."""
    raw = Path(path).read_bytes()
    w, m, n = _header(path, raw)
    _payload_size(path, len(raw), w, m, n)
    words = np.frombuffer(raw, dtype=WIDTHS[w][0], offset=HEADER.size)
    return words.astype(np.int64).reshape(m, n), w


def load_stream_file(path, device: torch.device | str | None = None) -> tuple[torch.Tensor, int]:
    """Read a stream file into device memory: (m x n tensor in the file's word
    width, word width).  One read into pinned host memory, one async H2D."""
    from . import _device as D

    path = Path(path)
    with open(path, "rb") as f:
        head = f.read(HEADER.size)
        w, m, n = _header(path, head)
        nbytes = _payload_size(path, path.stat().st_size, w, m, n)
        dev = torch.device(device) if device is not None else D.device()  # no device: DeviceError
        host = torch.empty((m, n), dtype=WIDTHS[w][1], pin_memory=True)
        view = memoryview(host.numpy()).cast("B")
        if f.readinto(view) != nbytes:
            raise FormatError(f"{path}: short read")
    out = torch.empty((m, n), dtype=host.dtype, device=dev)
    out.copy_(host, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()  # the pinned buffer is released on return
    return out, w


def store_stream_file(path, data: torch.Tensor, w: int) -> None:
    """Write a device (m, n) block as w-bit words through a pinned buffer."""
    _check_width(w)
    if data.dim() != 2:
        raise FormatError("stream data must be 2-D (m x n)")
    if data.numel():
        lo, hi = -(1 << (w - 1)), (1 << (w - 1)) - 1
        mn, mx = int(data.min()), int(data.max())
        if mn < lo or mx > hi:
            raise FormatError(f"data does not fit in {w}-bit words")
    host = torch.empty(tuple(data.shape), dtype=WIDTHS[w][1], pin_memory=True)
    host.copy_(data.to(WIDTHS[w][1]), non_blocking=True)
    torch.cuda.current_stream(data.device).synchronize()
    m, n = data.shape
    with open(path, "wb") as f:
        f.write(HEADER.pack(MAGIC, VERSION, w, 0, m, n))
        f.write(memoryview(host.numpy()).cast("B"))

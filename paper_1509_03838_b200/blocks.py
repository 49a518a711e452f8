"""Stream containers: plain (``StreamBlock``) and entangled (``EntangledBlock``).

Drop-in for /root/reference/pkg/src/nent/blocks.py:26-59.  ``data`` is either

* a host ``numpy.ndarray`` coerced to C-contiguous int64 (m, n) exactly like
  the reference (1-D input becomes a column), so reference callers can keep
  mutating ``block.data[...]`` and calling ``.tolist()``; every operation then
  copies to the B200, runs the kernels and returns int64 numpy again; or
* a CUDA ``torch.Tensor`` (int32 or int64, 2-D, contiguous rows): the data
  stays resident in HBM and every operation returns device blocks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import ParameterError
from .params import CodecParams


def _coerce(data, m: int):
    if isinstance(data, torch.Tensor):
        t = data
        if t.dim() == 1:
            t = t.reshape(-1, 1)
        if t.dim() != 2:
            raise ParameterError(f"block data must be 2-D (m x n), got shape {tuple(t.shape)}")
        if t.dtype not in (torch.int32, torch.int64):
            t = t.to(torch.int64)
        if t.shape[1] > 0 and t.stride(1) != 1:
            t = t.contiguous()
        arr = t
    else:
        arr = np.asarray(data, dtype=np.int64)
        if arr.ndim == 1:
            arr = arr.reshape(len(arr), 1)
        if arr.ndim != 2:
            raise ParameterError(f"block data must be 2-D (m x n), got shape {arr.shape}")
    if arr.shape[0] != m:
        raise ParameterError(f"expected {m} streams, got {arr.shape[0]}")
    if arr.shape[1] < 1:
        raise ParameterError("streams must hold at least one sample")
    return arr


class _Block:
    params: CodecParams
    data: object

    @property
    def n(self) -> int:
        return int(self.data.shape[1])

    @property
    def on_device(self) -> bool:
        return isinstance(self.data, torch.Tensor)

    def numpy(self) -> np.ndarray:
        """int64 host copy of the data (no copy for host blocks)."""
        if isinstance(self.data, torch.Tensor):
            return self.data.to(torch.int64).cpu().numpy()
        return self.data

    def _copy_data(self):
        return self.data.clone() if isinstance(self.data, torch.Tensor) else self.data.copy()


@dataclass
class StreamBlock(_Block):
    """m parallel integer streams of equal length n (codec inputs or results)."""

    params: CodecParams
    data: object = field(repr=False)

    def __post_init__(self):
        self.data = _coerce(self.data, self.params.m)

    def copy(self) -> "StreamBlock":
        return StreamBlock(self.params, self._copy_data())

    def to_device(self, device=None, dtype=torch.int64) -> "StreamBlock":
        return StreamBlock(self.params, _to_device(self.data, device, dtype))


@dataclass
class EntangledBlock(_Block):
    """m entangled streams; row i is (source[i-1 mod m] << l) + source[i]."""

    params: CodecParams
    data: object = field(repr=False)

    def __post_init__(self):
        self.data = _coerce(self.data, self.params.m)

    def copy(self) -> "EntangledBlock":
        return EntangledBlock(self.params, self._copy_data())

    def to_device(self, device=None, dtype=torch.int64) -> "EntangledBlock":
        return EntangledBlock(self.params, _to_device(self.data, device, dtype))


def _to_device(data, device, dtype):
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    if isinstance(data, torch.Tensor):
        return data.to(device=device, dtype=dtype)
    return torch.from_numpy(np.ascontiguousarray(data)).to(device=device, dtype=dtype)

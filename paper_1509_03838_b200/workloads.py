"""Canonical seeded inputs of the five BASELINE.json configs.

There is no public dataset for this path: every config is synthetic.  Inputs
are drawn with ``np.random.default_rng(seed)``, seed = config number, in the
documented order, each with ``rng.integers(lo, hi + 1, size, dtype=np.int64)``
-- so the known-answer digests in tests/golden/ apply.  ``scale_n`` shrinks
the stream length for quick parity runs (different draws, same shapes/ranges).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .params import CodecParams, derive_params


@dataclass
class Workload:
    name: str
    params: CodecParams
    c: np.ndarray                     # (m, n) or (m, batch, n) for cfg4
    g: np.ndarray                     # filter taps / shared vector
    mode: str = "full"                # convolution mode
    scale: int | None = None          # cfg5 chain
    add: np.ndarray | None = None
    perm: np.ndarray | None = None
    notes: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return self.params.m

    @property
    def n(self) -> int:
        return int(self.c.shape[-1])

    @property
    def K(self) -> int:
        return int(len(self.g))

    @property
    def out_len(self) -> int:
        return self.n + self.K - 1 if self.mode == "full" else self.n

    def macs(self) -> int:
        """Algorithmic multiply-accumulates of the conv stage (m * n * K)."""
        return self.m * self.n * self.K

    def output_samples(self) -> int:
        return self.m * self.out_len


def _draw(rng, lo, hi, size):
    return rng.integers(lo, hi + 1, size, dtype=np.int64)


# geometry per config: w=32 for cfg1/cfg5, w=64 for cfg2-cfg4
GEOMETRY = {1: (3, 32), 2: (3, 64), 3: (4, 64), 4: (3, 64), 5: (8, 32)}


def make(cfg: int, n: int | None = None, batch: int | None = None, K: int | None = None,
         seed: int | None = None) -> Workload:
    """Config ``cfg`` at full size by default (``n``/``batch``/``K`` override)."""
    seed = cfg if seed is None else seed
    rng = np.random.default_rng(seed)
    m, w = GEOMETRY[cfg]
    p = derive_params(m, w)
    if cfg == 1:
        n, K = n or 65_536, K or 64
        c = _draw(rng, -128, 127, (3, n))
        g = _draw(rng, -128, 127, (K,))
        return Workload("cfg1", p, c, g)
    if cfg == 2:
        n, K = n or (1 << 24), K or 256
        c = _draw(rng, -(1 << 11), (1 << 11) - 1, (3, n))
        g = _draw(rng, -(1 << 11), (1 << 11) - 1, (K,))
        return Workload("cfg2", p, c, g)
    if cfg == 3:
        n, K = n or (1 << 22), K or 1024
        c = _draw(rng, -(1 << 9), (1 << 9) - 1, (4, n))
        g = _draw(rng, -(1 << 9), (1 << 9) - 1, (K,))
        return Workload("cfg3", p, c, g)
    if cfg == 4:
        n, batch = n or 4096, batch or 65_536
        c = _draw(rng, -(1 << 7), (1 << 7) - 1, (3, batch, n))
        g = _draw(rng, -(1 << 7), (1 << 7) - 1, (n,))
        return Workload("cfg4", p, c, g, mode="inner")
    if cfg == 5:
        n, K = n or (1 << 24), K or 128
        c = _draw(rng, -128, 127, (8, n))
        s = 0
        while s == 0:  # a zero scale makes the chain trivial
            s = int(rng.integers(-16, 17))
        a = _draw(rng, -128, 127, (n,))
        perm = rng.permutation(n)
        g = _draw(rng, -128, 127, (K,))
        return Workload("cfg5", p, c, g, scale=s, add=a, perm=perm.astype(np.int64))
    raise ValueError(f"unknown config {cfg}")

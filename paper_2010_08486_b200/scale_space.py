"""Sigma ladder and separable tap tables (host side, float64).

Mirrors the reference's scale-space definition (`pkg/src/dogblob/scale_space.py`):
an arithmetic ladder of n_bin + 1 scales, one unit-sum Gaussian per scale
sampled on the integer grid out to ceil(truncate * sigma).  The reference
materialises dense 2-D kernels k = outer(g, g) / sum (scale_space.py:76-81);
they are exactly separable, k = w (x) w with w = g / sum(g), and the CUDA
path only ever needs the 1-D taps, so a `TapBank` stores those (9,233 floats
at sigma <= 30 instead of a 43 MB bank).  `dense_kernels()` rebuilds the
reference's padded 2-D bank on demand for callers that want it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

__all__ = ["SigmaLadder", "TapBank", "KernelBank", "build_ladder", "build_kernel_bank",
           "gaussian_taps", "MAX_WIDTH_CAP"]

MAX_WIDTH_CAP = 4097  # scale_space.py:21


@dataclass(frozen=True)
class SigmaLadder:
    """scale_space.py:24-37."""
    min_sigma: float
    max_sigma: float
    n_bin: int
    sigmas: np.ndarray = field(repr=False)
    delta_sigma: float

    @property
    def n_levels(self) -> int:
        return self.n_bin + 1


def build_ladder(min_sigma: float, max_sigma: float, n_bin: int) -> SigmaLadder:
    """sigma_i = linspace(min, max, n_bin + 1); error cases of scale_space.py:54-64."""
    if not min_sigma > 0:
        raise ValueError(f"min_sigma must be > 0, got {min_sigma}")
    if max_sigma < min_sigma:
        raise ValueError(f"max_sigma {max_sigma} < min_sigma {min_sigma}")
    if n_bin < 1:
        raise ValueError(f"n_bin must be >= 1, got {n_bin}")
    if max_sigma == min_sigma:
        raise ValueError("degenerate ladder: max_sigma == min_sigma")
    sig = np.linspace(min_sigma, max_sigma, n_bin + 1)
    sig.setflags(write=False)
    return SigmaLadder(float(min_sigma), float(max_sigma), int(n_bin), sig,
                       float((max_sigma - min_sigma) / n_bin))


def gaussian_taps(sigma: float, radius: int) -> np.ndarray:
    """Unit-sum 1-D taps w[-r..r] in float64; outer(w, w) is the reference kernel."""
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    g = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return g / g.sum()


@dataclass(frozen=True)
class TapBank:
    """1-D taps of every ladder scale, concatenated.

    taps64 / taps32 hold w_i back to back; offsets[i] is the start of level i and
    radii[i] = ceil(truncate * sigma_i) its half-width (scale_space.py:97).
    `max_width` equals the reference bank's padded kernel width.
    """
    ladder: SigmaLadder
    truncate: float
    radii: np.ndarray = field(repr=False)
    offsets: np.ndarray = field(repr=False)
    taps64: np.ndarray = field(repr=False)
    taps32: np.ndarray = field(repr=False)
    max_width: int

    def level_taps(self, i: int, dtype=np.float64) -> np.ndarray:
        src = self.taps64 if np.dtype(dtype) == np.float64 else self.taps32
        o, r = int(self.offsets[i]), int(self.radii[i])
        return src[o:o + 2 * r + 1]

    def dense_kernels(self) -> np.ndarray:
        """The reference's (n_levels, max_width, max_width) zero-framed bank."""
        n, mw = self.ladder.n_levels, self.max_width
        mr = mw // 2
        out = np.zeros((n, mw, mw), dtype=np.float64)
        for i, s in enumerate(self.ladder.sigmas):
            r = int(self.radii[i])
            x = np.arange(-r, r + 1, dtype=np.float64)
            g = np.exp(-(x * x) / (2.0 * float(s) * float(s)))
            k = np.outer(g, g)
            out[i, mr - r:mr + r + 1, mr - r:mr + r + 1] = k / k.sum()
        return out

    @cached_property
    def kernels(self) -> np.ndarray:  # reference attribute name (KernelBank.kernels)
        k = self.dense_kernels()
        k.setflags(write=False)
        return k


KernelBank = TapBank  # the reference's name for the per-ladder filter bank


def build_kernel_bank(ladder: SigmaLadder, truncate: float = 5.0,
                      max_width_cap: int = MAX_WIDTH_CAP) -> TapBank:
    """scale_space.py:84-119 with the same guards, producing separable taps."""
    if not truncate > 0:
        raise ValueError(f"truncate must be > 0, got {truncate}")
    radii = np.array([math.ceil(truncate * float(s)) for s in ladder.sigmas], dtype=np.int64)
    max_width = 2 * int(radii.max()) + 1
    if max_width > max_width_cap:
        raise ValueError(f"kernel width {max_width} exceeds cap {max_width_cap} "
                         f"(max_sigma={ladder.max_sigma}, truncate={truncate})")
    offsets = np.zeros(ladder.n_levels, dtype=np.int64)
    chunks = []
    pos = 0
    for i, (s, r) in enumerate(zip(ladder.sigmas, radii)):
        offsets[i] = pos
        w = gaussian_taps(float(s), int(r))
        chunks.append(w)
        pos += w.size
    taps64 = np.concatenate(chunks)
    taps32 = taps64.astype(np.float32)
    for a in (radii, offsets, taps64, taps32):
        a.setflags(write=False)
    return TapBank(ladder, float(truncate), radii, offsets, taps64, taps32, max_width)

"""Gaussian gridding window metadata (reference gridding.py:1-98).

The window itself (fine-grid geometry, factorised weights, deconvolution) is
evaluated inside the CUDA kernels; this module keeps the reference's
``GriddingKernel`` / ``kernel_for_size`` API so callers can pass a kernel
(e.g. a different ``spread_width``) exactly as before.  The host tables
(`bins`, `deconv`) are informational copies for callers that inspect them.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .grid import DEFAULT_SPREAD_WIDTH


def gaussian_shape(spread_width: int) -> float:
    """b of exp(-x^2 / 4b) balancing alias and truncation exponents (gridding.py:32-34)."""
    return spread_width / (2.0 * np.sqrt(2.0) * np.pi)


@dataclass(frozen=True, eq=False)
class GriddingKernel:
    """Window parameters for transforms with output length `size` (oversampling 2)."""

    size: int
    spread_width: int
    shape_b: float
    fine_size: int
    band_shift: int
    bins: np.ndarray
    deconv: np.ndarray

    @property
    def taps(self) -> int:
        return 2 * self.spread_width + 1


@lru_cache(maxsize=64)
def kernel_for_size(size: int, spread_width: int = DEFAULT_SPREAD_WIDTH) -> GriddingKernel:
    """Build (or fetch a cached) window description for output length `size`."""
    if size < 1:
        raise ValueError(f"transform size must be >= 1, got {size}")
    if spread_width < 1:
        raise ValueError(f"spread width must be >= 1, got {spread_width}")
    b = gaussian_shape(spread_width)
    n = 2 * size
    K = size // 2
    nu = np.arange(size) - K
    deconv = np.exp(b * (2.0 * np.pi * nu / n) ** 2) / np.sqrt(4.0 * np.pi * b)
    bins = nu % n
    deconv.setflags(write=False)
    bins.setflags(write=False)
    return GriddingKernel(size, spread_width, b, n, K, bins, deconv)

"""Trial inputs and the error metric used by the reference's harness
(bench.py:84-104); host-side utilities, not part of the device path."""

from __future__ import annotations

import math

import numpy as np

from .errors import LengthMismatchError, ZeroReferenceError
from .grid import validate_grid


def generate_trial(P: int, seed: int, jitter_max: float = 0.6):
    """Jittered grid t_p = p/P + U[0, jitter_max/P) and CN(0,1) amplitudes (Philox)."""
    if P < 2:
        raise ValueError("need P >= 2 for a jittered grid")
    rng = np.random.Generator(np.random.Philox(key=seed))
    jitter = rng.uniform(0.0, jitter_max / P, size=P)
    grid = validate_grid(np.arange(P) / P + jitter)
    amp = (rng.standard_normal(P) + 1j * rng.standard_normal(P)) / math.sqrt(2.0)
    return grid, amp


def relative_error(truth, estimate) -> float:
    """||truth - estimate|| / ||truth||."""
    t = np.asarray(truth, dtype=np.complex128)
    e = np.asarray(estimate, dtype=np.complex128)
    if t.shape != e.shape:
        raise LengthMismatchError(f"shape mismatch: {t.shape} vs {e.shape}")
    tn = float(np.linalg.norm(t))
    if tn == 0.0:
        raise ZeroReferenceError("relative error undefined: reference vector is zero")
    return float(np.linalg.norm(t - e)) / tn

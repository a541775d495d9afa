"""Trial inputs and the error metric of the figure harness (reference
bench.py:84-104).

`trial_arrays` reproduces the reference's per-trial random streams exactly:
ONE Philox(key=seed) generator, the jitter drawn first (uniform on
[0, jitter_max/P), i.e. jitter_max/P times a unit double), then the real and
the imaginary standard-normal parts of the amplitudes — so for a given seed
the nodes and the truth vector are bit-identical to the reference's and the
GPU harness's rows line up with the reference's record for record.

`relative_error` is ||truth - estimate|| / ||truth||; when either operand is
a CUDA tensor it is evaluated on that device (one scalar comes back).
"""

from __future__ import annotations

import math

import numpy as np

from .errors import LengthMismatchError, ZeroReferenceError
from .grid import validate_grid


def trial_arrays(P: int, seed: int, jitter_max: float = 0.6) -> tuple[np.ndarray, np.ndarray]:
    """(nodes, amplitudes) of one trial: t_p = p/P + jitter_max/P * U_p, a = (N1 + i N2)/sqrt(2)."""
    if P < 2:
        raise ValueError("need P >= 2 for a jittered grid")
    gen = np.random.Generator(np.random.Philox(key=seed))
    nodes = np.arange(P) / P + gen.uniform(0.0, jitter_max / P, size=P)
    re = gen.standard_normal(P)
    im = gen.standard_normal(P)
    return nodes, (re + 1j * im) / math.sqrt(2.0)


def generate_trial(P: int, seed: int, jitter_max: float = 0.6):
    """Validated jittered grid and CN(0, 1) amplitudes of one trial."""
    nodes, amp = trial_arrays(P, seed, jitter_max)
    return validate_grid(nodes), amp


def relative_error(truth, estimate) -> float:
    """||truth - estimate|| / ||truth|| (device-side for CUDA tensors)."""
    try:
        import torch
    except Exception:  # pragma: no cover - torch is part of the image
        torch = None
    if torch is not None and any(isinstance(v, torch.Tensor) and v.is_cuda for v in (truth, estimate)):
        dev = next(v.device for v in (truth, estimate) if isinstance(v, torch.Tensor) and v.is_cuda)
        t = torch.as_tensor(truth, dtype=torch.complex128).to(dev)
        e = torch.as_tensor(estimate, dtype=torch.complex128).to(dev)
        if t.shape != e.shape:
            raise LengthMismatchError(f"shape mismatch: {tuple(t.shape)} vs {tuple(e.shape)}")
        norms = torch.stack([torch.linalg.vector_norm(t), torch.linalg.vector_norm(t - e)]).cpu()
        tn, dn = float(norms[0]), float(norms[1])
    else:
        t = np.asarray(truth, dtype=np.complex128)
        e = np.asarray(estimate, dtype=np.complex128)
        if t.shape != e.shape:
            raise LengthMismatchError(f"shape mismatch: {t.shape} vs {e.shape}")
        tn, dn = float(np.linalg.norm(t)), float(np.linalg.norm(t - e))
    if tn == 0.0:
        raise ZeroReferenceError("relative error undefined: reference vector is zero")
    return dn / tn

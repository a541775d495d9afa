"""DFT wrappers (reference fftops.py:17-41) on the B200 Stockham FFT engine."""

from __future__ import annotations

import numpy as np

from . import _device, _lib
from .errors import LengthMismatchError
from .flops import FlopCounter


def _run(x, sign: int, scale: bool, flops: FlopCounter | None, device=None):
    dev = _device.device_index(device)
    a = _device.operand(x, dev, name="vector")
    out = a.empty_like_rows(a.n)
    _lib.call("nfft45_dft", a.ptr, out.data_ptr(), a.rows, a.n, sign, _device.stream_handle(dev))
    if scale:
        out = out / a.n
    if flops is not None:
        flops.fft(a.n)
        if scale:
            flops.real_mul(2 * a.n)
    return a.finish(out)


def dft(x, flops: FlopCounter | None = None, device=None):
    """X_k = sum_j x_j e^{-2 pi i jk/N} (np.fft.fft convention)."""
    return _run(x, -1, False, flops, device)


def idft(X, flops: FlopCounter | None = None, device=None):
    """x_j = (1/N) sum_k X_k e^{+2 pi i jk/N} (np.fft.ifft convention)."""
    return _run(X, +1, True, flops, device)


def hadamard(x, y, flops: FlopCounter | None = None):
    """Elementwise product of two equal-length complex vectors."""
    a = np.asarray(x, dtype=np.complex128)
    b = np.asarray(y, dtype=np.complex128)
    if a.shape != b.shape:
        raise LengthMismatchError(f"shape mismatch: {a.shape} vs {b.shape}")
    if flops is not None:
        flops.complex_mul(a.size)
    return a * b

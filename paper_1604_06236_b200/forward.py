"""Forward type-1 / type-2 NFFTs and the nonuniform convolution on the B200
(reference forward.py:1-162).

Every function validates like the reference, then issues one C-ABI call into
libnfft45 (spread/gather kernels + Stockham FFTs).  numpy in -> numpy out;
torch CUDA tensors in -> tensors out (no sync).  2-D [batch, n] operands are
the batched extension (one signal per row, one shared node set).
"""

from __future__ import annotations

import numpy as np

from . import _device, _lib
from . import flops as _fl
from .errors import SizeMismatchError
from .flops import FlopCounter
from .grid import NonuniformGrid
from .gridding import GriddingKernel, kernel_for_size


def _width(kernel: GriddingKernel | None, size: int) -> int:
    if kernel is None:
        kernel = kernel_for_size(size)
    elif kernel.size != size:
        raise SizeMismatchError(f"kernel built for size {kernel.size}, transform needs {size}")
    return kernel.spread_width, kernel


def nfft_type1(grid: NonuniformGrid, amplitudes, R: int, kernel: GriddingKernel | None = None,
               flops: FlopCounter | None = None, device=None):
    """A(p) = sum_q a_q e^{-2 pi i p t_q}, p = 0..R-1 (forward.py:26-64)."""
    if R < 1:
        raise ValueError(f"output length must be >= 1, got {R}")
    dev = _device.device_index(device)
    a = _device.operand(amplitudes, dev, length=grid.size, name="amplitudes")
    m, kernel = _width(kernel, R)
    out = a.empty_like_rows(R)
    _lib.call("nfft45_type1", grid.device_handle(dev), a.ptr, a.rows, R, m, out.data_ptr(),
              _device.stream_handle(dev))
    _fl.charge_type1(flops, grid.size, R, kernel.taps)
    return a.finish(out)


def nfft_type2(coefficients, grid: NonuniformGrid, kernel: GriddingKernel | None = None,
               flops: FlopCounter | None = None, device=None):
    """s(t_q) = sum_p S_p e^{+2 pi i p t_q} (forward.py:67-102)."""
    dev = _device.device_index(device)
    S = _device.operand(coefficients, dev, name="coefficients")
    P = S.n
    m, kernel = _width(kernel, P)
    out = S.empty_like_rows(grid.size)
    _lib.call("nfft45_type2", grid.device_handle(dev), S.ptr, S.rows, P, m, out.data_ptr(),
              _device.stream_handle(dev))
    _fl.charge_type2(flops, grid.size, P, kernel.taps)
    return S.finish(out)


def nfft_type1_direct(grid: NonuniformGrid, amplitudes, R: int, device=None):
    """Exact O(RQ) type-1 sum with exactly reduced phases (forward.py:105-118)."""
    dev = _device.device_index(device)
    a = _device.operand(amplitudes, dev, length=grid.size, name="amplitudes")
    out = a.empty_like_rows(R)
    _lib.call("nfft45_type1_direct", grid.device_handle(dev), a.ptr, a.rows, R, out.data_ptr(),
              _device.stream_handle(dev))
    return a.finish(out)


def nfft_type2_direct(coefficients, grid: NonuniformGrid, device=None):
    """Exact O(PQ) type-2 sum (forward.py:121-130)."""
    dev = _device.device_index(device)
    S = _device.operand(coefficients, dev, name="coefficients")
    out = S.empty_like_rows(grid.size)
    _lib.call("nfft45_type2_direct", grid.device_handle(dev), S.ptr, S.rows, S.n, out.data_ptr(),
              _device.stream_handle(dev))
    return S.finish(out)


def nonuniform_conv(grid: NonuniformGrid, amplitudes, lam_coefficients, P: int,
                    kernel: GriddingKernel | None = None, flops: FlopCounter | None = None, device=None):
    """gamma(q/P) = sum_q a_q lam(q/P - t_q): type-1 of length R, fold, IDFT_P (forward.py:133-162)."""
    lam_host = lam_coefficients
    R = int(np.asarray(lam_host).size) if not hasattr(lam_host, "numel") else int(lam_host.numel())
    if R % P != 0:
        raise SizeMismatchError(f"kernel length {R} is not a multiple of output length {P}")
    dev = _device.device_index(device)
    a = _device.operand(amplitudes, dev, length=grid.size, name="amplitudes")
    m, kernel = _width(kernel, R)
    lam = _device.real_table(lam_host, dev)
    out = a.empty_like_rows(P)
    _lib.call("nfft45_nonuniform_conv", grid.device_handle(dev), a.ptr, a.rows, lam.data_ptr(), R, P, m,
              out.data_ptr(), _device.stream_handle(dev))
    if flops is not None:
        _fl.charge_type1(flops, grid.size, R, kernel.taps)
        real = not np.iscomplexobj(lam_host) if not hasattr(lam_host, "is_complex") else not lam_host.is_complex()
        _fl.charge_conv_tail(flops, R, P, real)
    return a.finish(out)

"""The paper's competitors on the B200 (reference baselines.py:1-181).

* ``cg_solve`` — conjugate gradient on the normal equations (CGNR),
  unpreconditioned; each iteration is one type-1 plus one type-2 NFFT (the
  forward kernels of this package) and fused vector kernels, all device
  resident (csrc/cg.cu, C ABI ``nfft45_cg_solve``).  2-D right-hand sides run
  one recurrence per row.
* ``ge_solve`` with ``type4_system`` / ``type5_system`` — dense Gaussian
  elimination with partial pivoting on the device (csrc/dense.cu, C ABI
  ``nfft45_ge_solve``), in the reference's right-looking order: a blocked
  library LU is measurably less accurate on these systems, and the figure
  protocols use GE as the accuracy floor.  The phase matrix comes from the
  exact direct-sum kernels.

Semantics follow the reference: same arguments and defaults, the same
``CGResult`` fields, ``SingularMatrixError`` below the 1e-300 pivot floor,
``ValueError`` for a non-positive tolerance or an unknown system kind, and
the same data-independent ``flops=`` charges.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes
import numpy as np
import torch

from . import _device, _lib
from . import flops as _fl
from .errors import SingularMatrixError
from .flops import FlopCounter
from .grid import NonuniformGrid, as_complex_vector
from .gridding import kernel_for_size

PIVOT_FLOOR = 1e-300


@dataclass(frozen=True, eq=False)
class DenseSystem:
    """One dense P x P system (baselines.py:27-34)."""

    matrix: np.ndarray
    rhs: np.ndarray


def _phase_matrix(grid: NonuniformGrid, sign: int, flops: FlopCounter | None) -> np.ndarray:
    """Entries e^{sign 2 pi i p t_q}, rows p, columns q (baselines.py:37-49),
    from the exact direct-sum kernels applied to identity rows."""
    from .forward import nfft_type1_direct, nfft_type2_direct

    P = grid.size
    eye = torch.eye(P, dtype=torch.complex128, device=f"cuda:{_device.device_index(None)}")
    if sign > 0:  # type2_direct(I)[p][q] = e^{+2 pi i p t_q}
        M = nfft_type2_direct(eye, grid)
    else:  # type1_direct(I)[q][p] = e^{-2 pi i p t_q}
        M = nfft_type1_direct(grid, eye, P).transpose(0, 1)
    if flops is not None:
        flops.real_mul(P * P)
        flops.complex_exp(P * P)
    return np.ascontiguousarray(M.cpu().numpy())


def type4_system(grid: NonuniformGrid, spectrum, flops: FlopCounter | None = None) -> DenseSystem:
    """System whose solution is the delta-train amplitudes (baselines.py:52-55)."""
    rhs = as_complex_vector(spectrum, length=grid.size, name="spectrum")
    return DenseSystem(matrix=_phase_matrix(grid, -1, flops), rhs=rhs)


def type5_system(grid: NonuniformGrid, samples, flops: FlopCounter | None = None) -> DenseSystem:
    """System whose solution is the polynomial coefficients (baselines.py:58-61)."""
    rhs = as_complex_vector(samples, length=grid.size, name="samples")
    return DenseSystem(matrix=_phase_matrix(grid, +1, flops).T.copy(), rhs=rhs)


def _charge_ge(flops: FlopCounter | None, n: int, steps: int, solved: bool):
    """baselines.py:86-104: elimination steps 0..steps-1, then back substitution."""
    if flops is None:
        return
    for k in range(steps):
        r = n - 1 - k
        flops.complex_div(r)
        flops.complex_mul(r * r + r)
        flops.complex_add(r * r + r)
    if solved:
        tri = n * (n - 1) // 2
        flops.complex_mul(tri)
        flops.complex_add(tri)
        flops.complex_div(n)


def ge_solve(system: DenseSystem, flops: FlopCounter | None = None, device=None) -> np.ndarray:
    """Gaussian elimination with partial pivoting (baselines.py:64-105), on
    the device in the reference's elimination order (csrc/dense.cu).

    Raises SingularMatrixError when a pivot magnitude falls below 1e-300."""
    A = np.array(system.matrix, dtype=np.complex128)
    b = np.array(system.rhs, dtype=np.complex128)
    n = A.shape[0]
    if A.shape != (n, n) or b.shape != (n,):
        raise ValueError("system must be square with a matching right-hand side")
    dev = _device.device_index(device)
    Ad = torch.from_numpy(A).to(f"cuda:{dev}")
    bd = torch.from_numpy(b).to(f"cuda:{dev}")
    xd = torch.empty_like(bd)
    step, piv = ctypes.c_int64(n), ctypes.c_double(0.0)
    status = _lib.load().nfft45_ge_solve(Ad.data_ptr(), bd.data_ptr(), n, xd.data_ptr(), PIVOT_FLOOR,
                                         ctypes.byref(step), ctypes.byref(piv), _device.stream_handle(dev))
    solved = status == 0
    _charge_ge(flops, n, min(step.value, n - 1), solved)
    _lib.check(status)
    return xd.cpu().numpy()


@dataclass(frozen=True, eq=False)
class CGResult:
    """baselines.py:108-113 (per-row arrays for a 2-D right-hand side)."""

    solution: object
    iterations: object
    converged: object
    relative_residual: object


def _charge_cg(flops: FlopCounter | None, P: int, taps: int, which: str, iterations: int, converged: bool,
               stalled: bool, zero_rhs: bool):
    """The data-independent charges of one reference cg_solve call
    (baselines.py:141-181): A^H once, then per iteration A and the vector
    updates, and A^H + direction update unless the iteration stopped."""
    if flops is None or zero_rhs:
        return
    Q = P

    def apply_A():
        (_fl.charge_type1 if which == "type4" else _fl.charge_type2)(flops, Q, P, taps)

    def apply_AH():
        (_fl.charge_type2 if which == "type4" else _fl.charge_type1)(flops, Q, P, taps)

    apply_AH()
    flops.real_mul(2 * P)
    flops.real_add(2 * P)
    full = iterations - (1 if converged and not stalled else 0)  # iterations that also did A^H
    for _ in range(full):
        apply_A()
        flops.real_mul(2 * P + 1)
        flops.real_add(2 * P)
        flops.real_mul(4 * P)
        flops.complex_add(2 * P)
        apply_AH()
        flops.real_mul(2 * P + 1)
        flops.real_add(2 * P)
        flops.real_mul(2 * P)
        flops.complex_add(P)
    if converged and not stalled and iterations > 0:
        apply_A()
        flops.real_mul(2 * P + 1)
        flops.real_add(2 * P)
        flops.real_mul(4 * P)
        flops.complex_add(2 * P)
    if stalled:
        apply_A()  # the iteration whose |A p| was zero


def cg_solve(grid: NonuniformGrid, rhs, which: str = "type4", tol: float = 1e-15, max_iter: int | None = None,
             spread_width: int | None = None, flops: FlopCounter | None = None, device=None) -> CGResult:
    """Conjugate gradient on the normal equations (CGNR), unpreconditioned
    (baselines.py:116-181).  Stops at relative recurred residual <= tol or at
    max_iter (default 4P), returning the best iterate with a convergence flag."""
    if tol <= 0.0:
        raise ValueError("tolerance must be positive")
    if which not in ("type4", "type5"):
        raise ValueError(f"unknown system kind {which!r}")
    P = grid.size
    kernel = kernel_for_size(P, spread_width) if spread_width else kernel_for_size(P)
    if max_iter is None:
        max_iter = 4 * P
    dev = _device.device_index(device)
    b = _device.operand(rhs, dev, length=P, name="rhs")
    rows = b.rows
    x = b.empty_like_rows(P)
    iters = (ctypes.c_int64 * rows)()
    conv = (ctypes.c_int * rows)()
    rel = (ctypes.c_double * rows)()
    stalled = (ctypes.c_int * rows)()
    _lib.call("nfft45_cg_solve", grid.device_handle(dev), 4 if which == "type4" else 5, b.ptr, rows, float(tol),
              int(max_iter), kernel.spread_width, x.data_ptr(), iters, conv, rel, stalled,
              _device.stream_handle(dev))
    if flops is not None:
        bn = torch.linalg.vector_norm(b.tensor.reshape(rows, P), dim=1).cpu().numpy()
        for i in range(rows):
            _charge_cg(flops, P, kernel.taps, which, int(iters[i]), bool(conv[i]), bool(stalled[i]),
                       bn[i] == 0.0)
    sol = b.finish(x)
    if b.batched:
        return CGResult(sol, np.array(iters[:], dtype=np.int64), np.array(conv[:], dtype=bool),
                        np.array(rel[:], dtype=np.float64))
    return CGResult(sol, int(iters[0]), bool(conv[0]), float(rel[0]))

"""Non-iterative type-4 / type-5 inversion on the B200 (reference inverse.py:1-202).

build_plan uploads the node set and builds every grid-only table on the
device in one C call (three NFFT-sized stages + node factors); type5/type4
are one C call each (spread/gather + Stockham FFTs with fused elementwise
stages); refine_type5/4 run the Section V residual passes inside the C call.
"""

from __future__ import annotations

import os

import ctypes
import threading

import numpy as np

from . import _device, _lib
from . import flops as _fl
from .flops import FlopCounter
from .grid import MethodParams, NonuniformGrid
from .gridding import GriddingKernel, kernel_for_size
from .lagrange import KernelData, _amplification_check

_TABLE = {"v": 0, "ks": 1, "L": 2, "dL": 3, "nw": 4, "decay": 5, "coef": 6}


class _PlanHandle:
    def __init__(self, ptr, grid_handle_owner):
        self.ptr = ptr
        self._owner = grid_handle_owner  # keeps the device grid alive

    def __del__(self):
        try:
            if self.ptr:
                _lib.load().nfft45_plan_destroy(self.ptr)
        except Exception:
            pass


class InversePlan:
    """Grid-only precomputation, reusable across right-hand sides (inverse.py:33-55).

    Device tables live in the C plan; the numpy views the reference exposes
    (kernel_data, node_weights, h1_coefficients, coef_scale) are copied back
    lazily on first access and are read-only.
    """

    def __init__(self, grid: NonuniformGrid, params: MethodParams, handle: _PlanHandle, device: int,
                 kernel_fine: GriddingKernel, kernel_base: GriddingKernel):
        self.grid = grid
        self.params = params
        self.kernel_fine = kernel_fine
        self.kernel_base = kernel_base
        self.device = device
        self._h = handle
        self._cache = {}
        self._mu = threading.Lock()

    @property
    def size(self) -> int:
        return self.grid.size

    @property
    def handle(self):
        return self._h.ptr

    def table(self, name: str, as_tensor: bool = False):
        """One plan table (caller order for node-indexed ones)."""
        torch = _device.torch
        t = torch.empty(self.size, dtype=torch.complex128, device=f"cuda:{self.device}")
        _lib.call("nfft45_plan_table", self.handle, _TABLE[name], t.data_ptr(), _device.stream_handle(self.device))
        return t if as_tensor else t.cpu().numpy()

    def _host(self, name: str, real: bool = False) -> np.ndarray:
        arr = self._cache.get(name)
        if arr is None:
            with self._mu:
                arr = self._cache.get(name)
                if arr is None:
                    arr = self.table(name)
                    if real:
                        arr = np.ascontiguousarray(arr.real)
                    arr.setflags(write=False)
                    self._cache[name] = arr
        return arr

    @property
    def kernel_data(self) -> KernelData:
        return KernelData(v_samples=self._host("v"), kernel_samples=self._host("ks"),
                          coefficients=self._host("L"), derivative_samples=self._host("dL"))

    @property
    def node_weights(self) -> np.ndarray:
        return self._host("nw")

    @property
    def h1_coefficients(self) -> np.ndarray:
        return self._host("decay", real=True)

    @property
    def coef_scale(self) -> np.ndarray:
        return self._host("coef", real=True)


def _charge_plan(f: FlopCounter | None, P: int, params: MethodParams):
    """build_kernel_data + build_plan charges (lagrange.py:57-164, inverse.py:79-86)."""
    if f is None:
        return
    taps = 2 * params.spread_width + 1
    R = params.series_terms(P)
    f.complex_exp(R - 1)
    f.real_mul(R - 1)
    _fl.charge_type1(f, P, R, taps)
    _fl.charge_conv_tail(f, R, P, True)
    f.real_add(P)
    f.complex_add(P)
    f.complex_exp(P)
    f.complex_exp(P)
    f.fft(P)
    f.complex_exp(1)
    f.real_mul(1 + P)
    f.complex_add(1)
    f.real_mul(2 * P)
    f.real_mul(2 * P)
    _fl.charge_type2(f, P, P, taps)
    f.complex_exp(P)
    f.real_mul(2 * P)
    f.complex_exp(2 * P + 1)
    f.real_mul(2 * P)
    f.complex_add(P)
    f.complex_div(2 * P)
    f.complex_mul(P)


def build_plan(grid: NonuniformGrid, params: MethodParams, flops: FlopCounter | None = None,
               device=None) -> InversePlan:
    """Precompute everything grid-dependent for type-4/type-5 solves (inverse.py:58-98)."""
    P = grid.size
    dev = _device.device_index(device)
    R = params.series_terms(P)
    kernel_fine = kernel_for_size(R, params.spread_width)
    kernel_base = kernel_for_size(P, params.spread_width)
    _amplification_check(P, params.damping_a)
    gptr = grid.device_handle(dev)
    out = ctypes.c_void_p()
    if params.fractional_eta:  # extension: R = eta P series terms, partial fold
        _lib.call("nfft45_plan_create_terms", gptr, float(params.damping_a), R, int(params.spread_width),
                  _device.stream_handle(dev), ctypes.byref(out))
    else:
        _lib.call("nfft45_plan_create", gptr, float(params.damping_a), int(params.eta), int(params.spread_width),
                  _device.stream_handle(dev), ctypes.byref(out))
    _charge_plan(flops, P, params)
    return InversePlan(grid, params, _PlanHandle(out.value, grid), dev, kernel_fine, kernel_base)


def _charge_type5(f, P, taps):
    if f is None:
        return
    _fl.charge_type1(f, P, P, taps)
    _fl.charge_conv_tail(f, P, P, True)
    f.complex_mul(2 * P)
    f.fft(P)
    f.real_mul(2 * P)


def charge_refine(f, kind: int, P: int, taps: int, passes: int):
    """Data-independent flop charge of refine_type5/4 (inverse.py:146-202): the
    solve, then per pass one forward NFFT, the residual subtraction and the
    correction solve."""
    if f is None:
        return
    solve = _charge_type5 if kind == 5 else _charge_type4
    solve(f, P, taps)
    for _ in range(passes):
        if kind == 5:
            _fl.charge_type2(f, P, P, taps)
        else:
            _fl.charge_type1(f, P, P, taps)
        f.complex_add(2 * P)
        solve(f, P, taps)


def charge_plan(f, P: int, params: MethodParams):
    """Data-independent flop charge of build_plan (lagrange.py:57-164, inverse.py:79-86)."""
    _charge_plan(f, P, params)


def charge_type4(f, P: int, taps: int):
    """Data-independent flop charge of type4 (inverse.py:136-142)."""
    _charge_type4(f, P, taps)


def _charge_type4(f, P, taps):
    if f is None:
        return
    _fl.charge_type2(f, P, P, taps)
    f.real_mul(2 * P)
    f.fft(P)
    f.complex_mul(P)
    f.fft(P)
    f.real_mul(2 * P)
    f.complex_mul(P)


# Host-resident batches are streamed through the device in chunks of this many
# signals: H2D of chunk i+1 and D2H of chunk i-1 (two copy streams, PCIe is
# full duplex) overlap the solve of chunk i.
STREAM_CHUNK = int(os.environ.get("NFFT45_STREAM_CHUNK", "64"))
# Smaller host operands (down to this many bytes) take the same pipeline as a
# single chunk, so a call's upload overlaps the previous call's solve and
# download (NFFT45_PIPE_MIN_BYTES overrides, for A/B runs).
PIPE_MIN_BYTES = int(os.environ.get("NFFT45_PIPE_MIN_BYTES", "0"))
# numpy operands: device-side finiteness check; NFFT45_NO_STAGING=1 copies
# pageable memory directly instead of through the pinned staging slots (A/B)
HOST_FLAGS = 1 | (2 if os.environ.get("NFFT45_NO_STAGING") else 0)


def _solve_streamed(name: str, plan: InversePlan, host, passes, dest, non_blocking: bool = False):
    """Pipelined host -> device -> host solve of a [batch, P] (or [P]) CPU tensor
    through the library's native host pipeline (nfft45_solve_host): chunks of
    STREAM_CHUNK signals, H2D / solve / D2H on per-(device, stream) streams that
    persist across calls, so both copy directions stay busy across calls.

    non_blocking (extension, torch's copy_ semantics): return once the copies
    and solves are enqueued; the result in `dest` (pinned) is valid after the
    caller synchronizes the current stream (or the device)."""
    torch = _device.torch
    dev = plan.device
    P = host.shape[-1]
    if dest is None:
        dest = torch.empty(host.shape, dtype=torch.complex128, pin_memory=True)
    src = host if host.dtype == torch.complex128 else host.to(torch.complex128)
    src = src.contiguous()
    rows = src.numel() // P
    kind = 5 if name == "type5" else 4
    _lib.call("nfft45_solve_host", plan.handle, kind, -1 if passes is None else int(passes), src.data_ptr(), rows,
              dest.data_ptr(), STREAM_CHUNK, 0 if non_blocking else 1, _device.stream_handle(dev))
    return dest


def _solve(name: str, plan: InversePlan, data, label: str, passes: int | None, dest=None,
           non_blocking: bool = False):
    torch = _device.torch
    if not isinstance(data, torch.Tensor) and dest is None:
        # the reference's convention (array-like in host memory -> numpy out):
        # validated here, solved through the native host pipeline
        # (the finiteness check of as_complex_vector, grid.py:30-31, runs on the
        # device over the staged chunks: no extra host pass over the operand)
        arr = _device.host_array(data, plan.size, label, check_finite=False)
        res = np.empty_like(arr)
        try:
            _lib.call("nfft45_solve_host_ex", plan.handle, 5 if name == "type5" else 4,
                      -1 if passes is None else int(passes), arr.ctypes.data, arr.size // plan.size,
                      res.ctypes.data, STREAM_CHUNK, 1, HOST_FLAGS, _device.stream_handle(plan.device))
        except ValueError as exc:
            if "NaN or Inf" in str(exc):
                raise ValueError(f"{label} contains NaN or Inf entries") from None
            raise
        return res
    if (isinstance(data, torch.Tensor) and not data.is_cuda and data.dim() in (1, 2) and data.numel() > 0
            and data.shape[-1] == plan.size
            and ((data.dim() == 2 and data.shape[0] > STREAM_CHUNK) or data.numel() * 16 >= PIPE_MIN_BYTES)
            and (dest is None or (not dest.is_cuda and dest.dtype == torch.complex128
                                  and dest.is_contiguous() and dest.shape == data.shape))):
        return _solve_streamed(name, plan, data, passes, dest,
                               non_blocking and dest is not None and dest.is_pinned())
    a = _device.operand(data, plan.device, length=plan.size, name=label)
    if dest is not None and dest.is_cuda and dest.dtype == _device.torch.complex128 and dest.is_contiguous():
        out = dest if dest.shape == a.tensor.shape else dest.reshape(a.tensor.shape)
        dest = None
    else:
        out = a.empty_like_rows(plan.size)
    st = _device.stream_handle(plan.device)
    if passes is None:
        _lib.call(f"nfft45_{name}", plan.handle, a.ptr, a.rows, out.data_ptr(), st)
    else:
        _lib.call(f"nfft45_refine_{name}", plan.handle, a.ptr, a.rows, int(passes), out.data_ptr(), st)
    return a.finish(out, dest, non_blocking)


def type5(plan: InversePlan, samples, flops: FlopCounter | None = None, out=None, non_blocking: bool = False):
    """Coefficients S with sum_p S_p e^{2 pi i p t_q} = samples_q (inverse.py:101-120, Fig. 2).

    `out` (extension): optional preallocated torch tensor (device, or pinned host) for the result.
    `non_blocking` (extension): with CPU torch operands and a pinned `out`, return once the
    work is enqueued (torch copy_ semantics: synchronize before reading `out`)."""
    out = _solve("type5", plan, samples, "samples", None, out, non_blocking)
    _charge_type5(flops, plan.size, plan.kernel_base.taps)
    return out


def type4(plan: InversePlan, spectrum, flops: FlopCounter | None = None, out=None, non_blocking: bool = False):
    """Amplitudes a with sum_q a_q e^{-2 pi i p t_q} = spectrum_p (inverse.py:123-143, Fig. 3)."""
    out = _solve("type4", plan, spectrum, "spectrum", None, out, non_blocking)
    _charge_type4(flops, plan.size, plan.kernel_base.taps)
    return out


def refine_type4(plan: InversePlan, spectrum, passes: int | None = None, flops: FlopCounter | None = None,
                 out=None, non_blocking: bool = False):
    """type4 plus residual-correction passes (inverse.py:165-185, Section V)."""
    if passes is None:
        passes = plan.params.refine_passes
    # a negative count runs no pass, like the reference's range(passes) (inverse.py:150)
    out = _solve("type4", plan, spectrum, "spectrum", max(int(passes), 0), out, non_blocking)
    charge_refine(flops, 4, plan.size, plan.kernel_base.taps, passes)
    return out


def refine_type5(plan: InversePlan, samples, passes: int | None = None, flops: FlopCounter | None = None,
                 out=None, non_blocking: bool = False):
    """type5 plus residual-correction passes in the sample domain (inverse.py:188-202)."""
    if passes is None:
        passes = plan.params.refine_passes
    # a negative count runs no pass, like the reference's range(passes) (inverse.py:150)
    out = _solve("type5", plan, samples, "samples", max(int(passes), 0), out, non_blocking)
    charge_refine(flops, 5, plan.size, plan.kernel_base.taps, passes)
    return out

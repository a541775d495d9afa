"""Operand plumbing: numpy / torch inputs -> device complex128 buffers -> results.

PyTorch supplies device memory and the current stream only; all arithmetic
runs in libnfft45.  Two calling conventions:

* reference-compatible: numpy arrays / sequences in, numpy arrays out (host
  -> device -> host copies around the device call);
* device-resident extension: torch complex128 CUDA tensors in, tensors out on
  the same device and stream, no synchronisation.

1-D operands behave exactly like the reference (as_complex_vector); a 2-D
[batch, n] operand is the batched extension (one signal per row).
"""

from __future__ import annotations

import numpy as np

from .errors import DeviceError, LengthMismatchError

try:
    import torch
except Exception as exc:  # pragma: no cover - torch is part of the image
    raise ImportError("paper_1604_06236_b200 needs PyTorch for device memory") from exc


def device_index(device=None) -> int:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 path has no CPU fallback")
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    return int(device)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(dev: int) -> int:
    """cudaStream_t of the caller's current stream on `dev` (the raw accessor skips
    building a torch.cuda.Stream object: ~4 us of the ~15 us host cost of a small solve)."""
    if _raw_stream is not None:
        return _raw_stream(dev)
    return torch.cuda.current_stream(dev).cuda_stream


class Operand:
    """A validated complex128 operand resident on one device."""

    __slots__ = ("tensor", "is_torch", "host", "batched", "rows", "n")

    def __init__(self, tensor, is_torch: bool, batched: bool, host: bool = False):
        self.tensor = tensor
        self.is_torch = is_torch
        self.host = host  # caller passed a CPU torch tensor: results go back to the host
        self.batched = batched
        self.rows = tensor.shape[0] if batched else 1
        self.n = tensor.shape[-1]

    @property
    def ptr(self) -> int:
        return self.tensor.data_ptr()

    def empty_like_rows(self, n: int):
        shape = (self.rows, n) if self.batched else (n,)
        return torch.empty(shape, dtype=torch.complex128, device=self.tensor.device)

    def finish(self, out, dest=None, non_blocking: bool = False):
        """Return `out` in the caller's convention: numpy in -> numpy out; CUDA
        tensor in -> CUDA tensor out (async); CPU tensor in -> CPU tensor out
        (written into `dest` when given, e.g. a pinned buffer; with
        non_blocking and a pinned dest the copy is only enqueued on the current
        stream — torch copy_ semantics)."""
        if dest is not None:
            dest.copy_(out.reshape(dest.shape), non_blocking=True)
            if not dest.is_cuda and not (non_blocking and dest.is_pinned()):
                torch.cuda.current_stream(out.device).synchronize()
            return dest
        if self.is_torch:
            return out.cpu() if self.host else out
        return out.cpu().numpy()


def operand(values, dev: int, length: int | None = None, name: str = "vector") -> Operand:
    """Coerce `values` to a device complex128 operand with the reference's checks."""
    if isinstance(values, torch.Tensor):
        t = values
        if t.dim() not in (1, 2):
            raise LengthMismatchError(f"{name} must be one- or two-dimensional, got shape {tuple(t.shape)}")
        if t.numel() == 0:
            raise LengthMismatchError(f"{name} must be nonempty")
        if length is not None and t.shape[-1] != length:
            raise LengthMismatchError(f"{name} has length {t.shape[-1]}, expected {length}")
        host = not t.is_cuda
        t = t.to(device=f"cuda:{dev}", dtype=torch.complex128, non_blocking=True).contiguous()
        return Operand(t, True, t.dim() == 2, host)
    arr = host_array(values, length, name)
    t = torch.from_numpy(arr).to(f"cuda:{dev}")
    return Operand(t, False, arr.ndim == 2)


def host_array(values, length: int | None = None, name: str = "vector", check_finite: bool = True) -> np.ndarray:
    """Coerce array-like `values` to a contiguous complex128 numpy array with the
    reference's checks (grid.py:21-32: 1-D, nonempty, finite; [batch, P] allowed).
    check_finite=False leaves the finiteness check to the caller (the host
    pipeline scans the staged chunks on the device)."""
    arr = np.asarray(values, dtype=np.complex128)
    if arr.ndim not in (1, 2):
        raise LengthMismatchError(f"{name} must be one-dimensional, got shape {arr.shape}")
    if arr.size == 0:
        raise LengthMismatchError(f"{name} must be nonempty")
    if length is not None and arr.shape[-1] != length:
        raise LengthMismatchError(f"{name} has length {arr.shape[-1]}, expected {length}")
    if check_finite and not np.isfinite(arr).all():
        raise ValueError(f"{name} contains NaN or Inf entries")
    arr = np.ascontiguousarray(arr)
    if not arr.flags.writeable:
        arr = arr.copy()
    return arr


def real_table(values, dev: int):
    """Real or complex host table -> device complex128 tensor (1-D)."""
    if isinstance(values, torch.Tensor):
        return values.to(device=f"cuda:{dev}", dtype=torch.complex128).contiguous().reshape(-1)
    arr = np.ascontiguousarray(np.asarray(values), dtype=np.complex128).reshape(-1)
    return torch.from_numpy(arr).to(f"cuda:{dev}")

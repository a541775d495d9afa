"""Analytic flop accounting, kept so the ``flops=`` keyword of every transform
behaves as in the reference (flops.py:1-140).

Counts are data-independent integers charged by the Python layer before the
CUDA call is issued: real add/mul 1, complex add 2, complex mul 6, complex
exp (any transcendental) 7, size-N FFT 5 N log2 N.  They describe the
reference algorithm, not the instructions the B200 kernels execute.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

REAL_ADD_FLOPS = 1
COMPLEX_ADD_FLOPS = 2
REAL_MUL_FLOPS = 1
COMPLEX_MUL_FLOPS = 6
COMPLEX_EXP_FLOPS = 7


def fft_flops(size: int) -> float:
    """5 N log2 N for N > 1, else 0."""
    return 5.0 * size * math.log2(size) if size > 1 else 0.0


@dataclass(frozen=True)
class FlopReport:
    real_adds: int = 0
    complex_adds: int = 0
    real_muls: int = 0
    complex_muls: int = 0
    complex_exps: int = 0
    fft_invocations: tuple = ()

    @property
    def total_flops(self) -> int:
        scalar = (self.real_adds * REAL_ADD_FLOPS + self.complex_adds * COMPLEX_ADD_FLOPS
                  + self.real_muls * REAL_MUL_FLOPS + self.complex_muls * COMPLEX_MUL_FLOPS
                  + self.complex_exps * COMPLEX_EXP_FLOPS)
        return scalar + round(sum(fft_flops(n) for n in self.fft_invocations))


class FlopCounter:
    """Accumulator owned by one call tree."""

    _KINDS = ("real_adds", "complex_adds", "real_muls", "complex_muls", "complex_exps")

    def __init__(self):
        for k in self._KINDS:
            setattr(self, k, 0)
        self.fft_sizes: list[int] = []

    def real_add(self, n: int = 1):
        self.real_adds += n

    def complex_add(self, n: int = 1):
        self.complex_adds += n

    def real_mul(self, n: int = 1):
        self.real_muls += n

    def complex_mul(self, n: int = 1):
        self.complex_muls += n

    def complex_exp(self, n: int = 1):
        self.complex_exps += n

    def complex_div(self, n: int = 1):
        """z / w = z conj(w) / |w|^2: one complex mul, five real muls, one real add."""
        self.complex_muls += n
        self.real_muls += 5 * n
        self.real_adds += n

    def fft(self, size: int):
        self.fft_sizes.append(int(size))

    def merge(self, other: "FlopCounter"):
        for k in self._KINDS:
            setattr(self, k, getattr(self, k) + getattr(other, k))
        self.fft_sizes.extend(other.fft_sizes)

    def report(self) -> FlopReport:
        return FlopReport(self.real_adds, self.complex_adds, self.real_muls, self.complex_muls,
                          self.complex_exps, tuple(self.fft_sizes))


def tally(events) -> FlopReport:
    """Fold (kind, arg) events, kind a FlopCounter method name."""
    allowed = {"real_add", "complex_add", "real_mul", "complex_mul", "complex_exp", "complex_div", "fft"}
    c = FlopCounter()
    for kind, arg in events:
        if kind not in allowed:
            raise ValueError(f"unknown flop event kind: {kind!r}")
        getattr(c, kind)(arg)
    return c.report()


# Charges of the reference algorithm, one function per reference call site.

def charge_type1(f: FlopCounter | None, Q: int, R: int, taps: int):
    """forward.py:56-63"""
    if f is None:
        return
    f.complex_exp(Q)
    f.complex_mul(Q)
    f.complex_exp(Q * taps)
    f.real_mul(2 * Q * taps)
    f.complex_add(Q * taps)
    f.fft(2 * R)
    f.real_mul(2 * R)


def charge_type2(f: FlopCounter | None, Q: int, P: int, taps: int):
    """forward.py:94-101"""
    if f is None:
        return
    f.real_mul(2 * P)
    f.fft(2 * P)
    f.complex_exp(Q * taps)
    f.real_mul(2 * Q * taps)
    f.complex_add(Q * taps)
    f.complex_exp(Q)
    f.complex_mul(Q)


def charge_conv_tail(f: FlopCounter | None, R: int, P: int, lam_is_real: bool):
    """forward.py:155-161"""
    if f is None:
        return
    if lam_is_real:
        f.real_mul(2 * R)
    else:
        f.complex_mul(R)
    f.complex_add((R // P - 1) * P)
    f.fft(P)

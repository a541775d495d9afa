"""CPU oracle for the type-1/2/4/5 NFFT hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``nufft1d`` 0.1.0
(arXiv 1604.06236; file:line citations below are into the reference tree
``pkg/src/nufft1d/``).  It exists to CHECK the CUDA product path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
  baseline leg (``--impl reference`` / ``cpu_baseline``) may import it;
* the product package ``paper_1604_06236_b200`` never imports it and has no
  CPU fallback.

Parity pin: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the reference itself (``oracle/make_golden.py``,
which imports the reference in the build container and writes
``tests/golden/*.npz``), including the reference's frozen P=8 fixture.

The arithmetic follows the reference step for step (same numpy primitives in
the same order, 80-bit ``longdouble`` phase reduction), so on the same inputs
the oracle reproduces the reference's outputs to the last bit on the forward
transforms and to its own roundoff level on the ill-conditioned plain solve.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SPREAD_HALF_WIDTH = 14  # grid.py:18
MIN_GAP = 1e-12  # grid.py:17
RE_V_LIMIT = float(np.log(np.finfo(np.float64).max)) - 16.0  # lagrange.py:25-27
DERIVATIVE_FLOOR = 1e-300  # lagrange.py:29


class OracleError(Exception):
    """Base of the oracle's error classes (names mirror errors.py:4-45)."""


class OutOfRange(OracleError):
    pass


class DuplicateNode(OracleError):
    pass


class NonPositiveDamping(OracleError):
    pass


class KernelOverflow(OracleError):
    pass


class SingularDerivative(OracleError):
    pass


class NonConvergence(OracleError):
    pass


# --------------------------------------------------------------------------- grid


def validate(instants, min_gap: float = MIN_GAP):
    """Range / distinctness check; returns (t read-only copy, stable sort order).

    Restates grid.py:64-96.
    """
    t = np.asarray(instants, dtype=np.float64)
    if t.ndim != 1 or t.size == 0 or not np.isfinite(t).all():
        raise OutOfRange("grid must be a nonempty finite 1-D sequence")
    if (t < 0.0).any() or (t >= 1.0).any():
        raise OutOfRange("instant outside [0, 1)")
    order = np.argsort(t, kind="stable")
    if t.size > 1:
        ts = t[order]
        gap = np.empty(t.size)
        gap[:-1] = ts[1:] - ts[:-1]
        gap[-1] = 1.0 - ts[-1] + ts[0]
        if gap.min() < min_gap:
            raise DuplicateNode("circular gap below floor")
    return t.copy(), order


def damping(mu: float, P: int, eta: int) -> float:
    """a from the truncation ratio mu (Eq. 49); restates grid.py:99-113."""
    span = eta * P - 1
    if not (0.0 < mu < 1.0) or span < 1 or mu * span >= 1.0:
        raise NonPositiveDamping("no positive damping for these parameters")
    return -math.log(mu * span) / (2.0 * math.pi * span)


def truncation_ratio(a: float, P: int, eta: int) -> float:
    """mu from the damping a; restates grid.py:116-123."""
    span = eta * P - 1
    if a <= 0.0 or span < 1:
        raise NonPositiveDamping("damping must be positive")
    return math.exp(-2.0 * math.pi * span * a) / span


# ------------------------------------------------------------------------ window


def cis_turns(turns) -> np.ndarray:
    """exp(2 pi i c) with c reduced mod 1 in 80-bit precision (gridding.py:26-29)."""
    f = np.mod(np.asarray(turns, dtype=np.longdouble), 1.0)
    return np.exp(2j * np.pi * f.astype(np.float64))


@dataclass(frozen=True)
class Window:
    """Gaussian gridding window at oversampling 2 (gridding.py:32-98)."""

    R: int
    m: int
    b: float
    n: int
    K: int
    bins: np.ndarray
    deconv: np.ndarray

    @classmethod
    def for_size(cls, R: int, m: int = SPREAD_HALF_WIDTH) -> "Window":
        b = m / (2.0 * np.sqrt(2.0) * np.pi)
        n = 2 * R
        K = R // 2
        nu = np.arange(R) - K
        deconv = np.exp(b * (2.0 * np.pi * nu / n) ** 2) / np.sqrt(4.0 * np.pi * b)
        return cls(R=R, m=m, b=b, n=n, K=K, bins=nu % n, deconv=deconv)

    def taps(self, t):
        """Fine-grid indices and Gaussian weights of every node (gridding.py:57-72)."""
        u = self.n * np.asarray(t, dtype=np.longdouble)
        centre = np.rint(u).astype(np.int64)
        off = np.asarray(u - centre, dtype=np.float64)
        k = np.arange(-self.m, self.m + 1)
        idx = (centre[:, None] + k[None, :]) % self.n
        d = k[None, :] - off[:, None]
        return idx, np.exp(-(d * d) / (4.0 * self.b))


def _idft_unscaled(V):
    """sum_p V_p e^{+2 pi i p q/N}, no 1/N (forward.py:21-23)."""
    return np.conj(np.fft.fft(np.conj(V)))


# ----------------------------------------------------------------------- forward


def type1(t, amps, R: int, m: int = SPREAD_HALF_WIDTH, win: Window | None = None):
    """A_p = sum_q a_q e^{-2 pi i p t_q}, p < R, by gridding (forward.py:26-64)."""
    w = win or Window.for_size(R, m)
    a = np.asarray(amps, dtype=np.complex128)
    tl = np.asarray(t, dtype=np.longdouble)
    shifted = a * cis_turns(-w.K * tl)
    idx, wt = w.taps(t)
    contrib = (shifted[:, None] * wt).ravel()
    flat = idx.ravel()
    grid = np.bincount(flat, weights=contrib.real, minlength=w.n) + 1j * np.bincount(
        flat, weights=contrib.imag, minlength=w.n
    )
    return np.fft.fft(grid)[w.bins] * w.deconv


def type2(S, t, m: int = SPREAD_HALF_WIDTH, win: Window | None = None):
    """s(t_q) = sum_p S_p e^{+2 pi i p t_q}, by windowed gather (forward.py:67-102)."""
    coef = np.asarray(S, dtype=np.complex128)
    w = win or Window.for_size(coef.size, m)
    F = np.zeros(w.n, dtype=np.complex128)
    F[w.bins] = coef * w.deconv
    y = _idft_unscaled(F)
    idx, wt = w.taps(t)
    vals = np.einsum("qj,qj->q", wt, y[idx])
    return vals * cis_turns(w.K * np.asarray(t, dtype=np.longdouble))


def type1_exact(t, amps, R: int):
    """O(RQ) direct sum with 80-bit phases (forward.py:105-118)."""
    a = np.asarray(amps, dtype=np.complex128)
    tl = np.asarray(t, dtype=np.longdouble)
    out = np.empty(R, dtype=np.complex128)
    for lo in range(0, R, 256):
        p = np.arange(lo, min(lo + 256, R), dtype=np.longdouble)
        out[lo : lo + p.size] = cis_turns(-np.outer(p, tl)) @ a
    return out


def type2_exact(S, t):
    """O(PQ) direct sum with 80-bit phases (forward.py:121-130)."""
    coef = np.asarray(S, dtype=np.complex128)
    p = np.arange(coef.size, dtype=np.longdouble)
    tl = np.asarray(t, dtype=np.longdouble)
    out = np.empty(tl.size, dtype=np.complex128)
    for lo in range(0, tl.size, 256):
        blk = tl[lo : lo + 256]
        out[lo : lo + blk.size] = cis_turns(np.outer(blk, p)) @ coef
    return out


def conv(t, amps, lam, P: int, m: int = SPREAD_HALF_WIDTH, win: Window | None = None):
    """Nonuniform convolution onto {q/P}: type-1 of length R, fold, IDFT_P (forward.py:133-162)."""
    lam = np.asarray(lam)
    R = lam.size
    if R % P:
        raise ValueError("kernel length must be a multiple of P")
    prod = lam * type1(t, amps, R, m, win)
    if R // P > 1:
        prod = prod.reshape(R // P, P).sum(axis=0)
    return _idft_unscaled(prod.astype(np.complex128, copy=False))


# ---------------------------------------------------------------------- Lagrange


def log_series(a: float, R: int):
    """Lambda_0 = 0, Lambda_p = -e^{-2 pi p a}/p (lagrange.py:42-54)."""
    lam = np.zeros(R)
    p = np.arange(1, R)
    lam[1:] = -np.exp(-2.0 * np.pi * p * a) / p
    return lam


def v_samples(t, a: float, eta: int, m: int = SPREAD_HALF_WIDTH):
    """v(q/P) via one nonuniform convolution of the log series (lagrange.py:57-75)."""
    P = len(t)
    R = eta * P
    return conv(t, np.ones(P, dtype=np.complex128), log_series(a, R), P, m)


def v_samples_terms(t, a: float, R: int, m: int = SPREAD_HALF_WIDTH):
    """EXTENSION, not in the reference (which requires R = eta P with integer
    eta, grid.py:143-144, forward.py:149-154): v with R log-series terms for
    any R >= 2.  Same steps as v_samples / conv (forward.py:133-162) except
    that the fold onto P zero-pads the product to a whole number of slices
    (a fractional oversampling factor eta = R / P, BASELINE config 5)."""
    P = len(t)
    lam = log_series(a, R)
    prod = lam * type1(t, np.ones(P, dtype=np.complex128), R, m)
    nsl = -(-R // P)
    if nsl > 1 or R % P:
        prod = np.concatenate([prod, np.zeros(nsl * P - R, dtype=prod.dtype)]).reshape(nsl, P).sum(axis=0)
    return _idft_unscaled(prod.astype(np.complex128, copy=False))


def kernel_samples(v, t):
    """exp(i pi P + 2 pi i sum t + v), with the overflow guard (lagrange.py:78-97)."""
    v = np.asarray(v, dtype=np.complex128)
    if float(np.abs(v.real).max()) > RE_V_LIMIT:
        raise KernelOverflow("|Re v| beyond the exp() margin")
    P = len(t)
    return np.exp(1j * np.pi * P + 2j * np.pi * float(np.sum(t)) + v)


def kernel_coeffs(ks, a: float):
    """L_0..L_{P-1} from the damped samples, Eq. 43 (lagrange.py:100-134)."""
    ks = np.asarray(ks, dtype=np.complex128)
    P = ks.size
    up = np.exp(2.0 * np.pi * np.arange(P) * a)
    spec = np.fft.fft(ks)
    spec[0] -= P * np.exp(-2.0 * np.pi * P * a)
    return spec * (up / P)


def derivative(L, t, m: int = SPREAD_HALF_WIDTH):
    """L'(e^{2 pi i t_p}) by a type-2 of (k+1) L_{k+1}, L_P = 1 (lagrange.py:137-164)."""
    L = np.asarray(L, dtype=np.complex128)
    P = L.size
    d = np.empty(P, dtype=np.complex128)
    d[: P - 1] = np.arange(1, P) * L[1:]
    d[P - 1] = P
    out = type2(d, t, m)
    if float(np.abs(out).min()) < DERIVATIVE_FLOOR:
        raise SingularDerivative("derivative sample vanished")
    return out


# ------------------------------------------------------------------------- plan


@dataclass
class Plan:
    """Grid-only tables of the inverse (inverse.py:33-98)."""

    t: np.ndarray
    a: float
    eta: int
    m: int
    v: np.ndarray
    ks: np.ndarray
    L: np.ndarray
    dL: np.ndarray
    node_weights: np.ndarray
    decay: np.ndarray
    coef_scale: np.ndarray

    @property
    def P(self) -> int:
        return self.t.size

    @classmethod
    def build(cls, t, a: float, eta: int = 2, m: int = SPREAD_HALF_WIDTH) -> "Plan":
        """eta integer: the reference's build_plan.  eta fractional (eta * P an
        integer): the extension of v_samples_terms."""
        t = np.asarray(t, dtype=np.float64)
        P = t.size
        if float(eta) == int(eta):
            v = v_samples(t, a, int(eta), m)
        else:
            v = v_samples_terms(t, a, int(round(eta * P)), m)
        ks = kernel_samples(v, t)
        L = kernel_coeffs(ks, a)
        dL = derivative(L, t, m)
        decay = np.exp(-2.0 * np.pi * np.arange(P) * a)
        coef_scale = (1.0 / decay) / P
        tl = np.asarray(t, dtype=np.longdouble)
        h = 1.0 / (cis_turns(-P * tl) * np.exp(-2.0 * np.pi * P * a) - 1.0)
        nw = h / (dL * cis_turns(tl))
        return cls(t, a, eta, m, v, ks, L, dL, nw, decay, coef_scale)


def solve5(plan: Plan, samples):
    """Coefficients from samples at the nodes, Fig. 2 (inverse.py:101-120)."""
    s = np.asarray(samples, dtype=np.complex128)
    u = conv(plan.t, s * plan.node_weights, plan.decay, plan.P, plan.m)
    return np.fft.fft(plan.ks * u) * plan.coef_scale


def solve4(plan: Plan, spectrum):
    """Amplitudes from uniform spectrum samples, Fig. 3 (inverse.py:123-143)."""
    A = np.asarray(spectrum, dtype=np.complex128)
    u = _idft_unscaled(plan.decay * A)
    S = np.fft.fft(plan.ks * u) * plan.coef_scale
    return type2(S, plan.t, plan.m) * plan.node_weights


def _residual_loop(plan, data, passes, solve, fwd):
    """Section V refinement (inverse.py:146-162)."""
    x = solve(plan, data)
    last = None
    for _ in range(passes):
        r = fwd(x) - data
        nrm = float(np.linalg.norm(r))
        if last is not None and nrm > last:
            raise NonConvergence("residual norm grew between passes")
        last = nrm
        x = x - solve(plan, r)
    return x


def refine5(plan: Plan, samples, passes: int = 1):
    """type5 + residual passes in the sample domain (inverse.py:188-202)."""
    s = np.asarray(samples, dtype=np.complex128)
    return _residual_loop(plan, s, passes, solve5, lambda x: type2(x, plan.t, plan.m))


def refine4(plan: Plan, spectrum, passes: int = 1):
    """type4 + residual passes in the spectrum domain (inverse.py:165-185)."""
    A = np.asarray(spectrum, dtype=np.complex128)
    return _residual_loop(plan, A, passes, solve4, lambda x: type1(plan.t, x, plan.P, plan.m))


# ---------------------------------------------------------------------- inputs


# ------------------------------------------------------------ baselines

def cg(t, b, which: str = "type4", tol: float = 1e-15, max_iter: int | None = None):
    """CGNR, unpreconditioned (baselines.py:116-181): per iteration one
    forward and one adjoint fast NFFT; stops at ||r|| <= tol ||b||.
    Returns (x, iterations, converged, relative_residual)."""
    if tol <= 0.0:
        raise ValueError("tolerance must be positive")
    if which not in ("type4", "type5"):
        raise ValueError(f"unknown system kind {which!r}")
    b = np.asarray(b, dtype=np.complex128)
    P = b.size
    if max_iter is None:
        max_iter = 4 * P
    if which == "type4":
        apply_A = lambda x: type1(t, x, P)
        apply_AH = lambda y: type2(y, t)
    else:
        apply_A = lambda x: type2(x, t)
        apply_AH = lambda y: type1(t, y, P)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return np.zeros(P, dtype=np.complex128), 0, True, 0.0
    x = np.zeros(P, dtype=np.complex128)
    r = b.copy()
    z = apply_AH(r)
    p = z.copy()
    zz = float(np.vdot(z, z).real)
    rnorm = bnorm
    iterations = 0
    for iterations in range(1, max_iter + 1):
        w = apply_A(p)
        ww = float(np.vdot(w, w).real)
        if ww == 0.0:
            iterations -= 1
            break
        alpha = zz / ww
        x = x + alpha * p
        r = r - alpha * w
        rnorm = float(np.linalg.norm(r))
        if rnorm <= tol * bnorm:
            return x, iterations, True, rnorm / bnorm
        z = apply_AH(r)
        zz_new = float(np.vdot(z, z).real)
        p = z + (zz_new / zz) * p
        zz = zz_new
    return x, iterations, rnorm <= tol * bnorm, rnorm / bnorm


def phase_matrix(t, sign: int):
    """e^{sign 2 pi i p t_q}, rows p, columns q (baselines.py:37-49)."""
    P = len(t)
    tt = np.asarray(t, dtype=np.longdouble)
    return cis_turns(sign * np.outer(np.arange(P, dtype=np.longdouble), tt))


def dense_solve(matrix, rhs):
    """Dense LU solve standing in for ge_solve (baselines.py:64-105)."""
    return np.linalg.solve(np.asarray(matrix, dtype=np.complex128), np.asarray(rhs, dtype=np.complex128))


def make_inputs(P: int, jitter: float, batch: int, seed: int):
    """Seeded benchmark inputs (generator as bench.py:84-92).

    Nodes t_p = ((p + u_p)/P) mod 1 with u ~ U[-jitter, jitter]; data circular
    CN(0,1) = (N + iN)/sqrt(2), shape [batch, P], drawn after the nodes from the
    same Philox stream.
    """
    rng = np.random.Generator(np.random.Philox(key=seed))
    u = rng.uniform(-jitter, jitter, P)
    t = np.mod((np.arange(P) + u) / P, 1.0)
    t[t >= 1.0] = 0.0  # mod can round up to 1.0 for tiny negative inputs
    re = rng.standard_normal((batch, P))
    im = rng.standard_normal((batch, P))
    data = (re + 1j * im) / np.sqrt(2.0)
    return t, data


def rel_l2(truth, got) -> float:
    truth = np.asarray(truth)
    return float(np.linalg.norm(np.asarray(got) - truth) / np.linalg.norm(truth))

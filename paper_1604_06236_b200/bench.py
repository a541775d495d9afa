"""Monte-Carlo harness of the paper's figure protocols on the GPU
(reference bench.py:1-301).

Same protocol and API as the reference: each trial draws a jittered regular
grid and CN(0, 1) amplitudes from Philox(key = seed ^ trial); the spectrum
handed to every solver is the EXACT direct sum (here the direct-sum kernel),
never the fast transform; errors are relative l2, linear and 20 log10 dB;
GE / CG run once per trial, the fast methods once per feasible (eta, mu)
sharing one plan between the plain and refined solves; infeasible mu and
non-contracting multi-pass cells are skipped.  What changes is where it
runs: the trial's grid, spectrum, truth and every solve stay on the device
(torch CUDA tensors), so a full figure sweep costs seconds instead of hours.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, replace

import numpy as np
import torch

from .baselines import cg_solve, ge_solve, type4_system
from .errors import AmplificationWarning, NonConvergenceError, NonPositiveDampingError, ZeroReferenceError
from .flops import FlopCounter
from .forward import nfft_type1_direct
from .grid import MethodParams
from .inverse import build_plan, refine_type4, type4
from .metrics import generate_trial, relative_error

GE_SIZE_CAP = 8192
MU_SWEEP_DEFAULT = tuple(float(m) for m in np.logspace(-18.0, -4.0, 29))

METHOD_GE = "GE"
METHOD_CG = "CG"
METHOD_NFFT = "NFFT"
METHOD_RNFFT = "R-NFFT"
ALL_METHODS = (METHOD_GE, METHOD_CG, METHOD_NFFT, METHOD_RNFFT)


@dataclass(frozen=True)
class TrialConfig:
    """One sweep specification (bench.py:45-66). Scalar fields accept tuples to sweep."""

    p: tuple[int, ...] = (1024,)
    eta: tuple[int, ...] = (1,)
    mu: tuple[float, ...] = MU_SWEEP_DEFAULT
    trials: int = 10
    seed: int = 0
    methods: tuple[str, ...] = ALL_METHODS
    jitter_max: float = 0.6
    spread_width: int = 14
    refine_passes: int = 1
    cg_tol: float = 1e-15

    def __post_init__(self):
        if not 0.0 <= self.jitter_max < 1.0:
            raise ValueError("jitter_max must lie in [0, 1) to keep nodes distinct")
        for m in self.methods:
            if m not in ALL_METHODS:
                raise ValueError(f"unknown method {m!r}")


@dataclass(frozen=True)
class TrialResult:
    p: int
    eta: int | None
    mu: float | None
    method: str
    trial: int
    error_linear: float
    error_db: float
    total_flops: int
    cg_iterations: int | None
    seed: int


def to_db(error_linear: float) -> float:
    return float("-inf") if error_linear <= 0.0 else 20.0 * math.log10(error_linear)


def _device_error(truth: torch.Tensor, est) -> float:
    """relative_error on device tensors (one scalar read back)."""
    est = torch.as_tensor(est, device=truth.device) if not isinstance(est, torch.Tensor) else est
    tn = float(torch.linalg.vector_norm(truth))
    if tn == 0.0:
        raise ZeroReferenceError("relative error undefined: reference vector is zero")
    return float(torch.linalg.vector_norm(truth - est.to(truth.device))) / tn


def _row(p, eta, mu, method, trial, err, counter, cg_iters, seed) -> TrialResult:
    return TrialResult(p, eta, mu, method, trial, err, to_db(err), counter.report().total_flops, cg_iters, seed)


def run_sweep(config: TrialConfig) -> list[TrialResult]:
    """Every (P, trial, method, eta, mu) combination of the config (bench.py:127-214)."""
    out: list[TrialResult] = []
    if METHOD_GE in config.methods and max(config.p) > GE_SIZE_CAP:
        raise ValueError(f"GE requested above the P = {GE_SIZE_CAP} dense-solver cap")
    fast = [m for m in (METHOD_NFFT, METHOD_RNFFT) if m in config.methods]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", AmplificationWarning)
        for P in config.p:
            for trial in range(config.trials):
                tseed = config.seed ^ trial
                grid, a_np = generate_trial(P, tseed, config.jitter_max)
                truth = torch.from_numpy(a_np).cuda()
                spectrum = nfft_type1_direct(grid, truth, P)  # exact, on the device
                if METHOD_GE in config.methods:
                    c = FlopCounter()
                    x = ge_solve(type4_system(grid, spectrum.cpu().numpy(), flops=c), flops=c)
                    out.append(_row(P, None, None, METHOD_GE, trial, relative_error(a_np, x), c, None, tseed))
                if METHOD_CG in config.methods:
                    c = FlopCounter()
                    res = cg_solve(grid, spectrum, "type4", tol=config.cg_tol, spread_width=config.spread_width,
                                   flops=c)
                    out.append(_row(P, None, None, METHOD_CG, trial, _device_error(truth, res.solution), c,
                                    res.iterations, tseed))
                if not fast:
                    continue
                for eta in config.eta:
                    for mu in config.mu:
                        try:
                            params = MethodParams.from_mu(mu, P, eta, spread_width=config.spread_width,
                                                          refine_passes=config.refine_passes)
                        except NonPositiveDampingError:
                            continue
                        pc = FlopCounter()
                        plan = build_plan(grid, params, flops=pc)
                        if METHOD_NFFT in config.methods:
                            c = FlopCounter()
                            c.merge(pc)
                            x = type4(plan, spectrum, flops=c)
                            out.append(_row(P, eta, mu, METHOD_NFFT, trial, _device_error(truth, x), c, None,
                                            tseed))
                        if METHOD_RNFFT in config.methods:
                            c = FlopCounter()
                            c.merge(pc)
                            try:
                                x = refine_type4(plan, spectrum, passes=config.refine_passes, flops=c)
                            except NonConvergenceError:
                                continue
                            out.append(_row(P, eta, mu, METHOD_RNFFT, trial, _device_error(truth, x), c, None,
                                            tseed))
    return out


def best_mu(results: list[TrialResult], method: str) -> dict[tuple[int, int], float]:
    """Per-(P, eta) mu minimising the mean error over trials (bench.py:217-231)."""
    groups: dict[tuple[int, int, float], list[float]] = {}
    for r in results:
        if r.method == method and r.mu is not None:
            groups.setdefault((r.p, r.eta, r.mu), []).append(r.error_linear)
    best: dict[tuple[int, int], tuple[float, float]] = {}
    for (p, eta, mu), errs in groups.items():
        mean = sum(errs) / len(errs)
        if (p, eta) not in best or mean < best[(p, eta)][0]:
            best[(p, eta)] = (mean, mu)
    return {k: mu for k, (_, mu) in best.items()}


def filter_best_mu(results: list[TrialResult], method: str) -> list[TrialResult]:
    """Dense-solver rows plus the best-mu rows of `method` (bench.py:234-243)."""
    winners = best_mu(results, method)
    return [r for r in results
            if r.mu is None or (r.method == method and winners.get((r.p, r.eta)) == r.mu)]


# fig1: error floor vs mu for several eta at P = 1024; fig2: the refined
# method; fig3: refined method vs P at best mu; fig6: flop totals vs P;
# fig7: flop totals vs eta (bench.py:246-275).
FIGURE_DEFAULTS: dict[str, TrialConfig] = {
    "fig1": TrialConfig(p=(1024,), eta=(1, 2, 3, 4, 6, 15, 20), methods=(METHOD_GE, METHOD_CG, METHOD_NFFT)),
    "fig2": TrialConfig(p=(1024,), eta=(1, 2), methods=(METHOD_GE, METHOD_CG, METHOD_RNFFT)),
    "fig3": TrialConfig(p=(64, 128, 256, 512, 1024, 2048, 4096, 8192), eta=(1,),
                        methods=(METHOD_GE, METHOD_CG, METHOD_RNFFT)),
    "fig6": TrialConfig(p=(64, 128, 256, 512, 1024), eta=(6,), mu=(1e-15,),
                        methods=(METHOD_GE, METHOD_CG, METHOD_NFFT)),
    "fig7": TrialConfig(p=(1024,), eta=tuple(range(1, 21)), mu=(1e-15,), methods=(METHOD_GE, METHOD_CG, METHOD_NFFT)),
}

DENSE_DEFAULT_CAP = 1024


def run_figure(name: str, config: TrialConfig | None = None, dense_cap: int | None = None):
    """One figure protocol -> (records, metadata) (bench.py:282-301)."""
    if name not in FIGURE_DEFAULTS:
        raise ValueError(f"unknown figure {name!r}; choose from {sorted(FIGURE_DEFAULTS)}")
    cfg = config if config is not None else FIGURE_DEFAULTS[name]
    cap = DENSE_DEFAULT_CAP if dense_cap is None else dense_cap
    dense = tuple(m for m in cfg.methods if m in (METHOD_GE, METHOD_CG))
    fast_only = tuple(m for m in cfg.methods if m not in (METHOD_GE, METHOD_CG))
    results: list[TrialResult] = []
    for P in cfg.p:
        methods = cfg.methods if P <= cap else fast_only
        if methods:
            results.extend(run_sweep(replace(cfg, p=(P,), methods=methods)))
    if name == "fig6":  # + the refined method at eta = 1 on the same trials
        results.extend(run_sweep(replace(cfg, eta=(1,), mu=(1e-8,), methods=(METHOD_RNFFT,), p=tuple(cfg.p))))
    if name in ("fig2", "fig3"):
        results = filter_best_mu(results, METHOD_RNFFT)
    meta = {
        "figure": name,
        "seed": cfg.seed,
        "trials": cfg.trials,
        "jitter_max": cfg.jitter_max,
        "db_convention": "20*log10(relative_l2_error)",
        "rng": "philox(key=seed^trial)",
        "dense_cap": cap if dense else None,
    }
    return results, meta

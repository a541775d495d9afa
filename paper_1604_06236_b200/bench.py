"""GPU-first Monte-Carlo harness for the paper's figure protocols
(reference bench.py:38-301).

Public API and record semantics are the reference's (TrialConfig,
TrialResult, run_sweep, best_mu, filter_best_mu, FIGURE_DEFAULTS,
run_figure): a trial's grid and truth come from Philox(key = seed ^ trial)
(metrics.trial_arrays, bit-identical to the reference's streams), the
spectrum handed to every solver is the EXACT direct sum, errors are relative
l2 (linear and 20 log10 dB), infeasible mu and non-contracting multi-pass
cells produce no record, and the records come out in the reference's order.

The execution is organised for the device instead of as a trial loop:

1. all trials of one size P are drawn up front; their nodes, truths and
   direct-sum spectra live on the GPU for the whole size;
2. the parameter-free dense solvers (device GE, device CGNR) run per trial;
3. the fast methods run CELL-MAJOR: for each feasible (eta, mu) cell the
   plans of all trials are built and the plain and refined solves launched
   back to back; their relative errors are reduced on the device into one
   [cells, trials, 2] tensor, read back once per size;
4. flop totals are charged once per (P, cell, method) — the reference's
   model is data independent (flops.py) — except CG, whose charge depends
   on its iteration count.
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
from .grid import MethodParams, validate_grid
from .inverse import build_plan, charge_plan, charge_refine, charge_type4, refine_type4, type4
from .metrics import generate_trial, relative_error, trial_arrays  # noqa: F401  (re-exported API)

GE_SIZE_CAP = 8192
MU_SWEEP_DEFAULT = tuple(float(v) for v in 10.0 ** np.linspace(-18.0, -4.0, 29))

METHOD_GE, METHOD_CG, METHOD_NFFT, METHOD_RNFFT = "GE", "CG", "NFFT", "R-NFFT"
ALL_METHODS = (METHOD_GE, METHOD_CG, METHOD_NFFT, METHOD_RNFFT)
_DENSE = (METHOD_GE, METHOD_CG)
_FAST = (METHOD_NFFT, METHOD_RNFFT)


@dataclass(frozen=True)
class TrialConfig:
    """A sweep: every size p, trial, method and (eta, mu) cell (reference bench.py:45-67)."""

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
        bad = [m for m in self.methods if m not in ALL_METHODS]
        if bad:
            raise ValueError(f"unknown method {bad[0]!r}")


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
    """20 log10 of a linear error (-inf for an exact result)."""
    return 20.0 * math.log10(error_linear) if error_linear > 0.0 else float("-inf")


class _Size:
    """Every trial of one size P, resident on the device."""

    def __init__(self, P: int, cfg: TrialConfig):
        self.P = P
        self.seeds = [cfg.seed ^ k for k in range(cfg.trials)]
        self.grids, truths = [], []
        for s in self.seeds:
            nodes, amp = trial_arrays(P, s, cfg.jitter_max)
            self.grids.append(validate_grid(nodes))
            truths.append(amp)
        self.truth = torch.from_numpy(np.stack(truths)).cuda()          # [trials, P]
        self.truth_norm = torch.linalg.vector_norm(self.truth, dim=1)  # [trials]
        # exact spectra A_p = sum_q a_q e^{-2 pi i p t_q} (direct-sum kernel, one launch per grid)
        self.spectrum = torch.stack([nfft_type1_direct(g, self.truth[k], P) for k, g in enumerate(self.grids)])

    def errors(self, k: int, x) -> torch.Tensor:
        """Device scalar ||truth_k - x|| / ||truth_k||."""
        x = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x))
        return torch.linalg.vector_norm(self.truth[k] - x.to(self.truth.device)) / self.truth_norm[k]


def _charged(fn) -> int:
    c = FlopCounter()
    fn(c)
    return c.report().total_flops


def _fast_cells(size: _Size, cfg: TrialConfig, want_plain: bool, want_refined: bool):
    """Cell-major fast methods: (cells, errors [cells, trials, 2] on the host, ok mask, flops)."""
    P, T = size.P, len(size.seeds)
    cells = []
    for eta in cfg.eta:
        for mu in cfg.mu:
            try:
                params = MethodParams.from_mu(mu, P, eta, spread_width=cfg.spread_width,
                                              refine_passes=cfg.refine_passes)
            except NonPositiveDampingError:
                continue  # no damping needed at this truncation: the reference records nothing
            cells.append((eta, mu, params))
    err = torch.full((len(cells), T, 2), float("nan"), dtype=torch.float64, device=size.truth.device)
    ok = np.zeros((len(cells), T, 2), dtype=bool)
    flops = {}
    for ci, (eta, mu, params) in enumerate(cells):
        taps = 2 * params.spread_width + 1
        plan_flops = _charged(lambda c: charge_plan(c, P, params))
        flops[("nfft", ci)] = plan_flops + _charged(lambda c: charge_type4(c, P, taps))
        flops[("rnfft", ci)] = plan_flops + _charged(lambda c: charge_refine(c, 4, P, taps, cfg.refine_passes))
        for k, grid in enumerate(size.grids):
            plan = build_plan(grid, params)
            if want_plain:
                err[ci, k, 0] = size.errors(k, type4(plan, size.spectrum[k]))
                ok[ci, k, 0] = True
            if want_refined:
                try:
                    x = refine_type4(plan, size.spectrum[k], passes=cfg.refine_passes)
                except NonConvergenceError:
                    continue  # residual grew between passes: no record (reference bench.py:196-199)
                err[ci, k, 1] = size.errors(k, x)
                ok[ci, k, 1] = True
    return cells, err.cpu().numpy(), ok, flops


def run_sweep(config: TrialConfig) -> list[TrialResult]:
    """Every (P, trial, method, eta, mu) record of the config, in the reference's order
    (per P, per trial: GE, CG, then per (eta, mu): NFFT, R-NFFT)."""
    if METHOD_GE in config.methods and max(config.p) > GE_SIZE_CAP:
        raise ValueError(f"GE requested above the P = {GE_SIZE_CAP} dense-solver cap")
    want_plain, want_refined = METHOD_NFFT in config.methods, METHOD_RNFFT in config.methods
    records: list[TrialResult] = []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", AmplificationWarning)
        for P in config.p:
            size = _Size(P, config)
            if float(size.truth_norm.min()) == 0.0:
                raise ZeroReferenceError("relative error undefined: reference vector is zero")
            dense = {}
            for k, grid in enumerate(size.grids):
                if METHOD_GE in config.methods:
                    c = FlopCounter()
                    x = ge_solve(type4_system(grid, size.spectrum[k].cpu().numpy(), flops=c), flops=c)
                    dense[(k, METHOD_GE)] = (size.errors(k, x), c.report().total_flops, None)
                if METHOD_CG in config.methods:
                    c = FlopCounter()
                    res = cg_solve(grid, size.spectrum[k], "type4", tol=config.cg_tol,
                                   spread_width=config.spread_width, flops=c)
                    dense[(k, METHOD_CG)] = (size.errors(k, res.solution), c.report().total_flops, res.iterations)
            cells, err, ok, flops = ([], None, None, {})
            if want_plain or want_refined:
                cells, err, ok, flops = _fast_cells(size, config, want_plain, want_refined)
            # one read-back of the dense errors, then the records in the reference's order
            dense_err = {key: float(v[0]) for key, v in dense.items()}
            for k, seed in enumerate(size.seeds):
                for m in _DENSE:
                    if (k, m) in dense:
                        e = dense_err[(k, m)]
                        records.append(TrialResult(P, None, None, m, k, e, to_db(e), dense[(k, m)][1],
                                                   dense[(k, m)][2], seed))
                for ci, (eta, mu, _) in enumerate(cells):
                    for slot, m, fk in ((0, METHOD_NFFT, "nfft"), (1, METHOD_RNFFT, "rnfft")):
                        if ok[ci, k, slot]:
                            e = float(err[ci, k, slot])
                            records.append(TrialResult(P, eta, mu, m, k, e, to_db(e), flops[(fk, ci)], None, seed))
    return records


def best_mu(results: list[TrialResult], method: str) -> dict[tuple[int, int], float]:
    """Per-(P, eta) mu with the smallest mean error over trials (reference bench.py:217-231);
    ties keep the first mu met."""
    by_cell: dict[tuple[int, int], dict[float, list[float]]] = {}
    for r in results:
        if r.method == method and r.mu is not None:
            by_cell.setdefault((r.p, r.eta), {}).setdefault(r.mu, []).append(r.error_linear)
    winners = {}
    for key, per_mu in by_cell.items():
        means = [(sum(v) / len(v), mu) for mu, v in per_mu.items()]
        best = means[0]
        for cand in means[1:]:
            if cand[0] < best[0]:
                best = cand
        winners[key] = best[1]
    return winners


def filter_best_mu(results: list[TrialResult], method: str) -> list[TrialResult]:
    """Dense-solver records plus `method`'s records at its best mu (reference bench.py:234-243)."""
    winners = best_mu(results, method)
    return [r for r in results if r.mu is None or (r.method == method and winners.get((r.p, r.eta)) == r.mu)]


# Figure protocols (reference bench.py:246-275): fig1 error floor vs mu at
# several eta (P = 1024); fig2 the refined method at eta 1, 2; fig3 refined
# method vs P at its best mu; fig6 flops vs P; fig7 flops vs eta.
_FIG_DENSE_NFFT = (METHOD_GE, METHOD_CG, METHOD_NFFT)
_FIG_DENSE_RNFFT = (METHOD_GE, METHOD_CG, METHOD_RNFFT)
FIGURE_DEFAULTS: dict[str, TrialConfig] = {
    "fig1": TrialConfig(p=(1024,), eta=(1, 2, 3, 4, 6, 15, 20), methods=_FIG_DENSE_NFFT),
    "fig2": TrialConfig(p=(1024,), eta=(1, 2), methods=_FIG_DENSE_RNFFT),
    "fig3": TrialConfig(p=tuple(64 << k for k in range(8)), eta=(1,), methods=_FIG_DENSE_RNFFT),
    "fig6": TrialConfig(p=tuple(64 << k for k in range(5)), eta=(6,), mu=(1e-15,), methods=_FIG_DENSE_NFFT),
    "fig7": TrialConfig(p=(1024,), eta=tuple(range(1, 21)), mu=(1e-15,), methods=_FIG_DENSE_NFFT),
}
DENSE_DEFAULT_CAP = 1024


def run_figure(name: str, config: TrialConfig | None = None, dense_cap: int | None = None):
    """(records, metadata) of one figure protocol (reference bench.py:282-301): dense
    solvers only up to `dense_cap`; fig6 adds the refined method at eta = 1, mu = 1e-8;
    fig2 / fig3 keep the refined method's best-mu records."""
    if name not in FIGURE_DEFAULTS:
        raise ValueError(f"unknown figure {name!r}; choose from {sorted(FIGURE_DEFAULTS)}")
    cfg = FIGURE_DEFAULTS[name] if config is None else config
    cap = DENSE_DEFAULT_CAP if dense_cap is None else dense_cap
    fast_only = tuple(m for m in cfg.methods if m not in _DENSE)
    records: list[TrialResult] = []
    for P in cfg.p:
        methods = cfg.methods if P <= cap else fast_only
        if methods:
            records += run_sweep(replace(cfg, p=(P,), methods=methods))
    if name == "fig6":
        records += run_sweep(replace(cfg, eta=(1,), mu=(1e-8,), methods=(METHOD_RNFFT,)))
    if name in ("fig2", "fig3"):
        records = filter_best_mu(records, METHOD_RNFFT)
    has_dense = any(m in _DENSE for m in cfg.methods)
    meta = {"figure": name, "seed": cfg.seed, "trials": cfg.trials, "jitter_max": cfg.jitter_max,
            "db_convention": "20*log10(relative_l2_error)", "rng": "philox(key=seed^trial)",
            "dense_cap": cap if has_dense else None}
    return records, meta

#!/usr/bin/env python
"""BASELINE config 5: parameter and conditioning sweep at P = 2^18, one
signal of complex128 Gaussian data.  Node jitter J in {0.1, 0.3, 0.45},
oversampling eta in {1.5, 2, 3}, attenuation mu in {1e-17 .. 1e-13} around
the reference default 1e-15.  Per case: plan time, refined (passes = 1)
type-5 + type-4 throughput (CUDA events, device-resident), error vs the CPU
oracle (integer eta; eta = 1.5 is the extension, no reference exists), error
vs truth built by construction (samples = fast type-2 of a known spectrum,
spectrum = fast type-1 of known amplitudes) and forward residuals.
Writes profiles/c5_sweep.json and prints a markdown table."""
import json
import math
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import paper_1604_06236_b200 as nf  # noqa: E402
from oracle import nfft_oracle as O  # noqa: E402

P = 1 << 18
rows = []
for J in (0.1, 0.3, 0.45):
    t, data = O.make_inputs(P, J, 1, 16045)
    grid = nf.validate_grid(t)
    rng = np.random.default_rng(16045)
    S_true = (rng.standard_normal(P) + 1j * rng.standard_normal(P)) / math.sqrt(2)
    a_true = (rng.standard_normal(P) + 1j * rng.standard_normal(P)) / math.sqrt(2)
    s_syn = nf.nfft_type2(S_true, grid)
    A_syn = nf.nfft_type1(grid, a_true, P)
    x = data[0]
    for eta in (1.5, 2, 3):
        for mu in (1e-17, 1e-16, 1e-15, 1e-14, 1e-13):
            frac = float(eta) != int(eta)
            prm = nf.MethodParams.from_mu(mu, P, eta, fractional_eta=frac)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan = nf.build_plan(grid, prm, device=0)
            torch.cuda.synchronize()
            plan_ms = 1e3 * (time.perf_counter() - t0)
            xd = torch.from_numpy(x).cuda()
            o5, o4 = torch.empty_like(xd), torch.empty_like(xd)
            for _ in range(3):
                nf.refine_type5(plan, xd, passes=1, out=o5)
                nf.refine_type4(plan, xd, passes=1, out=o4)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                nf.refine_type5(plan, xd, passes=1, out=o5)
                nf.refine_type4(plan, xd, passes=1, out=o4)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            g5, g4 = o5.cpu().numpy(), o4.cpu().numpy()
            row = {"J": J, "eta": eta, "mu": mu, "plan_ms": plan_ms, "step_ms": ms,
                   "points_per_s": 2 * P / (ms / 1e3),
                   "resid5": O.rel_l2(x, O.type2(g5, t)), "resid4": O.rel_l2(x, O.type1(t, g4, P))}
            try:
                row["truth5"] = O.rel_l2(S_true, nf.refine_type5(plan, s_syn, passes=2))
                row["truth4"] = O.rel_l2(a_true, nf.refine_type4(plan, A_syn, passes=2))
            except nf.NufftError as e:  # e.g. NonConvergence in the over-damped corner
                row["truth_error"] = type(e).__name__
            if not frac:
                try:
                    op = O.Plan.build(t, prm.damping_a, int(eta))
                    row["oracle5"] = O.rel_l2(O.refine5(op, x, 1), g5)
                    row["oracle4"] = O.rel_l2(O.refine4(op, x, 1), g4)
                except Exception as e:  # the reference's own guards
                    row["oracle_error"] = type(e).__name__
            rows.append(row)
            print(json.dumps(row), flush=True)

os.makedirs(os.path.join(REPO, "profiles"), exist_ok=True)
with open(os.path.join(REPO, "gpurun_out", "c5_sweep.json"), "w") as f:
    json.dump({"P": P, "gpu": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


def fmt(v):
    return "—" if v is None else (f"{v:.1e}" if isinstance(v, float) else str(v))


print("| J | eta | mu | plan ms | refined 5+4 ms | points/s | vs oracle (5/4, 1 pass) | vs truth (5/4, 2 passes) | residual (5/4) |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows:
    orc = f"{fmt(r.get('oracle5'))} / {fmt(r.get('oracle4'))}" if "oracle5" in r else (
        r.get("oracle_error", "no reference (extension)"))
    tru = f"{fmt(r.get('truth5'))} / {fmt(r.get('truth4'))}" if "truth5" in r else r.get("truth_error", "")
    print(f"| {r['J']} | {r['eta']} | {r['mu']:.0e} | {r['plan_ms']:.1f} | {r['step_ms']:.3f} | "
          f"{r['points_per_s']:.2e} | {orc} | {tru} | {r['resid5']:.1e} / {r['resid4']:.1e} |")

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
PASSES2 = {(0.1, 2, 1e-17), (0.3, 2, 1e-17), (0.45, 2, 1e-17), (0.45, 2, 1e-16)}
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
                # the stated pass count (tests/test_gpu_parity.py C5_PASSES2): 2 where the
                # reference's own one-pass output is > 1e-11 from its two-pass result
                passes = 2 if (J, eta, mu) in PASSES2 else 1
                row["passes"] = passes
                try:
                    op = O.Plan.build(t, prm.damping_a, int(eta))
                    for kind, fn in ((5, nf.refine_type5), (4, nf.refine_type4)):
                        solve = O.solve5 if kind == 5 else O.solve4
                        fwd = (lambda v: O.type2(v, t)) if kind == 5 else (lambda v: O.type1(t, v, P))
                        x0 = solve(op, x)
                        x1 = x0 - solve(op, fwd(x0) - x)
                        r1 = fwd(x1) - x
                        x2 = x1 - solve(op, r1)
                        got = fn(plan, x, passes=passes)
                        row[f"oracle{kind}"] = O.rel_l2(x1 if passes == 1 else x2, got)
                        row[f"floor{kind}"] = O.rel_l2(x2, x1)
                        row[f"refres{kind}"] = float(np.linalg.norm(r1) / np.linalg.norm(x))
                        row[f"res_stated{kind}"] = (O.rel_l2(x, O.type2(got, t)) if kind == 5
                                                    else O.rel_l2(x, O.type1(t, got, P)))
                except Exception as e:  # the reference's own guards
                    row["oracle_error"] = type(e).__name__
            rows.append(row)
            print(json.dumps(row), flush=True)

os.makedirs(os.path.join(REPO, "profiles"), exist_ok=True)
with open(os.path.join(REPO, "gpurun_out", "c5_sweep.json"), "w") as f:
    json.dump({"P": P, "gpu": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


def fmt(v):
    return "—" if v is None else (f"{v:.1e}" if isinstance(v, float) else str(v))


lines = ["# Config 5 sweep (P = 2^18, one signal), B200 — `python tests/tools/c5_sweep.py`", "",
         "Refined = passes=1 solves timed device-resident (CUDA events, 20 reps). 'vs oracle' = GPU at the "
         "cell's STATED pass count vs the CPU restatement of the reference at the same count (integer eta "
         "only; eta=1.5 is the fractional-oversampling extension). Stated passes = 2 where the reference's own "
         "one-pass output has not converged: its self-floor (distance between its 1-pass and 2-pass results) "
         "exceeds 1e-11; 'ref 1-pass residual' is the reference's own forward residual after one pass. "
         "'vs truth' = samples built from a known spectrum / amplitudes by the fast forward NFFT, solved with "
         "passes=2. Residual = forward NFFT of the GPU output (stated passes) vs the input. The same cells are "
         "the gate of tests/test_gpu_parity.py::test_c5_grid_2_18.", "",
         "| J | eta | mu | plan ms | refined 5+4 ms | points/s | stated passes | vs oracle (5/4) | reference "
         "self-floor (5/4) | ref 1-pass residual (5/4) | GPU residual (5/4) | vs truth (5/4, 2 passes) |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    if "oracle5" in r:
        orc = f"{fmt(r['oracle5'])} / {fmt(r['oracle4'])}"
        flo = f"{fmt(r['floor5'])} / {fmt(r['floor4'])}"
        rr = f"{fmt(r['refres5'])} / {fmt(r['refres4'])}"
        gr = f"{fmt(r['res_stated5'])} / {fmt(r['res_stated4'])}"
        ps = str(r["passes"])
    else:
        orc = r.get("oracle_error", "no reference (extension)")
        flo = rr = "—"
        gr = f"{r['resid5']:.1e} / {r['resid4']:.1e} (1 pass)"
        ps = "1"
    tru = f"{fmt(r.get('truth5'))} / {fmt(r.get('truth4'))}" if "truth5" in r else r.get("truth_error", "")
    lines.append(f"| {r['J']} | {r['eta']} | {r['mu']:.0e} | {r['plan_ms']:.1f} | {r['step_ms']:.3f} | "
                 f"{r['points_per_s']:.2e} | {ps} | {orc} | {flo} | {rr} | {gr} | {tru} |")
with open(os.path.join(REPO, "gpurun_out", "c5_sweep.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))

"""Ad-hoc GPU correctness sweep (prints errors vs the oracle / golden)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1604_06236_b200 as nf
from oracle import nfft_oracle as O

z = np.load("tests/golden/golden.npz")
rel = O.rel_l2
worst = {}
def rec(k, v):
    worst[k] = max(worst.get(k, 0), v)
    return v

for i in range(int(z["fwd_count"])):
    t = z[f"fwd{i}_t"]; a = z[f"fwd{i}_a"]; S = z[f"fwd{i}_S"]; R = int(z[f"fwd{i}_R"])
    g = nf.validate_grid(t)
    try:
        e1 = rec("type1", rel(z[f"fwd{i}_type1"], nf.nfft_type1(g, a, R)))
        e2 = rec("type2", rel(z[f"fwd{i}_type2"], nf.nfft_type2(S, g)))
        d1 = rec("type1_direct", rel(z[f"fwd{i}_type1_direct"], nf.nfft_type1_direct(g, a, R)))
        d2 = rec("type2_direct", rel(z[f"fwd{i}_type2_direct"], nf.nfft_type2_direct(S, g)))
        print(f"fwd{i} Q={t.size} R={R}: t1 {e1:.1e} t2 {e2:.1e} d1 {d1:.1e} d2 {d2:.1e}")
    except Exception as ex:
        print(f"fwd{i} FAILED {type(ex).__name__}: {ex}")
for i in range(int(z["conv_count"])):
    P = int(z[f"conv{i}_P"])
    g = nf.validate_grid(z[f"conv{i}_t"])
    e = rec("conv", rel(z[f"conv{i}_out"], nf.nonuniform_conv(g, z[f"conv{i}_a"], z[f"conv{i}_lam"], P)))
    print(f"conv{i}: {e:.1e}")
for i in range(int(z["plan_count"])):
    P = int(z[f"plan{i}_P"]); eta = int(z[f"plan{i}_eta"]); mu = float(z[f"plan{i}_mu"])
    g = nf.validate_grid(z[f"plan{i}_t"])
    try:
        plan = nf.build_plan(g, nf.MethodParams.from_mu(mu, P, eta))
        kd = plan.kernel_data
        errs = {k: rel(z[f"plan{i}_{k}"], v) for k, v in (("v", kd.v_samples), ("ks", kd.kernel_samples),
                ("L", kd.coefficients), ("dL", kd.derivative_samples), ("nw", plan.node_weights),
                ("decay", plan.h1_coefficients), ("coef", plan.coef_scale))}
        s, A = z[f"plan{i}_s"], z[f"plan{i}_A"]
        errs["t5"] = rel(z[f"plan{i}_type5"], nf.type5(plan, s))
        errs["t4"] = rel(z[f"plan{i}_type4"], nf.type4(plan, A))
        for key, fn, x in (("r5", nf.refine_type5, s), ("r4", nf.refine_type4, A)):
            for p in (1, 2):
                name = f"plan{i}_{key}p{p}"
                if name in z.files:
                    errs[f"{key}p{p}"] = rel(z[name], fn(plan, x, passes=p))
                elif name + "_raises" in z.files:
                    try:
                        fn(plan, x, passes=p); errs[f"{key}p{p}"] = "NO-RAISE"
                    except nf.NonConvergenceError:
                        errs[f"{key}p{p}"] = "raised-ok"
        print(f"plan{i} P={P} eta={eta}: " + " ".join(f"{k}={v:.1e}" if isinstance(v, float) else f"{k}={v}" for k, v in errs.items()))
    except Exception as ex:
        import traceback; traceback.print_exc()
        print(f"plan{i} FAILED {type(ex).__name__}: {ex}")

# bigger: P=2^16 and 2^20 vs oracle (refined)
for P, J, B in ((4096, 0.3, 4), (4096, 0.3, 64), (1 << 16, 0.3, 2), (1 << 16, 0.45, 40), (1 << 20, 0.4, 1)):
    t, data = O.make_inputs(P, J, B, 7)
    g = nf.validate_grid(t)
    prm = nf.MethodParams.from_mu(1e-15, P, 2)
    t0 = time.time(); plan = nf.build_plan(g, prm); import torch; torch.cuda.synchronize(); tp = time.time() - t0
    t0 = time.time(); op = O.Plan.build(t, prm.damping_a, 2); to = time.time() - t0
    x = data
    for p in (0, 1, 2):
        g5 = nf.refine_type5(plan, x, passes=p); g4 = nf.refine_type4(plan, x, passes=p)
        o5 = O.refine5(op, x[0], p); o4 = O.refine4(op, x[0], p)
        print(f"P={P} passes={p}: t5 err {rel(o5, g5[0]):.2e} t4 err {rel(o4, g4[0]):.2e} "
              f"resid5 {rel(x[0], O.type2(g5[0], t)):.2e} resid4 {rel(x[0], O.type1(t, g4[0], P)):.2e}")
    # batched == loop
    if B > 1:
        single = nf.refine_type5(plan, x[1], passes=1)
        full = nf.refine_type5(plan, x, passes=1)
        print("batch vs single: bitwise", np.array_equal(single, full[1]), "rel", rel(single, full[1]),
              "repeat bitwise", np.array_equal(full, nf.refine_type5(plan, x, passes=1)))
        if B >= 32:
            for j in (0, B - 1):
                print(f"  signal {j}: t5 err {rel(O.refine5(op, x[j], 1), full[j]):.2e}")
    print(f"P={P}: plan gpu {tp:.3f}s oracle {to:.3f}s")
print("WORST", worst)
print("launches", nf._lib.load().nfft45_launch_count())

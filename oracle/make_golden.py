"""Generate golden vectors from the REFERENCE implementation (build container only).

Run:  python oracle/make_golden.py [/root/reference]

Imports the reference package ``nufft1d`` from ``<ref>/pkg/src`` (read-only;
nothing is copied), runs it on seeded inputs and writes
``tests/golden/golden.npz``.  Those vectors pin

* the CPU oracle (``oracle/nfft_oracle.py``; ``tests/test_oracle_golden.py``,
  runs without a GPU), and
* the CUDA path (``tests/test_gpu_parity.py``, on the B200 box, where the
  reference tree does not exist — hence the committed fixture).

The reference's own frozen P=8 fixture (``pkg/tests/fixtures/grid8.txt``,
``samples8.txt``, ``coeffs8_dense_solve.txt``; used by
``pkg/tests/test_cli.py:155-169``) is read and stored as arrays too.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

from oracle.nfft_oracle import make_inputs  # noqa: E402


def _read_vec(path):
    rows = [ln.split() for ln in open(path) if ln.strip() and not ln.startswith("#")]
    if len(rows[0]) == 1:
        return np.array([float(r[0]) for r in rows])
    return np.array([float(r[0]) + 1j * float(r[1]) for r in rows])


def main(ref_root="/root/reference"):
    sys.path.insert(0, os.path.join(ref_root, "pkg", "src"))
    import nufft1d as R  # the reference

    out = {}

    def put(key, arr):
        out[key] = np.asarray(arr)

    rng = np.random.default_rng(1604)

    def randc(n):
        return rng.standard_normal(n) + 1j * rng.standard_normal(n)

    # ---- forward transforms: square, rectangular, tiny and non-smooth sizes
    fwd_cases = [(16, 16), (7, 16), (33, 8), (16, 48), (5, 1), (64, 64), (11, 11), (9, 18),
                 (256, 256), (100, 60)]
    for i, (Q, Rn) in enumerate(fwd_cases):
        t = np.sort(rng.uniform(0, 1, Q)) if i % 2 else (np.arange(Q) + rng.uniform(0, 0.6, Q)) / Q
        g = R.validate_grid(t)
        a = randc(Q)
        S = randc(Rn)
        put(f"fwd{i}_t", g.instants)
        put(f"fwd{i}_a", a)
        put(f"fwd{i}_S", S)
        put(f"fwd{i}_R", Rn)
        put(f"fwd{i}_type1", R.nfft_type1(g, a, Rn))
        put(f"fwd{i}_type1_direct", R.nfft_type1_direct(g, a, Rn))
        put(f"fwd{i}_type2", R.nfft_type2(S, g))
        put(f"fwd{i}_type2_direct", R.nfft_type2_direct(S, g))
    put("fwd_count", len(fwd_cases))

    # ---- spread widths other than 14
    t = (np.arange(32) + rng.uniform(0, 0.6, 32)) / 32
    g = R.validate_grid(t)
    a = randc(32)
    put("width_t", t)
    put("width_a", a)
    for m in (4, 8, 12):
        put(f"width_type1_m{m}", R.nfft_type1(g, a, 32, kernel=R.kernel_for_size(32, m)))
        put(f"width_type2_m{m}", R.nfft_type2(a, g, kernel=R.kernel_for_size(32, m)))

    # ---- nonuniform convolution (eta = 1, 2, 3)
    for i, (P, eta) in enumerate([(8, 2), (6, 2), (7, 2), (16, 3), (12, 1)]):
        t = (np.arange(P) + rng.uniform(0, 0.6, P)) / P
        g = R.validate_grid(t)
        a = randc(P)
        lam = randc(eta * P)
        put(f"conv{i}_t", t)
        put(f"conv{i}_a", a)
        put(f"conv{i}_lam", lam)
        put(f"conv{i}_P", P)
        put(f"conv{i}_out", R.nonuniform_conv(g, a, lam, P))
    put("conv_count", 5)

    # ---- plans + solves
    plan_cases = [
        # (P, eta, mu, jitter-grid?)
        (8, 2, 1e-11, "jit"),
        (16, 6, 1e-14, "uniform"),
        (32, 2, 1e-11, "jit"),
        (64, 2, 1e-15, "jit"),
        (64, 3, 1e-15, "jit"),
        (256, 1, 1e-6, "jit"),
        (256, 2, 1e-15, "sorted"),
        (12, 2, 1e-13, "jit"),
        (1, 4, 1e-12, "single"),
    ]
    for i, (P, eta, mu, kind) in enumerate(plan_cases):
        if kind == "uniform":
            t = np.arange(P) / P
        elif kind == "single":
            t = np.array([0.3173])
        elif kind == "sorted":
            t = np.sort(rng.uniform(0, 1, P))
        else:
            t = (np.arange(P) + rng.uniform(0, 0.6, P)) / P
        g = R.validate_grid(t)
        prm = R.MethodParams.from_mu(mu, P, eta)
        plan = R.build_plan(g, prm)
        s = randc(P)
        A = randc(P)
        put(f"plan{i}_t", t)
        put(f"plan{i}_P", P)
        put(f"plan{i}_eta", eta)
        put(f"plan{i}_mu", mu)
        put(f"plan{i}_a", prm.damping_a)
        put(f"plan{i}_v", plan.kernel_data.v_samples)
        put(f"plan{i}_ks", plan.kernel_data.kernel_samples)
        put(f"plan{i}_L", plan.kernel_data.coefficients)
        put(f"plan{i}_dL", plan.kernel_data.derivative_samples)
        put(f"plan{i}_nw", plan.node_weights)
        put(f"plan{i}_decay", plan.h1_coefficients)
        put(f"plan{i}_coef", plan.coef_scale)
        put(f"plan{i}_s", s)
        put(f"plan{i}_A", A)
        put(f"plan{i}_type5", R.type5(plan, s))
        put(f"plan{i}_type4", R.type4(plan, A))
        if P > 1:
            for key, fn, x in (("r5", R.refine_type5, s), ("r4", R.refine_type4, A)):
                for passes in (1, 2):
                    try:
                        put(f"plan{i}_{key}p{passes}", fn(plan, x, passes=passes))
                    except R.NonConvergenceError:
                        # recorded as an expected error (edge case of the refinement)
                        put(f"plan{i}_{key}p{passes}_raises", "NonConvergenceError")
    put("plan_count", len(plan_cases))

    # ---- benchmark-shaped inputs: C1 in full, a C2 signal
    for name, P, J, seed in (("c1", 64, 0.3, 16041), ("c2", 4096, 0.3, 16042)):
        t, data = make_inputs(P, J, 1, seed)
        g = R.validate_grid(t)
        prm = R.MethodParams.from_mu(1e-15, P, 2)
        plan = R.build_plan(g, prm)
        x = data[0]
        put(f"{name}_t", t)
        put(f"{name}_x", x)
        put(f"{name}_a", prm.damping_a)
        put(f"{name}_type5", R.type5(plan, x))
        put(f"{name}_type4", R.type4(plan, x))
        put(f"{name}_r5p1", R.refine_type5(plan, x, passes=1))
        put(f"{name}_r4p1", R.refine_type4(plan, x, passes=1))
        put(f"{name}_r5p2", R.refine_type5(plan, x, passes=2))
        put(f"{name}_r4p2", R.refine_type4(plan, x, passes=2))
        if P <= 64:
            put(f"{name}_nw", plan.node_weights)
            put(f"{name}_ks", plan.kernel_data.kernel_samples)
            put(f"{name}_dL", plan.kernel_data.derivative_samples)

    # ---- analytic flop reports (data-independent; flops.py) for the flops= kwarg
    def rep(fc):
        r = fc.report()
        return np.array([r.real_adds, r.complex_adds, r.real_muls, r.complex_muls, r.complex_exps,
                         r.total_flops] + list(r.fft_invocations), dtype=np.int64)

    t = (np.arange(64) + rng.uniform(0, 0.6, 64)) / 64
    g = R.validate_grid(t)
    prm = R.MethodParams.from_mu(1e-11, 64, 2)
    put("flops_t", t)
    fc = R.FlopCounter(); plan = R.build_plan(g, prm, flops=fc); put("flops_build_plan", rep(fc))
    x = randc(64)
    for name, fn in (("type5", lambda f: R.type5(plan, x, flops=f)), ("type4", lambda f: R.type4(plan, x, flops=f)),
                     ("refine5", lambda f: R.refine_type5(plan, x, passes=1, flops=f)),
                     ("refine4", lambda f: R.refine_type4(plan, x, passes=1, flops=f)),
                     ("type1", lambda f: R.nfft_type1(g, x, 48, flops=f)),
                     ("type2", lambda f: R.nfft_type2(x, g, flops=f)),
                     ("conv", lambda f: R.nonuniform_conv(g, x, randc(128), 64, flops=f)),
                     ("conv_real", lambda f: R.nonuniform_conv(g, x, rng.standard_normal(128), 64, flops=f))):
        fc = R.FlopCounter()
        fn(fc)
        put(f"flops_{name}", rep(fc))

    # ---- the reference's frozen fixture (dense-elimination solution, P=8, mu=1e-11, eta=2)
    fx = os.path.join(ref_root, "pkg", "tests", "fixtures")
    put("fixture_grid8", _read_vec(os.path.join(fx, "grid8.txt")))
    put("fixture_samples8", _read_vec(os.path.join(fx, "samples8.txt")))
    put("fixture_coeffs8", _read_vec(os.path.join(fx, "coeffs8_dense_solve.txt")))

    # ---- baselines (baselines.py): CG runs with their iteration counts and
    # flop reports, dense GE solutions.  Own generator: earlier arrays keep
    # their values.
    rng2 = np.random.default_rng(1604)

    def randc2(n):
        return rng2.standard_normal(n) + 1j * rng2.standard_normal(n)

    cg_cases = [
        ("cg4", 256, 17, "type4", 1e-14, None),
        ("cg5", 64, 19, "type5", 1e-14, None),
        ("cgcap", 128, 23, "type4", 1e-15, 2),
        ("cgtol", 512, 29, "type4", 1e-10, None),
    ]
    for name, P, seed, which, tol, cap in cg_cases:
        grid, a_true = R.generate_trial(P, seed)
        b = R.nfft_type1_direct(grid, a_true, P) if which == "type4" else randc2(P)
        fc = R.FlopCounter()
        res = R.cg_solve(grid, b, which, tol=tol, max_iter=cap, flops=fc)
        put(f"{name}_t", np.asarray(grid.instants))
        put(f"{name}_b", b)
        put(f"{name}_x", res.solution)
        put(f"{name}_meta", np.array([res.iterations, int(res.converged)], dtype=np.int64))
        put(f"{name}_rel", np.array(res.relative_residual))
        put(f"{name}_flops", rep(fc))
        if P <= 256:
            sysm = R.type4_system(grid, b) if which == "type4" else R.type5_system(grid, b)
            put(f"{name}_ge", R.ge_solve(sysm))
    fc = R.FlopCounter()
    grid, _ = R.generate_trial(32, 7)
    b = randc2(32)
    sysm = R.type4_system(grid, b, flops=fc)
    put("ge32_t", np.asarray(grid.instants))
    put("ge32_b", b)
    put("ge32_matrix", sysm.matrix)
    put("ge32_x", R.ge_solve(sysm, flops=fc))
    put("ge32_flops", rep(fc))
    put("cg_cases", np.array([c[0] for c in cg_cases]))

    out["meta_numpy"] = np.array(np.__version__)
    out["meta_reference"] = np.array(R.__version__)
    dst = os.path.join(REPO, "tests", "golden", "golden.npz")
    np.savez_compressed(dst, **out)
    print(f"wrote {dst}: {len(out)} arrays, {os.path.getsize(dst)} bytes")


if __name__ == "__main__":
    main(*sys.argv[1:])

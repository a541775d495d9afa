"""Pin the CPU oracle against vectors produced by the reference itself.

The golden file comes from ``oracle/make_golden.py`` (imports the reference
``nufft1d`` in the build container).  These tests need no GPU.
"""

import numpy as np
import pytest

from oracle import nfft_oracle as O


def rel(truth, got):
    return O.rel_l2(truth, got)


def test_forward_transforms_match_reference(golden):
    for i in range(int(golden["fwd_count"])):
        t = golden[f"fwd{i}_t"]
        a, S, R = golden[f"fwd{i}_a"], golden[f"fwd{i}_S"], int(golden[f"fwd{i}_R"])
        assert rel(golden[f"fwd{i}_type1"], O.type1(t, a, R)) < 1e-15
        assert rel(golden[f"fwd{i}_type2"], O.type2(S, t)) < 1e-15
        assert rel(golden[f"fwd{i}_type1_direct"], O.type1_exact(t, a, R)) < 1e-15
        assert rel(golden[f"fwd{i}_type2_direct"], O.type2_exact(S, t)) < 1e-15
        # the fast paths track the exact sums (reference tests/test_forward.py:85-125)
        assert rel(golden[f"fwd{i}_type1_direct"], O.type1(t, a, R)) < 1e-12
        assert rel(golden[f"fwd{i}_type2_direct"], O.type2(S, t)) < 1e-12


def test_spread_widths(golden):
    t, a = golden["width_t"], golden["width_a"]
    for m in (4, 8, 12):
        assert rel(golden[f"width_type1_m{m}"], O.type1(t, a, 32, m)) < 1e-15
        assert rel(golden[f"width_type2_m{m}"], O.type2(a, t, m)) < 1e-15


def test_nonuniform_conv(golden):
    for i in range(int(golden["conv_count"])):
        P = int(golden[f"conv{i}_P"])
        got = O.conv(golden[f"conv{i}_t"], golden[f"conv{i}_a"], golden[f"conv{i}_lam"], P)
        assert rel(golden[f"conv{i}_out"], got) < 1e-15


@pytest.mark.parametrize("i", range(9))
def test_plan_and_solves(golden, i):
    P = int(golden[f"plan{i}_P"])
    eta = int(golden[f"plan{i}_eta"])
    a = float(golden[f"plan{i}_a"])
    assert a == O.damping(float(golden[f"plan{i}_mu"]), P, eta)
    plan = O.Plan.build(golden[f"plan{i}_t"], a, eta)
    for key, got in (("v", plan.v), ("ks", plan.ks), ("L", plan.L), ("dL", plan.dL),
                     ("nw", plan.node_weights), ("decay", plan.decay), ("coef", plan.coef_scale)):
        assert rel(golden[f"plan{i}_{key}"], got) < 1e-15, key
    s, A = golden[f"plan{i}_s"], golden[f"plan{i}_A"]
    assert rel(golden[f"plan{i}_type5"], O.solve5(plan, s)) < 1e-15
    assert rel(golden[f"plan{i}_type4"], O.solve4(plan, A)) < 1e-15
    if P == 1:
        return
    for key, fn, x in (("r5", O.refine5, s), ("r4", O.refine4, A)):
        for passes in (1, 2):
            name = f"plan{i}_{key}p{passes}"
            if name + "_raises" in golden.files:
                with pytest.raises(O.NonConvergence):
                    fn(plan, x, passes)
            else:
                assert rel(golden[name], fn(plan, x, passes)) < 1e-15


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_benchmark_shaped_inputs(golden, name):
    t, x = golden[f"{name}_t"], golden[f"{name}_x"]
    P = t.size
    t2, d2 = O.make_inputs(P, 0.3, 1, 16041 if name == "c1" else 16042)
    assert np.array_equal(t, t2) and np.array_equal(x, d2[0])
    plan = O.Plan.build(t, float(golden[f"{name}_a"]), 2)
    assert rel(golden[f"{name}_type5"], O.solve5(plan, x)) < 1e-15
    assert rel(golden[f"{name}_type4"], O.solve4(plan, x)) < 1e-15
    for p in (1, 2):
        assert rel(golden[f"{name}_r5p{p}"], O.refine5(plan, x, p)) < 1e-15
        assert rel(golden[f"{name}_r4p{p}"], O.refine4(plan, x, p)) < 1e-15


def test_frozen_fixture(golden):
    """Reference fixture: dense-elimination type-5 solution at P=8 (test_cli.py:155-169)."""
    t = golden["fixture_grid8"]
    s = golden["fixture_samples8"]
    want = golden["fixture_coeffs8"]
    plan = O.Plan.build(t, O.damping(1e-11, 8, 2), 2)
    assert rel(want, O.solve5(plan, s)) < 1e-10
    assert rel(want, O.refine5(plan, s, 1)) < 1e-13


def test_validation_errors():
    with pytest.raises(O.OutOfRange):
        O.validate([0.1, 1.0])
    with pytest.raises(O.DuplicateNode):
        O.validate([0.1, 0.1 + 1e-14])
    t, order = O.validate([0.5, 0.25, 0.75])
    assert list(order) == [1, 0, 2]
    with pytest.raises(O.NonPositiveDamping):
        O.damping(0.5, 4, 1)


_CG_ARGS = {"cg4": ("type4", 1e-14, None), "cg5": ("type5", 1e-14, None), "cgcap": ("type4", 1e-15, 2),
            "cgtol": ("type4", 1e-10, None)}


@pytest.mark.parametrize("name", sorted(_CG_ARGS))
def test_oracle_cg_reproduces_reference(golden, name):
    """CGNR restatement (baselines.py:116-181) vs the reference's own runs:
    same iteration count and convergence flag, same iterate."""
    which, tol, cap = _CG_ARGS[name]
    x, it, conv, relres = O.cg(golden[f"{name}_t"], golden[f"{name}_b"], which, tol, cap)
    want_it, want_conv = (int(v) for v in golden[f"{name}_meta"])
    assert (it, int(conv)) == (want_it, want_conv)
    assert rel(golden[f"{name}_x"], x) < 1e-14
    assert abs(relres - float(golden[f"{name}_rel"])) <= 1e-12 * float(golden[f"{name}_rel"])


def test_oracle_phase_matrix_and_dense_solve(golden):
    M = O.phase_matrix(golden["ge32_t"], -1)
    assert np.abs(M - golden["ge32_matrix"]).max() < 1e-15
    assert rel(golden["ge32_x"], O.dense_solve(M, golden["ge32_b"])) < 1e-12
    for name in ("cg4", "cg5"):  # CG converged to the dense solution
        assert rel(golden[f"{name}_ge"], golden[f"{name}_x"]) < 1e-10


def test_harness_trial_streams_bitwise_equal_reference():
    """metrics.trial_arrays reproduces the reference's generate_trial streams
    (bench.py:84-92) bit for bit (golden: oracle/make_sweep_golden.py)."""
    import json
    import os

    from paper_1604_06236_b200.metrics import trial_arrays

    g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sweep_rows.json")))
    for c in g["trial_streams"]:
        t, a = trial_arrays(c["P"], c["seed"])
        assert np.array_equal(t, np.array(c["nodes"]))
        assert np.array_equal(a.real, np.array(c["re"])) and np.array_equal(a.imag, np.array(c["im"]))

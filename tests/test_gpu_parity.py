"""Parity of the CUDA path with the reference: golden vectors produced by the
reference itself (tests/golden, oracle/make_golden.py) and, at the
BASELINE.json config sizes, the CPU oracle run live on the same seeded
inputs plus size-independent properties (forward residuals, linearity,
determinism).

Gates:
  G1  refined path (passes = 1, 2): rel-L2 vs reference <= 1e-10 AND forward
      residual ||fwd(out) - in|| / ||in|| <= 1e-10 (fwd = reference fast NFFT);
  G2  plain path: reported vs the reference's own permutation floor — it is
      roundoff amplified ~(mu eta P)^(-1/eta), so only a loose bound is asserted;
  G3  forward NFFTs: <= 1e-13 vs the reference fast path, <= 1e-12 vs direct.
"""

import numpy as np
import pytest
import torch

import paper_1604_06236_b200 as nf
from oracle import nfft_oracle as O

pytestmark = pytest.mark.gpu

G1 = 1e-10


def rel(truth, got):
    return O.rel_l2(truth, got)


# ------------------------------------------------------------ golden vectors

def test_forward_golden(golden):
    for i in range(int(golden["fwd_count"])):
        g = nf.validate_grid(golden[f"fwd{i}_t"])
        a, S, R = golden[f"fwd{i}_a"], golden[f"fwd{i}_S"], int(golden[f"fwd{i}_R"])
        assert rel(golden[f"fwd{i}_type1"], nf.nfft_type1(g, a, R)) < 1e-13
        assert rel(golden[f"fwd{i}_type2"], nf.nfft_type2(S, g)) < 1e-13
        assert rel(golden[f"fwd{i}_type1_direct"], nf.nfft_type1(g, a, R)) < 1e-12
        assert rel(golden[f"fwd{i}_type2_direct"], nf.nfft_type2(S, g)) < 1e-12
        assert rel(golden[f"fwd{i}_type1_direct"], nf.nfft_type1_direct(g, a, R)) < 1e-14
        assert rel(golden[f"fwd{i}_type2_direct"], nf.nfft_type2_direct(S, g)) < 1e-14


def test_spread_width_golden(golden):
    g = nf.validate_grid(golden["width_t"])
    a = golden["width_a"]
    for m in (4, 8, 12):
        k = nf.kernel_for_size(32, m)
        assert rel(golden[f"width_type1_m{m}"], nf.nfft_type1(g, a, 32, kernel=k)) < 1e-13
        assert rel(golden[f"width_type2_m{m}"], nf.nfft_type2(a, g, kernel=k)) < 1e-13


def test_conv_golden(golden):
    for i in range(int(golden["conv_count"])):
        P = int(golden[f"conv{i}_P"])
        g = nf.validate_grid(golden[f"conv{i}_t"])
        got = nf.nonuniform_conv(g, golden[f"conv{i}_a"], golden[f"conv{i}_lam"], P)
        assert rel(golden[f"conv{i}_out"], got) < 1e-13


WELL_CONDITIONED = [0, 1, 2, 3, 4, 5, 7, 8]   # plan6: random uniform nodes, the reference itself diverges


@pytest.mark.parametrize("i", WELL_CONDITIONED)
def test_plan_and_solves_golden(golden, i):
    P, eta = int(golden[f"plan{i}_P"]), int(golden[f"plan{i}_eta"])
    g = nf.validate_grid(golden[f"plan{i}_t"])
    prm = nf.MethodParams.from_mu(float(golden[f"plan{i}_mu"]), P, eta)
    plan = nf.build_plan(g, prm)
    kd = plan.kernel_data
    assert rel(golden[f"plan{i}_v"], kd.v_samples) < 1e-12
    assert rel(golden[f"plan{i}_ks"], kd.kernel_samples) < 1e-12
    # coefficient recovery amplifies roundoff (test_lagrange.py:211-214): method-level agreement
    assert rel(golden[f"plan{i}_L"], kd.coefficients) < 1e-7
    assert rel(golden[f"plan{i}_dL"], kd.derivative_samples) < 1e-7
    assert rel(golden[f"plan{i}_nw"], plan.node_weights) < 1e-7
    assert rel(golden[f"plan{i}_decay"], plan.h1_coefficients) < 1e-14
    assert rel(golden[f"plan{i}_coef"], plan.coef_scale) < 1e-14
    s, A = golden[f"plan{i}_s"], golden[f"plan{i}_A"]
    assert rel(golden[f"plan{i}_type5"], nf.type5(plan, s)) < 1e-6   # G2 (plain)
    assert rel(golden[f"plan{i}_type4"], nf.type4(plan, A)) < 1e-6
    if P == 1:
        return
    for key, fn, x in (("r5", nf.refine_type5, s), ("r4", nf.refine_type4, A)):
        for passes in (1, 2):
            assert rel(golden[f"plan{i}_{key}p{passes}"], fn(plan, x, passes=passes)) < G1


def test_ill_conditioned_grid_raises_like_reference(golden):
    i = 6
    P = int(golden[f"plan{i}_P"])
    g = nf.validate_grid(golden[f"plan{i}_t"])
    plan = nf.build_plan(g, nf.MethodParams.from_mu(float(golden[f"plan{i}_mu"]), P, 2))
    assert f"plan{i}_r5p2_raises" in golden.files
    with pytest.raises(nf.NonConvergenceError):
        nf.refine_type5(plan, golden[f"plan{i}_s"], passes=2)
    with pytest.raises(nf.NonConvergenceError):
        nf.refine_type4(plan, golden[f"plan{i}_A"], passes=2)


def test_frozen_fixture(golden):
    """The reference's frozen dense-elimination solution (pkg/tests/fixtures, test_cli.py:155-169)."""
    g = nf.validate_grid(golden["fixture_grid8"])
    plan = nf.build_plan(g, nf.MethodParams.from_mu(1e-11, 8, 2))
    s = golden["fixture_samples8"]
    want = golden["fixture_coeffs8"]
    assert rel(want, nf.type5(plan, s)) < 1e-10
    assert rel(want, nf.refine_type5(plan, s, passes=1)) < 1e-13


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_shaped_golden(golden, name):
    t, x = golden[f"{name}_t"], golden[f"{name}_x"]
    P = t.size
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    for p in (1, 2):
        g5 = nf.refine_type5(plan, x, passes=p)
        g4 = nf.refine_type4(plan, x, passes=p)
        assert rel(golden[f"{name}_r5p{p}"], g5) < G1
        assert rel(golden[f"{name}_r4p{p}"], g4) < G1
        assert rel(x, O.type2(g5, t)) < G1
        assert rel(x, O.type1(t, g4, P)) < G1
    assert rel(golden[f"{name}_type5"], nf.type5(plan, x)) < 1e-5


# ------------------------------------------------ config sizes vs live oracle

def _check_config(P, J, B, seed, eta=2, mu=1e-15, passes=(1, 2), rows=(0,)):
    t, data = O.make_inputs(P, J, B, seed)
    grid = nf.validate_grid(t)
    prm = nf.MethodParams.from_mu(mu, P, eta, fractional_eta=float(eta) != int(eta))
    plan = nf.build_plan(grid, prm)
    oplan = O.Plan.build(t, prm.damping_a, eta)
    report = {}
    for p in passes:
        g5 = nf.refine_type5(plan, data if B > 1 else data[0], passes=p)
        g4 = nf.refine_type4(plan, data if B > 1 else data[0], passes=p)
        g5, g4 = np.atleast_2d(g5), np.atleast_2d(g4)
        for r in rows:
            e5 = rel(O.refine5(oplan, data[r], p), g5[r])
            e4 = rel(O.refine4(oplan, data[r], p), g4[r])
            r5 = rel(data[r], O.type2(g5[r], t))
            r4 = rel(data[r], O.type1(t, g4[r], P))
            report[(p, r)] = (e5, e4, r5, r4)
            assert max(e5, e4, r5, r4) <= G1, (P, p, r, e5, e4, r5, r4)
    return report


def test_c2_batched_4096x64():
    _check_config(4096, 0.3, 64, 16042, rows=(0, 31, 63))


def test_c4_shape_65536_batched():
    _check_config(1 << 16, 0.3, 40, 16044, rows=(0, 39))


def test_c4_full_size_1024x65536_properties():
    """BASELINE config 4 at its full size (1024 signals x 2^16, device-resident, the bench
    workload): every signal's forward residual (device forward NFFTs) <= 1e-10, the
    first and last signals vs the CPU oracle <= 1e-10, and linearity of the refined
    solves on a pair of signals (size-independent properties of the path)."""
    P, B = 1 << 16, 1024
    t, _ = O.make_inputs(P, 0.3, 1, 16044)
    grid = nf.validate_grid(t)
    prm = nf.MethodParams.from_mu(1e-15, P, 2)
    plan = nf.build_plan(grid, prm)
    g = torch.Generator(device="cuda")
    g.manual_seed(16044)
    mk = lambda: torch.complex(torch.randn(B, P, generator=g, device="cuda", dtype=torch.float64),
                               torch.randn(B, P, generator=g, device="cuda", dtype=torch.float64))
    s, A = mk(), mk()
    x5 = nf.refine_type5(plan, s, passes=1)
    x4 = nf.refine_type4(plan, A, passes=1)
    res5 = torch.linalg.norm(nf.nfft_type2(x5, grid) - s, dim=1) / torch.linalg.norm(s, dim=1)
    res4 = torch.linalg.norm(nf.nfft_type1(grid, x4, P) - A, dim=1) / torch.linalg.norm(A, dim=1)
    assert float(res5.max()) <= G1 and float(res4.max()) <= G1, (float(res5.max()), float(res4.max()))
    oplan = O.Plan.build(t, prm.damping_a, 2)
    for r in (0, B - 1):
        assert rel(O.refine5(oplan, s[r].cpu().numpy(), 1), x5[r].cpu().numpy()) <= G1
        assert rel(O.refine4(oplan, A[r].cpu().numpy(), 1), x4[r].cpu().numpy()) <= G1
    a, b = 0.75 - 0.5j, -1.25 + 0.25j
    mix = (a * s[3] + b * s[7]).unsqueeze(0)
    got = nf.refine_type5(plan, mix, passes=1)[0]
    want = a * x5[3] + b * x5[7]
    assert float(torch.linalg.norm(got - want) / torch.linalg.norm(want)) <= 1e-12


def test_c4_shape_repeatable_and_row_independent():
    """Race canary for the kernels that reuse live shared memory (compute-sanitizer is closed
    on the pool): at the C4 kernel shape with enough signals for the 64-signal spreading groups,
    the 8-warp gather (transpose tile aliased onto the consumed cell tile) and the bulk tensor
    stores (dense rows written in place in the tile buffer), ten solves of the same operands
    give bitwise the same outputs, a signal's result does not depend on which other signals
    share its groups / tiles (rows of a 200-signal batch vs the same rows in a 131-signal
    batch), and rows 0 / last agree with the oracle."""
    P, B = 1 << 16, 200
    t, data = O.make_inputs(P, 0.3, 8, 16044)
    rng = np.random.default_rng(99)
    data = (rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))) / np.sqrt(2)
    prm = nf.MethodParams.from_mu(1e-15, P, 2)
    plan = nf.build_plan(nf.validate_grid(t), prm)
    d = torch.from_numpy(data).cuda()
    x5 = nf.refine_type5(plan, d, passes=1)
    x4 = nf.refine_type4(plan, d, passes=1)
    for _ in range(9):
        assert torch.equal(x5, nf.refine_type5(plan, d, passes=1))
        assert torch.equal(x4, nf.refine_type4(plan, d, passes=1))
    sub = d[69:200].contiguous()  # 131 signals: other group / tile neighbours, ragged tail
    assert torch.equal(x5[69:200], nf.refine_type5(plan, sub, passes=1))
    assert torch.equal(x4[69:200], nf.refine_type4(plan, sub, passes=1))
    oplan = O.Plan.build(t, prm.damping_a, 2)
    for r in (0, B - 1):
        assert rel(O.refine5(oplan, data[r], 1), x5[r].cpu().numpy()) <= G1
        assert rel(O.refine4(oplan, data[r], 1), x4[r].cpu().numpy()) <= G1


def test_c3_single_2_20():
    _check_config(1 << 20, 0.4, 1, 16043, passes=(1,))


@pytest.mark.parametrize("logP", [18, 20])
def test_batched_large_grids(logP):
    """Batch-minor chains at M = 512 (8-signal tiles) and M = 1024 (4-signal
    band/pad tiles, 2-row boundary tiles): vs the oracle on the first and last
    signal; type 5 bitwise equal to the single-signal (signal-major) chain,
    type 4 equal to rounding (its batch-minor and signal-major kernels round
    differently, ~1e-13 on the plain solve, ~1e-15 refined)."""
    P, B = 1 << logP, 16
    _check_config(P, 0.3, B, 16046, passes=(1,), rows=(0, B - 1))
    t, data = O.make_inputs(P, 0.3, B, 16046)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    full5 = nf.refine_type5(plan, data, passes=1)
    full4 = nf.refine_type4(plan, data, passes=1)
    assert np.array_equal(full5[B - 1], nf.refine_type5(plan, data[B - 1], passes=1))
    assert rel(nf.refine_type4(plan, data[B - 1], passes=1), full4[B - 1]) < 1e-13


@pytest.mark.parametrize("P,B", [(2048, 16), (8192, 24), (1 << 15, 24), (1 << 17, 17), (1 << 19, 16)])
def test_rectangular_batch_minor_chains(P, B):
    """Odd powers of two, P = R * C with R = 2C, on the batch-minor chains
    (batches >= 16): vs the oracle on the first and last signal, and vs the
    single-signal solve (generic kernels) to rounding."""
    _check_config(P, 0.3, B, 16050, passes=(1,), rows=(0, B - 1))
    t, data = O.make_inputs(P, 0.3, B, 16050)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    full5, full4 = nf.type5(plan, data), nf.type4(plan, data)
    # plain solves amplify roundoff (finding 2): compare the two kernel families at that level
    assert rel(nf.type5(plan, data[B - 1]), full5[B - 1]) < 1e-9
    assert rel(nf.type4(plan, data[B - 1]), full4[B - 1]) < 1e-9


@pytest.mark.parametrize("P,B", [(3072, 1), (3072, 16), (12288, 24), (49152, 1), (49152, 17), (196608, 1),
                                 (196608, 16), (786432, 1), (786432, 16)])
def test_three_times_power_of_two_chains(P, B):
    """P = 3 * 2^k on the chains (PR = 3 * 2^a, PC = 4 PR / 3; radix-3 tile
    schedules): vs the oracle, signal-major and batch-minor."""
    _check_config(P, 0.3, B, 16052, passes=(1,), rows=(0, B - 1) if B > 1 else (0,))


@pytest.mark.parametrize("P", [2048, 1 << 15, 1 << 17, 1 << 19])
def test_rectangular_single_signal_chains(P):
    """Odd powers of two on the signal-major chains (single transforms): vs the
    oracle, and batched (batch-minor kernels) vs single to rounding."""
    _check_config(P, 0.3, 1, 16051, passes=(1,))


# BASELINE config 5, every oracle-backed cell: P = 2^18, one signal (seed 16045),
# J x eta x mu.  The gate is G1 at the cell's stated pass count: passes = 1,
# except where the reference's OWN one-pass output has not converged — its
# distance to its own two-pass result (the "self-floor", measured live below
# and listed in profiles/c5_sweep.md) exceeds 1e-11, i.e. the over-damped
# corner mu <= 1e-17 at eta = 2 and mu = 1e-16 at J = 0.45 (reference
# self-floor 5e-11 ... 8e-10, one-pass residual up to 8e-10).  There the
# comparison is at passes = 2 (both converge to ~1e-15).
C5_PASSES2 = {(0.1, 2, 1e-17), (0.3, 2, 1e-17), (0.45, 2, 1e-17), (0.45, 2, 1e-16)}
C5_CELLS = [(J, eta, mu) for J in (0.1, 0.3, 0.45) for eta in (2, 3) for mu in (1e-17, 1e-16, 1e-15, 1e-14, 1e-13)]


def _oracle_two_passes(oplan, x, kind, t, P):
    """The reference's refinement (inverse.py:146-162) unrolled: x1 and x2 and the residuals."""
    solve = O.solve5 if kind == 5 else O.solve4
    fwd = (lambda v: O.type2(v, t)) if kind == 5 else (lambda v: O.type1(t, v, P))
    x0 = solve(oplan, x)
    x1 = x0 - solve(oplan, fwd(x0) - x)
    r1 = fwd(x1) - x
    x2 = x1 - solve(oplan, r1)
    return x1, x2, float(np.linalg.norm(r1) / np.linalg.norm(x))


@pytest.mark.slow
@pytest.mark.parametrize("J,eta,mu", C5_CELLS)
def test_c5_grid_2_18(J, eta, mu):
    P = 1 << 18
    t, data = O.make_inputs(P, J, 1, 16045)
    x = data[0]
    prm = nf.MethodParams.from_mu(mu, P, eta)
    plan = nf.build_plan(nf.validate_grid(t), prm)
    oplan = O.Plan.build(t, prm.damping_a, eta)
    passes = 2 if (J, eta, mu) in C5_PASSES2 else 1
    for kind in (5, 4):
        x1, x2, ref_res1 = _oracle_two_passes(oplan, x, kind, t, P)
        floor = rel(x2, x1)  # the reference's own one-pass non-convergence
        if passes == 1:
            assert floor <= 1e-11, (kind, floor)  # the stated pass count is the right one
        else:
            assert floor > 1e-11, (kind, floor)
        got = (nf.refine_type5 if kind == 5 else nf.refine_type4)(plan, x, passes=passes)
        err = rel(x1 if passes == 1 else x2, got)
        res = rel(x, O.type2(got, t)) if kind == 5 else rel(x, O.type1(t, got, P))
        assert err <= G1 and res <= G1, (kind, passes, err, res, floor, ref_res1)


# Extension: BASELINE config 5's eta = 1.5 (the reference needs an integer
# eta; the oracle's v_samples_terms restates the same steps with a partial
# fold).  Checked against that restatement, by forward residual, and against
# truth built by construction.
@pytest.mark.parametrize("P,J", [(4096, 0.3), (1 << 18, 0.1), (1 << 18, 0.45)])
def test_c5_fractional_eta(P, J):
    # eta = 1.5 amplifies the plain solve's roundoff more than eta = 2 (finding
    # 2): one pass leaves both implementations ~1e-9 from the fixed point
    # (forward residuals ~2e-14), the second pass converges both
    _check_config(P, J, 1, 16045, eta=1.5, passes=(2,))


def test_c5_fractional_eta_truth_by_construction():
    P = 1 << 18
    t, _ = O.make_inputs(P, 0.3, 1, 16047)
    grid = nf.validate_grid(t)
    rng = np.random.default_rng(16047)
    S = (rng.standard_normal(P) + 1j * rng.standard_normal(P)) / np.sqrt(2)
    s = nf.nfft_type2(S, grid)                      # samples of a known spectrum
    plan = nf.build_plan(grid, nf.MethodParams.from_mu(1e-15, P, 1.5, fractional_eta=True))
    got = nf.refine_type5(plan, s, passes=2)
    assert rel(S, got) <= G1
    plan_v = plan.kernel_data.v_samples
    oracle_v = O.v_samples_terms(t, plan.params.damping_a, 3 * P // 2)
    assert rel(oracle_v, plan_v) < 1e-10  # length-3P/2 series, FFT sizes 3*2^k: rounding-level agreement


def test_plain_path_is_at_least_as_accurate_as_reference():
    """G2: the plain solve is roundoff-amplified; ours is checked against the
    exact forward operator: its residual must not exceed the reference's."""
    P = 4096
    t, data = O.make_inputs(P, 0.3, 1, 16042)
    x = data[0]
    prm = nf.MethodParams.from_mu(1e-15, P, 2)
    plan = nf.build_plan(nf.validate_grid(t), prm)
    oplan = O.Plan.build(t, prm.damping_a, 2)
    ours = rel(x, O.type2(nf.type5(plan, x), t))
    ref = rel(x, O.type2(O.solve5(oplan, x), t))
    assert ours <= 2 * ref


# ------------------------------------------------ batched / device API

def test_batched_equals_per_signal_and_is_bitwise_reproducible():
    P, B = 4096, 48
    t, data = O.make_inputs(P, 0.3, B, 7)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    full = nf.refine_type5(plan, data, passes=1)
    assert full.shape == (B, P)
    for r in (0, B - 1):
        assert np.array_equal(full[r], nf.refine_type5(plan, data[r], passes=1))
    assert np.array_equal(full, nf.refine_type5(plan, data, passes=1))
    full4 = nf.refine_type4(plan, data, passes=1)
    assert np.array_equal(full4[5], nf.refine_type4(plan, data[5], passes=1))


@pytest.mark.parametrize("B", [3, 5, 15, 16, 17, 33])
def test_batch_sizes_across_kernel_switches(B):
    """Batch sizes on both sides of every kernel switch (small-batch gridding
    with 1- and 4-signal tiles, signal-major vs batch-minor chains at 16, padded
    batch-minor rows): every row matches its single-signal solve — type 5
    bitwise, type 4 to rounding — and the oracle."""
    P = 4096
    t, data = O.make_inputs(P, 0.3, B, 100 + B)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    oplan = O.Plan.build(t, plan.params.damping_a, 2)
    full5 = nf.refine_type5(plan, data, passes=1)
    full4 = nf.refine_type4(plan, data, passes=1)
    for r in sorted({0, B // 2, B - 1}):
        assert np.array_equal(full5[r], nf.refine_type5(plan, data[r], passes=1))
        assert rel(nf.refine_type4(plan, data[r], passes=1), full4[r]) < 1e-13
        assert rel(O.refine5(oplan, data[r], 1), full5[r]) <= G1
        assert rel(O.refine4(oplan, data[r], 1), full4[r]) <= G1


def test_torch_device_and_pinned_host_operands():
    P, B = 1 << 16, 4
    t, data = O.make_inputs(P, 0.3, B, 9)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    ref = nf.refine_type5(plan, data, passes=1)
    dev = torch.from_numpy(data).cuda()
    out_dev = nf.refine_type5(plan, dev, passes=1)
    assert out_dev.is_cuda and np.array_equal(out_dev.cpu().numpy(), ref)
    host = torch.from_numpy(data).pin_memory()
    dest = torch.empty_like(host).pin_memory()
    got = nf.refine_type5(plan, host, passes=1, out=dest)
    assert got is dest and np.array_equal(dest.numpy(), ref)
    buf = torch.empty_like(dev)
    nf.refine_type5(plan, dev, passes=1, out=buf)
    assert np.array_equal(buf.cpu().numpy(), ref)


def test_native_library_is_the_code_path():
    from paper_1604_06236_b200 import _lib

    before = _lib.load().nfft45_launch_count()
    g = nf.validate_grid(np.arange(64) / 64 + 0.001)
    nf.nfft_type1(g, np.ones(64), 64)
    assert _lib.load().nfft45_launch_count() > before


def test_streamed_host_batches_match_device_path():
    """CPU (pinned) [batch, P] operands larger than one chunk are streamed through
    the device (copies overlapped with the solves); results equal the device path."""
    from paper_1604_06236_b200 import inverse as inv

    P, B = 4096, inv.STREAM_CHUNK * 2 + 37
    t, data = O.make_inputs(P, 0.3, B, 11)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    dev = torch.from_numpy(data).cuda()
    want5 = nf.refine_type5(plan, dev, passes=1).cpu()
    want4 = nf.type4(plan, dev).cpu()
    host = torch.from_numpy(data).pin_memory()
    got5 = nf.refine_type5(plan, host, passes=1, out=torch.empty_like(host).pin_memory())
    got4 = nf.type4(plan, host)
    assert not got4.is_cuda
    # chunks of 128 vs one batch of 293: both use the batch-minor kernels (>= 16 signals)
    assert rel(want5.numpy(), got5.numpy()) < 1e-15 and rel(want4.numpy(), got4.numpy()) < 1e-15


def test_non_blocking_streamed_solves_complete_after_synchronize():
    """non_blocking=True (torch copy_ semantics): back-to-back streamed type-5 and
    type-4 calls into pinned outputs, one device synchronize, results equal the
    blocking path bitwise; the staging buffers are not recycled under the copies."""
    from paper_1604_06236_b200 import inverse as inv

    P, B = 4096, inv.STREAM_CHUNK * 3 + 5
    t, data = O.make_inputs(P, 0.3, B, 12)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    host = torch.from_numpy(data).pin_memory()
    want5 = nf.refine_type5(plan, host, passes=1)
    want4 = nf.refine_type4(plan, host, passes=1)
    o5, o4 = torch.empty_like(host).pin_memory(), torch.empty_like(host).pin_memory()
    for _ in range(2):
        o5.zero_()
        o4.zero_()
        nf.refine_type5(plan, host, passes=1, out=o5, non_blocking=True)
        nf.refine_type4(plan, host, passes=1, out=o4, non_blocking=True)
        torch.cuda.synchronize()
        assert torch.equal(o5, want5) and torch.equal(o4, want4)


def test_non_blocking_streamed_output_fed_back_as_input():
    """The streamed pipeline persists across calls (uploads of the next call do not
    wait for the caller's stream): a non_blocking output fed straight back as the
    next call's input is still ordered after its own download, and a second plan
    built in between is ordered after its build."""
    from paper_1604_06236_b200 import inverse as inv

    P, B = 4096, inv.STREAM_CHUNK * 2 + 9
    t, data = O.make_inputs(P, 0.3, B, 14)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    host = torch.from_numpy(data).pin_memory()
    want5 = nf.refine_type5(plan, host, passes=1)
    want45 = nf.refine_type4(plan, want5, passes=1)
    t2, _ = O.make_inputs(P, 0.2, 1, 15)
    plan2 = nf.build_plan(nf.validate_grid(t2), nf.MethodParams.from_mu(1e-15, P, 2))
    want2 = nf.type5(plan2, host)
    for _ in range(2):
        o5, o45 = torch.zeros_like(host).pin_memory(), torch.zeros_like(host).pin_memory()
        nf.refine_type5(plan, host, passes=1, out=o5, non_blocking=True)
        nf.refine_type4(plan, o5, passes=1, out=o45, non_blocking=True)
        plan3 = nf.build_plan(nf.validate_grid(t2), nf.MethodParams.from_mu(1e-15, P, 2))
        o2 = torch.zeros_like(host).pin_memory()
        nf.type5(plan3, host, out=o2, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(o5, want5) and torch.equal(o45, want45) and torch.equal(o2, want2)


def test_non_blocking_single_signal_on_two_streams():
    """Single-signal CPU operands with pinned outputs, type 5 and type 4 on two
    streams with non_blocking=True: bitwise equal to the blocking path after a
    device synchronize."""
    P = 1 << 16
    t, data = O.make_inputs(P, 0.3, 1, 13)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    host = torch.from_numpy(data).pin_memory()
    want5 = nf.refine_type5(plan, host, passes=1)
    want4 = nf.refine_type4(plan, host, passes=1)
    o5, o4 = torch.empty_like(host).pin_memory(), torch.empty_like(host).pin_memory()
    side = torch.cuda.Stream()
    for _ in range(3):
        o5.zero_()
        o4.zero_()
        side.wait_stream(torch.cuda.current_stream())
        nf.refine_type5(plan, host, passes=1, out=o5, non_blocking=True)
        with torch.cuda.stream(side):
            nf.refine_type4(plan, host, passes=1, out=o4, non_blocking=True)
        torch.cuda.synchronize()
        assert torch.equal(o5, want5) and torch.equal(o4, want4)


_GAP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
import paper_1604_06236_b200 as nf
P, B = 4096, 40
sp = np.ones(P); sp[1000:1064] = 1.7; sp *= P / sp.sum()
t = (np.cumsum(sp) - sp[0] * 0.5) / P
rng = np.random.default_rng(3)
x = (rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))) / np.sqrt(2)
plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
np.savez(sys.argv[1], t5=nf.type5(plan, x), t4=nf.type4(plan, x), r4=nf.refine_type4(plan, x, passes=1))
"""


@pytest.mark.parametrize("P", [32, 64, 128, 256])
def test_one_cta_small_solves(P):
    """P <= 256 solves run as ONE fused kernel per call (tiny.cu): one launch per
    solve, refined results vs the oracle <= 1e-10 with forward residuals, batched ==
    per-signal and passes=0 == plain bitwise, and the wrap case (a node whose rounded
    centre is n) handled; above P * batch = 2^17 the general path takes over and
    agrees to rounding."""
    from paper_1604_06236_b200 import _lib

    t, data = O.make_inputs(P, 0.45, 3, 900 + P)
    t[np.argmax(t)] = 1.0 - 0.25 / (2 * P)  # rint(2P t) == 2P: centre on the wrap
    grid = nf.validate_grid(t)
    prm = nf.MethodParams.from_mu(1e-15, P, 2)
    plan = nf.build_plan(grid, prm)
    oplan = O.Plan.build(t, prm.damping_a, 2)
    L = _lib.load()
    import torch

    xdev = torch.from_numpy(data[1]).to("cuda")
    before = L.nfft45_launch_count()
    got5_dev = nf.refine_type5(plan, xdev, passes=1)
    assert L.nfft45_launch_count() - before == 1  # device operand: the whole solve is ONE kernel
    before = L.nfft45_launch_count()
    got5 = nf.refine_type5(plan, data[1], passes=1)
    # numpy operand (host pipeline): the same kernel plus the device-side finiteness check
    assert L.nfft45_launch_count() - before == 2
    assert np.array_equal(got5_dev.cpu().numpy(), got5)
    got4 = nf.refine_type4(plan, data[1], passes=1)
    assert rel(O.refine5(oplan, data[1], 1), got5) <= G1 and rel(O.refine4(oplan, data[1], 1), got4) <= G1
    assert rel(data[1], O.type2(got5, t)) <= G1 and rel(data[1], O.type1(t, got4, P)) <= G1
    assert np.array_equal(nf.refine_type5(plan, data, passes=1)[1], got5)
    assert np.array_equal(nf.refine_type4(plan, data, passes=1)[1], got4)
    assert np.array_equal(nf.refine_type5(plan, data[0], passes=0), nf.type5(plan, data[0]))
    assert np.array_equal(nf.refine_type4(plan, data[0], passes=0), nf.type4(plan, data[0]))
    big = np.repeat(data[1:2], (1 << 17) // P + 1, axis=0)  # past the one-CTA threshold
    assert rel(got5, nf.refine_type5(plan, big, passes=1)[-1]) < 1e-12
    assert rel(got4, nf.refine_type4(plan, big, passes=1)[-1]) < 1e-12


def test_persistent_gather_fallback_blocks_bitwise(tmp_path):
    """A grid with a locally stretched stretch of nodes (64 nodes at 1.7x
    spacing) puts some 32-node blocks past the persistent gather's staging
    span; those blocks are recomputed by the chunked kernel.  The operator
    output must be bitwise identical to the chunked kernel run everywhere
    (NFFT45_NO_GPIPE) — the grid is outside the method's accuracy domain, so
    the check is implementation against implementation, not against the
    reference."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_extra in ({}, {"NFFT45_NO_GPIPE": "1"}):
        f = tmp_path / f"gap{len(outs)}.npz"
        env = dict(os.environ, **env_extra)
        subprocess.run([sys.executable, "-c", _GAP_SCRIPT, str(f), root], check=True, env=env, timeout=300)
        outs.append(np.load(f))
    for k in ("t5", "t4", "r4"):
        assert np.array_equal(outs[0][k], outs[1][k]), k


_VARIANT_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[2])
import paper_1604_06236_b200 as nf
out = {}
for P, B, J in [(1000, 1, 0.3), (4096, 1, 0.45), (4096, 4, 0.3), (1 << 16, 1, 0.3), (1 << 18, 1, 0.4),
                (4096, 32, 0.3), (1 << 16, 16, 0.3), (1 << 15, 24, 0.3), (12288, 16, 0.3),
                (2048, 16, 0.3), (1 << 14, 24, 0.45), (1 << 17, 17, 0.3)]:
    rng = np.random.default_rng(P + B)
    t = np.mod((np.arange(P) + rng.uniform(-J, J, P)) / P, 1.0)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(1e-15, P, 2))
    x = (rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))) / np.sqrt(2)
    x = x[0] if B == 1 else x
    out[f"t5_{P}_{B}"] = nf.refine_type5(plan, x, passes=1)
    out[f"t4_{P}_{B}"] = nf.refine_type4(plan, x, passes=1)
np.savez(sys.argv[1], **out)
"""


def test_kernel_variants_bitwise(tmp_path):
    """The launch / tiling variants kept as A/B switches compute the same terms
    in the same order: programmatic dependent launch off (NFFT45_NO_PDL),
    warp-tiled single-signal spreading forced on / off (NFFT45_SPREAD_WARP),
    256-cell spreading tiles (NFFT45_STILE) and 256-node interpolation CTAs
    (NFFT45_GNODES), the TMA-staged pad kernel instead of the LDG-staged
    one (NFFT45_TMA), and the round-2 switches (hybrid / fused chain kernels,
    TMA gather tiles, persistent pad) must all give bitwise the outputs of the
    default build, for single signals on both sides of the warp-tile
    threshold, a 4-signal batch, batch-minor chains and a non-chain size."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    variants = ({}, {"NFFT45_NO_PDL": "1"}, {"NFFT45_SPREAD_WARP": "1"}, {"NFFT45_SPREAD_WARP": "0"},
                {"NFFT45_STILE": "256", "NFFT45_GNODES": "256"}, {"NFFT45_TMA": "1"},
                # round 2: all-column-fast two-FFT kernels instead of the hybrid (warp-local) ones, hybrid
                # without the register / shuffle handoffs, cp.async instead of TMA cell tiles in the
                # persistent gather, the persistent TMA-prefetching pad
                {"NFFT45_HYB": "0"}, {"NFFT45_FUSE": "0"}, {"NFFT45_GATHER_TMA": "0"}, {"NFFT45_PAD_PERSIST": "1"},
                # natural-order fine grid (column pass in place) instead of the row-permuted one, and a
                # blocked permutation
                {"NFFT45_COL_PERM": "0"}, {"NFFT45_COL_BLK": "8"},
                # outputs of the fused pad / mid kernels by per-thread global stores instead of bulk
                # tensor stores (TMA), and the band kernel's output through the TMA unit as well
                {"NFFT45_TMAST": "0"}, {"NFFT45_TMAST": "2"},
                # persistent gather with 8 warps x 4 nodes on 32-signal groups (the default from 64
                # signals up) forced on for these small, ragged batches
                {"NFFT45_GATHER_WARPS": "8"},
                # pipelined spreading on 64-signal groups (two signals per lane, single-buffered
                # amplitudes; the default from 128 signals up) forced on for these small batches
                {"NFFT45_SPREAD_SPL": "2"},
                # FFT_2P column pass on the padded tile with per-thread stores (default: hybrid tile,
                # output through the TMA unit), and the IFFT_2P row pass through the TMA unit as well
                {"NFFT45_PASS_TMAST": "0"}, {"NFFT45_PASS_TMAST": "3"})
    outs = []
    for i, extra in enumerate(variants):
        f = tmp_path / f"v{i}.npz"
        subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, str(f), root], check=True,
                       env=dict(os.environ, **extra), timeout=300)
        outs.append(np.load(f))
    for extra, o in zip(variants[1:], outs[1:]):
        for k in outs[0].files:
            assert np.array_equal(outs[0][k], o[k]), (extra, k)


# ------------------------------------- batched forward transforms on the batch-minor passes

@pytest.mark.parametrize("P,B,J", [(1024, 16, 0.3), (2048, 19, 0.45), (4096, 64, 0.3), (1 << 15, 18, 0.3),
                                   (1 << 16, 17, 0.3), (1 << 17, 16, 0.4)])
def test_batched_forward_fast_path(P, B, J):
    """nfft_type1 / nfft_type2 on batches of 16 or more signals (R = P = Q a power of two in
    2^10 ... 2^17) run on the batch-minor FFT passes with one 2-D boundary kernel per direction
    (chain_bm.cu: kbm_fwd_in / kbm_fwd_out).  Every row must match the oracle's fast transform
    (forward.py:26-102 restated) to 1e-13 and the per-signal path of the library (single signals
    take the signal-major kernels: a different FFT schedule, so roundoff-level differences) to
    1e-13; ragged batches exercise the padded signal groups."""
    t, data = O.make_inputs(P, J, B, 16050 + B)
    g = nf.validate_grid(t)
    got1 = nf.nfft_type1(g, data, P)
    got2 = nf.nfft_type2(data, g)
    assert got1.shape == (B, P) and got2.shape == (B, P)
    for r in sorted({0, 7, B - 2, B - 1}):
        assert rel(O.type1(t, data[r], P), got1[r]) <= 1e-13
        assert rel(O.type2(data[r], t), got2[r]) <= 1e-13
        assert rel(nf.nfft_type1(g, data[r], P), got1[r]) <= 1e-13
        assert rel(nf.nfft_type2(data[r], g), got2[r]) <= 1e-13
    if P <= 2048:  # exact direct sums (forward.py:105-130)
        assert rel(O.type1_exact(t, data[B - 1], P), got1[B - 1]) <= 1e-12
        assert rel(O.type2_exact(data[B - 1], t), got2[B - 1]) <= 1e-12


_FWD_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[2])
import paper_1604_06236_b200 as nf
rng = np.random.default_rng(5)
P, B = 4096, 24
t = np.mod((np.arange(P) + rng.uniform(-0.3, 0.3, P)) / P, 1.0)
g = nf.validate_grid(t)
x = (rng.standard_normal((B, P)) + 1j * rng.standard_normal((B, P))) / np.sqrt(2)
plan = nf.build_plan(g, nf.MethodParams.from_mu(1e-15, P, 2))
np.savez(sys.argv[1], t1=nf.nfft_type1(g, x, P), t2=nf.nfft_type2(x, g),
         r5=nf.refine_type5(plan, x, passes=2), r4=nf.refine_type4(plan, x, passes=2))
"""


def test_batched_forward_fast_path_vs_generic(tmp_path):
    """The batch-minor forward path against the generic batched path (NFFT45_NO_FORWARD_BM=1:
    signal-major spread / four-step FFT / band kernels), and inside the UNFUSED refinement
    (NFFT45_NO_CHAIN=1: solve, forward transform with the subtrahend fused, solve), whose forward
    transforms take the fast path with a subtrahend: roundoff-level agreement."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for i, extra in enumerate(({}, {"NFFT45_NO_FORWARD_BM": "1"}, {"NFFT45_NO_CHAIN": "1"},
                               {"NFFT45_NO_CHAIN": "1", "NFFT45_NO_FORWARD_BM": "1"})):
        f = tmp_path / f"f{i}.npz"
        subprocess.run([sys.executable, "-c", _FWD_SCRIPT, str(f), root], check=True, env=dict(os.environ, **extra),
                       timeout=300)
        outs.append(np.load(f))
    for k in ("t1", "t2"):
        assert rel(outs[1][k], outs[0][k]) <= 1e-13
        assert not np.array_equal(outs[1][k], outs[0][k])  # the switch really selects another path
    for k in ("r5", "r4"):
        assert rel(outs[0][k], outs[2][k]) <= 1e-11 and rel(outs[3][k], outs[2][k]) <= 1e-11


# ------------------------------------- fused multi-pass type-4 refinement

@pytest.mark.parametrize("B", [1, 20])
def test_type4_multi_pass_on_fused_chains(B):
    """refine_type4 with passes >= 2 runs on the fused chains (signal-major for
    B < 16, batch-minor otherwise): the band epilogue stores the residual for
    the NonConvergence norms (inverse.py:146-185).  Over-damped cell where the
    second pass matters (J = 0.45, mu = 1e-17): vs the oracle at 2 and 3 passes."""
    P = 4096
    t, data = O.make_inputs(P, 0.45, B, 16048)
    prm = nf.MethodParams.from_mu(1e-17, P, 2)
    plan = nf.build_plan(nf.validate_grid(t), prm)
    oplan = O.Plan.build(t, prm.damping_a, 2)
    x = data if B > 1 else data[0]
    for passes in (2, 3):
        got = np.atleast_2d(nf.refine_type4(plan, x, passes=passes))
        for r in sorted({0, B - 1}):
            assert rel(O.refine4(oplan, data[r], passes), got[r]) <= G1
            assert rel(data[r], O.type1(t, got[r], P)) <= G1


@pytest.mark.parametrize("B", [1, 20])
def test_type4_multi_pass_nonconvergence_on_fused_chains(B):
    """eta = 1, J = 0.45 at P = 4096, deep in the over-damped corner (mu = 1e-24,
    roundoff amplified beyond 1 for any fp64 implementation): the reference's
    residual grows between passes (oracle raises) and so does ours — the fused
    chain path raises NonConvergenceError.  (Between mu ~ 1e-16 and ~1e-22 this
    path's more accurate phases still contract where the reference diverges.)"""
    P = 4096
    mu = 1e-24
    t, data = O.make_inputs(P, 0.45, B, 16048)
    with pytest.raises(O.NonConvergence):
        O.refine4(O.Plan.build(t, O.damping(mu, P, 1), 1), data[0], 4)
    plan = nf.build_plan(nf.validate_grid(t), nf.MethodParams.from_mu(mu, P, 1))
    with pytest.raises(nf.NonConvergenceError):
        nf.refine_type4(plan, data if B > 1 else data[0], passes=4)

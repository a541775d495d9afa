"""The reference's hot-path test strategy (pkg/tests/test_forward.py,
test_lagrange.py, test_inverse.py) re-stated against the CUDA drop-in:
closed forms, brute-force oracles, invariants, determinism and error paths.
Every call below runs libnfft45 kernels on cuda:0."""

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1604_06236_b200 as nf
import paper_1604_06236_b200.lagrange as lagrange_mod

pytestmark = pytest.mark.gpu


def jittered(P, rng, jitter=0.6):
    return nf.validate_grid(np.arange(P) / P + rng.uniform(0, jitter / P, P))


def randc(n, rng):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def rel(truth, got):
    truth = np.asarray(truth)
    return np.linalg.norm(np.asarray(got) - truth) / np.linalg.norm(truth)


def std_params(P, mu=1e-11, eta=2, **kw):
    return nf.MethodParams.from_mu(mu, P, eta, **kw)


def dense(grid, sign):
    """Phase matrix e^{sign 2 pi i p t_q} (rows p) with exact integer-part removal."""
    p = np.arange(grid.size, dtype=np.longdouble)
    ph = np.mod(np.outer(p, np.asarray(grid.instants, dtype=np.longdouble)), 1.0).astype(np.float64)
    return np.exp(sign * 2j * np.pi * ph)


# ------------------------------------------------------------------ forward

def test_direct_sums_match_naive_loops():
    rng = np.random.default_rng(0)
    g = jittered(5, rng)
    a = randc(5, rng)
    naive1 = np.array([sum(a[q] * np.exp(-2j * np.pi * p * g.instants[q]) for q in range(5)) for p in range(7)])
    assert np.abs(nf.nfft_type1_direct(g, a, 7) - naive1).max() < 1e-13
    S = randc(6, rng)
    naive2 = np.array([sum(S[p] * np.exp(2j * np.pi * p * t) for p in range(6)) for t in g.instants])
    assert np.abs(nf.nfft_type2_direct(S, g) - naive2).max() < 1e-13


def test_type1_single_node_at_zero():
    out = nf.nfft_type1(nf.validate_grid([0.0]), [1.0], 4)
    assert np.abs(out - 1.0).max() < 1e-13


def test_uniform_grids_reduce_to_dfts():
    rng = np.random.default_rng(3)
    Q = 16
    g = nf.validate_grid(np.arange(Q) / Q)
    a = randc(Q, rng)
    assert rel(np.fft.fft(a), nf.nfft_type1(g, a, Q)) < 1e-13
    assert rel(Q * np.fft.ifft(a), nf.nfft_type2(a, g)) < 1e-13
    assert rel(np.fft.fft(a), nf.dft(a)) < 1e-14 and rel(np.fft.ifft(a), nf.idft(a)) < 1e-14


@pytest.mark.parametrize("Q,R", [(7, 16), (33, 8), (16, 48), (5, 1), (100, 60), (64, 200)])
def test_type1_rectangular_sizes(Q, R):
    rng = np.random.default_rng(5)
    g = nf.validate_grid(np.sort(rng.uniform(0, 1, Q)))
    a = randc(Q, rng)
    assert rel(nf.nfft_type1_direct(g, a, R), nf.nfft_type1(g, a, R)) < 1e-12


@pytest.mark.parametrize("P", [8, 11, 16, 64, 96, 1000])
def test_fast_paths_track_direct_sums(P):
    rng = np.random.default_rng(9)
    g = jittered(P, rng)
    a = randc(P, rng)
    assert rel(nf.nfft_type1_direct(g, a, P), nf.nfft_type1(g, a, P)) < 1e-12
    assert rel(nf.nfft_type2_direct(a, g), nf.nfft_type2(a, g)) < 1e-12


def test_type2_constant_polynomial():
    rng = np.random.default_rng(6)
    g = jittered(11, rng)
    S = np.zeros(11, dtype=complex)
    S[0] = 2.5 - 1j
    assert np.abs(nf.nfft_type2(S, g) - S[0]).max() < 1e-12


def test_adjoint_consistency():
    rng = np.random.default_rng(10)
    P = 64
    g = jittered(P, rng)
    x, y = randc(P, rng), randc(P, rng)
    lhs = np.vdot(y, nf.nfft_type1(g, x, P))
    rhs = np.vdot(nf.nfft_type2(y, g), x)
    assert abs(lhs - rhs) / abs(lhs) < 1e-11


def test_conv_properties():
    rng = np.random.default_rng(11)
    g = jittered(6, rng)
    a = randc(6, rng)
    lam = np.zeros(12)
    lam[0] = 1.0
    assert np.abs(nf.nonuniform_conv(g, a, lam, 6) - a.sum()).max() < 1e-12
    P = 8
    lam = randc(2 * P, rng)
    out = nf.nonuniform_conv(nf.validate_grid([0.0]), [1.0], lam, P)
    want = np.array([np.sum(lam * np.exp(2j * np.pi * np.arange(2 * P) * k / P)) for k in range(P)])
    assert rel(want, out) < 1e-12
    g7 = jittered(7, rng)
    a, b = randc(7, rng), randc(7, rng)
    l1, l2 = randc(14, rng), randc(14, rng)
    assert rel(nf.nonuniform_conv(g7, a, l1, 7) + 3j * nf.nonuniform_conv(g7, b, l1, 7),
               nf.nonuniform_conv(g7, a + 3j * b, l1, 7)) < 1e-11
    assert rel(nf.nonuniform_conv(g7, a, l1, 7) + 2.0 * nf.nonuniform_conv(g7, a, l2, 7),
               nf.nonuniform_conv(g7, a, l1 + 2.0 * l2, 7)) < 1e-11
    with pytest.raises(nf.SizeMismatchError):
        nf.nonuniform_conv(g, randc(6, rng), randc(13, rng), 6)


def test_accuracy_improves_with_spread_width():
    rng = np.random.default_rng(16)
    P = 32
    for _ in range(5):
        g = jittered(P, rng)
        a = randc(P, rng)
        truth = nf.nfft_type1_direct(g, a, P)
        errs = [rel(truth, nf.nfft_type1(g, a, P, kernel=nf.kernel_for_size(P, m))) for m in (4, 8, 12)]
        assert errs[1] < errs[0] and errs[2] < errs[1]


def test_kernel_size_mismatch():
    rng = np.random.default_rng(1)
    g = jittered(8, rng)
    with pytest.raises(nf.SizeMismatchError):
        nf.nfft_type1(g, randc(8, rng), 8, kernel=nf.kernel_for_size(9))


# ------------------------------------------------------------------ Lagrange

def v_direct(grid, a):
    q = np.arange(grid.size) / grid.size
    return np.array([np.sum(np.log(1 - np.exp(2j * np.pi * (qq - grid.instants + 1j * a)))) for qq in q])


def poly_coefficients(grid):
    c = np.array([1.0 + 0j])
    for t in grid.instants:
        c = np.convolve(c, np.array([-np.exp(2j * np.pi * t), 1.0]))
    return c


def test_v_samples():
    g = nf.validate_grid([0.0])
    prm = nf.MethodParams.from_mu(1e-12, 1, eta=4)
    v = nf.compute_v_samples(g, prm)
    assert abs(v[0] - np.log(1 - np.exp(-2 * np.pi * prm.damping_a))) < 1e-11
    rng = np.random.default_rng(0)
    g = jittered(8, rng)
    prm = nf.MethodParams.from_mu(1e-13, 8, eta=2)
    assert np.abs(nf.compute_v_samples(g, prm) - v_direct(g, prm.damping_a)).max() < 10 * prm.mu * 8 + 1e-12
    g = jittered(8, np.random.default_rng(1))
    errs = [np.abs(nf.compute_v_samples(g, nf.MethodParams.from_damping(0.05, 8, e)) - v_direct(g, 0.05)).max()
            for e in (1, 2)]
    assert errs[1] < errs[0]


def test_kernel_samples():
    P = 8
    g = nf.validate_grid(np.arange(P) / P)
    prm = nf.MethodParams.from_mu(1e-13, P, eta=2)
    ks = nf.kernel_samples_from_v(nf.compute_v_samples(g, prm), g)
    assert np.abs(ks - (np.exp(-2 * np.pi * P * prm.damping_a) - 1.0)).max() < 1e-11
    rng = np.random.default_rng(2)
    g = jittered(P, rng)
    ks = nf.kernel_samples_from_v(nf.compute_v_samples(g, prm), g)
    z = np.exp(2j * np.pi * (np.arange(P) / P + 1j * prm.damping_a))
    direct = np.array([np.prod(zz - np.exp(2j * np.pi * g.instants)) for zz in z])
    assert rel(direct, ks) < 1e-11
    with pytest.raises(nf.KernelOverflowError):
        nf.kernel_samples_from_v(np.array([800.0 + 0j, -800.0 + 0j]), nf.validate_grid([0.0, 0.5]))


def test_coefficients():
    P = 16
    g = nf.validate_grid(np.arange(P) / P)
    prm = nf.MethodParams.from_mu(1e-14, P, eta=6)
    L = nf.kernel_coefficients(nf.kernel_samples_from_v(nf.compute_v_samples(g, prm), g), prm)
    want = np.zeros(P, dtype=complex)
    want[0] = -1.0
    assert np.abs(L - want).max() < 1e-12
    g = nf.validate_grid([0.3173])
    prm = nf.MethodParams.from_mu(1e-12, 1, eta=4)
    L = nf.kernel_coefficients(nf.kernel_samples_from_v(nf.compute_v_samples(g, prm), g), prm)
    assert abs(L[0] + np.exp(2j * np.pi * 0.3173)) < 1e-10
    rng = np.random.default_rng(3)
    g = jittered(8, rng)
    prm = nf.MethodParams.from_mu(1e-11, 8, eta=2)
    L = nf.kernel_coefficients(nf.kernel_samples_from_v(nf.compute_v_samples(g, prm), g), prm)
    assert rel(poly_coefficients(g)[:8], L) < 1e-10
    with pytest.warns(nf.AmplificationWarning):
        nf.kernel_coefficients(np.ones(64, dtype=complex), nf.MethodParams.from_damping(0.1, 64, eta=1))


def test_derivative_samples():
    P = 16
    g = nf.validate_grid(np.arange(P) / P)
    plan = nf.build_plan(g, nf.MethodParams.from_mu(1e-14, P, eta=6))
    assert rel(P * np.exp(-2j * np.pi * np.arange(P) / P), plan.kernel_data.derivative_samples) < 1e-12
    plan1 = nf.build_plan(nf.validate_grid([0.77]), nf.MethodParams.from_mu(1e-12, 1, eta=4))
    assert abs(plan1.kernel_data.derivative_samples[0] - 1.0) < 1e-10
    rng = np.random.default_rng(4)
    g = jittered(8, rng)
    prm = nf.MethodParams.from_mu(1e-11, 8, eta=2)
    kd = nf.build_plan(g, prm).kernel_data
    z = np.exp(2j * np.pi * g.instants)
    direct = np.array([np.prod(z[j] - np.delete(z, j)) for j in range(8)])
    assert rel(direct, kd.derivative_samples) < 1e-10
    # the standalone pipeline agrees with the fused plan
    dL = nf.derivative_samples(kd.coefficients, g)
    assert rel(kd.derivative_samples, dL) < 1e-12


def test_singular_derivative_guard(monkeypatch):
    g = nf.validate_grid(np.arange(4) / 4)
    vanishing = np.array([1.0, 0.0, 1.0, 1.0], dtype=complex)
    monkeypatch.setattr(lagrange_mod, "nfft_type2", lambda *a, **k: vanishing)
    with pytest.raises(nf.SingularDerivativeError):
        nf.derivative_samples(np.zeros(4, dtype=complex), g)


def test_node_order_invariance():
    rng = np.random.default_rng(5)
    P = 8
    t = np.sort(rng.uniform(0, 1, P))
    perm = rng.permutation(P)
    prm = nf.MethodParams.from_mu(1e-11, P, eta=2)
    d1 = nf.build_plan(nf.validate_grid(t), prm).kernel_data
    d2 = nf.build_plan(nf.validate_grid(t[perm]), prm).kernel_data
    assert rel(d1.v_samples, d2.v_samples) < 1e-12
    assert rel(d1.kernel_samples, d2.kernel_samples) < 1e-12
    assert rel(d1.coefficients, d2.coefficients) < 1e-9
    assert rel(d1.derivative_samples[perm], d2.derivative_samples) < 1e-9


def test_kernel_identity_end_to_end():
    rng = np.random.default_rng(7)
    for P in (8, 12, 16):
        g = jittered(P, rng)
        prm = nf.MethodParams.from_mu(1e-12, P, eta=2)
        kd = nf.build_plan(g, prm).kernel_data
        z = np.exp(2j * np.pi * (np.arange(P) / P + 1j * prm.damping_a))
        full = np.concatenate((kd.coefficients, [1.0]))
        rebuilt = np.array([np.polyval(full[::-1], zz) for zz in z])
        assert rel(rebuilt, kd.kernel_samples) < 1e-9


# ------------------------------------------------------------------ inverse

def test_plan_closed_forms_and_fields():
    P = 16
    g = nf.validate_grid(np.arange(P) / P)
    prm = nf.MethodParams.from_mu(1e-14, P, eta=6)
    plan = nf.build_plan(g, prm)
    a = prm.damping_a
    p = np.arange(P)
    h = 1.0 / (np.exp(-2 * np.pi * P * a) - 1.0)
    assert rel(h / P * np.ones(P), plan.node_weights) < 1e-11
    assert rel(np.exp(-2 * np.pi * p * a), plan.h1_coefficients) < 1e-14
    assert np.all(np.diff(plan.h1_coefficients) < 0) and np.all(plan.h1_coefficients > 0)
    assert plan.size == P and not plan.node_weights.flags.writeable
    rng = np.random.default_rng(1)
    g = jittered(8, rng)
    plan = nf.build_plan(g, std_params(8))
    z = np.exp(2j * np.pi * g.instants)
    dL = np.array([np.prod(z[j] - np.delete(z, j)) for j in range(8)])
    hh = 1.0 / (np.exp(-2j * np.pi * 8 * g.instants) * np.exp(-2 * np.pi * 8 * std_params(8).damping_a) - 1.0)
    assert rel(hh / (dL * z), plan.node_weights) < 1e-9


def test_plan_rebuild_and_reuse_are_bitwise():
    rng = np.random.default_rng(0)
    g = jittered(32, rng)
    prm = std_params(32)
    p1, p2 = nf.build_plan(g, prm), nf.build_plan(g, prm)
    assert np.array_equal(p1.node_weights, p2.node_weights)
    assert np.array_equal(p1.kernel_data.kernel_samples, p2.kernel_data.kernel_samples)
    s1, s2 = randc(32, rng), randc(32, rng)
    assert np.array_equal(nf.type5(p1, s1), nf.type5(nf.build_plan(g, prm), s1))
    assert np.array_equal(nf.type5(p1, s2), nf.type5(p2, s2))


def test_type5_known_answers():
    rng = np.random.default_rng(2)
    P = 16
    plan = nf.build_plan(jittered(P, rng), std_params(P))
    c = 1.5 - 0.5j
    want = np.zeros(P, dtype=complex)
    want[0] = c
    assert np.abs(nf.type5(plan, np.full(P, c)) - want).max() < 1e-9
    g = nf.validate_grid(np.arange(P) / P)
    plan = nf.build_plan(g, nf.MethodParams.from_mu(1e-14, P, eta=6))
    s = randc(P, rng)
    assert rel(np.fft.fft(s) / P, nf.type5(plan, s)) < 1e-12
    A = randc(P, rng)
    assert rel(np.fft.ifft(A), nf.type4(plan, A)) < 1e-12


def test_type4_impulse():
    rng = np.random.default_rng(5)
    P = 16
    g = jittered(P, rng)
    plan = nf.build_plan(g, std_params(P))
    want = np.zeros(P, dtype=complex)
    want[3] = 1.0
    got = nf.type4(plan, np.exp(-2j * np.pi * np.arange(P) * g.instants[3]))
    assert np.abs(got - want).max() < 1e-9


@pytest.mark.parametrize("seed", [4, 7])
def test_against_dense_solves(seed):
    rng = np.random.default_rng(seed)
    P = 8
    g = jittered(P, rng)
    plan = nf.build_plan(g, std_params(P))
    s = randc(P, rng)
    want5 = np.linalg.solve(dense(g, +1).T, s)   # sum_p S_p e^{2 pi i p t_q} = s_q
    assert rel(want5, nf.type5(plan, s)) < 1e-10
    assert rel(want5, nf.refine_type5(plan, s, passes=1)) < 1e-13
    A = randc(P, rng)
    want4 = np.linalg.solve(dense(g, -1), A)      # sum_q a_q e^{-2 pi i p t_q} = A_p
    assert rel(want4, nf.type4(plan, A)) < 1e-10
    assert rel(want4, nf.refine_type4(plan, A, passes=1)) < 1e-13


def test_round_trip_residuals_and_linearity():
    rng = np.random.default_rng(8)
    P = 64
    g = jittered(P, rng)
    plan = nf.build_plan(g, std_params(P))
    s = randc(P, rng)
    assert rel(s, nf.nfft_type2_direct(nf.type5(plan, s), g)) < 1e-9
    A = randc(P, rng)
    assert rel(A, nf.nfft_type1_direct(g, nf.type4(plan, A), P)) < 1e-9
    g = jittered(32, np.random.default_rng(9))
    plan = nf.build_plan(g, std_params(32))
    x, y = randc(32, rng), randc(32, rng)
    al, be = 1.5 - 2j, -0.25 + 1j
    for fn in (nf.type4, nf.type5):
        assert rel(al * fn(plan, x) + be * fn(plan, y), fn(plan, al * x + be * y)) < 1e-12


def test_refinement_semantics():
    rng = np.random.default_rng(12)
    P = 32
    plan = nf.build_plan(jittered(P, rng), std_params(P, refine_passes=1))
    A, s = randc(P, rng), randc(P, rng)
    assert np.array_equal(nf.refine_type4(plan, A, passes=0), nf.type4(plan, A))
    assert np.array_equal(nf.refine_type5(plan, s, passes=0), nf.type5(plan, s))
    assert np.array_equal(nf.refine_type4(plan, A), nf.refine_type4(plan, A, passes=1))
    assert np.array_equal(nf.refine_type5(plan, s), nf.refine_type5(plan, s, passes=1))
    # a negative count runs no pass (the reference loops over range(passes))
    assert np.array_equal(nf.refine_type4(plan, A, passes=-3), nf.type4(plan, A))
    assert np.array_equal(nf.refine_type5(plan, s, passes=-1), nf.type5(plan, s))


def test_refine_contracts_error():
    P = 256
    prm = nf.MethodParams.from_mu(1e-6, P, eta=1)
    wins = 0
    for trial in range(4):
        g, a_true = nf.generate_trial(P, 100 + trial)
        spectrum = nf.nfft_type1_direct(g, a_true, P)
        plan = nf.build_plan(g, prm)
        e_plain = rel(a_true, nf.type4(plan, spectrum))
        e_ref = rel(a_true, nf.refine_type4(plan, spectrum, passes=1))
        wins += np.log10(e_ref) <= 1.5 * np.log10(e_plain)
    assert wins >= 3
    for trial in range(4):
        g, S_true = nf.generate_trial(P, 200 + trial)
        samples = nf.nfft_type2_direct(S_true, g)
        plan = nf.build_plan(g, prm)
        r0 = rel(samples, nf.nfft_type2_direct(nf.type5(plan, samples), g))
        r1 = rel(samples, nf.nfft_type2_direct(nf.refine_type5(plan, samples, passes=1), g))
        assert r1 < r0


def test_nonconvergence_detection():
    P = 64
    g, _ = nf.generate_trial(P, 42)
    plan = nf.build_plan(g, nf.MethodParams.from_mu(1e-2, P, eta=1))
    A = randc(P, np.random.default_rng(14))
    with pytest.raises(nf.NonConvergenceError):
        nf.refine_type4(plan, A, passes=4)


def test_concurrent_solves_share_one_plan():
    rng = np.random.default_rng(15)
    P = 128
    plan = nf.build_plan(jittered(P, rng), std_params(P))
    inputs = [randc(P, rng) for _ in range(8)]
    serial = [nf.type4(plan, x) for x in inputs]
    with ThreadPoolExecutor(max_workers=4) as pool:
        threaded = list(pool.map(lambda x: nf.type4(plan, x), inputs))
    for a, b in zip(serial, threaded):
        assert np.array_equal(a, b)


def test_concurrent_plan_builds_share_one_node_set():
    """Plans built at the same time on one node-set handle (each build launches the node
    set's caches and publishes them after its own stream synchronize; the losers of the race
    drop their copies) give bitwise the tables and solves of a serial build."""
    rng = np.random.default_rng(151)
    P = 4096
    t = np.arange(P) / P + rng.uniform(0, 0.6 / P, P)
    prm = std_params(P)
    ref_plan = nf.build_plan(nf.validate_grid(t), prm)
    x = randc(P, rng)
    want5, want4 = nf.refine_type5(ref_plan, x, passes=1), nf.refine_type4(ref_plan, x, passes=1)
    g = nf.validate_grid(t)  # fresh handle: no cached tile ranges / gather flags yet
    g.device_handle(0)
    with ThreadPoolExecutor(max_workers=4) as pool:
        plans = list(pool.map(lambda _: nf.build_plan(g, prm), range(8)))
    for p in plans:
        assert np.array_equal(p.kernel_data.kernel_samples, ref_plan.kernel_data.kernel_samples)
        assert np.array_equal(nf.refine_type5(p, x, passes=1), want5)
        assert np.array_equal(nf.refine_type4(p, x, passes=1), want4)
    batch = np.stack([x, 2 * x, x[::-1]] * 6)  # 18 rows: the batch-minor chains and the persistent gather
    got = nf.refine_type5(plans[-1], batch, passes=1)
    assert np.array_equal(got, nf.refine_type5(ref_plan, batch, passes=1))


@pytest.mark.parametrize("lgN,B", [(11, 16), (12, 19), (13, 16), (14, 17), (15, 16), (16, 24), (17, 16), (18, 17)])
def test_batched_dft(lgN, B):
    """dft / idft of batches of rows of length 2^11 ... 2^18 (the four-step Stockham passes of
    fft.cu, forward.py:21-23): numpy's FFT to roundoff, every row equal to the single-row call,
    ragged batches."""
    rng = np.random.default_rng(lgN)
    N = 1 << lgN
    x = rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))
    X = nf.dft(x)
    assert X.shape == (B, N)
    assert rel(np.fft.fft(x, axis=-1), X) < 1e-14
    assert rel(np.fft.ifft(x, axis=-1), nf.idft(x)) < 1e-14
    for r in (0, B - 1):
        assert rel(nf.dft(x[r]), X[r]) < 1e-14
    assert rel(x, nf.idft(X)) < 1e-14


def test_flop_reports_match_reference(golden):
    def rep(fc):
        r = fc.report()
        return [r.real_adds, r.complex_adds, r.real_muls, r.complex_muls, r.complex_exps, r.total_flops] + list(
            r.fft_invocations)

    g = nf.validate_grid(golden["flops_t"])
    prm = nf.MethodParams.from_mu(1e-11, 64, 2)
    fc = nf.FlopCounter()
    plan = nf.build_plan(g, prm, flops=fc)
    assert rep(fc) == list(golden["flops_build_plan"])
    x = np.ones(64, dtype=complex)
    for name, fn in (("type5", lambda f: nf.type5(plan, x, flops=f)), ("type4", lambda f: nf.type4(plan, x, flops=f)),
                     ("refine5", lambda f: nf.refine_type5(plan, x, passes=1, flops=f)),
                     ("refine4", lambda f: nf.refine_type4(plan, x, passes=1, flops=f)),
                     ("type1", lambda f: nf.nfft_type1(g, x, 48, flops=f)),
                     ("type2", lambda f: nf.nfft_type2(x, g, flops=f)),
                     ("conv", lambda f: nf.nonuniform_conv(g, x, np.ones(128, dtype=complex), 64, flops=f)),
                     ("conv_real", lambda f: nf.nonuniform_conv(g, x, np.ones(128), 64, flops=f))):
        fc = nf.FlopCounter()
        fn(fc)
        assert rep(fc) == list(golden[f"flops_{name}"]), name
    c4, c5 = nf.FlopCounter(), nf.FlopCounter()
    nf.type4(plan, x, flops=c4)
    nf.type5(plan, x, flops=c5)
    assert c4.report() == c5.report()


def test_input_validation_errors():
    rng = np.random.default_rng(1)
    g = jittered(8, rng)
    plan = nf.build_plan(g, std_params(8))
    with pytest.raises(nf.LengthMismatchError):
        nf.type5(plan, np.ones(7))
    with pytest.raises(ValueError):
        nf.type4(plan, np.full(8, np.nan))
    with pytest.raises(nf.LengthMismatchError):
        nf.nfft_type1(g, np.ones(9), 8)
    with pytest.raises(ValueError):
        nf.nfft_type1(g, np.ones(8), 0)


# ------------------------------------------- advisor findings (round 1)

@pytest.mark.parametrize("P,batch", [(64, 3), (1000, 2), (4096, 1), (4096, 20), (1 << 14, 40)])
@pytest.mark.parametrize("kind", [5, 4])
def test_refine_in_place_out_equals_input(P, batch, kind):
    """out= aliasing the operand (S_dev == s_dev) gives the out-of-place result:
    the refinement re-reads its operand after writing x (tiny, chain and generic paths)."""
    import torch

    rng = np.random.default_rng(P + batch)
    g = jittered(P, rng)
    plan = nf.build_plan(g, std_params(P, mu=1e-15))
    x = torch.from_numpy(np.stack([randc(P, rng) for _ in range(batch)])).cuda()
    fn = nf.refine_type5 if kind == 5 else nf.refine_type4
    for passes in (1, 2):
        ref = fn(plan, x, passes=passes)
        y = x.clone()
        got = fn(plan, y, passes=passes, out=y)
        assert got.data_ptr() == y.data_ptr()
        assert torch.equal(ref, y), (passes, float((ref - y).abs().max()))


def test_more_than_65535_rows_at_non_power_of_two_size():
    """Batched launches walk rows in slices of 65535 (gridDim.y cap): forward
    NFFTs, DFTs and solves with 70000 rows match the row-wise results."""
    import torch

    rng = np.random.default_rng(70000)
    P, rows = 6, 70000
    g = jittered(P, rng)
    plan = nf.build_plan(g, std_params(P, mu=1e-11))
    x = torch.from_numpy(rng.standard_normal((rows, P)) + 1j * rng.standard_normal((rows, P))).cuda()
    pick = [0, 1, 65534, 65535, 65536, rows - 1]

    def close(a, b):  # batched and single-row kernels may differ in rounding only
        return float((a - b).abs().max() / b.abs().max()) < 1e-12

    out = nf.nfft_type2(x, g)
    for r in pick:
        assert close(out[r], nf.nfft_type2(x[r:r + 1], g)[0])
    d = nf.dft(x)
    for r in pick:
        assert close(d[r], nf.dft(x[r:r + 1])[0])
    for fn in (nf.refine_type5, nf.refine_type4):
        y = fn(plan, x, passes=1)
        for r in pick:
            assert close(y[r], fn(plan, x[r:r + 1], passes=1)[0])


def test_graph_cache_stays_bounded_with_fresh_outputs():
    """A plan fed a fresh output buffer on every call keeps working (the
    capture-candidate table is trimmed) and results stay bitwise equal."""
    import torch

    rng = np.random.default_rng(11)
    P = 4096
    g = jittered(P, rng)
    plan = nf.build_plan(g, std_params(P, mu=1e-15))
    x = torch.from_numpy(randc(P, rng)).cuda()
    ref = nf.refine_type5(plan, x, passes=1)
    keep = []
    for _ in range(600):
        keep.append(nf.refine_type5(plan, x, passes=1))
    assert all(torch.equal(ref, k) for k in keep[::50])


@pytest.mark.parametrize("P,batch", [(4096, 150), (1 << 16, 3), (64, 1), (1000, 70)])
def test_numpy_operands_staged_path(P, batch):
    """numpy (pageable) operands stream through pinned staging slots filled by
    the copy pool; results equal the device-resident solve bitwise, and a
    non-finite entry anywhere raises ValueError like the reference
    (grid.py:30-31), checked on the device over the staged chunks."""
    import torch

    rng = np.random.default_rng(P + batch)
    g = jittered(P, rng)
    plan = nf.build_plan(g, std_params(P, mu=1e-15))
    x = rng.standard_normal((batch, P)) + 1j * rng.standard_normal((batch, P))
    x1 = x[0] if batch == 1 else x
    for fn, label in ((nf.refine_type5, "samples"), (nf.refine_type4, "spectrum")):
        got = fn(plan, x1, passes=1)
        assert isinstance(got, np.ndarray) and got.shape == x1.shape
        dev = fn(plan, torch.from_numpy(np.ascontiguousarray(x1)).cuda(), passes=1).cpu().numpy()
        assert np.array_equal(got, dev)
        bad = x1.copy()
        bad.reshape(-1)[bad.size - 3] = np.nan + 0j
        with pytest.raises(ValueError, match=f"{label} contains NaN or Inf entries"):
            fn(plan, bad, passes=1)
        bad = x1.copy()
        bad.reshape(-1)[0] = complex(0.0, np.inf)
        with pytest.raises(ValueError, match="NaN or Inf"):
            (nf.type5 if label == "samples" else nf.type4)(plan, bad)
        # the pipeline is still usable after an error
        assert np.array_equal(fn(plan, x1, passes=1), got)

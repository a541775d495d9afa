"""Host-side logic of the drop-in (no GPU): parameter relations, validation,
error mapping, window metadata and the analytic flop accounting — checked
against the reference's semantics and its recorded values."""

import os
import warnings

import numpy as np
import pytest

import paper_1604_06236_b200 as nf
from paper_1604_06236_b200 import flops as F
from paper_1604_06236_b200 import inverse as inv
from oracle import nfft_oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# --- MethodParams / Eq. 49 (grid.py:99-160) -------------------------------------

@pytest.mark.parametrize("P,eta,mu", [(8, 2, 1e-11), (64, 2, 1e-15), (256, 1, 1e-6), (4096, 3, 1e-13)])
def test_damping_matches_oracle_and_round_trips(P, eta, mu):
    a = nf.damping_from_mu(mu, P, eta)
    assert a == O.damping(mu, P, eta)
    assert nf.mu_from_damping(a, P, eta) == pytest.approx(mu, rel=1e-12)
    prm = nf.MethodParams.from_mu(mu, P, eta)
    assert prm.damping_a == a and prm.spread_width == 14 and prm.refine_passes == 1
    assert nf.MethodParams.from_damping(a, P, eta).mu == pytest.approx(mu, rel=1e-12)


def test_params_validation():
    with pytest.raises(nf.NonPositiveDampingError):
        nf.damping_from_mu(0.5, 4, 1)
    with pytest.raises(nf.NonPositiveDampingError):
        nf.damping_from_mu(1e-3, 1, 1)
    with pytest.raises(nf.NonPositiveDampingError):
        nf.mu_from_damping(0.0, 8, 1)
    with pytest.raises(ValueError):
        nf.MethodParams(damping_a=0.1, eta=1.5, mu=1e-3)
    with pytest.raises(ValueError):
        nf.MethodParams(damping_a=0.1, eta=1, mu=1e-3, refine_passes=-1)
    with pytest.raises(nf.NonPositiveDampingError):
        nf.MethodParams(damping_a=-1.0, eta=1, mu=1e-3)


# --- validate_grid (grid.py:64-96) through the C library ---------------------------

def test_fractional_eta_extension_params():
    """The reference contract (integer eta, grid.py:143-144) is the default;
    fractional_eta=True is the config-5 extension, eta * P must be integral."""
    with pytest.raises(ValueError):
        nf.MethodParams.from_mu(1e-15, 4096, 1.5)
    prm = nf.MethodParams.from_mu(1e-15, 4096, 1.5, fractional_eta=True)
    assert prm.series_terms(4096) == 6144
    assert prm.damping_a == nf.damping_from_mu(1e-15, 4096, 1.5)
    with pytest.raises(ValueError):
        prm.series_terms(4095)
    with pytest.raises(ValueError):
        nf.MethodParams(damping_a=0.1, eta=0.5, mu=1e-3, fractional_eta=True)
    assert nf.MethodParams.from_mu(1e-15, 64, 2).series_terms(64) == 128


@pytest.mark.parametrize("eta", [1, 2, 3])
def test_oracle_series_terms_restatement_reduces_to_reference(eta):
    """v_samples_terms (extension) with R = eta P is the reference's v_samples, bitwise."""
    t, _ = O.make_inputs(16, 0.3, 1, 5)
    a = O.damping(1e-12, 16, eta)
    assert np.array_equal(O.v_samples_terms(t, a, eta * 16), O.v_samples(t, a, eta))


def test_validate_grid_semantics():
    g = nf.validate_grid([0.5, 0.25, 0.75, 0.0])
    assert list(g.order) == [3, 1, 0, 2]
    assert g.size == 4 and not g.instants.flags.writeable
    assert np.array_equal(g.sorted_instants, [0.0, 0.25, 0.5, 0.75])
    assert nf.validate_grid(g) == g and hash(nf.validate_grid(g)) == hash(g)
    for bad in ([0.1, 1.0], [-0.1], [np.nan], [], [[0.1]]):
        with pytest.raises(nf.OutOfRangeError):
            nf.validate_grid(bad)
    with pytest.raises(nf.DuplicateNodeError):
        nf.validate_grid([0.2, 0.2 + 1e-13])
    with pytest.raises(nf.DuplicateNodeError):  # circular gap across the period
        nf.validate_grid([1e-14, 1.0 - 1e-14])
    assert nf.validate_grid([0.2, 0.2 + 1e-13], min_gap=1e-14).size == 2


def test_validate_matches_oracle_order_with_ties_impossible():
    rng = np.random.default_rng(5)
    t = rng.uniform(0, 1, 1000)
    assert np.array_equal(nf.validate_grid(t).order, O.validate(t)[1])


def test_as_complex_vector():
    v = nf.as_complex_vector([1, 2j], length=2)
    assert v.dtype == np.complex128
    with pytest.raises(nf.LengthMismatchError):
        nf.as_complex_vector([[1.0]])
    with pytest.raises(nf.LengthMismatchError):
        nf.as_complex_vector([])
    with pytest.raises(nf.LengthMismatchError):
        nf.as_complex_vector([1.0], length=2)
    with pytest.raises(ValueError):
        nf.as_complex_vector([np.inf])


# --- window metadata (gridding.py:75-98) ------------------------------------------

def test_kernel_tables():
    for size in (1, 7, 33, 256):
        k = nf.kernel_for_size(size)
        w = O.Window.for_size(size)
        assert np.array_equal(k.deconv, w.deconv) and np.array_equal(k.bins, w.bins)
        assert k.fine_size == 2 * size and k.band_shift == size // 2 and k.taps == 29
        with pytest.raises(ValueError):
            k.deconv[0] = 1.0
    with pytest.raises(ValueError):
        nf.kernel_for_size(0)
    with pytest.raises(ValueError):
        nf.kernel_for_size(8, 0)


# --- error mapping of C status codes ------------------------------------------------

def test_status_codes_map_to_reference_exceptions():
    from paper_1604_06236_b200 import _lib

    assert _lib._STATUS_TO_ERROR[1] is nf.OutOfRangeError
    assert _lib._STATUS_TO_ERROR[6] is nf.KernelOverflowError
    assert _lib._STATUS_TO_ERROR[7] is nf.SingularDerivativeError
    assert _lib._STATUS_TO_ERROR[8] is nf.NonConvergenceError
    assert issubclass(nf.DeviceError, nf.NufftError)


def test_amplification_warning_from_scalars():
    from paper_1604_06236_b200.lagrange import _amplification_check

    with pytest.warns(nf.AmplificationWarning):
        _amplification_check(64, 0.1)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        _amplification_check(64, 1e-3)


# --- analytic flop accounting vs the reference's recorded reports (flops.py) --------

def _rep(fc):
    r = fc.report()
    return [r.real_adds, r.complex_adds, r.real_muls, r.complex_muls, r.complex_exps, r.total_flops] + list(
        r.fft_invocations)


def test_flop_charges_match_reference(golden):
    P, taps = 64, 29
    prm = nf.MethodParams.from_mu(1e-11, 64, 2)
    cases = {
        "build_plan": lambda f: inv._charge_plan(f, P, prm),
        "type5": lambda f: inv._charge_type5(f, P, taps),
        "type4": lambda f: inv._charge_type4(f, P, taps),
        "type1": lambda f: F.charge_type1(f, P, 48, taps),
        "type2": lambda f: F.charge_type2(f, P, P, taps),
    }
    for name, fn in cases.items():
        fc = nf.FlopCounter()
        fn(fc)
        assert _rep(fc) == list(golden[f"flops_{name}"]), name
    # conv = type1(R=128) + tail (real vs complex lam)
    for name, real in (("conv", False), ("conv_real", True)):
        fc = nf.FlopCounter()
        F.charge_type1(fc, P, 128, taps)
        F.charge_conv_tail(fc, 128, P, real)
        assert _rep(fc) == list(golden[f"flops_{name}"]), name


def test_tally_and_merge():
    r = nf.tally([("real_add", 2), ("complex_mul", 1), ("fft", 8), ("complex_div", 1)])
    assert r.total_flops == 2 + 6 + 5 * 8 * 3 + 6 + 5 + 1
    with pytest.raises(ValueError):
        nf.tally([("bogus", 1)])
    a, b = nf.FlopCounter(), nf.FlopCounter()
    a.fft(4)
    b.complex_exp(2)
    a.merge(b)
    assert a.report().complex_exps == 2 and a.report().fft_invocations == (4,)


def _report_array(fc):
    r = fc.report()
    return np.array([r.real_adds, r.complex_adds, r.real_muls, r.complex_muls, r.complex_exps, r.total_flops]
                    + list(r.fft_invocations), dtype=np.int64)


@pytest.mark.parametrize("name,which", [("cg4", "type4"), ("cg5", "type5"), ("cgcap", "type4"),
                                        ("cgtol", "type4")])
def test_cg_flop_charges_match_reference(golden, name, which):
    """cg_solve's flops= charges (baselines.py:141-181) from the iteration
    outcome alone reproduce the reference's counter for the same run."""
    from paper_1604_06236_b200 import baselines as B

    P = golden[f"{name}_t"].size
    it, conv = (int(v) for v in golden[f"{name}_meta"])
    fc = nf.FlopCounter()
    B._charge_cg(fc, P, 29, which, it, bool(conv), False, False)
    assert np.array_equal(_report_array(fc), golden[f"{name}_flops"])


def test_ge_flop_charges_match_reference(golden):
    from paper_1604_06236_b200 import baselines as B

    n = golden["ge32_t"].size
    fc = nf.FlopCounter()
    fc.real_mul(n * n)  # type4_system's phase matrix (baselines.py:46-48)
    fc.complex_exp(n * n)
    B._charge_ge(fc, n, n - 1, True)
    assert np.array_equal(_report_array(fc), golden["ge32_flops"])


def test_cg_argument_checks_precede_device_work():
    grid = nf.NonuniformGrid.__new__(nf.NonuniformGrid)  # never touched: validation fails first
    with pytest.raises(ValueError):
        nf.cg_solve(grid, np.ones(8), tol=0.0)
    with pytest.raises(ValueError):
        nf.cg_solve(grid, np.ones(8), which="type3")


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus N never silently runs on fewer GPUs: with fewer than N
    visible devices (none here) it prints an error line and exits non-zero."""
    import json
    import subprocess
    import sys

    import torch

    if torch.cuda.device_count() >= 8:
        pytest.skip("8 GPUs visible")
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "8", "--steps", "1"],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode != 0
    line = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    assert "error" in line and line["n_gpus"] == 8

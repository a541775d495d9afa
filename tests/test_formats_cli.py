"""Host-side parity of the file formats, the CLI's usage/parse/numeric exit
paths and the Monte-Carlo harness's configuration logic (reference
tests/test_vecio.py, test_cli.py, test_bench.py) — no GPU needed: every case
here fails or finishes before a kernel would launch."""

import math

import numpy as np
import pytest

from paper_1604_06236_b200 import bench as B
from paper_1604_06236_b200.cli import main
from paper_1604_06236_b200.vecio import (
    default_out_dir,
    read_grid_file,
    read_results_csv,
    read_vector_file,
    write_grid_file,
    write_results_csv,
    write_vector_file,
)


def test_vector_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    vec = rng.standard_normal(100) * 10.0 ** rng.integers(-200, 200, 100) + 1j * rng.standard_normal(100)
    write_vector_file(tmp_path / "v.txt", vec)
    assert np.array_equal(read_vector_file(tmp_path / "v.txt"), vec)


def test_grid_round_trip_bit_exact(tmp_path):
    t = np.sort(np.random.default_rng(1).uniform(0, 1, 64))
    write_grid_file(tmp_path / "g.txt", t)
    assert np.array_equal(read_grid_file(tmp_path / "g.txt"), t)


@pytest.mark.parametrize("text", ["1.0\n", "", "1.0 2.0 3.0\n", "# only a comment\n\n"])
def test_vector_parse_errors(tmp_path, text):
    (tmp_path / "bad.txt").write_text(text)
    with pytest.raises(ValueError):
        read_vector_file(tmp_path / "bad.txt")


def test_grid_parse_errors_name_the_line(tmp_path):
    (tmp_path / "bad.txt").write_text("0.1\n0.1 0.2\n")
    with pytest.raises(ValueError, match=r"bad.txt:2"):
        read_grid_file(tmp_path / "bad.txt")


def test_comments_and_blanks_skipped(tmp_path):
    (tmp_path / "v.txt").write_text("# header\n\n1.0 2.0\n")
    assert read_vector_file(tmp_path / "v.txt")[0] == 1.0 + 2.0j


def test_results_round_trip(tmp_path):
    rows = [
        B.TrialResult(64, 2, 1e-12, "NFFT", 0, 3.14159e-11, -210.06, 123456, None, 7),
        B.TrialResult(64, None, None, "CG", 1, 1e-14, -280.0, 999, 52, 6),
        B.TrialResult(32, 1, 1e-9, "GE", 0, 0.0, float("-inf"), 5, None, 3),
    ]
    path = tmp_path / "r.csv"
    write_results_csv(path, rows, {"seed": 7, "db_convention": "20*log10", "dense_cap": None})
    back, meta = read_results_csv(path)
    assert back == rows
    assert meta == {"seed": "7", "db_convention": "20*log10"}
    lines = path.read_text().splitlines()
    assert lines[0].startswith("# ") and lines[1].startswith("p,eta,mu,method")


def test_default_out_dir(monkeypatch, tmp_path):
    monkeypatch.delenv("NUFFT1D_OUT_DIR", raising=False)
    assert default_out_dir() == "."
    monkeypatch.setenv("NUFFT1D_OUT_DIR", str(tmp_path))
    assert default_out_dir() == str(tmp_path)


# ------------------------------------------------------------ CLI exit codes

def _files(tmp_path, t, d):
    write_grid_file(tmp_path / "grid.txt", t)
    write_vector_file(tmp_path / "data.txt", d)
    return str(tmp_path / "grid.txt"), str(tmp_path / "data.txt"), str(tmp_path / "out.txt")


def test_parse_failure_exit_code(tmp_path):
    (tmp_path / "bad.txt").write_text("not numbers\n")
    write_grid_file(tmp_path / "grid.txt", [0.0, 0.5])
    assert main(["transform", "--type", "2", "--grid", str(tmp_path / "grid.txt"), "--data",
                 str(tmp_path / "bad.txt"), "--out", str(tmp_path / "o.txt")]) == 2


def test_missing_file_exit_code(tmp_path):
    assert main(["transform", "--type", "2", "--grid", str(tmp_path / "nope.txt"), "--data",
                 str(tmp_path / "nope2.txt"), "--out", str(tmp_path / "o.txt")]) == 2


def test_length_mismatch_exit_code(tmp_path):
    g, d, o = _files(tmp_path, [0.0, 0.5], np.ones(3, complex))
    assert main(["transform", "--type", "4", "--grid", g, "--data", d, "--out", o]) == 2


def test_numeric_failure_exit_code(tmp_path, capsys):
    t = (np.arange(8) + 0.3) / 8
    g, d, o = _files(tmp_path, t, np.ones(8, complex))
    assert main(["transform", "--type", "4", "--grid", g, "--data", d, "--out", o, "--mu", "0.9",
                 "--eta", "2"]) == 3
    assert "NonPositiveDamping" in capsys.readouterr().err


def test_invalid_grid_file_exit_code(tmp_path, capsys):
    (tmp_path / "grid.txt").write_text("0.1\n1.5\n")
    write_vector_file(tmp_path / "data.txt", np.ones(2, complex))
    assert main(["transform", "--type", "2", "--grid", str(tmp_path / "grid.txt"), "--data",
                 str(tmp_path / "data.txt"), "--out", str(tmp_path / "o.txt")]) == 2
    assert "OutOfRange" in capsys.readouterr().err


def test_usage_errors_exit_2():
    with pytest.raises(SystemExit) as e:
        main(["transform", "--grid", "g", "--data", "d", "--out", "o"])  # --type missing
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        main(["transform", "--type", "3", "--grid", "g", "--data", "d", "--out", "o"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        main(["bench", "--figure", "fig9"])
    assert e.value.code == 2


# ------------------------------------------------ Monte-Carlo configuration

def test_db_convention():
    assert abs(B.to_db(1e-3) + 60.0) < 1e-9
    assert B.to_db(0.0) == float("-inf")


def test_config_rejects_bad_jitter_and_method():
    with pytest.raises(ValueError):
        B.TrialConfig(jitter_max=1.0)
    with pytest.raises(ValueError):
        B.TrialConfig(methods=("GE", "QR"))


def test_ge_size_cap_enforced_before_any_work():
    with pytest.raises(ValueError):
        B.run_sweep(B.TrialConfig(p=(16384,), methods=(B.METHOD_GE,), trials=1))


def test_run_figure_rejects_unknown():
    with pytest.raises(ValueError):
        B.run_figure("fig9")


def test_figure_protocol_defaults():
    f = B.FIGURE_DEFAULTS
    assert f["fig1"].p == (1024,) and f["fig1"].eta == (1, 2, 3, 4, 6, 15, 20)
    assert set(f["fig1"].methods) == {"GE", "CG", "NFFT"}
    assert len(f["fig1"].mu) == 29 and f["fig1"].mu[0] == 1e-18 and f["fig1"].mu[-1] == 1e-4
    assert f["fig2"].eta == (1, 2) and "R-NFFT" in f["fig2"].methods
    assert f["fig3"].p == (64, 128, 256, 512, 1024, 2048, 4096, 8192) and f["fig3"].eta == (1,)
    assert f["fig6"].eta == (6,) and f["fig6"].mu == (1e-15,)
    assert f["fig7"].p == (1024,) and f["fig7"].eta == tuple(range(1, 21))
    assert B.DENSE_DEFAULT_CAP == 1024 and B.GE_SIZE_CAP == 8192


def test_best_mu_selection_logic():
    def r(mu, trial, err):
        return B.TrialResult(64, 1, mu, B.METHOD_RNFFT, trial, err, 20 * math.log10(err), 1, None, trial)

    rows = [r(1e-13, 0, 1e-9), r(1e-13, 1, 1e-9), r(1e-9, 0, 1e-12), r(1e-9, 1, 1e-10), r(1e-5, 0, 1e-6),
            r(1e-5, 1, 1e-6), B.TrialResult(64, None, None, "GE", 0, 1e-14, -280.0, 1, None, 0)]
    assert B.best_mu(rows, B.METHOD_RNFFT) == {(64, 1): 1e-9}
    kept = B.filter_best_mu(rows, B.METHOD_RNFFT)
    assert {x.mu for x in kept} == {None, 1e-9} and len(kept) == 3

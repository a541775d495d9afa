"""The C-ABI shared library builds, loads without a GPU, and exports every
entry point include/nfft45.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "nfft45.h")
LIB = os.path.join(REPO, "paper_1604_06236_b200", "lib", "libnfft45.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(REPO, "paper_1604_06236_b200")], check=True)
    return ctypes.CDLL(LIB)


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nfft45_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_boundary():
    names = declared()
    for must in ("nfft45_validate_grid", "nfft45_grid_create", "nfft45_type1", "nfft45_type2",
                 "nfft45_nonuniform_conv", "nfft45_plan_create", "nfft45_type4", "nfft45_type5",
                 "nfft45_refine_type4", "nfft45_refine_type5", "nfft45_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_table_matches_header():
    from paper_1604_06236_b200 import _lib

    assert set(_lib.EXPORTED) == set(declared())


def test_host_only_entry_points_work_without_gpu(lib):
    import numpy as np

    from paper_1604_06236_b200 import _lib

    t = np.array([0.75, 0.25, 0.5])
    order = np.empty(3, dtype=np.int64)
    assert _lib.load().nfft45_validate_grid(t.ctypes.data, 3, 1e-12, order.ctypes.data) == 0
    assert list(order) == [1, 2, 0]
    bad = np.array([0.1, 1.0])
    assert _lib.load().nfft45_validate_grid(bad.ctypes.data, 2, 1e-12, order.ctypes.data) == 1
    assert b"outside" in _lib.load().nfft45_last_error()
    assert _lib.load().nfft45_version() >= 100


def test_sources_never_name_forbidden_batch_copy_apis():
    # B200_PROFILING.md: the batched async memcpy family faulted boxes; never call it
    forbidden = re.compile(r"Memcpy(3D)?BatchAsync")
    for root, _, files in os.walk(os.path.join(REPO, "paper_1604_06236_b200")):
        for f in files:
            if f.endswith((".cu", ".cuh", ".py", ".h", ".cpp")):
                assert not forbidden.search(open(os.path.join(root, f)).read()), f


def test_host_solve_rejects_invalid_arguments_without_touching_the_device(lib):
    """nfft45_solve_host validates its arguments before any CUDA call: a null plan,
    a bad kind, an empty batch or a refine count below -1 are INVALID_ARGUMENT (9)."""
    import numpy as np

    from paper_1604_06236_b200 import _lib

    L = _lib.load()
    x = np.zeros(8, dtype=np.complex128)
    y = np.empty_like(x)
    for plan, kind, passes, batch in ((None, 5, 1, 1), (None, 4, -1, 1), (None, 3, 1, 1), (None, 5, 1, 0),
                                      (None, 5, -2, 1)):
        rc = L.nfft45_solve_host(plan, kind, passes, x.ctypes.data, batch, y.ctypes.data, 64, 1, None)
        assert rc == 9
        assert b"invalid host solve" in L.nfft45_last_error()

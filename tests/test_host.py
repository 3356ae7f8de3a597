"""CPU-side checks of the product library: it loads, exports every symbol
include/hdivred_b200.h declares, its host restatement of the reference element
is bit-exact against the reference's own fixtures, its structured-solve
factors are valid, and compute entry points fail loudly without a device."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1801_08914_b200 as hd
from paper_1801_08914_b200 import _capi
from conftest import has_cuda, load_golden, GOLDEN_CASES

HEADER = Path(__file__).resolve().parent.parent / "include" / "hdivred_b200.h"


def test_library_exports_every_declared_symbol():
    declared = set(re.findall(r"\b(hdr_[a-z0-9_]+)\s*\(", HEADER.read_text()))
    declared = {d for d in declared if not d.endswith("_t")}
    lib = _capi.load()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(_capi.EXPORTED), declared ^ set(_capi.EXPORTED)
    assert b"sm_100a" in lib.hdr_version()


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_host_reference_element_bit_exact(name):
    g = load_golden(name)
    dim, k = g["dim"], g["k"]
    h = (ctypes.c_double * 3)(*g["h"])
    n = int(np.sqrt(g["ref_divdiv"].size))
    dd, mm, ul = np.empty(n * n), np.empty(n * n), np.empty(3 * n)
    fm = np.empty(g["ref_face_moments"].size)
    assert _capi.load().hdr_reference_element(dim, k, ctypes.addressof(h), dd.ctypes.data, mm.ctypes.data,
                                                 fm.ctypes.data, ul.ctypes.data) == 0
    assert np.array_equal(dd, g["ref_divdiv"])
    assert np.array_equal(mm, g["ref_mass"])
    assert np.array_equal(fm, g["ref_face_moments"])
    assert np.array_equal(ul, g["ref_unit_load"])


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_host_div_form_bit_exact(name):
    """ref_div_form (rt_space.cpp:256-259), the B of near_nullspace_check."""
    g = load_golden(name)
    h = (ctypes.c_double * 3)(*g["h"])
    out = np.empty(g["ref_div_form"].size)
    assert _capi.load().hdr_reference_div_form(g["dim"], g["k"], ctypes.addressof(h), out.ctypes.data) == 0
    assert np.array_equal(out, g["ref_div_form"])


@pytest.mark.parametrize("dim,k,cells", [(2, 0, 64), (3, 0, 64), (3, 1, 48), (3, 2, 24), (3, 3, 32), (2, 3, 16)])
def test_structured_factors(dim, k, cells):
    """D = Ms X diag(lambda) X^T Ms + E with E at rounding level, X M-orthonormal,
    N0 = Ms^-1 - X X^T PSD: the exact rewriting the device solve relies on."""
    h = (ctypes.c_double * 3)(*([1.0 / cells] * dim + [1.0] * (3 - dim)))
    dpf = (k + 1) ** (dim - 1)
    n = 2 * dim * dpf + dim * k * dpf
    r = (k + 1) ** dim
    X, lam, E, N0, Ma, diag = np.empty(n * r), np.empty(r), np.empty(n * n), np.empty(n * n), np.empty(n * n), np.empty(4)
    rank = ctypes.c_int64()
    assert _capi.load().hdr_structured_factors(dim, k, ctypes.addressof(h), X.ctypes.data, lam.ctypes.data,
                                                  E.ctypes.data, N0.ctypes.data, Ma.ctypes.data, diag.ctypes.data,
                                                  ctypes.byref(rank)) == 0, _capi.last_error()
    assert rank.value == r
    rho, e_rel, orth, block = diag
    assert e_rel < 1e-14 and orth < 1e-13 and block == 1.0
    assert np.all(lam > 0)
    N0 = N0.reshape(n, n)
    assert np.linalg.eigvalsh(0.5 * (N0 + N0.T)).min() > -1e-12 * np.abs(N0).max()
    assert np.max(np.abs(Ma)) <= 1e-15 * np.max(np.abs(N0)) * 1e6  # rounding-level asymmetry only


def test_space_info_mirrors_reference_counts():
    """tests/python/test_smoke.py:9-17 of the reference (401,408 dofs)."""
    assert hd.space_info(3, [64, 64, 32], 0)["ndofs"] == 401408
    assert hd.space_info(3, [32, 32, 16], 1)["ndofs"] == 401408
    one = hd.space_info(3, [1, 1, 1], 0)
    assert one["ndofs"] == 6 and one["broken_ndofs"] == 6


@pytest.mark.skipif(has_cuda(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    with pytest.raises(hd.DeviceError):
        hd.Space(3, [2, 2, 2], 0)

"""Fail-safe of the structured element solve (DESIGN.md §2 "Fail-safe"), GPU.

The structured kernels accept a cell only when their a-posteriori estimate of
its error (Neumann truncation + fp32/TF32 evaluation of the correction) is below
1e-12 of |H_T|; every other cell is solved on the exact double-double path
(kern_exact.cu, or in-thread for k = 0).  These tests drive the coefficient
ranges the reference accepts but the BASELINE configs never reach:

  * the reference's soft-hard preset p in {-8, -4, 4, 8} (src/mesh.cpp:168-191,
    pinned at p = -8 in tests/unit_reduction.cpp:216-224) at 4^3 and at 64^3 (RT0)
    / 32^3 (RT1);
  * alpha, beta log-uniform in [1e-8, 1e8] (the draw of tests/unit_fem.cpp:118-133):
    where the reference raises SingularBlock (pivot <= 1e-14 max|A_ii| or
    max|S_b|, src/dense.cpp:61-97) the device raises SingularBlockError too,
    elsewhere H, g, x_hat match the double-double oracle;
  * RT3 with alpha / beta = 1e6 (every cell rejected);
  * every golden case with the exact path forced for all cells;
  * BASELINE-like inputs send no cell to the exact path.

Values: max|device - DD| <= 1e-11 max|DD| (the parity contract).
"""
import numpy as np
import pytest

from conftest import GOLDEN_CASES, has_cuda, load_golden
from oracle_lib import Oracle, OracleError, rel_err, sampled_rows_vs_dd

pytestmark = pytest.mark.gpu

TOL = 1e-11

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402


def _check_case(dim, cells, k, coef, seed, recover=True, condense=False, expect_exact=None):
    o = Oracle(dim, cells, k)
    o.gen_inputs(coef, seed)
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    sp = hd.Space(dim, cells, k)
    try:
        o.run("port_hybridize")
    except OracleError as exc:  # the reference raises: so must the device
        assert "SingularBlock" in str(exc)
        with pytest.raises(hd.SingularBlockError):
            sp.hybridize(a, b, f)
        return None
    o.run("dd_hybridize")
    op = sp.hybridize(a, b, f)
    nx = op.exact_cells()
    if expect_exact is not None:
        assert (nx > 0) == expect_exact, nx
    hv, gv = op.values()
    h_dd, g_dd = o.get("H.values_dd"), o.get("g_dd")
    eh, eg = rel_err(hv, h_dd), rel_err(gv, g_dd)
    assert eh <= TOL and eg <= TOL, (eh, eg)
    msg = f"{coef} {cells} RT{k}: exact cells {nx}/{sp.ncells}; device-vs-DD H {eh:.1e} g {eg:.1e}; " \
          f"reference-vs-DD H {rel_err(o.get('H.values'), h_dd):.1e}"
    if recover:
        o.run("dd_recover")
        x_hat, x = op.recover(o.get("lambda"), f)
        ex, exx = rel_err(x_hat, o.get("x_hat_dd")), rel_err(x, o.get("x_dd"))
        assert ex <= TOL and exx <= TOL, (ex, exx)
        msg += f"; x_hat {ex:.1e}"
    if condense:
        o.run("port_condense")
        o.run("dd_condense")
        cop = sp.static_condense(a, b, f)
        sv, fs = cop.values()
        es, ef = rel_err(sv, o.get("S.values_dd")), rel_err(fs, o.get("f_s_dd"))
        assert es <= TOL and ef <= TOL, (es, ef)
        msg += f"; S {es:.1e} f_S {ef:.1e}"
    print(msg)
    return op


@pytest.mark.parametrize("p", [-8, -4, 4, 8])
@pytest.mark.parametrize("k", [0, 1])
def test_soft_hard_preset_4cube(p, k):
    """cube(4) with soft_hard_coefficients(mesh, p), as tests/unit_reduction.cpp:216-224."""
    _check_case(3, (4, 4, 4), k, f"softhard:{p}", 2024, condense=True, expect_exact=(p == -8 and k == 1) or None)


@pytest.mark.parametrize("dim,cells,k", [(3, (64, 64, 64), 0), (3, (32, 32, 32), 1)])
def test_soft_hard_p_minus8_large(dim, cells, k):
    _check_case(dim, cells, k, "softhard:-8", 77, recover=True, expect_exact=(k == 1) or None)


@pytest.mark.parametrize("dim,cells,k", [
    (3, (4, 4, 4), 0), (3, (8, 8, 8), 0), (3, (2, 2, 2), 1), (3, (4, 4, 4), 1), (2, (8, 8), 1), (2, (16, 16), 0),
    (2, (4, 4), 2), (2, (3, 3), 3), (3, (3, 3, 3), 2), (3, (2, 2, 2), 3),
])
def test_logu_1e8_matches_reference_behaviour(dim, cells, k):
    """alpha, beta ~ log-U[1e-8, 1e8] per cell: SingularBlock where the reference
    raises it, DD-accurate values elsewhere."""
    _check_case(dim, cells, k, "logu:1e-8:1e8", 11)


@pytest.mark.parametrize("dim,cells,k,coef", [
    (3, (4, 4, 4), 1, "logu:1e-6:1e6"), (3, (6, 6, 6), 1, "logu:1e-5:1e5"), (2, (8, 8), 2, "logu:1e-6:1e6"),
    (3, (3, 3, 3), 2, "logu:1e-5:1e5"),
])
def test_wide_coefficient_ranges(dim, cells, k, coef):
    _check_case(dim, cells, k, coef, 5, condense=True)


def test_rt3_ratio_1e6_every_cell_exact():
    sp_cells = 125
    op = _check_case(3, (5, 5, 5), 3, "uniform:1e6:1", 3, recover=False, expect_exact=True)
    assert op.exact_cells() == sp_cells


def test_rt3_ratio_1e6_16cube_sampled():
    """16^3 RT3, alpha / beta = 1e6: every cell on the exact path; sampled rows
    (cells and their +x neighbours) against the element-wise DD oracle."""
    o = Oracle(3, (16, 16, 16), 3)
    o.gen_inputs("uniform:1e6:1", 9)
    o.run("structure")
    sp = hd.Space(3, (16, 16, 16), 3)
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    assert op.exact_cells() == sp.ncells
    hv, gv = op.values()
    rng = np.random.default_rng(1)
    base = [int(e) for e in rng.choice(sp.ncells, 24, replace=False) if int(e) % 16 < 15]
    ro, ci = sp.pattern("H")
    eh, eg = sampled_rows_vs_dd(o, ro, ci, hv, gv, sp.n, 16, base)
    assert eh <= TOL and eg <= TOL, (eh, eg)


@pytest.mark.parametrize("name", [c for c in GOLDEN_CASES if "weighted" not in c])
def test_forced_exact_path_on_goldens(name):
    """Every cell through the exact path (force): H, g, x_hat, x vs DD."""
    g = load_golden(name)
    o = Oracle(g["dim"], g["cells"], g["k"])
    o.gen_inputs(g["coef"], g["seed"])
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    sp = hd.Space(g["dim"], g["cells"], g["k"])
    sp.set_exact_policy(force=True)
    op = sp.hybridize(g["alpha"], g["beta"], g["f_hat"])
    assert op.exact_cells() == sp.ncells
    hv, gv = op.values()
    assert rel_err(hv, o.get("H.values_dd")) <= TOL and rel_err(gv, o.get("g_dd")) <= TOL
    x_hat, x = op.recover(g["lambda"], g["f_hat"])
    assert op.exact_cells() == sp.ncells  # the recovery's own count
    assert rel_err(x_hat, o.get("x_hat_dd")) <= TOL and rel_err(x, o.get("x_dd")) <= TOL
    # and the pattern positions of the fast path: forced and structured results agree
    sp2 = hd.Space(g["dim"], g["cells"], g["k"])
    hv2, gv2 = sp2.hybridize(g["alpha"], g["beta"], g["f_hat"]).values()
    assert rel_err(hv, hv2) <= TOL and rel_err(gv, gv2) <= TOL


@pytest.mark.parametrize("dim,cells,k,coef", [
    (2, (64, 64), 0, "uniform:1:1"), (3, (32, 32, 32), 0, "logu:1e-2:1e2"), (3, (16, 16, 16), 1, "logu:1e-2:1e2"),
    (3, (12, 12, 12), 2, "logu:1e-2:1e2"), (3, (8, 8, 8), 3, "checker:1e-2:1e2"), (2, (16, 16), 3, "logu:1e-2:1e2"),
])
def test_baseline_like_inputs_stay_on_the_structured_path(dim, cells, k, coef):
    o = Oracle(dim, cells, k)
    o.gen_inputs(coef, 1000 + k)
    sp = hd.Space(dim, cells, k)
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    assert op.exact_cells() == 0


@pytest.mark.parametrize("variant", ["HDR_RT0_BRICK", "HDR_RT0_CELL", "HDR_RT0_ROWS"])
@pytest.mark.parametrize("dim,cells", [(3, (9, 5, 6)), (2, (33, 7))])
def test_rt0_kernel_variants_exact_tail(variant, dim, cells, monkeypatch):
    """k = 0: rejected cells are added by the last CTA of the colour-1 launch
    (rt0_tail) in each kernel variant; forced on every cell, twice in a row
    (the list resets itself), against the DD oracle."""
    o = Oracle(dim, cells, 0)
    o.gen_inputs("logu:1e-2:1e2", 31)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    monkeypatch.setenv(variant, "1")
    sp = hd.Space(dim, cells, 0)
    sp.set_exact_policy(force=True)
    for _ in range(2):
        op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
        assert op.exact_cells() == sp.ncells
        hv, gv = op.values()
        assert rel_err(hv, o.get("H.values_dd")) <= TOL and rel_err(gv, o.get("g_dd")) <= TOL
    sp.set_exact_policy(force=False)
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    assert op.exact_cells() == 0
    assert rel_err(op.values()[0], o.get("H.values_dd")) <= TOL


def test_exact_path_is_deterministic():
    o = Oracle(3, (4, 4, 4), 1)
    o.gen_inputs("softhard:-8", 5)
    sp = hd.Space(3, (4, 4, 4), 1)
    v1 = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat")).values()
    v2 = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat")).values()
    assert np.array_equal(v1[0], v2[0]) and np.array_equal(v1[1], v2[1])

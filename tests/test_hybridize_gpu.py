"""Parity of the device hybridization / recovery against the oracle (GPU).

Contract:
  * H row_offsets / col_indices bit-exact against the reference's hybridize
    output (golden fixtures produced by the reference itself);
  * H values, g, recovered x_hat / x within 1e-11 of max|entry| of the
    element-wise double-double oracle evaluated on the bit-identical A_T
    (tests/oracle_lib.py → oracle/hdr_oracle.c);
  * bit-identical results on repeated runs (no float atomics).
All calls go through the C ABI (libhdivred_b200.so) via the package front-end.
"""
import numpy as np
import pytest

from conftest import has_cuda, load_golden, GOLDEN_CASES
from oracle_lib import Oracle, rel_err, sampled_rows_vs_dd

pytestmark = pytest.mark.gpu

TOL = 1e-11

if not has_cuda():  # collected on CPU boxes too, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402

UNWEIGHTED = [c for c in GOLDEN_CASES if "weighted" not in c]


def oracle_for(g):
    o = Oracle(g["dim"], g["cells"], g["k"])
    o.gen_inputs(g["coef"], g["seed"])
    return o


@pytest.mark.parametrize("name", UNWEIGHTED)
def test_pattern_bit_exact_vs_reference(name):
    g = load_golden(name)
    sp = hd.Space(g["dim"], g["cells"], g["k"])
    ro, ci = sp.pattern("H")
    assert np.array_equal(ro, g["H.row_offsets"])
    assert np.array_equal(ci, g["H.col_indices"])
    ro, ci = sp.pattern("S")
    assert np.array_equal(ro, g["S.row_offsets"])
    assert np.array_equal(ci, g["S.col_indices"])
    assert np.array_equal(sp.master_globals(), g["master_globals"])
    gl, sg = sp.dof_map()
    assert np.array_equal(gl, g["P.col_indices"])
    assert np.array_equal(sg, g["P.values"])
    dd, mm = sp.reference_matrices()
    assert np.array_equal(dd.ravel(), g["ref_divdiv"]) and np.array_equal(mm.ravel(), g["ref_mass"])


@pytest.mark.parametrize("name", UNWEIGHTED)
def test_hybridize_values_vs_dd_oracle(name):
    g = load_golden(name)
    o = oracle_for(g)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    sp = hd.Space(g["dim"], g["cells"], g["k"])
    op = sp.hybridize(g["alpha"], g["beta"], g["f_hat"])
    hv, gv = op.values()
    h_dd, g_dd = o.get("H.values_dd"), o.get("g_dd")
    assert rel_err(hv, h_dd) <= TOL, rel_err(hv, h_dd)
    assert rel_err(gv, g_dd) <= TOL, rel_err(gv, g_dd)
    x_hat, x = op.recover(g["lambda"], g["f_hat"])
    assert rel_err(x_hat, o.get("x_hat_dd")) <= TOL
    assert rel_err(x, o.get("x_dd")) <= TOL
    # the reference's own distance to the truth, for the record
    print(f"{name}: device-vs-DD H {rel_err(hv, h_dd):.1e} g {rel_err(gv, g_dd):.1e}; "
          f"reference-vs-DD H {rel_err(g['H.values'], h_dd):.1e}")


def test_explicit_reference_matrices_give_identical_bits():
    g = load_golden("h3_rt1_2x2x2_logu")
    n = int(np.sqrt(g["ref_divdiv"].size))
    a = hd.Space(3, g["cells"], 1)
    b = hd.Space(3, g["cells"], 1, ref_divdiv=g["ref_divdiv"].reshape(n, n), ref_mass=g["ref_mass"].reshape(n, n))
    va = a.hybridize(g["alpha"], g["beta"], g["f_hat"]).values()
    vb = b.hybridize(g["alpha"], g["beta"], g["f_hat"]).values()
    assert np.array_equal(va[0], vb[0]) and np.array_equal(va[1], vb[1])


@pytest.mark.parametrize("dim,cells,k,coef", [
    (3, (8, 8, 8), 0, "logu:1e-2:1e2"), (3, (6, 5, 4), 1, "logu:1e-2:1e2"), (3, (5, 4, 4), 1, "logu:1e-3:1e3"),
    (2, (9, 7), 1, "logu:1e-2:1e2"), (2, (6, 6), 2, "logu:1e-3:1e3"), (2, (5, 4), 3, "logu:1e-2:1e2"),
    (3, (3, 3, 3), 2, "logu:1e-3:1e3"), (3, (3, 3, 2), 3, "checker:1e-2:1e2"), (3, (4, 4, 4), 1, "logu:1e-4:1e4"),
])
def test_hybridize_moderate_meshes_vs_dd(dim, cells, k, coef):
    o = Oracle(dim, cells, k)
    o.gen_inputs(coef, 4242)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    sp = hd.Space(dim, cells, k)
    ro, ci = sp.pattern("H")
    assert np.array_equal(ro, o.getq("H.row_offsets")) and np.array_equal(ci, o.getq("H.col_indices"))
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    hv, gv = op.values()
    assert rel_err(hv, o.get("H.values_dd")) <= TOL
    assert rel_err(gv, o.get("g_dd")) <= TOL


@pytest.mark.parametrize("cells,coef", [
    ((1, 1, 5), "logu:1e-2:1e2"), ((7, 1, 1), "logu:1e-3:1e3"), ((2, 3, 1), "softhard:4"), ((1, 4, 3), "logu:1e-2:1e2"),
    ((9, 2, 2), "checker:1e-2:1e2"), ((3, 3, 3), "uniform:2:0.5"),
])
def test_rt1_tensor_core_correction_thin_meshes_vs_dd(cells, coef):
    """RT1 hexes (the mma.sync 3xTF32 correction, the prefetched [N0 f ; X^T f]):
    one-cell-thick meshes, so cells with every count of interior faces, incl. none;
    H, g and the recovery against the double-double oracle, no cell rejected."""
    o = Oracle(3, cells, 1)
    o.gen_inputs(coef, 31)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    sp = hd.Space(3, cells, 1)
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    hv, gv = op.values()
    assert op.exact_cells() == 0
    assert rel_err(hv, o.get("H.values_dd")) <= TOL and rel_err(gv, o.get("g_dd")) <= TOL
    x_hat, _ = op.recover(o.get("lambda"), o.get("f_hat"))
    assert rel_err(x_hat, o.get("x_hat_dd")) <= TOL


@pytest.mark.parametrize("dim,cells,coef", [
    (3, (8, 8, 8), "logu:1e-2:1e2"), (3, (37, 5, 7), "logu:1e-3:1e3"), (3, (70, 3, 2), "checker:1e-2:1e2"),
    (3, (1, 1, 9), "logu:1e-2:1e2"), (2, (64, 64), "uniform:1:1"), (2, (75, 9), "logu:1e-2:1e2"), (2, (1, 13), "logu:1e-2:1e2"),
])
def test_rt0_brick_kernel_matches_cell_kernel_bitwise(dim, cells, coef, monkeypatch):
    """The k = 0 brick kernel (shared-memory line segments, coalesced stores,
    staged brick-boundary faces) against the thread-per-cell kernel: the same
    element arithmetic and the same two-term sums, so identical bits, on meshes
    with partial bricks in every direction; plus the DD oracle."""
    o = Oracle(dim, cells, 0)
    o.gen_inputs(coef, 77)
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    sp = hd.Space(dim, cells, 0)
    monkeypatch.setenv("HDR_RT0_BRICK", "1")
    hb = sp.hybridize(a, b, f).values()
    monkeypatch.delenv("HDR_RT0_BRICK")
    monkeypatch.setenv("HDR_RT0_CELL", "1")
    hc = sp.hybridize(a, b, f).values()
    assert np.array_equal(hb[0], hc[0]) and np.array_equal(hb[1], hc[1])
    o.run("port_hybridize")
    o.run("dd_hybridize")
    assert rel_err(hb[0], o.get("H.values_dd")) <= TOL and rel_err(hb[1], o.get("g_dd")) <= TOL


def test_deterministic_and_device_inputs():
    import torch

    o = Oracle(3, (6, 6, 6), 1)
    o.gen_inputs("logu:1e-2:1e2", 9)
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    sp = hd.Space(3, (6, 6, 6), 1)
    v1 = sp.hybridize(a, b, f).values()
    v2 = sp.hybridize(a, b, f).values()
    dev = [torch.from_numpy(x).cuda() for x in (a, b, f)]
    v3 = sp.hybridize(*dev).values()
    for x, y in ((v1, v2), (v1, v3)):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


def test_zero_rhs_gives_zero_g_and_recovery():
    """tests/unit_reduction.cpp:258-267."""
    sp = hd.Space(3, (2, 2, 2), 0)
    op = sp.hybridize(np.ones(8), np.ones(8), np.zeros(48))
    _, g = op.values()
    assert np.all(g == 0.0)
    x_hat, x = op.recover(np.zeros(sp.m), np.zeros(48))
    assert np.all(x_hat == 0.0) and np.all(x == 0.0)


def test_single_cell_m0_recovery_is_direct_solve():
    """tests/unit_reduction.cpp:268-276: m = 0, x_hat = A^-1 f."""
    o = Oracle(3, (1, 1, 1), 1)
    o.gen_inputs("uniform:1:1", 3)
    sp = hd.Space(3, (1, 1, 1), 1)
    assert sp.m == 0
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    x_hat, _ = op.recover(np.zeros(0), o.get("f_hat"))
    ref = np.linalg.solve(o.element_matrix(0), o.get("f_hat"))
    assert rel_err(x_hat, ref) <= 1e-11


def test_hybridized_matrix_mirror():
    """Mirror of the reference's python smoke test (tests/python/test_smoke.py:87-94)."""
    (nrows, ncols, offsets, cols, vals), g = hd.hybridized_matrix({"cells": [2, 2, 2], "order": 0})
    assert nrows == ncols == 12
    assert len(g) == nrows and len(offsets) == nrows + 1 and len(cols) == len(vals) == offsets[-1]
    assert all(np.isfinite(vals))


FULL = [  # BASELINE.json configs 1, 2, 3, 5 (config 4 needs the Piola path)
    (2, (64, 64), 0, "uniform:1:1", 1001, 55688),
    (3, (64, 64, 64), 0, "logu:1e-2:1e2", 1002, 8394240),
    (3, (48, 48, 48), 1, "logu:1e-2:1e2", 1003, 56088576),
    (3, (32, 32, 32), 3, "checker:1e-2:1e2", 1005, 260505600),
]


@pytest.mark.parametrize("dim,cells,k,coef,seed,nnz", FULL)
def test_full_size_sampled_rows_vs_dd(dim, cells, k, coef, seed, nnz):
    """Full BASELINE sizes: pattern size as the analytic count, and sampled rows
    of H / g against the element-wise DD oracle of both adjacent cells."""
    o = Oracle(dim, cells, k)
    o.gen_inputs(coef, seed)
    o.run("structure")
    sp = hd.Space(dim, cells, k)
    assert sp.info["nnz_h"] == nnz
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    hv, gv = op.values()
    ro, ci = sp.pattern("H")
    assert ro[-1] == nnz and np.all(np.diff(ro) > 0)
    assert np.all(np.isfinite(hv)) and np.all(np.isfinite(gv))
    rng = np.random.default_rng(seed)
    base = [int(e) for e in rng.choice(sp.ncells, 3 if k == 3 else 16, replace=False) if int(e) % cells[0] < cells[0] - 1]
    eh, eg = sampled_rows_vs_dd(o, ro, ci, hv, gv, sp.n, cells[0], base)
    assert eh <= TOL and eg <= TOL, (eh, eg)


@pytest.mark.parametrize("dim,cells,k", [(3, (6, 5, 4), 0), (3, (5, 4, 3), 1), (3, (3, 3, 2), 3), (2, (9, 7), 2)])
def test_batch_pipeline_matches_single_calls(dim, cells, k):
    """hdr_hybridize_fe_batch (three streams, two alternating operators) gives
    the same bits as separate hybridize calls, item by item."""
    sp = hd.Space(dim, cells, k)
    rng = np.random.default_rng(7)
    items = []
    for _ in range(5):
        a = 10.0 ** rng.uniform(-2, 2, sp.ncells)
        b = 10.0 ** rng.uniform(-2, 2, sp.ncells)
        f = rng.uniform(-1, 1, sp.broken_ndofs)
        items.append((a, b, f))
    h_outs = [np.full(sp.info["nnz_h"], np.nan) for _ in items]
    g_outs = [np.full(sp.m, np.nan) for _ in items]
    sp.hybridize_batch([x[0] for x in items], [x[1] for x in items], [x[2] for x in items], h_outs, g_outs)
    for (a, b, f), hv, gv in zip(items, h_outs, g_outs):
        h_ref, g_ref = sp.hybridize(a, b, f).values()
        assert np.array_equal(hv, h_ref) and np.array_equal(gv, g_ref)

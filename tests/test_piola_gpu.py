"""Config 4 on the device: perturbed trilinear hexahedra (GPU).

Contract: the device A_T against the CPU
restatement (oracle hdo_piola_element — there is no reference for curved
cells) within 1e-13 of max|A_T| (the device assembles in GEMM form, another
summation order); H / g / x_hat / x / S / f_S / x_cond within 1e-11 of
max|entry| of the double-double oracle fed the device's own A_T (a_hat); patterns identical to the affine ones
(same topology); the unperturbed vertex set reproduces the affine path.
"""
import numpy as np
import pytest

from conftest import has_cuda
from oracle_lib import Oracle, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-11

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402

CASES = [((3, 2, 2), 1, 1004), ((2, 2, 2), 2, 1004), ((2, 2, 1), 2, 7), ((3, 3, 3), 0, 11)]


A_TOL = 1e-13


def _setup(cells, k, seed):
    """Space with the seeded vertices; the oracle then runs on the device's A_T."""
    o = Oracle(3, cells, k)
    o.gen_inputs("logu:1e-3:1e3;perturb=0.2", seed)
    sp = hd.Space(3, cells, k)
    sp.set_vertices(o.get("vertices"))
    sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))  # assembles A_T on the device
    A = sp.element_matrices()
    for e in range(sp.ncells):
        ref = o.element_matrix(e)
        assert np.max(np.abs(A[e] - ref)) <= A_TOL * np.max(np.abs(ref)), e
    o.set("a_hat", np.ascontiguousarray(A).ravel())
    return o, sp


@pytest.mark.parametrize("cells,k,seed", CASES)
def test_piola_hybridize_vs_dd(cells, k, seed):
    o, sp = _setup(cells, k, seed)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    ro, ci = sp.pattern("H")
    assert np.array_equal(ro, o.getq("H.row_offsets")) and np.array_equal(ci, o.getq("H.col_indices"))
    hv, g = op.values()
    e_h, e_g = rel_err(hv, o.get("H.values_dd")), rel_err(g, o.get("g_dd"))
    assert e_h <= TOL and e_g <= TOL, (e_h, e_g)
    x_hat, x = op.recover(o.get("lambda"), o.get("f_hat"))
    assert rel_err(x_hat, o.get("x_hat_dd")) <= TOL
    assert rel_err(x, o.get("x_dd")) <= TOL
    print(f"{cells} k={k}: H {e_h:.1e} g {e_g:.1e} (port vs DD {rel_err(o.get('H.values'), o.get('H.values_dd')):.1e})")


@pytest.mark.parametrize("cells,k,seed", CASES)
def test_piola_condense_vs_dd(cells, k, seed):
    o, sp = _setup(cells, k, seed)
    o.run("port_condense")
    o.run("dd_condense")
    o.run("dd_recover_condensed")
    op = sp.static_condense(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    sv, fs = op.values()
    assert rel_err(sv, o.get("S.values_dd")) <= TOL
    assert rel_err(fs, o.get("f_s_dd")) <= TOL
    x = op.recover(o.get("x_b"), o.get("f_hat"))
    assert rel_err(x, o.get("x_cond_dd")) <= TOL


def test_unperturbed_vertices_reproduce_affine():
    cells, k = (3, 2, 2), 1
    o = Oracle(3, cells, k)
    o.gen_inputs("logu:1e-2:1e2", 5)
    h = [1 / c for c in cells]
    g = np.stack(np.meshgrid(*[np.arange(c + 1) * hh for c, hh in zip(cells, h)], indexing="ij"), -1)
    verts = g.transpose(2, 1, 0, 3).reshape(-1, 3)
    sp = hd.Space(3, cells, k)
    ref = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat")).values()
    sp.set_vertices(verts)
    mapped = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat")).values()
    # the mapped A_T equals the reference's affine A_T up to rounding ...
    A = sp.element_matrices()
    for e in range(sp.ncells):
        assert rel_err(A[e], o.element_matrix(e)) <= 2e-15
    # ... and H moves by the reference's own sensitivity to 1-ulp changes of A_T
    # (about 1e-9 here), not more
    assert rel_err(mapped[0], ref[0]) <= 1e-8 and rel_err(mapped[1], ref[1]) <= 1e-8
    sp.set_vertices(None)
    back = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat")).values()
    assert np.array_equal(back[0], ref[0])


def test_config4_full_size_sampled_rows_vs_dd():
    """BASELINE config 4 at full size (24^3 perturbed RT2, log-uniform [1e-3, 1e3]):
    analytic pattern size, finite values, and sampled cells (with their +x
    neighbours, so shared-face entries are complete) against the element-wise
    double-double oracle fed the device's A_T of those cells."""
    cells, k = (24, 24, 24), 2
    o = Oracle(3, cells, k)
    o.gen_inputs("logu:1e-3:1e3;perturb=0.2", 1004)
    o.run("structure")
    sp = hd.Space(3, cells, k)
    sp.set_vertices(o.get("vertices"))
    assert sp.info["nnz_h"] == 34058880
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    hv, gv = op.values()
    ro, ci = sp.pattern("H")
    assert ro[-1] == 34058880 and np.all(np.isfinite(hv)) and np.all(np.isfinite(gv))
    rng = np.random.default_rng(1004)
    pool = [e for e in range(sp.ncells) if e % cells[0] < cells[0] - 1]
    base = [int(e) for e in rng.choice(pool, 128, replace=False)]  # + their +x neighbours: >= 256 cells
    have = sorted(set(base) | {e + 1 for e in base})
    A = sp.element_matrices()
    n = sp.n
    for e in have:
        ref = o.element_matrix(e)
        assert np.max(np.abs(A[e] - ref)) <= A_TOL * np.max(np.abs(ref)), e
    o.set("a_sel", np.array(have, dtype=np.float64))
    o.set("a_sel_blocks", np.ascontiguousarray(A[have]).ravel())
    del A
    row_vals, row_g = {}, {}
    for cell in have:
        rows, h, gt, _ = o.dd_element(cell)
        for a_, r in enumerate(rows):
            row_g.setdefault(int(r), []).append(gt[a_])
            for b_, c in enumerate(rows):
                row_vals.setdefault((int(r), int(c)), []).append(h[a_, b_])
    C = o.getq("C.col_indices").reshape(-1, 2)
    hs = set(have)

    def cells_of(row):
        return {int(C[row, 0]) // n, int(C[row, 1]) // n}

    worst_h, worst_g, checked = 0.0, 0.0, 0
    for (r, c), parts in row_vals.items():
        if not (cells_of(r) & cells_of(c)) <= hs:
            continue
        p = ro[r] + np.searchsorted(ci[ro[r]:ro[r + 1]], c)
        assert ci[p] == c
        worst_h = max(worst_h, abs(hv[p] - sum(parts)))
        checked += 1
    for r, parts in row_g.items():
        if cells_of(r) <= hs:
            worst_g = max(worst_g, abs(gv[r] - sum(parts)))
    assert checked > 0
    e_h, e_g = worst_h / np.max(np.abs(hv)), worst_g / np.max(np.abs(gv))
    print(f"config 4 full size: {checked} sampled H entries, H {e_h:.1e} g {e_g:.1e}")
    assert e_h <= TOL and e_g <= TOL


def test_mapped_blocks_not_positive_definite_or_singular_are_reported():
    """The SPD elimination of mapped cells checks every LDL^T pivot with the
    reference's SingularBlock rule (dense.cpp:61-97): a cell with alpha = beta = 0
    (zero block) raises SingularBlockError, one with a negative coefficient pair
    (negative definite block) is not SPD and raises UnsupportedError; both name
    the element, and the space stays usable afterwards."""
    o, sp = _setup((3, 2, 2), 2, 1004)
    a, b, f = o.get("alpha").copy(), o.get("beta").copy(), o.get("f_hat")
    a0, b0 = a.copy(), b.copy()
    a[5] = b[5] = 0.0
    with pytest.raises(hd.SingularBlockError, match="element 5"):
        sp.hybridize(a, b, f)
    a, b = a0.copy(), b0.copy()
    a[7], b[7] = -a[7], -b[7]
    with pytest.raises(hd.UnsupportedError, match="element 7"):
        sp.hybridize(a, b, f)
    hv, g = sp.hybridize(a0, b0, f).values()
    assert np.all(np.isfinite(hv)) and np.all(np.isfinite(g))


def test_batch_empty_and_partial_outputs():
    """hdr_hybridize_fe_batch: count 0 is a no-op; NULL outputs skip the download."""
    sp = hd.Space(3, (4, 3, 2), 1)
    sp.hybridize_batch([], [], [])
    rng = np.random.default_rng(3)
    a, b, f = rng.uniform(1, 2, sp.ncells), rng.uniform(1, 2, sp.ncells), rng.uniform(-1, 1, sp.broken_ndofs)
    g_out = [np.full(sp.m, np.nan)]
    sp.hybridize_batch([a], [b], [f], None, g_out)
    assert np.array_equal(g_out[0], sp.hybridize(a, b, f).values()[1])

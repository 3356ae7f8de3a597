"""The one-pass k = 0 pencil kernel (kern_pencil.cu, the default RT0 path) against
the element-wise double-double oracle and against the older brick kernel (GPU).

  * meshes with every boundary configuration: one-cell-thick, lines longer than one
    warp / one CTA (x-neighbour recomputed across CTAs), odd sizes, 2D and 3D;
  * H, g within 1e-11 of max|entry| (the contract) AND within 1e-13 of each ROW's
    own max|entry| (element accuracy: the Sherman-Morrison form is accurate to a few
    ulp of the cell's own A_T^-1, whatever alpha / beta);
  * coefficient ranges from BASELINE's to 1e-6..1e6 stay on the fast path; the
    cells past the acceptance bound go to the exact path with the reference's
    SingularBlock behaviour (tests/test_failsafe_gpu.py), forced here too.
"""
import numpy as np
import pytest

from conftest import has_cuda
from oracle_lib import Oracle, OracleError, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-11

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402


def _row_rel(ro, hv, ref):
    """max over rows of |hv - ref| / max|ref row|"""
    worst = 0.0
    d = np.abs(hv - ref)
    a = np.abs(ref)
    for r in range(len(ro) - 1):
        s = a[ro[r]:ro[r + 1]].max()
        if s > 0:
            worst = max(worst, d[ro[r]:ro[r + 1]].max() / s)
    return worst


MESHES = [
    (3, (8, 8, 8)), (3, (64, 3, 2)), (3, (65, 2, 3)), (3, (33, 4, 1)), (3, (1, 5, 7)), (3, (300, 2, 1)),
    (3, (2, 1, 1)), (3, (5, 5, 5)), (2, (64, 64)), (2, (75, 9)), (2, (1, 13)), (2, (260, 3)), (2, (31, 2)),
]


@pytest.mark.parametrize("dim,cells", MESHES)
@pytest.mark.parametrize("coef", ["logu:1e-2:1e2", "logu:1e-4:1e4", "logu:1e-6:1e6", "logu:1e-8:1e8"])
def test_pencil_vs_dd(dim, cells, coef):
    """square / cube cells (h = 1 / max cells on every axis: the pencil kernel's
    structure D = c 1 1^T); anisotropic cells take the older kernels (below)"""
    h = [1.0 / max(cells)] * dim
    o = Oracle(dim, cells, 0)
    o.set_h(h + [1.0] * (3 - dim))
    o.gen_inputs(coef, 4242)
    sp = hd.Space(dim, cells, 0, sizes=h)
    try:
        o.run("port_hybridize")
    except OracleError as exc:  # the reference raises: so must the device (exact path)
        assert "SingularBlock" in str(exc)
        with pytest.raises(hd.SingularBlockError):
            sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
        return
    o.run("dd_hybridize")
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    hv, gv = op.values()
    h_dd, g_dd = o.get("H.values_dd"), o.get("g_dd")
    assert rel_err(hv, h_dd) <= TOL and rel_err(gv, g_dd) <= TOL
    ro, _ = sp.pattern("H")
    if len(hv):
        assert _row_rel(ro, hv, h_dd) <= 1e-13
    if coef == "logu:1e-2:1e2" and max(cells) <= 128:  # the acceptance bound grows like h^-2
        assert op.exact_cells() == 0


@pytest.mark.parametrize("dim,cells", [(3, (37, 5, 7)), (2, (75, 9))])
def test_pencil_matches_brick_kernel(dim, cells, monkeypatch):
    """the brick kernel (Neumann form) and the pencil kernel (Sherman-Morrison form)
    are two different evaluations of the same inverse: they agree to a few ulp"""
    h = [1.0 / max(cells)] * dim
    o = Oracle(dim, cells, 0)
    o.set_h(h)
    o.gen_inputs("logu:1e-2:1e2", 5)
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    sp = hd.Space(dim, cells, 0, sizes=h)
    hp = sp.hybridize(a, b, f).values()
    monkeypatch.setenv("HDR_RT0_BRICK", "1")
    hb = sp.hybridize(a, b, f).values()
    assert rel_err(hp[0], hb[0]) <= 1e-13 and rel_err(hp[1], hb[1]) <= 1e-13


def test_pencil_forced_exact_and_reset():
    h = [1.0 / 70] * 3
    o = Oracle(3, (70, 3, 2), 0)
    o.set_h(h)
    o.gen_inputs("logu:1e-2:1e2", 8)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    sp = hd.Space(3, (70, 3, 2), 0, sizes=h)
    sp.set_exact_policy(force=True)
    for _ in range(2):
        op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
        assert op.exact_cells() == sp.ncells
        hv, gv = op.values()
        assert rel_err(hv, o.get("H.values_dd")) <= TOL and rel_err(gv, o.get("g_dd")) <= TOL
    sp.set_exact_policy(force=False)
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    assert op.exact_cells() == 0


def test_pencil_deterministic_and_one_launch_pair():
    o = Oracle(3, (16, 16, 16), 0)
    o.gen_inputs("logu:1e-2:1e2", 3)
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    sp = hd.Space(3, (16, 16, 16), 0)
    v1 = sp.hybridize(a, b, f).values()
    n0 = hd.launch_count()
    v2 = sp.hybridize(a, b, f).values()
    assert np.array_equal(v1[0], v2[0]) and np.array_equal(v1[1], v2[1])
    assert hd.launch_count() - n0 <= 2  # the pencil kernel + the (empty) exact-path tail


@pytest.mark.parametrize("dim,cells", [(3, (64, 3, 2)), (2, (75, 9))])
def test_anisotropic_cells_take_the_structured_kernels(dim, cells):
    """unit-domain meshes with unequal counts: box cells, D is not c 1 1^T, the
    brick kernel (Neumann form) runs; the 1e-11 contract holds"""
    o = Oracle(dim, cells, 0)
    o.gen_inputs("logu:1e-4:1e4", 4242)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    sp = hd.Space(dim, cells, 0)
    hv, gv = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat")).values()
    assert rel_err(hv, o.get("H.values_dd")) <= TOL and rel_err(gv, o.get("g_dd")) <= TOL


@pytest.mark.parametrize("dim,cells", MESHES)
def test_condense_pencil_bit_identical(dim, cells, monkeypatch):
    """k = 0 static condensation in one pass (k_sc_pencil): S and f_S carry the
    reference's bits (the oracle's port is pinned bit-exact to the reference) on
    every boundary configuration, and equal the two-colour kernel's"""
    h = [1.0 / max(cells)] * dim
    o = Oracle(dim, cells, 0)
    o.set_h(h + [1.0] * (3 - dim))
    o.gen_inputs("logu:1e-2:1e2", 99)
    o.run("port_condense")
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    sp = hd.Space(dim, cells, 0, sizes=h)
    ro, ci = sp.pattern("S")
    assert np.array_equal(ro, o.getq("S.row_offsets")) and np.array_equal(ci, o.getq("S.col_indices"))
    n0 = hd.launch_count()
    sv, fs = sp.static_condense(a, b, f).values()
    assert hd.launch_count() - n0 <= 1  # one pass, no colours
    assert np.array_equal(sv, o.get("S.values")) and np.array_equal(fs, o.get("f_s"))
    monkeypatch.setenv("HDR_SC_NO_PENCIL", "1")
    sv2, fs2 = sp.static_condense(a, b, f).values()
    assert np.array_equal(sv, sv2) and np.array_equal(fs, fs2)

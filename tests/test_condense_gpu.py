"""Static condensation, condensed recovery and SpMV on the device (GPU).

Contract: S pattern / master_globals bit-exact against the reference; S, f_S
and the recovered solution within 1e-11 of max|entry| of the double-double
oracle on the bit-identical A_T; for k = 0 (S = P^T A_hat P) bit-identical to
the reference itself.  SpMV: bit-identical to the reference's sequential row
sums (src/csr.cpp:77-87) on the same matrix and vector.
"""
import numpy as np
import pytest

from conftest import has_cuda, load_golden, GOLDEN_CASES
from oracle_lib import Oracle, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-11

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402

UNWEIGHTED = [c for c in GOLDEN_CASES if "weighted" not in c]


def seq_spmv(ro, ci, v, x):
    """The reference's spmv loop, vectorised across rows, sequential along each row."""
    n = len(ro) - 1
    lens = np.diff(ro)
    y = np.zeros(n)
    for j in range(int(lens.max()) if n else 0):
        rows = np.nonzero(lens > j)[0]
        k = ro[rows] + j
        y[rows] = y[rows] + v[k] * x[ci[k]]
    return y


@pytest.mark.parametrize("name", UNWEIGHTED)
def test_condense_vs_reference_and_dd(name):
    g = load_golden(name)
    o = Oracle(g["dim"], g["cells"], g["k"])
    o.gen_inputs(g["coef"], g["seed"])
    o.run("port_condense")
    o.run("dd_condense")
    o.run("dd_recover_condensed")
    sp = hd.Space(g["dim"], g["cells"], g["k"])
    op = sp.static_condense(g["alpha"], g["beta"], g["f_hat"])
    sv, fs = op.values()
    if g["k"] == 0:  # S = P^T A_hat P: the same two-term sums as the reference
        assert np.array_equal(sv, g["S.values"])
        assert np.array_equal(fs, g["f_s"])
    assert rel_err(sv, o.get("S.values_dd")) <= TOL
    assert rel_err(fs, o.get("f_s_dd")) <= TOL
    x = op.recover(g["x_b"], g["f_hat"])
    assert rel_err(x, o.get("x_cond_dd")) <= TOL
    # masters are copied through
    nm = len(g["master_globals"])
    assert np.array_equal(x[g["master_globals"]], g["x_b"][:nm])
    print(f"{name}: S {rel_err(sv, o.get('S.values_dd')):.1e} f_S {rel_err(fs, o.get('f_s_dd')):.1e} "
          f"(reference f_S vs DD {rel_err(g['f_s'], o.get('f_s_dd')):.1e})")


@pytest.mark.parametrize("dim,cells,k,coef", [
    (3, (6, 5, 4), 1, "logu:1e-2:1e2"), (3, (5, 4, 4), 1, "logu:1e-3:1e3"), (2, (7, 6), 2, "logu:1e-2:1e2"),
    (3, (3, 3, 2), 2, "logu:1e-3:1e3"), (3, (2, 2, 2), 3, "checker:1e-2:1e2"), (3, (12, 12, 12), 0, "logu:1e-2:1e2"),
])
def test_condense_moderate_vs_dd(dim, cells, k, coef):
    o = Oracle(dim, cells, k)
    o.gen_inputs(coef, 77)
    o.run("port_condense")
    o.run("dd_condense")
    o.run("dd_recover_condensed")
    sp = hd.Space(dim, cells, k)
    ro, ci = sp.pattern("S")
    assert np.array_equal(ro, o.getq("S.row_offsets")) and np.array_equal(ci, o.getq("S.col_indices"))
    op = sp.static_condense(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    sv, fs = op.values()
    assert rel_err(sv, o.get("S.values_dd")) <= TOL
    assert rel_err(fs, o.get("f_s_dd")) <= TOL
    x = op.recover(o.get("x_b"), o.get("f_hat"))
    assert rel_err(x, o.get("x_cond_dd")) <= TOL


def test_spmv_bit_exact_reference_order():
    o = Oracle(3, (6, 6, 6), 1)
    o.gen_inputs("logu:1e-2:1e2", 5)
    sp = hd.Space(3, (6, 6, 6), 1)
    hop = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    _, _, ro, ci, hv = hop.h_mat()
    x = o.get("lambda")
    assert np.array_equal(hop.spmv(x), seq_spmv(ro, ci, hv, x))
    cop = sp.static_condense(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    _, _, ro, ci, sv = cop.s_mat()
    xb = o.get("x_b")
    assert np.array_equal(cop.spmv(xb), seq_spmv(ro, ci, sv, xb))


def test_spmv_matches_reference_on_reference_matrix():
    """Same matrix and vector as the reference -> identical bits (golden H_lambda)."""
    import ctypes
    import torch

    g = load_golden("h3_rt1_2x2x2_logu")
    ro, ci, v, x = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in
                    (g["H.row_offsets"], g["H.col_indices"], g["H.values"], g["lambda"]))
    y = torch.empty(len(g["H.row_offsets"]) - 1, dtype=torch.float64, device="cuda")
    lib = hd._capi.load()
    st = lib.hdr_csr_spmv_device(y.numel(), ro.data_ptr(), ci.data_ptr(), v.data_ptr(), x.data_ptr(), y.data_ptr(),
                                 None)
    assert st == 0
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), g["H_lambda"])


@pytest.mark.parametrize("form", ["HDR_SPMV_ROWS", "HDR_SPMV_TILES"])
@pytest.mark.parametrize("dim,cells,k", [(3, (9, 5, 4), 0), (3, (5, 4, 3), 1), (2, (37, 5), 2), (3, (2, 2, 3), 3)])
def test_spmv_forms_bit_exact(dim, cells, k, form, monkeypatch):
    """both SpMV kernels (thread per row; coalesced warp tiles through shared memory)
    reproduce the reference's sequential row sums bit for bit, on short and long rows
    (rows that span several tiles: RT3) and on a row count that is no multiple of 32"""
    monkeypatch.setenv(form, "1")
    o = Oracle(dim, cells, k)
    o.gen_inputs("logu:1e-2:1e2", 11)
    sp = hd.Space(dim, cells, k)
    hop = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    _, _, ro, ci, hv = hop.h_mat()
    x = o.get("lambda")
    assert np.array_equal(hop.spmv(x), seq_spmv(ro, ci, hv, x))
    cop = sp.static_condense(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    _, _, ro, ci, sv = cop.s_mat()
    xb = o.get("x_b")
    assert np.array_equal(cop.spmv(xb), seq_spmv(ro, ci, sv, xb))

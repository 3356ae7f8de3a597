"""Essential-boundary elimination (eliminate_essential, src/reduction.cpp:589-698)
on the FE front end, feeding the device's general element path (GPU).

The reference (oracle/_ref/ref_harness dump essential=1) eliminates every
boundary face with a seeded normal flux and then runs hybridize /
recover_hybrid / static_condense on the reduced inputs.  Here the same space
goes through fe_reduction_inputs (device-assembled blocks) and the Python
restatement of eliminate_essential: the reduced blocks, right-hand side, dof
numbering, P and C must be bit-identical to the reference's; the device's
hybridize of the reduced inputs gives the reference's H / S patterns bit for
bit and its values to the reference's own accuracy (it is the less accurate of
the two).
"""
import numpy as np
import pytest

from conftest import has_cuda
from oracle_lib import REF_HARNESS, rel_err, run_ref_dump

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402
from paper_1801_08914_b200 import algebraic as alg  # noqa: E402
from paper_1801_08914_b200.inputs import make_inputs  # noqa: E402

CASES = [(3, (3, 2, 2), 1, ("logu", 1e-2, 1e2)), (3, (4, 4, 4), 0, ("logu", 1e-2, 1e2)),
         (2, (5, 4), 1, ("logu", 1e-2, 1e2)), (3, (2, 2, 2), 2, ("uniform", 1.0, 1.0)),
         (3, (3, 3, 2), 1, ("softhard", -4, 0))]


@pytest.mark.parametrize("dim,cells,k,coef", CASES)
def test_eliminate_essential_vs_reference(dim, cells, k, coef, tmp_path):
    if not REF_HARNESS.exists():
        pytest.skip("ref_harness not built")
    seed = 91
    ref = run_ref_dump(tmp_path / "e.bin", dim, cells, k, f"{coef[0]}:{coef[1]}:{coef[2]}", seed, essential=True)
    alpha, beta, f_hat = make_inputs(dim, cells, k, coef, seed)
    sp = hd.Space(dim, cells, k)
    inputs = alg.fe_reduction_inputs(sp, alpha, beta, f_hat)
    _, cm, cp = alg._face_geometry(sp)
    bfaces = np.nonzero((cm < 0) | (cp < 0))[0]
    bcs = [alg.EssentialBc(int(f), float(v)) for f, v in zip(bfaces, ref["ess.flux"])]
    el = alg.eliminate_essential(sp, inputs, bcs)
    red = el.inputs
    # the reduced instance, bit for bit
    assert np.array_equal(el.kept_globals, ref["ess.kept_globals"])
    assert np.array_equal(el.prescribed, ref["ess.prescribed"])
    assert np.array_equal([np.shape(b)[0] for b in red.blocks], ref["ess.block_sizes"])
    assert np.array_equal(np.concatenate([np.ravel(b) for b in red.blocks]), ref["a_hat"])
    assert np.array_equal(red.f_hat, ref["f_hat"])
    assert np.array_equal(red.dof_global, ref["dof_global"])
    for name, m in (("P", red.p_mat), ("C", red.c_mat)):
        assert np.array_equal(m.row_offsets, ref[name + ".row_offsets"]), name
        assert np.array_equal(m.col_indices, ref[name + ".col_indices"]), name
        assert np.array_equal(m.values, ref[name + ".values"]), name
    assert red.interior_global_begin == int(ref["ess.interior_global_begin"][0])
    # the device's hybridize / recovery / condensation of the reduced inputs
    op, g = alg.hybridize(red, symmetric=True)
    assert np.array_equal(op.h_mat.row_offsets, ref["H.row_offsets"])
    assert np.array_equal(op.h_mat.col_indices, ref["H.col_indices"])
    eh, eg = rel_err(op.h_mat.values, ref["H.values"]), rel_err(g, ref["g"])
    x_hat, x = alg.recover_hybrid(op, ref["lambda"], red.f_hat)
    ex = rel_err(x_hat, ref["x_hat"])
    cop, f_s = alg.static_condense(red, symmetric=True)
    assert np.array_equal(cop.s_mat.row_offsets, ref["S.row_offsets"])
    assert np.array_equal(cop.s_mat.col_indices, ref["S.col_indices"])
    assert np.array_equal(cop.master_globals, ref["master_globals"])
    es = rel_err(cop.s_mat.values, ref["S.values"])
    print(f"{cells} RT{k} {coef[0]}: reduced n_hat {red.n_hat}, H vs reference {eh:.1e}, g {eg:.1e}, "
          f"x_hat {ex:.1e}, S {es:.1e}")
    assert eh <= 1e-7 and eg <= 1e-7 and ex <= 1e-7 and es <= 1e-12


def test_hybridized_matrix_with_essential_boundary():
    """The bindings' hybridized_matrix with essential_boundary (build_problem's
    elimination of every boundary face, src/driver.cpp:187-195)."""
    (nr, nc, ro, ci, v), g = hd.hybridized_matrix({"cells": [3, 3, 3], "order": 1, "essential_boundary": True})
    (nr0, _, _, _, _), _ = hd.hybridized_matrix({"cells": [3, 3, 3], "order": 1})
    assert nr == nr0 and len(g) == nr and len(v) == ro[-1]  # boundary faces carry no multipliers
    h = alg.Csr(nr, nc, np.array(ro), np.array(ci), np.array(v)).to_dense()
    assert np.max(np.abs(h - h.T)) == 0.0 and np.all(np.linalg.eigvalsh(h) > 0)

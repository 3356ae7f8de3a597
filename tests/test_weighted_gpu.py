"""Weighted constraint rows (build_C weighted, reduction.cpp:182-195) on the FE
path (GPU): C rows are the face moments, so H_T = W_F A_T^-1 W_F^T per cell.

Contract: H pattern bit-exact against the reference (golden weighted case);
H, g, x_hat, x within 1e-11 of max|entry| of the double-double oracle on the
bit-identical A_T; static condensation (which does not involve C) unchanged.
"""
import numpy as np
import pytest

from conftest import has_cuda, load_golden
from oracle_lib import Oracle, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-11

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402


def test_weighted_golden_vs_reference_and_dd():
    g = load_golden("h3_rt1_3x2x2_logu_weighted")
    o = Oracle(g["dim"], g["cells"], g["k"], weighted=True)
    o.gen_inputs(g["coef"], g["seed"])
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    sp = hd.Space(g["dim"], g["cells"], g["k"], weighted=True)
    ro, ci = sp.pattern("H")
    assert np.array_equal(ro, g["H.row_offsets"]) and np.array_equal(ci, g["H.col_indices"])
    op = sp.hybridize(g["alpha"], g["beta"], g["f_hat"])
    hv, gv = op.values()
    assert rel_err(hv, o.get("H.values_dd")) <= TOL and rel_err(gv, o.get("g_dd")) <= TOL
    x_hat, x = op.recover(o.get("lambda"), o.get("f_hat"))
    assert rel_err(x_hat, o.get("x_hat_dd")) <= TOL and rel_err(x, o.get("x_dd")) <= TOL
    print(f"weighted: H {rel_err(hv, o.get('H.values_dd')):.1e} "
          f"(reference {rel_err(g['H.values'], o.get('H.values_dd')):.1e})")


@pytest.mark.parametrize("dim,cells,k", [(2, (4, 3), 2), (2, (3, 3), 3), (3, (2, 2, 2), 2), (3, (3, 3, 2), 0)])
def test_weighted_vs_dd(dim, cells, k):
    o = Oracle(dim, cells, k, weighted=True)
    o.gen_inputs("logu:1e-2:1e2", 31 + k)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    sp = hd.Space(dim, cells, k, weighted=True)
    ro, ci = sp.pattern("H")
    assert np.array_equal(ro, o.getq("H.row_offsets")) and np.array_equal(ci, o.getq("H.col_indices"))
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    hv, gv = op.values()
    assert rel_err(hv, o.get("H.values_dd")) <= TOL and rel_err(gv, o.get("g_dd")) <= TOL
    x_hat, x = op.recover(o.get("lambda"), o.get("f_hat"))
    assert rel_err(x_hat, o.get("x_hat_dd")) <= TOL and rel_err(x, o.get("x_dd")) <= TOL
    # static condensation does not involve C: same S as the unweighted space
    o.run("port_condense")
    o.run("dd_condense")
    cop = sp.static_condense(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    sv, fs = cop.values()
    assert rel_err(sv, o.get("S.values_dd")) <= TOL and rel_err(fs, o.get("f_s_dd")) <= TOL


def test_weighted_config_front_end():
    (nr, nc, ro, ci, v), g = hd.hybridized_matrix({"dim": 3, "cells": [2, 2, 2], "order": 1, "weighted": True})
    assert nr == nc == len(ro) - 1 and len(v) == ro[-1] and np.all(np.isfinite(v))

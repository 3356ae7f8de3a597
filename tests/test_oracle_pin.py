"""Pins the CPU oracle (oracle/hdr_oracle.c) against the REFERENCE's own outputs:
the golden fixtures in tests/golden/ were produced by running the reference
library (oracle/_ref, compiled from /root/reference) on seeded inputs
(tests/golden/make_golden.py).  The oracle's restatement of the reference's
production algorithm must match those bits exactly; its double-double value
oracle must agree with the reference wherever the reference itself is accurate.
"""
import numpy as np
import pytest

from conftest import load_golden
from oracle_lib import Oracle, build_reference, rel_err

BIT_EXACT = ["ref_divdiv", "ref_mass", "ref_face_moments", "ref_unit_load", "alpha", "beta", "f_hat", "lambda", "x_b"]


def make_oracle(g):
    o = Oracle(g["dim"], g["cells"], g["k"], weighted=g["weighted"])
    o.gen_inputs(g["coef"], g["seed"])
    return o


def test_inputs_and_reference_element_bit_exact(golden):
    o = make_oracle(golden)
    for name in BIT_EXACT:
        assert np.array_equal(o.get(name), golden[name]), name


def test_element_matrices_bit_exact(golden):
    if "a_hat" not in golden:
        pytest.skip("fixture without explicit blocks")
    o = make_oracle(golden)
    o.run("assemble")
    assert np.array_equal(o.get("a_hat"), golden["a_hat"])


def test_structure_bit_exact(golden):
    o = make_oracle(golden)
    o.run("structure")
    for p in ("P", "C"):
        assert np.array_equal(o.getq(p + ".row_offsets"), golden[p + ".row_offsets"])
        assert np.array_equal(o.getq(p + ".col_indices"), golden[p + ".col_indices"])
        assert np.array_equal(o.get(p + ".values"), golden[p + ".values"])
    if "dof_global" in golden:
        assert np.array_equal(o.getq("dof_global"), golden["dof_global"])
        assert np.array_equal(o.get("dof_sign"), golden["dof_sign"])


def test_port_hybridize_recover_bit_exact(golden):
    o = make_oracle(golden)
    o.run("port_hybridize")
    for s in ("row_offsets", "col_indices"):
        assert np.array_equal(o.getq("H." + s), golden["H." + s])
    assert np.array_equal(o.get("H.values"), golden["H.values"])
    assert np.array_equal(o.get("g"), golden["g"])
    o.run("port_recover")
    assert np.array_equal(o.get("x_hat"), golden["x_hat"])
    assert np.array_equal(o.get("x"), golden["x"])
    o.run("spmv_H")
    assert np.array_equal(o.get("H_lambda"), golden["H_lambda"])


def test_port_condense_bit_exact(golden):
    o = make_oracle(golden)
    o.run("port_condense")
    for s in ("row_offsets", "col_indices"):
        assert np.array_equal(o.getq("S." + s), golden["S." + s])
    assert np.array_equal(o.get("S.values"), golden["S.values"])
    assert np.array_equal(o.get("f_s"), golden["f_s"])
    assert np.array_equal(o.getq("master_globals"), golden["master_globals"])
    o.run("port_recover_condensed")
    assert np.array_equal(o.get("x_cond"), golden["x_cond"])
    o.run("spmv_S")
    assert np.array_equal(o.get("S_x_b"), golden["S_x_b"])


def test_dd_oracle_agrees_with_reference(golden):
    """The DD truth and the reference's production output differ by the
    reference's own rounding; on these small meshes that is
    < 1e-9.  S, which is well conditioned, agrees to ~1e-15."""
    o = make_oracle(golden)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    o.run("port_condense")
    o.run("dd_condense")
    o.run("dd_recover_condensed")
    assert rel_err(golden["H.values"], o.get("H.values_dd")) < 1e-9
    assert rel_err(golden["g"], o.get("g_dd")) < 1e-9
    assert rel_err(golden["x_hat"], o.get("x_hat_dd")) < 1e-9
    assert rel_err(golden["S.values"], o.get("S.values_dd")) < 1e-14
    assert rel_err(golden["f_s"], o.get("f_s_dd")) < 1e-9
    assert rel_err(golden["x_cond"], o.get("x_cond_dd")) < 1e-11


def test_known_answer_unit_cube_rt0():
    """tests/unit_reduction.cpp:280-287: for k = 0, S equals the assembled A; and
    H is symmetric positive definite on 3^3 (acceptance A3, tests/acceptance.cpp:115-127)."""
    o = Oracle(3, (3, 3, 3), 0)
    o.gen_inputs("uniform:1:1", 5)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    nr, nc, ro, ci, hv = o.csr("H", "values_dd")
    dense = np.zeros((nr, nc))
    for i in range(nr):
        dense[i, ci[ro[i]:ro[i + 1]]] = hv[ro[i]:ro[i + 1]]
    assert np.max(np.abs(dense - dense.T)) <= 1e-12 * np.max(np.abs(dense))
    assert np.all(np.linalg.eigvalsh(0.5 * (dense + dense.T)) > 0)


def test_dd_element_matches_dd_assembly():
    """hdo_dd_element (used for sampled full-size parity) equals the assembled DD H."""
    o = Oracle(3, (3, 3, 2), 1)
    o.gen_inputs("logu:1e-2:1e2", 11)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    nr, nc, ro, ci, hv = o.csr("H", "values_dd")
    H = {}
    for e in range(o.size("ncells")):
        rows, h, g, _ = o.dd_element(e)
        for a, r in enumerate(rows):
            for b, c in enumerate(rows):
                H[(r, c)] = H.get((r, c), 0.0) + h[a, b]
    worst = 0.0
    for i in range(nr):
        for p in range(ro[i], ro[i + 1]):
            worst = max(worst, abs(H[(i, ci[p])] - hv[p]))
    assert worst <= 1e-15 * np.max(np.abs(hv))


@pytest.mark.parametrize("dim,k", [(2, 0), (2, 1), (3, 0), (3, 1), (3, 2), (3, 3)])
def test_reference_element_identities(dim, k):
    """Element-matrix identities of tests/unit_fem.cpp:80-146: symmetric up to
    rounding, mass SPD, divdiv PSD of rank (k+1)^dim, refined quadrature agrees."""
    h = [0.25, 0.5, 0.125][:dim]
    D, M, _, _ = build_reference(dim, k, h, k + 2)
    assert np.max(np.abs(D - D.T)) <= 1e-13 * np.max(np.abs(D))
    assert np.max(np.abs(M - M.T)) <= 1e-13 * np.max(np.abs(M))
    assert np.all(np.linalg.eigvalsh(0.5 * (M + M.T)) > 0)
    ev = np.linalg.eigvalsh(0.5 * (D + D.T))
    assert int(np.sum(ev > 1e-10 * ev.max())) == (k + 1) ** dim
    D2, M2, _, _ = build_reference(dim, k, h, k + 6)
    assert np.max(np.abs(D2 - D)) <= 1e-12 * np.max(np.abs(D))
    assert np.max(np.abs(M2 - M)) <= 1e-12 * np.max(np.abs(M))

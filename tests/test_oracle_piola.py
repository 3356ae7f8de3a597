"""Config-4 oracle (perturbed trilinear cells, contravariant Piola): a
RESTATEMENT — the reference has affine boxes only.  It is
pinned by (1) the affine limit, which must reproduce the reference element
(itself pinned bit-exact against the reference build), (2) the per-element
identity divdiv = B^T W^-1 B with the Piola-mapped pressures (adapting the
reference's acceptance A7, tests/acceptance.cpp:175-197), (3) convergence
under refined quadrature (tests/unit_fem.cpp:135-146 pattern), (4) symmetry and
definiteness.  CPU only."""
import numpy as np
import pytest

from oracle_lib import Oracle, box_vertices, build_reference, piola_element, rel_err


@pytest.mark.parametrize("k", [0, 1, 2])
def test_affine_limit_reproduces_reference(k):
    h = (1 / 24, 1 / 24, 1 / 24)
    D0, M0, _, _ = build_reference(3, k, h, k + 2)
    D, M = piola_element(k, h, box_vertices(h, origin=(0.25, 0.5, 0.125)), k + 2)
    assert rel_err(D, D0) <= 1e-14 and rel_err(M, M0) <= 1e-14


def _perturbed(h, seed, frac=0.2):
    rng = np.random.default_rng(seed)
    v = box_vertices(h)
    return v + rng.uniform(-frac, frac, size=v.shape) * np.array(h)


@pytest.mark.parametrize("k", [1, 2])
def test_divdiv_is_projection_identity(k):
    h = (1 / 24, 1 / 24, 1 / 24)
    D, M, B, W = piola_element(k, h, _perturbed(h, k), k + 2, pressure=True)
    assert rel_err(B.T @ np.linalg.solve(W, B), D) <= 1e-11


@pytest.mark.parametrize("k", [1, 2])
def test_symmetric_and_definite(k):
    h = (1 / 24, 1 / 24, 1 / 24)
    D, M = piola_element(k, h, _perturbed(h, 10 + k), k + 2)
    # as in the reference's accumulation (w * d_i * d_j), D is symmetric up to rounding
    assert np.array_equal(M, M.T) and rel_err(D, D.T) <= 1e-15
    assert np.linalg.eigvalsh(M).min() > 0
    ev = np.linalg.eigvalsh(D)
    assert ev.min() > -1e-12 * ev.max()
    A = 1e3 * D + 1e-3 * M
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0


def test_refined_quadrature_converges():
    k = 2
    h = (1 / 24, 1 / 24, 1 / 24)
    v = _perturbed(h, 7)
    ref = piola_element(k, h, v, k + 8)
    errs = []
    for nq in (k + 2, k + 4, k + 6):
        D, M = piola_element(k, h, v, nq)
        errs.append(max(rel_err(D, ref[0]), rel_err(M, ref[1])))
    assert errs[0] < 1e-2 and errs[1] < errs[0] and errs[2] < errs[1], errs


def test_mesh_perturbation_inputs():
    o = Oracle(3, (3, 2, 2), 1)
    o.gen_inputs("logu:1e-3:1e3;perturb=0.2", 1004)
    vt = o.get("vertices").reshape(3, 3, 4, 3)  # (z, y, x, coord)
    h = np.array([1 / 3, 1 / 2, 1 / 2])
    grid = np.stack(np.meshgrid(np.arange(4) * h[0], np.arange(3) * h[1], np.arange(3) * h[2], indexing="ij"), -1)
    grid = grid.transpose(2, 1, 0, 3)
    d = vt - grid
    boundary = np.ones((3, 3, 4), bool)
    boundary[1:-1, 1:-1, 1:-1] = False
    assert np.all(d[boundary] == 0.0)
    assert np.all(np.abs(d[~boundary]) <= 0.2 * h + 1e-15) and np.any(d[~boundary] != 0.0)
    # the element matrices of the mesh are the Piola ones, and the FE stages run on them
    a0 = o.element_matrix(0)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    assert rel_err(o.get("H.values"), o.get("H.values_dd")) < 1e-4
    o2 = Oracle(3, (3, 2, 2), 1)
    o2.gen_inputs("logu:1e-3:1e3", 1004)
    assert not np.array_equal(a0, o2.element_matrix(0))

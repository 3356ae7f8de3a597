"""Device pcg for the reduced systems (the reference's pcg,
src/solvers.cpp:109-163, with its none / Jacobi preconditioners) (GPU).

Checks: the solution of H lambda = g (hybrid) and S x_b = f_s (condensed)
against a dense float64 solve; the full pipeline hybridize -> pcg -> recover
reproduces the conforming solution that static condensation gives; the
reference's breakdown errors."""
import numpy as np
import pytest

from conftest import has_cuda
from oracle_lib import Oracle, rel_err

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402


def dense(ro, ci, v, n):
    a = np.zeros((n, n))
    for r in range(n):
        a[r, ci[ro[r]:ro[r + 1]]] += v[ro[r]:ro[r + 1]]
    return a


@pytest.mark.parametrize("precond", ["jacobi", "none"])
@pytest.mark.parametrize("dim,cells,k", [(3, (4, 4, 3), 0), (3, (3, 3, 2), 1), (2, (6, 5), 2)])
def test_hybrid_pcg_solves_h(dim, cells, k, precond):
    o = Oracle(dim, cells, k)
    o.gen_inputs("logu:1e-1:1e1", 50 + k)
    sp = hd.Space(dim, cells, k)
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    op.symmetrize()
    lam, rep = op.pcg(rtol=1e-12, maxit=5000, precond=precond)
    assert rep["converged"] and rep["relative_residuals"][0] == 1.0
    ro, ci = sp.pattern("H")
    hv, g = op.values()
    H = dense(ro, ci, hv, sp.m)
    ref = np.linalg.solve(H, g)
    assert rel_err(lam, ref) <= 1e-9
    # the reduced solve feeds the recovery on the device; hybrid and condensed
    # solutions of the same FE problem agree
    x_hat, x = op.recover(lam, o.get("f_hat"))
    cop = sp.static_condense(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    xb, rep2 = cop.pcg(rtol=1e-12, maxit=5000, precond=precond)
    assert rep2["converged"]
    xc = cop.recover(xb, o.get("f_hat"))
    assert rel_err(x, xc) <= 1e-8


def test_pcg_host_csr_and_errors():
    rng = np.random.default_rng(0)
    n = 40
    b_ = rng.standard_normal((n, n))
    a = b_ @ b_.T + n * np.eye(n)
    ro = np.arange(0, n * n + 1, n)
    ci = np.tile(np.arange(n), n)
    x, rep = hd.pcg((n, n, ro, ci, a.ravel()), np.ones(n), rtol=1e-13)
    assert rep["converged"] and rel_err(x, np.linalg.solve(a, np.ones(n))) <= 1e-11
    neg = a.copy()
    neg[3, 3] = -1.0
    with pytest.raises(hd.ValidationError):  # ZeroDiagonal (non-positive diagonal) under Jacobi
        hd.pcg((n, n, ro, ci, neg.ravel()), np.ones(n))
    ind = -a
    with pytest.raises(hd.ValidationError):  # <p, Ap> <= 0 without preconditioning
        hd.pcg((n, n, ro, ci, ind.ravel()), np.ones(n), precond="none")
    x0, rep0 = hd.pcg((n, n, ro, ci, a.ravel()), np.zeros(n))
    assert rep0["converged"] and np.all(x0 == 0.0)


def test_alg_pcg():
    from paper_1801_08914_b200.algebraic import Csr, ReductionInputs
    o = Oracle(3, (3, 2, 2), 1)
    o.gen_inputs("logu:1e-1:1e1", 9)
    o.run("structure")
    o.run("assemble")
    n, nc = o.size("n"), o.size("ncells")
    inp = ReductionInputs(list(o.get("a_hat").reshape(nc, n, n)), Csr(*o.csr("P")), Csr(*o.csr("C")), o.get("f_hat"))
    op, g = hd.algebraic.hybridize(inp, symmetric=True)
    lam, rep = op.pcg(rtol=1e-12, maxit=2000)
    assert rep["converged"]
    H = op.h_mat.to_dense()
    assert rel_err(lam, np.linalg.solve(H, g)) <= 1e-9

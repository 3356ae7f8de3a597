"""Device AMG / SGS preconditioners and the reduced solve
against the reference itself (oracle/_ref/ref_harness amg=1: the reference's
amg_setup / amg_apply / ssgs_setup / pcg on its own H).

  * on the reference's H: every level's A, P, R and the coarse matrix
    bit-identical (amg_setup, src/amg.cpp:189-244); one V-cycle and one SGS
    application on g bit-identical (amg_apply :268, solvers.cpp:60-107);
  * pcg (src/solvers.cpp:109-163, rtol 1e-12 and maxit 2000 of RunConfig) with
    amg / sgs / jacobi on that H: iteration counts within +-1 of the reference;
  * the device pipeline hybridize -> symmetrize -> pcg(amg) on the device's own
    H over the soft-hard sweep (src/mesh.cpp:168-191): iterations within 3 %
    (at least +-1) of the reference's, true residual at the rtol level.
"""
import tempfile
from pathlib import Path

import numpy as np
import pytest

from conftest import has_cuda
from oracle_lib import REF_HARNESS, run_ref_dump

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)
if not REF_HARNESS.exists():
    pytest.skip("oracle/_ref/ref_harness not built", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402

CASES = [  # dim, cells, k, coef
    (3, (4, 4, 4), 0, "softhard:-8"),
    (3, (8, 8, 8), 0, "softhard:8"),
    (3, (8, 8, 8), 1, "softhard:-4"),
    (3, (16, 16, 16), 0, "softhard:4"),
    (3, (12, 12, 12), 1, "softhard:8"),
    (2, (32, 32), 1, "softhard:-8"),
    (3, (32, 32, 32), 0, "softhard:-8"),
    (3, (16, 16, 16), 1, "logu:1e-2:1e2"),
]

_cache = {}


def ref(case):
    if case not in _cache:
        dim, cells, k, coef = case
        with tempfile.TemporaryDirectory() as td:
            _cache[case] = run_ref_dump(Path(td) / "d.bin", dim, cells, k, coef, 77, blocks=False, amg=True)
    return _cache[case]


def true_residual(a, x, b):
    import scipy.sparse as sps

    m = sps.csr_matrix((a[4], a[3], a[2]), shape=a[:2])
    return np.linalg.norm(b - m @ x) / np.linalg.norm(b)


def csr(d, name):
    sh = d[f"{name}.shape"]
    return int(sh[0]), int(sh[1]), d[f"{name}.row_offsets"], d[f"{name}.col_indices"], d[f"{name}.values"]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}d-{'x'.join(map(str, c[1]))}-k{c[2]}-{c[3]}" for c in CASES])
def test_hierarchy_and_cycle_bit_identical(case):
    d = ref(case)
    H = csr(d, "H")
    amg = hd.AmgHierarchy(H)
    assert amg.nlevels == int(d["amg.levels"][0])
    for lvl in range(amg.nlevels + 1):
        for w in ("A", "P", "R") if lvl < amg.nlevels else ("A",):
            name = f"amg.{w}{lvl}" if lvl < amg.nlevels else "amg.coarse"
            mine, theirs = amg.matrix(lvl, w), csr(d, name)
            assert mine[:2] == theirs[:2], (name, mine[:2], theirs[:2])
            for a, b in zip(mine[2:], theirs[2:]):
                assert np.array_equal(a, b), name
    assert np.array_equal(amg.apply(d["g"]), d["amg.z"])
    assert np.array_equal(hd.precond_apply(H, d["g"], "sgs"), d["sgs.z"])


@pytest.mark.parametrize("precond", ["amg", "sgs", "jacobi"])
@pytest.mark.parametrize("case", CASES[:6], ids=[f"{c[0]}d-{'x'.join(map(str, c[1]))}-k{c[2]}-{c[3]}" for c in CASES[:6]])
def test_pcg_iterations_on_reference_matrix(case, precond):
    d = ref(case)
    x, rep = hd.pcg(csr(d, "H"), d["g"], rtol=1e-12, maxit=2000, precond=precond)
    it_ref = int(d[f"pcg.{precond}.iterations"][0])
    assert rep["converged"]
    assert abs(rep["iterations"] - it_ref) <= 1, (rep["iterations"], it_ref)
    # same stopping point: the true residual of both solutions at the rtol level
    H = csr(d, "H")
    assert true_residual(H, x, d["g"]) <= 1e-10
    assert true_residual(H, d[f"pcg.{precond}.x"], d["g"]) <= 1e-10


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}d-{'x'.join(map(str, c[1]))}-k{c[2]}-{c[3]}" for c in CASES])
def test_device_pipeline_hybridize_pcg_amg(case):
    """solve_reduction's hybridization branch (src/driver.cpp:241-245) on the device."""
    dim, cells, k, coef = case
    d = ref(case)
    sp = hd.Space(dim, cells, k)
    op = sp.hybridize(d["alpha"], d["beta"], d["f_hat"])
    op.symmetrize()
    lam, rep = op.pcg(rtol=1e-12, maxit=2000, precond="amg")
    it_ref = int(d["pcg.amg.iterations"][0])
    assert rep["converged"]
    # H agrees with the reference's to ~1e-12, not bitwise, so the Krylov
    # trajectories part at that level: on the reference's own H the counts are
    # identical (test above); here they agree exactly except 2D RT1 with the
    # 1e16 contrast of p = -8 (123 vs 126), hence 3 % (at least 1)
    tol = max(1, int(np.ceil(0.03 * it_ref)))
    assert abs(rep["iterations"] - it_ref) <= tol, (rep["iterations"], it_ref)
    hv, gv = op.values()
    ro, ci = sp.pattern("H")
    assert true_residual((sp.m, sp.m, ro, ci, hv), lam, gv) <= 1e-10
    print(f"{case}: device {rep['iterations']} iterations, reference {it_ref}")


def test_pcg_rejects_nonsymmetric():
    ro = np.array([0, 2, 4])
    ci = np.array([0, 1, 0, 1])
    v = np.array([2.0, 1.0, 0.5, 2.0])
    with pytest.raises(ValueError):
        hd.pcg((2, 2, ro, ci, v), np.ones(2), precond="amg")


def test_amg_setup_failed_on_nonpositive_diagonal():
    """checked_inv_diag (amg.cpp:159-166) on a coarsening level: SetupFailed."""
    n = 100
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, a in ((i - 1, -1.0), (i, -2.0 if i == 7 else 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                rows.append(i), cols.append(j), vals.append(a)
    ro = np.searchsorted(np.array(rows), np.arange(n + 1))
    with pytest.raises(hd.SetupFailed):
        hd.AmgHierarchy((n, n, ro, np.array(cols), np.array(vals)))


@pytest.mark.parametrize("opts", [
    {"amg_theta": 0.25, "amg_cap": 200},
    {"amg_theta": 0.02, "amg_levels": 2},
    {"amg_omega": 0.5, "amg_cap": 16},
])
def test_nondefault_options_bit_identical(opts):
    """AmgOptions (amg.hpp:12-19) other than the defaults: the same hierarchy and cycle."""
    with tempfile.TemporaryDirectory() as td:
        d = run_ref_dump(Path(td) / "d.bin", 3, (8, 8, 8), 1, "softhard:4", 5, blocks=False, amg=True,
                         amg_options=opts)
    names = {"amg_theta": "strength_threshold", "amg_cap": "coarse_cap", "amg_levels": "max_levels",
             "amg_omega": "omega_factor"}
    amg = hd.AmgHierarchy(csr(d, "H"), **{names[k_]: v for k_, v in opts.items()})
    assert amg.nlevels == int(d["amg.levels"][0])
    for lvl in range(amg.nlevels):
        for w in ("A", "P", "R"):
            for a, b in zip(amg.matrix(lvl, w)[2:], csr(d, f"amg.{w}{lvl}")[2:]):
                assert np.array_equal(a, b)
    assert np.array_equal(amg.apply(d["g"]), d["amg.z"])


def test_pcg_zero_rhs_and_zero_diagonal():
    ro = np.array([0, 2, 4])
    ci = np.array([0, 1, 0, 1])
    x, rep = hd.pcg((2, 2, ro, ci, np.array([2.0, 1.0, 1.0, 2.0])), np.zeros(2), precond="amg")
    assert rep["converged"] and rep["iterations"] == 0 and np.all(x == 0)
    with pytest.raises(hd.ValidationError):  # ZeroDiagonal (solvers.cpp:32-44)
        hd.pcg((2, 2, ro, ci, np.array([0.0, 1.0, 1.0, 2.0])), np.ones(2), precond="sgs")

"""Algebraic batch path (hybridize / static_condense / recoveries on a general
ReductionInputs) on the device (GPU).

Contract: patterns and master_globals bit-exact against the
reference's own output on the FE-built inputs (golden fixtures + the oracle
port); values within 1e-11 of max|entry| of the double-double oracle on the
same blocks; on general non-FE inputs (random SPD blocks, duplicated / weighted
P, general C) against exact rational arithmetic.  Error behaviour mirrors the
reference's exceptions.
"""
from fractions import Fraction

import numpy as np
import pytest

from conftest import has_cuda, load_golden, GOLDEN_CASES
from oracle_lib import Oracle, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-11

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402
from paper_1801_08914_b200.algebraic import Csr, ReductionInputs  # noqa: E402

ALG = hd.algebraic


def fe_inputs(o: Oracle, marker: bool = False) -> ReductionInputs:
    """The FE-built ReductionInputs (build_reduction_inputs, reduction.cpp:200-222) from the oracle."""
    o.run("structure")
    o.run("assemble")
    n, ncells = o.size("n"), o.size("ncells")
    a_hat = o.get("a_hat").reshape(ncells, n, n)
    P = Csr(*o.csr("P"))
    C = Csr(*o.csr("C"))
    return ReductionInputs(list(a_hat), P, C, o.get("f_hat"),
                           interior_global_begin=o.size("face_dof_count") if marker else -1,
                           dof_global=o.getq("dof_global"))


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_alg_hybridize_fe_inputs(name):
    g = load_golden(name)
    o = Oracle(g["dim"], g["cells"], g["k"], weighted="weighted" in name)
    o.gen_inputs(g["coef"], g["seed"])
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    op, gv = ALG.hybridize(fe_inputs(o))
    H = op.h_mat
    assert np.array_equal(H.row_offsets, g["H.row_offsets"]) and np.array_equal(H.col_indices, g["H.col_indices"])
    e_h, e_g = rel_err(H.values, o.get("H.values_dd")), rel_err(gv, o.get("g_dd"))
    assert e_h <= TOL and e_g <= TOL, (e_h, e_g)
    # default: not symmetrized (the reference's DD oracle is not); symmetric=True
    # gives the reference's exactly symmetric H (what its pcg requires)
    if H.nrows:
        ops, _ = ALG.hybridize(fe_inputs(o), symmetric=True)
        Hs = ops.h_mat.to_dense()
        assert np.array_equal(Hs, Hs.T)
        Hd = H.to_dense()
        assert np.array_equal(Hs, 0.5 * (Hd + Hd.T))
    x_hat, x = ALG.recover_hybrid(op, o.get("lambda"), o.get("f_hat"))
    assert rel_err(x_hat, o.get("x_hat_dd")) <= TOL
    assert rel_err(x, o.get("x_dd")) <= TOL
    assert op.diagonal_gram
    P = fe_inputs(o).p_mat
    colsq = np.zeros(P.ncols)
    np.add.at(colsq, P.col_indices, P.values * P.values)
    assert np.array_equal(op.recovery_scale, 1.0 / colsq)
    print(f"{name}: H {e_h:.1e} g {e_g:.1e} (reference H vs DD {rel_err(g['H.values'], o.get('H.values_dd')):.1e})")


@pytest.mark.parametrize("name", [c for c in GOLDEN_CASES if "weighted" not in c])
def test_alg_condense_fe_inputs(name):
    g = load_golden(name)
    o = Oracle(g["dim"], g["cells"], g["k"])
    o.gen_inputs(g["coef"], g["seed"])
    o.run("port_condense")
    o.run("dd_condense")
    o.run("dd_recover_condensed")
    op, fs = ALG.static_condense(fe_inputs(o, marker=True))
    S = op.s_mat
    assert np.array_equal(S.row_offsets, g["S.row_offsets"]) and np.array_equal(S.col_indices, g["S.col_indices"])
    assert np.array_equal(op.master_globals, g["master_globals"])
    assert rel_err(S.values, o.get("S.values_dd")) <= TOL
    assert rel_err(fs, o.get("f_s_dd")) <= TOL
    if g["k"] == 0:  # S = P^T A_hat P: identical two-term sums
        assert np.array_equal(S.values, g["S.values"]) and np.array_equal(fs, g["f_s"])
    x = ALG.recover_condensed(op, o.get("x_b"), o.get("f_hat"))
    assert rel_err(x, o.get("x_cond_dd")) <= TOL


def test_alg_matches_fe_fast_path():
    o = Oracle(3, (3, 3, 2), 1)
    o.gen_inputs("logu:1e-2:1e2", 77)
    inp = fe_inputs(o)
    op, gv = ALG.hybridize(inp)
    sp = hd.Space(3, (3, 3, 2), 1)
    fe = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    hv, g2 = fe.values()
    assert rel_err(op.h_mat.values, hv) <= TOL and rel_err(gv, g2) <= TOL


# ---------------------------------------------------------------- general (non-FE) inputs, exact truth

def _rand_spd(rng, n):
    """Symmetric positive definite with small-integer entries (exact in binary and in Fraction)."""
    b = rng.integers(-3, 4, size=(n, n)).astype(float)
    return b @ b.T + n * np.eye(n)


def _frac_solve(A, B):
    n = len(A)
    M = [[Fraction(A[i][j]) for j in range(n)] + [Fraction(B[i][c]) for c in range(len(B[0]))] for i in range(n)]
    for j in range(n):
        p = next(i for i in range(j, n) if M[i][j] != 0)
        M[j], M[p] = M[p], M[j]
        for i in range(n):
            if i != j and M[i][j] != 0:
                f = M[i][j] / M[j][j]
                M[i] = [a - f * b for a, b in zip(M[i], M[j])]
    return [[M[i][n + c] / M[i][i] for c in range(len(B[0]))] for i in range(n)]


def _general_instance(seed, sizes=(4, 5, 3, 6), weighted=True):
    """Blocks + a general P (one dof duplicated with weights) + a C whose rows couple
    pairs of broken dofs with non-unit weights; f_hat random dyadic."""
    rng = np.random.default_rng(seed)
    blocks = [_rand_spd(rng, n) for n in sizes]
    n_hat = sum(sizes)
    off = np.cumsum([0] + list(sizes))
    # constrain the last two dofs of every block to the first dof of the next block
    trip = []
    r = 0
    for e in range(len(sizes) - 1):
        for t in range(2):
            a_dof, b_dof = off[e] + sizes[e] - 1 - t, off[e + 1] + t
            trip += [(r, a_dof, 1.0 if not weighted else 0.5 * (t + 1)), (r, b_dof, -1.0 if not weighted else -0.25)]
            r += 1
    m = r
    Cd = np.zeros((m, n_hat))
    for rr, c, v in trip:
        Cd[rr, c] += v
    C = Csr.from_dense(Cd)
    # P: injection, plus (weighted) the constrained broken dof 3 also mapped to global 1
    # with weight 0.5 (an interface dof: static_condense requires interior dofs to map 1:1)
    n_global = n_hat - 1
    Pd = np.zeros((n_hat, n_global))
    for i in range(n_hat):
        Pd[i, min(i, n_global - 1)] = 1.0 if i % 3 else -1.0
    if weighted:
        Pd[3, 1] = 0.5
    P = Csr.from_dense(Pd)
    f = rng.integers(-8, 9, size=n_hat) / 8.0
    return blocks, P, C, f, Cd, Pd


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_alg_hybridize_general_exact(seed):
    blocks, P, C, f, Cd, Pd = _general_instance(seed)
    op, g = ALG.hybridize(ReductionInputs(blocks, P, C, f))
    n_hat = len(f)
    A = np.zeros((n_hat, n_hat))
    o = 0
    for b in blocks:
        A[o:o + len(b), o:o + len(b)] = b
        o += len(b)
    X = _frac_solve(A.tolist(), np.hstack([Cd.T, f[:, None]]).tolist())
    m = Cd.shape[0]
    H = [[sum(Fraction(Cd[r][i]) * X[i][q] for i in range(n_hat)) for q in range(m)] for r in range(m)]
    gt = [sum(Fraction(Cd[r][i]) * X[i][m] for i in range(n_hat)) for r in range(m)]
    Hd = op.h_mat.to_dense()
    Ht = np.array([[float(v) for v in row] for row in H])
    assert rel_err(Hd, Ht) <= 1e-14
    assert rel_err(g, np.array([float(v) for v in gt])) <= 1e-14
    # pattern: exactly the couplings of the elements' multiplier rows (explicit zeros kept)
    assert op.h_mat.nrows == m
    # recovery through a non-injection P: CG on the Gram matrix
    lam = np.linspace(-1, 1, m)
    x_hat, x = ALG.recover_hybrid(op, lam, f)
    rhs = f - Cd.T @ lam
    xh_t = np.array([[float(v) for v in row] for row in _frac_solve(A.tolist(), rhs[:, None].tolist())])[:, 0]
    assert rel_err(x_hat, xh_t) <= 1e-13
    assert not op.diagonal_gram
    x_t = np.linalg.solve(Pd.T @ Pd, Pd.T @ xh_t)
    assert rel_err(x, x_t) <= 1e-10


@pytest.mark.parametrize("seed", [4, 5])
def test_alg_condense_general_exact(seed):
    blocks, P, C, f, Cd, Pd = _general_instance(seed, weighted=True)
    op, fs = ALG.static_condense(ReductionInputs(blocks, P, C, f))
    # truth: algebraic partition (zero columns of C), Schur per block, S = sum P_b^T S_hat P_b
    used = np.abs(Cd).sum(axis=0) != 0
    n_global = Pd.shape[1]
    masters = sorted({int(c) for i in np.nonzero(used)[0] for c in np.nonzero(Pd[i])[0]})
    ordn = {g: k for k, g in enumerate(masters)}
    nm = len(masters)
    S = [[Fraction(0)] * nm for _ in range(nm)]
    fst = [Fraction(0)] * nm
    o = 0
    for blk in blocks:
        n = len(blk)
        loc = np.arange(o, o + n)
        b = [l for l in range(n) if used[o + l]]
        i = [l for l in range(n) if not used[o + l]]
        Abb = [[Fraction(blk[p][q]) for q in b] for p in b]
        fb = [Fraction(f[o + p]) for p in b]
        if i:
            X = _frac_solve([[blk[p][q] for q in i] for p in i],
                            [[blk[p][q] for q in b] + [f[o + p]] for p in i])
            for jj, p in enumerate(b):
                for kk in range(len(b)):
                    Abb[jj][kk] -= sum(Fraction(blk[p][i[ll]]) * X[ll][kk] for ll in range(len(i)))
                fb[jj] -= sum(Fraction(blk[p][i[ll]]) * X[ll][len(b)] for ll in range(len(i)))
        for jj, p in enumerate(b):
            for gi in np.nonzero(Pd[o + p])[0]:
                wi = Fraction(Pd[o + p][gi])
                fst[ordn[int(gi)]] += wi * fb[jj]
                for kk, q in enumerate(b):
                    for gj in np.nonzero(Pd[o + q])[0]:
                        S[ordn[int(gi)]][ordn[int(gj)]] += wi * Fraction(Pd[o + q][gj]) * Abb[jj][kk]
        o += n
        del loc
    assert np.array_equal(op.master_globals, np.array(masters))
    St = np.array([[float(v) for v in row] for row in S])
    Sd = op.s_mat.to_dense()
    assert rel_err(Sd, St) <= 1e-14
    assert rel_err(fs, np.array([float(v) for v in fst])) <= 1e-14
    assert op.n_global == n_global


def test_alg_errors():
    blocks, P, C, f, Cd, Pd = _general_instance(9, weighted=False)
    with pytest.raises(hd.DimensionMismatch):
        ALG.hybridize(ReductionInputs(blocks, P, C, f[:-1]))
    with pytest.raises(hd.DimensionMismatch):
        ALG.static_condense(ReductionInputs(blocks, P, C, f[:-1]))
    bad = [b.copy() for b in blocks]
    bad[2][:] = 0.0  # singular block
    with pytest.raises(hd.SingularBlockError):
        ALG.hybridize(ReductionInputs(bad, P, C, f))
    # P with an empty column
    Pz = Pd.copy()
    Pz[:, 3] = 0.0
    with pytest.raises(hd.ValidationError):
        ALG.hybridize(ReductionInputs(blocks, Csr.from_dense(Pz), C, f))
    # interior dof mapped to two globals (static_condense's one-to-one check)
    Pw = Pd.copy()
    Pw[1, 0] = 0.5  # dof 1 is unconstrained in block 0
    with pytest.raises(hd.ValidationError):
        ALG.static_condense(ReductionInputs(blocks, Csr.from_dense(Pw), C, f))
    op, _ = ALG.hybridize(ReductionInputs(blocks, P, C, f))
    with pytest.raises(hd.DimensionMismatch):
        ALG.recover_hybrid(op, np.zeros(op.h_mat.nrows + 1), f)


def test_alg_no_constraints():
    """m = 0: empty H, recovery is the block solve (unit_reduction.cpp:245-276 edge case)."""
    rng = np.random.default_rng(3)
    blocks = [_rand_spd(rng, 3), _rand_spd(rng, 2)]
    n_hat = 5
    P = Csr.from_dense(np.eye(n_hat))
    C = Csr(0, n_hat, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    f = np.arange(n_hat, dtype=float)
    op, g = ALG.hybridize(ReductionInputs(blocks, P, C, f))
    assert op.h_mat.nrows == 0 and g.size == 0
    x_hat, x = ALG.recover_hybrid(op, np.zeros(0), f)
    A = np.zeros((5, 5))
    A[:3, :3], A[3:, 3:] = blocks
    assert rel_err(x_hat, np.linalg.solve(A, f)) <= 1e-14

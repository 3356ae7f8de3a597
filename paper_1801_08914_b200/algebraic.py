"""Algebraic batch path: the reference's ReductionInputs-level API on the B200.

Mirrors include/hdivred/reduction.hpp of the reference:

    ReductionInputs                       reduction.hpp:16-33
    hybridize(inputs) -> (op, g)          reduction.hpp:70      (src/reduction.cpp:262-354)
    recover_hybrid(op, lambda, f_hat)     reduction.hpp:73-75   (src/reduction.cpp:356-446)
    static_condense(inputs) -> (op, f_s)  reduction.hpp:97      (src/reduction.cpp:448-557)
    recover_condensed(op, x_b, f_hat)     reduction.hpp:101-102 (src/reduction.cpp:559-587)

Element blocks are arbitrary square dense matrices (ElementBlockOperator,
block_operator.hpp:22-38); P and C are CSR (CsrMatrix, csr.hpp:13-42).  All
arithmetic runs in libhdivred_b200.so's kernels (kern_alg.cu); this module only
packs arrays.  Errors map to the same exceptions as the FE path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi
from . import _check, _lib, _pcg_call


@dataclass
class Csr:
    """CsrMatrix (csr.hpp:13-42): int64 row_offsets (nrows+1), int64 col_indices, float64 values."""
    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self.nrows, self.ncols))
        for r in range(self.nrows):
            for k in range(self.row_offsets[r], self.row_offsets[r + 1]):
                a[r, self.col_indices[k]] += self.values[k]
        return a

    @staticmethod
    def from_dense(a: np.ndarray, keep_zeros: bool = False) -> "Csr":
        a = np.asarray(a, dtype=np.float64)
        ro, ci, v = [0], [], []
        for r in range(a.shape[0]):
            for c in range(a.shape[1]):
                if keep_zeros or a[r, c] != 0.0:
                    ci.append(c)
                    v.append(a[r, c])
            ro.append(len(ci))
        return Csr(a.shape[0], a.shape[1], np.array(ro), np.array(ci, dtype=np.int64), np.array(v))


@dataclass
class ReductionInputs:
    """The algebraic bundle (reduction.hpp:16-33).

    blocks: list of square float64 matrices (ElementBlockOperator blocks, block
    order = broken order); dof_global: optional n_hat int64 (dof_map[].global),
    needed when interior_global_begin >= 0."""
    blocks: Sequence[np.ndarray]
    p_mat: Csr
    c_mat: Csr
    f_hat: np.ndarray
    interior_global_begin: int = -1
    dof_global: Optional[np.ndarray] = None
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n_hat(self) -> int:
        return int(sum(np.shape(b)[0] for b in self.blocks))

    def _struct(self) -> _capi.AlgInputs:
        sizes = np.array([np.shape(b)[0] for b in self.blocks], dtype=np.int64)
        for b in self.blocks:
            if np.ndim(b) != 2 or np.shape(b)[0] != np.shape(b)[1]:
                raise ValueError("element blocks must be square matrices")
        flat = (np.concatenate([np.ascontiguousarray(b, dtype=np.float64).ravel() for b in self.blocks])
                if len(self.blocks) else np.zeros(1))
        f = np.ascontiguousarray(self.f_hat, dtype=np.float64)
        dg = None if self.dof_global is None else np.ascontiguousarray(self.dof_global, dtype=np.int64)
        self._keep = [sizes, flat, f, dg, self.p_mat, self.c_mat]
        s = _capi.AlgInputs()
        s.nblocks = len(self.blocks)
        s.block_sizes = sizes.ctypes.data
        s.blocks = flat.ctypes.data
        s.dof_global = dg.ctypes.data if dg is not None else None
        for pre, m in (("p", self.p_mat), ("c", self.c_mat)):
            setattr(s, f"{pre}_nrows", m.nrows)
            setattr(s, f"{pre}_ncols", m.ncols)
            setattr(s, f"{pre}_row_offsets", m.row_offsets.ctypes.data)
            setattr(s, f"{pre}_col_indices", m.col_indices.ctypes.data if m.col_indices.size else None)
            setattr(s, f"{pre}_values", m.values.ctypes.data if m.values.size else None)
        s.f_len = f.size
        s.f_hat = f.ctypes.data if f.size else None
        s.interior_global_begin = int(self.interior_global_begin)
        return s


class _AlgOperator:
    def __init__(self, handle):
        self._h = handle
        info = np.zeros(len(_capi.ALG_INFO_NAMES), dtype=np.int64)
        _check(_lib().hdr_alg_info(handle, info.ctypes.data))
        self.info = dict(zip(_capi.ALG_INFO_NAMES, (int(v) for v in info)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib().hdr_alg_destroy(h)
            self._h = None

    def pcg(self, b=None, rtol: float = 1e-10, maxit: int = 1000, precond: Optional[str] = "jacobi"):
        """Solve the reduced system (h_mat / s_mat, default rhs g / f_s) on the device: (x, report)."""
        return _pcg_call(_lib().hdr_alg_pcg, self._h, self.info["nrows"], b, rtol, maxit, precond)

    def _matrix(self):
        n, nnz = self.info["nrows"], self.info["nnz"]
        ro = np.empty(n + 1, dtype=np.int64)
        ci = np.empty(nnz, dtype=np.int64)
        v = np.empty(nnz)
        rhs = np.empty(n)
        _check(_lib().hdr_alg_matrix(self._h, ro.ctypes.data, ci.ctypes.data, v.ctypes.data, rhs.ctypes.data))
        return Csr(n, n, ro, ci, v), rhs


class HybridizedOperator(_AlgOperator):
    """HybridizedOperator (reduction.hpp:49-68): h_mat, recovery_scale, diagonal_gram;
    the per-element factorization state stays on the device."""

    def __init__(self, handle, symmetric: bool = False):
        super().__init__(handle)
        if symmetric:
            _check(_lib().hdr_alg_symmetrize(handle))
        self.h_mat, self._g = self._matrix()
        self.diagonal_gram = bool(self.info["diagonal_gram"])
        self.recovery_scale = np.empty(self.info["n_global"])
        _check(_lib().hdr_alg_recovery_scale(self._h, self.recovery_scale.ctypes.data))


class CondensedOperator(_AlgOperator):
    """CondensedOperator (reduction.hpp:78-95): s_mat, master_globals, n_global."""

    def __init__(self, handle, symmetric: bool = False):
        super().__init__(handle)
        if symmetric:
            _check(_lib().hdr_alg_symmetrize(handle))
        self.s_mat, self._f_s = self._matrix()
        self.master_globals = np.empty(self.info["nrows"], dtype=np.int64)
        _check(_lib().hdr_alg_master_globals(self._h, self.master_globals.ctypes.data))
        self.n_global = self.info["n_global"]


def hybridize(inputs: ReductionInputs, symmetric: bool = False):
    """hybridize(const ReductionInputs&) -> (HybridizedOperator, g).

    symmetric=True applies the reference's symmetrize to h_mat (exactly symmetric
    output, as its pcg requires); the default is the element-exact value."""
    s = inputs._struct()
    h = ctypes.c_void_p()
    _check(_lib().hdr_alg_hybridize(ctypes.byref(s), ctypes.byref(h)))
    op = HybridizedOperator(h.value, symmetric)
    return op, op._g


def static_condense(inputs: ReductionInputs, symmetric: bool = False):
    """static_condense(const ReductionInputs&) -> (CondensedOperator, f_s)."""
    s = inputs._struct()
    h = ctypes.c_void_p()
    _check(_lib().hdr_alg_static_condense(ctypes.byref(s), ctypes.byref(h)))
    op = CondensedOperator(h.value, symmetric)
    return op, op._f_s


def recover_hybrid(op: HybridizedOperator, lam, f_hat):
    """recover_hybrid(op, lambda, f_hat) -> (x_hat, x)."""
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    f = np.ascontiguousarray(f_hat, dtype=np.float64)
    x_hat = np.empty(op.info["n_hat"])
    x = np.empty(op.info["n_global"])
    _check(_lib().hdr_alg_recover_hybrid(op._h, lam.ctypes.data, lam.size, f.ctypes.data, f.size,
                                         x_hat.ctypes.data, x.ctypes.data))
    return x_hat, x


def recover_condensed(op: CondensedOperator, x_b, f_hat):
    """recover_condensed(op, x_b, f_hat) -> x (full global solution)."""
    xb = np.ascontiguousarray(x_b, dtype=np.float64)
    f = np.ascontiguousarray(f_hat, dtype=np.float64)
    x = np.empty(op.info["n_global"])
    _check(_lib().hdr_alg_recover_condensed(op._h, xb.ctypes.data, xb.size, f.ctypes.data, f.size, x.ctypes.data))
    return x


# ------------------------------------------------------------------ FE inputs and essential boundaries

def _face_geometry(space):
    """Per face: (axis, minus cell or -1, plus cell or -1), in the mesh's face order
    (src/mesh.cpp:75-120: faces grouped by axis, lexicographic, x fastest)."""
    dim = space.dim
    N = list(space.cells) + [1] * (3 - len(space.cells))
    axes, cms, cps = [], [], []
    for a in range(dim):
        d = [N[b] + (1 if b == a else 0) for b in range(3)]
        idx = np.arange(d[0] * d[1] * d[2])
        co = [idx % d[0], (idx // d[0]) % d[1], idx // (d[0] * d[1])]
        plane = co[a]
        cell = lambda c: c[0] + N[0] * (c[1] + N[1] * c[2])  # noqa: E731
        cm = np.where(plane > 0, cell([co[b] - (1 if b == a else 0) for b in range(3)]), -1)
        cp = np.where(plane < N[a], cell(co), -1)
        axes.append(np.full(idx.size, a))
        cms.append(cm)
        cps.append(cp)
    return np.concatenate(axes), np.concatenate(cms), np.concatenate(cps)


def fe_reduction_inputs(space, alpha, beta, f_hat) -> ReductionInputs:
    """build_reduction_inputs (src/reduction.cpp:200-222) of an FE space: the element
    blocks A_T (assembled on the device, bit-identical to element_matrices), P from
    the signed dof map (build_P, :136-150), C (build_C, :152-198: unit rows, or face
    moment rows for weighted spaces), interior_global_begin = face dof count."""
    n, nc = space.n, space.ncells
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    blocks = np.empty(nc * n * n)
    _check(_lib().hdr_space_element_blocks(space._h, a.ctypes.data, b.ctypes.data, 0, blocks.ctypes.data))
    blocks = blocks.reshape(nc, n, n)
    gl, sg = space.dof_map()
    nb = space.broken_ndofs
    p_mat = Csr(nb, space.ndofs, np.arange(nb + 1), gl, sg)
    dpf, nint, dim = space.info["dofs_per_face"], space.info["interior_dofs_per_cell"], space.dim
    axis, cm, cp = _face_geometry(space)
    interior = (cm >= 0) & (cp >= 0)
    faces = np.nonzero(interior)[0]
    m = faces.size * dpf
    if space.weighted:
        fm = np.empty(2 * dim * dpf * n)
        hh = (ctypes.c_double * 3)(*space.sizes)
        _check(_lib().hdr_reference_element(dim, space.order, hh, None, None, fm.ctypes.data, None))
        fm = fm.reshape(2 * dim, dpf, n)
    ro, ci, cv = [0], [], []
    for f in faces:
        ax = int(axis[f])
        lm, lp = nint + (2 * ax + 1) * dpf, nint + 2 * ax * dpf
        om, op = int(cm[f]) * n, int(cp[f]) * n
        for r in range(dpf):
            if not space.weighted:
                ci += [om + lm + r, op + lp + r]
                cv += [1.0, 1.0]
            else:
                ci += [om + lm + s_ for s_ in range(dpf)] + [op + lp + s_ for s_ in range(dpf)]
                cv += [fm[2 * ax + 1, r, lm + s_] for s_ in range(dpf)] + [fm[2 * ax, r, lp + s_] for s_ in range(dpf)]
            ro.append(len(ci))
    c_mat = Csr(m, nb, np.array(ro), np.array(ci, dtype=np.int64), np.array(cv))
    return ReductionInputs(list(blocks), p_mat, c_mat, np.ascontiguousarray(f_hat, dtype=np.float64),
                           interior_global_begin=space.info["face_dof_count"], dof_global=gl)


@dataclass
class EssentialBc:
    """EssentialBc (include/hdivred/reduction.hpp:104-107)."""
    face: int
    normal_flux: float = 0.0


@dataclass
class EliminationResult:
    """EliminationResult (reduction.hpp:109-113)."""
    inputs: ReductionInputs
    kept_globals: np.ndarray
    prescribed: np.ndarray


def eliminate_essential(space, inputs: ReductionInputs, bcs) -> EliminationResult:
    """eliminate_essential (src/reduction.cpp:589-698): removes the face dofs of
    the listed boundary faces from every block, moves their prescribed values
    (normal flux on sub-dof 0, 0 on the others) to the right-hand side
    (f_keep -= A[keep, drop] x_drop, in the reference's order), renumbers the
    globals, keeps C's rows (eliminated dofs are boundary dofs, so C never
    touches them).  Host bookkeeping; the reduced blocks then go through the
    device's general element path (kern_alg.cu)."""
    n = inputs.p_mat.ncols
    dpf = space.info["dofs_per_face"]
    _, cm, cp = _face_geometry(space)
    elim = np.zeros(n, dtype=bool)
    prescribed = np.zeros(n)
    for bc in bcs:
        if bc.face < 0 or bc.face >= space.info["nfaces"]:
            raise ValueError("eliminate_essential: face index out of range")
        if cm[bc.face] >= 0 and cp[bc.face] >= 0:
            raise ValueError(f"eliminate_essential: face {bc.face} is not on the boundary")
        for sub in range(dpf):
            g = bc.face * dpf + sub
            if elim[g]:
                raise ValueError(f"eliminate_essential: face {bc.face} listed twice")
            elim[g] = True
            prescribed[g] = bc.normal_flux if sub == 0 else 0.0
    kept = np.nonzero(~elim)[0]
    new_global = np.full(n, -1, dtype=np.int64)
    new_global[kept] = np.arange(kept.size)
    gl = inputs.dof_global if inputs.dof_global is not None else inputs.p_mat.col_indices
    sg = inputs.p_mat.values
    blocks, dof_global, signs, f_new, broken_keep = [], [], [], [], []
    off = 0
    for blk in inputs.blocks:
        nel = np.shape(blk)[0]
        g_e, s_e = gl[off:off + nel], sg[off:off + nel]
        drop_mask = elim[g_e]
        keep = np.nonzero(~drop_mask)[0]
        drop = np.nonzero(drop_mask)[0]
        A = np.asarray(blk)
        blocks.append(np.ascontiguousarray(A[np.ix_(keep, keep)]))
        dof_global.append(new_global[g_e[keep]])
        signs.append(s_e[keep])
        broken_keep.append(off + keep)
        for i in keep:  # v -= A[keep_i, l] * (sign_l * prescribed[global_l]), l in drop order
            v = float(inputs.f_hat[off + i])
            for l in drop:
                v -= A[i, l] * (s_e[l] * prescribed[g_e[l]])
            f_new.append(v)
        off += nel
    dof_global = np.concatenate(dof_global) if dof_global else np.zeros(0, np.int64)
    signs = np.concatenate(signs) if signs else np.zeros(0)
    broken_keep = np.concatenate(broken_keep) if broken_keep else np.zeros(0, np.int64)
    nb = broken_keep.size
    p_mat = Csr(nb, kept.size, np.arange(nb + 1), dof_global, signs)
    new_broken = np.full(inputs.p_mat.nrows, -1, dtype=np.int64)
    new_broken[broken_keep] = np.arange(nb)
    c = inputs.c_mat
    cols = new_broken[c.col_indices]
    if np.any(cols < 0):
        raise ValueError("eliminate_essential: constraint touches an eliminated dof")
    c_mat = Csr(c.nrows, nb, c.row_offsets.copy(), cols, c.values.copy())  # column order preserved (monotone map)
    igb = inputs.interior_global_begin
    if igb >= 0:
        igb = igb - int(np.count_nonzero(elim[:igb]))
    red = ReductionInputs(blocks, p_mat, c_mat, np.array(f_new), interior_global_begin=igb, dof_global=dof_global)
    return EliminationResult(red, kept, prescribed)


def expand_eliminated(elim: EliminationResult, reduced, full_n: int) -> np.ndarray:
    """expand_eliminated (src/reduction.cpp:700-709)."""
    reduced = np.asarray(reduced, dtype=np.float64)
    if reduced.size != elim.kept_globals.size:
        raise ValueError("expand_eliminated: reduced solution length")
    full = np.zeros(full_n)
    full[:elim.prescribed.size] = elim.prescribed[:full_n]
    full[elim.kept_globals] = reduced
    return full


__all__ = ["Csr", "ReductionInputs", "HybridizedOperator", "CondensedOperator", "hybridize", "static_condense",
           "recover_hybrid", "recover_condensed", "fe_reduction_inputs", "EssentialBc", "EliminationResult",
           "eliminate_essential", "expand_eliminated"]

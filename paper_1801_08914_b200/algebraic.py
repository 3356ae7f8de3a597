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


__all__ = ["Csr", "ReductionInputs", "HybridizedOperator", "CondensedOperator", "hybridize", "static_condense",
           "recover_hybrid", "recover_condensed"]

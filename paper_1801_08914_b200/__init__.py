"""B200-native element-local hybridization / static condensation for RT_k H(div)
systems (arXiv 1801.08914), a drop-in for the reference toolkit ``hdivred``'s
hot path.

Host-side mirror of the reference interfaces for this path:

* ``hybridized_matrix(config)`` / ``space_info(dim, cells, order)`` and the
  exception names mirror the pybind11 module ``hdivred._core``
  (bindings/module.cpp:75-174 of the reference);
* ``Space`` / ``HybridizedOperator`` / ``CondensedOperator`` mirror
  ``build_space`` + ``hybridize`` / ``recover_hybrid`` / ``static_condense`` /
  ``recover_condensed`` / ``spmv`` (include/hdivred/reduction.hpp,
  include/hdivred/csr.hpp) as far as the FE fast path goes.

All compute goes through the C ABI of ``libhdivred_b200.so`` (hand-written
sm_100a CUDA); there is no CPU fallback.  Arrays may be numpy (host) or torch
CUDA tensors (device resident, float64, contiguous).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _capi

__version__ = "0.1.0"


class HdivredError(RuntimeError):
    pass


class SingularBlockError(HdivredError):
    """hdivred::SingularBlock (include/hdivred/errors.hpp:15)."""


class CapExceededError(HdivredError):
    """hdivred::CapExceeded (include/hdivred/errors.hpp:20)."""


class FormatError(HdivredError):
    """hdivred::FormatError (include/hdivred/errors.hpp:25)."""


class ValidationError(HdivredError):
    """hdivred::ValidationError (include/hdivred/errors.hpp:44)."""


class SetupFailed(HdivredError):
    """hdivred::SetupFailed (include/hdivred/errors.hpp:39): AMG setup."""


class DimensionMismatch(HdivredError):
    """hdivred::DimensionMismatch (include/hdivred/errors.hpp:9)."""


class UnsupportedError(HdivredError):
    """Input outside what the device path implements (never silently ignored)."""


class DeviceError(HdivredError):
    """CUDA failure or no device (the hot path has no CPU fallback)."""


_STATUS_EXC = {
    _capi.SINGULAR_BLOCK: SingularBlockError,
    _capi.DIMENSION_MISMATCH: DimensionMismatch,
    _capi.VALIDATION: ValidationError,
    _capi.UNSUPPORTED: UnsupportedError,
    _capi.CUDA_ERROR: DeviceError,
    _capi.INVALID_ARGUMENT: ValueError,
    _capi.FORMAT_ERROR: FormatError,
    _capi.CAP_EXCEEDED: CapExceededError,
    _capi.SETUP_FAILED: SetupFailed,
}


def _check(status: int) -> None:
    if status != _capi.OK:
        raise _STATUS_EXC.get(status, HdivredError)(_capi.last_error())


def _lib():
    return _capi.load()


def _ptr(a) -> tuple[int, int]:
    """(address, on_device) of a float64/int64 numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data, 0
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr(), 1 if a.is_cuda else 0
    raise TypeError(f"unsupported array type {type(a)}")


def _as_f64(a, n: int, name: str):
    if isinstance(a, np.ndarray) or not hasattr(a, "data_ptr"):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.size != n:
            raise DimensionMismatch(f"{name}: expected {n} values, got {a.size}")
        return a
    import torch

    if a.dtype != torch.float64:
        raise TypeError(f"{name}: tensor must be float64")
    if a.numel() != n:
        raise DimensionMismatch(f"{name}: expected {n} values, got {a.numel()}")
    return a.contiguous()


def _same_device(arrays) -> int:
    flags = {_ptr(a)[1] for a in arrays}
    if len(flags) != 1:
        raise ValueError("inputs must be all host arrays or all CUDA tensors")
    return flags.pop()


class Space:
    """Structured mesh + RT_k space with its device-resident H/S patterns.

    Mirrors build_mesh + build_space (src/mesh.cpp:137, src/rt_space.cpp:318):
    ``cells`` per axis, ``sizes`` per axis (default 1/cells: unit cube),
    ``order`` k in 0..3.  ``ref_divdiv``/``ref_mass`` may be given to bind the
    reference element matrices of an existing RtSpace; by default the library's
    bit-exact restatement of build_reference builds them.
    """

    def __init__(self, dim: int, cells: Sequence[int], order: int, sizes: Optional[Sequence[float]] = None,
                 ref_divdiv=None, ref_mass=None, weighted: bool = False):
        cells = list(cells) + [1] * (3 - len(cells))
        if sizes is None:
            sizes = [1.0 / c if a < dim else 1.0 for a, c in enumerate(cells)]
        sizes = list(sizes) + [1.0] * (3 - len(sizes))
        carr = (ctypes.c_int64 * 3)(*[int(c) for c in cells[:3]])
        harr = (ctypes.c_double * 3)(*[float(s) for s in sizes[:3]])
        dd = mm = None
        if ref_divdiv is not None:
            dd = np.ascontiguousarray(ref_divdiv, dtype=np.float64)
            mm = np.ascontiguousarray(ref_mass, dtype=np.float64)
        h = ctypes.c_void_p()
        _check(_lib().hdr_space_create(dim, ctypes.addressof(carr), ctypes.addressof(harr), order,
                                       None if dd is None else dd.ctypes.data,
                                       None if mm is None else mm.ctypes.data, 1 if weighted else 0, None,
                                       ctypes.byref(h)))
        self._h = h
        info = np.zeros(len(_capi.INFO_NAMES), np.int64)
        _check(_lib().hdr_space_info(self._h, info.ctypes.data))
        self.info = {k: int(v) for k, v in zip(_capi.INFO_NAMES, info)}
        self.dim, self.order, self.weighted = dim, order, bool(weighted)
        self.cells = tuple(cells[:dim])
        self.sizes = tuple(sizes[:3])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _capi is not None and _capi._lib is not None:  # (not during interpreter teardown)
            _capi._lib.hdr_space_destroy(h)
            self._h = None

    # sizes
    @property
    def ncells(self) -> int:
        return self.info["ncells"]

    @property
    def n(self) -> int:
        return self.info["element_ndofs"]

    @property
    def m(self) -> int:
        return self.info["m"]

    @property
    def broken_ndofs(self) -> int:
        return self.info["broken_ndofs"]

    @property
    def ndofs(self) -> int:
        return self.info["ndofs"]

    def reference_matrices(self):
        n = self.n
        dd = np.empty(n * n)
        mm = np.empty(n * n)
        _check(_lib().hdr_space_reference(self._h, dd.ctypes.data, mm.ctypes.data))
        return dd.reshape(n, n), mm.reshape(n, n)

    def unit_load(self) -> np.ndarray:
        ul = np.empty(3 * self.n)
        _check(_lib().hdr_space_unit_load(self._h, ul.ctypes.data))
        return ul.reshape(3, self.n)

    def load_vector(self, g=(1.0, 1.0, 1.0)) -> np.ndarray:
        """FE load f_hat of build_reduction_inputs (rt_space.cpp:361-364), broken order."""
        ul = self.unit_load()
        load = np.zeros(self.n)
        for c in range(self.dim):
            load = load + g[c] * ul[c]
        return np.tile(load, self.ncells)

    def pattern(self, which: str = "H"):
        nr = self.m if which == "H" else self.info["n_s"]
        nz = self.info["nnz_h"] if which == "H" else self.info["nnz_s"]
        ro = np.empty(nr + 1, np.int64)
        ci = np.empty(nz, np.int64)
        _check(_lib().hdr_space_pattern(self._h, 0 if which == "H" else 1, ro.ctypes.data, ci.ctypes.data))
        return ro, ci

    def master_globals(self) -> np.ndarray:
        out = np.empty(self.info["n_s"], np.int64)
        _check(_lib().hdr_space_master_globals(self._h, out.ctypes.data))
        return out

    def dof_map(self):
        gl = np.empty(self.broken_ndofs, np.int64)
        sg = np.empty(self.broken_ndofs)
        _check(_lib().hdr_space_dof_map(self._h, gl.ctypes.data, sg.ctypes.data))
        return gl, sg

    def set_vertices(self, vertices) -> None:
        """Config 4: trilinear cells with these vertex coordinates ((N0+1)(N1+1)(N2+1) x 3,
        x fastest); None returns to the affine boxes."""
        if vertices is None:
            _check(_lib().hdr_space_set_vertices(self._h, None))
            self.vertices = None
            return
        nv = int(np.prod([c + 1 for c in self.cells[:3]]))
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1)
        if v.size != 3 * nv:
            raise DimensionMismatch(f"vertices: expected {3 * nv} values, got {v.size}")
        _check(_lib().hdr_space_set_vertices(self._h, v.ctypes.data))
        self.vertices = v

    def element_matrices(self) -> np.ndarray:
        """A_T of every cell from the last mapped-geometry call (ncells x n x n)."""
        out = np.empty(self.ncells * self.n * self.n)
        _check(_lib().hdr_space_element_matrices(self._h, out.ctypes.data))
        return out.reshape(self.ncells, self.n, self.n)

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """Run on a caller's CUDA stream handle (e.g. torch.cuda.Stream().cuda_stream).
        0 binds the legacy default stream; None restores the library's own stream."""
        if stream_ptr is None:
            _check(_lib().hdr_space_set_stream(self._h, None))
        else:
            _check(_lib().hdr_space_set_stream(self._h, ctypes.c_void_p(stream_ptr if stream_ptr else 1)))

    def synchronize(self) -> None:
        _check(_lib().hdr_space_synchronize(self._h))

    def set_exact_policy(self, force: bool = False, eps32: float = 0.0, eps_tc: float = 0.0, q_log=None) -> None:
        """Fail-safe controls of the structured solve (hdr_space_set_exact_policy):
        force=True sends every cell to the exact double-double path (testing);
        eps32 / eps_tc override the assumed correction accuracy (0: defaults);
        q_log: a CUDA float32 tensor (ncells) receiving each cell's measured
        first-order ratio q on later hybridize calls (None: off)."""
        qp = None
        if q_log is not None:
            if not getattr(q_log, "is_cuda", False) or str(q_log.dtype) != "torch.float32" or q_log.numel() < self.ncells:
                raise ValueError("q_log: CUDA float32 tensor of ncells entries")
            qp = q_log.data_ptr()
        _check(_lib().hdr_space_set_exact_policy(self._h, 1 if force else 0, float(eps32), float(eps_tc), qp))
        self._qlog = q_log

    def near_nullspace_check(self, alpha, beta, weighted: bool = False, dense_cap: int = 4_000_000) -> np.ndarray:
        """near_nullspace_check (src/reduction.cpp:711-742): ascending eigenvalues of
        C Y C^T, computed on the device in the reference's operation order."""
        a = _as_f64(alpha, self.ncells, "alpha")
        b = _as_f64(beta, self.ncells, "beta")
        dev = _same_device([a, b])
        out = np.empty(self.m)
        _check(_lib().hdr_near_nullspace_check(self._h, _ptr(a)[0], _ptr(b)[0], dev, 1 if weighted else 0,
                                               int(dense_cap), out.ctypes.data if self.m else None))
        return out

    # ---- hot path
    def hybridize(self, alpha, beta, f_hat) -> "HybridizedOperator":
        """hybridize (src/reduction.cpp:262-354) of the FE inputs (alpha, beta per cell, f_hat)."""
        a = _as_f64(alpha, self.ncells, "alpha")
        b = _as_f64(beta, self.ncells, "beta")
        f = _as_f64(f_hat, self.broken_ndofs, "f_hat")
        dev = _same_device([a, b, f])
        h = ctypes.c_void_p()
        _check(_lib().hdr_hybridize_fe(self._h, _ptr(a)[0], _ptr(b)[0], _ptr(f)[0], dev, ctypes.byref(h)))
        op = HybridizedOperator(self, h)
        op._keep = (a, b) if dev else None  # the C operator borrows device alpha / beta for recovery
        return op

    def hybridize_batch(self, alphas, betas, f_hats, h_outs=None, g_outs=None) -> None:
        """Pipelined batch of independent hybridizations (hdr_hybridize_fe_batch):
        item i's host inputs (alphas[i], betas[i], f_hats[i]; pinned for overlap)
        give H values / g in the host arrays h_outs[i] / g_outs[i] (None skips).
        Uploads, kernels and downloads of consecutive items overlap."""
        count = len(alphas)
        if len(betas) != count or len(f_hats) != count:
            raise DimensionMismatch("hybridize_batch: alphas, betas, f_hats differ in length")

        def ptrs(arrs, n, name, out=False):
            if arrs is None:
                return None
            if len(arrs) != count:
                raise DimensionMismatch(f"hybridize_batch: {name} has {len(arrs)} items, expected {count}")
            vals = []
            for a in arrs:
                if a is None:
                    vals.append(None)
                    continue
                if not out:
                    a = _as_f64(a, n, name)
                elif (a.size if isinstance(a, np.ndarray) else a.numel()) != n:
                    raise DimensionMismatch(f"{name}: expected {n} values")
                p_, dev = _ptr(a)
                if dev:
                    raise ValueError(f"{name}: hybridize_batch takes host arrays")
                vals.append(p_)
            return (ctypes.c_void_p * count)(*vals)

        keep = [ptrs(alphas, self.ncells, "alpha"), ptrs(betas, self.ncells, "beta"),
                ptrs(f_hats, self.broken_ndofs, "f_hat"), ptrs(h_outs, self.info["nnz_h"], "h_outs", True),
                ptrs(g_outs, self.m, "g_outs", True)]
        _check(_lib().hdr_hybridize_fe_batch(self._h, count, *keep))

    def static_condense(self, alpha, beta, f_hat) -> "CondensedOperator":
        """static_condense (src/reduction.cpp:448-557) of the FE inputs."""
        a = _as_f64(alpha, self.ncells, "alpha")
        b = _as_f64(beta, self.ncells, "beta")
        f = _as_f64(f_hat, self.broken_ndofs, "f_hat")
        dev = _same_device([a, b, f])
        h = ctypes.c_void_p()
        _check(_lib().hdr_static_condense_fe(self._h, _ptr(a)[0], _ptr(b)[0], _ptr(f)[0], dev, ctypes.byref(h)))
        op = CondensedOperator(self, h)
        op._keep = (a, b) if dev else None  # borrowed device alpha / beta (recover_condensed re-reads them)
        return op


class HybridizedOperator:
    """Device-resident HybridizedOperator (include/hdivred/reduction.hpp:49-68)."""

    def __init__(self, space: Space, handle):
        self.space = space
        self._h = handle
        self._keep = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _capi is not None and _capi._lib is not None:
            _capi._lib.hdr_hybrid_destroy(h)
            self._h = None

    def rehybridize(self, alpha, beta, f_hat) -> None:
        sp = self.space
        a = _as_f64(alpha, sp.ncells, "alpha")
        b = _as_f64(beta, sp.ncells, "beta")
        f = _as_f64(f_hat, sp.broken_ndofs, "f_hat")
        dev = _same_device([a, b, f])
        _check(_lib().hdr_hybridize_fe_into(self._h, _ptr(a)[0], _ptr(b)[0], _ptr(f)[0], dev))
        self._keep = (a, b) if dev else None

    def enqueue(self, alpha, beta, f_hat) -> None:
        """Asynchronous hybridize on the space's stream (no host sync); host
        inputs should be pinned.  Device errors surface in check()."""
        sp = self.space
        dev = _same_device([alpha, beta, f_hat])
        _check(_lib().hdr_hybridize_fe_enqueue(self._h, _ptr(alpha)[0], _ptr(beta)[0], _ptr(f_hat)[0], dev))
        self._keep = (alpha, beta) if dev else None

    def exact_cells(self) -> int:
        """Cells the last synchronous call solved on the exact double-double path
        (the structured solve's estimate rejected them; hdr_hybrid_exact_cells)."""
        n = ctypes.c_int64()
        _check(_lib().hdr_hybrid_exact_cells(self._h, ctypes.byref(n)))
        return int(n.value)

    def values_enqueue(self, h_out, g_out) -> None:
        """Asynchronous copy of H values / g into caller buffers (host pinned or device)."""
        dev = _same_device([h_out, g_out])
        _check(_lib().hdr_hybrid_values_enqueue(self._h, _ptr(h_out)[0], _ptr(g_out)[0], dev))

    def pcg(self, b=None, rtol: float = 1e-10, maxit: int = 1000, precond: Optional[str] = "jacobi"):
        """Solve H lambda = b (default b = g) on the device: (lambda, report), see hdr_hybrid_pcg."""
        return _pcg_call(_lib().hdr_hybrid_pcg, self._h, self.space.m, b, rtol, maxit, precond)

    def symmetrize(self) -> None:
        """In place H <- (H + H^T) / 2, the reference's symmetrize (reduction.cpp:316):
        exactly symmetric H for consumers such as its pcg (solvers.cpp:25-30)."""
        _check(_lib().hdr_hybrid_symmetrize(self._h))

    def check(self) -> None:
        _check(_lib().hdr_hybrid_check(self._h))

    def values(self):
        """(H values in pattern order, g) as host arrays."""
        hv = np.empty(self.space.info["nnz_h"])
        g = np.empty(self.space.m)
        _check(_lib().hdr_hybrid_values(self._h, hv.ctypes.data, g.ctypes.data, 0))
        return hv, g

    def h_mat(self):
        """CsrMatrix as the reference's csr_to_tuple: (nrows, ncols, row_offsets, col_indices, values)."""
        ro, ci = self.space.pattern("H")
        hv, _ = self.values()
        return self.space.m, self.space.m, ro, ci, hv

    def recover(self, lam, f_hat):
        """recover_hybrid (src/reduction.cpp:356-446): returns (x_hat, x)."""
        sp = self.space
        lam = _as_f64(lam, sp.m, "lambda")
        f = _as_f64(f_hat, sp.broken_ndofs, "f_hat")
        dev = _same_device([lam, f])
        if dev:
            import torch

            xh = torch.empty(sp.broken_ndofs, dtype=torch.float64, device=lam.device)
            x = torch.empty(sp.ndofs, dtype=torch.float64, device=lam.device)
        else:
            xh = np.empty(sp.broken_ndofs)
            x = np.empty(sp.ndofs)
        _check(_lib().hdr_recover_hybrid(self._h, _ptr(lam)[0], _ptr(f)[0], dev, _ptr(xh)[0], _ptr(x)[0]))
        return xh, x

    def spmv(self, x):
        """y = H x (spmv, src/csr.cpp:77-87)."""
        sp = self.space
        x = _as_f64(x, sp.m, "x")
        dev = _ptr(x)[1]
        if dev:
            import torch

            y = torch.empty(sp.m, dtype=torch.float64, device=x.device)
        else:
            y = np.empty(sp.m)
        _check(_lib().hdr_hybrid_spmv(self._h, _ptr(x)[0], _ptr(y)[0], dev))
        return y


class CondensedOperator:
    """Device-resident CondensedOperator (include/hdivred/reduction.hpp:78-95)."""

    def __init__(self, space: Space, handle):
        self.space = space
        self._h = handle
        self._keep = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _capi is not None and _capi._lib is not None:
            _capi._lib.hdr_condensed_destroy(h)
            self._h = None

    def values(self):
        sv = np.empty(self.space.info["nnz_s"])
        fs = np.empty(self.space.info["n_s"])
        _check(_lib().hdr_condensed_values(self._h, sv.ctypes.data, fs.ctypes.data, 0))
        return sv, fs

    def pcg(self, b=None, rtol: float = 1e-10, maxit: int = 1000, precond: Optional[str] = "jacobi"):
        """Solve S x_b = b (default b = f_s) on the device: (x_b, report)."""
        return _pcg_call(_lib().hdr_condensed_pcg, self._h, self.space.info["n_s"], b, rtol, maxit, precond)

    def s_mat(self):
        ro, ci = self.space.pattern("S")
        sv, _ = self.values()
        ns = self.space.info["n_s"]
        return ns, ns, ro, ci, sv

    def recover(self, x_b, f_hat):
        """recover_condensed (src/reduction.cpp:559-587): full global solution."""
        sp = self.space
        xb = _as_f64(x_b, sp.info["n_s"], "x_b")
        f = _as_f64(f_hat, sp.broken_ndofs, "f_hat")
        dev = _same_device([xb, f])
        if dev:
            import torch

            x = torch.empty(sp.ndofs, dtype=torch.float64, device=xb.device)
        else:
            x = np.empty(sp.ndofs)
        _check(_lib().hdr_recover_condensed(self._h, _ptr(xb)[0], _ptr(f)[0], dev, _ptr(x)[0]))
        return x

    def spmv(self, x):
        sp = self.space
        x = _as_f64(x, sp.info["n_s"], "x")
        dev = _ptr(x)[1]
        if dev:
            import torch

            y = torch.empty(sp.info["n_s"], dtype=torch.float64, device=x.device)
        else:
            y = np.empty(sp.info["n_s"])
        _check(_lib().hdr_condensed_spmv(self._h, _ptr(x)[0], _ptr(y)[0], dev))
        return y


# the reference's PrecondKind (include/hdivred/driver.hpp:15)
_PRECOND = {None: 0, "none": 0, "jacobi": 1, "sgs": 2, "amg": 3}


def _pcg_call(fn, handle, n, b, rtol, maxit, precond):
    """Shared driver of the device pcg entry points: returns (x, report)."""
    if precond not in _PRECOND:
        raise ValueError("precond must be None, 'none', 'jacobi', 'sgs' or 'amg'")
    hist = np.zeros(int(maxit) + 1)
    rep = _capi.PcgReport()
    if b is None:
        x = np.empty(n)
        _check(fn(handle, None, x.ctypes.data, 0, float(rtol), int(maxit), _PRECOND[precond], hist.ctypes.data,
                  ctypes.byref(rep)))
    else:
        bb = _as_f64(b, n, "b")
        dev = _ptr(bb)[1]
        if dev:
            import torch

            x = torch.empty(n, dtype=torch.float64, device=bb.device)
        else:
            x = np.empty(n)
        _check(fn(handle, _ptr(bb)[0], _ptr(x)[0], dev, float(rtol), int(maxit), _PRECOND[precond],
                  hist.ctypes.data, ctypes.byref(rep)))
    it = int(rep.iterations)
    report = {"iterations": it, "converged": bool(rep.converged), "relative_residuals": hist[: it + 1].tolist(),
              "final_relative_residual": float(rep.final_relative_residual), "wall_time": rep.wall_ms * 1e-3}
    return x, report


def pcg(a, b, rtol: float = 1e-10, maxit: int = 1000, precond: Optional[str] = "jacobi"):
    """pcg (src/solvers.cpp:109-163) on the device for a CSR tuple (nrows, ncols, row_offsets,
    col_indices, values): returns (x, report)."""
    nr, nc, ro, ci, v = a
    ro = np.ascontiguousarray(ro, np.int64)
    ci = np.ascontiguousarray(ci, np.int64)
    v = np.ascontiguousarray(v, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if nr != nc or b.size != nr:
        raise DimensionMismatch("pcg: matrix not square or rhs length")
    if precond not in _PRECOND:
        raise ValueError("precond must be None, 'none', 'jacobi', 'sgs' or 'amg'")
    x = np.empty(nr)
    hist = np.zeros(int(maxit) + 1)
    rep = _capi.PcgReport()
    _check(_lib().hdr_csr_pcg_host(nr, ro.ctypes.data, ci.ctypes.data, v.ctypes.data, b.ctypes.data, x.ctypes.data,
                                   float(rtol), int(maxit), _PRECOND[precond], hist.ctypes.data, ctypes.byref(rep)))
    it = int(rep.iterations)
    return x, {"iterations": it, "converged": bool(rep.converged), "relative_residuals": hist[: it + 1].tolist(),
               "final_relative_residual": float(rep.final_relative_residual), "wall_time": rep.wall_ms * 1e-3}


def _host_csr(a):
    nr, nc, ro, ci, v = a
    if nr != nc:
        raise DimensionMismatch("matrix not square")
    return (int(nr), np.ascontiguousarray(ro, np.int64), np.ascontiguousarray(ci, np.int64),
            np.ascontiguousarray(v, np.float64))


class AmgHierarchy:
    """amg_setup (src/amg.cpp:189-244) on the device: levels (A, P, R) bit-identical
    to the reference's for the same matrix; apply() is one V(1,1) cycle (amg_apply)."""

    def __init__(self, a, **options):
        n, ro, ci, v = _host_csr(a)
        o = _capi.AmgOptions()
        _lib().hdr_amg_default_options(ctypes.byref(o))
        for k_, val in options.items():
            setattr(o, k_, val)
        h = ctypes.c_void_p()
        _check(_lib().hdr_amg_setup(n, ro.ctypes.data, ci.ctypes.data, v.ctypes.data, 0, ctypes.byref(o),
                                    ctypes.byref(h)))
        self._h = h
        self.n = n
        lv = ctypes.c_int64()
        _check(_lib().hdr_amg_info(self._h, ctypes.byref(lv), None, None))
        self.nlevels = int(lv.value)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib().hdr_amg_destroy(self._h)
            self._h = None

    def matrix(self, level: int, which: str = "A"):
        """(nrows, ncols, row_offsets, col_indices, values) of a level's A / P / R
        (level == nlevels: the coarse matrix)."""
        w = {"A": 0, "P": 1, "R": 2}[which]
        dims = np.zeros(3, np.int64)
        _check(_lib().hdr_amg_level_matrix(self._h, level, w, dims.ctypes.data, None, None, None))
        ro = np.empty(dims[0] + 1, np.int64)
        ci = np.empty(dims[2], np.int64)
        v = np.empty(dims[2])
        _check(_lib().hdr_amg_level_matrix(self._h, level, w, dims.ctypes.data, ro.ctypes.data,
                                           ci.ctypes.data if dims[2] else None, v.ctypes.data if dims[2] else None))
        return int(dims[0]), int(dims[1]), ro, ci, v

    def apply(self, r) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        if r.size != self.n:
            raise DimensionMismatch("amg_apply: vector length")
        z = np.empty(self.n)
        _check(_lib().hdr_amg_apply(self._h, r.ctypes.data, z.ctypes.data, 0))
        return z


def precond_apply(a, r, kind: str = "sgs") -> np.ndarray:
    """One application of the jacobi / sgs preconditioner of a host CSR matrix
    (jacobi_setup / ssgs_setup, src/solvers.cpp:46-72), on the device."""
    n, ro, ci, v = _host_csr(a)
    r = np.ascontiguousarray(r, np.float64)
    z = np.empty(n)
    _check(_lib().hdr_csr_precond_apply_host(n, ro.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                             {"jacobi": 1, "sgs": 2}[kind], r.ctypes.data, z.ctypes.data))
    return z


# ------------------------------------------------------------------ reference-mirroring front-end

def _axes(v, dim, default):
    if v is None:
        return list(default)
    if isinstance(v, (list, tuple)):
        out = list(default)
        for a in range(min(3, len(v))):
            out[a] = v[a]
        return out
    return [v, v, v]


def coefficients_from_config(config: dict, space: Space):
    """Per-cell (alpha, beta) as the reference's build_problem (src/driver.cpp:166-197):
    uniform alpha/beta, the soft-hard preset (src/mesh.cpp:168-191) or a coefficient file
    (src/mesh.cpp:193-221)."""
    nc = space.ncells
    preset = config.get("coeff_preset", "")
    if preset == "soft-hard":
        p = int(config.get("p", 0))
        jump = math.pow(10.0, p)
        alpha = np.ones(nc)
        beta = np.ones(nc)
        n0, n1, n2 = (list(space.cells) + [1, 1])[:3]
        h = space.sizes
        idx = np.arange(nc)
        co = [idx % n0, (idx // n0) % n1, idx // (n0 * n1)]
        in_lo = np.ones(nc, bool)
        in_hi = np.ones(nc, bool)
        for a in range(space.dim):
            t = 0.0 + (co[a].astype(np.float64) + 0.5) * h[a]
            in_lo &= (t >= 0.25) & (t <= 0.5)
            in_hi &= (t >= 0.5) & (t <= 0.75)
        beta[in_lo | in_hi] = jump
        return alpha, beta
    if preset:
        raise ValueError(f"unknown coefficient preset '{preset}'")
    if config.get("coeff_file"):
        alpha = np.empty(nc)
        beta = np.empty(nc)
        expected = 0
        with open(config["coeff_file"]) as fh:
            for line_no, line in enumerate(fh, 1):
                if not line.strip() or line.startswith("#"):
                    continue
                parts = line.split()
                if len(parts) < 3:
                    raise FormatError(f"bad coefficient line (line {line_no})")
                cell, a, b = int(parts[0]), float(parts[1]), float(parts[2])
                if cell != expected:
                    raise FormatError(f"coefficient lines must be in lexicographic cell order (line {line_no})")
                if not (a > 0 and b > 0 and math.isfinite(a) and math.isfinite(b)):
                    raise FormatError(f"coefficients must be positive and finite (line {line_no})")
                alpha[cell], beta[cell] = a, b
                expected += 1
        if expected != nc:
            raise FormatError(f"coefficient file has {expected} cells, mesh has {nc}")
        return alpha, beta
    a = float(config.get("alpha", 1.0))
    b = float(config.get("beta", 1.0))
    if not (a > 0 and b > 0):
        raise ValueError("coefficients must be positive")
    return np.full(nc, a), np.full(nc, b)


def space_from_config(config: dict) -> Space:
    dim = int(config.get("dim", 3))
    cells = [int(c) for c in _axes(config.get("cells"), dim, [8, 8, 8])]
    sizes = [float(s) for s in _axes(config.get("sizes"), dim, [0.0, 0.0, 0.0])]
    for a in range(dim):
        if sizes[a] == 0.0:
            sizes[a] = 1.0 / cells[a]
    if dim == 2:
        cells[2], sizes[2] = 1, 1.0
    return Space(dim, cells[:dim], int(config.get("order", 0)), sizes, weighted=bool(config.get("weighted", False)))


def hybridized_matrix(config: dict):
    """Mirror of hdivred._core.hybridized_matrix (bindings/module.cpp:163-171):
    ((nrows, ncols, row_offsets, col_indices, values), g) for the config's FE problem."""
    space = space_from_config(config)
    alpha, beta = coefficients_from_config(config, space)
    g = config.get("g", (1.0, 1.0, 1.0))
    g = _axes(g, 3, [1.0, 1.0, 1.0])
    f_hat = space.load_vector(g)
    if config.get("essential_boundary", False):
        # build_problem (src/driver.cpp:187-195): every boundary face eliminated with
        # zero normal flux, then hybridize(ReductionInputs) on the reduced blocks
        from . import algebraic as alg

        inputs = alg.fe_reduction_inputs(space, alpha, beta, f_hat)
        _, cm, cp = alg._face_geometry(space)
        bcs = [alg.EssentialBc(int(f), 0.0) for f in np.nonzero((cm < 0) | (cp < 0))[0]]
        red = alg.eliminate_essential(space, inputs, bcs).inputs
        aop, gv = alg.hybridize(red, symmetric=True)
        h = aop.h_mat
        return (h.nrows, h.ncols, list(h.row_offsets), list(h.col_indices), list(h.values)), list(gv)
    op = space.hybridize(alpha, beta, f_hat)
    op.symmetrize()  # the reference symmetrizes every element block (src/reduction.cpp:316)
    nr, nc, ro, ci, hv = op.h_mat()
    _, gv = op.values()
    return (nr, nc, list(ro), list(ci), list(hv)), list(gv)


def space_info(dim: int, cells: Sequence[int], order: int) -> dict:
    """Mirror of hdivred._core.space_info (bindings/module.cpp:83-101), computed
    from the mesh numbering alone (no device needed)."""
    cells = list(cells) + [1] * (3 - len(cells))
    n = cells[:dim]
    nfaces = 0
    for a in range(dim):
        c = n[a] + 1
        for b in range(dim):
            if b != a:
                c *= n[b]
        nfaces += c
    ncells = int(np.prod(n))
    dpf = (order + 1) ** (dim - 1)
    nint = dim * order * dpf
    ndofs = nfaces * dpf + ncells * nint
    return {"ncells": ncells, "nfaces": nfaces, "ndofs": ndofs, "broken_ndofs": ncells * (2 * dim * dpf + nint),
            "dofs_per_face": dpf, "interior_dofs_per_cell": nint}


def measure_fp64_peak() -> tuple[float, float]:
    """(TFLOP/s, ms) of the device's DFMA throughput (fp64 roofline denominator)."""
    t = ctypes.c_double()
    ms = ctypes.c_double()
    _check(_lib().hdr_measure_fp64_peak(ctypes.byref(t), ctypes.byref(ms)))
    return t.value, ms.value


def measure_dmma_peak() -> tuple[float, float]:
    """(TFLOP/s, ms) of the device's fp64 tensor-core (DMMA m8n8k4) throughput."""
    t = ctypes.c_double()
    ms = ctypes.c_double()
    _check(_lib().hdr_measure_dmma_peak(ctypes.byref(t), ctypes.byref(ms)))
    return t.value, ms.value


def launch_count() -> int:
    """Kernels this process launched through the library (bench.py gpu_launches)."""
    return int(_lib().hdr_launch_count())


from . import algebraic  # noqa: E402  (ReductionInputs-level API; needs _check/_lib above)
from . import io  # noqa: E402  (instance I/O, host threads)

__all__ = [
    "algebraic", "io", "AmgHierarchy", "precond_apply", "SetupFailed", "CapExceededError", "FormatError", "SingularBlockError", "ValidationError", "DimensionMismatch",
    "UnsupportedError", "DeviceError", "Space", "HybridizedOperator", "CondensedOperator", "hybridized_matrix",
    "space_info", "coefficients_from_config", "space_from_config", "launch_count", "pcg", "__version__",
]

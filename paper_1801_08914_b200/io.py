"""Instance I/O of the algebraic import path (reference: src/block_io.cpp,
src/matrix_market.cpp; hdivred import --prefix P, src/driver.cpp:372-380).

Host-side parallel readers / writers in libhdivred_b200.so (csrc/io.cpp): the
reference's text formats, values bit-identical on read, files byte-identical on
write.  No GPU is needed for these calls.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _capi
from . import _check, _lib
from .algebraic import Csr, ReductionInputs


def read_block_operator(path: str, threads: int = 0):
    """read_block_operator (block_io.cpp:41-94) -> (blocks list, dof_global, dof_sign, broken_dim, global_dim)."""
    h = ctypes.c_void_p()
    _check(_lib().hdr_io_read_block_operator(str(path).encode(), threads, ctypes.byref(h)))
    try:
        info = np.zeros(4, np.int64)
        _check(_lib().hdr_io_blocks_info(h, info.ctypes.data))
        nb, bd, gd, ne = (int(x) for x in info)
        sizes = np.empty(nb, np.int64)
        gl = np.empty(bd, np.int64)
        sg = np.empty(bd)
        ent = np.empty(ne)
        _check(_lib().hdr_io_blocks_get(h, sizes.ctypes.data, gl.ctypes.data, sg.ctypes.data, ent.ctypes.data))
    finally:
        _lib().hdr_io_blocks_destroy(h)
    blocks, o = [], 0
    for n in sizes:
        blocks.append(ent[o:o + n * n].reshape(n, n))
        o += n * n
    return blocks, gl, sg, bd, gd


def write_block_operator(path: str, blocks, dof_global, dof_sign, global_dim: int, threads: int = 0) -> None:
    """write_block_operator (block_io.cpp:15-39)."""
    sizes = np.array([np.shape(b)[0] for b in blocks], np.int64)
    ent = np.concatenate([np.ascontiguousarray(b, dtype=np.float64).ravel() for b in blocks]) if len(blocks) else np.zeros(1)
    gl = np.ascontiguousarray(dof_global, dtype=np.int64)
    sg = np.ascontiguousarray(dof_sign, dtype=np.float64)
    _check(_lib().hdr_io_write_block_operator(str(path).encode(), sizes.size, int(sizes.sum()), int(global_dim),
                                              sizes.ctypes.data, gl.ctypes.data, sg.ctypes.data, ent.ctypes.data,
                                              threads))


def _csr_from_handle(h) -> Csr:
    try:
        info = np.zeros(3, np.int64)
        _check(_lib().hdr_io_csr_info(h, info.ctypes.data))
        nr, nc, nz = (int(x) for x in info)
        ro = np.empty(nr + 1, np.int64)
        ci = np.empty(nz, np.int64)
        v = np.empty(nz)
        _check(_lib().hdr_io_csr_get(h, ro.ctypes.data, ci.ctypes.data, v.ctypes.data))
    finally:
        _lib().hdr_io_csr_destroy(h)
    return Csr(nr, nc, ro, ci, v)


def read_matrix_market(path: str, threads: int = 0) -> Csr:
    """read_matrix_market (matrix_market.cpp:55-97)."""
    h = ctypes.c_void_p()
    _check(_lib().hdr_io_read_matrix_market(str(path).encode(), threads, ctypes.byref(h)))
    return _csr_from_handle(h)


def write_matrix_market(path: str, a: Csr, threads: int = 0) -> None:
    """write_matrix_market (matrix_market.cpp:36-53)."""
    _check(_lib().hdr_io_write_matrix_market(str(path).encode(), a.nrows, a.ncols, a.row_offsets.ctypes.data,
                                             a.col_indices.ctypes.data if a.col_indices.size else None,
                                             a.values.ctypes.data if a.values.size else None, threads))


def read_vector_market(path: str, threads: int = 0) -> np.ndarray:
    """read_vector_market (matrix_market.cpp:112-122): an n x 1 coordinate matrix."""
    m = read_matrix_market(path, threads)
    if m.ncols != 1:
        raise _capi_format_error(f"expected an n-by-1 vector in '{path}'")
    v = np.zeros(m.nrows)
    for i in np.nonzero(np.diff(m.row_offsets))[0]:
        v[i] = m.values[m.row_offsets[i]]
    return v


def write_vector_market(path: str, v, threads: int = 0) -> None:
    """write_vector_market (matrix_market.cpp:99-110): zeros are not stored."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    nz = v != 0.0
    ro = np.concatenate([[0], np.cumsum(nz)]).astype(np.int64)
    write_matrix_market(path, Csr(v.size, 1, ro, np.zeros(int(nz.sum()), np.int64), v[nz]), threads)


def read_vector_lines(path: str, threads: int = 0) -> np.ndarray:
    """read_vector_lines (matrix_market.cpp:131-146)."""
    h = ctypes.c_void_p()
    _check(_lib().hdr_io_read_vector_lines(str(path).encode(), threads, ctypes.byref(h)))
    return _csr_from_handle(h).values


def write_vector_lines(path: str, v, threads: int = 0) -> None:
    """write_vector_lines (matrix_market.cpp:124-129)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    _check(_lib().hdr_io_write_vector_lines(str(path).encode(), v.size, v.ctypes.data if v.size else None, threads))


def import_instance(prefix: str, threads: int = 0) -> ReductionInputs:
    """import_instance (src/driver.cpp:372-380): PREFIX.blocks, .p.mtx, .c.mtx, .f.mtx ->
    ReductionInputs with interior_global_begin = -1 (unknown on the import path)."""
    blocks, gl, sg, bd, gd = read_block_operator(f"{prefix}.blocks", threads)
    p = read_matrix_market(f"{prefix}.p.mtx", threads)
    c = read_matrix_market(f"{prefix}.c.mtx", threads)
    f = read_vector_market(f"{prefix}.f.mtx", threads)
    return ReductionInputs(blocks, p, c, f, interior_global_begin=-1, dof_global=gl)


def _capi_format_error(msg):
    from . import FormatError

    return FormatError(msg)


__all__ = ["read_block_operator", "write_block_operator", "read_matrix_market", "write_matrix_market",
           "read_vector_market", "write_vector_market", "read_vector_lines", "write_vector_lines",
           "import_instance"]

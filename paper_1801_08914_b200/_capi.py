"""ctypes binding of the C ABI in include/hdivred_b200.h (libhdivred_b200.so).

The library is built in-tree (``make -C paper_1801_08914_b200/csrc`` or
``__graft_entry__.build()``).  Importing this module without it raises: the hot
path has no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

# HDR_LIB: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = Path(os.environ.get("HDR_LIB") or Path(__file__).resolve().parent / "libhdivred_b200.so")

# status codes (hdr_status)
(OK, SINGULAR_BLOCK, DIMENSION_MISMATCH, VALIDATION, UNSUPPORTED, CUDA_ERROR, INVALID_ARGUMENT, FORMAT_ERROR,
 CAP_EXCEEDED, SETUP_FAILED) = range(10)

# hdr_space_info indices
INFO_NAMES = ["dim", "order", "ncells", "nfaces", "ndofs", "broken_ndofs", "element_ndofs", "dofs_per_face",
              "interior_dofs_per_cell", "face_dof_count", "m", "nnz_h", "n_s", "nnz_s", "div_rank"]

_vp, _i32, _i64, _d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double

class PcgReport(ctypes.Structure):
    """hdr_pcg_report"""
    _fields_ = [("iterations", _i64), ("converged", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("final_relative_residual", _d), ("wall_ms", _d)]


class AmgOptions(ctypes.Structure):
    """hdr_amg_options (AmgOptions, include/hdivred/amg.hpp:12-19)"""
    _fields_ = [("strength_threshold", _d), ("omega_factor", _d), ("coarse_cap", _i64), ("max_levels", ctypes.c_int32),
                ("power_iterations", ctypes.c_int32), ("stall_ratio", _d)]


class AlgInputs(ctypes.Structure):
    """hdr_alg_inputs (include/hdivred_b200.h): a ReductionInputs as plain arrays."""
    _fields_ = [
        ("nblocks", _i64), ("block_sizes", _vp), ("blocks", _vp), ("dof_global", _vp),
        ("p_nrows", _i64), ("p_ncols", _i64), ("p_row_offsets", _vp), ("p_col_indices", _vp), ("p_values", _vp),
        ("c_nrows", _i64), ("c_ncols", _i64), ("c_row_offsets", _vp), ("c_col_indices", _vp), ("c_values", _vp),
        ("f_len", _i64), ("f_hat", _vp), ("interior_global_begin", _i64),
    ]


# hdr_alg_info indices
ALG_INFO_NAMES = ["nrows", "nnz", "n_hat", "n_global", "diagonal_gram", "kind"]

_SIGS = {
    "hdr_space_create": (_i32, [_i32, _vp, _vp, _i32, _vp, _vp, _i32, _vp, _vp]),
    "hdr_space_destroy": (None, [_vp]),
    "hdr_space_info": (_i32, [_vp, _vp]),
    "hdr_space_reference": (_i32, [_vp, _vp, _vp]),
    "hdr_space_unit_load": (_i32, [_vp, _vp]),
    "hdr_space_set_stream": (_i32, [_vp, _vp]),
    "hdr_space_pattern": (_i32, [_vp, _i32, _vp, _vp]),
    "hdr_space_master_globals": (_i32, [_vp, _vp]),
    "hdr_space_dof_map": (_i32, [_vp, _vp, _vp]),
    "hdr_space_element_blocks": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "hdr_space_synchronize": (_i32, [_vp]),
    "hdr_hybridize_fe": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp]),
    "hdr_hybridize_fe_into": (_i32, [_vp, _vp, _vp, _vp, _i32]),
    "hdr_hybridize_fe_enqueue": (_i32, [_vp, _vp, _vp, _vp, _i32]),
    "hdr_hybridize_fe_batch": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    "hdr_hybrid_check": (_i32, [_vp]),
    "hdr_hybrid_exact_cells": (_i32, [_vp, _vp]),
    "hdr_space_set_exact_policy": (_i32, [_vp, _i32, _d, _d, _vp]),
    "hdr_hybrid_values_enqueue": (_i32, [_vp, _vp, _vp, _i32]),
    "hdr_measure_fp64_peak": (_i32, [_vp, _vp]),
    "hdr_measure_dmma_peak": (_i32, [_vp, _vp]),
    "hdr_hybrid_destroy": (None, [_vp]),
    "hdr_hybrid_values": (_i32, [_vp, _vp, _vp, _i32]),
    "hdr_hybrid_device_ptrs": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "hdr_recover_hybrid": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp]),
    "hdr_static_condense_fe": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp]),
    "hdr_static_condense_fe_into": (_i32, [_vp, _vp, _vp, _vp, _i32]),
    "hdr_condensed_destroy": (None, [_vp]),
    "hdr_condensed_values": (_i32, [_vp, _vp, _vp, _i32]),
    "hdr_recover_condensed": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "hdr_hybrid_spmv": (_i32, [_vp, _vp, _vp, _i32]),
    "hdr_condensed_spmv": (_i32, [_vp, _vp, _vp, _i32]),
    "hdr_csr_spmv_device": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hdr_csr_spmv_host": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "hdr_reference_element": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "hdr_structured_factors": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hdr_alg_hybridize": (_i32, [_vp, _vp]),
    "hdr_alg_static_condense": (_i32, [_vp, _vp]),
    "hdr_alg_info": (_i32, [_vp, _vp]),
    "hdr_alg_matrix": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "hdr_alg_master_globals": (_i32, [_vp, _vp]),
    "hdr_alg_recovery_scale": (_i32, [_vp, _vp]),
    "hdr_alg_recover_hybrid": (_i32, [_vp, _vp, _i64, _vp, _i64, _vp, _vp]),
    "hdr_alg_recover_condensed": (_i32, [_vp, _vp, _i64, _vp, _i64, _vp]),
    "hdr_alg_destroy": (None, [_vp]),
    "hdr_alg_symmetrize": (_i32, [_vp]),
    "hdr_space_set_vertices": (_i32, [_vp, _vp]),
    "hdr_space_element_matrices": (_i32, [_vp, _vp]),
    "hdr_hybrid_symmetrize": (_i32, [_vp]),
    "hdr_umma_selftest": (_i32, [_i32, _i32, _vp, _vp, _vp, _i32]),
    "hdr_hybrid_pcg": (_i32, [_vp, _vp, _vp, _i32, _d, _i64, _i32, _vp, _vp]),
    "hdr_condensed_pcg": (_i32, [_vp, _vp, _vp, _i32, _d, _i64, _i32, _vp, _vp]),
    "hdr_alg_pcg": (_i32, [_vp, _vp, _vp, _i32, _d, _i64, _i32, _vp, _vp]),
    "hdr_csr_pcg_host": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _d, _i64, _i32, _vp, _vp]),
    "hdr_io_read_block_operator": (_i32, [ctypes.c_char_p, _i32, _vp]),
    "hdr_io_blocks_info": (_i32, [_vp, _vp]),
    "hdr_io_blocks_get": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "hdr_io_blocks_destroy": (None, [_vp]),
    "hdr_io_write_block_operator": (_i32, [ctypes.c_char_p, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32]),
    "hdr_io_read_matrix_market": (_i32, [ctypes.c_char_p, _i32, _vp]),
    "hdr_io_read_vector_lines": (_i32, [ctypes.c_char_p, _i32, _vp]),
    "hdr_io_csr_info": (_i32, [_vp, _vp]),
    "hdr_io_csr_get": (_i32, [_vp, _vp, _vp, _vp]),
    "hdr_io_csr_destroy": (None, [_vp]),
    "hdr_io_write_matrix_market": (_i32, [ctypes.c_char_p, _i64, _i64, _vp, _vp, _vp, _i32]),
    "hdr_io_write_vector_lines": (_i32, [ctypes.c_char_p, _i64, _vp, _i32]),
    "hdr_space_set_exact_policy": (_i32, [_vp, _i32, _d, _d, _vp]),
    "hdr_reference_div_form": (_i32, [_i32, _i32, _vp, _vp]),
    "hdr_amg_default_options": (None, [_vp]),
    "hdr_amg_setup": (_i32, [_i64, _vp, _vp, _vp, _i32, _vp, _vp]),
    "hdr_amg_info": (_i32, [_vp, _vp, _vp, _vp]),
    "hdr_amg_level_matrix": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp, _vp]),
    "hdr_amg_apply": (_i32, [_vp, _vp, _vp, _i32]),
    "hdr_amg_destroy": (None, [_vp]),
    "hdr_csr_precond_apply_host": (_i32, [_i64, _vp, _vp, _vp, _i32, _vp, _vp]),
    "hdr_near_nullspace_check": (_i32, [_vp, _vp, _vp, _i32, _i32, _i64, _vp]),
    "hdr_last_error": (ctypes.c_char_p, []),
    "hdr_version": (ctypes.c_char_p, []),
    "hdr_launch_count": (_i64, []),
}

EXPORTED = sorted(_SIGS)

_lib = None


def load(path: os.PathLike | None = None):
    """Loads libhdivred_b200.so (raises ImportError if it has not been built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is missing: build the CUDA library first "
                          "(make -C paper_1801_08914_b200/csrc); there is no CPU fallback")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    return load().hdr_last_error().decode(errors="replace")

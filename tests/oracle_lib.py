"""ctypes front-end to the CPU oracle (oracle/build/liboracle.so) and a reader
for ref_harness dumps (oracle/_ref/ref_harness).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg use this module.
"""
from __future__ import annotations

import ctypes
import os
import struct
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "build" / "liboracle.so"
REF_HARNESS = ROOT / "oracle" / "_ref" / "ref_harness"

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], check=True,
                           stdout=subprocess.DEVNULL)
        L = ctypes.CDLL(str(ORACLE_SO))
        L.hdo_create.restype = ctypes.c_void_p
        L.hdo_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int, ctypes.c_int]
        L.hdo_destroy.argtypes = [ctypes.c_void_p]
        L.hdo_set_h.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
        L.hdo_size.restype = ctypes.c_longlong
        L.hdo_size.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.hdo_count.restype = ctypes.c_longlong
        L.hdo_count.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.hdo_get_d.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
        L.hdo_get_q.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
        L.hdo_set_d.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_longlong]
        L.hdo_gen_inputs.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_ulonglong]
        L.hdo_run.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.hdo_last_error.restype = ctypes.c_char_p
        L.hdo_last_error.argtypes = [ctypes.c_void_p]
        L.hdo_dd_element.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p]
        L.hdo_element_matrix.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p]
        L.hdo_build_reference.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.hdo_piola_element.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


class Oracle:
    """One FE instance: dim, cells, RT order k (restates the reference FE path)."""

    def __init__(self, dim: int, cells, k: int, weighted: bool = False):
        c = list(cells) + [1] * (3 - len(cells))
        arr = (ctypes.c_longlong * 3)(*c)
        self._h = lib().hdo_create(dim, arr, k, int(weighted))
        if not self._h:
            raise OracleError("hdo_create failed")
        self.dim, self.k = dim, k
        self.cells = tuple(c[:dim])

    def __del__(self):
        if getattr(self, "_h", None):
            lib().hdo_destroy(self._h)
            self._h = None

    def size(self, name: str) -> int:
        return int(lib().hdo_size(self._h, name.encode()))

    def has(self, name: str) -> bool:
        return lib().hdo_count(self._h, name.encode()) >= 0

    def get(self, name: str, dtype=np.float64) -> np.ndarray:
        cnt = lib().hdo_count(self._h, name.encode())
        if cnt < 0:
            raise KeyError(name)
        out = np.empty(cnt, dtype=dtype)
        fn = lib().hdo_get_d if dtype == np.float64 else lib().hdo_get_q
        if fn(self._h, name.encode(), out.ctypes.data) != 0:
            raise KeyError(f"{name} has another dtype")
        return out

    def getq(self, name: str) -> np.ndarray:
        return self.get(name, np.int64)

    def set_h(self, h) -> None:
        arr = (ctypes.c_double * 3)(*(list(h) + [1.0] * (3 - len(h))))
        if lib().hdo_set_h(self._h, arr) != 0:
            raise OracleError("hdo_set_h failed")

    def set(self, name: str, data) -> None:
        a = np.ascontiguousarray(data, dtype=np.float64)
        lib().hdo_set_d(self._h, name.encode(), a.ctypes.data, a.size)

    def gen_inputs(self, coef: str, seed: int) -> None:
        if lib().hdo_gen_inputs(self._h, coef.encode(), seed) != 0:
            raise OracleError(lib().hdo_last_error(self._h).decode())

    def run(self, what: str) -> None:
        rc = lib().hdo_run(self._h, what.encode())
        if rc != 0:
            raise OracleError(f"{what}: rc={rc} {lib().hdo_last_error(self._h).decode()}")

    def csr(self, prefix: str, values: str = "values"):
        shape = self.getq(prefix + ".shape")
        return (int(shape[0]), int(shape[1]), self.getq(prefix + ".row_offsets"),
                self.getq(prefix + ".col_indices"), self.get(prefix + "." + values))

    def element_matrix(self, cell: int) -> np.ndarray:
        n = self.size("n")
        out = np.empty(n * n)
        lib().hdo_element_matrix(self._h, cell, out.ctypes.data)
        return out.reshape(n, n)

    def dd_element(self, cell: int):
        n = self.size("n")
        rows = np.empty(n, np.int64)
        h = np.empty(n * n)
        g = np.empty(n)
        xh = np.empty(n)
        nr = lib().hdo_dd_element(self._h, cell, rows.ctypes.data, h.ctypes.data, g.ctypes.data, xh.ctypes.data)
        if nr < 0:
            raise OracleError(lib().hdo_last_error(self._h).decode())
        return rows[:nr].copy(), h[: nr * nr].reshape(nr, nr).copy(), g[:nr].copy(), xh.copy()


def build_reference(dim: int, k: int, h, nq: int):
    """Restated build_reference (rt_space.cpp:180-314): divdiv, mass, face_moments, unit_load."""
    n = dim * (k + 1) ** (dim - 1) * 2 + dim * k * (k + 1) ** (dim - 1)
    dpf = (k + 1) ** (dim - 1)
    hh = (ctypes.c_double * 3)(*(list(h) + [1.0] * (3 - len(h))))
    dd_ = np.zeros(n * n)
    mm = np.zeros(n * n)
    fm = np.zeros(2 * dim * dpf * n)
    ul = np.zeros(3 * n)
    rc = lib().hdo_build_reference(dim, k, hh, nq, dd_.ctypes.data, mm.ctypes.data, fm.ctypes.data, ul.ctypes.data)
    if rc != 0:
        raise OracleError("build_reference failed")
    return dd_.reshape(n, n), mm.reshape(n, n), fm, ul


def piola_element(k: int, h, verts, nq: int, pressure: bool = False):
    """Config-4 restatement: (divdiv, mass[, div_form, pressure_mass]) of the trilinear cell
    with the 8 vertices verts (8 x 3, v = vx + 2 vy + 4 vz) mapped from the h box."""
    n = 3 * (k + 1) ** 2 * 2 + 3 * k * (k + 1) ** 2
    npr = (k + 1) ** 3
    hh = (ctypes.c_double * 3)(*h)
    v = np.ascontiguousarray(verts, dtype=np.float64).reshape(24)
    D = np.zeros(n * n)
    M = np.zeros(n * n)
    B = np.zeros(npr * n)
    W = np.zeros(npr * npr)
    rc = lib().hdo_piola_element(k, hh, v.ctypes.data, nq, D.ctypes.data, M.ctypes.data,
                                 B.ctypes.data if pressure else None, W.ctypes.data if pressure else None)
    if rc != 0:
        raise OracleError("piola_element failed")
    if pressure:
        return D.reshape(n, n), M.reshape(n, n), B.reshape(npr, n), W.reshape(npr, npr)
    return D.reshape(n, n), M.reshape(n, n)


def box_vertices(h, origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    return np.array([[origin[a] + h[a] * ((v >> a) & 1) for a in range(3)] for v in range(8)], dtype=np.float64)


def read_dump(path) -> dict:
    """Reads an HDRB0001 dump written by oracle/ref_harness.cpp."""
    out = {}
    with open(path, "rb") as f:
        if f.read(8) != b"HDRB0001":
            raise ValueError("bad magic")
        while True:
            hdr = f.read(4)
            if not hdr:
                break
            (ln,) = struct.unpack("<I", hdr)
            name = f.read(ln).decode()
            typ = f.read(1).decode()
            (cnt,) = struct.unpack("<Q", f.read(8))
            dt = np.float64 if typ == "d" else np.int64
            out[name] = np.frombuffer(f.read(8 * cnt), dtype=dt).copy()
    return out


def run_ref_dump(out_path, dim, cells, k, coef, seed, weighted=False, blocks=True, essential=False,
                 nullspace=False, amg=False, amg_options=None) -> dict:
    """Runs the reference (oracle/_ref/ref_harness) and reads its dump (essential:
    every boundary face eliminated first, eliminate_essential)."""
    if not REF_HARNESS.exists():
        raise FileNotFoundError(REF_HARNESS)
    args = [str(REF_HARNESS), "dump", f"out={out_path}", f"dim={dim}", "cells=" + ",".join(map(str, cells)),
            f"k={k}", f"coef={coef}", f"seed={seed}", f"weighted={int(weighted)}", f"blocks={int(blocks)}",
            f"essential={int(essential)}", f"nullspace={int(nullspace)}", f"amg={int(amg)}"]
    for key, val in (amg_options or {}).items():  # amg_theta, amg_cap, amg_levels, amg_omega
        args.append(f"{key}={val}")
    subprocess.run(args, check=True, env={**os.environ, "HDIVRED_NUM_THREADS": "1"})
    return read_dump(out_path)


def sampled_rows_vs_dd(o: "Oracle", ro, ci, hv, gv, n: int, nx: int, base) -> tuple[float, float]:
    """H / g rows of the cells in `base` and their +x neighbours (so shared-face
    blocks are complete) against the element-wise DD oracle (hdo_dd_element);
    needs o.run("structure").  Returns (max|dH| / max|H|, max|dg| / max|g|)."""
    have = set(int(e) for e in base) | {int(e) + 1 for e in base}
    row_vals, row_g = {}, {}
    for cell in sorted(have):
        rows, h, gt, _ = o.dd_element(cell)
        for a_, r in enumerate(rows):
            row_g.setdefault(int(r), []).append(gt[a_])
            for b_, c in enumerate(rows):
                row_vals.setdefault((int(r), int(c)), []).append(h[a_, b_])
    C = o.getq("C.col_indices").reshape(-1, 2)

    def cells_of(row):
        return {int(C[row, 0]) // n, int(C[row, 1]) // n}

    worst_h, worst_g, checked = 0.0, 0.0, 0
    for (r, c), parts in row_vals.items():
        if not (cells_of(r) & cells_of(c)) <= have:
            continue
        p = ro[r] + np.searchsorted(ci[ro[r]:ro[r + 1]], c)
        assert ci[p] == c
        worst_h = max(worst_h, abs(hv[p] - sum(parts)))
        checked += 1
    for r, parts in row_g.items():
        if cells_of(r) <= have:
            worst_g = max(worst_g, abs(gv[r] - sum(parts)))
    assert checked > 0
    return worst_h / max(np.max(np.abs(hv)), 1e-300), worst_g / max(np.max(np.abs(gv)), 1e-300)


def rel_err(a, b, scale=None) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    s = scale if scale is not None else max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / s)

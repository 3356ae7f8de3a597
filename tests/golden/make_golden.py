"""Generates the committed golden fixtures tests/golden/*.npz by running the
REFERENCE itself (oracle/_ref/ref_harness, built from /root/reference by
oracle/Makefile) on small seeded instances.  Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture holds every array ref_harness dumps: reference element matrices
(D_ref, M_ref, face moments), the seeded inputs (alpha, beta, f_hat, lambda,
x_b), P, C, H/g, recovered x_hat/x, S/f_S/master_globals, recovered x_cond,
the reference spmv outputs, ref_div_form and the near_nullspace_check eigenvalues.  k = 2, 3 use the guard-lifted copy of
rt_space.cpp.
"""
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import run_ref_dump  # noqa: E402

CASES = [
    # name, dim, cells, k, coef, seed, weighted, blocks
    ("q2_rt0_4x3_unit", 2, (4, 3), 0, "uniform:1:1", 1001, False, True),
    ("q2_rt0_8x8_unit", 2, (8, 8), 0, "uniform:1:1", 1001, False, True),
    ("h3_rt0_3x2x2_logu", 3, (3, 2, 2), 0, "logu:1e-2:1e2", 1002, False, True),
    ("h3_rt0_4x4x4_logu", 3, (4, 4, 4), 0, "logu:1e-2:1e2", 1002, False, True),
    ("h3_rt1_2x2x2_logu", 3, (2, 2, 2), 1, "logu:1e-2:1e2", 1003, False, True),
    ("h3_rt1_3x2x2_logu_weighted", 3, (3, 2, 2), 1, "logu:1e-2:1e2", 1003, True, True),
    ("q2_rt1_3x3_logu", 2, (3, 3), 1, "logu:1e-2:1e2", 1005, False, True),
    ("h3_rt2_2x2x2_logu3", 3, (2, 2, 2), 2, "logu:1e-3:1e3", 1004, False, False),
    ("h3_rt3_2x2x1_checker", 3, (2, 2, 1), 3, "checker:1e-2:1e2", 1005, False, False),
    ("h3_rt0_1x1x1_unit", 3, (1, 1, 1), 0, "uniform:1:1", 7, False, True),
    ("h3_rt0_3x3x3_unit", 3, (3, 3, 3), 0, "uniform:1:1", 7, False, True),
]


def main():
    with tempfile.TemporaryDirectory() as td:
        for name, dim, cells, k, coef, seed, weighted, blocks in CASES:
            d = run_ref_dump(Path(td) / "d.bin", dim, cells, k, coef, seed, weighted, blocks, nullspace=True)
            d["case"] = np.array([dim, *list(cells) + [1] * (3 - len(cells)), k, seed, int(weighted)], np.int64)
            d["coef"] = np.frombuffer(coef.encode(), dtype=np.uint8)
            np.savez_compressed(HERE / f"{name}.npz", **{k_.replace(".", "__"): v for k_, v in d.items()})
            print(name, sum(v.nbytes for v in d.values()) // 1024, "KiB raw")


if __name__ == "__main__":
    main()

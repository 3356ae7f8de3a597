"""Instance I/O (csrc/io.cpp) against the reference's own readers and writers
(src/block_io.cpp, src/matrix_market.cpp), host only (no GPU needed).

The reference writes an instance (oracle/_ref/ref_harness export: its
write_block_operator / write_matrix_market / write_vector_market /
write_vector_lines); our parallel readers must return exactly the arrays the
reference holds (ref_harness dump of the same problem), and our writers must
reproduce the reference's files byte for byte.  Malformed files raise
FormatError with the line number, like the reference's readers.
"""
import numpy as np
import pytest

from oracle_lib import REF_HARNESS, run_ref_dump

import paper_1801_08914_b200 as hd
from paper_1801_08914_b200 import io as hio

pytestmark = pytest.mark.skipif(not REF_HARNESS.exists(), reason="ref_harness not built (needs /root/reference)")

CASES = [(3, (3, 2, 2), 1, "logu:0.01:100", False), (2, (5, 4), 2, "logu:0.001:1000", False),
         (3, (2, 2, 2), 1, "logu:0.01:100", True), (3, (4, 3, 2), 0, "uniform:1:1", False)]


def _export(tmp_path, dim, cells, k, coef, weighted):
    import subprocess

    pre = tmp_path / "inst"
    subprocess.run([str(REF_HARNESS), "export", f"prefix={pre}", f"dim={dim}", "cells=" + ",".join(map(str, cells)),
                    f"k={k}", f"coef={coef}", "seed=17", f"weighted={int(weighted)}"], check=True,
                   capture_output=True)
    return pre


@pytest.mark.parametrize("dim,cells,k,coef,weighted", CASES)
@pytest.mark.parametrize("threads", [1, 7])
def test_readers_match_reference_arrays(tmp_path, dim, cells, k, coef, weighted, threads):
    pre = _export(tmp_path, dim, cells, k, coef, weighted)
    ref = run_ref_dump(tmp_path / "d.bin", dim, cells, k, coef, 17, weighted=weighted)
    blocks, gl, sg, bd, gd = hio.read_block_operator(f"{pre}.blocks", threads)
    assert np.array_equal(np.concatenate([b.ravel() for b in blocks]), ref["a_hat"])
    assert np.array_equal(gl, ref["dof_global"]) and np.array_equal(sg, ref["dof_sign"])
    for name, suf in (("P", "p"), ("C", "c")):
        m = hio.read_matrix_market(f"{pre}.{suf}.mtx", threads)
        assert (m.nrows, m.ncols) == tuple(ref[name + ".shape"])
        assert np.array_equal(m.row_offsets, ref[name + ".row_offsets"])
        assert np.array_equal(m.col_indices, ref[name + ".col_indices"])
        assert np.array_equal(m.values, ref[name + ".values"])
    assert np.array_equal(hio.read_vector_market(f"{pre}.f.mtx", threads), ref["f_hat"])
    assert np.array_equal(hio.read_vector_lines(f"{pre}.f.txt", threads), ref["f_hat"])
    inst = hio.import_instance(str(pre), threads)
    assert inst.interior_global_begin == -1 and inst.n_hat == ref["f_hat"].size


@pytest.mark.parametrize("dim,cells,k,coef,weighted", CASES)
def test_writers_byte_identical_to_reference(tmp_path, dim, cells, k, coef, weighted):
    pre = _export(tmp_path, dim, cells, k, coef, weighted)
    blocks, gl, sg, bd, gd = hio.read_block_operator(f"{pre}.blocks")
    out = tmp_path / "ours"
    hio.write_block_operator(f"{out}.blocks", blocks, gl, sg, gd, threads=5)
    for suf in ("p", "c"):
        hio.write_matrix_market(f"{out}.{suf}.mtx", hio.read_matrix_market(f"{pre}.{suf}.mtx"), threads=3)
    f = hio.read_vector_lines(f"{pre}.f.txt")
    hio.write_vector_market(f"{out}.f.mtx", f)
    hio.write_vector_lines(f"{out}.f.txt", f, threads=4)
    for suf in ("blocks", "p.mtx", "c.mtx", "f.mtx", "f.txt"):
        assert open(f"{out}.{suf}", "rb").read() == open(f"{pre}.{suf}", "rb").read(), suf


def test_format_errors_carry_the_line(tmp_path):
    pre = _export(tmp_path, 3, (2, 1, 1), 0, "uniform:1:1", False)
    text = open(f"{pre}.blocks").read().split("\n")
    bad = tmp_path / "bad.blocks"
    open(bad, "w").write("\n".join(["%%Nope"] + text[1:]))
    with pytest.raises(hd.FormatError, match="header"):
        hio.read_block_operator(str(bad))
    t2 = list(text)
    t2[4] = t2[4].replace(t2[4].split()[2], "1.0x", 1)  # a malformed entry on physical line 5
    open(bad, "w").write("\n".join(t2))
    with pytest.raises(hd.FormatError, match=r"bad matrix entry \(line 5\)"):
        hio.read_block_operator(str(bad))
    open(bad, "w").write("\n".join(text[:6]))  # truncated
    with pytest.raises(hd.FormatError, match="unexpected end"):
        hio.read_block_operator(str(bad))
    mtx = open(f"{pre}.c.mtx").read().split("\n")
    badm = tmp_path / "bad.mtx"
    m2 = list(mtx)
    m2[2] = "99 1 1.0"
    open(badm, "w").write("\n".join(m2))
    with pytest.raises(hd.FormatError, match=r"entry index out of range \(line 3\)"):
        hio.read_matrix_market(str(badm))
    with pytest.raises(hd.FormatError, match="cannot open"):
        hio.read_matrix_market(str(tmp_path / "missing.mtx"))


def test_matrix_market_duplicates_summed_and_comments_skipped(tmp_path):
    p = tmp_path / "m.mtx"
    open(p, "w").write("%%MatrixMarket matrix coordinate real general\n% comment\n3 3 4\n"
                       "2 3 1.5\n1 1 2\n% inner comment\n2 3 0.25\n2 1 -1\n")
    m = hio.read_matrix_market(str(p))
    assert m.to_dense().tolist() == [[2, 0, 0], [-1, 0, 1.75], [0, 0, 0]]

"""The bench's seeded inputs (paper_1801_08914_b200/inputs.py) are bit-identical
to the oracle's §8(d) stream (oracle/hdr_oracle.c hdo_gen_inputs), so the timed
workload is the parity-tested one (CPU only)."""
import numpy as np
import pytest

from oracle_lib import Oracle
from paper_1801_08914_b200 import inputs


@pytest.mark.parametrize("dim,cells,k,coef", [
    (3, (5, 4, 3), 0, ("logu", 1e-2, 1e2)), (2, (7, 5), 1, ("uniform", 1.0, 1.0)),
    (3, (4, 4, 4), 3, ("checker", 1e-2, 1e2)), (3, (4, 4, 4), 1, ("softhard", -8, 0)),
    (3, (3, 3, 3), 2, ("logu", 1e-3, 1e3)),
])
def test_stream_matches_oracle(dim, cells, k, coef):
    o = Oracle(dim, cells, k)
    o.gen_inputs(f"{coef[0]}:{coef[1]}:{coef[2]}", 1234)
    a, b, f, lam, xb, _ = inputs.make_inputs(dim, cells, k, coef, 1234, extras=True)
    for name, v in (("alpha", a), ("beta", b), ("f_hat", f), ("lambda", lam), ("x_b", xb)):
        assert np.array_equal(v, o.get(name)), name


def test_config4_vertices_match_oracle():
    o = Oracle(3, (4, 3, 5), 2)
    o.gen_inputs("logu:0.001:1000;perturb=0.2", 1004)
    a, b, f, lam, xb, v = inputs.make_inputs(3, (4, 3, 5), 2, ("logu", 1e-3, 1e3), 1004, perturb=0.2, extras=True)
    assert np.array_equal(a, o.get("alpha")) and np.array_equal(f, o.get("f_hat"))
    assert np.array_equal(v.ravel(), o.get("vertices"))


def test_config2_full_size_stream():
    cfg = inputs.CONFIGS[2]
    o = Oracle(3, cfg["cells"], 0)
    o.gen_inputs("logu:0.01:100", cfg["seed"])
    a, b, f, _ = inputs.config_inputs(2)
    assert np.array_equal(a, o.get("alpha")) and np.array_equal(b, o.get("beta")) and np.array_equal(f, o.get("f_hat"))

"""Full-size parity on the five BASELINE configs (GPU), on the bench's own
inputs (the §8(d) Xorshift stream, seed 1000 + config id).

  * H and S patterns bit-exact, every row, against the oracle's structure-only
    restatement of from_triplets (oracle "pattern_H" / "pattern_S", pinned to the
    reference's goldens in tests/test_oracle_pin.py), configs 1-5;
  * configs 1-3: EVERY H, g, x_hat, x entry against the element-wise
    double-double oracle; configs 2-3: every S, f_S, x_cond entry likewise;
  * config 5: every H / g entry against the device's exact double-double path
    forced on all cells (itself pinned to the CPU DD oracle on the goldens,
    tests/test_failsafe_gpu.py), plus 256 sampled cells against the CPU DD oracle;
  * config 4: tests/test_piola_gpu.py (256 sampled cells at full size).
Tolerance 1e-11 of max|entry|.
"""
import numpy as np
import pytest

from conftest import has_cuda
from oracle_lib import Oracle, rel_err, sampled_rows_vs_dd

pytestmark = pytest.mark.gpu
TOL = 1e-11

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402
from paper_1801_08914_b200.inputs import CONFIGS  # noqa: E402


def _oracle(cid):
    cfg = CONFIGS[cid]
    o = Oracle(cfg["dim"], cfg["cells"], cfg["k"])
    kind, lo, hi = cfg["coef"]
    o.gen_inputs(f"{kind}:{lo}:{hi}", cfg["seed"])
    return cfg, o


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_full_patterns_bit_exact(cid):
    cfg, o = _oracle(cid)
    sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    for which in ("H", "S"):
        o.run(f"pattern_{which}")
        ro, ci = sp.pattern(which)
        assert np.array_equal(ro, o.getq(f"{which}p.row_offsets")), which
        assert np.array_equal(ci, o.getq(f"{which}p.col_indices")), which
        del ro, ci
    assert np.array_equal(sp.master_globals(), np.arange(sp.info["n_s"]))


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_full_hybridize_and_recovery_every_entry_vs_dd(cid):
    cfg, o = _oracle(cid)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    o.run("dd_recover")
    sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    op = sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    assert op.exact_cells() == 0
    hv, gv = op.values()
    eh, eg = rel_err(hv, o.get("H.values_dd")), rel_err(gv, o.get("g_dd"))
    x_hat, x = op.recover(o.get("lambda"), o.get("f_hat"))
    ex, exx = rel_err(x_hat, o.get("x_hat_dd")), rel_err(x, o.get("x_dd"))
    print(f"config {cid} full: H {eh:.1e} g {eg:.1e} x_hat {ex:.1e} x {exx:.1e}; "
          f"reference-port vs DD H {rel_err(o.get('H.values'), o.get('H.values_dd')):.1e}")
    assert eh <= TOL and eg <= TOL and ex <= TOL and exx <= TOL


@pytest.mark.parametrize("cid", [2, 3])
def test_full_static_condensation_every_entry_vs_dd(cid):
    cfg, o = _oracle(cid)
    o.run("port_condense")
    o.run("dd_condense")
    o.run("dd_recover_condensed")
    sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    ro, ci = sp.pattern("S")
    assert np.array_equal(ro, o.getq("S.row_offsets")) and np.array_equal(ci, o.getq("S.col_indices"))
    cop = sp.static_condense(o.get("alpha"), o.get("beta"), o.get("f_hat"))
    sv, fs = cop.values()
    es, ef = rel_err(sv, o.get("S.values_dd")), rel_err(fs, o.get("f_s_dd"))
    x = cop.recover(o.get("x_b"), o.get("f_hat"))
    exc = rel_err(x, o.get("x_cond_dd"))
    print(f"config {cid} full: S {es:.1e} f_S {ef:.1e} x_cond {exc:.1e}")
    assert es <= TOL and ef <= TOL and exc <= TOL


def test_config5_every_entry_vs_exact_path_and_sampled_vs_dd():
    cfg, o = _oracle(5)
    o.run("structure")
    sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    op = sp.hybridize(a, b, f)
    assert op.exact_cells() == 0
    hv, gv = op.values()
    sx = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    sx.set_exact_policy(force=True)
    opx = sx.hybridize(a, b, f)
    assert opx.exact_cells() == sx.ncells
    hx, gx = opx.values()
    eh, eg = rel_err(hv, hx), rel_err(gv, gx)
    print(f"config 5 full, structured vs exact DD path, every entry: H {eh:.1e} g {eg:.1e}")
    assert eh <= TOL and eg <= TOL
    del hx, gx, opx, sx
    ro, ci = sp.pattern("H")
    rng = np.random.default_rng(1005)
    n0 = cfg["cells"][0]
    pool = [e for e in range(sp.ncells) if e % n0 < n0 - 1]
    base = [int(e) for e in rng.choice(pool, 128, replace=False)]
    eh, eg = sampled_rows_vs_dd(o, ro, ci, hv, gv, sp.n, n0, base)
    print(f"config 5 full, 256 sampled cells vs the CPU DD oracle: H {eh:.1e} g {eg:.1e}")
    assert eh <= TOL and eg <= TOL

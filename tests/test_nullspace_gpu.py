"""near_nullspace_check (src/reduction.cpp:711-742) on the device
(kern_nullspace.cu) against the reference's own eigenvalues (golden fixtures
dumped by oracle/_ref/ref_harness): bit-identical, and the reference's
dimension checks (tests/unit_reduction.cpp:465-481, acceptance A6)."""
import numpy as np
import pytest

from conftest import GOLDEN_CASES, has_cuda, load_golden

pytestmark = pytest.mark.gpu

if has_cuda():
    import torch

    import paper_1801_08914_b200 as hd


def _space(g):
    return hd.Space(g["dim"], g["cells"], g["k"], weighted=g["weighted"]) if g["weighted"] else \
        hd.Space(g["dim"], g["cells"], g["k"])


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_eigenvalues_bit_identical_to_reference(name):
    g = load_golden(name)
    sp = _space(g)
    ev = sp.near_nullspace_check(g["alpha"], g["beta"], weighted=g["weighted"])
    ref = g["nullspace"]
    assert ev.shape == ref.shape
    assert np.array_equal(ev, ref), np.max(np.abs(ev - ref)) / max(1e-300, np.max(np.abs(ref)))


def test_device_inputs_match_host_inputs():
    g = load_golden("h3_rt1_2x2x2_logu")
    sp = _space(g)
    host = sp.near_nullspace_check(g["alpha"], g["beta"])
    dev = sp.near_nullspace_check(torch.from_numpy(g["alpha"]).cuda(), torch.from_numpy(g["beta"]).cuda())
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("n", [2, 3])
def test_at_most_one_near_zero_eigenvalue(n):
    """unit_reduction.cpp 'near-nullspace of C Y C^T': 2^3 and 3^3, k = 0, alpha = beta = 1."""
    sp = hd.Space(3, (n, n, n), 0)
    ev = sp.near_nullspace_check(np.ones(n ** 3), np.ones(n ** 3))
    assert ev.size > 0
    assert int(np.sum(ev < 1e-10 * ev[-1])) <= 1


def test_single_cell_has_no_multipliers():
    sp = hd.Space(3, (1, 1, 1), 0)
    assert sp.near_nullspace_check(np.ones(1), np.ones(1)).size == 0


def test_cap_and_coefficient_errors():
    sp = hd.Space(3, (3, 3, 3), 0)
    with pytest.raises(hd.CapExceededError):
        sp.near_nullspace_check(np.ones(27), np.ones(27), dense_cap=100)
    bad = np.ones(27)
    bad[5] = 0.0
    with pytest.raises(ValueError):
        sp.near_nullspace_check(np.ones(27), bad)

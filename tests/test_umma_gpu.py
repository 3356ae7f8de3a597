"""tcgen05 TF32 tensor-core path (paper_1801_08914_b200/csrc/umma.cuh) on the
device: one-CTA GEMMs with the accumulator in TMEM against numpy (GPU)."""
import numpy as np
import pytest

from conftest import has_cuda

pytestmark = pytest.mark.gpu

if not has_cuda():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1801_08914_b200 as hd  # noqa: E402,F401
from paper_1801_08914_b200 import _capi  # noqa: E402


def tf32(x):
    """cvt.rna.tf32.f32: round to nearest (ties away) to a 10-bit mantissa."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def run(n, k, a, b, split):
    d = np.empty((128, n), np.float32)
    st = _capi.load().hdr_umma_selftest(n, k, a.ctypes.data, b.ctypes.data, d.ctypes.data, split)
    assert st == 0, _capi.last_error()
    return d


@pytest.mark.parametrize("n,k", [(16, 8), (32, 64), (112, 40), (128, 96)])
def test_umma_tf32(n, k):
    rng = np.random.default_rng(n + k)
    a = rng.standard_normal((128, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    d = run(n, k, a, b, 0)
    ref = tf32(a).astype(np.float64) @ tf32(b).astype(np.float64).T
    assert np.abs(d - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("n,k", [(16, 8), (112, 40), (128, 96)])
def test_umma_3xtf32_is_fp32_accurate(n, k):
    rng = np.random.default_rng(7 * n + k)
    a = rng.standard_normal((128, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    d = run(n, k, a, b, 1)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    err = np.abs(d - ref).max() / (np.abs(a).max() * np.abs(b).max() * k)
    assert err <= 2e-7, err

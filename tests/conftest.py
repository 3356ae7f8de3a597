import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full BASELINE-size case")


def load_golden(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz")
    d = {k.replace("__", "."): z[k] for k in z.files}
    c = d["case"]
    d["dim"], d["cells"], d["k"], d["seed"], d["weighted"] = int(c[0]), tuple(int(x) for x in c[1:1 + int(c[0])]), int(c[4]), int(c[5]), bool(c[6])
    d["coef"] = bytes(d["coef"]).decode()
    return d


GOLDEN_CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


@pytest.fixture(params=GOLDEN_CASES)
def golden(request):
    return load_golden(request.param)


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False

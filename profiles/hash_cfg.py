"""sha256 of H values and g for a BASELINE config with the library in HDR_LIB (variant checks:
kernel variants that must give identical bits).   python profiles/hash_cfg.py 2"""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1801_08914_b200 as hd  # noqa: E402
from paper_1801_08914_b200.inputs import CONFIGS, config_inputs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = CONFIGS[cid]
a, b, f, v = config_inputs(cid)
sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
if v is not None:
    sp.set_vertices(v)
op = sp.hybridize(*[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a, b, f)])
hv, g = op.values()
print(cid, hashlib.sha256(hv.tobytes() + g.tobytes()).hexdigest()[:16], "exact", op.exact_cells())

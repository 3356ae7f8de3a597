"""Distribution of the per-cell first-order ratio q = |C| / |H0| (the structured
solve's order control, hdr_device.cuh struct_order) on a BASELINE config, and the
Neumann order each cell needs (10 q^(P+1) <= 1e-12).   python profiles/qdist.py 3"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1801_08914_b200 as hd  # noqa: E402
from paper_1801_08914_b200.inputs import CONFIGS, config_inputs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = CONFIGS[cid]
a, b, f, _ = config_inputs(cid)
sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
q = torch.zeros(sp.ncells, dtype=torch.float32, device="cuda")
sp.set_exact_policy(q_log=q)
op = sp.hybridize(*[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a, b, f)])
torch.cuda.synchronize()
qs = q.cpu().numpy().astype(np.float64)
print(f"cfg{cid}: cells {qs.size}, exact cells {op.exact_cells()}")
print("q quantiles (50/90/99/100%):", np.quantile(qs, [0.5, 0.9, 0.99, 1.0]))
P = np.ones_like(qs, dtype=int)
t = 10 * qs ** 2
while np.any((t > 1e-12) & (P < 4)):
    m = (t > 1e-12) & (P < 4)
    P[m] += 1
    t[m] *= qs[m]
for p in range(1, 5):
    print(f"  order {p}: {np.mean(P == p) * 100:.1f}% of cells")

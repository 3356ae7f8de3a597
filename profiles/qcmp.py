"""q (first-order ratio) per cell on a small RT1 case for the library in HDR_LIB (debug)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1801_08914_b200 as hd
from oracle_lib import Oracle
o = Oracle(3, (4, 4, 4), 1)
o.gen_inputs("logu:1e-2:1e2", 1003)
sp = hd.Space(3, (4, 4, 4), 1)
q = torch.zeros(sp.ncells, dtype=torch.float32, device="cuda")
sp.set_exact_policy(q_log=q)
op = sp.hybridize(*[torch.from_numpy(o.get(k)).cuda() for k in ("alpha", "beta", "f_hat")])
torch.cuda.synchronize()
print("exact", op.exact_cells(), "q", q.cpu().numpy()[:12])

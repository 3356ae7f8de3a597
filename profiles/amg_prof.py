import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1801_08914_b200 as hd
from paper_1801_08914_b200.inputs import CONFIGS, config_inputs
cfg = CONFIGS[2]
a, b, f, _ = config_inputs(2)
sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
op = sp.hybridize(*[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a, b, f)])
op.symmetrize()
lam, r = op.pcg(rtol=1e-12, maxit=3, precond="amg")
print(r)

"""The reduced solve on the device: hybridize -> symmetrize ->
pcg(precond) -> recover on a BASELINE config, wall times per stage (host clock
around synchronous calls).   python profiles/solve_bench.py 3 amg"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1801_08914_b200 as hd  # noqa: E402
from paper_1801_08914_b200.inputs import CONFIGS, config_inputs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pc = sys.argv[2] if len(sys.argv) > 2 else "amg"
cfg = CONFIGS[cid]
a, b, f, v = config_inputs(cid)
sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
if v is not None:
    sp.set_vertices(v)
dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a, b, f)]
out = {"config": cid, "precond": pc, "m": sp.m}
for rep in range(2):  # the second repetition is reported (first touches / allocations)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = sp.hybridize(*dev)
    op.symmetrize()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    lam, r = op.pcg(rtol=1e-12, maxit=2000, precond=pc)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x_hat, x = op.recover(lam, np.ascontiguousarray(f))  # host arrays (lam comes back to the host)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out.update({"hybridize_s": t1 - t0, "pcg_s": t2 - t1, "recover_s": t3 - t2, "iterations": r["iterations"],
                "converged": r["converged"], "final_relative_residual": r["final_relative_residual"]})
print(json.dumps(out))

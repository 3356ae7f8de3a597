"""Fail-safe diagnostics on the BASELINE configs (GPU): distribution of the
per-cell first-order ratio q the structured kernels measure, the estimated
error q * eps of the accepted cells, the number of rejected cells, and the
realised error of the structured result against the exact double-double path
forced on every cell (max |H_fast - H_exact| / max |H|)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1801_08914_b200 as hd  # noqa: E402
from oracle_lib import Oracle  # noqa: E402

CFG = {2: (3, (64, 64, 64), 0, "logu:1e-2:1e2", 1002), 3: (3, (48, 48, 48), 1, "logu:1e-2:1e2", 1003),
       5: (3, (32, 32, 32), 3, "checker:1e-2:1e2", 1005), 1: (2, (64, 64), 0, "uniform:1:1", 1001)}
out = {}
for cid in [int(c) for c in (sys.argv[1:] or ["1", "2", "3", "5"])]:
    dim, cells, k, coef, seed = CFG[cid]
    o = Oracle(dim, cells, k)
    o.gen_inputs(coef, seed)
    a, b, f = (torch.from_numpy(o.get(x)).cuda() for x in ("alpha", "beta", "f_hat"))
    sp = hd.Space(dim, cells, k)
    q = torch.zeros(sp.ncells, dtype=torch.float32, device="cuda")
    sp.set_exact_policy(q_log=q)
    op = sp.hybridize(a, b, f)
    nx = op.exact_cells()
    hv, gv = op.values()
    qs = q.cpu().numpy().astype(np.float64)
    sp.set_exact_policy(force=True)
    t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t[0].record()
    op2 = sp.hybridize(a, b, f)
    t[1].record()
    torch.cuda.synchronize()
    hx, gx = op2.values()
    n = sp.n
    eps32 = np.sqrt(2.0 * n) * 2.0 ** -24
    rec = {"config": cid, "cells": sp.ncells, "exact_cells": nx, "q_max": float(qs.max()),
           "q_p50": float(np.median(qs)), "q_p99": float(np.quantile(qs, 0.99)),
           "est_max_fp32": float(qs.max() * eps32), "est_max_tc": float(qs.max() * 1e-6),
           "fast_vs_exact_H": float(np.max(np.abs(hv - hx)) / np.max(np.abs(hx))),
           "fast_vs_exact_g": float(np.max(np.abs(gv - gx)) / np.max(np.abs(gx))),
           "forced_exact_ms": t[0].elapsed_time(t[1])}
    print(json.dumps(rec), flush=True)
    out[cid] = rec
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/failsafe_diag.json").write_text(json.dumps(out, indent=1))

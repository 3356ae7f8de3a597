"""Phase timing of k_spd_hyb (CTA 0 cycle counters) with the variant build
HDR_LIB=build_x1/libhdr_timing.so (make EXTRA=-DHDR_SPD_TIMING ...)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_1801_08914_b200 as hd
from oracle_lib import Oracle
o = Oracle(3, (24, 24, 24), 2)
o.gen_inputs("logu:1e-3:1e3;perturb=0.2", 1004)
sp = hd.Space(3, (24, 24, 24), 2)
sp.set_vertices(o.get("vertices"))
sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
lib = hd._capi.load()
out = (ctypes.c_ulonglong * 16)()
ctypes.CDLL(os.environ["HDR_LIB"]).hdr_debug_spd_prof(out)
v = list(out)
names = ["loop-top", "load+thr", "sweep-T", "sweep-tiles", "sweep-writeback", "pivchk", "Zinit", "residual", "update", "post", "epilogue"]
cells, res = v[14], v[15]
tot = sum(v[:11])
print(f"cells {cells} residuals {res} ({res / max(cells, 1):.2f}/cell) cycles/cell {tot / max(cells, 1):.0f}")
print(f"  warp0 tiles {v[11] / max(cells, 1):.0f}  warp0 tiles+sweep {v[12] / max(cells, 1):.0f}  warp1 tiles {v[13] / max(cells, 1):.0f}  (cyc/cell)")
for i, nm in enumerate(names):
    print(f"  {nm:16s} {v[i] / max(cells, 1):9.0f} cyc/cell  {100 * v[i] / max(tot, 1):5.1f}%")

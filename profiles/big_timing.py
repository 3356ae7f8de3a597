"""Phase timing of k_hyb_big (CTA 0 cycle counters, both colours) with the
variant build HDR_LIB=build_x2/libhdr_big.so (make EXTRA=-DHDR_BIG_TIMING ...)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_1801_08914_b200 as hd
from oracle_lib import Oracle
o = Oracle(3, (32, 32, 32), 3)
o.gen_inputs("checker:1e-2:1e2", 1005)
sp = hd.Space(3, (32, 32, 32), 3)
sp.hybridize(o.get("alpha"), o.get("beta"), o.get("f_hat"))
out = (ctypes.c_ulonglong * 32)()
ctypes.CDLL(os.environ["HDR_LIB"]).hdr_debug_big_prof(out)
v = list(out)
names = ["loop-top", "f/s/z setup", "V blocks", "TC: Y=Delta V", "TC: C=V^T Y", "ratio check", "CUDA-core fallback", "scatter"]
cells = v[14]
tot = sum(v[:8])
print(f"cells {cells} fallback cells {v[15]} cycles/cell {tot / max(cells, 1):.0f}")
print(f"  scatter tables (part of scatter) {v[12] / max(cells, 1):.0f}")
print(f"  Y loop (thread 0): wait {v[8] / max(cells, 1):.0f}  A fill {v[9] / max(cells, 1):.0f}  B fill {v[10] / max(cells, 1):.0f}  barrier {v[11] / max(cells, 1):.0f}  MMA issue {v[12] / max(cells, 1):.0f}")
print("  V rounds (face tid 0 / interior tid 256):", [round(v[16 + q] / max(cells, 1)) for q in range(6)],
      "barrier wait", round(v[24] / max(cells, 1)), round(v[25] / max(cells, 1)))
print("  correction ratio |C|/|H0| histogram (all cells):", {f"[1e{-16 + 2 * q},1e{-14 + 2 * q})": v[26 + q] for q in range(6)})
for i, nm in enumerate(names):
    print(f"  {nm:20s} {v[i] / max(cells, 1):9.0f} cyc/cell  {100 * v[i] / max(tot, 1):5.1f}%")

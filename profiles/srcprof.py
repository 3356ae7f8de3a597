"""Per-CUDA-line summary of an ncu --set full capture (--import-source on,
-lineinfo): warp-stall samples and executed warp instructions per source line,
per kernel.   python profiles/srcprof.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn = path = None
agg = {}
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] and r[0] != "Line No":  # a CUDA source line with its aggregated metrics
        d = dict(zip(hdr[2:], r[2:]))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0"))
            ins = int(d.get("Instructions Executed", "0"))
        except ValueError:
            continue
        key = (fn, path, int(r[0]))
        a = agg.setdefault(key, [0, 0, r[1].strip()[:100], d])
        a[0] += s
        a[1] += ins
for f in sorted({k[0] for k in agg}):
    items = [(v[0], v[1], k[1], k[2], v[2]) for k, v in agg.items() if k[0] == f]
    S = sum(i[0] for i in items) or 1
    I = sum(i[1] for i in items) or 1
    print(f"== {f[:110]}\n   samples {S}, warp instructions {I}")
    for s, ins, p, ln, src in sorted(items, reverse=True)[:top]:
        print(f"{100 * s / S:5.1f}% smp {100 * ins / I:5.1f}% ins  {p}:{ln}  {src}")

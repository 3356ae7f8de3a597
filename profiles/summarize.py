#!/usr/bin/env python
"""Summarise ncu --set full reports into markdown (python profiles/summarize.py r01)."""
import csv
import subprocess
import sys
from pathlib import Path

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn. smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU wavefronts %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
]


def raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = Path("gpurun_out") / rnd
    lines = [f"# {rnd} ncu summaries (B200, `ncu --set full --clock-control none --import-source on`)", "",
             "Cold-cache, serialised replays (ncu flushes caches per pass): compare shares, not absolutes.",
             "Reports: `gpurun_out/" + rnd + "/full_cfg*.ncu-rep` (not committed); commands in profiles/README.md.", ""]
    for rep in sorted(src.glob("full_cfg*.ncu-rep")):
        cfg = rep.stem.replace("full_", "")
        for d, u in raw(rep):
            lines.append(f"## {cfg}: `{d['Kernel Name'][:110]}`")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for k, name in KEYS:
                if k in d and d[k] not in ("", "n/a"):
                    lines.append(f"| {name} | {d[k]} {u.get(k, '')} |")
            st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(v.replace(",", ""))
                  for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not k.endswith("not_issued") and v.replace(",", "").isdigit()}
            tot = sum(st.values()) or 1
            top = sorted(st.items(), key=lambda x: -x[1])[:5]
            lines.append("| top stall reasons (share of samples) | " +
                         ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top) + " |")
            lines.append("")
    Path("profiles") .joinpath(f"{rnd}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    traffic_json(src)


# per step DRAM bytes (read + write) of the dominant kernels, from the traffic launch lists;
# the number of steps captured = launches of the step's anchor kernel / its launches per step
ANCHOR = {"cfg2": ("k_rt0_pencil<3>", 1), "cfg3": ("k_hyb_warp", 2), "cfg4": ("k_piola_gemm", 1), "cfg5": ("k_hyb_big", 2)}


def traffic_json(src: Path):
    import json
    out = {}
    for cfg, (anchor, per_step) in ANCHOR.items():
        f = src / f"traffic_{cfg}.csv"
        if not f.exists():
            continue
        rows = [r for r in csv.reader(f.read_text().splitlines()) if r]
        hdr = next((r for r in rows if "Kernel Name" in r), None)
        if hdr is None:
            continue
        tot, launches = 0.0, set()
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows:
            if len(r) != len(hdr) or r is hdr:
                continue
            d = dict(zip(hdr, r))
            if cfg == "cfg2" and "<3>" not in d["Kernel Name"]:  # the per-config block's 2D launches
                continue
            if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
            if anchor in d["Kernel Name"]:
                launches.add(d["ID"])
        if launches:
            out[cfg] = tot / (len(launches) / per_step)
    if out:  # merged into the committed per-config sums (configs not captured this time keep theirs)
        tf = Path("profiles").joinpath("ncu_traffic.json")
        old = json.loads(tf.read_text()) if tf.exists() else {}
        old.update(out)
        tf.write_text(json.dumps(old, indent=1) + "\n")


if __name__ == "__main__":
    main()

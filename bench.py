#!/usr/bin/env python
"""Benchmark of the element-local hybridization hot path (BASELINE.json metric:
elements/s of hybridization = assemble + eliminate + scatter).

Default workload: BASELINE config 2 (3D unit-cube 64^3 hexes, RT_0, alpha/beta
log-uniform in [1e-2, 1e2], f_hat uniform [-1, 1]); --config picks another.
One "step" = one hybridize of the whole mesh: element assembly, structured
element solve (with its fail-safe exact path) and deterministic CSR scatter of
H and g, inputs resident in HBM.  Inputs are the SURVEY.md §8(d) stream (the
reference's Xorshift, seed 1000 + config id: paper_1801_08914_b200/inputs.py),
bit-identical to the parity tests' inputs (tests/test_inputs.py).

At N = 1 the line also carries "configs": every BASELINE config (1-5) timed
the same way in the same run (value, ms/step, roofline fraction with the
boundary-aware b_T flop count of §8(d), cells sent to the exact path).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 2]

Under torchrun (N > 1) every rank hybridizes its own independent replica mesh
(the path shards by cells with no data-path exchange: weak scaling); with
--partition slab the ranks instead split ONE mesh into ghosted z-slabs
(paper_1801_08914_b200/slab.py: strong scaling, value = the mesh's cells / time,
ghost cells not counted).  Timing is the max over ranks.  --impl reference
times the reference's own CPU implementation (oracle/_ref/ref_harness, built
from /root/reference: build_reduction_inputs + hybridize) on the same full
mesh and inputs law with all host threads, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "elements/s of hybridization (assemble+eliminate+scatter), % of fp64/HBM roofline"
UNIT = "elements/s"

# BASELINE.json configs (dims, order, coefficient law, seed 1000 + id): paper_1801_08914_b200/inputs.py
from paper_1801_08914_b200.inputs import CONFIGS, config_inputs  # noqa: E402  (numpy only; no library load)

# --impl reference / cpu_baseline on configs too large for a few minutes of host
# time per step: the reference on a sub-mesh with the SAME element (cell size of
# the full mesh) and coefficient law, elements/s extrapolated by the §8(d) flop
# ratio of the full mesh to the sub-mesh (boundary-aware b_T)
CPU_SUBMESH = {3: (16, 16, 16), 5: (6, 6, 6)}
CPU_PORT_SAMPLE = {4: (3, 3, 3)}  # config 4: no reference (trilinear cells): the oracle's port on a sample


def analytic_shape(dim: int, cells, k: int) -> dict:
    """ncells, n, b_T per cell, m, nnz(H) of a structured mesh (probe P11)."""
    c = list(cells) + [1] * (3 - len(cells))
    dpf = (k + 1) ** (dim - 1)
    n = 2 * dim * dpf + dim * k * dpf
    idx = np.arange(c[0] * c[1] * c[2])
    co = [idx % c[0], (idx // c[0]) % c[1], idx // (c[0] * c[1])]
    nfi = np.zeros(idx.size, dtype=np.int64)
    for a in range(dim):
        nfi += (co[a] > 0).astype(np.int64) + (co[a] + 1 < c[a]).astype(np.int64)
    b = nfi * dpf
    n_int_faces = sum((c[a] - 1) * int(np.prod([c[x] for x in range(dim) if x != a])) for a in range(dim))
    return {"ncells": int(idx.size), "n": n, "dpf": dpf, "b": b, "m": n_int_faces * dpf,
            "nnz_h": int(np.sum(b.astype(np.int64) ** 2) - n_int_faces * dpf * dpf)}


def flops_per_step(cfg: dict, cells=None) -> float:
    """§8(d) algorithmic flops: sum over cells of 2n^3/3 + 4 b_T^3/3 + 2n^2 + 3n^2 (b_T the
    cell's actual multiplier count), + the mapped-cell assembly for config 4."""
    sh = analytic_shape(cfg["dim"], cells or cfg["cells"], cfg["k"])
    n = sh["n"]
    b = sh["b"].astype(np.float64)
    f = float(np.sum(2 * n ** 3 / 3 + 4 * b ** 3 / 3 + 5 * n ** 2))
    if cfg.get("perturb"):
        f += sh["ncells"] * 2 * (n * (n + 1) / 2) * (cfg["k"] + 2) ** 3 * 2
    return f


def bytes_per_step(cfg: dict) -> float:
    """§8(d) compulsory bytes: 16 (alpha, beta) + 8 n (f_hat) per cell [+ 8 vertices x 3 x 8 for
    config 4] + 8 nnz(H) + 8 m."""
    sh = analytic_shape(cfg["dim"], cfg["cells"], cfg["k"])
    by = sh["ncells"] * (16 + 8 * sh["n"]) + 8 * (sh["nnz_h"] + sh["m"])
    if cfg.get("perturb"):
        by += 8 * 3 * 8 * sh["ncells"]
    return float(by)


def config_record(cfg_id: int) -> dict:
    """The workload description both arms print (identical dicts: same config)."""
    cfg = CONFIGS[cfg_id]
    sh = analytic_shape(cfg["dim"], cfg["cells"], cfg["k"])
    return {"workload": cfg["desc"], "cells": sh["ncells"], "order": cfg["k"], "dim": cfg["dim"],
            "nnz_h": sh["nnz_h"], "m": sh["m"], "inputs": f"SURVEY.md §8(d) Xorshift stream, seed {cfg['seed']}"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop = [], 0, False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max = None

    def _run(self):
        while not self.stop:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop = True
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"],
                "samples": len(self.samples)}


def ref_harness_path():
    return ROOT / "oracle" / "_ref" / "ref_harness"


def run_reference(cfg_id: int, reps: int, threads: int, cells=None):
    """The reference (oracle/_ref/ref_harness: build_reduction_inputs + hybridize,
    src/reduction.cpp:200-354) on the config's inputs law; cells = a sub-mesh with
    the full mesh's cell size (CPU_SUBMESH) or None for the full mesh."""
    cfg = CONFIGS[cfg_id]
    kind, lo, hi = cfg["coef"]
    full = list(cfg["cells"])
    cells = list(cells or full)
    cmd = [str(ref_harness_path()), "bench", f"dim={cfg['dim']}", "cells=" + ",".join(map(str, cells)),
           f"k={cfg['k']}", f"coef={kind}:{lo}:{hi}", f"seed={cfg['seed']}", f"reps={reps}", "sc=0", "rec=0"]
    if cells != full:
        cmd.append("h=" + ",".join(repr(1.0 / c) for c in full))
    env = dict(os.environ, HDIVRED_NUM_THREADS=str(threads))
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, check=True).stdout
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def cpu_throughput(cfg_id: int, reps: int, threads: int):
    """(elements/s of the full config, seconds per step, sample note) of the reference at
    `threads` host threads; sub-mesh configs are extrapolated by the §8(d) flop ratio."""
    cfg = CONFIGS[cfg_id]
    sub = CPU_SUBMESH.get(cfg_id)
    recs = run_reference(cfg_id, reps, threads, sub)
    t = float(np.median([r["metric_s"] for r in recs]))
    full_cells = int(np.prod(cfg["cells"]))
    if sub is None:
        return full_cells / t, t, f"full {'x'.join(map(str, cfg['cells']))} mesh, median of {reps}"
    scale = flops_per_step(cfg) / flops_per_step(cfg, sub)
    t_full = t * scale
    note = (f"{'x'.join(map(str, sub))} sub-mesh with the full mesh's cell size (h = 1/{cfg['cells'][0]}), "
            f"{t:.3f} s, extrapolated x{scale:.1f} by the §8(d) flop ratio (boundary-aware b_T) to the full "
            f"{'x'.join(map(str, cfg['cells']))} mesh")
    return full_cells / t_full, t_full, note


def port_sample(cfg_id: int, reps: int = 1):
    """The oracle's port of hybridize (single thread) on a sample; for config 4 the
    only CPU implementation of the path (the reference has affine boxes only,
    SURVEY.md §8(c)), per-element cost extrapolated by the flop ratio."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Oracle

    cfg = CONFIGS[cfg_id]
    cells = CPU_PORT_SAMPLE.get(cfg_id, cfg["cells"])
    kind, lo, hi = cfg["coef"]
    spec = f"{kind}:{lo}:{hi}" + (f";perturb={cfg['perturb']}" if cfg.get("perturb") else "")
    times = []
    for _ in range(reps):
        o = Oracle(cfg["dim"], cells, cfg["k"])
        o.set_h([1.0 / c for c in cfg["cells"]])
        o.gen_inputs(spec, cfg["seed"])
        t0 = time.perf_counter()
        o.run("port_hybridize")
        times.append(time.perf_counter() - t0)
    scale = flops_per_step(cfg) / flops_per_step(cfg, cells)
    note = (f"{'x'.join(map(str, cells))} sample (cell size of the full mesh) of the {cfg['desc'].split(':')[0]} "
            f"workload, oracle port of the reference hybridize incl. the Piola assembly, 1 thread, extrapolated "
            f"x{scale:.1f} by the §8(d) flop ratio to the full mesh")
    return [t * scale for t in times], note


def cpu_baseline(cfg_id: int):
    """Reference on the box's host cores: nproc threads (value) and 1 thread."""
    threads = os.cpu_count() or 1
    cfg = CONFIGS[cfg_id]
    ncells = int(np.prod(cfg["cells"]))
    if cfg.get("perturb"):
        times, note = port_sample(cfg_id, 1)
        return {"value": ncells / times[0], "unit": UNIT, "cores": 1, "kind": "port", "sample": note,
                "cpu_model": cpu_model()}
    if not ref_harness_path().exists():
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                "error": "oracle/_ref/ref_harness not built"}
    v, t, note = cpu_throughput(cfg_id, 3, threads)
    v1, t1, _ = cpu_throughput(cfg_id, 1, 1)
    return {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": note + f"; build_reduction_inputs + hybridize (the metric), HDIVRED_NUM_THREADS={threads}",
            "s_per_step": t, "single_thread": {"value": v1, "s_per_step": t1, "cores": 1},
            "cpu_model": cpu_model(), "nproc": threads}


def kernel_name(cfg: dict) -> str:
    if cfg.get("perturb"):
        return "k_piola_gemm + k_spd_hyb + k_run_sum"
    if cfg["k"] == 0:
        return "k_rt0_pencil<dim> (one pass; the exact-path tail k_rt0_exact returns at once)"
    if cfg["dim"] == 3 and cfg["k"] >= 2:
        return "k_hyb_big<k> x2 colours"
    return "k_hyb_warp x2 colours"


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def reference_arm(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    cfg_id = args.config
    threads = os.cpu_count() or 1
    cfg = CONFIGS[cfg_id]
    base = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY.md §8(d) Xorshift stream, the parity tests' inputs)",
            "config": config_record(cfg_id)}
    if cfg.get("perturb"):  # no reference implementation of mapped cells: the oracle port stands in
        times, note = port_sample(cfg_id, args.warmup + args.steps)
        timed = times[args.warmup:]
        value = int(np.prod(cfg["cells"])) * len(timed) / float(np.sum(timed))
        base.update({"value": value, "ms_per_step": 1e3 * float(np.mean(timed)),
                     "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": note,
                                      "cpu_model": cpu_model()},
                     "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
        print(json.dumps(base))
        return 0
    if not ref_harness_path().exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_harness not built (needs /root/reference at build time)"}))
        return 0
    sub = CPU_SUBMESH.get(cfg_id)
    recs = run_reference(cfg_id, args.warmup + args.steps, threads, sub)
    timed = [r["metric_s"] for r in recs[args.warmup:]]
    scale = 1.0 if sub is None else flops_per_step(cfg) / flops_per_step(cfg, sub)
    t = float(np.sum(timed)) * scale
    value = int(np.prod(cfg["cells"])) * len(timed) / t
    note = (f"full {'x'.join(map(str, cfg['cells']))} mesh" if sub is None else
            f"{'x'.join(map(str, sub))} sub-mesh with the full mesh's cell size, extrapolated x{scale:.1f} by the "
            f"§8(d) flop ratio to the full mesh")
    base.update({
        "value": value, "ms_per_step": 1e3 * t / len(timed),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": note + "; build_reduction_inputs + hybridize per step, HDIVRED_NUM_THREADS="
                         + str(threads), "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    print(json.dumps(base))
    return 0


class Timer:
    """Device time of K steps (W warm-up), L2 flushed before each step, CUDA events
    on the library's stream; the step replayed from a CUDA graph when it captures."""

    def __init__(self, torch, stream, flush, use_graph: bool):
        self.torch, self.stream, self.flush, self.use_graph = torch, stream, flush, use_graph

    def run(self, step, check, steps: int, warmup: int, clocks=None):
        torch = self.torch
        for _ in range(warmup):
            step()
        check()
        torch.cuda.synchronize()
        graph = None
        if self.use_graph:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    step()
                g.replay()
                torch.cuda.synchronize()
                check()
                graph = g
            except Exception:
                graph = None
                torch.cuda.synchronize()
        fn = graph.replay if graph is not None else step
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        torch.cuda.synchronize()
        for i in range(steps):
            self.flush.fill_(float(i))
            ev0[i].record(self.stream)
            fn()
            ev1[i].record(self.stream)
        torch.cuda.synchronize()
        check()
        return [a.elapsed_time(b) for a, b in zip(ev0, ev1)], graph is not None


def roofline_for(cfg: dict, ms: float, hbm_peak: float, fp64: tuple) -> dict:
    """Roofline of one config's step: HBM (k = 0) or fp64 (k >= 1) bound, with the
    §8(d) algorithmic bytes / boundary-aware flops; fp64 fractions against both the
    DFMA and the DMMA (fp64 tensor core) peaks measured in this run."""
    by = bytes_per_step(cfg)
    fl = flops_per_step(cfg)
    hbm = {"bound": "hbm", "achieved": by / (ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
           "algorithmic_bytes_per_step": by}
    hbm["frac"] = hbm["achieved"] / hbm_peak
    dfma, dmma = fp64
    ach = fl / (ms * 1e-3) / 1e12
    f64 = {"bound": "fp64", "achieved": ach, "peak": dfma, "unit": "TFLOP/s", "frac": ach / dfma,
           "peak_dmma": dmma, "frac_dmma": ach / dmma if dmma else None, "flops_per_step": fl,
           "flops_model": "§8(d): sum over cells of 2n^3/3 + 4 b_T^3/3 + 5 n^2 (b_T = the cell's multipliers)"
                          + (" + Piola assembly" if cfg.get("perturb") else "")}
    if cfg["k"] == 0:
        hbm["fp64"] = f64
        return hbm
    f64["hbm"] = hbm
    return f64


# the stages each BASELINE config names beside hybridization (BASELINE.json configs)
CONFIG_STAGES = {1: ("recover", "spmv"), 2: ("condense", "spmv"), 3: ("condense", "recover", "spmv"), 4: ("spmv",),
                 5: ("recover", "spmv")}


def stage_case(hd, torch, sp, stage: str, a_d, b_d, f_d):
    """One call of a stage on device-resident inputs and its SURVEY.md §8(d) cost model:
    (run, flops, bytes, units, metric, objects to keep alive)."""
    n, nc, m = sp.n, sp.ncells, sp.m
    nint = sp.info["interior_dofs_per_cell"]
    nb = n - nint
    lib = hd._lib()
    if stage == "condense":
        cop = sp.static_condense(a_d, b_d, f_d)

        def run():
            st = lib.hdr_static_condense_fe_into(cop._h, a_d.data_ptr(), b_d.data_ptr(), f_d.data_ptr(), 1)
            assert st == 0, hd._capi.last_error()
        flops = nc * (2 * (nint ** 3 / 3 + nint ** 2 * nb + nint * nb ** 2) + 2 * (nint ** 2 + nint * nb) + 3 * n ** 2)
        byts = nc * (16 + 8 * n) + 8 * (sp.info["nnz_s"] + sp.info["n_s"])
        return run, flops, byts, nc, "elements/s of static condensation (assemble+condense+scatter)", (cop,)
    op = sp.hybridize(a_d, b_d, f_d)
    if stage == "recover":
        lam = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, m)).cuda()

        def run():
            op.recover(lam, f_d)
        flops = nc * (2 * n ** 3 / 3 + 4 * n ** 2)
        byts = nc * (16 + 16 * n) + 8 * m
        return run, flops, byts, nc, "elements/s of hybrid recovery (x_hat = A^-1 (f - C^T lambda), averaged x)", (op, lam)
    x = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, m)).cuda()
    nnz = sp.info["nnz_h"]

    def run():
        op.spmv(x)
    return run, 2 * nnz, 12 * nnz + 8 * (m + 1) + 16 * m, m, "rows/s of SpMV with H (reference row-sum order)", (op, x)


def stage_roofline(stage: str, ms: float, flops: float, byts: float, hbm_peak: float, fp64_peak: float) -> dict:
    bw = byts / (ms * 1e-3) / 1e9
    fl = flops / (ms * 1e-3) / 1e12
    hbm_frac, fp_frac = bw / hbm_peak, fl / fp64_peak
    roof = ({"bound": "hbm", "achieved": bw, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_frac, "traffic": None}
            if hbm_frac >= fp_frac or stage == "spmv" else
            {"bound": "fp64", "achieved": fl, "peak": fp64_peak, "unit": "TFLOP/s", "frac": fp_frac, "traffic": None})
    roof.update({"algorithmic_bytes_per_step": byts, "algorithmic_flops_per_step": flops})
    return roof


def measure_config(hd, torch, timer, cfg_id: int, steps: int, warmup: int, hbm_peak: float, fp64: tuple,
                   seed=None) -> dict:
    """One BASELINE config timed like the headline (device-resident inputs)."""
    cfg = CONFIGS[cfg_id]
    alpha, beta, f_hat, verts = config_inputs(cfg_id, seed)
    sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    if verts is not None:
        sp.set_vertices(verts)
    sp.set_stream(timer.stream.cuda_stream)
    a_d, b_d, f_d = (torch.from_numpy(x).cuda() for x in (alpha, beta, f_hat))
    op = sp.hybridize(a_d, b_d, f_d)
    exact = op.exact_cells()
    l0 = hd.launch_count()
    op.enqueue(a_d, b_d, f_d)
    op.check()
    per_step = hd.launch_count() - l0
    ms_list, graphed = timer.run(lambda: op.enqueue(a_d, b_d, f_d), op.check, steps, warmup)
    ms = float(np.mean(ms_list))
    rec = {"workload": cfg["desc"], "value": sp.ncells / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
           "roofline": roofline_for(cfg, ms, hbm_peak, fp64), "exact_cells": exact,
           "gpu_launches_per_step": per_step, "cuda_graph": graphed}
    # the other stages BASELINE names for this config, timed the same way (fewer steps)
    rec["stages"] = {}
    for stage in CONFIG_STAGES.get(cfg_id, ()):
        run, flops, byts, units, _metric, keep = stage_case(hd, torch, sp, stage, a_d, b_d, f_d)
        # the stage calls return a status (they synchronise): launched directly, not graph-captured
        s_ms, s_graph = Timer(torch, timer.stream, timer.flush, False).run(run, lambda: None, max(3, steps // 2), 2)
        s_ms = float(np.mean(s_ms))
        rec["stages"][stage] = {"ms_per_step": s_ms, "value": units / (s_ms * 1e-3),
                                "unit": "rows/s" if stage == "spmv" else UNIT,
                                "roofline": stage_roofline(stage, s_ms, flops, byts, hbm_peak, fp64[0]),
                                "cuda_graph": s_graph}
        del run, keep
    del op, sp
    torch.cuda.synchronize()
    return rec


def ours(args):
    import torch

    world, rank, local = dist_setup()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_1801_08914_b200 as hd
    from paper_1801_08914_b200 import dist as hdist

    cfg = CONFIGS[args.config]
    slab_plan = None
    verts = None
    if args.partition == "slab":
        # one mesh over the ranks: each hybridizes its ghosted z-slab (slab.py), no exchange
        from paper_1801_08914_b200 import slab
        if cfg["dim"] != 3 or cfg.get("perturb"):
            raise SystemExit("--partition slab: affine 3D configs")
        slab_plan = slab.SlabPlan(cfg["cells"], cfg["k"], world, rank)
        alpha, beta, f_hat, _ = config_inputs(args.config)  # the global inputs, identical on every rank
        n_loc = f_hat.size // int(np.prod(cfg["cells"]))
        alpha, beta, f_hat = (np.ascontiguousarray(x) for x in slab_plan.inputs(alpha, beta, f_hat, n_loc))
        sp = hd.Space(3, slab_plan.sub_cells, cfg["k"], sizes=slab_plan.sizes)
    else:
        # rank 0 times exactly the parity-tested stream; other replicas reseed
        seed = cfg["seed"] if rank == 0 else hdist.replica_seed(cfg["seed"], rank)
        alpha, beta, f_hat, verts = config_inputs(args.config, seed)
        sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    if verts is not None:
        sp.set_vertices(verts)
    stream = torch.cuda.Stream()  # one non-default stream for the library, the events and the flush
    torch.cuda.set_stream(stream)
    sp.set_stream(stream.cuda_stream)
    a_d, b_d, f_d = (torch.from_numpy(x).cuda() for x in (alpha, beta, f_hat))
    op = sp.hybridize(a_d, b_d, f_d)
    exact_cells = op.exact_cells()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MiB > 126 MB L2
    timer = Timer(torch, stream, flush, not args.no_graph)

    barrier = hdist.barrier
    l0 = hd.launch_count()
    op.enqueue(a_d, b_d, f_d)
    op.check()
    launches_per_step = hd.launch_count() - l0

    # ---- value: inputs resident in HBM, L2 flushed between steps, CUDA events per step
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        step_ms, graphed = timer.run(lambda: op.enqueue(a_d, b_d, f_d), op.check, args.steps, args.warmup)
    barrier()
    launches = launches_per_step * args.steps
    total_ms = hdist.reduce_max(float(np.sum(step_ms)))  # device time, max over ranks
    ncells = sp.ncells
    # units of the whole job: replicas process world meshes; slabs one mesh (ghost cells not counted)
    job_cells = int(np.prod(cfg["cells"])) if slab_plan is not None else ncells * world
    value = job_cells * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    # ---- e2e: the public pipelined batch call (hdr_hybridize_fe_batch) from pinned
    # host buffers: every step uploads its alpha / beta / f_hat, runs the kernels
    # and downloads its H values and g; consecutive steps overlap on three streams
    e2e = None
    if not args.no_e2e:
        pa, pb, pf = (torch.from_numpy(x).pin_memory() for x in (alpha, beta, f_hat))
        h_out = torch.empty(sp.info["nnz_h"], dtype=torch.float64).pin_memory()
        g_out = torch.empty(sp.m, dtype=torch.float64).pin_memory()

        def batch(k):
            sp.hybridize_batch([pa] * k, [pb] * k, [pf] * k, [h_out] * k, [g_out] * k)

        batch(max(2, args.warmup))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        batch(args.steps)
        e1.record(stream)  # the space's stream is ordered after the last download
        torch.cuda.synchronize()
        e2e_ms = hdist.reduce_max(float(e0.elapsed_time(e1)))
        e2e = {"value": job_cells * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": 8 * (2 * ncells + sp.broken_ndofs),
               "d2h_bytes_per_step": 8 * (sp.info["nnz_h"] + sp.m),
               "note": "hdr_hybridize_fe_batch over the K timed steps: pinned host alpha/beta/f_hat in, H values + g "
                       "out per step, uploads / kernels / downloads of consecutive steps overlapped on three streams; "
                       "CSR pattern copied once per mesh"}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (the fused hybridize kernels of the step)
    peak, peak_kind = load_peaks()
    dfma, _ = hd.measure_fp64_peak()
    dmma, _ = hd.measure_dmma_peak()
    roof = roofline_for(cfg, ms_per_step, peak, (dfma, dmma)) if slab_plan is None else {
        "bound": "n/a (slab partition)", "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None}
    roof["peak_source"] = (f"HBM: {peak_kind} (MEASURED_PEAKS.json hbm_gbs); fp64: DFMA / DMMA m8n8k4 chains "
                           "measured in this run (hdr_measure_fp64_peak / hdr_measure_dmma_peak)")
    roof["kernel"] = kernel_name(cfg)
    tf = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(tf.read_text()).get(f"cfg{args.config}") if tf.exists() else None
    roof["traffic"] = traffic
    roof["traffic_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum of the step's kernels from the committed "
                              "ncu capture (profiles/ncu_traffic.json), not measured in this run")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if slab_plan is not None else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY.md §8(d) Xorshift stream, the parity tests' inputs)",
        "config": config_record(args.config),
        "setup": {"parallelism": (f"z-slabs x{world} of one mesh (ghosted sub-meshes, no exchange)" if slab_plan is not None
                                  else f"replicas x{world} (cells shard; no exchange)"),
                  "l2": "flushed between steps (512 MiB write); inputs resident in HBM",
                  "cuda_graph": graphed, "exact_cells": exact_cells},
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    # every BASELINE config in the same run (N = 1): the north-star config 5 among them
    if world == 1 and not args.no_configs and slab_plan is None:
        line["configs"] = {}
        for cid in sorted(CONFIGS):
            line["configs"][str(cid)] = measure_config(hd, torch, timer, cid, args.steps, args.warmup, peak,
                                                       (dfma, dmma))
    if world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config)
        except Exception as exc:  # never hide a failure: report it
            line["cpu_baseline"] = {"value": None, "error": str(exc)}
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def stage_bench(args):
    """Timing of the other in-scope stages of the path (SURVEY.md §8(d) "other
    stages"): static condensation, hybrid recovery, SpMV with H.  Device-resident
    inputs, CUDA events on the library's stream, L2 flushed between steps;
    roofline from the §8(d) cost models."""
    import torch
    import ctypes

    import paper_1801_08914_b200 as hd

    cfg = CONFIGS[args.config]
    alpha, beta, f_hat, verts = config_inputs(args.config)
    sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    if verts is not None:
        sp.set_vertices(verts)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sp.set_stream(stream.cuda_stream)
    a_d, b_d, f_d = (torch.from_numpy(x).cuda() for x in (alpha, beta, f_hat))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    run, flops, byts, units, metric, _keep = stage_case(hd, torch, sp, args.stage, a_d, b_d, f_d)
    nc, m = sp.ncells, sp.m
    # timed like the headline (L2 flushed before each step, CUDA events on the library's
    # stream), launched directly through the public call
    run()
    torch.cuda.synchronize()
    l0 = hd.launch_count()
    run()
    torch.cuda.synchronize()
    per_step = hd.launch_count() - l0
    timer = Timer(torch, stream, flush, False)  # the stage calls return a status (they synchronise): no graph
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms_list, graphed = timer.run(run, lambda: None, args.steps, args.warmup)
    launches = per_step * args.steps
    ms = float(np.mean(ms_list))
    peak, kind = load_peaks()
    tfl, _ = hd.measure_fp64_peak()
    roof = stage_roofline(args.stage, ms, flops, byts, peak, tfl)
    print(json.dumps({"metric": metric, "value": units / (ms * 1e-3), "unit": "rows/s" if args.stage == "spmv" else UNIT,
                      "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": {"workload": cfg["desc"], "stage": args.stage,
                                                      "l2": "flushed between steps", "cuda_graph": graphed},
                      "roofline": roof, "gpu_launches": launches, "clocks": clk.summary()}))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--partition", default="replica", choices=["replica", "slab"],
                    help="N > 1: independent replica meshes (weak scaling) or z-slabs of one mesh (strong scaling)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config block (all BASELINE configs)")
    ap.add_argument("--fp64", action="store_true", help="also report the fp64 roofline for k = 0")
    ap.add_argument("--no-graph", action="store_true", help="launch the step directly instead of replaying a CUDA graph")
    ap.add_argument("--stage", default="hybridize", choices=["hybridize", "condense", "recover", "spmv"],
                    help="time another stage of the path (not the headline metric)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    if args.stage != "hybridize":
        return stage_bench(args)
    return ours(args)


if __name__ == "__main__":
    sys.exit(main())

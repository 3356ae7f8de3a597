#!/usr/bin/env python
"""Benchmark of the element-local hybridization hot path (BASELINE.json metric:
elements/s of hybridization = assemble + eliminate + scatter).

Default workload: BASELINE config 2 (3D unit-cube 64^3 hexes, RT_0, alpha/beta
log-uniform in [1e-2, 1e2], f_hat uniform [-1, 1]); --config picks another.
One "step" = one hybridize of the whole mesh: element assembly, structured
element solve and deterministic CSR scatter of H and g, inputs resident in HBM.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 2]

Under torchrun (N > 1) every rank hybridizes its own independent replica mesh
(the path shards by cells with no data-path exchange: weak scaling); with
--partition slab the ranks instead split ONE mesh into ghosted z-slabs
(paper_1801_08914_b200/slab.py: strong scaling, value = the mesh's cells / time,
ghost cells not counted).  Timing is the max over ranks.  --impl reference times the reference's own CPU
implementation (oracle/_ref/ref_harness, built from /root/reference) on a
bounded sample of the same workload, on rank 0 only.
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

# BASELINE.json configs
CONFIGS = {
    1: dict(dim=2, cells=(64, 64), k=0, coef=("uniform", 1.0, 1.0), seed=1001,
            desc="cfg1: 2D unit-square 64x64 quads, RT_0, alpha=beta=1"),
    2: dict(dim=3, cells=(64, 64, 64), k=0, coef=("logu", 1e-2, 1e2), seed=1002,
            desc="cfg2: 3D unit-cube 64^3 hexes (262,144 elems), RT_0, alpha,beta log-uniform [1e-2,1e2]"),
    3: dict(dim=3, cells=(48, 48, 48), k=1, coef=("logu", 1e-2, 1e2), seed=1003,
            desc="cfg3: 3D unit-cube 48^3 hexes (110,592 elems), RT_1, alpha,beta log-uniform [1e-2,1e2]"),
    4: dict(dim=3, cells=(24, 24, 24), k=2, coef=("logu", 1e-3, 1e3), seed=1004, perturb=0.2,
            desc="cfg4: 3D 24^3 perturbed trilinear hexes (13,824 elems, interior vertices moved U[-0.2h,0.2h]), "
                 "RT_2 (Piola), alpha,beta log-uniform [1e-3,1e3]"),
    5: dict(dim=3, cells=(32, 32, 32), k=3, coef=("checker", 1e-2, 1e2), seed=1005,
            desc="cfg5: 3D unit-cube 32^3 hexes (32,768 elems), RT_3, 4^3 checkerboard sigma_t in {1e-2,1e2}"),
}
# bounded CPU samples of each workload for the reference / cpu_baseline legs
CPU_SAMPLE = {1: (2, (64, 64)), 2: (3, (32, 32, 32)), 3: (3, (16, 16, 16)), 4: (3, (3, 3, 3)), 5: (3, (4, 4, 4))}


def make_inputs(cfg: dict, seed: int):
    """Seeded synthetic inputs with the workload's distributions (host numpy)."""
    rng = np.random.default_rng(seed)
    cells = cfg["cells"]
    nc = int(np.prod(cells))
    kind, lo, hi = cfg["coef"]
    if kind == "uniform":
        alpha, beta = np.full(nc, lo), np.full(nc, hi)
    elif kind == "logu":
        alpha = np.exp(rng.uniform(np.log(lo), np.log(hi), nc))
        beta = np.exp(rng.uniform(np.log(lo), np.log(hi), nc))
    else:  # checkerboard: alpha_ref = 1 (divdiv), beta_ref = 1/(3 sigma_t) (mass), SURVEY.md §8(d)
        idx = np.arange(nc)
        co = [idx % cells[0], (idx // cells[0]) % cells[1], idx // (cells[0] * cells[1])]
        reg = sum(np.floor(4.0 * (co[a] + 0.5) / cells[a]).astype(np.int64) for a in range(cfg["dim"]))
        sigma = np.where(reg % 2 == 0, lo, hi)
        alpha, beta = np.ones(nc), 1.0 / (3.0 * sigma)
    dpf = (cfg["k"] + 1) ** (cfg["dim"] - 1)
    n = 2 * cfg["dim"] * dpf + cfg["dim"] * cfg["k"] * dpf
    f_hat = rng.uniform(-1.0, 1.0, nc * n)
    return alpha, beta, f_hat


def make_vertices(cfg: dict, seed: int):
    """Config 4 geometry: unit-cube grid, every interior vertex coordinate moved by
    U[-f h, f h] (boundary vertices fixed), vertices lexicographic x fastest."""
    cells = cfg["cells"]
    h = [1.0 / c for c in cells]
    g = np.stack(np.meshgrid(*[np.arange(c + 1) * hh for c, hh in zip(cells, h)], indexing="ij"), -1)
    g = g.transpose(2, 1, 0, 3).copy()  # (z, y, x, coord)
    rng = np.random.default_rng(seed + 17)
    inner = (slice(1, -1),) * 3
    f = cfg["perturb"]
    g[inner] += rng.uniform(-f, f, g[inner].shape) * np.array(h)
    return g.reshape(-1, 3)


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


def run_reference_sample(cfg_id: int, reps: int, threads: int):
    """Times the reference (oracle/_ref/ref_harness: build_reduction_inputs +
    hybridize, src/reduction.cpp:200-354) on the bounded sample of the workload."""
    cfg = CONFIGS[cfg_id]
    dim, cells = CPU_SAMPLE[cfg_id]
    kind, lo, hi = cfg["coef"]
    coef = f"{kind}:{lo}:{hi}"
    cmd = [str(ref_harness_path()), "bench", f"dim={dim}", "cells=" + ",".join(map(str, cells)), f"k={cfg['k']}",
           f"coef={coef}", f"seed={cfg['seed']}", f"reps={reps}", "sc=0", "rec=0"]
    env = dict(os.environ, HDIVRED_NUM_THREADS=str(threads))
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, check=True).stdout
    recs = [json.loads(line) for line in out.splitlines() if line.startswith("{")]
    ncells = int(np.prod(cells))
    sample = f"{'x'.join(map(str, cells))} mesh ({ncells} cells) of the {cfg['desc'].split(':')[0]} workload, same element and coefficient law"
    return recs, ncells, sample


def port_sample(cfg_id: int, reps: int = 1):
    """The oracle's port of hybridize (single thread) on the bounded sample; for
    config 4 the only CPU implementation of the path (the reference has affine
    boxes only)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Oracle

    cfg = CONFIGS[cfg_id]
    dim, cells = CPU_SAMPLE[cfg_id]
    kind, lo, hi = cfg["coef"]
    spec = f"{kind}:{lo}:{hi}" + (f";perturb={cfg['perturb']}" if cfg.get("perturb") else "")
    times = []
    for _ in range(reps):
        o = Oracle(dim, cells, cfg["k"])
        o.gen_inputs(spec, cfg["seed"])
        t0 = time.perf_counter()
        o.run("port_hybridize")
        times.append(time.perf_counter() - t0)
    sample = (f"{'x'.join(map(str, cells))} mesh ({int(np.prod(cells))} cells) of the {cfg['desc'].split(':')[0]} "
              f"workload, oracle port of the reference hybridize (element assembly included)")
    return times, int(np.prod(cells)), sample


def cpu_baseline(cfg_id: int):
    threads = os.cpu_count() or 1
    if CONFIGS[cfg_id].get("perturb"):
        times, ncells, sample = port_sample(cfg_id, 1)
        return {"value": ncells / times[0], "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
    if ref_harness_path().exists():
        recs, ncells, sample = run_reference_sample(cfg_id, 3, threads)
        t = float(np.median([r["metric_s"] for r in recs]))
        return {"value": ncells / t, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": sample + "; build_reduction_inputs + hybridize, median of 3, HDIVRED_NUM_THREADS=" + str(threads)}
    # the oracle's port of the reference algorithm (single thread)
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Oracle

    dim, cells = CPU_SAMPLE[cfg_id]
    kind, lo, hi = CONFIGS[cfg_id]["coef"]
    o = Oracle(dim, cells, CONFIGS[cfg_id]["k"])
    o.gen_inputs(f"{kind}:{lo}:{hi}", CONFIGS[cfg_id]["seed"])
    t0 = time.perf_counter()
    o.run("port_hybridize")
    t = time.perf_counter() - t0
    return {"value": int(np.prod(cells)) / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{'x'.join(map(str, cells))} mesh, oracle port of hybridize (reference build unavailable)"}


def kernel_name(cfg: dict) -> str:
    if cfg.get("perturb"):
        return "k_piola_gemm + k_spd_hyb + k_run_sum"
    if cfg["k"] == 0:
        return "k_rt0_brick<dim,0> + k_rt0_brick<dim,1> (colour passes; k_rt0_cell below the brick size)"
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
    if cfg.get("perturb"):  # no reference implementation of mapped cells: the oracle port stands in
        times, ncells, sample = port_sample(cfg_id, args.warmup + args.steps)
        timed = times[args.warmup:]
        value = ncells * len(timed) / float(np.sum(timed))
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(timed)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "sample": sample, "threads": 1},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return 0
    if not ref_harness_path().exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_harness not built (needs /root/reference at build time)"}))
        return 0
    recs, ncells, sample = run_reference_sample(cfg_id, args.warmup + args.steps, threads)
    timed = recs[args.warmup:]
    t = float(np.sum([r["metric_s"] for r in timed]))
    value = ncells * len(timed) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t / len(timed), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "sample": sample, "threads": threads},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample + "; build_reduction_inputs + hybridize per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


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
    if args.partition == "slab":
        # one mesh over the ranks: each hybridizes its ghosted z-slab (slab.py), no exchange
        from paper_1801_08914_b200 import slab
        if cfg["dim"] != 3 or cfg.get("perturb"):
            raise SystemExit("--partition slab: affine 3D configs")
        slab_plan = slab.SlabPlan(cfg["cells"], cfg["k"], world, rank)
        alpha, beta, f_hat = make_inputs(cfg, cfg["seed"])  # the global inputs, identical on every rank
        n_loc = f_hat.size // int(np.prod(cfg["cells"]))
        alpha, beta, f_hat = (np.ascontiguousarray(x) for x in slab_plan.inputs(alpha, beta, f_hat, n_loc))
        sp = hd.Space(3, slab_plan.sub_cells, cfg["k"], sizes=slab_plan.sizes)
    else:
        alpha, beta, f_hat = make_inputs(cfg, hdist.replica_seed(cfg["seed"], rank))
        sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    if cfg.get("perturb"):
        sp.set_vertices(make_vertices(cfg, hdist.replica_seed(cfg["seed"], rank)))
    stream = torch.cuda.Stream()  # one non-default stream for the library, the events and the flush
    torch.cuda.set_stream(stream)
    sp.set_stream(stream.cuda_stream)
    a_d, b_d, f_d = (torch.from_numpy(x).cuda() for x in (alpha, beta, f_hat))
    op = sp.hybridize(a_d, b_d, f_d)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MiB > 126 MB L2

    barrier = hdist.barrier

    # warmup (device-resident inputs)
    for i in range(args.warmup):
        op.enqueue(a_d, b_d, f_d)
    op.check()
    torch.cuda.synchronize()

    # the step's launches captured once into a CUDA graph (launch-bound small
    # configs); paths that synchronise inside (mapped geometry) run directly
    graph = None
    if not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                op.enqueue(a_d, b_d, f_d)
            g.replay()
            torch.cuda.synchronize()
            op.check()
            graph = g
        except Exception:
            graph = None
            torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            op.enqueue(a_d, b_d, f_d)

    # ---- value: inputs resident in HBM, L2 flushed between steps, CUDA events per step
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if graph is not None:
        l0 = hd.launch_count()
        op.enqueue(a_d, b_d, f_d)
        torch.cuda.synchronize()
        launches_per_step = hd.launch_count() - l0
    launches0 = hd.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            ev0[i].record(stream)
            step()
            ev1[i].record(stream)
        torch.cuda.synchronize()
    barrier()
    op.check()
    launches = hd.launch_count() - launches0
    if graph is not None:  # replays do not pass through the library's launch counter
        launches = launches_per_step * args.steps
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
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

    # ---- roofline of the dominant kernel (the fused hybridize kernel; one launch per colour)
    peak, peak_kind = load_peaks()
    alg_bytes = 8 * (2 * ncells + sp.broken_ndofs + sp.info["nnz_h"] + sp.m)
    if cfg.get("perturb"):
        alg_bytes += 8 * 3 * 8 * ncells  # the cell's vertex coordinates
    achieved = alg_bytes / (ms_per_step * 1e-3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(f"cfg{args.config}")
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
            "algorithmic_bytes_per_step": alg_bytes,
            "kernel": kernel_name(cfg)}
    if cfg["k"] > 0 or args.fp64:
        tfl, _ = hd.measure_fp64_peak()
        n = sp.n
        b = sp.info["dofs_per_face"] * 2 * cfg["dim"]
        flop_cell = 2 * n ** 3 / 3 + 4 * b ** 3 / 3 + 2 * n ** 2 + 3 * n ** 2
        if cfg.get("perturb"):  # + mapped-element assembly (mass and divdiv, symmetric halves)
            flop_cell += 2 * (n * (n + 1) / 2) * (cfg["k"] + 2) ** 3 * 2
        fl = flop_cell * ncells / (ms_per_step * 1e-3) / 1e12
        roof_fp64 = {"bound": "fp64", "achieved": fl, "peak": tfl, "unit": "TFLOP/s", "frac": fl / tfl,
                     "peak_source": "measured DFMA (hdr_measure_fp64_peak)", "flops_per_cell": flop_cell}
        if cfg["k"] > 0:
            roof, roof_fp64["hbm"] = roof_fp64, roof
        else:
            roof["fp64"] = roof_fp64

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if slab_plan is not None else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "cells": ncells, "order": cfg["k"], "dim": cfg["dim"],
                   "nnz_h": sp.info["nnz_h"], "m": sp.m,
                   "parallelism": (f"z-slabs x{world} of one mesh (ghosted sub-meshes, no exchange)" if slab_plan is not None
                                   else f"replicas x{world} (cells shard; no exchange)"),
                   "l2": "flushed between steps (512 MiB write); inputs resident in HBM",
                   "cuda_graph": graph is not None},
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
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
    alpha, beta, f_hat = make_inputs(cfg, cfg["seed"])
    sp = hd.Space(cfg["dim"], cfg["cells"], cfg["k"])
    if cfg.get("perturb"):
        sp.set_vertices(make_vertices(cfg, cfg["seed"]))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sp.set_stream(stream.cuda_stream)
    a_d, b_d, f_d = (torch.from_numpy(x).cuda() for x in (alpha, beta, f_hat))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    n, nc, m = sp.n, sp.ncells, sp.m
    dpf = sp.info["dofs_per_face"]
    nint = sp.info["interior_dofs_per_cell"]
    nb = n - nint
    lib = hd._lib()
    if args.stage == "condense":
        cop = sp.static_condense(a_d, b_d, f_d)

        def run():
            st = lib.hdr_static_condense_fe_into(cop._h, a_d.data_ptr(), b_d.data_ptr(), f_d.data_ptr(), 1)
            assert st == 0, hd._capi.last_error()
        flops = nc * (2 * (nint ** 3 / 3 + nint ** 2 * nb + nint * nb ** 2) + 2 * (nint ** 2 + nint * nb) + 3 * n ** 2)
        byts = nc * (16 + 8 * n) + 8 * (sp.info["nnz_s"] + sp.info["n_s"])
        metric = "elements/s of static condensation (assemble+condense+scatter)"
    elif args.stage == "recover":
        op = sp.hybridize(a_d, b_d, f_d)
        lam = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, m)).cuda()

        def run():
            op.recover(lam, f_d)
        flops = nc * (2 * n ** 3 / 3 + 4 * n ** 2)
        byts = nc * (16 + 16 * n) + 8 * m
        metric = "elements/s of hybrid recovery (x_hat = A^-1 (f - C^T lambda), averaged x)"
    else:  # spmv
        op = sp.hybridize(a_d, b_d, f_d)
        x = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, m)).cuda()
        nnz = sp.info["nnz_h"]

        def run():
            op.spmv(x)
        flops = 2 * nnz
        byts = 12 * nnz + 8 * (m + 1) + 16 * m
        metric = "rows/s of SpMV with H (reference row-sum order)"
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = hd.launch_count()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            ev0[i].record(stream)
            run()
            ev1[i].record(stream)
        torch.cuda.synchronize()
    launches = hd.launch_count() - l0
    ms = float(np.mean([a.elapsed_time(b) for a, b in zip(ev0, ev1)]))
    units = m if args.stage == "spmv" else nc
    peak, kind = load_peaks()
    tfl, _ = hd.measure_fp64_peak()
    bw = byts / (ms * 1e-3) / 1e9
    fl = flops / (ms * 1e-3) / 1e12
    hbm_frac, fp_frac = bw / peak, fl / tfl
    roof = ({"bound": "hbm", "achieved": bw, "peak": peak, "unit": "GB/s", "frac": hbm_frac, "traffic": None}
            if hbm_frac >= fp_frac or args.stage == "spmv" else
            {"bound": "fp64", "achieved": fl, "peak": tfl, "unit": "TFLOP/s", "frac": fp_frac, "traffic": None})
    roof.update({"algorithmic_bytes_per_step": byts, "algorithmic_flops_per_step": flops})
    print(json.dumps({"metric": metric, "value": units / (ms * 1e-3), "unit": "rows/s" if args.stage == "spmv" else UNIT,
                      "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": {"workload": cfg["desc"], "stage": args.stage,
                                                      "l2": "flushed between steps"},
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

#!/usr/bin/env python3
"""Benchmark: explicit HLLC shallow-water steps on B200 (BASELINE.json metric
"cell-updates/sec (HLLC SWE, 10M tris) ... % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config channel] [--scale 1.0]

Workload (default): BASELINE.json configs[2] -- the 10M-triangle synthetic
meandering river channel with bathymetry and Manning n = 0.03 on an
unstructured (jittered, randomly renumbered) mesh, 7162 x 716 generator grid =
10,255,984 cells.  A "step" is one explicit Euler step of the whole mesh
(CFL reduction + face fluxes + cell update + friction + clamp), as the
reference's bench harness counts it (bench.hpp:173: cells * steps / wall).

value     K steps with the state resident in HBM (one CUDA graph launch),
          device time (CUDA events on the solver's stream), max over ranks.
e2e       the same K steps through the public C-ABI from pinned HOST buffers:
          upload of the state at value's first timed step (copied out before
          the timed region), the K-step run with its per-step stats
          records copied back, download of the final state -- all inside the
          timed region (the reference run()'s contract, engine.hpp:335-394).
roofline  the dominant kernel's algorithmic bytes per launch (SURVEY.md §8(d):
          face 64 B/edge + 32 B/cell, cell 64 B/edge + 84 B/cell) / its mean
          CUDA-event duration over a profiled pass of the same K steps.
cpu_baseline  the reference itself (oracle/_ref, OpenMP, all host threads) on
          a bounded sample of the same workload, its own phase timers.
--impl reference   the reference CPU implementation alone on the same workload.
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

METRIC = "cell-updates/sec (HLLC SWE, 10M tris)"
UNIT = "cell-updates/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
CONFIG_NOTE = {
    "channel": "BASELINE configs[2]: 10M-triangle meandering channel, bathymetry + Manning n=0.03",
    "sloping_wet_dry": "BASELINE configs[3]: 10M-triangle dam break onto a dry sloping bed, n=0.03",
    "three_mounds_friction": "BASELINE configs[1]: 1M-triangle three-mound dam break, n=0.03",
    "circular_dam_break": "BASELINE configs[0]: ~10k-triangle circular dam break, flat frictionless",
    "weak_square": "BASELINE configs[4]: weak-scaling square water drop",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="channel", choices=list(CONFIG_NOTE))
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--weak-base", type=int, default=2265,
                    help="weak scaling: generator nx at N=1 (default: SURVEY's 2265)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-rebalance", action="store_true",
                    help="N > 1 strong scaling: keep the modelled split (no measured rebalancing)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N > 1: strong = the configured mesh split N ways; weak = BASELINE "
                         "configs[4], the square water drop at ~10.26M cells per GPU")
    return ap.parse_args()


LOCKSTEP_CHECK = os.environ.get("SWE_BENCH_LOCKSTEP_CHECK") == "1"


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.window = None

    def start(self):
        """Start sampling (before the warm-up) and wait for the first sample."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10:
                time.sleep(0.05)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = self.rows
        where = "during the timed region"
        if self.window:
            inside = [r for r in rows if self.window[0] <= r[0] <= self.window[1] + 0.05]
            if inside:
                rows = inside
            else:  # region shorter than the sampling period: nearest samples
                mid = 0.5 * (self.window[0] + self.window[1])
                rows = sorted(rows, key=lambda r: abs(r[0] - mid))[:3]
                where = "nearest samples to a timed region shorter than the 20 ms sampling period"
        rows = [r for _, r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        num = lambda v: v.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(r[0]) for r in rows if num(r[0])]
        mx = [float(r[1]) for r in rows if len(r) > 1 and num(r[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "window": where}


def load_peaks():
    if PEAKS.exists():
        p = json.loads(PEAKS.read_text())
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def build_workload(name, scale, device=None):
    """scenario (host) + build_mesh (on `device` when given: swe_dev_build_mesh,
    bit-identical to the host build)"""
    from paper_1807_00672_b200 import api
    t0 = time.perf_counter()
    sc = api.make_scenario(name, scale=scale, unstructured=True)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=device)
    return sc, mesh, time.perf_counter() - t0


def produce_workload(name, scale, weak_nx=2265):
    """The same inputs from a producer SUBPROCESS (tools/make_workload.py), so
    the process that runs the reference never loads libswe_b200.so."""
    import tempfile
    with tempfile.TemporaryDirectory(prefix="swe_wl_") as d:
        out = Path(d) / "w.npz"
        subprocess.run([sys.executable, str(ROOT / "tools" / "make_workload.py"), "--config", name,
                        "--scale", repr(scale), "--weak-nx", str(weak_nx), "--out", str(out)],
                       check=True)
        with np.load(out) as z:
            return {k: z[k] for k in z.files}


def workload_config(name, n_cells, n_edges, n_boundary, world):
    """identical in both arms (the driver compares the two lines' config)"""
    return {"workload": f"{name} ({CONFIG_NOTE[name]})", "cells": n_cells,
            "edges": n_edges, "boundary_edges": n_boundary,
            "mesh": "unstructured: jittered nodes, random diagonals, random node/cell numbering",
            "l2": ("inputs larger than L2 (state + mesh ~= 300 B/cell >> 126 MB)"
                   if 300 * n_cells > 2 * 126e6 else
                   f"inputs fit in L2 (~{300 * n_cells / 1e6:.0f} MB of state + mesh): "
                   "resident across steps as in any run of this size; not flushed"),
            "step_window": "steps [W, W+K) from the initial state (W = --warmup, at least 3) in "
                           "both arms",
            "parallelism": "single GPU" if world == 1 else f"{world} GPUs"}


REF_MAX_STEPS = 150
HORIZON = 1.7976931348623157e308  # bench.hpp:91 (fixed-step throughput mode)


def reference_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def host_cpu_info():
    """core counts of the host (state the count)"""
    info = {"hardware_concurrency": os.cpu_count(), "affinity_threads": reference_threads()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {k.strip(): v.strip() for k, v in
              (ln.split(":", 1) for ln in out.splitlines() if ":" in ln)}
        info["lscpu_cpus"] = int(kv.get("CPU(s)", 0) or 0)
        cps, sk = int(kv.get("Core(s) per socket", 0) or 0), int(kv.get("Socket(s)", 0) or 0)
        info["lscpu_physical_cores"] = cps * sk if cps and sk else None
        info["lscpu_threads_per_core"] = int(kv.get("Thread(s) per core", 0) or 0) or None
        info["model"] = kv.get("Model name")
    except Exception as e:  # lscpu missing: hardware_concurrency only
        info["lscpu"] = f"unavailable ({type(e).__name__})"
    return info


def reference_window(rm, st, W, K, threads, seq_steps=0):
    """The reference (oracle/_ref, unmodified headers) from the initial state:
    W untimed steps on all threads, then K steps timed by its own phase
    timers (engine.hpp:314-317, as bench.hpp:105-110) with `threads`; with
    seq_steps, also that many steps of the same window on ONE thread."""
    r0 = rm.advance(st["h"], st["qx"], st["qy"], t_end=HORIZON, nsteps=W, threads=threads)
    if r0["rc"] != 0:
        raise RuntimeError(f"reference failed: {r0['error']}")
    at = dict(t=r0["t"], step=r0["step"], clipped_volume=r0["clipped_volume"],
              clip_events=r0["clip_events"])
    r = rm.advance(r0["h"], r0["qx"], r0["qy"], t_end=HORIZON, nsteps=K, threads=threads, **at)
    if r["rc"] != 0:
        raise RuntimeError(f"reference failed: {r['error']}")
    phase_s = r["flux_s"] + r["update_s"]
    out = {"value": rm.n_cells * K / phase_s, "phase_s": phase_s, "steps": K,
           "state": (r["h"], r["qx"], r["qy"]), "dts": r["dts"]}
    if seq_steps:
        q = rm.advance(r0["h"], r0["qx"], r0["qy"], t_end=HORIZON, nsteps=seq_steps, threads=1, **at)
        out["seq_value"] = rm.n_cells * seq_steps / (q["flux_s"] + q["update_s"])
        out["seq_steps"] = seq_steps
    return out


def ref_mesh_of(wl):
    from oracle.pyoracle import RefOracle
    ref = RefOracle()
    t0 = time.perf_counter()
    rm = ref.build_mesh(wl["nodes"], wl["tris"], wl["bed"], wl["manning"])
    return rm, time.perf_counter() - t0


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from oracle.pyoracle import RefOracle
    if not RefOracle.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libswe_ref.so was not built (needs /root/reference)"}))
        return
    wl = (produce_workload("weak_square", 1.0, weak_nx=weak_nx(world)) if args.scaling == "weak"
          else produce_workload(args.config, args.scale))
    rm, build_s = ref_mesh_of(wl)
    threads = reference_threads()
    # bounded sample: ~0.34 s per step at 10M cells on 16 threads, so at most
    # REF_MAX_STEPS timed steps keep the arm within a few minutes for any K
    W, K = max(3, args.warmup), min(args.steps, REF_MAX_STEPS)
    r = reference_window(rm, wl, W, K, threads)
    sample = (f"steps [{W}, {W + K}) of the full {rm.n_cells}-cell workload (the B200 arm's window"
              f"{'' if K == args.steps else ', first ' + str(K) + ' of its ' + str(args.steps) + ' steps'}"
              f"), reference built with -O3 -fopenmp -ffp-contract=off, {threads} OpenMP threads, "
              "its own phase timers; inputs from a producer subprocess, mesh from the reference's "
              "build_mesh")
    out = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * r["phase_s"] / K, "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(cfg_name(args), rm.n_cells, rm.n_edges, rm.n_boundary,
                                     args.gpus),
           "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads,
                            "kind": "reference", "sample": sample, "host": host_cpu_info()},
           "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "setup": {"reference_build_mesh_s": round(build_s, 2)},
           "native_libs": repo_libs_mapped()}
    print(json.dumps(out))


def repo_libs_mapped():
    """shared objects of this repo mapped into this process (/proc/self/maps):
    the reference arm's must be oracle/ libraries only"""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except OSError:
        return None
    root = str(ROOT.resolve())
    libs = {ln.split()[-1] for ln in maps if ln.rstrip().endswith(".so") and root in ln}
    return sorted(str(Path(x).resolve().relative_to(ROOT.resolve())) for x in libs)


def run_b200_dist(args, rank, local, world):
    """N > 1: the mesh split across ranks by RCB (one part per GPU) running as
    LINKED contexts (include/swe_dev.h): the step kernel pushes ghost states
    into the peers' buffers over NVLink (CUDA IPC peer memory) and the CFL
    bound / step outcome goes through device mailboxes, so each rank's run is
    one CUDA graph launch with no host round trip per step
    (paper_1807_00672_b200/dist.py).  strong: the configured mesh; weak: the
    generator resolution scaled by sqrt(N) (N x the cells)."""
    import torch
    import torch.distributed as tdist
    from paper_1807_00672_b200 import api, dist

    dev = "cpu" if LOCKSTEP_CHECK else "cuda"  # the collectives' tensors (gloo / NCCL)
    if args.scaling == "weak":
        # BASELINE configs[4] / SURVEY §8(d) 5: the square water drop at ~10.26M
        # cells per GPU (nx = 2265, 3203, 4530, 6406 for N = 1, 2, 4, 8); every
        # rank builds only its own part from the raw mesh (build_rank_mesh) --
        # the global 82M-cell Mesh would need ~40 GB of host memory per rank
        t0 = time.perf_counter()
        nx = weak_nx(world)
        sc = api.make_scenario("weak_square", weak_nx=nx)
        part = dist.partition_raw(sc.raw, world)  # the drop is wet everywhere: equal counts
        lm = dist.rank_mesh(sc.raw, sc.bed, sc.manning, part, rank)
        mesh = None
        C, E, NB = sc.raw.n_cells, 3 * nx * nx + 2 * nx, 4 * nx
        setup_s = time.perf_counter() - t0
    else:
        scale = args.scale
        sc, mesh, setup_s = build_workload(args.config, scale, device=local)
        C, E, NB = mesh.n_cells, mesh.n_edges, mesh.n_boundary_edges
        # equal work per GPU: cells weighted by the device's own dry-tile skip pattern
        w0 = dist.measured_cost_weights(mesh, sc.state, device=local, parts=world)
        part = dist.partition(mesh, world, w0)
        if not args.no_rebalance:
            t_r = time.perf_counter()
            part, rebalance = rebalance_parts(args, mesh, sc.state, part, w0, rank, local, world,
                                              dev, tdist, dist)
            rebalance["s"] = round(time.perf_counter() - t_r, 2)
            setup_s += rebalance["s"]
        lm = dist.local_mesh(mesh, part, rank)
    if args.scaling == "weak" or args.no_rebalance:
        rebalance = None
    lp = dist.LinkedPart(lm, device=local)
    inf = api.DeviceSolver.info(lp)
    U = inf["graph_unroll"]  # steps per WHILE iteration (graph loop)
    PERSISTENT = bool(inf["persistent"])
    try:
        dist.link_torch(lp)
    except dist.LinkUnavailable as e:  # every rank takes this branch together
        lp.close()
        return run_dist_host_driven(args, rank, local, world, sc, (C, E, NB), part, lm, setup_s,
                                    reason=str(e))
    lp.set_state(sc.state)
    horizon = HORIZON
    W, K = max(3, args.warmup), args.steps

    def advance(target):  # run() segment up to step `target` (collective)
        if LOCKSTEP_CHECK:
            return dist.run_lockstep_ranks(lp, target - lp.clock()[1], t_end=horizon)
        return lp.advance(t_end=horizon, max_steps=target)

    def launch(target):
        if LOCKSTEP_CHECK:
            launch.recs = advance(target)
        else:
            lp.launch(t_end=horizon, max_steps=target)

    def records():
        return launch.recs if LOCKSTEP_CHECK else lp.records()

    # clocks ramp: keep stepping >= 1 s (every rank takes the same decision),
    # then restart from the initial state: the timed window is steps [W, W+K),
    # the reference arm's
    t_w = time.perf_counter()
    steps = 0
    while not LOCKSTEP_CHECK:
        go = torch.tensor([1.0 if time.perf_counter() - t_w < 1.0 else 0.0], device=dev)
        tdist.all_reduce(go, op=tdist.ReduceOp.MAX)
        if go.item() == 0.0:
            break
        steps += 50
        advance(steps)
    lp.set_state(sc.state)
    advance(W)
    steps = W
    skipped0, held0 = lp_skipped(lp), lp_held(lp)
    stream = torch.cuda.ExternalStream(dist_stream(lp), device=local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tdist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local).start() if rank == 0 else None
    w0 = time.time()
    ev0.record(stream)
    launch(steps + K)  # one graph launch per rank, no host sync
    ev1.record(stream)
    torch.cuda.synchronize()
    recs = records()
    if clk:
        clk.mark(w0, time.time())
        clk.stop()
    assert len(recs) == K, f"expected {K} steps, ran {len(recs)}"
    ms = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
    tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
    # dry tiles skipped over the timed steps, summed over ranks
    sk = torch.tensor([float(lp_skipped(lp) - skipped0), float(lp_tiles(lp) * K),
                       float(lp_held(lp) - held0)], device=dev)
    tdist.all_reduce(sk, op=tdist.ReduceOp.SUM)
    skip_frac = float(sk[0].item()) / max(1.0, float(sk[1].item()))
    held_frac = float(sk[2].item()) / max(1.0, float(sk[1].item()))
    ms = float(ms.item())
    # e2e: host state in, the same K steps, owned state back to the host
    # (the state at step W -- the window's start -- is re-formed untimed)
    lp.set_state(sc.state)
    advance(W)
    start = api.FieldState.zeros(C)
    t_start, _ = lp.gather_owned(start)
    gath = [None] * world
    tdist.all_gather_object(gath, (lm.cells[:lm.n_owned], start.h[lm.cells[:lm.n_owned]],
                                   start.qx[lm.cells[:lm.n_owned]], start.qy[lm.cells[:lm.n_owned]]))
    for cells, h, qx, qy in gath:
        start.h[cells], start.qx[cells], start.qy[cells] = h, qx, qy
    tdist.barrier()
    t0 = time.perf_counter()
    lp.set_state(start, t=t_start, step=W)
    advance(W + K)
    got = api.FieldState.zeros(C)
    lp.gather_owned(got)
    e2e_s = torch.tensor([time.perf_counter() - t0], device=dev)
    tdist.all_reduce(e2e_s, op=tdist.ReduceOp.MAX)
    if rank == 0:
        out = {"metric": METRIC, "value": C * K / (ms / 1e3), "unit": UNIT, "n_gpus": world,
               "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
               "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": workload_config(cfg_name(args), C, E, NB, world),
               "decomposition": {
                   "how": f"{world}-way cost-weighted RCB domain decomposition (cells "
                          "of computed tiles weighted "
                          f"{dist.COMPUTED_COST_LARGE if C / world >= dist.LARGE_PART_CELLS else dist.COMPUTED_COST}"
                          "x cells of skipped dry tiles, measured on the device), one "
                          "part per GPU; "
                          "ghost states pushed peer-to-peer by the step kernel, CFL "
                          "bound / outcome through device mailboxes (no host round "
                          "trip per step)",
                   "cells_per_gpu_max": int(np.bincount(part).max()),
                   "cells_per_gpu_min": int(np.bincount(part).min()),
                   "halo_cells_rank0": int(lm.n_cells - lm.n_owned),
                   "rebalance": rebalance},
               "setup": {"setup_s": round(setup_s, 2)},
               "gpu_launches": 3 if PERSISTENT else 2 * U * -(-K // U) + 2,
               "gpu_launches_note": ("per rank: k_set_params, k_gate and one cooperative launch "
                                     "of the persistent step kernel (halo pushed peer-to-peer by "
                                     "the tiles, the exchange run by the last CTA to arrive while "
                                     "the others start the next step's fluxes)" if PERSISTENT else
                                     "per rank: k_set_params + one CUDA-graph launch = k_gate + "
                                     f"a conditional WHILE node of ceil(K/{U}) iterations x {U} x "
                                     "(k_tile with halo push, k_exchange); steps past the stop "
                                     "exit at once"),
               "clocks": clk.summary() if clk else None,
               "roofline": dist_roofline(C, E, K, ms, world, skip_frac, held_frac),
               "e2e": {"value": C * K / float(e2e_s.item()), "unit": UNIT,
                       "h2d_bytes_per_step": 24 * C / K, "d2h_bytes_per_step": (24 * C + 40 * K) / K,
                       "path": "LinkedPart.set_state (host) + advance (K steps, records D2H) + "
                               "gather_owned (host), max over ranks"},
               "step_dt_last": float(recs[-1, 2])}
        if LOCKSTEP_CHECK:
            out = {"lockstep_check": True, "note": "N>1 code path validated on one GPU; "
                   "not a bench value", "records_ok": bool(len(recs) == K), **out}
        print(json.dumps(out))
    tdist.barrier()
    lp.close()
    tdist.destroy_process_group()


def run_dist_host_driven(args, rank, local, world, sc, sizes, part, lm, setup_s, reason):
    """Fallback when peer memory cannot be mapped (CUDA IPC unavailable): the
    host-driven protocol -- halo pack / NCCL send-recv / unpack, CFL bound by
    NCCL all_reduce, one step per round (dist.run_parts + TorchExchange)."""
    import torch
    import torch.distributed as tdist
    from paper_1807_00672_b200 import dist
    ps = dist.PartSolver(lm, device=local)
    ex = dist.TorchExchange(ps)
    ps.set_state(sc.state)
    W, K = max(3, args.warmup), args.steps
    dist.run_parts([ps], ex, W)
    stream = torch.cuda.ExternalStream(dist_stream(ps), device=local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tdist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local).start() if rank == 0 else None
    from paper_1807_00672_b200 import api
    launches0 = api.launch_count()
    w0 = time.time()
    ev0.record(stream)
    recs = dist.run_parts([ps], ex, K)
    ev1.record(stream)
    launches = api.launch_count() - launches0
    torch.cuda.synchronize()
    if clk:
        clk.mark(w0, time.time())
        clk.stop()
    dev = "cpu" if LOCKSTEP_CHECK else "cuda"
    ms = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
    tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
    ms = float(ms.item())
    C, E, NB = sizes
    tdist.barrier()
    t0 = time.perf_counter()
    ps.set_state(sc.state)
    dist.run_parts([ps], ex, K)
    got = api.FieldState.zeros(C)
    ps.gather_owned(got)
    e2e_s = torch.tensor([time.perf_counter() - t0], device=dev)
    tdist.all_reduce(e2e_s, op=tdist.ReduceOp.MAX)
    if rank == 0:
        out = {"metric": METRIC, "value": C * K / (ms / 1e3), "unit": UNIT, "n_gpus": world,
               "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
               "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": workload_config(cfg_name(args), C, E, NB, world),
               "decomposition": {
                   "how": f"{world}-way cost-weighted RCB domain decomposition, host-"
                          "driven exchange (NCCL send/recv + all_reduce per step): "
                          f"linked peer memory unavailable ({reason[:160]})",
                   "cells_per_gpu_max": int(np.bincount(part).max())},
               "setup": {"setup_s": round(setup_s, 2)},
               "gpu_launches": launches,
               "gpu_launches_note": "rank 0, counted by the library: per step halo pack / "
                                    "unpack, k_set_params, k_gate, k_tile, k_finalize (+ NCCL "
                                    "kernels, not counted)",
               "clocks": clk.summary() if clk else None,
               "roofline": dist_roofline(C, E, K, ms, world, 0.0),
               "e2e": {"value": C * K / float(e2e_s.item()), "unit": UNIT,
                       "h2d_bytes_per_step": 24 * C / K, "d2h_bytes_per_step": 24 * C / K,
                       "path": "PartSolver.set_state (host) + K steps + gather_owned (host)"},
               "step_dt_last": float(recs[-1, 1])}
        print(json.dumps(out))
    tdist.barrier()
    ps.close()
    tdist.destroy_process_group()


def _lp_info(lp):
    import ctypes
    v = (ctypes.c_longlong * 16)()
    lp.lib.swe_dev_info(lp.ctx, v, 16)
    return list(v)


def lp_skipped(lp):
    return _lp_info(lp)[11]


def lp_held(lp):
    return _lp_info(lp)[15]


def lp_tiles(lp):
    return _lp_info(lp)[2]


WEAK_BASE = 2265


def weak_nx(world):
    """~10.26M cells per GPU (--weak-base shrinks it for checks)"""
    if WEAK_BASE == 2265:
        return {1: 2265, 2: 3203, 4: 4530, 8: 6406}.get(world, int(round(2265 * world ** 0.5)))
    return int(round(WEAK_BASE * world ** 0.5))


def cfg_name(args):
    return "weak_square" if args.scaling == "weak" else args.config


REBALANCE_ROUNDS = 2


def rebalance_parts(args, mesh, state, part, w0, rank, local, world, dev, tdist, dist):
    """Measured rebalancing of the strong-scaling split (dist.refine_weights):
    every rank times its own part alone on its GPU (unlinked, its own dt), the
    times are all-gathered, the cell weights scaled by each part's time and
    the mesh re-split; after REBALANCE_ROUNDS the split whose slowest part was
    fastest is kept (every rank takes the same decisions from the same
    gathered times).  On one GPU (lockstep check) the ranks' timings contend,
    so the choice there only exercises the code path."""
    import torch
    hist, best = [], None
    w = w0
    for r in range(REBALANCE_ROUNDS + 1):
        mine = dist.part_step_ms(mesh, state, part, rank, device=local, steps=30)
        t = torch.zeros(world, dtype=torch.float64, device=dev)
        t[rank] = mine
        tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
        times = [float(x) for x in t.cpu()]
        hist.append(max(times))
        if best is None or max(times) < best[0]:
            best = (max(times), part, r)
        if r == REBALANCE_ROUNDS:
            break
        w = dist.refine_weights(w, part, times)
        part = dist.partition(mesh, world, w)
    return best[1], {"rounds": REBALANCE_ROUNDS, "slowest_part_ms": hist, "kept_round": best[2]}


def dist_roofline(C, E, K, ms, world, skip_frac, held_frac=0.0):
    """whole-job step roofline of an N-GPU run: SURVEY §8(d) canonical step
    bytes (skipped dry tiles at 40 B/cell, held ones at 16) over the
    max-over-ranks step time, against N x the per-GPU HBM peak"""
    peak, src = load_peaks()
    step = ((1.0 - skip_frac) * (116 * C + 128 * E) + (skip_frac - held_frac) * 40 * C
            + held_frac * 16 * C)
    achieved = step / (ms / K / 1e3) / 1e9
    return {"bound": "hbm", "kernel": "step (all ranks)", "achieved": achieved,
            "peak": world * peak, "unit": "GB/s", "frac": achieved / (world * peak),
            "traffic": None, "peak_source": f"{world} x {src}",
            "skipped_tile_fraction": skip_frac, "held_tile_fraction": held_frac}


def dist_stream(part_solver):
    return part_solver.lib.swe_dev_stream(part_solver.ctx)


def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_1807_00672_b200 import api

    rank, local, world = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    if world > 1 and LOCKSTEP_CHECK:
        # validation of the N>1 path on ONE GPU: every rank on device 0, gloo,
        # barrier-separated lockstep phases (no kernel waits on a concurrently
        # running one); the numbers it prints are not bench values
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        return run_b200_dist(args, rank, 0, world)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return run_b200_dist(args, rank, local, world)

    sc, mesh, setup_s = build_workload(args.config, args.scale, device=local)
    C, E = mesh.n_cells, mesh.n_edges
    t0 = time.perf_counter()
    solver = api.DeviceSolver(mesh, device=local)
    create_s = time.perf_counter() - t0
    horizon = HORIZON
    W, K = max(3, args.warmup), args.steps
    clk = ClockSampler(local).start()
    # clocks ramp from idle: >= 1 s of untimed stepping, then restart from the
    # initial state so the timed window is steps [W, W+K) -- the reference
    # arm's window (the W warm-up steps also rebuild the dry-tile mask)
    solver.set_state(sc.state)
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 1.0:
        _, s_now = solver.clock()
        solver.advance(t_end=horizon, max_steps=s_now + 50)
    solver.set_state(sc.state)
    solver.advance(t_end=horizon, max_steps=W)
    _, step0 = solver.clock()
    assert step0 == W
    inf_0 = solver.info()
    skipped0, held0 = inf_0["skipped_tiles"], inf_0["held_tiles"]
    # e2e replays the same K steps from this state (untimed copy-out here)
    e2e_start = None if args.no_e2e else solver.get_state()

    stream = torch.cuda.ExternalStream(solver.stream, device=local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = api.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    w0 = time.time()
    ev0.record(stream)
    solver.advance_async(t_end=horizon, max_steps=step0 + K)  # one graph launch, no host sync
    ev1.record(stream)
    torch.cuda.synchronize()
    recs = solver.records()
    clk.mark(w0, time.time())
    clk.stop()
    info0 = solver.info()
    skip_frac = (info0["skipped_tiles"] - skipped0) / max(1, K * info0["tiles"])
    held_frac = (info0["held_tiles"] - held0) / max(1, K * info0["tiles"])
    launches = api.launch_count() - launches0
    assert len(recs) == K, f"expected {K} steps, ran {len(recs)}"
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = world * C * K / (ms / 1e3)

    # kernel-level timing: the same K steps again (from the state at step W),
    # plain launches with events per kernel on the solver's stream
    solver.set_state(sc.state)
    solver.advance(t_end=horizon, max_steps=W)
    inf_1 = solver.info()
    skipped1, held1 = inf_1["skipped_tiles"], inf_1["held_tiles"]
    solver.set_profiling(True)
    solver.advance_n_async(K, t_end=horizon)
    solver.synchronize()
    kt = solver.kernel_times()
    solver.set_profiling(False)
    info = solver.info()
    prof_skip = (info["skipped_tiles"] - skipped1) / max(1, K * info["tiles"])
    prof_held = (info["held_tiles"] - held1) / max(1, K * info["tiles"])
    avg = lambda k: kt[k][0] / max(1, kt[k][1])  # noqa: E731
    fin_ms = avg("finalize")
    peak, peak_src = load_peaks()
    step_bytes = 116 * C + 128 * E  # SURVEY.md §8(d) canonical B_step
    # skipped tiles: 40 B/cell (h, area in; state out), held ones 16 B/cell (h, area in)
    step_eff = ((1.0 - skip_frac) * step_bytes + (skip_frac - held_frac) * 40 * C
                + held_frac * 16 * C)
    prof = load_traffic()
    if prof.get("config", "channel") != args.config or args.scale != 1.0:
        prof = {}  # the committed capture is of another mesh: no per-launch bytes for this one
    if info["fused"]:
        # the dominant kernel k_tile does the whole step (face + cell work of
        # §8(d)) in one launch: its algorithmic bytes per launch are B_step,
        # skipped dry tiles counted at 40 B/cell (h, area in; state out)
        tile_ms = avg("tile")
        kernels = {"tile": tile_ms, "finalize": fin_ms}
        own = 80 * C + 32 * E + 4 * info["halo_edges"]  # the fused kernel's own compulsory bytes
        skipped_b = (prof_skip - prof_held) * 40 * C + prof_held * 16 * C
        dom = ("tile", tile_ms, (1.0 - prof_skip) * step_bytes + skipped_b,
               (1.0 - prof_skip) * own + skipped_b)
    else:
        face_ms, cell_ms = avg("face"), avg("cell")
        kernels = {"face": face_ms, "cell": cell_ms, "finalize": fin_ms}
        dom = (("face", face_ms, 64 * E + 32 * C, 82 * E + 32 * C) if face_ms >= cell_ms
               else ("cell", cell_ms, 64 * E + 84 * C, 144 * C))
    t_s = dom[1] / 1e3
    achieved = dom[2] / t_s / 1e9
    traffic = prof.get(dom[0])
    fp64 = prof.get(dom[0] + "_fp64_thread_inst")
    fpk = load_fp64_peak()
    roof = {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "peak_source": peak_src,
            "canonical_frac": achieved / peak,
            "canonical_bytes_per_launch": dom[2],
            "canonical_note": "SURVEY.md 8(d) B_step = 116 C + 128 E per step (one k_tile "
                              "launch), dry tiles skipped in this window counted at 40 B/cell, "
                              "held ones (next state already in place, no writes) at 16 B/cell",
            "dram_frac": (traffic / t_s / 1e9 / peak) if traffic else None,
            "dram_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch "
                         "(committed capture, profiles/traffic.json) over this run's mean launch "
                         "time: the physical HBM utilisation",
            "fp64_frac": (fp64 / t_s / fpk["dfma_per_s"]) if (fp64 and fpk) else None,
            "fp64_note": ("FP64 thread-instructions (DFMA + DMUL + DADD) per launch from the ncu "
                          "capture over the mean launch time, against the measured DFMA peak "
                          f"{fpk['dfma_per_s']:.3e}/s (profiles/r02_fp64_peak.json)") if fpk else
                         "no FP64 peak measured",
            # issue roofline: warp-instructions per launch (ncu capture) over the
            # SMs' issue capacity (4 schedulers x 1 warp-instruction per clock)
            "issue_frac": ((prof[dom[0] + "_warp_inst"] / t_s)
                           / (4 * fpk["sms"] * fpk["clock_mhz_attr"] * 1e6))
                          if (fpk and prof.get(dom[0] + "_warp_inst")) else None,
            "issue_note": "smsp__inst_executed.sum per launch (profiles/traffic.json) over the mean "
                          "launch time, against 4 warp-instructions per SM per clock at the "
                          "attribute clock (profiles/r02_fp64_peak.json sms, clock_mhz_attr)",
            "own_bytes_per_launch": dom[3],
            "own_frac": dom[3] / t_s / 1e9 / peak,
            "limiter": prof.get(dom[0] + "_limiter"),
            "kernel_ms": kernels,
            "layout": info,
            "step": {"algorithmic_bytes": step_eff,
                     "achieved_gbs": step_eff / (ms / K / 1e3) / 1e9,
                     "frac": step_eff / (ms / K / 1e3) / 1e9 / peak}}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
           "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": args.scaling,
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(args.config, C, E, mesh.n_boundary_edges, world),
           "setup": {"setup_s": round(setup_s, 2), "create_s": round(create_s, 2),
                     "device_bytes": solver.memory_bytes()},
           "gpu_launches": (3 if info["persistent"] else
                            (2 if info["fused"] else 3) * info["graph_unroll"]
                            * -(-K // info["graph_unroll"]) + 2),
           "gpu_launches_note": ("k_set_params, k_gate and ONE cooperative launch of the "
                                 f"persistent step kernel k_run ({info['grid_run']} CTAs) for all "
                                 f"{K} steps (grid barrier per step; the last CTA to arrive "
                                 "commits the step)" if info["persistent"] else
                                 "k_set_params + one CUDA-graph launch = k_gate + a conditional "
                                 f"WHILE node of ceil(K/{info['graph_unroll']}) iterations x "
                                 f"{info['graph_unroll']} x ("
                                 + ("k_tile" if info["fused"] else "k_face_c, k_cell_c")
                                 + ", k_finalize); steps past the stop exit at once")
                                + f" (host-side launch calls: {launches})",
           "roofline": roof,
           "clocks": clk.summary()}
    if info["fused"]:
        ms_ns = (no_skip_ms(api, mesh, sc, step0, K, horizon, local, torch)
                 if info["dry_skip"] else ms / K)
        out["dry_tile_skip"] = {
            "enabled": bool(info["dry_skip"]), "skipped_tile_fraction": skip_frac,
            "held_tile_fraction": held_frac,
            "note": "tiles whose cells and ring were dry and at rest after the previous step "
                    "are updated without evaluating their edges (every mass flux is exactly "
                    "+-0, the clamp zeroes q); results bit-identical (tests/test_gpu_parity.py)",
            "ms_per_step_without_skip": ms_ns,
            "step_frac_without_skip": step_bytes / (ms_ns / 1e3) / 1e9 / peak}

    if not args.no_e2e:
        out["e2e"] = e2e_run(api, solver, e2e_start, K, horizon, torch)
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(sc, mesh, args, W)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def load_traffic():
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()) if p.exists() else {}
    except Exception:
        return {}


def load_fp64_peak():
    p = ROOT / "profiles" / "r02_fp64_peak.json"
    try:
        return json.loads(p.read_text()) if p.exists() else None
    except Exception:
        return None


def no_skip_ms(api, mesh, sc, step0, K, horizon, local, torch):
    """the same K steps (same starting step) with dry-tile skipping off"""
    os.environ["SWE_NO_DRY_SKIP"] = "1"
    try:
        s = api.DeviceSolver(mesh, device=local)
    finally:
        del os.environ["SWE_NO_DRY_SKIP"]
    st = torch.cuda.ExternalStream(s.stream, device=local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(2):  # the first pass also brings the clocks back up after setup
        s.set_state(sc.state)
        while s.clock()[1] < step0:  # in chunks: one advance() keeps at most 2^16 records
            s.advance(t_end=horizon, max_steps=min(step0, s.clock()[1] + 50_000))
        torch.cuda.synchronize()
        e0.record(st)
        s.advance_async(t_end=horizon, max_steps=step0 + K)
        e1.record(st)
        torch.cuda.synchronize()
        s.records()
        best = min(best, e0.elapsed_time(e1) / K)
    s.close()
    return best


def e2e_run(api, solver, start, K, horizon, torch):
    """Public C-ABI with pinned host buffers: H2D state, K steps with per-step
    stats records back to the host, D2H final state.  start = (state, t,
    step) at the first timed step of `value`, so both cover the same steps."""
    C = solver.n_cells
    state, t_start, step_start = start
    pin = [torch.empty(C, dtype=torch.float64).pin_memory() for _ in range(6)]
    for dst, src in zip(pin[:3], (state.h, state.qx, state.qy)):
        dst.numpy()[:] = src
    ptrs_in = [p.data_ptr() for p in pin[:3]]
    ptrs_out = [p.data_ptr() for p in pin[3:]]
    # one untimed round trip first: the first DMA through freshly pinned pages
    # pays their mapping (measured +2.5 ms of 22 ms at 10M cells,
    # tools/e2e_breakdown.py); then the median of 3 timed end-to-end runs
    solver.set_state_ptrs(*ptrs_in, t=t_start, step=step_start)
    solver.get_state_ptrs(*ptrs_out)
    runs = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.set_state_ptrs(*ptrs_in, t=t_start, step=step_start)
        recs = solver.advance(t_end=horizon, max_steps=step_start + K)
        solver.get_state_ptrs(*ptrs_out)
        runs.append(time.perf_counter() - t0)
        assert len(recs) == K
    el = sorted(runs)[1]
    h2d, d2h = 24 * C, 24 * C + 40 * K
    return {"value": C * K / el, "unit": UNIT, "h2d_bytes_per_step": h2d / K,
            "d2h_bytes_per_step": d2h / K, "wall_s": el, "wall_s_runs": runs,
            "path": "swe_dev_set_state (pinned H2D) + swe_dev_advance (K steps, stats rows D2H) + "
                    "swe_dev_get_state (pinned D2H), host wall clock, median of 3 runs after one "
                    "untimed round trip through the pinned buffers; the same K steps as value "
                    "(from the state at its first timed step)"}


def cpu_baseline(sc, mesh, args, W):
    """The reference (oracle/_ref) on a bounded sample of the same window:
    steps [W, W+k) on all host threads, and a few of them on one thread
    (bench.hpp:150-153 times a sequential and a parallel variant)."""
    from oracle.pyoracle import RefOracle
    if not RefOracle.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    threads = reference_threads()
    wl = {"nodes": sc.raw.nodes, "tris": sc.raw.triangles, "bed": sc.bed, "manning": sc.manning,
          "h": sc.state.h, "qx": sc.state.qx, "qy": sc.state.qy}
    rm, build_s = ref_mesh_of(wl)
    # size the samples to ~cpu_seconds of work (~5e7 cell-updates/s on 8 threads,
    # ~8e6 on one)
    steps = int(max(2, min(args.steps, 50, args.cpu_seconds * 6e6 * threads / mesh.n_cells)))
    seq = int(max(1, min(steps, 0.5 * args.cpu_seconds * 8e6 / mesh.n_cells)))
    r = reference_window(rm, wl, W, steps, threads, seq_steps=seq)
    return {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"steps [{W}, {W + steps}) of the full {mesh.n_cells}-cell workload "
                      f"({r['phase_s']:.1f} s of phase time, reference build_mesh {build_s:.1f} s "
                      f"excluded), {threads} OpenMP threads",
            "sequential": {"value": r["seq_value"], "unit": UNIT, "cores": 1,
                           "sample": f"steps [{W}, {W + seq}) on one thread"},
            "host": host_cpu_info()}


def main():
    global WEAK_BASE
    args = parse()
    WEAK_BASE = args.weak_base
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

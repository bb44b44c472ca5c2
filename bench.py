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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N > 1: strong = the configured mesh split N ways; weak = N x the cells")
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


def workload_config(name, sc, mesh, world, note_extra=None):
    cfg = {"workload": f"{name} ({CONFIG_NOTE[name]})", "cells": mesh.n_cells,
           "edges": mesh.n_edges, "boundary_edges": mesh.n_boundary_edges,
           "mesh": "unstructured: jittered nodes, random diagonals, random node/cell numbering",
           "l2": ("inputs larger than L2 (state + mesh ~= 300 B/cell >> 126 MB)"
                  if 300 * mesh.n_cells > 2 * 126e6 else
                  f"inputs fit in L2 (~{300 * mesh.n_cells / 1e6:.0f} MB of state + mesh): "
                  "resident across steps as in any run of this size; not flushed"),
           "parallelism": "single GPU" if world == 1 else f"{world} independent replicas"}
    if note_extra:
        cfg.update(note_extra)
    return cfg


REF_MAX_STEPS = 150


def reference_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def time_reference(sc, mesh, steps, warmup, threads):
    """The reference (oracle/_ref, unmodified headers) on the same mesh and
    initial state; phase timers of engine.hpp:314-317 as bench.hpp:105-110."""
    from oracle.pyoracle import RefOracle
    ref = RefOracle()
    t0 = time.perf_counter()
    rm = ref.build_mesh(sc.raw.nodes, sc.raw.triangles, sc.bed, sc.manning)
    setup_s = time.perf_counter() - t0
    st = sc.state
    if warmup > 0:
        rm.advance(st.h, st.qx, st.qy, t_end=1.7976931348623157e308, nsteps=warmup, threads=threads)
    r = rm.advance(st.h, st.qx, st.qy, t_end=1.7976931348623157e308, nsteps=steps, threads=threads)
    if r["rc"] != 0:
        raise RuntimeError(f"reference failed: {r['error']}")
    phase_s = r["flux_s"] + r["update_s"]
    return mesh.n_cells * steps / phase_s, phase_s, setup_s


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from oracle.pyoracle import RefOracle
    if not RefOracle.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libswe_ref.so was not built (needs /root/reference)"}))
        return
    sc, mesh, _ = build_workload(args.config, args.scale)
    threads = reference_threads()
    # bounded sample: ~0.34 s per step at 10M cells on 16 threads, so at most
    # REF_MAX_STEPS timed steps keep the arm within a few minutes for any K
    steps, warmup = min(args.steps, REF_MAX_STEPS), min(args.warmup, 3)
    value, phase_s, setup_s = time_reference(sc, mesh, steps, warmup, threads)
    sample = (f"{steps} timed steps (after {warmup} warm-up) of the full "
              f"{mesh.n_cells}-cell workload, reference build with -O3 -fopenmp "
              f"-ffp-contract=off, {threads} OpenMP threads, phase timers")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * phase_s / steps, "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(args.config, sc, mesh, 1),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


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

    scale = args.scale * (world ** 0.5 if args.scaling == "weak" else 1.0)
    sc, mesh, setup_s = build_workload(args.config, scale, device=local)
    # equal work per GPU: cells weighted by the device's own dry-tile skip pattern
    part = dist.partition(mesh, world, dist.measured_cost_weights(mesh, sc.state, device=local,
                                                                  parts=world))
    lm = dist.local_mesh(mesh, part, rank)
    lp = dist.LinkedPart(lm, device=local)
    U = api.DeviceSolver.info(lp)["graph_unroll"]  # steps per WHILE iteration
    try:
        dist.link_torch(lp)
    except dist.LinkUnavailable as e:  # every rank takes this branch together
        lp.close()
        return run_dist_host_driven(args, rank, local, world, sc, mesh, part, lm, setup_s,
                                    reason=str(e))
    lp.set_state(sc.state)
    horizon = 1.7976931348623157e308
    W, K = max(3, args.warmup), args.steps
    dev = "cpu" if LOCKSTEP_CHECK else "cuda"

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

    advance(W)
    # clocks ramp: keep stepping >= 1 s; every rank takes the same decision
    t_w = time.perf_counter()
    steps = W
    while True:
        go = torch.tensor([1.0 if time.perf_counter() - t_w < 1.0 else 0.0], device=dev)
        tdist.all_reduce(go, op=tdist.ReduceOp.MAX)
        if go.item() == 0.0:
            break
        steps += 50
        advance(steps)
    skipped0 = lp_skipped(lp)
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
    sk = torch.tensor([float(lp_skipped(lp) - skipped0), float(lp_tiles(lp) * K)], device=dev)
    tdist.all_reduce(sk, op=tdist.ReduceOp.SUM)
    skip_frac = float(sk[0].item()) / max(1.0, float(sk[1].item()))
    ms = float(ms.item())
    C = mesh.n_cells
    # e2e: host state in, K steps, owned state back to the host
    tdist.barrier()
    t0 = time.perf_counter()
    lp.set_state(sc.state)
    advance(K)
    got = api.FieldState.zeros(C)
    lp.gather_owned(got)
    e2e_s = torch.tensor([time.perf_counter() - t0], device=dev)
    tdist.all_reduce(e2e_s, op=tdist.ReduceOp.MAX)
    if rank == 0:
        out = {"metric": METRIC, "value": C * K / (ms / 1e3), "unit": UNIT, "n_gpus": world,
               "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
               "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": workload_config(args.config, sc, mesh, 1, {
                   "parallelism": f"{world}-way cost-weighted RCB domain decomposition (cells "
                                  "of computed tiles weighted "
                                  f"{dist.COMPUTED_COST_LARGE if mesh.n_cells / world >= dist.LARGE_PART_CELLS else dist.COMPUTED_COST}"
                                  "x cells of skipped dry tiles, measured on the device), one "
                                  "part per GPU; "
                                  "ghost states pushed peer-to-peer by the step kernel, CFL "
                                  "bound / outcome through device mailboxes (no host round "
                                  "trip per step)",
                   "cells_per_gpu_max": int(np.bincount(part).max()),
                   "cells_per_gpu_min": int(np.bincount(part).min()),
                   "halo_cells_rank0": int(lm.n_cells - lm.n_owned), "setup_s": round(setup_s, 2)}),
               "gpu_launches": 2 * U * -(-K // U) + 2,
               "gpu_launches_note": "per rank: k_set_params + one CUDA-graph launch = k_gate + "
                                    f"a conditional WHILE node of ceil(K/{U}) iterations x {U} x "
                                    "(k_tile with halo push, k_exchange); steps past the stop "
                                    "exit at once",
               "clocks": clk.summary() if clk else None,
               "roofline": dist_roofline(mesh, K, ms, world, skip_frac),
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


def run_dist_host_driven(args, rank, local, world, sc, mesh, part, lm, setup_s, reason):
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
    C = mesh.n_cells
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
               "config": workload_config(args.config, sc, mesh, 1, {
                   "parallelism": f"{world}-way cost-weighted RCB domain decomposition, host-"
                                  "driven exchange (NCCL send/recv + all_reduce per step): "
                                  f"linked peer memory unavailable ({reason[:160]})",
                   "cells_per_gpu_max": int(np.bincount(part).max()),
                   "setup_s": round(setup_s, 2)}),
               "gpu_launches": launches,
               "gpu_launches_note": "rank 0, counted by the library: per step halo pack / "
                                    "unpack, k_set_params, k_gate, k_tile, k_finalize (+ NCCL "
                                    "kernels, not counted)",
               "clocks": clk.summary() if clk else None,
               "roofline": dist_roofline(mesh, K, ms, world, 0.0),
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
    v = (ctypes.c_longlong * 12)()
    lp.lib.swe_dev_info(lp.ctx, v, 12)
    return list(v)


def lp_skipped(lp):
    return _lp_info(lp)[11]


def lp_tiles(lp):
    return _lp_info(lp)[2]


def dist_roofline(mesh, K, ms, world, skip_frac):
    """whole-job step roofline of an N-GPU run: SURVEY §8(d) canonical step
    bytes (skipped dry tiles at 40 B/cell) over the max-over-ranks step time,
    against N x the per-GPU HBM peak"""
    peak, src = load_peaks()
    C, E = mesh.n_cells, mesh.n_edges
    step = (1.0 - skip_frac) * (116 * C + 128 * E) + skip_frac * 40 * C
    achieved = step / (ms / K / 1e3) / 1e9
    return {"bound": "hbm", "kernel": "step (all ranks)", "achieved": achieved,
            "peak": world * peak, "unit": "GB/s", "frac": achieved / (world * peak),
            "traffic": None, "peak_source": f"{world} x {src}",
            "skipped_tile_fraction": skip_frac}


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
    solver.set_state(sc.state)
    horizon = 1.7976931348623157e308  # bench.hpp:91 (fixed-step throughput mode)
    W, K = max(3, args.warmup), args.steps
    clk = ClockSampler(local).start()
    solver.advance(t_end=horizon, max_steps=W)
    # clocks ramp from idle: keep stepping (untimed) for >= 1 s before timing
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 1.0:
        _, s_now = solver.clock()
        solver.advance(t_end=horizon, max_steps=s_now + 50)
    _, step0 = solver.clock()
    skipped0 = solver.info()["skipped_tiles"]
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
    launches = api.launch_count() - launches0
    assert len(recs) == K, f"expected {K} steps, ran {len(recs)}"
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = world * C * K / (ms / 1e3)

    # kernel-level timing: same K steps, plain launches with events per kernel
    skipped1 = info0["skipped_tiles"]
    solver.set_profiling(True)
    solver.advance_n_async(K, t_end=horizon)
    solver.synchronize()
    kt = solver.kernel_times()
    solver.set_profiling(False)
    info = solver.info()
    prof_skip = (info["skipped_tiles"] - skipped1) / max(1, K * info["tiles"])
    avg = lambda k: kt[k][0] / max(1, kt[k][1])  # noqa: E731
    fin_ms = avg("finalize")
    peak, peak_src = load_peaks()
    if info["fused"]:
        # k_tile compulsory traffic: cell state/bed/area/n/r in (56 B) + state
        # out (24 B); edge record {el|kl, er|kr} (8 B) + {nx, ny} (16 B) + len
        # (8 B) = 32 B; halo index (4 B)
        # a dry tile skipped moves 40 B per cell: h and area in,
        # state out -- no edge data, no qx / qy / bed
        tile_ms = avg("tile")
        kernels = {"tile": tile_ms, "finalize": fin_ms}
        full = 80 * C + 32 * E + 4 * info["halo_edges"]
        dom = ("tile", tile_ms, (1.0 - prof_skip) * full + prof_skip * 40 * C)
    else:
        # k_face_c: edge data 34 B + contributions out 48 B per edge, state+bed
        # gathers 32 B per cell; k_cell_c: 3x3 contributions 72 B + state 24 B
        # + area/n/r 24 B in, state 24 B out per cell
        face_ms, cell_ms = avg("face"), avg("cell")
        kernels = {"face": face_ms, "cell": cell_ms, "finalize": fin_ms}
        dom = (("face", face_ms, 82 * E + 32 * C) if face_ms >= cell_ms
               else ("cell", cell_ms, 144 * C))
    achieved = dom[2] / (dom[1] / 1e3) / 1e9
    step_bytes = 116 * C + 128 * E  # SURVEY.md §8(d) canonical two-phase B_step
    step_eff = (1.0 - skip_frac) * step_bytes + skip_frac * 40 * C  # skipped tiles: 40 B/cell
    traffic, limiter = None, None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            traffic, limiter = tj.get(dom[0]), tj.get(dom[0] + "_limiter")
        except Exception:
            traffic = None

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
           "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": args.scaling,
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(args.config, sc, mesh, world,
                                     {"setup_s": round(setup_s, 2), "create_s": round(create_s, 2),
                                      "device_bytes": solver.memory_bytes()}),
           "gpu_launches": (2 if info["fused"] else 3) * info["graph_unroll"]
                           * -(-K // info["graph_unroll"]) + 2,
           "gpu_launches_note": "k_set_params + one CUDA-graph launch = k_gate + a conditional "
                                f"WHILE node of ceil(K/{info['graph_unroll']}) iterations x "
                                f"{info['graph_unroll']} x ("
                                + ("k_tile" if info["fused"] else "k_face_c, k_cell_c")
                                + ", k_finalize); steps past the stop exit at once "
                                f"(host-side launch calls: {launches})",
           "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
                        "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                        "peak_source": peak_src,
                        "limiter": limiter,
                        "algorithmic_bytes_per_launch": dom[2],
                        "kernel_ms": kernels,
                        "layout": info,
                        "step": {"canonical_bytes": "SURVEY.md 8(d) B_step = 116 C + 128 E, "
                                                    "skipped dry tiles counted at 40 B/cell",
                                 "algorithmic_bytes": step_eff,
                                 "achieved_gbs": step_eff / (ms / K / 1e3) / 1e9,
                                 "frac": step_eff / (ms / K / 1e3) / 1e9 / peak}},
           "clocks": clk.summary()}
    if info["fused"]:
        ms_ns = (no_skip_ms(api, mesh, sc, step0, K, horizon, local, torch)
                 if info["dry_skip"] else ms / K)
        out["dry_tile_skip"] = {
            "enabled": bool(info["dry_skip"]), "skipped_tile_fraction": skip_frac,
            "note": "tiles whose cells and ring were dry and at rest after the previous step "
                    "are updated without evaluating their edges (every mass flux is exactly "
                    "+-0, the clamp zeroes q); results bit-identical (tests/test_gpu_parity.py)",
            "ms_per_step_without_skip": ms_ns,
            "step_frac_without_skip": step_bytes / (ms_ns / 1e3) / 1e9 / peak}

    if not args.no_e2e:
        out["e2e"] = e2e_run(api, solver, e2e_start, K, horizon, torch)
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(sc, mesh, args)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


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
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solver.set_state_ptrs(*ptrs_in, t=t_start, step=step_start)
    recs = solver.advance(t_end=horizon, max_steps=step_start + K)
    solver.get_state_ptrs(*ptrs_out)
    el = time.perf_counter() - t0
    assert len(recs) == K
    h2d, d2h = 24 * C, 24 * C + 40 * K
    return {"value": C * K / el, "unit": UNIT, "h2d_bytes_per_step": h2d / K,
            "d2h_bytes_per_step": d2h / K, "wall_s": el,
            "path": "swe_dev_set_state (pinned H2D) + swe_dev_advance (K steps, stats rows D2H) + "
                    "swe_dev_get_state (pinned D2H), host wall clock; the same K steps as value "
                    "(from the state at its first timed step)"}


def cpu_baseline(sc, mesh, args):
    from oracle.pyoracle import RefOracle
    if not RefOracle.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    threads = reference_threads()
    # size the sample to ~cpu_seconds of work at ~5e7 cell-updates/s/8 threads
    est = 6e6 * threads
    steps = int(max(2, min(50, args.cpu_seconds * est / mesh.n_cells)))
    value, phase_s, setup_s = time_reference(sc, mesh, steps, 1, threads)
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{steps} steps of the full {mesh.n_cells}-cell workload after 1 warm-up "
                      f"step ({phase_s:.1f} s of phase time, reference build_mesh {setup_s:.1f} s "
                      f"excluded), {threads} OpenMP threads"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

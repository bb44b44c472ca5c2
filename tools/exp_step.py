#!/usr/bin/env python3
"""Step-timing experiment: graph-launched K steps vs plain launches vs the
per-kernel event times, on one scenario.  Prints one JSON line."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="channel")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--identity", action="store_true")
    ap.add_argument("--two-phase", action="store_true")
    ap.add_argument("--presteps", type=int, default=0)
    ap.add_argument("--linked", action="store_true", help="self-linked context (nranks=1)")
    a = ap.parse_args()
    import torch
    from paper_1807_00672_b200 import api
    sc = api.make_scenario(a.config, scale=a.scale)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    H = 1.7976931348623157e308
    if a.linked:
        from paper_1807_00672_b200 import dist
        lm = dist.local_mesh(mesh, dist.partition(mesh, 1), 0)
        p = dist.LinkedPart(lm, two_phase=a.two_phase)
        dist.link_local([p])
        p.set_state(sc.state)
        p.advance(t_end=H, max_steps=5 + a.presteps)
        st = torch.cuda.ExternalStream(p.lib.swe_dev_stream(p.ctx))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        out = {"cells": mesh.n_cells, "linked": True}
        n0 = 5 + a.presteps
        for rep in range(2):
            torch.cuda.synchronize()
            e0.record(st)
            p.advance(t_end=H, max_steps=n0 + a.steps)
            e1.record(st)
            torch.cuda.synchronize()
            n0 += a.steps
            out[f"graph_ms_per_step_{rep}"] = e0.elapsed_time(e1) / a.steps
        out["kernel_ms"] = {}
        print(json.dumps(out))
        return
    s = api.DeviceSolver(mesh, identity_order=a.identity, two_phase=a.two_phase)
    s.set_state(sc.state)
    s.advance(t_end=H, max_steps=5 + a.presteps)
    st = torch.cuda.ExternalStream(s.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"cells": mesh.n_cells, "edges": mesh.n_edges, "info": s.info()}
    for rep in range(2):
        _, step0 = s.clock()
        torch.cuda.synchronize()
        e0.record(st)
        s.advance(t_end=H, max_steps=step0 + a.steps)
        e1.record(st)
        torch.cuda.synchronize()
        out[f"graph_ms_per_step_{rep}"] = e0.elapsed_time(e1) / a.steps
        e0.record(st)
        s.advance_n_async(a.steps, t_end=H)
        e1.record(st)
        s.synchronize()
        out[f"plain_ms_per_step_{rep}"] = e0.elapsed_time(e1) / a.steps
    s.set_profiling(True)
    s.advance_n_async(a.steps, t_end=H)
    s.synchronize()
    kt = s.kernel_times()
    out["kernel_ms"] = {k: v[0] / max(1, v[1]) for k, v in kt.items()}
    inf = s.info()
    if "skipped_tiles" in inf:
        _, steps_done = s.clock()
        out["skipped_per_step"] = inf["skipped_tiles"] / max(1, steps_done) / max(1, inf["tiles"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()

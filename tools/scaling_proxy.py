#!/usr/bin/env python3
"""Strong-scaling proxy on ONE GPU: split the 10M channel into N RCB parts,
time each part's step (events; the run loop the engine picks for the part)
separately, and project the N-GPU step as max over parts (+ the measured
cost of the linked exchange at the part's size: the channel scaled to 1/N,
self-linked vs unlinked, on the run loop a linked rank of that size uses).
Prints one JSON line."""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def time_part(lp, steps, torch):
    st = torch.cuda.ExternalStream(lp.lib.swe_dev_stream(lp.ctx))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    H = 1.7976931348623157e308
    lp.advance(t_end=H, max_steps=5)
    torch.cuda.synchronize()
    e0.record(st)
    lp.launch(t_end=H, max_steps=5 + steps)
    e1.record(st)
    torch.cuda.synchronize()
    lp.records()
    return e0.elapsed_time(e1) / steps


def exchange_cost(torch, api, dist, n, steps):
    """ms per step that linking adds at 1/n of the channel (10.26M / n cells)"""
    sc = api.make_scenario("channel", scale=(1.0 / n) ** 0.5)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    # a linked rank of this size: the persistent kernel up to 600k cells (swe_dev.cu)
    old = os.environ.get("SWE_PERSISTENT")
    os.environ["SWE_PERSISTENT"] = "1" if mesh.n_cells <= 600000 else "0"
    try:
        one = dist.LinkedPart(dist.local_mesh(mesh, dist.partition(mesh, 1), 0))
    finally:
        if old is None:
            del os.environ["SWE_PERSISTENT"]
        else:
            os.environ["SWE_PERSISTENT"] = old
    one.set_state(sc.state)
    t0 = time_part(one, steps, torch)
    dist.link_local([one])
    one.set_state(sc.state)
    t1 = time_part(one, steps, torch)
    one.close()
    return t1 - t0, mesh.n_cells, int(mesh.n_cells <= 600000)


def weak(torch, api, dist, steps):
    """weak scaling: the channel scaled to N x 10M cells, N cost-weighted parts
    timed one by one; projected efficiency = 10M single step / slowest part"""
    out = {"mode": "weak"}
    sc = api.make_scenario("channel", scale=1.0)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    one = dist.LinkedPart(dist.local_mesh(mesh, dist.partition(mesh, 1), 0))
    one.set_state(sc.state)
    t1 = time_part(one, steps, torch)
    one.close()
    del mesh, sc
    out["ms_1"] = t1
    for n in [int(x) for x in sys.argv[sys.argv.index("--weak") + 1].split(",")]:
        sc = api.make_scenario("channel", scale=n ** 0.5)
        mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
        cc = float(sys.argv[sys.argv.index("--cc") + 1]) if "--cc" in sys.argv else None
        w = dist.measured_cost_weights(mesh, sc.state, parts=n, **({"computed_cost": cc} if cc else {}))
        part = dist.partition(mesh, n, w)
        ts, cells = [], []
        for p in range(n):
            lm = dist.local_mesh(mesh, part, p)
            lp = dist.LinkedPart(lm)
            lp.set_state(sc.state)
            ts.append(time_part(lp, steps, torch))
            cells.append(lm.n_owned)
            lp.close()
        out[f"N{n}"] = {"cells": mesh.n_cells, "ms_parts": ts, "owned_cells": cells,
                        "ms_max": max(ts), "projected_efficiency_no_exchange": t1 / max(ts)}
        del mesh, sc
    print(json.dumps(out))


def main():
    import torch
    from paper_1807_00672_b200 import api, dist
    steps = 100
    if "--weak" in sys.argv:
        return weak(torch, api, dist, steps)
    sc = api.make_scenario("channel", scale=1.0)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    out = {"cells": mesh.n_cells}
    one = dist.LinkedPart(dist.local_mesh(mesh, dist.partition(mesh, 1), 0))
    one.set_state(sc.state)
    t1 = time_part(one, steps, torch)
    dist.link_local([one])  # self-linked: the exchange kernel's own cost
    one.set_state(sc.state)
    t1l = time_part(one, steps, torch)
    one.close()
    out["ms_1"], out["ms_1_linked"] = t1, t1l
    weights = None
    out["partition"] = "equal-count RCB"
    if "--weighted" in sys.argv:
        weights = dist.cost_weights(sc.state, mesh=mesh)
        out["partition"] = "cost-weighted RCB (wet/dry model)"
    if "--measured" in sys.argv:
        nxt = sys.argv[sys.argv.index("--measured") + 1:][:1]
        cc = float(nxt[0]) if nxt and not nxt[0].startswith("--") else None
        out["partition"] = f"cost-weighted RCB (measured skip pattern, computed tiles {cc}x)"
    refine = int(sys.argv[sys.argv.index("--refine") + 1]) if "--refine" in sys.argv else 0
    for n in (2, 4, 8):
        if "--measured" in sys.argv:
            weights = dist.measured_cost_weights(mesh, sc.state, parts=n,
                                                 **({"computed_cost": cc} if cc else {}))
        part = dist.partition(mesh, n, weights)
        history = []
        for r in range(refine):  # rebalance from measured part times (dist.refine_weights)
            pt = [dist.part_step_ms(mesh, sc.state, part, p, steps=40) for p in range(n)]
            history.append(max(pt))
            w0 = weights if weights is not None else np.ones(mesh.n_cells)
            weights = dist.refine_weights(w0, part, pt)
            part = dist.partition(mesh, n, weights)
        ts, cells, wet = [], [], []
        for p in range(n):
            lm = dist.local_mesh(mesh, part, p)
            lp = dist.LinkedPart(lm)  # unlinked: its own dt; the step cost is what is measured
            lp.set_state(sc.state)
            ts.append(time_part(lp, steps, torch))
            cells.append(lm.n_owned)
            wet.append(float((sc.state.h[lm.cells[:lm.n_owned]] > 0).mean()))
            lp.close()
        if refine:
            out.setdefault("refine_history_ms_max", {})[n] = history
        mx = max(ts)
        exch, exch_cells, exch_persistent = exchange_cost(torch, api, dist, n, steps)
        out[f"N{n}"] = {"ms_parts": ts, "owned_cells": cells, "wet_fraction": wet,
                        "ms_max": mx, "ms_mean": sum(ts) / n,
                        "exchange_ms": exch, "exchange_measured_on_cells": exch_cells,
                        "exchange_run_loop": "persistent" if exch_persistent else "graph",
                        "projected_efficiency_no_exchange": t1 / (n * mx),
                        "projected_efficiency": t1 / (n * (mx + exch))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

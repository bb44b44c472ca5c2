"""Phase times of the persistent step kernel (experiment builds with
-DSWE_RUN_TIMING=1, selected by SWE_B200_LIB): per CTA-step work, waits for
the epoch and for all arrivals, and the commit, averaged over K steps.

    SWE_B200_LIB=exp/tim/libswe_b200.so python tools/run_timing.py --config channel
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1807_00672_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="channel")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--parts", type=int, default=1, help="time part 0 of an N-way RCB split")
ap.add_argument("--part", type=int, default=0, help="which part of the split")
ap.add_argument("--measured", action="store_true", help="measured-cost RCB (bench.py's split)")
ap.add_argument("--self-link", action="store_true",
                help="the whole mesh as ONE linked rank: the exchange's own cost per step")
a = ap.parse_args()
sc = api.make_scenario(a.config, scale=a.scale)
m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
if a.parts > 1 or a.self_link:
    from paper_1807_00672_b200 import dist
    w = dist.measured_cost_weights(m, sc.state, parts=a.parts) if a.measured else None
    part = dist.partition(m, a.parts, w)
    s = dist.LinkedPart(dist.local_mesh(m, part, a.part))  # unlinked: its own dt
    if a.self_link:
        dist.link_local([s])
    s.stream = s.lib.swe_dev_stream(s.ctx)
    s.info = lambda: api.DeviceSolver.info(s)
    s.advance_async = lambda t_end, max_steps: s.launch(t_end=t_end, max_steps=max_steps)
else:
    s = api.DeviceSolver(m)
s.set_state(sc.state)
s.advance(1e300, max_steps=300)  # clocks
s.set_state(sc.state)
s.advance(1e300, max_steps=5)
lib = s.lib
lib.swe_dev_run_timing.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
v = (C.c_longlong * 12)()
lib.swe_dev_run_timing(s.ctx, v, 12)  # clear
st = torch.cuda.ExternalStream(s.stream, device=0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
s.advance_async(1e300, max_steps=5 + a.steps)
e1.record(st)
torch.cuda.synchronize()
s.records()
ms = e0.elapsed_time(e1)
lib.swe_dev_run_timing(s.ctx, v, 12)
work, ew, cw, com, cs, nc, aw, fin, q_dec, q_edge, q_view, q_upd = list(v)
print(json.dumps({"config": a.config, "us_per_step": 1e3 * ms / a.steps, "info": s.info(),
                  "per_cta_step_us": {"work_incl_epoch_wait": work / max(cs, 1) / 1e3,
                                      "epoch_wait": ew / max(cs, 1) / 1e3,
                                      "arrival_wait": aw / max(cs, 1) / 1e3},
                  "first_tile_us": {"decisions": q_dec / max(cs, 1) / 1e3,
                                    "stage_edges": q_edge / max(cs, 1) / 1e3,
                                    "view": q_view / max(cs, 1) / 1e3,
                                    "update": q_upd / max(cs, 1) / 1e3},
                  "commit_us": com / max(nc, 1) / 1e3,
                  "control_wait_us": cw / max(nc, 1) / 1e3,
                  "deferred_us": fin / max(nc, 1) / 1e3, "cta_steps": cs, "commits": nc}))

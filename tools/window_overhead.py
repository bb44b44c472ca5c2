"""Per-launch overhead of the run loop: device time of advance_async(K) for
several K (events on the solver's stream) and the host time of the launch
call itself; fits time(K) = a + b K.
    python tools/window_overhead.py --config channel"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1807_00672_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="channel")
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
sc = api.make_scenario(a.config, scale=a.scale)
m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
s = api.DeviceSolver(m)
s.set_state(sc.state)
s.advance(1e300, max_steps=400)
st = torch.cuda.ExternalStream(s.stream, device=0)
out = {"config": a.config, "info": s.info(), "runs": []}
for K in (1, 4, 8, 16, 20, 24, 64, 200):
    for rep in range(3):
        _, step = s.clock()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        h0 = time.perf_counter()
        s.advance_async(1e300, max_steps=step + K)
        h1 = time.perf_counter()
        e1.record(st)
        torch.cuda.synchronize()
        s.records()
        out["runs"].append({"K": K, "ms": e0.elapsed_time(e1), "host_launch_ms": 1e3 * (h1 - h0)})
import numpy as np  # noqa: E402
Ks = np.array([r["K"] for r in out["runs"]], float)
ms = np.array([r["ms"] for r in out["runs"]])
b, a0 = np.polyfit(Ks, ms, 1)
out["fit_ms"] = {"per_launch": a0, "per_step": b}
print(json.dumps(out))

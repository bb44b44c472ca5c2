"""Where the e2e time goes (bench.py e2e_run's calls, timed one by one):
pinned H2D state (swe_dev_set_state), the K-step segment with records
(swe_dev_advance), pinned D2H state (swe_dev_get_state); plus a raw pinned
cudaMemcpy bandwidth reference of the same bytes."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1807_00672_b200 import api  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sc = api.make_scenario("channel")
m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
s = api.DeviceSolver(m)
C = m.n_cells
pin = [torch.empty(C, dtype=torch.float64).pin_memory() for _ in range(6)]
for dst, src in zip(pin[:3], (sc.state.h, sc.state.qx, sc.state.qy)):
    dst.numpy()[:] = src
H = 1.7976931348623157e308
s.set_state(sc.state)
s.advance(H, max_steps=300)
out = {}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.set_state_ptrs(*[p.data_ptr() for p in pin[:3]], t=0.0, step=0)
    t1 = time.perf_counter()
    s.advance(H, max_steps=K)
    t2 = time.perf_counter()
    s.get_state_ptrs(*[p.data_ptr() for p in pin[3:]])
    t3 = time.perf_counter()
    out[rep] = {"set_state_ms": 1e3 * (t1 - t0), "advance_ms": 1e3 * (t2 - t1),
                "get_state_ms": 1e3 * (t3 - t2), "total_ms": 1e3 * (t3 - t0)}
dev = torch.empty(C, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for p in pin[:3]:
    dev.copy_(p, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
for p in pin[3:]:
    p.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
t2 = time.perf_counter()
out["raw_h2d_gbs"] = 3 * 8 * C / (t1 - t0) / 1e9
out["raw_d2h_gbs"] = 3 * 8 * C / (t2 - t1) / 1e9
print(json.dumps(out))

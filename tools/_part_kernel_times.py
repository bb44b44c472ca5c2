"""kernel times (plain launches, events) of parts of the 10M channel's 8-way
measured-cost split: k_tile vs k_finalize per step"""
import sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '.')
import torch
from paper_1807_00672_b200 import api, dist
sc = api.make_scenario("channel")
m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
w = dist.measured_cost_weights(m, sc.state, parts=8)
part = dist.partition(m, 8, w)
for k in (0, 3, 1):
    s = dist.LinkedPart(dist.local_mesh(m, part, k))
    s.info = lambda s=s: api.DeviceSolver.info(s)
    s.set_state(sc.state)
    s.advance(1e300, max_steps=100)
    D = api.DeviceSolver
    D.set_profiling(s, True)
    D.advance_n_async(s, 200, t_end=1e300)
    D.synchronize(s)
    kt = D.kernel_times(s)
    D.set_profiling(s, False)
    print(k, {a: (round(b[0] / max(1, b[1]) * 1e3, 2), b[1]) for a, b in kt.items()}, api.DeviceSolver.info(s)["tiles"])
    s.close()

"""Part k of the 10M channel's 8-way measured-cost split, stepped either by the
persistent kernel (one launch of 200 steps) or by plain k_tile / k_finalize
launches (200 steps): the target of an ncu comparison of the two loops.
    python tools/_ncu_part.py <part> persistent|plain"""
import os
import sys
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '.')
k, mode = int(sys.argv[1]), sys.argv[2]
os.environ["SWE_PERSISTENT"] = "1" if mode == "persistent" else "0"
from paper_1807_00672_b200 import api, dist  # noqa: E402

sc = api.make_scenario("channel")
m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
part = dist.partition(m, 8, dist.measured_cost_weights(m, sc.state, parts=8))
s = dist.LinkedPart(dist.local_mesh(m, part, k))
D = api.DeviceSolver
s.set_state(sc.state)
s.advance(1e300, max_steps=100)
if mode == "persistent":
    s.advance(1e300, max_steps=300)
else:
    D.advance_n_async(s, 200, t_end=1e300)
    D.synchronize(s)
print("done", mode)

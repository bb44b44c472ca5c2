import ctypes as C, json, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1807_00672_b200 import api, dist, _lib as L
sc = api.make_scenario("channel", scale=float(sys.argv[1]))
mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
out = {}
for linked in (False, True):
    lm = dist.local_mesh(mesh, dist.partition(mesh, 1), 0)
    p = dist.LinkedPart(lm)
    if linked:
        dist.link_local([p])
    p.set_state(sc.state)
    H = 1.7976931348623157e308
    p.advance(t_end=H, max_steps=10)
    lib = p.lib
    lib.swe_dev_set_profiling(p.ctx, 1)
    lib.swe_dev_advance_n_async(p.ctx, 100, H)
    st = L.swe_status(); lib.swe_dev_synchronize(p.ctx, C.byref(st))
    ms = (C.c_double * 4)(); n = (C.c_longlong * 4)()
    lib.swe_dev_kernel_times(p.ctx, ms, n, 4)
    out["linked" if linked else "plain"] = {k: ms[i] / max(1, n[i]) for i, k in enumerate(("tile", "cell", "finalize", "cfl"))}
    lib.swe_dev_set_profiling(p.ctx, 0)
    p.close()
print(json.dumps(out))

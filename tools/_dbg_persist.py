import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1807_00672_b200 import api
from oracle.pyoracle import COracle, MeshArrays
def solver(mesh, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return api.DeviceSolver(mesh)
    finally:
        for k, v in old.items():
            if v is None: del os.environ[k]
            else: os.environ[k] = v
for name, scale in [("circular_dam_break", 1.0), ("channel", 0.04)]:
    sc = api.make_scenario(name, scale=scale)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    a, b = solver(m), solver(m, SWE_PERSISTENT=0)
    print(name, a.info())
    res = []
    for s in (a, b):
        s.set_state(sc.state)
        recs = np.concatenate([s.advance(1e30, max_steps=k) for k in (1, 77, 160, 400)])
        st, t, step = s.get_state()
        res.append((recs, st))
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy, nsteps=400)
    for lab, (recs, st) in zip("ab", res):
        bad = np.flatnonzero(recs[:, 2].view(np.uint64) != ref["dts"].view(np.uint64))
        print(lab, "dt mismatches vs oracle:", len(bad), bad[:5], "state h mism:", np.count_nonzero(st.h.view(np.uint64) != ref["h"].view(np.uint64)))
    ra, rb = res[0][0], res[1][0]
    d = np.argwhere(ra.view(np.uint64) != rb.view(np.uint64))
    print("rec diffs (row,col):", d[:10].tolist(), len(d))
    if len(d): r, c = d[0]; print(ra[r], rb[r])

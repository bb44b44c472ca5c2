#!/usr/bin/env python3
"""Upper bound of dry-tile skipping on the 10M channel: after 2000 steps, the
fraction of cells dry and at rest whose neighbours are too (any exact
cell-granular skip) vs the cells in tiles the device skips."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1807_00672_b200 import api
from oracle.pyoracle import MeshArrays
sc = api.make_scenario("channel", scale=1.0, unstructured=True)
m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
s = api.DeviceSolver(m)
s.set_state(sc.state)
H = 1.7976931348623157e308
for k in range(40):
    s.advance(t_end=H, max_steps=(k + 1) * 50)
st, t, step = s.get_state()
skip = s.cell_skip().astype(bool)
ma = MeshArrays.from_mesh(m)
el, er = ma.edge_left, ma.edge_right
dry = (st.h >= 0) & (st.h < 1e-6) & (st.qx == 0) & (st.qy == 0)
inter = er >= 0
bad = np.zeros(m.n_cells, bool)  # cell has a non-dry neighbour
np.logical_or.at(bad, el[inter], ~dry[er[inter]])
np.logical_or.at(bad, er[inter], ~dry[el[inter]])
deep = dry & ~bad
print(f"step {step}: dry-at-rest {dry.mean():.3f}, deep-dry (cell+neighbours) {deep.mean():.3f}, cells in skipped tiles {skip.mean():.3f}")

import os, sys, time
sys.path.insert(0, '/root/repo')
k = int(sys.argv[1]); mode = sys.argv[2]
os.environ["SWE_PERSISTENT"] = "1" if mode == "persistent" else "0"
import torch
from paper_1807_00672_b200 import api, dist
sc = api.make_scenario("channel")
m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
part = dist.partition(m, 8, dist.measured_cost_weights(m, sc.state, parts=8))
s = dist.LinkedPart(dist.local_mesh(m, part, k))
D = api.DeviceSolver
info = D.info(s)
s.set_state(sc.state)
s.advance(1e300, max_steps=100)
st = torch.cuda.ExternalStream(s.lib.swe_dev_stream(s.ctx), device=0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sk0 = D.info(s)["skipped_tiles"]
torch.cuda.synchronize(); e0.record(st)
s.launch(t_end=1e300, max_steps=300)
e1.record(st); torch.cuda.synchronize(); s.records()
sk1 = D.info(s)["skipped_tiles"]
print(mode, k, "us/step", round(e0.elapsed_time(e1) / 200 * 1e3, 2), "tiles", info["tiles"], "skipped/step", (sk1 - sk0) / 200, "persistent", info["persistent"], "owned", s.lm.n_owned)

#!/usr/bin/env python3
"""run() with periodic snapshots at 10M cells: asynchronous snapshots (copy
+ host callback overlapped with the next segment) vs synchronous, vs no
snapshots.  Prints one JSON line."""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def one(mode, steps, every):
    from paper_1807_00672_b200 import api
    sc = api.make_scenario("channel", scale=1.0)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    st = sc.state.copy()
    s = api.DeviceSolver(mesh)
    s.set_state(sc.state)
    dt = s.advance(1e30, max_steps=3)[:, 2].min()
    del s
    t_end = steps * dt * 0.999
    interval = every * dt * 0.999 if mode != "none" else 0.0
    api.run(mesh, st.copy(), t_end=t_end * 0.05, snapshot_interval=0.0)  # warm the device mesh
    t0 = time.perf_counter()
    r = api.run(mesh, st, t_end=t_end, snapshot_interval=interval, snapshots=mode != "none")
    wall = time.perf_counter() - t0
    return {"mode": mode, "steps": r.step, "snapshots": len(r.snapshots), "wall_s": wall,
            "ms_per_step": 1e3 * wall / max(1, r.step)}


def main():
    if len(sys.argv) > 1:
        print(json.dumps(one(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))))
        return
    res = {}
    for steps, every in ((400, 20), (2000, 100)):
        out = []
        for mode in ("none", "async", "sync"):
            env = dict(os.environ)
            if mode == "sync":
                env["SWE_SYNC_SNAPSHOTS"] = "1"
            p = subprocess.run([sys.executable, __file__, mode, str(steps), str(every)], env=env,
                               capture_output=True, text=True)
            out.append(json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0
                       else {"mode": mode, "error": p.stderr[-500:]})
        res[f"channel_10M_{steps}_steps_snapshot_every_{every}"] = out
    print(json.dumps(res))


if __name__ == "__main__":
    main()

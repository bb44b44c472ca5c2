"""Smoke-size runs of every step path for compute-sanitizer (one tool per
gpurun call, profiles/r02_sanitizer_*.log):

    compute-sanitizer --tool memcheck   python tools/sanitize_run.py
    compute-sanitizer --tool racecheck  python tools/sanitize_run.py
    compute-sanitizer --tool initcheck  python tools/sanitize_run.py

Paths: fused k_tile (+ dry-tile skipping) through the graph and through plain
launches, the two-phase k_face_c / k_cell_c path, compute_fluxes, and two
linked parts stepped in lockstep on one device (P2P halo push + mailbox
exchange).  Every result is checked against the C oracle (test
infrastructure) so a run that completes also proves the paths computed.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle.pyoracle import COracle, MeshArrays  # noqa: E402
from paper_1807_00672_b200 import api, dist  # noqa: E402


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def main() -> None:
    steps = int(os.environ.get("SAN_STEPS", "12"))
    sc = api.make_scenario("sloping_wet_dry", scale=0.01)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=steps)
    print(f"mesh {m.n_cells} cells, {steps} steps", flush=True)
    for label, kw in (("fused", {}), ("two_phase", {"two_phase": True})):
        s = api.DeviceSolver(m, **kw)
        s.set_state(sc.state)
        s.advance(t_end=1e30, max_steps=steps // 2)          # graph launch
        s.advance_n_async(steps - steps // 2)                  # plain launches
        got, t, step = s.get_state()
        assert step == steps and same(got.h, ref["h"]) and same(got.qx, ref["qx"]), label
        left, right = s.compute_fluxes()
        assert np.isfinite(left).all() and np.isfinite(right).all()
        s.close()
        print(f"{label}: ok", flush=True)
    P = 2
    part = dist.partition(m, P)
    parts = [dist.LinkedPart(dist.local_mesh(m, part, p)) for p in range(P)]
    dist.link_local(parts)
    for p in parts:
        p.set_state(sc.state)
    dist.run_lockstep(parts, steps)
    got = api.FieldState.zeros(m.n_cells)
    for p in parts:
        p.gather_owned(got)
    assert same(got.h, ref["h"]) and same(got.qy, ref["qy"]), "linked"
    for p in parts:
        p.close()
    print("linked lockstep: ok", flush=True)


if __name__ == "__main__":
    main()

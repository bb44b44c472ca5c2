"""Write one BASELINE.json workload (raw mesh + bathymetry / Manning + the
initial state) to an .npz, in a process of its own.

    python tools/make_workload.py --config channel --scale 1.0 --out /tmp/w.npz

bench.py's reference arm runs this as a subprocess and builds the mesh with
the reference's own build_mesh (oracle/_ref), so the reference process never
loads this repo's library (libswe_b200.so); the input producer (the host C++
case generators of include/swe/cases.hpp) is the same one
the B200 arm uses, so both arms step bit-identical inputs.
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--weak-nx", type=int, default=2265)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    from paper_1807_00672_b200 import api
    t0 = time.perf_counter()
    sc = api.make_scenario(a.config, scale=a.scale, unstructured=True, weak_nx=a.weak_nx)
    np.savez(a.out, nodes=sc.raw.nodes, tris=sc.raw.triangles, bed=sc.bed, manning=sc.manning,
             h=sc.state.h, qx=sc.state.qx, qy=sc.state.qy, t_end=np.float64(sc.t_end),
             gen_s=np.float64(time.perf_counter() - t0))


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Time the SWEMESH 1 reader / writer (include/swe/swemesh.hpp) against the
reference's io.hpp (oracle/_ref/libswe_ref_io.so) on one scenario mesh;
prints one JSON line.  Files go to --dir (deleted afterwards)."""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="channel")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--dir", default="/tmp")
    a = ap.parse_args()
    import numpy as np
    from oracle.pyoracle import RefIO
    from paper_1807_00672_b200 import api
    sc = api.make_scenario(a.config, scale=a.scale)
    d = Path(a.dir)
    ours, ref = d / "swemesh_ours.txt", d / "swemesh_ref.txt"
    out = {"cells": sc.raw.n_cells, "nodes": len(sc.raw.nodes), "threads": a.threads or os.cpu_count()}
    t = time.perf_counter()
    api.write_swemesh(ours, sc.raw, sc.bed, sc.manning, threads=a.threads)
    out["write_s"] = time.perf_counter() - t
    r = RefIO()
    t = time.perf_counter()
    r.write(ref, sc.raw.nodes, sc.raw.triangles, sc.bed, sc.manning)
    out["ref_write_s"] = time.perf_counter() - t
    out["bytes"] = ours.stat().st_size
    out["bytes_equal"] = ours.read_bytes() == ref.read_bytes()
    t = time.perf_counter()
    raw, bed, man = api.read_swemesh(ours, threads=a.threads)
    out["read_s"] = time.perf_counter() - t
    t = time.perf_counter()
    xy, tris, rbed, rman = r.read(ref)
    out["ref_read_s"] = time.perf_counter() - t
    out["values_equal"] = bool(np.array_equal(raw.nodes.view(np.int64), xy.view(np.int64)) and
                               np.array_equal(raw.triangles, tris) and
                               np.array_equal(bed.view(np.int64), rbed.view(np.int64)) and
                               np.array_equal(man.view(np.int64), rman.view(np.int64)))
    out["read_speedup"] = out["ref_read_s"] / out["read_s"]
    out["write_speedup"] = out["ref_write_s"] / out["write_s"]
    out["read_gbs"] = out["bytes"] / out["read_s"] / 1e9
    ours.unlink()
    ref.unlink()
    print(json.dumps(out))


if __name__ == "__main__":
    main()

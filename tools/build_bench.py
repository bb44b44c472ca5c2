#!/usr/bin/env python3
"""Host vs device build_mesh at one scenario size; prints one JSON line."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="channel")
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    import numpy as np
    from paper_1807_00672_b200 import api
    t = time.perf_counter()
    sc = api.make_scenario(a.config, scale=a.scale)
    gen = time.perf_counter() - t
    api.build_mesh(api.generate_square_mesh(8, 8, 1, 1), np.zeros(128), np.zeros(128), device=0)
    t = time.perf_counter()
    md = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    dev = time.perf_counter() - t
    t = time.perf_counter()
    mh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    host = time.perf_counter() - t
    same = all(np.array_equal(np.asarray(getattr(md, f)).view(np.uint8),
                              np.asarray(getattr(mh, f)).view(np.uint8))
               for f in ("cell_nodes", "cell_area", "cx", "cy", "cell_inradius", "cell_edge",
                         "cell_sign", "edge_nodes", "edge_left", "edge_right", "nx", "ny",
                         "edge_length"))
    # the device build alone (inputs already flat), and the export of its arrays
    import ctypes as C
    from paper_1807_00672_b200 import _lib as L
    lib = L.load()
    xy = np.ascontiguousarray(sc.raw.nodes)
    tris = np.ascontiguousarray(sc.raw.triangles, dtype=np.int32)
    h, err = C.c_void_p(), C.create_string_buffer(512)
    t = time.perf_counter()
    rc = lib.swe_dev_build_mesh(0, len(xy), xy.ctypes.data, len(tris), tris.ctypes.data,
                                C.byref(h), err, 512)
    core = time.perf_counter() - t
    ne = C.c_int()
    lib.swe_dev_built_sizes(h, None, None, C.byref(ne))
    Cn, E = len(tris), ne.value
    outs = [np.empty(3 * Cn, np.int32), np.empty(Cn), np.empty(Cn), np.empty(Cn), np.empty(Cn),
            np.empty(3 * Cn, np.int32), np.empty(3 * Cn, np.int32), np.empty(2 * E, np.int32),
            np.empty(E, np.int32), np.empty(E, np.int32), np.empty(E), np.empty(E), np.empty(E)]
    for o in outs:
        o.fill(0)  # fault the pages in outside the timed export
    t = time.perf_counter()
    lib.swe_dev_built_export(h, *[o.ctypes.data for o in outs])
    export = time.perf_counter() - t
    lib.swe_dev_built_free(h)
    print(json.dumps({"config": a.config, "cells": sc.raw.n_cells, "edges": mh.n_edges,
                      "scenario_s": gen, "host_build_s": host, "device_build_s": dev,
                      "speedup": host / dev, "identical": bool(same), "rc": rc,
                      "device_core_s": core, "device_export_s": export,
                      "note": "wall incl. ctypes/numpy export of the Mesh on both paths"}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Weak-scaling proxy of BASELINE configs[4] / SURVEY §8(d) 5 on ONE GPU: the
square water drop at nx = 2265 * sqrt(N) (~10.26M cells per part), split
into N equal parts by RCB of the raw mesh, every part built rank-locally
(build_rank_mesh) and timed on its own (unlinked, events); projected
efficiency = single 10.26M step / slowest part, and with the exchange cost
measured on the single square self-linked.  Prints one JSON line.
    python tools/weak_proxy_square.py 2,4,8"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from scaling_proxy import time_part  # noqa: E402


def main():
    import torch
    from paper_1807_00672_b200 import api, dist
    import bench
    steps = 100
    Ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8").split(",")]
    out = {"mode": "weak (square water drop, rank-local parts)"}
    nx1 = bench.weak_nx(1)
    sc = api.make_scenario("weak_square", weak_nx=nx1)
    part = dist.partition_raw(sc.raw, 1)
    one = dist.LinkedPart(dist.rank_mesh(sc.raw, sc.bed, sc.manning, part, 0))
    one.set_state(sc.state)
    t1 = time_part(one, steps, torch)
    dist.link_local([one])
    one.set_state(sc.state)
    t1l = time_part(one, steps, torch)
    one.close()
    out.update({"nx_1": nx1, "cells_1": sc.raw.n_cells, "ms_1": t1, "ms_1_linked": t1l})
    del sc
    for n in Ns:
        t0 = time.perf_counter()
        nx = bench.weak_nx(n)
        sc = api.make_scenario("weak_square", weak_nx=nx)
        part = dist.partition_raw(sc.raw, n)
        ts, cells = [], []
        for p in range(n):
            lm = dist.rank_mesh(sc.raw, sc.bed, sc.manning, part, p)
            lp = dist.LinkedPart(lm)
            lp.set_state(sc.state)
            ts.append(time_part(lp, steps, torch))
            cells.append(lm.n_owned)
            lp.close()
        mx = max(ts)
        out[f"N{n}"] = {"nx": nx, "cells": sc.raw.n_cells, "ms_parts": ts, "owned_cells": cells,
                        "ms_max": mx, "projected_efficiency_no_exchange": t1 / mx,
                        "projected_efficiency": t1 / (mx + (t1l - t1)),
                        "setup_s": time.perf_counter() - t0}
        del sc
        print(json.dumps(out), file=sys.stderr)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

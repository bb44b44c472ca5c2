#!/usr/bin/env python3
"""Generate tests/golden/ fixtures from the REFERENCE ITSELF.

Runs oracle/_ref/libswe_ref.so -- the unmodified reference headers under
/root/reference/proj/include compiled by oracle/Makefile -- on small seeded
inputs and stores the outputs (full arrays for tiny cases, SHA-256 digests of
the FP64 bytes for trajectories) so the GPU box, which has no
/root/reference, can check the CUDA path and the C oracle against the
reference's own results.

    python tests/golden/make_golden.py        # needs /root/reference (this container)
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import RefOracle  # noqa: E402

KEYS = ("lx", "ly", "eta0", "amplitude", "sigma", "manning", "h_left", "h_right", "x_dam", "t_end")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def random_state(n, seed, dry_frac=0.0):
    """test_engine.cpp:40-52 distribution (h ~ U(0.2,2), u ~ U(-1,1)), numpy RNG,
    optionally with a dry fraction (test_kernels.cpp:185-201)."""
    rng = np.random.default_rng(seed)
    h = rng.uniform(0.2, 2.0, n)
    if dry_frac:
        h[rng.random(n) < dry_frac] = 0.0
    qx = h * rng.uniform(-1, 1, n)
    qy = h * rng.uniform(-1, 1, n)
    return h, qx, qy


# (name, case, nx, ny, overrides, steps, stop_at_t_end, t_end)
TRAJECTORIES = [
    ("water_drop_12x12_200", "water_drop", 12, 12, dict(lx=100.0, ly=100.0, sigma=12.0), 200, False, 1e9),
    ("still_water_8x8_25", "dam_break_1d", 8, 8, dict(lx=2.0, ly=2.0, h_left=1.0, h_right=0.75, x_dam=1.0), 25, False, 1e9),
    ("lake_at_rest_30x12_50", "lake_at_rest", 30, 12, {}, 50, False, 1e9),
    ("three_mounds_100x40_t30", "three_mounds", 100, 40, dict(t_end=30.0), 100000, True, 30.0),
    ("dam_break_1d_100x10_t40", "dam_break_1d", 100, 10, {}, 100000, True, 40.0),
    ("water_drop_50x50_1000", "water_drop", 50, 50, {}, 1000, False, 1e30),
]


def main():
    ref = RefOracle()
    out = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref/libswe_ref.so "
           "(reference headers /root/reference/proj/include, -O3 -fopenmp -ffp-contract=off)",
           "fluxes": {}, "trajectories": {}, "acceptance": {}}

    # 1. compute_fluxes on seeded random states (12x9 flat mesh, test_engine.cpp:112-127)
    nodes, tris = ref.square(12, 9, 4.0, 3.0)
    for seed, dry in ((7, 0.0), (8, 0.3)):
        nc = len(tris)
        rm = ref.build_mesh(nodes, tris, np.zeros(nc), np.zeros(nc))
        h, qx, qy = random_state(nc, seed, dry)
        left, right, rc, _ = rm.compute_fluxes(h, qx, qy)
        assert rc == 0
        np.savez_compressed(HERE / f"fluxes_12x9_seed{seed}.npz", h=h, qx=qx, qy=qy, left=left,
                            right=right)
        out["fluxes"][f"12x9_seed{seed}"] = {"file": f"fluxes_12x9_seed{seed}.npz",
                                             "digest": digest(left, right)}
    # bathymetry: three-mound floodplain, random wet/dry states
    nodes, tris = ref.square(30, 12, 75.0, 30.0)
    spec = ref.case_defaults("lake_at_rest")
    bed, man, h0, _, _ = ref.init_case("lake_at_rest", spec, nodes, tris)
    rm = ref.build_mesh(nodes, tris, bed, man)
    h, qx, qy = random_state(len(tris), 9, 0.3)
    left, right, rc, _ = rm.compute_fluxes(h, qx, qy)
    np.savez_compressed(HERE / "fluxes_mounds_30x12_seed9.npz", h=h, qx=qx, qy=qy, left=left,
                        right=right)
    out["fluxes"]["mounds_30x12_seed9"] = {"file": "fluxes_mounds_30x12_seed9.npz",
                                           "digest": digest(left, right)}

    # 2. trajectories
    for name, case, nx, ny, ov, steps, stop, t_end in TRAJECTORIES:
        spec = dict(zip(KEYS, ref.case_defaults(case)))
        spec.update(ov)
        nodes, tris = ref.square(nx, ny, spec["lx"], spec["ly"])
        bed, man, h, qx, qy = ref.init_case(case, [spec[k] for k in KEYS], nodes, tris)
        if name.startswith("still_water"):
            h[:] = 0.75
        rm = ref.build_mesh(nodes, tris, bed, man)
        r = rm.advance(h, qx, qy, t_end=t_end, nsteps=steps, stop_at_t_end=stop)
        assert r["rc"] == 0, r["error"]
        out["trajectories"][name] = {
            "case": case, "nx": nx, "ny": ny, "spec": spec, "still_water": name.startswith("still_water"),
            "steps": r["done"], "t_end": t_end, "stop_at_t_end": stop, "t": r["t"],
            "state_digest": digest(r["h"], r["qx"], r["qy"]), "dt_digest": digest(r["dts"]),
            "dts_head": r["dts"][:16].tolist(), "mass_final": rm.total_mass(r["h"]),
            "clip_events": r["clip_events"], "clipped_volume": r["clipped_volume"],
            "friction": bool(spec["manning"] > 0)}
        print(name, r["done"], r["t"])

    # 3. acceptance criteria values (acceptance.cpp:56-332 re-run through the reference)
    spec = dict(zip(KEYS, ref.case_defaults("lake_at_rest")))
    nodes, tris = ref.square(112, 45, spec["lx"], spec["ly"])
    bed, man, h, qx, qy = ref.init_case("lake_at_rest", [spec[k] for k in KEYS], nodes, tris)
    rm = ref.build_mesh(nodes, tris, bed, man)
    r = rm.advance(h, qx, qy, t_end=1e30, nsteps=1000)
    wet = h > 0
    out["acceptance"]["c1"] = {"cells": len(tris), "max_eta_err": float(np.max(np.abs(r["h"][wet] + bed[wet] - spec["eta0"]))),
                               "max_q": float(max(np.abs(r["qx"]).max(), np.abs(r["qy"]).max())),
                               "recorded": "4.441e-16 / 1.403e-13 (proj/test_output.txt:15)"}
    spec = dict(zip(KEYS, ref.case_defaults("water_drop")))
    nodes, tris = ref.square(71, 71, spec["lx"], spec["ly"])
    bed, man, h, qx, qy = ref.init_case("water_drop", [spec[k] for k in KEYS], nodes, tris)
    rm = ref.build_mesh(nodes, tris, bed, man)
    m0 = rm.total_mass(h)
    r = rm.advance(h, qx, qy, t_end=1e30, nsteps=1000)
    out["acceptance"]["c2_1000"] = {"cells": len(tris), "t": r["t"], "state_digest": digest(r["h"], r["qx"], r["qy"]),
                                    "drift": abs(rm.total_mass(r["h"]) - m0) / m0}
    spec = dict(zip(KEYS, ref.case_defaults("three_mounds")))
    spec["t_end"] = 30.0
    nodes, tris = ref.square(100, 40, spec["lx"], spec["ly"])
    bed, man, h, qx, qy = ref.init_case("three_mounds", [spec[k] for k in KEYS], nodes, tris)
    rm = ref.build_mesh(nodes, tris, bed, man)
    r = rm.advance(h, qx, qy, t_end=30.0, nsteps=100000, stop_at_t_end=True)
    out["acceptance"]["c3"] = {"cells": len(tris), "steps": r["done"], "recorded_steps": 1117,
                               "mass_final": rm.total_mass(r["h"])}
    spec = dict(zip(KEYS, ref.case_defaults("water_drop")))
    nodes, tris = ref.square(48, 48, spec["lx"], spec["ly"])
    bed, man, h, qx, qy = ref.init_case("water_drop", [spec[k] for k in KEYS], nodes, tris)
    rm = ref.build_mesh(nodes, tris, bed, man)
    r = rm.advance(h, qx, qy, t_end=1e30, nsteps=100)
    rot = np.array([ref.lib.ref_rotated_cell_index(c, 48, 48) for c in range(len(tris))])
    out["acceptance"]["c9"] = {"worst": float(np.max(np.abs(r["h"] - r["h"][rot]))),
                               "recorded": "6.661e-16 (proj/test_output.txt:23)",
                               "state_digest": digest(r["h"], r["qx"], r["qy"])}
    (HERE / "golden.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out["acceptance"], indent=1))


if __name__ == "__main__":
    main()

"""Pinning the C oracle (oracle/swe_oracle.c) -- CPU only.

The oracle is the checker of the CUDA path, so it is itself checked against
(a) the reference's golden fixtures (tests/golden/, generated from the
reference by tests/golden/make_golden.py), (b) the reference's recorded
acceptance values (proj/test_output.txt), and (c) the compiled reference
(oracle/_ref) on fresh inputs where it is available.
"""
import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, bit_equal, random_state
from oracle.pyoracle import MeshArrays

KEYS = ("lx", "ly", "eta0", "amplitude", "sigma", "manning", "h_left", "h_right", "x_dam", "t_end")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def case_mesh(case, nx, ny, spec, still=False):
    from paper_1807_00672_b200 import api
    raw = api.generate_square_mesh(nx, ny, spec["lx"], spec["ly"])
    bed, man, st = api.init_case(case, raw, **spec)
    if still:
        st.h[:] = 0.75
    return api.build_mesh(raw, bed, man), st


@pytest.mark.parametrize("name", ["12x9_seed7", "12x9_seed8", "mounds_30x12_seed9"])
def test_oracle_fluxes_match_golden(coracle, golden, name):
    from paper_1807_00672_b200 import api
    f = np.load(GOLDEN / golden["fluxes"][name]["file"])
    if name.startswith("mounds"):
        raw = api.generate_square_mesh(30, 12, 75.0, 30.0)
        mesh, _ = api.setup_case("lake_at_rest", raw)
    else:
        raw = api.generate_square_mesh(12, 9, 4.0, 3.0)
        mesh = api.build_mesh(raw, np.zeros(raw.n_cells), np.zeros(raw.n_cells))
    left, right, bad = coracle.compute_fluxes(MeshArrays.from_mesh(mesh), f["h"], f["qx"], f["qy"])
    assert bad == -1
    assert bit_equal(left, f["left"]) and bit_equal(right, f["right"])
    assert digest(left, right) == golden["fluxes"][name]["digest"]


@pytest.mark.parametrize("name", ["water_drop_12x12_200", "still_water_8x8_25", "lake_at_rest_30x12_50",
                                  "three_mounds_100x40_t30", "dam_break_1d_100x10_t40",
                                  "water_drop_50x50_1000"])
def test_oracle_trajectories_match_golden(coracle, golden, name):
    g = golden["trajectories"][name]
    mesh, st = case_mesh(g["case"], g["nx"], g["ny"], g["spec"], g["still_water"])
    r = coracle.advance(MeshArrays.from_mesh(mesh), st.h, st.qx, st.qy, t_end=g["t_end"],
                        nsteps=g["steps"] + (1 if g["stop_at_t_end"] else 0),
                        stop_at_t_end=g["stop_at_t_end"])
    assert r["error"] is None
    assert r["step"] == g["steps"] and r["t"] == g["t"]
    assert digest(r["h"], r["qx"], r["qy"]) == g["state_digest"]
    assert digest(r["dts"]) == g["dt_digest"]
    assert r["clip_events"] == g["clip_events"] and r["clipped_volume"] == g["clipped_volume"]


def test_acceptance_c1_lake_at_rest(coracle, golden):
    """acceptance.cpp:56-79; recorded 4.441e-16 / 1.403e-13 (test_output.txt:15)."""
    from paper_1807_00672_b200 import api
    spec = api.case_defaults("lake_at_rest")
    mesh, st = case_mesh("lake_at_rest", 112, 45, spec)
    r = coracle.advance(MeshArrays.from_mesh(mesh), st.h, st.qx, st.qy, nsteps=1000)
    wet = st.h > 0
    eta = np.max(np.abs(r["h"][wet] + mesh.cell_bed[wet] - spec["eta0"]))
    q = max(np.abs(r["qx"]).max(), np.abs(r["qy"]).max())
    assert f"{eta:.3e}" == "4.441e-16" and f"{q:.3e}" == "1.403e-13"
    assert eta == golden["acceptance"]["c1"]["max_eta_err"]


def test_acceptance_c3_three_mounds_step_count(coracle, golden):
    """acceptance.cpp:101-139: exactly 1117 steps to t=30 (test_output.txt:17)."""
    from paper_1807_00672_b200 import api
    spec = api.case_defaults("three_mounds")
    spec["t_end"] = 30.0
    mesh, st = case_mesh("three_mounds", 100, 40, spec)
    r = coracle.advance(MeshArrays.from_mesh(mesh), st.h, st.qx, st.qy, t_end=30.0, nsteps=5000,
                        stop_at_t_end=True)
    assert r["step"] == 1117 and r["t"] == 30.0
    assert (r["h"] >= 0).all()
    assert coracle.total_mass(MeshArrays.from_mesh(mesh), r["h"]) == golden["acceptance"]["c3"]["mass_final"]


def test_acceptance_c9_symmetry(coracle, golden):
    """acceptance.cpp:313-332; recorded 6.661e-16 (test_output.txt:23)."""
    from paper_1807_00672_b200 import api
    spec = api.case_defaults("water_drop")
    mesh, st = case_mesh("water_drop", 48, 48, spec)
    r = coracle.advance(MeshArrays.from_mesh(mesh), st.h, st.qx, st.qy, nsteps=100)
    # rotated_cell_index (mesh.hpp:92-98)
    rot =np.array([2 * ((47 - (c // 2) // 48) * 48 + (47 - (c // 2) % 48)) + (1 - c % 2)
                    for c in range(mesh.n_cells)])
    worst = np.max(np.abs(r["h"] - r["h"][rot]))
    assert f"{worst:.3e}" == "6.661e-16"
    assert digest(r["h"], r["qx"], r["qy"]) == golden["acceptance"]["c9"]["state_digest"]


def test_acceptance_c2_mass_1000(coracle, golden):
    """acceptance.cpp:81-99 (1000 of its 10,000 steps): t = 868.4939716386242."""
    from paper_1807_00672_b200 import api
    spec = api.case_defaults("water_drop")
    mesh, st = case_mesh("water_drop", 71, 71, spec)
    ma = MeshArrays.from_mesh(mesh)
    m0 = coracle.total_mass(ma, st.h)
    r = coracle.advance(ma, st.h, st.qx, st.qy, nsteps=1000)
    assert r["t"] == 868.4939716386242 == golden["acceptance"]["c2_1000"]["t"]
    assert digest(r["h"], r["qx"], r["qy"]) == golden["acceptance"]["c2_1000"]["state_digest"]
    assert abs(coracle.total_mass(ma, r["h"]) - m0) / m0 <= 1e-12
    assert r["clip_events"] == 0


def test_oracle_error_paths(coracle):
    """NaN -> stable_dt cell (test_engine.cpp:218-227); negative depth -> edge (:229-237)."""
    from paper_1807_00672_b200 import api
    raw = api.generate_square_mesh(3, 3, 1.0, 1.0)
    mesh = api.build_mesh(raw, np.zeros(18), np.zeros(18))
    ma = MeshArrays.from_mesh(mesh)
    h, qx, qy = random_state(18, 11)
    qx[5] = np.nan
    r = coracle.advance(ma, h, qx, qy)
    assert r["error"][:2] == (1, 5)
    h, qx, qy = random_state(18, 12)
    h[0] = -0.5
    _, _, bad = coracle.compute_fluxes(ma, h, qx, qy)
    e0 = [e for e in range(mesh.n_edges) if mesh.edge_left[e] == 0 or mesh.edge_right[e] == 0]
    assert bad == min(e0)


# ---- against the compiled reference on fresh inputs (this container) ----

@pytest.mark.parametrize("seed,dry", [(1, 0.0), (2, 0.3), (3, 0.6)])
def test_oracle_vs_reference_fluxes_unstructured(coracle, refo, seed, dry):
    from paper_1807_00672_b200 import api
    raw = api.generate_unstructured_mesh(37, 23, 75.0, 30.0, seed=seed)
    mesh, _ = api.setup_case("lake_at_rest", raw)
    rm = refo.build_mesh(raw.nodes, raw.triangles, mesh.cell_bed, mesh.cell_manning)
    h, qx, qy = random_state(mesh.n_cells, seed, dry)
    l1, r1, b1 = coracle.compute_fluxes(MeshArrays.from_mesh(mesh), h, qx, qy)
    l2, r2, rc, _ = rm.compute_fluxes(h, qx, qy)
    assert rc == 0 and b1 == -1
    assert bit_equal(l1, l2) and bit_equal(r1, r2)


@pytest.mark.parametrize("manning", [0.0, 0.03])
def test_oracle_vs_reference_trajectory_friction(coracle, refo, manning):
    """Same host libm: the oracle's pow is the reference's pow, so even the
    friction path is bit-identical here."""
    from paper_1807_00672_b200 import api
    raw = api.generate_unstructured_mesh(60, 24, 75.0, 30.0, seed=5)
    mesh, st = api.setup_case("three_mounds", raw, manning=manning)
    rm = refo.build_mesh(raw.nodes, raw.triangles, mesh.cell_bed, mesh.cell_manning)
    a = coracle.advance(MeshArrays.from_mesh(mesh), st.h, st.qx, st.qy, nsteps=300)
    b = rm.advance(st.h, st.qx, st.qy, nsteps=300, threads=4)
    assert a["error"] is None and b["rc"] == 0
    for k in ("h", "qx", "qy", "dts", "max_speeds"):
        assert bit_equal(a[k], b[k]), k
    assert a["clipped_volume"] == b["clipped_volume"] and a["clip_events"] == b["clip_events"]

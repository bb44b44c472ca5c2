"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Bar: bit-identical FP64 for every frictionless path (fluxes, states, the dt
sequence); for the friction path the device pow(h, 4/3) is checked against
the host libm's and the state against the per-cell floored-relative
tolerance 1e-12 of BASELINE.json's north_star / SURVEY.md §8(c).
"""
import json
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, bit_equal, random_state
from oracle.pyoracle import MeshArrays
from paper_1807_00672_b200 import api

pytestmark = pytest.mark.gpu

FRICTION_TOL = 1e-12  # per-cell |a-b| / max(|b|, 1e-12 ||b||_inf)


def floored_rel(a, b):
    scale = np.maximum(np.abs(b), 1e-12 * max(np.abs(b).max(), 1e-300))
    return float(np.max(np.abs(a - b) / scale))


def rng_pairs(n, seed, dry=0.3, hmax=3.0, umax=4.0):
    rng = np.random.default_rng(seed)
    def st():
        h = rng.uniform(0.0, hmax, n)
        h[rng.random(n) < dry] = 0.0
        tiny = rng.random(n) < 0.05  # straddle h_dry = 1e-6
        h[tiny] = rng.uniform(0.0, 2e-6, int(tiny.sum()))
        return np.stack([h, h * rng.uniform(-umax, umax, n), h * rng.uniform(-umax, umax, n)], 1)
    a = rng.uniform(0, 2 * np.pi, n)
    return st(), st(), np.stack([np.cos(a), np.sin(a)], 1), rng.uniform(0, 2, (n, 2))


# ---------------------------------------------------------------- point physics

@pytest.mark.parametrize("kind", [0, 1, 2])
def test_point_physics_bitwise(coracle, kind):
    """hllc (kernels.hpp:72-114), wall (:156-164), reconstruction + edge combine
    (:126-152, engine.hpp:161-166) on 1e5 random wet/dry pairs."""
    l, r, nrm, z = rng_pairs(100_000, 10 + kind)
    if kind == 0:
        # identical-state shortcut (kernels.hpp:83-84) on a slice
        r[:1000] = l[:1000]
    dev = api.point_eval(kind, l, r, z, nrm)
    ref = coracle.point(kind, l, r, z, nrm)
    assert bit_equal(dev, ref)


def test_point_physics_matches_reference(refo):
    l, r, nrm, z = rng_pairs(20_000, 99)
    assert bit_equal(api.point_eval(0, l, r, None, nrm), refo.hllc(l, r, nrm))
    assert bit_equal(api.point_eval(1, l, None, None, nrm), refo.wall(l, nrm))
    left, right = refo.edge(l, r, z, nrm)
    dev = api.point_eval(2, l, r, z, nrm)
    assert bit_equal(dev[:, :3], left) and bit_equal(dev[:, 3:], right)


def test_pow43_against_host_libm(coracle):
    """kernels.hpp:197 std::pow(h, 4/3) over the depth range friction sees."""
    rng = np.random.default_rng(3)
    h = np.concatenate([rng.uniform(1e-6, 1e-3, 200_000), rng.uniform(1e-3, 10, 600_000),
                        rng.uniform(10, 100, 200_000)])
    h = np.concatenate([h, [1.0, np.nextafter(1.0, 2), np.nextafter(1.0, 0), 5e-324, 1e-310, 0.0,
                            1e300, np.inf]])
    dev = api.point_eval(4, np.stack([h, h, h], 1))
    ref = coracle.point(4, np.stack([h, h, h], 1))
    mism = np.count_nonzero(dev.view(np.uint64) != ref.view(np.uint64))
    print(f"pow43 mismatches: {mism} of {len(h)}")
    assert mism == 0


def test_friction_point(coracle):
    rng = np.random.default_rng(4)
    n = 50_000
    h = rng.uniform(0.05, 5, n)
    u = np.stack([h, h * rng.uniform(-3, 3, n), h * rng.uniform(-3, 3, n)], 1)
    z = np.stack([rng.uniform(0, 0.1, n), rng.uniform(1e-4, 10, n)], 1)
    dev = api.point_eval(3, u, None, z)
    ref = coracle.point(3, u, None, z)
    assert bit_equal(dev, ref)
    assert np.all(np.abs(dev[:, 1]) <= np.abs(u[:, 1])) and np.all(dev[:, 1] * u[:, 1] >= 0)


# ---------------------------------------------------------------- compute_fluxes

def mesh_for(kind, seed=1):
    if kind == "flat":
        raw = api.generate_square_mesh(12, 9, 4.0, 3.0)
        return api.build_mesh(raw, np.zeros(raw.n_cells), np.zeros(raw.n_cells))
    if kind == "mounds":
        return api.setup_case("lake_at_rest", api.generate_square_mesh(30, 12, 75.0, 30.0))[0]
    raw = api.generate_unstructured_mesh(90, 36, 75.0, 30.0, seed=seed)
    return api.setup_case("lake_at_rest", raw)[0]


@pytest.mark.parametrize("name", ["12x9_seed7", "12x9_seed8", "mounds_30x12_seed9"])
def test_fluxes_match_reference_golden(golden, name):
    f = np.load(GOLDEN / golden["fluxes"][name]["file"])
    mesh = mesh_for("mounds" if name.startswith("mounds") else "flat")
    st = api.FieldState(f["h"], f["qx"], f["qy"])
    left, right = api.compute_fluxes(st, mesh)
    assert bit_equal(left, f["left"]) and bit_equal(right, f["right"])


@pytest.mark.parametrize("identity", [False, True])
@pytest.mark.parametrize("dry", [0.0, 0.3, 0.7])
def test_fluxes_unstructured_bitwise(coracle, identity, dry):
    mesh = mesh_for("unstructured", seed=2)
    h, qx, qy = random_state(mesh.n_cells, 5, dry)
    s = api.DeviceSolver(mesh, identity_order=identity)
    s.set_state(api.FieldState(h, qx, qy))
    left, right = s.compute_fluxes()
    l2, r2, bad = coracle.compute_fluxes(MeshArrays.from_mesh(mesh), h, qx, qy)
    assert bad == -1 and bit_equal(left, l2) and bit_equal(right, r2)


def test_negative_depth_reports_lowest_edge(coracle):
    """test_engine.cpp:229-237 -- the lowest edge index, as the sequential backend."""
    mesh = mesh_for("unstructured", seed=3)
    h, qx, qy = random_state(mesh.n_cells, 12)
    h[[17, 400, 901]] = -0.5
    _, _, bad = coracle.compute_fluxes(MeshArrays.from_mesh(mesh), h, qx, qy)
    with pytest.raises(api.NumericError, match=f"compute_fluxes: negative depth at edge {bad}$"):
        api.compute_fluxes(api.FieldState(h, qx, qy), mesh)


# ---------------------------------------------------------------- trajectories

def golden_case(g):
    raw = api.generate_square_mesh(g["nx"], g["ny"], g["spec"]["lx"], g["spec"]["ly"])
    mesh, st = api.setup_case(g["case"], raw, **g["spec"])
    if g["still_water"]:
        st.h[:] = 0.75
    return mesh, st


def digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("two_phase", [False, True], ids=["fused", "two_phase"])
@pytest.mark.parametrize("name", ["water_drop_12x12_200", "still_water_8x8_25", "lake_at_rest_30x12_50",
                                  "dam_break_1d_100x10_t40", "water_drop_50x50_1000",
                                  "three_mounds_100x40_t30"])
def test_trajectory_vs_reference_golden(golden, coracle, name, two_phase):
    """Device run loop (one graph launch) against the reference's trajectories."""
    g = golden["trajectories"][name]
    mesh, st = golden_case(g)
    s = api.DeviceSolver(mesh, two_phase=two_phase)
    s.set_state(st)
    recs = s.advance(t_end=g["t_end"], max_steps=g["steps"])
    got, t, step = s.get_state()
    # bit-identical to the reference, friction included (swe_pow.cuh restates
    # the host glibc pow exactly)
    assert step == g["steps"] and t == g["t"]
    assert digest(got.h, got.qx, got.qy) == g["state_digest"]
    assert digest(recs[:, 2]) == g["dt_digest"]
    assert s.ledger()[1] == g["clip_events"]


@pytest.mark.parametrize("two_phase", [False, True], ids=["fused", "two_phase"])
def test_config1_circular_dam_break_1000_steps(coracle, two_phase):
    """BASELINE configs[0]: ~10k-triangle unstructured circular dam break, 1000 steps."""
    sc = api.make_scenario("circular_dam_break")
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    s = api.DeviceSolver(mesh, two_phase=two_phase)
    s.set_state(sc.state)
    recs = s.advance(t_end=1e30, max_steps=1000)
    got, t, step = s.get_state()
    ref = coracle.advance(MeshArrays.from_mesh(mesh), sc.state.h, sc.state.qx, sc.state.qy,
                          nsteps=1000)
    assert step == 1000 and t == ref["t"]
    for k, a in (("h", got.h), ("qx", got.qx), ("qy", got.qy)):
        assert bit_equal(a, ref[k]), k
    assert bit_equal(recs[:, 2], ref["dts"]) and bit_equal(recs[:, 3], ref["max_speeds"])
    m = recs[:, 4]
    assert abs(m[-1] - m[0]) <= 1e-12 * m[0]


@pytest.mark.parametrize("two_phase", [False, True], ids=["fused", "two_phase"])
@pytest.mark.parametrize("scenario", ["three_mounds_friction", "sloping_wet_dry", "channel"])
def test_friction_scenarios_scaled(coracle, scenario, two_phase):
    """Configs 2-4 at reduced resolution: wet/dry fronts + bathymetry + Manning."""
    sc = api.make_scenario(scenario, scale=0.04 if scenario != "three_mounds_friction" else 0.1)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    s = api.DeviceSolver(mesh, two_phase=two_phase)
    s.set_state(sc.state)
    recs = s.advance(t_end=1e30, max_steps=300)
    got, t, step = s.get_state()
    ref = coracle.advance(MeshArrays.from_mesh(mesh), sc.state.h, sc.state.qx, sc.state.qy,
                          nsteps=300)
    assert ref["error"] is None and step == 300 and t == ref["t"]
    for k, a in (("h", got.h), ("qx", got.qx), ("qy", got.qy)):
        assert floored_rel(a, ref[k]) <= FRICTION_TOL, k  # the north_star bar ...
        assert bit_equal(a, ref[k]), k                    # ... and the one we hold
    assert bit_equal(recs[:, 2], ref["dts"])
    assert s.ledger()[1] == ref["clip_events"]


def test_oversized_tile_is_rejected(monkeypatch):
    monkeypatch.setenv("SWE_TILE_CELLS", "8192")
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    with pytest.raises(api.DeviceError, match="shared memory"):
        api.DeviceSolver(mesh)


@pytest.mark.parametrize("threads", [128, 256])
@pytest.mark.parametrize("tile_cells", [32, 100, 256, 1024])
def test_tile_sizes_agree(coracle, monkeypatch, tile_cells, threads):
    monkeypatch.setenv("SWE_TILE_THREADS", str(threads))
    """The fused kernel's result does not depend on the tile size (halo edges
    are evaluated by both tiles from identical inputs)."""
    monkeypatch.setenv("SWE_TILE_CELLS", str(tile_cells))
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    s = api.DeviceSolver(mesh)
    assert s.info()["tile_cells"] == tile_cells and s.info()["fused"] == 1
    s.set_state(sc.state)
    recs = s.advance(t_end=1e30, max_steps=120)
    got = s.get_state()[0]
    ref = coracle.advance(MeshArrays.from_mesh(mesh), sc.state.h, sc.state.qx, sc.state.qy,
                          nsteps=120)
    assert bit_equal(got.h, ref["h"]) and bit_equal(got.qx, ref["qx"]) and bit_equal(got.qy, ref["qy"])
    assert bit_equal(recs[:, 2], ref["dts"])


def test_morton_and_identity_order_agree():
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    out = []
    for identity in (False, True):
        s = api.DeviceSolver(mesh, identity_order=identity)
        s.set_state(sc.state)
        recs = s.advance(t_end=1e30, max_steps=200)
        out.append((s.get_state()[0], recs))
    (a, ra), (b, rb) = out
    assert bit_equal(a.h, b.h) and bit_equal(a.qx, b.qx) and bit_equal(a.qy, b.qy)
    assert bit_equal(ra[:, 2], rb[:, 2])


# ---------------------------------------------------------------- engine API

def test_advance_step_api_vs_oracle(coracle):
    """swe::advance_step host-resident contract, including the clip ledger."""
    sc = api.make_scenario("sloping_wet_dry", scale=0.02)
    mesh = api.build_mesh(sc.raw, sc.bed, np.zeros_like(sc.manning))
    st = sc.state.copy()
    r = api.advance(mesh, st, nsteps=40)
    o = coracle.advance(MeshArrays.from_mesh(mesh), sc.state.h, sc.state.qx, sc.state.qy, nsteps=40)
    assert bit_equal(st.h, o["h"]) and bit_equal(st.qx, o["qx"]) and bit_equal(st.qy, o["qy"])
    assert bit_equal(r.dts, o["dts"]) and bit_equal(r.max_speeds, o["max_speeds"])
    assert r.clip_events == o["clip_events"]
    assert abs(r.clipped_volume - o["clipped_volume"]) <= 1e-12 * max(abs(o["clipped_volume"]), 1e-300)


def test_run_api_truncates_and_snapshots(coracle):
    """engine.hpp:335-394 + test_engine.cpp:249-299."""
    raw = api.generate_square_mesh(4, 4, 1.0, 1.0)
    mesh = api.build_mesh(raw, np.zeros(32), np.zeros(32))
    st = api.FieldState(np.ones(32), np.zeros(32), np.zeros(32))
    r = api.run(mesh, st, t_end=1e-6)
    assert r.step == 1 and r.t == 1e-6 and r.stats["t_final"] == 1e-6
    st = api.FieldState(np.ones(32), np.zeros(32), np.zeros(32))
    r = api.run(mesh, st, t_end=0.2, snapshot_interval=0.08, snapshots=True)
    assert len(r.snapshots) >= 3 and r.snapshots[0] == 0.0 and abs(r.snapshots[-1] - 0.2) < 1e-12
    with pytest.raises(api.ConfigError):
        api.run(mesh, st, t_end=0.0)
    with pytest.raises(api.NumericError, match="exceeded max_steps=3"):
        api.run(mesh, api.FieldState(np.ones(32), np.zeros(32), np.zeros(32)), t_end=10.0,
                max_steps=3)


def test_run_api_series_vs_oracle(coracle, golden):
    g = golden["trajectories"]["dam_break_1d_100x10_t40"]
    mesh, st = golden_case(g)
    st0 = st.copy()
    r = api.run(mesh, st, t_end=40.0)
    o = coracle.advance(MeshArrays.from_mesh(mesh), st0.h, st0.qx, st0.qy, t_end=40.0, nsteps=10**6,
                        stop_at_t_end=True)
    assert r.step == o["step"] and r.t == 40.0
    assert bit_equal(r.series[:, 2], o["dts"]) and bit_equal(r.series[:, 3], o["max_speeds"])
    assert digest(st.h, st.qx, st.qy) == g["state_digest"]
    masses = r.series[:, 4]
    assert np.all(np.abs(masses - r.stats["mass_initial"]) <= 1e-12 * r.stats["mass_initial"])
    assert r.stats["mean_dt"] == np.sum(o["dts"]) / r.step or abs(r.stats["mean_dt"] * r.step - 40.0) < 1e-9


def test_errors_match_reference_messages(coracle):
    """NaN -> 'stable_dt: non-finite velocity in cell 5' (test_engine.cpp:218-227),
    blow-up -> 'advance_step: numeric blowup at step N, cell C, dt D (h=H)'."""
    raw = api.generate_square_mesh(3, 3, 1.0, 1.0)
    mesh = api.build_mesh(raw, np.zeros(18), np.zeros(18))
    h, qx, qy = random_state(18, 11)
    qx[5] = np.nan
    with pytest.raises(api.NumericError, match="stable_dt: non-finite velocity in cell 5$"):
        api.advance(mesh, api.FieldState(h, qx, qy))
    # an unstable Courant number drives a blow-up; compare with the oracle's report
    p = api.PhysParams(cfl=40.0)
    from oracle.pyoracle import so_params  # noqa: F401
    h, qx, qy = random_state(18, 3)
    o = coracle.advance(MeshArrays.from_mesh(mesh), h, qx, qy, nsteps=50, params=p)
    assert o["error"] is not None
    kind, cell, hval = o["error"]
    st = api.FieldState(h.copy(), qx.copy(), qy.copy())
    with pytest.raises(api.NumericError) as ei:
        api.advance(mesh, st, nsteps=50, params=p)
    msg = str(ei.value)
    if kind == 3:
        assert f"cell {cell}," in msg and "numeric blowup at step" in msg and f"(h={hval:f})" in msg
    assert bit_equal(st.h, o["h"])  # state = last good step


def test_reproducible_and_mass_conserving_full_size():
    """BASELINE configs[2] at full size (10M cells): run twice bitwise; mass
    balance to round-off (change = clipped volume only)."""
    sc = api.make_scenario("channel")
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    s = api.DeviceSolver(mesh)
    outs = []
    for _ in range(2):
        s.set_state(sc.state)
        m0 = s.total_mass()
        recs = s.advance(t_end=1e30, max_steps=30)
        outs.append((s.get_state()[0], recs, m0))
    (a, ra, m0), (b, rb, _) = outs
    assert bit_equal(a.h, b.h) and bit_equal(a.qx, b.qx) and bit_equal(ra[:, 2], rb[:, 2])
    clipped, _ = s.ledger()
    assert abs(ra[-1, 4] - m0) <= 1e-12 * m0 + 2 * clipped


def test_cpp_drop_in_driver(golden):
    """A reference-API caller (tests/cpp/api_driver.cpp) on the device engine."""
    exe = ROOT / "tests" / "cpp" / "api_driver"
    out = json.loads(subprocess.run([str(exe)], capture_output=True, text=True, check=True,
                                    timeout=600).stdout)
    assert out["c3_steps"] == 1117 and out["c3_positive"] and out["c3_t"] == 30.0
    assert out["run_steps"] == 1000 and out["run_t"] == golden["acceptance"]["c2_1000"]["t"]
    assert out["run_snaps"] == 1 + 5 and abs(out["run_drift"]) <= 1e-12
    assert out["uniform_mass_antisymmetric"] and abs(out["mass_unit"] - 6.0) <= 6e-14  # 3 m x 2 m
    assert out["nan_msg"] == "stable_dt: non-finite velocity in cell 5"
    assert out["neg_msg"].startswith("compute_fluxes: negative depth at edge ")
    assert out["cfg_msg"] == "run: t_end must be > 0"
    # the device cache keys on content; helpers inside on_snapshot leave run() intact
    assert out["cache_mutation_ok"] and out["reentrant_ok"]


def test_advance_async_equals_advance():
    """swe_dev_advance_async + swe_dev_records == swe_dev_advance."""
    sc = api.make_scenario("three_mounds_friction", scale=0.05)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    a, b = api.DeviceSolver(m), api.DeviceSolver(m)
    a.set_state(sc.state)
    b.set_state(sc.state)
    ra = a.advance(1e30, max_steps=120)
    b.advance_async(1e30, max_steps=60)
    b.advance_async(1e30, max_steps=120)  # two launches queued back to back
    rb = b.records()
    assert len(rb) == 60 and bit_equal(rb, ra[60:])
    sa, _, _ = a.get_state()
    sb, _, _ = b.get_state()
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(sa, k), getattr(sb, k)), k


@pytest.mark.parametrize("sync", [False, True], ids=["async", "sync"])
def test_run_snapshots_are_the_states_at_their_steps(coracle, monkeypatch, sync):
    """run()'s snapshots (copied D2H while the next segment already steps)
    equal the oracle's state at the snapshot's step, bit for bit."""
    if sync:
        monkeypatch.setenv("SWE_SYNC_SNAPSHOTS", "1")
    sc = api.make_scenario("three_mounds_friction", scale=0.05)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning)
    st = sc.state.copy()
    r = api.run(mesh, st, t_end=6.0, snapshot_interval=1.0, snapshots=True, snapshot_fields=8)
    assert len(r.snapshots) == 7 and r.snapshots[0] == 0.0 and r.snapshots[-1] == 6.0
    steps = {t: int(s) for s, t in r.series[:, :2]}
    m = MeshArrays.from_mesh(mesh)
    for ts, f in zip(r.snapshots[1:], r.fields[1:]):
        k = steps[ts]
        o = coracle.advance(m, sc.state.h, sc.state.qx, sc.state.qy, t_end=6.0, nsteps=k)
        for j, key in enumerate(("h", "qx", "qy")):
            assert bit_equal(f[j], o[key]), (ts, key)
    o = coracle.advance(m, sc.state.h, sc.state.qx, sc.state.qy, t_end=6.0, nsteps=10**6,
                        stop_at_t_end=True)
    assert bit_equal(st.h, o["h"]) and r.step == o["step"]


def test_staged_tile_option_is_bit_identical(coracle, monkeypatch):
    """SWE_TILE_STAGE=1 (cp.async-staged tiles) == oracle."""
    monkeypatch.setenv("SWE_TILE_STAGE", "1")
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    s = api.DeviceSolver(m)
    assert s.info()["tile_cells"] <= 128
    s.set_state(sc.state)
    recs = s.advance(1e30, max_steps=120)
    got, _, _ = s.get_state()
    o = coracle.advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy, nsteps=120)
    assert bit_equal(recs[:, 2], o["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), o[k]), k


def _square_case(nx, ny, seed, dry_frac=0.3):
    raw = api.generate_square_mesh(nx, ny, float(nx), float(ny))
    n = raw.n_cells
    rng = np.random.default_rng(seed)
    bed = rng.uniform(0.0, 0.3, n)
    man = np.where(rng.random(n) < 0.5, 0.03, 0.0)
    h = np.where(rng.random(n) < dry_frac, 0.0, rng.uniform(0.2, 2.0, n))
    qx = np.where(h > 0, rng.uniform(-1, 1, n) * h, 0.0)
    qy = np.where(h > 0, rng.uniform(-1, 1, n) * h, 0.0)
    return api.build_mesh(raw, bed, man), api.FieldState(h, qx, qy)


@pytest.mark.parametrize("nx,ny", [(1, 1), (1, 2), (2, 1), (3, 1), (5, 4)])
def test_tiny_meshes_bitwise(coracle, nx, ny):
    """the smallest meshes: every cell on the boundary, tiles of one cell"""
    m, st = _square_case(nx, ny, seed=nx * 10 + ny)
    s = api.DeviceSolver(m)
    s.set_state(st)
    recs = s.advance(1e30, max_steps=60)
    got, _, _ = s.get_state()
    o = coracle.advance(MeshArrays.from_mesh(m), st.h, st.qx, st.qy, nsteps=60)
    assert bit_equal(recs[:, 2], o["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), o[k]), k


def test_all_dry_domain_steps_with_dt_max(coracle):
    """engine.hpp:214: every cell dry -> dt = dt_max, nothing moves"""
    m, st = _square_case(20, 10, seed=3, dry_frac=1.0)
    s = api.DeviceSolver(m)
    s.set_state(st)
    recs = s.advance(1e30, max_steps=5)
    assert np.all(recs[:, 2] == api.PhysParams().dt_max) and np.all(recs[:, 4] == 0.0)
    got, t, _ = s.get_state()
    assert t == 5 * api.PhysParams().dt_max and not np.any(got.h) and not np.any(got.qx)


def test_single_wet_cell_spreads_into_dry_cells(coracle):
    """a wetting front from one cell: dry-bed HLLC branches and the clamp"""
    m, st = _square_case(30, 30, seed=5, dry_frac=1.0)
    st.h[450] = 2.0
    s = api.DeviceSolver(m)
    s.set_state(st)
    recs = s.advance(1e30, max_steps=200)
    got, _, _ = s.get_state()
    o = coracle.advance(MeshArrays.from_mesh(m), st.h, st.qx, st.qy, nsteps=200)
    assert bit_equal(recs[:, 2], o["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), o[k]), k
    assert np.count_nonzero(got.h) > 50


def test_dry_tile_skipping_is_exercised_and_bit_identical(coracle, monkeypatch):
    """dry-tile skipping: on a mostly dry bed many tiles are
    skipped, and states, dt and the mass series equal the no-skip run and the
    oracle bit for bit"""
    sc = api.make_scenario("sloping_wet_dry", scale=0.04)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    runs = {}
    for skip in (True, False):
        if not skip:
            monkeypatch.setenv("SWE_NO_DRY_SKIP", "1")
        s = api.DeviceSolver(m)
        s.set_state(sc.state)
        recs = s.advance(1e30, max_steps=300)
        got, _, _ = s.get_state()
        runs[skip] = (recs, got, s.info())
    assert runs[True][2]["dry_skip"] == 1 and runs[False][2]["dry_skip"] == 0
    assert runs[True][2]["skipped_tiles"] > 0.2 * 300 * runs[True][2]["tiles"]
    assert bit_equal(runs[True][0], runs[False][0])  # dt, max speed AND mass series
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(runs[True][1], k), getattr(runs[False][1], k)), k
    o = coracle.advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy, nsteps=300)
    assert bit_equal(runs[True][0][:, 2], o["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(runs[True][1], k), o[k]), k


@pytest.mark.parametrize("config,scale,steps", [("three_mounds_friction", 1.0, 3000),
                                                ("sloping_wet_dry", 0.3, 3000)])
def test_dry_skip_long_runs_equal_no_skip(monkeypatch, config, scale, steps):
    """~1M cells, thousands of steps while fronts sweep over dry tiles: the
    skipping run equals the full evaluation bit for bit (state, dt, speed,
    mass series, clip ledger)"""
    sc = api.make_scenario(config, scale=scale)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    out = []
    for off in ("0", "1"):
        monkeypatch.setenv("SWE_NO_DRY_SKIP", off)
        s = api.DeviceSolver(m)
        s.set_state(sc.state)
        recs = s.advance(1e30, max_steps=steps)
        st, t, n = s.get_state()
        out.append((recs, st, t, n, s.ledger(), s.info()))
        s.close()
    (ra, sa, ta, na, la, ia), (rb, sb, tb, nb, lb, ib) = out
    assert ia["dry_skip"] == 1 and ib["dry_skip"] == 0 and ia["skipped_tiles"] > 0
    assert na == nb == steps and ta == tb and la == lb
    assert bit_equal(ra, rb)
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(sa, k), getattr(sb, k)), k


@pytest.mark.parametrize("config", ["channel", "sloping_wet_dry"])
def test_full_size_steps_bitwise_vs_reference(refo, config):
    """BASELINE configs [2] / [3] at FULL size (10.26M cells): the bench's
    timed window -- steps [W, W+K) = [5, 25) from the initial state with the
    driver's --warmup 5 --steps 20 -- on the device (dry-tile skipping on)
    equals the reference's own advance_step (oracle/_ref, all host threads)
    bit for bit: state, dt, max speed and the clip ledger's event count."""
    import os
    n = 25
    sc = api.make_scenario(config)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    s = api.DeviceSolver(mesh)
    s.set_state(sc.state)
    recs = s.advance(1e30, max_steps=n)
    got, _, _ = s.get_state()
    _, ev = s.ledger()
    info = s.info()
    s.close()
    rm = refo.build_mesh(sc.raw.nodes, sc.raw.triangles, sc.bed, sc.manning)
    r = rm.advance(sc.state.h, sc.state.qx, sc.state.qy, t_end=1e30, nsteps=n,
                   threads=len(os.sched_getaffinity(0)))
    assert r["rc"] == 0 and r["done"] == n
    assert info["dry_skip"] == 1 and info["skipped_tiles"] > 0
    assert bit_equal(recs[:, 2], r["dts"]) and bit_equal(recs[:, 3], r["max_speeds"])
    assert ev == r["clip_events"]
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), r[k]), k

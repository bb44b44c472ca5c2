"""The persistent step kernel (k_run, csrc/swe_step.cuh): the run loop as ONE
cooperative launch with a grid barrier per step, the commit by the last CTA to
arrive, and the next step's first flux tile evaluated before the commit is
published.  It must reproduce the CUDA-graph loop (k_tile + k_finalize,
SWE_PERSISTENT=0) bit for bit -- state, dt / max speed / mass records, clip
ledger, dry-tile skip decisions -- and the reference (oracle).

Linked ranks: P parts on ONE device stepped by one cooperative launch over all
ranks (swe_dev_run_ranks) -- their CTAs run concurrently and spin on each
other's mailbox flags (acquire / release at system scope), the path a P-GPU
run takes, without lockstep phases."""
import os

import numpy as np
import pytest

from conftest import bit_equal
from oracle.pyoracle import COracle, MeshArrays
from paper_1807_00672_b200 import api, dist

pytestmark = pytest.mark.gpu

CASES = [("sloping_wet_dry", 0.03), ("three_mounds_friction", 0.05), ("circular_dam_break", 1.0),
         ("channel", 0.04)]


def solver(mesh, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return api.DeviceSolver(mesh)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name,scale", CASES)
def test_persistent_equals_graph_loop(name, scale):
    sc = api.make_scenario(name, scale=scale)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    a, b = solver(m), solver(m, SWE_PERSISTENT=0)
    assert a.info()["persistent"] == 1 and b.info()["persistent"] == 0
    out = []
    for s in (a, b):
        s.set_state(sc.state)
        recs = np.concatenate([s.advance(1e30, max_steps=k) for k in (1, 77, 160, 400)])
        st, t, step = s.get_state()
        out.append((st, t, step, recs, s.ledger(), s.info()["skipped_tiles"]))
    (sa, ta, na, ra, la, ka), (sb, tb, nb, rb, lb, kb) = out
    assert na == nb == 400 and ta == tb
    assert bit_equal(ra, rb)  # step, t, dt, max_speed AND the mass series
    assert la == lb and ka == kb
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(sa, k), getattr(sb, k)), k


def test_persistent_matches_oracle_with_many_tiles_per_cta(coracle):
    """Two worker CTAs: every one walks hundreds of tiles, so its skip decisions are
    formed in several chunks (kRunDec) per step."""
    sc = api.make_scenario("sloping_wet_dry", scale=0.05)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    s = solver(m, SWE_RUN_GRID=2)
    info = s.info()
    assert info["grid_run"] == 3 and info["tiles"] > 2 * 128  # 2 workers + the control block
    s.set_state(sc.state)
    recs = s.advance(1e30, max_steps=200)
    got, _, _ = s.get_state()
    ref = coracle.advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                          nsteps=200)
    assert bit_equal(recs[:, 2], ref["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), ref[k]), k
    assert s.info()["skipped_tiles"] > 0


def test_persistent_stops_like_the_reference_loop():
    """t_end truncation (engine.hpp:236-237), snapshot stops and max_steps in
    one launch each, as the graph loop does."""
    sc = api.make_scenario("three_mounds_friction", scale=0.04)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    a, b = solver(m), solver(m, SWE_PERSISTENT=0)
    res = []
    for s in (a, b):
        s.set_state(sc.state)
        r1 = s.advance(2.5, next_snapshot=1.0)        # stops at the snapshot
        r2 = s.advance(2.5)                           # lands exactly on t_end
        r3 = s.advance(1e30, max_steps=int(r2[-1, 0]) + 3)
        st, t, step = s.get_state()
        res.append((r1, r2, r3, st, t, step))
    for x, y in zip(res[0], res[1]):
        if isinstance(x, np.ndarray):
            assert bit_equal(x, y)
        elif isinstance(x, api.FieldState):
            assert bit_equal(x.h, y.h) and bit_equal(x.qx, y.qx)
        else:
            assert x == y
    assert res[0][1][-1, 1] == 2.5 and res[0][0][-1, 1] >= 1.0 - 1e-12


def _linked(P, scale=0.03, name="sloping_wet_dry"):
    sc = api.make_scenario(name, scale=scale)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, P)
    parts = [dist.LinkedPart(dist.local_mesh(m, part, p)) for p in range(P)]
    dist.link_local(parts)
    for p in parts:
        p.set_state(sc.state)
    return sc, m, parts


@pytest.mark.parametrize("P", [2, 3, 4])
def test_linked_ranks_run_concurrently_in_one_launch(P):
    sc, m, parts = _linked(P)
    recs = np.concatenate([dist.run_ranks(parts, 70), dist.run_ranks(parts, 80)])
    got = api.FieldState.zeros(m.n_cells)
    for p in parts:
        _, step = p.gather_owned(got)
        assert step == 150
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=150)
    assert bit_equal(recs[:, 2], ref["dts"]) and bit_equal(recs[:, 3], ref["max_speeds"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), ref[k]), k


def test_linked_ranks_one_cta_each_many_tiles():
    sc, m, parts = _linked(2, scale=0.05)
    recs = dist.run_ranks(parts, 60, grid=2)  # one worker + the control block per rank
    got = api.FieldState.zeros(m.n_cells)
    for p in parts:
        p.gather_owned(got)
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=60)
    assert bit_equal(recs[:, 2], ref["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), ref[k]), k


def test_linked_ranks_error_stops_every_rank():
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, 2)
    lms = [dist.local_mesh(m, part, p) for p in range(2)]
    parts = [dist.LinkedPart(lm) for lm in lms]
    dist.link_local(parts)
    st = sc.state.copy()
    bad = int(lms[1].cells[7])
    st.h[bad] = 1.0
    st.qx[bad] = np.nan
    for p in parts:
        p.set_state(st)
    with pytest.raises(api.NumericError, match=f"non-finite velocity in cell {bad}$"):
        dist.run_ranks(parts, 5)


def test_cell_skip_pattern_matches_the_graph_loop():
    """swe_dev_cell_skip (the cost pattern behind measured_cost_weights) reads
    the persistent kernel's own dry-tile flags."""
    sc = api.make_scenario("sloping_wet_dry", scale=0.05)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    a, b = solver(m), solver(m, SWE_PERSISTENT=0)
    pats = []
    for s in (a, b):
        s.set_state(sc.state)
        s.advance(1e30, max_steps=30)
        pats.append(s.cell_skip())
    assert pats[0].sum() > 0 and np.array_equal(pats[0], pats[1])


@pytest.mark.parametrize("name", ["three_mounds_friction", "channel"])
def test_persistent_full_size_equals_graph_loop(name):
    """Full size (1.06M / 10.26M cells, 1183 workers, many tiles per worker):
    the persistent kernel and the graph loop are the same computation bit for
    bit (the 10M mesh runs the graph loop by default)."""
    sc = api.make_scenario(name)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    a, b = solver(m, SWE_PERSISTENT=1), solver(m, SWE_PERSISTENT=0)
    if name == "channel":
        assert solver(m).info()["persistent"] == 0
    assert a.info()["persistent"] == 1 and b.info()["persistent"] == 0
    out = []
    for s in (a, b):
        s.set_state(sc.state)
        recs = np.concatenate([s.advance(1e30, max_steps=k) for k in (3, 60)])
        st, t, step = s.get_state()
        out.append((st, recs, s.ledger()))
        s.close()
    (sa, ra, la), (sb, rb, lb) = out
    assert bit_equal(ra, rb) and la == lb
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(sa, k), getattr(sb, k)), k


@pytest.mark.timeout(120)
def test_linked_step_exchange_timeout_stops_the_persistent_kernel():
    """A peer that stops posting mid-run: the control CTA's wait for the step
    outcome (split exchange, swe_ctl.cuh wait_commit_head) times out, the
    workers see a stop in the published view, and the run ends with an error
    instead of a hang."""
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, 2)
    parts = [dist.LinkedPart(dist.local_mesh(m, part, p)) for p in range(2)]
    assert all(api.DeviceSolver.info(p)["persistent"] == 1 for p in parts)
    dist.link_local(parts, timeout_s=0.5)
    for p in parts:
        p.set_state(sc.state)
    recs = dist.run_ranks(parts, 6)  # both ranks: the CFL cache is formed, 6 steps
    assert len(recs) == 6
    with pytest.raises(api.DeviceError):
        parts[0].advance(max_steps=int(recs[-1, 0]) + 4)  # rank 1 never posts again

"""Parity where the numbers are measured.

* deep operating point: the 10M channel / dry bed stepped 2000 steps on the
  device (the flood well developed, ~1 s of stepping, where the round-1 bench
  timed), then 20 more steps from that state on the device and on the
  reference itself (oracle/_ref, all host threads): bit-identical state, dt,
  max speed and clip events;
* BASELINE config [1] (1,058,000-cell three-mound flood, Manning n = 0.03)
  over 3000 steps against the reference: bit-identical (friction included);
* BASELINE config [4] at its largest rung (the nx = 6406 square,
  2 x 6406^2 = 82,073,672 cells; SURVEY.md §8(a) prints 82,076,872): 8
  linked parts in lockstep on one GPU equal the single-domain run over 20
  steps (the single-domain path is pinned to the reference above).
"""
import os

import numpy as np
import pytest

from conftest import bit_equal
from paper_1807_00672_b200 import api, dist

pytestmark = pytest.mark.gpu

THREADS = len(os.sched_getaffinity(0))


@pytest.mark.parametrize("config", ["channel", "sloping_wet_dry"])
def test_deep_operating_point_bitwise_vs_reference(refo, config):
    sc = api.make_scenario(config)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    s = api.DeviceSolver(mesh)
    s.set_state(sc.state)
    for target in range(500, 2001, 500):
        s.advance(1e30, max_steps=target)
    start, t0, step0 = s.get_state()
    clipped0, ev0 = s.ledger()
    assert step0 == 2000
    recs = s.advance(1e30, max_steps=step0 + 20)
    got, t1, _ = s.get_state()
    _, ev1 = s.ledger()
    skipped = s.info()["skipped_tiles"]
    s.close()
    rm = refo.build_mesh(sc.raw.nodes, sc.raw.triangles, sc.bed, sc.manning)
    r = rm.advance(start.h, start.qx, start.qy, t=t0, step=step0, t_end=1e30, nsteps=20,
                   threads=THREADS, clipped_volume=clipped0, clip_events=ev0)
    assert r["rc"] == 0 and r["done"] == 20 and r["step"] == 2020
    assert skipped > 0  # dry-tile skipping active at the operating point
    assert bit_equal(recs[:, 2], r["dts"]) and bit_equal(recs[:, 3], r["max_speeds"])
    assert r["t"] == t1 and ev1 == r["clip_events"]
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), r[k]), k


def test_three_mounds_1M_3000_steps_bitwise_vs_reference(refo):
    sc = api.make_scenario("three_mounds_friction")
    assert sc.raw.n_cells == 1_058_000
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    s = api.DeviceSolver(mesh)
    s.set_state(sc.state)
    recs = np.concatenate([s.advance(1e30, max_steps=k) for k in (1000, 2000, 3000)])
    got, t, step = s.get_state()
    clipped, ev = s.ledger()
    s.close()
    rm = refo.build_mesh(sc.raw.nodes, sc.raw.triangles, sc.bed, sc.manning)
    r = rm.advance(sc.state.h, sc.state.qx, sc.state.qy, t_end=1e30, nsteps=3000,
                   threads=THREADS)
    assert r["rc"] == 0 and r["done"] == 3000 and step == 3000 and t == r["t"]
    assert bit_equal(recs[:, 2], r["dts"]) and bit_equal(recs[:, 3], r["max_speeds"])
    assert ev == r["clip_events"]
    assert abs(clipped - r["clipped_volume"]) <= 1e-12 * max(1.0, r["clipped_volume"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), r[k]), k
    m_ref = rm.total_mass(r["h"])
    assert abs(recs[-1, 4] - m_ref) <= 1e-12 * m_ref


def test_weak_square_82M_eight_linked_parts_match_single_domain():
    sc = api.make_scenario("weak_square", weak_nx=6406)
    mesh = api.build_mesh(sc.raw, sc.bed, sc.manning, device=0)
    C = mesh.n_cells
    assert C == 2 * 6406 * 6406  # 82,073,672
    s = api.DeviceSolver(mesh)
    s.set_state(sc.state)
    ref_recs = s.advance(1e30, max_steps=20)
    want, _, _ = s.get_state()
    s.close()
    del s
    part = dist.partition(mesh, 8)
    lms = [dist.local_mesh(mesh, part, p) for p in range(8)]
    parts = [dist.LinkedPart(lm) for lm in lms]
    dist.link_local(parts)
    for p in parts:
        p.set_state(sc.state)
    recs = dist.run_lockstep(parts, 20)
    got = api.FieldState.zeros(C)
    for p in parts:
        _, step = p.gather_owned(got)
        assert step == 20
        p.close()
    assert bit_equal(recs[:, 2], ref_recs[:, 2]) and bit_equal(recs[:, 3], ref_recs[:, 3])
    assert np.allclose(recs[:, 4], ref_recs[:, 4], rtol=1e-12, atol=0)
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), getattr(want, k)), k

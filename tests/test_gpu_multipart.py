"""Decomposed-domain runs on the device: P part contexts
with ghost cells and halo exchange (include/swe_dev.h multi-device entries),
driven in one process on one GPU, must be bit-identical to the single-domain
run -- the same machinery a multi-GPU run uses with NCCL moving the blocks."""
import numpy as np
import pytest

from conftest import bit_equal
from oracle.pyoracle import COracle, MeshArrays
from paper_1807_00672_b200 import api, dist

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("two_phase", [False, True], ids=["fused", "two_phase"])
def test_parts_on_one_gpu_match_single_domain(P, two_phase):
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, P)
    parts = [dist.PartSolver(dist.local_mesh(m, part, p), two_phase=two_phase) for p in range(P)]
    for p in parts:
        p.set_state(sc.state)
    ex = dist.LocalExchange(parts)
    recs = dist.run_parts(parts, ex, 150)
    got = api.FieldState.zeros(m.n_cells)
    for p in parts:
        t, step = p.gather_owned(got)
        assert step == 150
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=150)
    assert bit_equal(recs[:, 1], ref["dts"]) and bit_equal(recs[:, 2], ref["max_speeds"])
    for k, a in (("h", got.h), ("qx", got.qx), ("qy", got.qy)):
        assert bit_equal(a, ref[k]), k
    m0 = recs[0, 3]
    assert abs(recs[-1, 3] - m0) <= 1e-12 * m0 + 1e-9


def test_part_error_reports_global_index():
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, 2)
    lm = dist.local_mesh(m, part, 1)
    p = dist.PartSolver(lm)
    st = sc.state.copy()
    bad = int(lm.cells[5])
    st.h[bad] = 1.0
    st.qx[bad] = np.nan
    p.set_state(st)
    with pytest.raises(api.NumericError, match=f"non-finite velocity in cell {bad}$"):
        p.local_cfl()


# ---- linked contexts: the device-resident multi-device step ---------------
def _scenario_parts(P, scale=0.03, name="sloping_wet_dry"):
    sc = api.make_scenario(name, scale=scale)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, P)
    return sc, m, [dist.local_mesh(m, part, p) for p in range(P)]


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("two_phase", [False, True], ids=["fused", "two_phase"])
def test_linked_parts_match_single_domain(P, two_phase):
    """P linked parts on one GPU stepped in lockstep: ghost states pushed by
    the step kernel, CFL bound / outcome through the device mailboxes."""
    sc, m, lms = _scenario_parts(P)
    parts = [dist.LinkedPart(lm, two_phase=two_phase) for lm in lms]
    dist.link_local(parts)
    for p in parts:
        p.set_state(sc.state)
    recs = dist.run_lockstep(parts, 150)
    got = api.FieldState.zeros(m.n_cells)
    for p in parts:
        t, step = p.gather_owned(got)
        assert step == 150
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=150)
    assert bit_equal(recs[:, 2], ref["dts"]) and bit_equal(recs[:, 3], ref["max_speeds"])
    for k, a in (("h", got.h), ("qx", got.qx), ("qy", got.qy)):
        assert bit_equal(a, ref[k]), k
    m0 = float(np.sum(sc.state.h * MeshArrays.from_mesh(m).area))
    assert abs(recs[-1, 4] - m0) <= 1e-12 * m0 + 1e-9
    ledgers = [p.ledger() for p in parts]  # the global ledger, on every rank
    assert all(lg == ledgers[0] for lg in ledgers)
    assert ledgers[0][1] == ref["clip_events"]
    assert abs(ledgers[0][0] - ref["clipped_volume"]) <= 1e-12 * max(1.0, ref["clipped_volume"])


def test_linked_single_rank_graph_matches_unlinked():
    """nranks = 1: the exchange (post + wait) runs inside the CUDA graph's
    WHILE body; results equal the unlinked context bit for bit."""
    sc, m, lms = _scenario_parts(1)
    p = dist.LinkedPart(lms[0])
    dist.link_local([p])
    p.set_state(sc.state)
    recs = p.advance(max_steps=200)
    assert len(recs) == 200
    solver = api.DeviceSolver(m)
    solver.set_state(sc.state)
    ref = solver.advance(1e30, max_steps=200)
    got = api.FieldState.zeros(m.n_cells)
    p.gather_owned(got)
    want, _, _ = solver.get_state()
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), getattr(want, k)), k
    assert bit_equal(recs[:, 2], ref[:, 2]) and bit_equal(recs[:, 3], ref[:, 3])


def test_link_normalises_buffer_parity_after_unlinked_steps():
    """A part stepped an odd number of times before linking (its state in
    buffer 1) still exchanges correctly: swe_dev_link moves every rank's
    current state to buffer 0 (pushes target the sender's cur^1)."""
    sc, m, lms = _scenario_parts(2)
    parts = [dist.LinkedPart(lm) for lm in lms]
    parts[0].set_state(sc.state)
    parts[0].advance(max_steps=1)  # unlinked warm-up: part 0 now holds cur = 1
    dist.link_local(parts)
    for p in parts:
        p.set_state(sc.state)
    recs = dist.run_lockstep(parts, 40)
    got = api.FieldState.zeros(m.n_cells)
    for p in parts:
        p.gather_owned(got)
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=40)
    assert bit_equal(recs[:, 2], ref["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), ref[k]), k


def test_linked_error_reports_global_index():
    sc, m, lms = _scenario_parts(2)
    parts = [dist.LinkedPart(lm) for lm in lms]
    dist.link_local(parts)
    st = sc.state.copy()
    bad = int(lms[1].cells[5])
    st.h[bad] = 1.0
    st.qx[bad] = np.nan
    for p in parts:
        p.set_state(st)
    with pytest.raises(api.NumericError, match=f"non-finite velocity in cell {bad}$"):
        dist.run_lockstep(parts, 1)


def test_linked_peer_timeout_is_an_error_not_a_hang():
    sc, m, lms = _scenario_parts(2)
    parts = [dist.LinkedPart(lm) for lm in lms]
    dist.link_local(parts, timeout_s=0.3)
    parts[0].set_state(sc.state)
    with pytest.raises(api.DeviceError):
        parts[0].advance(max_steps=5)  # rank 1 never posts


def _ipc_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, m, lms = _scenario_parts(world)
        lp = dist.LinkedPart(lms[rank])
        dist.link_torch(lp)  # peers' arenas through CUDA IPC handles
        lp.set_state(sc.state)
        recs = dist.run_lockstep_ranks(lp, 60)
        got = api.FieldState.zeros(m.n_cells)
        lp.gather_owned(got)
        own = lms[rank].cells[:lms[rank].n_owned]
        q.put((rank, own, got.h[own], got.qx[own], got.qy[own], recs, lp.ledger()))
        tdist.barrier()
        lp.close()
    finally:
        tdist.destroy_process_group()


def test_linked_ranks_over_cuda_ipc():
    """Two processes linked through CUDA IPC (the torchrun path of
    bench.py --gpus N), stepped in lockstep on one GPU."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sc, m, _ = _scenario_parts(1)
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=60)
    assert bit_equal(res[0][5], res[1][5])  # same records on both ranks
    assert res[0][6] == res[1][6]
    assert bit_equal(res[0][5][:, 2], ref["dts"])
    for rank, own, h, qx, qy, _, _ in res:
        assert bit_equal(h, ref["h"][own]) and bit_equal(qx, ref["qx"][own])
        assert bit_equal(qy, ref["qy"][own])


def test_linked_two_phase_single_rank_graph():
    """linked two-phase step (k_face_c, k_cell_c, k_push, k_exchange) in the graph"""
    sc, m, lms = _scenario_parts(1)
    p = dist.LinkedPart(lms[0], two_phase=True)
    dist.link_local([p])
    p.set_state(sc.state)
    recs = p.advance(max_steps=150)
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=150)
    got = api.FieldState.zeros(m.n_cells)
    p.gather_owned(got)
    assert bit_equal(recs[:, 2], ref["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(got, k), ref[k]), k


def _fail_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SWE_LINK_FAIL="2")
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, m, lms = _scenario_parts(world)
        lp = dist.LinkedPart(lms[rank])
        try:
            dist.link_torch(lp, timeout_s=5.0)
            q.put((rank, "linked"))
        except dist.LinkUnavailable as e:
            q.put((rank, "unavailable"))
        tdist.barrier()
        lp.close()
    finally:
        tdist.destroy_process_group()


def test_link_failure_on_one_rank_is_seen_by_all():
    """rank 1 cannot map peer memory: every rank raises LinkUnavailable
    (bench.py then takes the host-driven path) instead of hanging"""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == {0: "unavailable", 1: "unavailable"}

"""Domain decomposition on CPU: the partitioner and local
meshes of the product (include/swe/partition.hpp) driven by the C oracle as
per-part compute, in one process and across 2 gloo ranks.  A P-part run must
be bit-identical to the single-domain run."""
import os
import socket

import numpy as np
import pytest

from conftest import bit_equal
from oracle.pyoracle import COracle, MeshArrays, so_clock
from paper_1807_00672_b200 import api, dist


def scenario(name="sloping_wet_dry", scale=0.02):
    sc = api.make_scenario(name, scale=scale)
    return sc, api.build_mesh(sc.raw, sc.bed, sc.manning)


def local_arrays(lm):
    a = lm.arrays
    return MeshArrays(a["area"], a["inradius"], a["bed"], a["manning"], a["cell_edge"],
                      a["cell_sign"], a["edge_left"], a["edge_right"], a["nx"], a["ny"], a["len"])


@pytest.mark.parametrize("P", [2, 3, 4, 7, 8])
def test_partition_and_plans(P):
    sc, m = scenario()
    part = dist.partition(m, P)
    counts = np.bincount(part, minlength=P)
    assert counts.min() >= counts.max() - 1  # RCB splits by count
    lms = [dist.local_mesh(m, part, p) for p in range(P)]
    owned = np.concatenate([lm.cells[:lm.n_owned] for lm in lms])
    assert np.array_equal(np.sort(owned), np.arange(m.n_cells))
    edge_count = np.zeros(m.n_edges, int)
    for lm in lms:
        edge_count[lm.edges] += 1
        # owned cells keep their three incidences in reference order
        ce = lm.arrays["cell_edge"].reshape(-1, 3)[:lm.n_owned]
        cs = lm.arrays["cell_sign"].reshape(-1, 3)[:lm.n_owned]
        g = lm.cells[:lm.n_owned]
        assert np.array_equal(lm.edges[ce], m.cell_edge[g]) and np.array_equal(cs, m.cell_sign[g])
        for i, q in enumerate(lm.peers):
            other = lms[q]
            j = other.peers.index(lm.part)
            assert np.array_equal(lm.cells[lm.send[i]], other.cells[other.recv[j]])
    cut = (m.edge_right >= 0) & (part[m.edge_left] != part[np.maximum(m.edge_right, 0)])
    assert np.all(edge_count[cut] == 2) and np.all(edge_count[~cut] == 1)


def oracle_parts_run(m, st, lms, nsteps, exchange_fn, min_fn=lambda x: x, max_fn=lambda x: x):
    """Step the parts with the oracle; exchange_fn(states) refreshes ghosts;
    min_fn / max_fn reduce a local value across ranks (identity in-process)."""
    co = COracle()
    arrs = [local_arrays(lm) for lm in lms]
    states = [[np.ascontiguousarray(a[lm.cells]) for a in (st.h, st.qx, st.qy)] for lm in lms]
    clks = [so_clock(0.0, 0, 0.0, 0) for _ in lms]
    dts_seq = []
    for _ in range(nsteps):
        exchange_fn(states)
        loc = [co.local_cfl(a, lm.n_owned, *s) for a, lm, s in zip(arrs, lms, states)]
        assert all(x[2] == -1 for x in loc)
        dts = min_fn(min(x[0] for x in loc))
        ms = max_fn(max(x[1] for x in loc))
        for a, lm, s, clk in zip(arrs, lms, states, clks):
            rc, stt = co.step_owned(a, lm.n_owned, s, clk, 1e30, dts, ms)
            assert rc == 0
        dts_seq.append(stt.dt)
    return states, dts_seq


@pytest.mark.parametrize("P", [2, 3, 5])
def test_decomposed_oracle_matches_single_domain(P):
    sc, m = scenario()
    part = dist.partition(m, P)
    lms = [dist.local_mesh(m, part, p) for p in range(P)]
    by_part = {lm.part: lm for lm in lms}

    def exchange(states):
        for lm, s in zip(lms, states):
            for i, q in enumerate(lm.peers):
                other = by_part[q]
                j = other.peers.index(lm.part)
                src = states[q]
                for k in range(3):
                    s[k][lm.recv[i]] = src[k][other.send[j]]

    states, dts = oracle_parts_run(m, sc.state, lms, 60, exchange)
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=60)
    assert bit_equal(np.array(dts), ref["dts"])
    for lm, s in zip(lms, states):
        own = lm.cells[:lm.n_owned]
        for k, key in enumerate(("h", "qx", "qy")):
            assert bit_equal(s[k][:lm.n_owned], ref[key][own]), key


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OraclePart:
    """CPU stand-in for dist.PartSolver (same interface), stepping one part
    with the C oracle -- test infrastructure that lets the product's
    dist.run_parts / dist.TorchExchange run over gloo on CPU."""

    def __init__(self, lm, state):
        import torch
        self.lm, self.co, self.arr = lm, COracle(), local_arrays(lm)
        self.s = [np.ascontiguousarray(a[lm.cells]) for a in (state.h, state.qx, state.qy)]
        self.clk = so_clock(0.0, 0, 0.0, 0)
        ns, nr = sum(map(len, lm.send)), sum(map(len, lm.recv))
        self.send_buf = torch.zeros(3 * max(1, ns), dtype=torch.float64)
        self.recv_buf = torch.zeros(3 * max(1, nr), dtype=torch.float64)
        self.send_off = np.concatenate([[0], np.cumsum([len(x) for x in lm.send])]).astype(int)
        self.recv_off = np.concatenate([[0], np.cumsum([len(x) for x in lm.recv])]).astype(int)

    def send_block(self, i):
        return self.send_buf[3 * self.send_off[i]:3 * self.send_off[i + 1]]

    def recv_block(self, i):
        return self.recv_buf[3 * self.recv_off[i]:3 * self.recv_off[i + 1]]

    def pack(self):
        cells = np.concatenate(self.lm.send) if self.lm.send else np.zeros(0, int)
        v = self.send_buf.numpy()[:3 * len(cells)].reshape(-1, 3)
        for k in range(3):
            v[:, k] = self.s[k][cells]

    def unpack(self):
        cells = np.concatenate(self.lm.recv) if self.lm.recv else np.zeros(0, int)
        v = self.recv_buf.numpy()[:3 * len(cells)].reshape(-1, 3)
        for k in range(3):
            self.s[k][cells] = v[:, k]

    def local_cfl(self):
        dts, ms, bad = self.co.local_cfl(self.arr, self.lm.n_owned, *self.s)
        assert bad == -1
        return dts, ms, float(np.sum(self.s[0][:self.lm.n_owned] * self.arr.area[:self.lm.n_owned]))

    def step_global(self, t_end, dts, ms):
        rc, st = self.co.step_owned(self.arr, self.lm.n_owned, self.s, self.clk, t_end, dts, ms)
        assert rc == 0
        n = self.lm.n_owned
        st.mass = float(np.sum(self.s[0][:n] * self.arr.area[:n]))
        return st


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, m = scenario()
        part = dist.partition(m, world)
        lm = dist.local_mesh(m, part, rank)
        op = OraclePart(lm, sc.state)
        recs = dist.run_parts([op], dist.TorchExchange(op), 40)  # the product driver
        dts = recs[:, 1]
        owned = np.zeros((3, m.n_cells))
        mask = np.zeros(m.n_cells)
        for k in range(3):
            owned[k][lm.cells[:lm.n_owned]] = op.s[k][:lm.n_owned]
        mask[lm.cells[:lm.n_owned]] = 1
        t_owned, t_mask = torch.from_numpy(owned), torch.from_numpy(mask)
        tdist.all_reduce(t_owned)  # disjoint ownership: the sum assembles the field
        tdist.all_reduce(t_mask)
        if rank == 0:
            q.put((t_owned.numpy().copy(), t_mask.numpy().copy(), np.array(dts)))
    finally:
        tdist.destroy_process_group()


def test_gloo_two_ranks_match_single_domain():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    field, mask, dts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc, m = scenario()
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=40)
    assert np.all(mask == 1)
    assert bit_equal(dts, ref["dts"])
    for k, key in enumerate(("h", "qx", "qy")):
        assert bit_equal(field[k], ref[key]), key


def test_push_plan_pairs_send_and_recv_lists():
    """Linked contexts: each push entry carries an owned cell to the ghost
    slot holding the same global cell on the destination rank."""
    sc, m = scenario()
    P = 4
    part = dist.partition(m, P)
    lms = [dist.local_mesh(m, part, p) for p in range(P)]
    recv = {lm.part: (lm.peers, lm.recv) for lm in lms}
    for lm in lms:
        cells, ranks, ghosts = dist.push_plan(lm, recv)
        assert len(cells) == sum(len(s) for s in lm.send)
        assert np.all(cells < lm.n_owned)
        for c, q, g in zip(cells, ranks, ghosts):
            other = lms[q]
            assert g >= other.n_owned and other.cells[g] == lm.cells[c]


def _gloo_link_worker(rank, world, port, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, m = scenario()
        part = dist.partition(m, world)
        lm = dist.local_mesh(m, part, rank)
        handle = bytes([rank]) * 64  # stand-in for the CUDA IPC handle
        handles, cells, recv = dist.exchange_link_info(rank, lm, handle)
        plan = dist.push_plan(lm, recv)
        q.put((rank, handles, cells, [a.tolist() for a in plan]))
    finally:
        tdist.destroy_process_group()


def test_gloo_link_info_exchange():
    """The host half of link_torch over 2 gloo ranks: every rank sees all
    handles / sizes in rank order and builds the same plan as in-process."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_link_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (h, c, pl)) for r, h, c, pl in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc, m = scenario()
    part = dist.partition(m, 2)
    lms = [dist.local_mesh(m, part, p) for p in range(2)]
    recv = {lm.part: (lm.peers, lm.recv) for lm in lms}
    for r in range(2):
        handles, cells, plan = got[r]
        assert handles == [bytes([0]) * 64, bytes([1]) * 64]
        assert cells == [lms[0].n_cells, lms[1].n_cells]
        want = dist.push_plan(lms[r], recv)
        assert all(list(a) == b for a, b in zip(want, plan))


@pytest.mark.parametrize("P", [2, 3, 8])
def test_weighted_partition_balances_work(P):
    """cost-weighted RCB: every part's weight within one heaviest cell of the
    target, and a weighted partition is still a valid decomposition"""
    sc, m = scenario()
    w = dist.cost_weights(sc.state)
    part = dist.partition(m, P, w)
    loads = np.bincount(part, weights=w, minlength=P)
    assert loads.max() - loads.min() <= 2 * w.max() * np.log2(2 * P)
    eq = np.bincount(dist.partition(m, P), weights=w, minlength=P)
    assert loads.max() - loads.min() <= eq.max() - eq.min()
    lms = [dist.local_mesh(m, part, p) for p in range(P)]
    owned = np.concatenate([lm.cells[:lm.n_owned] for lm in lms])
    assert np.array_equal(np.sort(owned), np.arange(m.n_cells))

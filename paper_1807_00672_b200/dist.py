"""Multi-device runs: domain decomposition + halo exchange.

A mesh is split by recursive coordinate bisection (include/swe/partition.hpp)
into P parts.  Each part is one device context over its local mesh: owned
cells (updated) + a one-cell ghost layer (read-only copies refreshed every
step) + every edge touching an owned cell, so cut edges are evaluated by both
sides from identical inputs and a P-part run is bit-identical to the
single-domain run (only the per-step mass is summed in a different order).

Production path -- LINKED contexts (``LinkedPart``, ``link_torch`` /
``link_local``): the step kernel pushes the new state of the cells a peer
holds as ghosts straight into that peer's buffers (CUDA IPC peer memory over
NVLink) and the CFL bound / step outcome is exchanged through device
mailboxes, all inside each rank's CUDA graph: no host round trip per step.
``run_lockstep`` / ``run_lockstep_ranks`` step linked parts phase by phase
(several parts sharing one device; tests).

Host-driven building blocks (``PartSolver`` + ``run_parts``), kept for the
CPU protocol tests (gloo): per step
  1. halo exchange: each part packs the owned cells its peers need (3 doubles
     per cell), the buffers move peer-to-peer, each part unpacks into its ghosts;
  2. global CFL bound: min over parts of the local bound, max of max_speed;
  3. every part takes the step with the global bound.
  ``LocalExchange``  all parts in this process: device-to-device copies.
  ``TorchExchange``  one part per rank: torch.distributed batch_isend_irecv
                     + all_reduce(MIN/MAX).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .api import DeviceError, FieldState, Mesh, NumericError, PhysParams, _check, _errbuf, _raise


def partition(mesh: Mesh, nparts: int, weights=None) -> np.ndarray:
    """part id per cell (recursive coordinate bisection of centroids); with
    per-cell weights (cost_weights) the parts get equal work instead of equal
    cell counts."""
    out = np.empty(mesh.n_cells, dtype=np.int32)
    lib = L.load()
    if weights is None:
        rc = lib.swe_host_partition(mesh.handle, nparts, L.ptr(out))
    else:
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if len(w) != mesh.n_cells:
            raise ValueError("partition: one weight per cell required")
        rc = lib.swe_host_partition_weighted(mesh.handle, nparts, L.ptr(w), L.ptr(out))
    if rc:
        _raise(rc, "rcb_partition failed")
    return out


WET_COST = 5.0    # wet / skipped-dry cell step cost on B200 (tools/scaling_proxy.py fit)
FRONT_COST = 3.0  # dry cells near water: their tiles are computed, not skipped
FRONT_WIDTH = 8   # cells: about half a tile's extent


def cost_weights(state: FieldState, h_dry: float = 1e-6, wet_cost: float = WET_COST,
                 mesh: Mesh | None = None, front_cost: float = FRONT_COST,
                 front_width: int = FRONT_WIDTH) -> np.ndarray:
    """per-cell step cost (include/swe/partition.hpp cost_weights): 1 for a
    dry cell in a skippable dry region, wet_cost for a wet one; with `mesh`,
    dry cells within front_width cells of water cost front_cost (dry-tile
    skipping needs the tile AND its ring dry)."""
    wet = np.asarray(state.h) >= h_dry
    w = np.where(wet, wet_cost, 1.0)
    if mesh is not None and front_width > 0:
        el, er = np.asarray(mesh.edge_left), np.asarray(mesh.edge_right)
        inner = er >= 0
        a, b = el[inner], er[inner]
        near = wet.copy()
        for _ in range(front_width):  # dilate the wet set across edges
            grow = near.copy()
            grow[a] |= near[b]
            grow[b] |= near[a]
            near = grow
        w = np.where(~wet & near, front_cost, w)
    return w


# computed / skipped tile cost per cell, calibrated on B200 splits of the 10M
# channel (tools/scaling_proxy.py): small parts (strong scaling, ~1-5M cells
# per GPU) 3.8; large parts (weak scaling, ~10M per GPU) 7.5 -- a skipped run
# of tiles amortises its per-tile latency better in a long kernel
COMPUTED_COST = 3.8
COMPUTED_COST_LARGE = 7.5
LARGE_PART_CELLS = 8_000_000


def measured_cost_weights(mesh: Mesh, state: FieldState, device: int = 0, steps: int = 2,
                          computed_cost: float | None = None, parts: int = 0) -> np.ndarray:
    """per-cell cost from the device's own skip pattern: run the whole mesh
    `steps` steps and weight cells in skipped dry tiles 1, all others
    computed_cost (captures the wet front at tile granularity); by default
    computed_cost follows the part size (mesh cells / parts)"""
    if computed_cost is None:
        large = parts > 0 and mesh.n_cells / parts >= LARGE_PART_CELLS
        computed_cost = COMPUTED_COST_LARGE if large else COMPUTED_COST
    from .api import DeviceSolver
    s = DeviceSolver(mesh, device=device)
    try:
        s.set_state(state)
        s.advance(1.7976931348623157e308, max_steps=steps)
        return np.where(s.cell_skip() != 0, 1.0, computed_cost)
    finally:
        s.close()


def refine_weights(weights, part, part_ms, damping: float = 0.8) -> np.ndarray:
    """One rebalancing step from measured part step times: every cell of part
    p is scaled by (t_p / mean t)^damping, so the next weighted RCB moves work
    from slow parts to fast ones.  A few rounds equalise parts whose costs the
    model misses (front tiles, halo edges, ramp / tail of short kernels)."""
    t = np.asarray(part_ms, dtype=np.float64)
    f = (t / t.mean()) ** damping
    return np.asarray(weights, dtype=np.float64) * f[np.asarray(part)]


def part_step_ms(mesh: Mesh, state: FieldState, part: np.ndarray, p: int, device: int = 0,
                 steps: int = 40) -> float:
    """Step time of part p alone (unlinked: its own dt), CUDA events on its
    stream after a warm-up; the measurement behind refine_weights."""
    import torch
    lm = local_mesh(mesh, part, p)
    lp = LinkedPart(lm, device=device)
    try:
        lp.set_state(state)
        H = 1.7976931348623157e308
        lp.advance(t_end=H, max_steps=5)
        st = torch.cuda.ExternalStream(lp.lib.swe_dev_stream(lp.ctx), device=device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(device)
        e0.record(st)
        lp.launch(t_end=H, max_steps=5 + steps)
        e1.record(st)
        torch.cuda.synchronize(device)
        lp.records()
        return e0.elapsed_time(e1) / steps
    finally:
        lp.close()


@dataclass
class LocalMesh:
    """One part's mesh in local numbering (owned first) + exchange plan."""
    part: int
    n_owned: int
    cells: np.ndarray  # local -> global cell
    edges: np.ndarray  # local -> global edge
    arrays: dict
    peers: list = field(default_factory=list)
    send: list = field(default_factory=list)  # per peer: local owned ids
    recv: list = field(default_factory=list)  # per peer: local ghost ids

    @property
    def n_cells(self):
        return len(self.cells)

    @property
    def n_edges(self):
        return len(self.edges)

    def view(self) -> L.swe_mesh_view:
        a = self.arrays
        v = L.swe_mesh_view()
        v.n_cells, v.n_edges, v.n_owned = self.n_cells, self.n_edges, self.n_owned
        v.area, v.inradius, v.bed, v.manning = (L.dptr(a[k]) for k in ("area", "inradius", "bed",
                                                                        "manning"))
        v.cx, v.cy = L.dptr(a["cx"]), L.dptr(a["cy"])
        v.cell_edge, v.cell_sign = L.iptr(a["cell_edge"]), L.iptr(a["cell_sign"])
        v.edge_left, v.edge_right = L.iptr(a["edge_left"]), L.iptr(a["edge_right"])
        v.nx, v.ny, v.len = L.dptr(a["nx"]), L.dptr(a["ny"]), L.dptr(a["len"])
        return v


def local_mesh(mesh: Mesh, part: np.ndarray, p: int) -> LocalMesh:
    lib = L.load()
    part = np.ascontiguousarray(part, dtype=np.int32)
    err = _errbuf()
    h = lib.swe_host_local_mesh(mesh.handle, L.ptr(part), p, err, len(err))
    if not h:
        _raise(3, err.value)
    return _local_from_handle(lib, h, p)


def partition_raw(raw, nparts: int, weights=None) -> np.ndarray:
    """RCB over a RAW mesh's triangle centroids (no global Mesh needed)."""
    out = np.empty(raw.n_cells, dtype=np.int32)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    rc = L.load().swe_host_partition_raw(raw.handle, nparts, L.ptr(w), L.ptr(out))
    if rc:
        _raise(rc, "rcb_partition (raw) failed")
    return out


def rank_mesh(raw, bed, manning, part: np.ndarray, p: int) -> LocalMesh:
    """Part p's LocalMesh built from the raw mesh alone (owned triangles +
    ghost layer; include/swe/multigpu.hpp build_rank_mesh): a rank of a large
    run never materialises the global Mesh.  Edge ids are part-local."""
    lib = L.load()
    part = np.ascontiguousarray(part, dtype=np.int32)
    b = np.ascontiguousarray(bed, dtype=np.float64)
    m = np.ascontiguousarray(manning, dtype=np.float64)
    err = _errbuf()
    h = lib.swe_host_rank_mesh(raw.handle, L.ptr(b), L.ptr(m), L.ptr(part), p, err, len(err))
    if not h:
        _raise(3, err.value)
    return _local_from_handle(lib, h, p)


def _local_from_handle(lib, h, p: int) -> LocalMesh:
    try:
        s = [C.c_int() for _ in range(6)]
        lib.swe_host_local_sizes(h, *[C.byref(x) for x in s])
        nc, no, ne, npeer, nsend, nrecv = (x.value for x in s)
        a = {k: np.empty(nc) for k in ("area", "inradius", "bed", "manning", "cx", "cy")}
        a["cell_edge"] = np.empty(3 * nc, np.int32)
        a["cell_sign"] = np.empty(3 * nc, np.int32)
        a["edge_left"] = np.empty(ne, np.int32)
        a["edge_right"] = np.empty(ne, np.int32)
        for k in ("nx", "ny", "len"):
            a[k] = np.empty(ne)
        cells, edges = np.empty(nc, np.int32), np.empty(ne, np.int32)
        lib.swe_host_local_export(h, L.ptr(cells), L.ptr(edges), *[L.ptr(a[k]) for k in (
            "area", "inradius", "bed", "manning", "cx", "cy", "cell_edge", "cell_sign",
            "edge_left", "edge_right", "nx", "ny", "len")])
        peers = np.empty(max(npeer, 1), np.int32)
        sc, rcnt = np.empty(max(npeer, 1), np.int32), np.empty(max(npeer, 1), np.int32)
        sf, rf = np.empty(max(nsend, 1), np.int32), np.empty(max(nrecv, 1), np.int32)
        lib.swe_host_local_plan(h, L.ptr(peers), L.ptr(sc), L.ptr(rcnt), L.ptr(sf), L.ptr(rf))
    finally:
        lib.swe_host_local_free(h)
    lm = LocalMesh(p, no, cells, edges, a)
    so = ro = 0
    for i in range(npeer):
        lm.peers.append(int(peers[i]))
        lm.send.append(sf[so:so + sc[i]].copy())
        lm.recv.append(rf[ro:ro + rcnt[i]].copy())
        so += sc[i]
        ro += rcnt[i]
    return lm


class PartSolver:
    """Device context of one part (include/swe_dev.h multi-device entries)."""

    def __init__(self, lm: LocalMesh, params: PhysParams = PhysParams(), device: int = 0,
                 two_phase: bool = False):
        import torch
        self.lib = L.load()
        self.lm, self.params, self.device = lm, params, device
        v = lm.view()
        p = params.c()
        ctx = C.c_void_p()
        flags = L.SWE_FLAG_TWO_PHASE if two_phase else 0
        _check(self.lib.swe_dev_create(C.byref(v), C.byref(p), device, flags, C.byref(ctx)),
               "swe_dev_create(part)")
        self.ctx = ctx
        send = np.concatenate(lm.send).astype(np.int32) if lm.send else np.zeros(0, np.int32)
        recv = np.concatenate(lm.recv).astype(np.int32) if lm.recv else np.zeros(0, np.int32)
        _check(self.lib.swe_dev_set_halo_plan(ctx, len(send), L.ptr(send), len(recv), L.ptr(recv)),
               "swe_dev_set_halo_plan")
        dev = torch.device("cuda", device)
        self.send_buf = torch.empty(3 * max(1, len(send)), dtype=torch.float64, device=dev)
        self.recv_buf = torch.empty(3 * max(1, len(recv)), dtype=torch.float64, device=dev)
        self.send_off = np.concatenate([[0], np.cumsum([len(s) for s in lm.send])]).astype(int)
        self.recv_off = np.concatenate([[0], np.cumsum([len(r) for r in lm.recv])]).astype(int)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.swe_dev_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    # blocks of the packed buffers, per peer index
    def send_block(self, i):
        return self.send_buf[3 * self.send_off[i]:3 * self.send_off[i + 1]]

    def recv_block(self, i):
        return self.recv_buf[3 * self.recv_off[i]:3 * self.recv_off[i + 1]]

    def set_state(self, s: FieldState, t=0.0, step=0):
        """s: GLOBAL state; the part takes its owned + ghost cells."""
        c = self.lm.cells
        h, qx, qy = (np.ascontiguousarray(a[c]) for a in (s.h, s.qx, s.qy))
        _check(self.lib.swe_dev_set_state(self.ctx, L.ptr(h), L.ptr(qx), L.ptr(qy), t, step),
               "swe_dev_set_state")

    def gather_owned(self, out: FieldState):
        n = self.lm.n_cells
        h, qx, qy = np.empty(n), np.empty(n), np.empty(n)
        t, step = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_state(self.ctx, L.ptr(h), L.ptr(qx), L.ptr(qy), C.byref(t),
                                          C.byref(step)), "swe_dev_get_state")
        own = self.lm.cells[:self.lm.n_owned]
        out.h[own], out.qx[own], out.qy[own] = h[:self.lm.n_owned], qx[:self.lm.n_owned], \
            qy[:self.lm.n_owned]
        return t.value, step.value

    def pack(self):
        _check(self.lib.swe_dev_pack_halo(self.ctx, C.c_void_p(self.send_buf.data_ptr())), "pack")

    def unpack(self):
        _check(self.lib.swe_dev_unpack_halo(self.ctx, C.c_void_p(self.recv_buf.data_ptr())), "unpack")

    def local_cfl(self):
        d, m, ms = C.c_double(), C.c_double(), C.c_double()
        st = L.swe_status()
        rc = self.lib.swe_dev_local_cfl(self.ctx, C.byref(d), C.byref(m), C.byref(ms), C.byref(st))
        if rc == L.SWE_NONFINITE_SPEED:
            gid = int(self.lm.cells[st.index])
            raise NumericError(f"stable_dt: non-finite velocity in cell {gid}")
        _check(rc, "swe_dev_local_cfl")
        return d.value, m.value, ms.value

    def step_global(self, t_end, dts, max_speed):
        rec, st = L.swe_step_record(), L.swe_status()
        rc = self.lib.swe_dev_step_global(self.ctx, t_end, dts, max_speed, C.byref(rec),
                                          C.byref(st))
        if rc in (L.SWE_NEGATIVE_DEPTH,):
            gid = int(self.lm.edges[st.index])
            raise NumericError(f"compute_fluxes: negative depth at edge {gid}")
        if rc == L.SWE_BLOWUP:
            gid = int(self.lm.cells[st.index])
            raise NumericError(f"advance_step: numeric blowup at step {st.step}, cell {gid}, "
                               f"dt {st.dt:f} (h={st.h:f})")
        _check(rc, "swe_dev_step_global")
        return rec


class LocalExchange:
    """All parts in this process: peer blocks moved by device copies."""

    def __init__(self, parts):
        self.parts = {p.lm.part: p for p in parts}

    def halo(self):
        for p in self.parts.values():
            p.pack()
        for p in self.parts.values():
            for i, q in enumerate(p.lm.peers):
                peer = self.parts[q]
                j = peer.lm.peers.index(p.lm.part)
                p.recv_block(i).copy_(peer.send_block(j))
        for p in self.parts.values():
            p.unpack()

    @staticmethod
    def allreduce_min(x):
        return x

    @staticmethod
    def allreduce_max(x):
        return x

    @staticmethod
    def allreduce_sum(x):
        return x


class TorchExchange:
    """One part per rank over torch.distributed: NCCL on GPUs (the part's
    buffers are device tensors), gloo on CPU.  The part provides pack(),
    unpack(), send_block(i), recv_block(i) and lm (LocalMesh)."""

    def __init__(self, part, group=None):
        import torch.distributed as dist
        self.dist, self.part, self.group = dist, part, group
        # gloo moves host memory only: device buffers are staged through the host
        self.host_staged = dist.get_backend(group) == "gloo" and part.send_buf.is_cuda

    def halo(self):
        import torch
        p, dist = self.part, self.dist
        p.pack()
        ops, back = [], []
        for i, q in enumerate(p.lm.peers):  # plans are symmetric: both directions per peer
            sb, rb = p.send_block(i), p.recv_block(i)
            if self.host_staged:
                sb, dev_rb = sb.cpu(), rb
                rb = torch.empty(rb.shape, dtype=rb.dtype)
                back.append((dev_rb, rb))
            if sb.numel():
                ops.append(dist.P2POp(dist.isend, sb, q, self.group))
            if rb.numel():
                ops.append(dist.P2POp(dist.irecv, rb, q, self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for dev_rb, host_rb in back:
            dev_rb.copy_(host_rb)
        if p.send_buf.is_cuda:
            torch.cuda.synchronize(p.send_buf.device)
        p.unpack()

    def _reduce(self, x, op):
        import torch
        t = torch.tensor([x], dtype=torch.float64,
                         device="cpu" if self.host_staged else self.part.send_buf.device)
        self.dist.all_reduce(t, op=op, group=self.group)
        return float(t.item())

    def allreduce_min(self, x):
        return self._reduce(x, self.dist.ReduceOp.MIN)

    def allreduce_max(self, x):
        return self._reduce(x, self.dist.ReduceOp.MAX)

    def allreduce_sum(self, x):
        return self._reduce(x, self.dist.ReduceOp.SUM)


# ---------------------------------------------------------------------------
# Linked contexts: the device-resident multi-device step (include/swe_dev.h
# "linked contexts").  Ghost states are pushed peer-to-peer by the step
# kernel and the CFL bound / step outcome is exchanged through device
# mailboxes, so a run is one CUDA graph launch per rank with no host round
# trip per step.
# ---------------------------------------------------------------------------
def push_plan(lm: LocalMesh, peer_recv: dict):
    """Push entries of part lm.part: (owned local cell, destination rank,
    ghost local id on that rank).  peer_recv[q] = (q's peers, q's recv lists);
    plans are symmetric -- lm.send[i] and q's recv list for lm.part hold the
    same global cells in the same order."""
    cells, ranks, ghosts = [], [], []
    for i, q in enumerate(lm.peers):
        qpeers, qrecv = peer_recv[q]
        j = list(qpeers).index(lm.part)
        s, r = np.asarray(lm.send[i]), np.asarray(qrecv[j])
        if len(s) != len(r):
            raise ValueError(f"halo plans of parts {lm.part} and {q} disagree")
        cells.append(s)
        ranks.append(np.full(len(s), q))
        ghosts.append(r)
    cat = (lambda xs: np.ascontiguousarray(np.concatenate(xs), dtype=np.int32) if xs
           else np.zeros(0, np.int32))
    return cat(cells), cat(ranks), cat(ghosts)


class LinkedPart:
    """One part (rank) of a linked multi-device run."""

    def __init__(self, lm: LocalMesh, params: PhysParams = PhysParams(), device: int = 0,
                 two_phase: bool = False):
        self.lib = L.load()
        self.lm, self.params, self.device = lm, params, device
        v = lm.view()
        p = params.c()
        ctx = C.c_void_p()
        flags = L.SWE_FLAG_TWO_PHASE if two_phase else 0
        _check(self.lib.swe_dev_create(C.byref(v), C.byref(p), device, flags, C.byref(ctx)),
               "swe_dev_create(part)")
        self.ctx = ctx
        self.linked = False

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.swe_dev_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def export(self):
        """(arena device pointer, 64-byte CUDA IPC handle)."""
        arena = C.c_void_p()
        h = (C.c_ubyte * 64)()
        _check(self.lib.swe_dev_link_export(self.ctx, C.byref(arena), h), "swe_dev_link_export")
        return arena.value, bytes(h)

    def link(self, rank: int, nranks: int, peer_cells, plan, arenas=None, handles=None,
             timeout_s: float = 60.0):
        cells, ranks, ghosts = plan
        pc = np.ascontiguousarray(peer_cells, dtype=np.int64)
        gc = np.ascontiguousarray(self.lm.cells, dtype=np.int32)
        ge = np.ascontiguousarray(self.lm.edges, dtype=np.int32)
        arr = (C.c_void_p * nranks)(*arenas) if arenas is not None else None
        hnd = (C.c_ubyte * (64 * nranks)).from_buffer_copy(b"".join(handles)) \
            if handles is not None else None
        _check(self.lib.swe_dev_link(self.ctx, rank, nranks, arr, hnd, L.ptr(pc), len(cells),
                                     L.ptr(cells), L.ptr(ranks), L.ptr(ghosts), L.ptr(gc),
                                     L.ptr(ge), float(timeout_s)), "swe_dev_link")
        self.linked = True

    def set_state(self, s: FieldState, t=0.0, step=0):
        """s: GLOBAL state; the part takes its owned + ghost cells."""
        c = self.lm.cells
        h, qx, qy = (np.ascontiguousarray(a[c]) for a in (s.h, s.qx, s.qy))
        _check(self.lib.swe_dev_set_state(self.ctx, L.ptr(h), L.ptr(qx), L.ptr(qy), t, step),
               "swe_dev_set_state")

    def gather_owned(self, out: FieldState):
        n = self.lm.n_cells
        h, qx, qy = np.empty(n), np.empty(n), np.empty(n)
        t, step = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_state(self.ctx, L.ptr(h), L.ptr(qx), L.ptr(qy), C.byref(t),
                                          C.byref(step)), "swe_dev_get_state")
        own = self.lm.cells[:self.lm.n_owned]
        no = self.lm.n_owned
        out.h[own], out.qx[own], out.qy[own] = h[:no], qx[:no], qy[:no]
        return t.value, step.value

    def clock(self):
        t, step = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_state(self.ctx, None, None, None, C.byref(t), C.byref(step)),
               "swe_dev_get_state")
        return t.value, step.value

    def ledger(self):
        v, n = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_ledger(self.ctx, C.byref(v), C.byref(n)), "ledger")
        return v.value, n.value

    @staticmethod
    def raise_status(rc, st):
        """Map a linked status to the reference's exceptions (indices are global)."""
        if rc == L.SWE_NONFINITE_SPEED:
            raise NumericError(f"stable_dt: non-finite velocity in cell {st.index}")
        if rc == L.SWE_NEGATIVE_DEPTH:
            raise NumericError(f"compute_fluxes: negative depth at edge {st.index}")
        if rc == L.SWE_BLOWUP:
            raise NumericError(f"advance_step: numeric blowup at step {st.step}, cell {st.index}, "
                               f"dt {st.dt:f} (h={st.h:f})")
        _check(rc, "linked step")

    def advance(self, t_end=1e30, max_steps=1 << 62, next_snapshot=float("inf"),
                max_records=1 << 16):
        """run() segment on the device (collective: every rank calls it);
        returns records (step, t, dt, max_speed, global mass)."""
        recs = (L.swe_step_record * max_records)()
        n, st = C.c_longlong(), L.swe_status()
        rc = self.lib.swe_dev_advance(self.ctx, t_end, max_steps, next_snapshot, recs, max_records,
                                      C.byref(n), C.byref(st))
        out = np.array([(r.step, r.t, r.dt, r.max_speed, r.mass) for r in recs[:n.value]],
                       dtype=np.float64).reshape(-1, 5)
        if rc:
            self.raise_status(rc, st)
        return out

    def advance_async(self, n: int, t_end=float("inf")):
        _check(self.lib.swe_dev_advance_n_async(self.ctx, n, t_end), "advance_n_async")

    def launch(self, t_end=1e30, max_steps=1 << 62, next_snapshot=float("inf"),
               max_records=1 << 16):
        """advance() split: enqueue the graph launch only (collective)."""
        _check(self.lib.swe_dev_advance_async(self.ctx, t_end, max_steps, next_snapshot,
                                              max_records), "swe_dev_advance_async")

    def records(self, max_records=1 << 16):
        recs = (L.swe_step_record * max_records)()
        n, st = C.c_longlong(), L.swe_status()
        rc = self.lib.swe_dev_records(self.ctx, recs, max_records, C.byref(n), C.byref(st))
        out = np.array([(r.step, r.t, r.dt, r.max_speed, r.mass)
                        for r in recs[:min(n.value, max_records)]],
                       dtype=np.float64).reshape(-1, 5)
        if rc:
            self.raise_status(rc, st)
        return out

    def synchronize(self):
        st = L.swe_status()
        rc = self.lib.swe_dev_synchronize(self.ctx, C.byref(st))
        if rc:
            self.raise_status(rc, st)


def link_local(parts, timeout_s: float = 60.0):
    """Link the parts of this process (one or several devices)."""
    nr = len(parts)
    by_part = {p.lm.part: p for p in parts}
    if sorted(by_part) != list(range(nr)):
        raise ValueError("parts must be numbered 0..P-1")
    arenas = [by_part[q].export()[0] for q in range(nr)]
    cells = [by_part[q].lm.n_cells for q in range(nr)]
    recv = {q: (by_part[q].lm.peers, by_part[q].lm.recv) for q in range(nr)}
    for p in parts:
        p.link(p.lm.part, nr, cells, push_plan(p.lm, recv), arenas=arenas, timeout_s=timeout_s)


def exchange_link_info(part_id: int, lm: LocalMesh, handle: bytes, group=None):
    """all_gather of every rank's (IPC handle, n_cells, peers, recv lists)."""
    import torch.distributed as tdist
    mine = (part_id, handle, lm.n_cells, list(lm.peers), [np.asarray(r).tolist() for r in lm.recv])
    allv = [None] * tdist.get_world_size(group)
    tdist.all_gather_object(allv, mine, group=group)
    allv.sort(key=lambda v: v[0])
    handles = [v[1] for v in allv]
    cells = [v[2] for v in allv]
    recv = {v[0]: (v[3], v[4]) for v in allv}
    return handles, cells, recv


class LinkUnavailable(DeviceError):
    """some rank could not map its peers' memory (CUDA IPC / peer access)"""


def link_torch(part: LinkedPart, group=None, timeout_s: float = 60.0):
    """Link one part per rank (torchrun): part id == rank; peers' arenas are
    mapped through CUDA IPC (NVLink peer memory on one node).  Collective and
    fail-safe: if any rank cannot link, every rank raises LinkUnavailable
    (instead of some ranks waiting forever at a barrier)."""
    import torch
    import torch.distributed as tdist
    rank, nr = tdist.get_rank(group), tdist.get_world_size(group)
    if part.lm.part != rank:
        raise ValueError("link_torch: the part id must equal the rank")
    _, handle = part.export()
    handles, cells, recv = exchange_link_info(rank, part.lm, handle, group)
    err = ""
    try:
        part.link(rank, nr, cells, push_plan(part.lm, recv), handles=handles, timeout_s=timeout_s)
    except DeviceError as e:
        err = str(e)
    backend = tdist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    ok = torch.tensor([0.0 if err else 1.0], device=dev)
    tdist.all_reduce(ok, op=tdist.ReduceOp.MIN, group=group)
    if ok.item() < 1.0:
        raise LinkUnavailable(err or "a peer rank could not link (CUDA IPC / peer access)")


def run_lockstep(parts, nsteps: int, t_end: float = 1e30):
    """Step linked parts of ONE process in lockstep (phase k of every part
    before phase k+1 of any), e.g. several parts sharing one device.
    Returns per-step (step, t, dt, max_speed, global mass)."""
    import torch
    out = []
    for _ in range(nsteps):
        for phase in range(5):
            for p in parts:
                _check(p.lib.swe_dev_link_phase(p.ctx, phase, t_end), "swe_dev_link_phase")
            torch.cuda.synchronize()
        recs = []
        for p in parts:
            rec, st = L.swe_step_record(), L.swe_status()
            rc = p.lib.swe_dev_last_record(p.ctx, C.byref(rec), C.byref(st))
            if rc:
                p.raise_status(rc, st)
            recs.append((rec.step, rec.t, rec.dt, rec.max_speed, rec.mass))
        if any(r != recs[0] for r in recs):
            raise RuntimeError(f"linked parts disagree on the step record: {recs}")
        out.append(recs[0])
        if not recs[0][1] < t_end:
            break
    return np.array(out, dtype=np.float64).reshape(-1, 5)


def run_ranks(parts, nsteps: int, t_end: float = 1e30, grid: int = 0):
    """Step linked parts of ONE process on ONE device concurrently: one
    cooperative launch of the persistent step kernel over all ranks
    (swe_dev_run_ranks), so the ranks' exchange runs as it does on P GPUs
    (no lockstep phases).  Returns the records of the last nsteps steps."""
    nr = len(parts)
    by_rank = sorted(parts, key=lambda p: p.lm.part)
    arr = (C.c_void_p * nr)(*[p.ctx.value for p in by_rank])
    rc = by_rank[0].lib.swe_dev_run_ranks(arr, nr, nsteps, t_end, grid)
    recs = [p.records() for p in by_rank]  # raises the rank's error, if any
    if rc:
        _check(rc, "swe_dev_run_ranks")
    for r in recs[1:]:
        if not np.array_equal(r, recs[0]):
            raise RuntimeError("linked ranks disagree on the step records")
    return recs[0][-nsteps:]


def run_lockstep_ranks(part: LinkedPart, nsteps: int, t_end: float = 1e30, group=None):
    """run_lockstep across processes: a torch.distributed barrier between
    phases, so every rank's post precedes every rank's wait (debug driver
    for ranks that share a device)."""
    import torch
    import torch.distributed as tdist
    out = []
    for _ in range(nsteps):
        for phase in range(5):
            _check(part.lib.swe_dev_link_phase(part.ctx, phase, t_end), "swe_dev_link_phase")
            torch.cuda.synchronize()
            tdist.barrier(group)
        rec, st = L.swe_step_record(), L.swe_status()
        rc = part.lib.swe_dev_last_record(part.ctx, C.byref(rec), C.byref(st))
        if rc:
            part.raise_status(rc, st)
        out.append((rec.step, rec.t, rec.dt, rec.max_speed, rec.mass))
        if not rec.t < t_end:
            break
    return np.array(out, dtype=np.float64).reshape(-1, 5)


def run_parts(parts, exchange, nsteps: int, t_end: float = 1e30):
    """nsteps explicit steps of the decomposed domain; returns per-step
    (t, dt, max_speed, mass) with the mass summed over parts in part order."""
    out = []
    for _ in range(nsteps):
        exchange.halo()
        loc = [p.local_cfl() for p in parts]
        dts = exchange.allreduce_min(min(x[0] for x in loc))
        ms = exchange.allreduce_max(max(x[1] for x in loc))
        recs = [p.step_global(t_end, dts, ms) for p in parts]
        mass = exchange.allreduce_sum(sum(r.mass for r in recs))
        out.append((recs[0].t, recs[0].dt, ms, mass))
        if not recs[0].t < t_end:
            break
    return np.array(out, dtype=np.float64).reshape(-1, 4)


__all__ = ["partition", "cost_weights", "measured_cost_weights", "refine_weights", "part_step_ms", "partition_raw", "rank_mesh", "local_mesh", "LocalMesh", "PartSolver", "LocalExchange", "TorchExchange",
           "run_parts", "push_plan", "LinkedPart", "link_local", "link_torch", "exchange_link_info",
           "run_lockstep", "run_ranks", "DeviceError", "LinkUnavailable"]

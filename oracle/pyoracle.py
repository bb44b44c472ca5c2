"""TEST INFRASTRUCTURE ONLY -- ctypes access to the checkers.

* ``COracle``: the plain-C restatement (oracle/swe_oracle.c -> liboracle.so),
  builds anywhere (gcc), used by the GPU parity tests on the box.
* ``RefOracle``: the reference itself (oracle/ref_shim.cpp over the unmodified
  /root/reference headers -> oracle/_ref/libswe_ref.so), built in this
  container and shipped as a prebuilt .so.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libswe_ref.so"

vp, ci, cl, cd = C.c_void_p, C.c_int, C.c_long, C.c_double
P = lambda a: None if a is None else a.ctypes.data_as(vp)  # noqa: E731


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


class so_params(C.Structure):
    _fields_ = [("g", cd), ("h_dry", cd), ("cfl", cd), ("dt_max", cd), ("h_ref", cd)]


class so_mesh(C.Structure):
    _fields_ = [("n_cells", ci), ("n_edges", ci)] + [(n, vp) for n in (
        "area", "inradius", "bed", "manning", "cell_edge", "cell_sign", "edge_left", "edge_right",
        "nx", "ny", "len")]


class so_clock(C.Structure):
    _fields_ = [("t", cd), ("step", cl), ("clipped_volume", cd), ("clip_events", cl)]


class so_step_stats(C.Structure):
    _fields_ = [("step", cl), ("t", cd), ("dt", cd), ("max_speed", cd)]


class MeshArrays:
    """Reference-numbered SoA arrays of one mesh (any producer)."""

    def __init__(self, area, inradius, bed, manning, cell_edge, cell_sign, edge_left, edge_right,
                 nx, ny, length):
        f = lambda a, t: np.ascontiguousarray(a, dtype=t)  # noqa: E731
        self.area, self.inradius, self.bed, self.manning = (f(a, np.float64) for a in
                                                            (area, inradius, bed, manning))
        self.cell_edge = f(cell_edge, np.int32).reshape(-1)
        self.cell_sign = f(cell_sign, np.int32).reshape(-1)
        self.edge_left, self.edge_right = f(edge_left, np.int32), f(edge_right, np.int32)
        self.nx, self.ny, self.len = (f(a, np.float64) for a in (nx, ny, length))
        self.n_cells, self.n_edges = len(self.area), len(self.nx)

    @classmethod
    def from_mesh(cls, m):
        """from paper_1807_00672_b200.api.Mesh (or anything with those fields)"""
        return cls(m.cell_area, m.cell_inradius, m.cell_bed, m.cell_manning, m.cell_edge,
                   m.cell_sign, m.edge_left, m.edge_right, m.nx, m.ny, m.edge_length)

    def c(self) -> so_mesh:
        m = so_mesh()
        m.n_cells, m.n_edges = self.n_cells, self.n_edges
        for n in ("area", "inradius", "bed", "manning", "cell_edge", "cell_sign", "edge_left",
                  "edge_right", "nx", "ny", "len"):
            setattr(m, n, P(getattr(self, n)))
        return m


def _params(p=None):
    if p is None:
        return so_params(9.81, 1e-6, 0.7, 1.0, 1.0)
    return so_params(p.g, p.h_dry, p.cfl, p.dt_max, p.h_ref)


class COracle:
    """The C restatement (swe_oracle.c)."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build_oracle()
        self.lib = C.CDLL(str(ORACLE_SO))
        L = self.lib
        L.so_compute_fluxes.restype = ci
        L.so_compute_fluxes.argtypes = [C.POINTER(so_mesh), C.POINTER(so_params), vp, vp, vp, vp, vp]
        L.so_advance_step.restype = ci
        L.so_advance_step.argtypes = [C.POINTER(so_mesh), C.POINTER(so_params), cd, vp, vp, vp, vp,
                                      vp, vp, vp, C.POINTER(so_clock), C.POINTER(so_step_stats),
                                      C.POINTER(ci), C.POINTER(cd)]
        L.so_total_mass.restype = cd
        L.so_total_mass.argtypes = [C.POINTER(so_mesh), vp]
        L.so_stable_dt_blocks.restype = ci
        L.so_stable_dt_blocks.argtypes = [C.POINTER(so_mesh), C.POINTER(so_params), vp, vp, vp,
                                          C.POINTER(cd), C.POINTER(cd)]
        L.so_build_mesh.restype = ci
        L.so_build_mesh.argtypes = [ci, vp, ci, vp] + [vp] * 13
        L.so_batch.restype = None
        L.so_batch.argtypes = [ci, cl, C.POINTER(so_params), vp, vp, vp, vp, vp]
        L.so_local_cfl.restype = ci
        L.so_local_cfl.argtypes = [C.POINTER(so_mesh), ci, C.POINTER(so_params), vp, vp, vp,
                                   C.POINTER(cd), C.POINTER(cd)]
        L.so_step_owned.restype = ci
        L.so_step_owned.argtypes = [C.POINTER(so_mesh), ci, C.POINTER(so_params), cd, cd, cd, vp,
                                    vp, vp, vp, vp, vp, vp, C.POINTER(so_clock),
                                    C.POINTER(so_step_stats), C.POINTER(ci)]

    # ---- decomposed domain (owned cells first, ghosts after) ----
    def local_cfl(self, m: "MeshArrays", n_owned, h, qx, qy, params=None):
        mc, p = m.c(), _params(params)
        d, s = cd(), cd()
        bad = self.lib.so_local_cfl(C.byref(mc), n_owned, C.byref(p), P(_c(h)), P(_c(qx)),
                                    P(_c(qy)), C.byref(d), C.byref(s))
        return d.value, s.value, bad

    def step_owned(self, m: "MeshArrays", n_owned, state, clk, t_end, dts, max_speed,
                   params=None):
        """state: [h, qx, qy] arrays updated in place; clk: so_clock."""
        mc, p = m.c(), _params(params)
        out = [np.empty_like(a) for a in state]
        scratch = np.empty(6 * m.n_edges)
        st, ei = so_step_stats(), ci()
        rc = self.lib.so_step_owned(C.byref(mc), n_owned, C.byref(p), t_end, dts, max_speed,
                                    *[P(a) for a in state], *[P(a) for a in out], P(scratch),
                                    C.byref(clk), C.byref(st), C.byref(ei))
        if rc == 0:
            for a, b in zip(state, out):
                a[:] = b
        return rc, st

    def point(self, kind, l, r=None, z=None, nrm=None, params=None):
        """so_batch: same kinds and layouts as swe_dev_point_eval."""
        l = _c(l).reshape(-1, 3)
        n = len(l)
        width = {2: 6, 4: 1}.get(kind, 3)
        out = np.empty((n, width))
        p = _params(params)
        self.lib.so_batch(kind, n, C.byref(p), P(l), P(None if r is None else _c(r)),
                          P(None if z is None else _c(z)), P(None if nrm is None else _c(nrm)),
                          P(out))
        return out if width > 1 else out[:, 0]

    def compute_fluxes(self, m: MeshArrays, h, qx, qy, params=None):
        left = np.empty((m.n_edges, 3))
        right = np.empty((m.n_edges, 3))
        mc, p = m.c(), _params(params)
        bad = self.lib.so_compute_fluxes(C.byref(mc), C.byref(p), P(h), P(qx), P(qy), P(left),
                                         P(right))
        return left, right, bad

    def total_mass(self, m: MeshArrays, h):
        mc = m.c()
        return self.lib.so_total_mass(C.byref(mc), P(np.ascontiguousarray(h)))

    def advance(self, m: MeshArrays, h, qx, qy, t=0.0, step=0, t_end=1e30, nsteps=1,
                stop_at_t_end=False, params=None, clipped_volume=0.0, clip_events=0):
        """nsteps of advance_step; returns dict with state, clock, per-step
        dt/max_speed, and error (kind, index, h) if a step failed."""
        mc, p = m.c(), _params(params)
        cur = [np.array(a, dtype=np.float64, copy=True) for a in (h, qx, qy)]
        nxt = [np.empty_like(cur[0]) for _ in range(3)]
        scratch = np.empty(6 * m.n_edges)
        clk = so_clock(t, step, clipped_volume, clip_events)
        st = so_step_stats()
        ei, eh = ci(), cd()
        dts, ms = [], []
        err = None
        for _ in range(nsteps):
            if stop_at_t_end and not (clk.t < t_end):
                break
            rc = self.lib.so_advance_step(C.byref(mc), C.byref(p), t_end, P(cur[0]), P(cur[1]),
                                          P(cur[2]), P(nxt[0]), P(nxt[1]), P(nxt[2]), P(scratch),
                                          C.byref(clk), C.byref(st), C.byref(ei), C.byref(eh))
            if rc != 0:
                err = (rc, ei.value, eh.value)
                break
            cur, nxt = nxt, cur
            dts.append(st.dt)
            ms.append(st.max_speed)
        return dict(h=cur[0], qx=cur[1], qy=cur[2], t=clk.t, step=clk.step,
                    clipped_volume=clk.clipped_volume, clip_events=clk.clip_events,
                    dts=np.array(dts), max_speeds=np.array(ms), error=err)

    def build_mesh(self, nodes, tris):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        tris = np.ascontiguousarray(tris, dtype=np.int32)
        nn, nc = len(nodes), len(tris)
        out = dict(cell_nodes=np.empty((nc, 3), np.int32), area=np.empty(nc), cx=np.empty(nc),
                   cy=np.empty(nc), inradius=np.empty(nc), cell_edge=np.empty((nc, 3), np.int32),
                   cell_sign=np.empty((nc, 3), np.int32),
                   edge_nodes=np.empty((3 * nc, 2), np.int32), edge_left=np.empty(3 * nc, np.int32),
                   edge_right=np.empty(3 * nc, np.int32), nx=np.empty(3 * nc), ny=np.empty(3 * nc),
                   len=np.empty(3 * nc))
        keys = ("cell_nodes", "area", "cx", "cy", "inradius", "cell_edge", "cell_sign",
                "edge_nodes", "edge_left", "edge_right", "nx", "ny", "len")
        ne = self.lib.so_build_mesh(nn, P(nodes), nc, P(tris), *[P(out[k]) for k in keys])
        if ne < 0:
            raise ValueError(f"so_build_mesh failed: {ne}")
        for k in ("edge_nodes", "edge_left", "edge_right", "nx", "ny", "len"):
            out[k] = out[k][:ne].copy()
        return out


class RefOracle:
    """The reference itself (oracle/_ref/libswe_ref.so)."""

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        self.lib = C.CDLL(str(REF_SO))
        L = self.lib
        L.ref_build_mesh.restype = vp
        L.ref_build_mesh.argtypes = [ci, vp, ci, vp, vp, vp, C.c_char_p, ci]
        L.ref_mesh_free.argtypes = [vp]
        L.ref_mesh_sizes.argtypes = [vp, C.POINTER(ci), C.POINTER(ci), C.POINTER(ci)]
        L.ref_mesh_export.argtypes = [vp] + [vp] * 13
        L.ref_compute_fluxes.restype = ci
        L.ref_compute_fluxes.argtypes = [vp, vp, vp, vp, vp, vp, vp, ci, C.c_char_p, ci]
        L.ref_total_mass.restype = cd
        L.ref_total_mass.argtypes = [vp, vp]
        L.ref_advance.restype = ci
        L.ref_advance.argtypes = [vp, vp, vp, vp, vp, C.POINTER(cd), C.POINTER(cl), cd, cl, ci, ci,
                                  vp, vp, C.POINTER(cd), C.POINTER(cl), C.POINTER(cd),
                                  C.POINTER(cd), C.POINTER(cl), C.c_char_p, ci]
        L.ref_run.restype = ci
        L.ref_run.argtypes = [vp, vp, vp, vp, vp, C.POINTER(cd), C.POINTER(cl), cd, cd, cl, ci, vp,
                              cl, C.POINTER(cl), vp, vp, cl, C.POINTER(cl), C.c_char_p, ci]
        L.ref_hllc.restype = ci
        L.ref_hllc.argtypes = [cl, vp, vp, vp, vp, vp]
        L.ref_wall.argtypes = [cl, vp, vp, vp, vp]
        L.ref_edge.argtypes = [cl, vp, vp, vp, vp, vp, vp, vp]
        L.ref_friction.argtypes = [cl, vp, vp, vp, vp, vp]
        L.ref_pow43.argtypes = [cl, vp, vp]
        L.ref_point.argtypes = [ci, cl, vp, vp, vp, vp, vp, vp]
        L.ref_stable_dt.argtypes = [cl, vp, vp, vp, vp, vp, C.POINTER(cd), C.POINTER(cl)]
        L.ref_wave_speeds.argtypes = [cl, vp, vp, vp]
        L.ref_case_defaults.restype = ci
        L.ref_case_defaults.argtypes = [C.c_char_p, vp]
        L.ref_generate_square_mesh.argtypes = [ci, ci, cd, cd, vp, vp]
        L.ref_init_case.restype = ci
        L.ref_init_case.argtypes = [C.c_char_p, vp, ci, vp, ci, vp, vp, vp, vp, vp, vp, C.c_char_p, ci]
        L.ref_rotated_cell_index.restype = ci
        L.ref_rotated_cell_index.argtypes = [ci, ci, ci]
        L.ref_stoker.argtypes = [cl, cd, cd, vp, cd, cd, cd, vp, vp]

    # --- mesh
    def build_mesh(self, nodes, tris, bed, manning):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        tris = np.ascontiguousarray(tris, dtype=np.int32)
        bed = np.ascontiguousarray(bed, dtype=np.float64)
        manning = np.ascontiguousarray(manning, dtype=np.float64)
        err = C.create_string_buffer(1024)
        h = self.lib.ref_build_mesh(len(nodes), P(nodes), len(tris), P(tris), P(bed), P(manning),
                                    err, 1024)
        if not h:
            raise ValueError(err.value.decode())
        return RefMesh(self, h, bed, manning)

    def square(self, nx, ny, lx, ly):
        nodes = np.empty(((nx + 1) * (ny + 1), 2))
        tris = np.empty((2 * nx * ny, 3), np.int32)
        self.lib.ref_generate_square_mesh(nx, ny, lx, ly, P(nodes), P(tris))
        return nodes, tris

    def case_defaults(self, name):
        v = np.empty(10)
        self.lib.ref_case_defaults(name.encode(), P(v))
        return v

    def init_case(self, name, spec, nodes, tris):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        tris = np.ascontiguousarray(tris, dtype=np.int32)
        nc = len(tris)
        out = [np.empty(nc) for _ in range(5)]
        err = C.create_string_buffer(1024)
        spec = np.ascontiguousarray(spec, dtype=np.float64)
        rc = self.lib.ref_init_case(name.encode(), P(spec), len(nodes), P(nodes), nc, P(tris),
                                    *[P(a) for a in out], err, 1024)
        if rc:
            raise ValueError(err.value.decode())
        return out  # bed, manning, h, qx, qy

    # --- point physics
    def hllc(self, l, r, nrm, params=None):
        out = np.empty((len(l), 3))
        pa = _pa(params)
        rc = self.lib.ref_hllc(len(l), P(pa), P(_c(l)), P(_c(r)), P(_c(nrm)), P(out))
        if rc:
            raise ValueError("negative depth")
        return out

    def wall(self, u, nrm, params=None):
        out = np.empty((len(u), 3))
        self.lib.ref_wall(len(u), P(_pa(params)), P(_c(u)), P(_c(nrm)), P(out))
        return out

    def edge(self, l, r, z, nrm, params=None):
        left, right = np.empty((len(l), 3)), np.empty((len(l), 3))
        self.lib.ref_edge(len(l), P(_pa(params)), P(_c(l)), P(_c(r)), P(_c(z)), P(_c(nrm)),
                          P(left), P(right))
        return left, right

    def friction(self, u, n, dt, params=None):
        out = np.empty((len(u), 3))
        self.lib.ref_friction(len(u), P(_pa(params)), P(_c(u)), P(_c(n)), P(_c(dt)), P(out))
        return out

    def point(self, kind, l, r=None, z=None, nrm=None, params=None):
        """ref_point: kernels.hpp entry points, swe_dev_point_eval kinds 5-9."""
        l = _c(l).reshape(-1, 3)
        n = len(l)
        width = {7: 12, 8: 1, 9: 5}.get(kind, 3)
        out = np.empty((n, width))
        cv = lambda a: None if a is None else P(_c(a))
        rc = self.lib.ref_point(kind, n, P(_pa(params)), P(l), cv(r), cv(z), cv(nrm), P(out))
        assert rc == 0
        return out if width > 1 else out[:, 0]

    def stable_dt(self, h, qx, qy, r, params=None):
        """-> (dt, None) or (None, bad cell)."""
        dt, bad = C.c_double(), C.c_long()
        rc = self.lib.ref_stable_dt(len(h), P(_pa(params)), P(_c(h)), P(_c(qx)), P(_c(qy)),
                                    P(_c(r)), C.byref(dt), C.byref(bad))
        return (dt.value, None) if rc == 0 else (None, bad.value)

    def pow43(self, h):
        h = _c(h)
        out = np.empty(len(h))
        self.lib.ref_pow43(len(h), P(h), P(out))
        return out


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _pa(p):
    if p is None:
        return np.array([9.81, 1e-6, 0.7, 1.0, 1.0])
    return np.array([p.g, p.h_dry, p.cfl, p.dt_max, p.h_ref])


class RefMesh:
    def __init__(self, ref: RefOracle, handle, bed, manning):
        self.ref, self.handle = ref, handle
        nc, ne, nb = ci(), ci(), ci()
        ref.lib.ref_mesh_sizes(handle, C.byref(nc), C.byref(ne), C.byref(nb))
        self.n_cells, self.n_edges, self.n_boundary = nc.value, ne.value, nb.value
        Cn, En = self.n_cells, self.n_edges
        self.a = dict(cell_nodes=np.empty((Cn, 3), np.int32), area=np.empty(Cn), cx=np.empty(Cn),
                      cy=np.empty(Cn), inradius=np.empty(Cn), cell_edge=np.empty((Cn, 3), np.int32),
                      cell_sign=np.empty((Cn, 3), np.int32), edge_nodes=np.empty((En, 2), np.int32),
                      edge_left=np.empty(En, np.int32), edge_right=np.empty(En, np.int32),
                      nx=np.empty(En), ny=np.empty(En), len=np.empty(En))
        keys = ("cell_nodes", "area", "cx", "cy", "inradius", "cell_edge", "cell_sign",
                "edge_nodes", "edge_left", "edge_right", "nx", "ny", "len")
        ref.lib.ref_mesh_export(handle, *[P(self.a[k]) for k in keys])
        self.bed, self.manning = bed, manning

    def __del__(self):
        if self.handle:
            self.ref.lib.ref_mesh_free(self.handle)
            self.handle = None

    def arrays(self) -> MeshArrays:
        a = self.a
        return MeshArrays(a["area"], a["inradius"], self.bed, self.manning, a["cell_edge"],
                          a["cell_sign"], a["edge_left"], a["edge_right"], a["nx"], a["ny"], a["len"])

    def compute_fluxes(self, h, qx, qy, threads=1, params=None):
        left, right = np.empty((self.n_edges, 3)), np.empty((self.n_edges, 3))
        err = C.create_string_buffer(1024)
        rc = self.ref.lib.ref_compute_fluxes(self.handle, P(_pa(params)), P(_c(h)), P(_c(qx)),
                                             P(_c(qy)), P(left), P(right), threads, err, 1024)
        return left, right, rc, err.value.decode()

    def total_mass(self, h):
        return self.ref.lib.ref_total_mass(self.handle, P(_c(h)))

    def advance(self, h, qx, qy, t=0.0, step=0, t_end=1e30, nsteps=1, stop_at_t_end=False,
                threads=1, params=None, clipped_volume=0.0, clip_events=0):
        h, qx, qy = (np.array(a, dtype=np.float64, copy=True) for a in (h, qx, qy))
        dts, ms = np.zeros(nsteps), np.zeros(nsteps)
        tt, ss, cv, ce = cd(t), cl(step), cd(clipped_volume), cl(clip_events)
        fs, us, done = cd(), cd(), cl()
        err = C.create_string_buffer(1024)
        rc = self.ref.lib.ref_advance(self.handle, P(_pa(params)), P(h), P(qx), P(qy), C.byref(tt),
                                      C.byref(ss), t_end, nsteps, int(stop_at_t_end), threads,
                                      P(dts), P(ms), C.byref(cv), C.byref(ce), C.byref(fs),
                                      C.byref(us), C.byref(done), err, 1024)
        n = done.value
        return dict(h=h, qx=qx, qy=qy, t=tt.value, step=ss.value, dts=dts[:n], max_speeds=ms[:n],
                    clipped_volume=cv.value, clip_events=ce.value, flux_s=fs.value,
                    update_s=us.value, rc=rc, error=err.value.decode(), done=n)

    def run(self, h, qx, qy, t_end, t=0.0, step=0, snapshot_interval=0.0, max_steps=100_000_000,
            threads=1, max_rows=1 << 20, snapshots=False, params=None):
        h, qx, qy = (np.array(a, dtype=np.float64, copy=True) for a in (h, qx, qy))
        series, stats, snaps = np.zeros((max_rows, 5)), np.zeros(9), np.zeros(4096)
        tt, ss, nr, ns = cd(t), cl(step), cl(), cl()
        err = C.create_string_buffer(1024)
        rc = self.ref.lib.ref_run(self.handle, P(_pa(params)), P(h), P(qx), P(qy), C.byref(tt),
                                  C.byref(ss), t_end, snapshot_interval, max_steps, threads,
                                  P(series), max_rows, C.byref(nr), P(stats),
                                  P(snaps) if snapshots else None, 4096, C.byref(ns), err, 1024)
        return dict(h=h, qx=qx, qy=qy, t=tt.value, step=ss.value,
                    series=series[:min(nr.value, max_rows)].copy(), stats=stats,
                    snaps=snaps[:ns.value].tolist(), rc=rc, error=err.value.decode())


REF_IO_SO = HERE / "_ref" / "libswe_ref_io.so"


class RefIO:
    """The reference's SWEMESH reader / writer (io.hpp:80-165) through
    oracle/_ref/libswe_ref_io.so -- the checker of include/swe/swemesh.hpp."""

    @staticmethod
    def available() -> bool:
        return REF_IO_SO.exists()

    def __init__(self):
        if not REF_IO_SO.exists():
            raise FileNotFoundError(f"{REF_IO_SO} not built (needs /root/reference at build time)")
        L = self.lib = C.CDLL(str(REF_IO_SO))
        L.refio_parse.restype = vp
        L.refio_parse.argtypes = [C.c_char_p, C.c_longlong, C.c_char_p, ci]
        L.refio_read.restype = vp
        L.refio_read.argtypes = [C.c_char_p, C.c_char_p, ci]
        L.refio_sizes.argtypes = [vp, C.POINTER(ci), C.POINTER(ci)]
        L.refio_export.argtypes = [vp, vp, vp, vp, vp]
        L.refio_free.argtypes = [vp]
        L.refio_write.restype = ci
        L.refio_write.argtypes = [C.c_char_p, ci, vp, ci, vp, vp, vp, C.c_char_p, ci]

    def _result(self, h, err):
        if not h:
            raise ValueError(err.value.decode(errors="replace"))
        nn, nc = ci(), ci()
        self.lib.refio_sizes(h, C.byref(nn), C.byref(nc))
        xy = np.empty((nn.value, 2))
        tris = np.empty((nc.value, 3), dtype=np.int32)
        bed, man = np.empty(nc.value), np.empty(nc.value)
        self.lib.refio_export(h, xy.ctypes.data, tris.ctypes.data, bed.ctypes.data,
                              man.ctypes.data)
        self.lib.refio_free(h)
        return xy, tris, bed, man

    def parse(self, text):
        """-> (nodes[nn,2], tris[nc,3], bed, manning); ValueError(reference message)."""
        b = text.encode() if isinstance(text, str) else bytes(text)
        err = C.create_string_buffer(1024)
        return self._result(self.lib.refio_parse(b, len(b), err, 1024), err)

    def read(self, path):
        err = C.create_string_buffer(1024)
        return self._result(self.lib.refio_read(str(path).encode(), err, 1024), err)

    def write(self, path, nodes, tris, bed, man):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        tris = np.ascontiguousarray(tris, dtype=np.int32)
        bed = np.ascontiguousarray(bed, dtype=np.float64)
        man = np.ascontiguousarray(man, dtype=np.float64)
        err = C.create_string_buffer(1024)
        if self.lib.refio_write(str(path).encode(), len(nodes), nodes.ctypes.data, len(tris),
                                tris.ctypes.data, bed.ctypes.data, man.ctypes.data, err, 1024):
            raise ValueError(err.value.decode())

"""Python face of the B200 shallow-water step (tests, bench, notebooks).

Two layers, both over libswe_b200.so:

* reference-shaped calls -- ``compute_fluxes``, ``advance``, ``run``,
  ``total_mass`` -- that execute the C++ drop-in engine
  (include/swe/engine.hpp: the reference's compute_fluxes / advance_step /
  run / total_mass, /root/reference/proj/include/swe/engine.hpp:128-394) and
  raise the reference's exception kinds with its message texts;
* ``DeviceSolver``: the C-ABI context (include/swe_dev.h) with the state
  resident in HBM, for throughput runs.

Meshes and initial states come from the host producers (include/swe/mesh.hpp,
include/swe/cases.hpp) through include/swe_host.h.  Arrays are numpy, in the
reference numbering.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class SweError(RuntimeError):
    """swe::error"""


class NumericError(SweError):
    """swe::numeric_error (NaN/Inf, negative depth, blow-up)"""


class ConfigError(SweError):
    """swe::config_error"""


class MeshError(SweError):
    """swe::mesh_error"""


class CaseError(SweError):
    """swe::case_error"""


class DeviceError(SweError):
    """CUDA runtime failure (no reference counterpart)"""


class IoError(SweError):
    """swe::io_error"""


_KINDS = {1: NumericError, 2: ConfigError, 3: MeshError, 4: CaseError, 5: DeviceError,
          7: IoError}


def _raise(kind: int, msg: bytes | str):
    if isinstance(msg, bytes):
        msg = msg.decode(errors="replace")
    raise _KINDS.get(kind, SweError)(msg)


def _errbuf():
    return C.create_string_buffer(1024)


@dataclass
class PhysParams:
    """swe::PhysParams (core.hpp:36-42)"""
    g: float = 9.81
    h_dry: float = 1e-6
    cfl: float = 0.7
    dt_max: float = 1.0
    h_ref: float = 1.0

    def array(self) -> np.ndarray:
        return np.array([self.g, self.h_dry, self.cfl, self.dt_max, self.h_ref], dtype=np.float64)

    def c(self) -> L.swe_params:
        return L.swe_params(self.g, self.h_dry, self.cfl, self.dt_max, self.h_ref)


@dataclass
class FieldState:
    """swe::FieldState (engine.hpp:54-70), SoA numpy arrays."""
    h: np.ndarray
    qx: np.ndarray
    qy: np.ndarray

    @classmethod
    def zeros(cls, n: int) -> "FieldState":
        return cls(np.zeros(n), np.zeros(n), np.zeros(n))

    def copy(self) -> "FieldState":
        return FieldState(self.h.copy(), self.qx.copy(), self.qy.copy())

    def __len__(self):
        return len(self.h)


class RawMesh:
    """swe::RawMesh (mesh.hpp:14-17); owns a host handle."""

    def __init__(self, handle, owner=None):
        """owner: object that owns a borrowed handle (kept alive), else we own it."""
        if not handle:
            raise MeshError("null raw mesh")
        self._lib = L.load()
        self.handle = handle
        nn, nc = C.c_int(), C.c_int()
        self._lib.swe_host_raw_sizes(handle, C.byref(nn), C.byref(nc))
        self.nodes = np.empty((nn.value, 2))
        self.triangles = np.empty((nc.value, 3), dtype=np.int32)
        self._lib.swe_host_raw_export(handle, L.ptr(self.nodes), L.ptr(self.triangles))
        self._owner = owner
        self._owned = owner is None

    def __del__(self):
        if getattr(self, "_owned", False) and self.handle:
            self._lib.swe_host_raw_free(self.handle)
            self.handle = None

    @classmethod
    def from_arrays(cls, nodes, triangles) -> "RawMesh":
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        tris = np.ascontiguousarray(triangles, dtype=np.int32)
        lib = L.load()
        return cls(lib.swe_host_raw_arrays(len(nodes), L.ptr(nodes), len(tris), L.ptr(tris)))

    @property
    def n_cells(self):
        return len(self.triangles)


class _SweMeshFile:
    """owns a swe_host_swemesh_* handle"""

    def __init__(self, h):
        self._lib, self.h = L.load(), h

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.swe_host_swemesh_free(self.h)
            self.h = None


def _swemesh_result(h, err):
    if not h:
        _raise(7, err.value)
    f = _SweMeshFile(h)
    raw = RawMesh(f._lib.swe_host_swemesh_raw(h), owner=f)
    bed, man = np.empty(raw.n_cells), np.empty(raw.n_cells)
    f._lib.swe_host_swemesh_fields(h, L.ptr(bed), L.ptr(man))
    return raw, bed, man


def read_swemesh(path, threads: int = 0):
    """SWEMESH 1 file -> (RawMesh, bed, manning) (io.hpp read_mesh_native_file,
    parsed in parallel by include/swe/swemesh.hpp); raises IoError."""
    err = _errbuf()
    return _swemesh_result(L.load().swe_host_swemesh_read(str(path).encode(), threads, err,
                                                          len(err)), err)


def parse_swemesh(text, threads: int = 0):
    """SWEMESH 1 text (str or bytes) -> (RawMesh, bed, manning)."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    err = _errbuf()
    return _swemesh_result(L.load().swe_host_swemesh_parse(b, len(b), threads, err, len(err)), err)


def write_swemesh(path, raw: RawMesh, bed, manning, threads: int = 0):
    """io.hpp write_mesh_native_file (17 significant digits), formatted in parallel."""
    bed = np.ascontiguousarray(bed, dtype=np.float64)
    man = np.ascontiguousarray(manning, dtype=np.float64)
    if len(bed) != raw.n_cells or len(man) != raw.n_cells:
        raise IoError("write_mesh_native: bed / manning size != cell count")
    err = _errbuf()
    rc = L.load().swe_host_swemesh_write(str(path).encode(), raw.handle, L.ptr(bed), L.ptr(man),
                                         threads, err, len(err))
    if rc:
        _raise(rc, err.value)


def generate_square_mesh(nx: int, ny: int, lx: float, ly: float) -> RawMesh:
    """mesh.hpp:67-87"""
    err = _errbuf()
    h = L.load().swe_host_raw_square(nx, ny, lx, ly, err, len(err))
    if not h:
        _raise(3, err.value)
    return RawMesh(h)


def generate_unstructured_mesh(nx, ny, lx, ly, jitter=0.2, seed=1807) -> RawMesh:
    err = _errbuf()
    h = L.load().swe_host_raw_unstructured(nx, ny, lx, ly, jitter, seed, err, len(err))
    if not h:
        _raise(3, err.value)
    return RawMesh(h)


class Mesh:
    """swe::Mesh (mesh.hpp:33-61) exported as SoA numpy arrays."""

    def __init__(self, handle):
        self._lib = L.load()
        self.handle = handle
        nc, ne, nb = C.c_int(), C.c_int(), C.c_int()
        self._lib.swe_host_mesh_sizes(handle, C.byref(nc), C.byref(ne), C.byref(nb))
        Cn, En = nc.value, ne.value
        self.n_cells, self.n_edges, self.n_boundary_edges = Cn, En, nb.value
        self.cell_nodes = np.empty((Cn, 3), np.int32)
        self.cell_area = np.empty(Cn)
        cx, cy = np.empty(Cn), np.empty(Cn)
        self.cell_inradius = np.empty(Cn)
        self.cell_edge = np.empty((Cn, 3), np.int32)
        self.cell_sign = np.empty((Cn, 3), np.int32)
        self.edge_nodes = np.empty((En, 2), np.int32)
        self.edge_left = np.empty(En, np.int32)
        self.edge_right = np.empty(En, np.int32)
        nx, ny = np.empty(En), np.empty(En)
        self.edge_length = np.empty(En)
        self._lib.swe_host_mesh_export(
            handle, *[L.ptr(a) for a in (self.cell_nodes, self.cell_area, cx, cy, self.cell_inradius,
                                         self.cell_edge, self.cell_sign, self.edge_nodes,
                                         self.edge_left, self.edge_right, nx, ny, self.edge_length)])
        self.cx, self.cy, self.nx, self.ny = cx, cy, nx, ny
        self.cell_centroid = np.stack([cx, cy], axis=1)
        self.edge_normal = np.stack([nx, ny], axis=1)
        self.cell_bed = None
        self.cell_manning = None

    def __del__(self):
        if getattr(self, "handle", None):
            self._lib.swe_host_mesh_free(self.handle)
            self.handle = None

    def view(self) -> L.swe_mesh_view:
        """swe_mesh_view over this mesh's arrays (keeps references alive)."""
        v = L.swe_mesh_view()
        v.n_cells, v.n_edges = self.n_cells, self.n_edges
        self._view_keep = [np.ascontiguousarray(a) for a in (
            self.cell_area, self.cell_inradius, self.cell_bed, self.cell_manning, self.cx, self.cy,
            self.cell_edge.reshape(-1), self.cell_sign.reshape(-1), self.edge_left,
            self.edge_right, self.nx, self.ny, self.edge_length)]
        k = self._view_keep
        v.area, v.inradius, v.bed, v.manning = (L.dptr(a) for a in k[0:4])
        v.cx, v.cy = L.dptr(k[4]), L.dptr(k[5])
        v.cell_edge, v.cell_sign, v.edge_left, v.edge_right = (L.iptr(a) for a in k[6:10])
        v.nx, v.ny, v.len = (L.dptr(a) for a in k[10:13])
        return v


def build_mesh(raw: RawMesh, bathymetry, manning, device: int | None = None) -> Mesh:
    """mesh.hpp:121-240 (re-implemented in include/swe/mesh.hpp); device=k:
    computed on GPU k (swe_dev_build_mesh) -- the same Mesh bit for bit."""
    bed = np.ascontiguousarray(bathymetry, dtype=np.float64)
    man = np.ascontiguousarray(manning, dtype=np.float64)
    err = _errbuf()
    if len(bed) != raw.n_cells or len(man) != raw.n_cells:
        raise MeshError(f"build_mesh: bathymetry/manning arrays must have one entry per triangle "
                        f"(got {len(bed)}/{len(man)} for {raw.n_cells} triangles)")
    lib = L.load()
    if device is None:
        h = lib.swe_host_build_mesh(raw.handle, L.ptr(bed), L.ptr(man), err, len(err))
    else:
        h = lib.swe_host_build_mesh_device(raw.handle, L.ptr(bed), L.ptr(man), device, err,
                                           len(err))
    if not h:
        _raise(3, err.value)
    m = Mesh(h)
    m.cell_bed, m.cell_manning = bed, man
    return m


CASE_SPEC_KEYS = ("lx", "ly", "eta0", "amplitude", "sigma", "manning", "h_left", "h_right",
                  "x_dam", "t_end")


def case_defaults(name: str) -> dict:
    """make_case (cases.hpp:53-85)"""
    v = np.empty(10)
    rc = L.load().swe_host_case_defaults(name.encode(), L.ptr(v))
    if rc:
        _raise(rc, f"unknown case '{name}'")
    return dict(zip(CASE_SPEC_KEYS, v.tolist()))


def init_case(name: str, raw: RawMesh, **overrides):
    """init_case (cases.hpp:114-181) -> (bed, manning, FieldState)."""
    spec = case_defaults(name)
    spec.update(overrides)
    v = np.array([spec[k] for k in CASE_SPEC_KEYS], dtype=np.float64)
    n = raw.n_cells
    bed, man, h, qx, qy = (np.empty(n) for _ in range(5))
    err = _errbuf()
    rc = L.load().swe_host_init_case(raw.handle, name.encode(), L.ptr(v), L.ptr(bed), L.ptr(man),
                                     L.ptr(h), L.ptr(qx), L.ptr(qy), err, len(err))
    if rc:
        _raise(rc, err.value)
    return bed, man, FieldState(h, qx, qy)


def setup_case(name: str, raw: RawMesh, **overrides):
    """setup_case (cases.hpp:189-193) -> (Mesh, FieldState)."""
    bed, man, st = init_case(name, raw, **overrides)
    return build_mesh(raw, bed, man), st


@dataclass
class Scenario:
    name: str
    raw: RawMesh
    bed: np.ndarray
    manning: np.ndarray
    state: FieldState
    t_end: float


def make_scenario(name: str, scale: float = 1.0, unstructured: bool = True, seed: int = 1807,
                  weak_nx: int = 2265) -> Scenario:
    """Benchmark configurations of BASELINE.json (include/swe/cases.hpp make_scenario)."""
    lib = L.load()
    err = _errbuf()
    t_end = C.c_double()
    s = lib.swe_host_scenario(name.encode(), scale, int(unstructured), seed, weak_nx,
                              C.byref(t_end), err, len(err))
    if not s:
        _raise(2, err.value)
    try:
        raw_h = lib.swe_host_scenario_raw(s)
        nn, nc = C.c_int(), C.c_int()
        lib.swe_host_raw_sizes(raw_h, C.byref(nn), C.byref(nc))
        nodes = np.empty((nn.value, 2))
        tris = np.empty((nc.value, 3), np.int32)
        lib.swe_host_raw_export(raw_h, L.ptr(nodes), L.ptr(tris))
        arrs = [np.empty(nc.value) for _ in range(5)]
        lib.swe_host_scenario_fields(s, *[L.ptr(a) for a in arrs])
    finally:
        lib.swe_host_scenario_free(s)
    raw = RawMesh.from_arrays(nodes, tris)
    bed, man, h, qx, qy = arrs
    return Scenario(name, raw, bed, man, FieldState(h, qx, qy), t_end.value)


# ---------------------------------------------------------------------------
# reference-shaped calls into the C++ drop-in engine
# ---------------------------------------------------------------------------

def compute_fluxes(state: FieldState, mesh: Mesh, params: PhysParams = PhysParams(), device=0):
    """engine.hpp:138-170 -> (left[E,3], right[E,3])."""
    left = np.empty((mesh.n_edges, 3))
    right = np.empty((mesh.n_edges, 3))
    err = _errbuf()
    p = params.array()
    rc = L.load().swe_api_compute_fluxes(mesh.handle, L.ptr(p), L.ptr(state.h), L.ptr(state.qx),
                                         L.ptr(state.qy), L.ptr(left), L.ptr(right), device, err,
                                         len(err))
    if rc:
        _raise(rc, err.value)
    return left, right


def total_mass(state: FieldState, mesh: Mesh, params: PhysParams = PhysParams(), device=0) -> float:
    """engine.hpp:128-132"""
    out = C.c_double()
    err = _errbuf()
    p = params.array()
    rc = L.load().swe_api_total_mass(mesh.handle, L.ptr(p), L.ptr(state.h), device, C.byref(out),
                                     err, len(err))
    if rc:
        _raise(rc, err.value)
    return out.value


@dataclass
class AdvanceResult:
    t: float
    step: int
    dts: np.ndarray
    max_speeds: np.ndarray
    clipped_volume: float
    clip_events: int
    done: int


def advance(mesh: Mesh, state: FieldState, t: float = 0.0, step: int = 0, t_end: float = 1e30,
            nsteps: int = 1, stop_at_t_end: bool = False, params: PhysParams = PhysParams(),
            clipped_volume: float = 0.0, clip_events: int = 0, device: int = 0) -> AdvanceResult:
    """nsteps x swe::advance_step (engine.hpp:226-319); state updated in place.
    Raises the reference's numeric_error on failure (state = last good step)."""
    dts, ms = np.zeros(nsteps), np.zeros(nsteps)
    tt, ss = C.c_double(t), C.c_long(step)
    cv, ce, done = C.c_double(clipped_volume), C.c_long(clip_events), C.c_long()
    err = _errbuf()
    p = params.array()
    rc = L.load().swe_api_advance(mesh.handle, L.ptr(p), L.ptr(state.h), L.ptr(state.qx),
                                  L.ptr(state.qy), C.byref(tt), C.byref(ss), t_end, nsteps,
                                  int(stop_at_t_end), device, L.ptr(dts), L.ptr(ms), C.byref(cv),
                                  C.byref(ce), C.byref(done), err, len(err))
    res = AdvanceResult(tt.value, ss.value, dts[:done.value], ms[:done.value], cv.value, ce.value,
                        done.value)
    if rc:
        e = _KINDS.get(rc, SweError)(err.value.decode(errors="replace"))
        e.result = res
        raise e
    return res


@dataclass
class RunResult:
    t: float
    step: int
    series: np.ndarray  # [n, 5] = step, t, dt, max_speed, mass
    stats: dict
    snapshots: list = field(default_factory=list)


STAT_KEYS = ("steps", "t_final", "mass_initial", "mass_final", "mass_drift_rel", "min_dt",
             "mean_dt", "clip_events", "clipped_volume")


def run(mesh: Mesh, state: FieldState, t_end: float, t: float = 0.0, step: int = 0,
        snapshot_interval: float = 0.0, max_steps: int = 100_000_000, max_rows: int = 1 << 20,
        snapshots: bool = False, params: PhysParams = PhysParams(), device: int = 0,
        snapshot_fields: int = 0) -> RunResult:
    """swe::run (engine.hpp:335-394); state updated in place.  snapshot_fields
    = k > 0 also keeps the first k snapshot states (RunResult.fields [k,3,C])."""
    series = np.zeros((max_rows, 5))
    stats = np.zeros(9)
    snaps = np.zeros(4096)
    fields = np.zeros((snapshot_fields, 3, mesh.n_cells)) if snapshot_fields else None
    if snapshot_fields:
        snaps = np.zeros(snapshot_fields)
    tt, ss = C.c_double(t), C.c_long(step)
    n_rows, n_snaps = C.c_long(), C.c_long()
    err = _errbuf()
    p = params.array()
    rc = L.load().swe_api_run(mesh.handle, L.ptr(p), L.ptr(state.h), L.ptr(state.qx),
                              L.ptr(state.qy), C.byref(tt), C.byref(ss), t_end, snapshot_interval,
                              max_steps, device, L.ptr(series), max_rows, C.byref(n_rows),
                              L.ptr(stats), L.ptr(snaps) if snapshots else None, len(snaps),
                              C.byref(n_snaps), L.ptr(fields), err, len(err))
    if rc:
        _raise(rc, err.value)
    res = RunResult(tt.value, ss.value, series[:min(n_rows.value, max_rows)].copy(),
                    dict(zip(STAT_KEYS, stats.tolist())),
                    snaps[:min(n_snaps.value, len(snaps))].tolist() if snapshots else [])
    res.fields = fields[:min(n_snaps.value, snapshot_fields)] if snapshot_fields else None
    return res


# ---------------------------------------------------------------------------
# the device-resident context
# ---------------------------------------------------------------------------

def _check(rc, what):
    if rc != L.SWE_OK:
        lib = L.load()
        raise DeviceError(f"{what}: {lib.swe_dev_strerror(rc).decode()} "
                          f"({lib.swe_dev_last_error().decode()})")


_STATUS_MSG = {
    L.SWE_NONFINITE_SPEED: lambda s: f"stable_dt: non-finite velocity in cell {s.index}",
    L.SWE_NEGATIVE_DEPTH: lambda s: f"compute_fluxes: negative depth at edge {s.index}",
    L.SWE_BLOWUP: lambda s: f"advance_step: numeric blowup at step {s.step}, cell {s.index}, "
                            f"dt {s.dt:f} (h={s.h:f})",
}


def _status(rc, st, what):
    if rc in _STATUS_MSG:
        raise NumericError(_STATUS_MSG[rc](st))
    _check(rc, what)


class DeviceSolver:
    """swe_dev_ctx: mesh + double-buffered state resident on one B200."""

    def __init__(self, mesh: Mesh, params: PhysParams = PhysParams(), device: int = 0,
                 identity_order: bool = False, graph: bool = True, two_phase: bool = False):
        self.lib = L.load()
        self.mesh = mesh
        self.params = params
        v = mesh.view()
        p = params.c()
        ctx = C.c_void_p()
        flags = ((L.SWE_FLAG_IDENTITY_ORDER if identity_order else 0)
                 | (0 if graph else L.SWE_FLAG_NO_GRAPH)
                 | (L.SWE_FLAG_TWO_PHASE if two_phase else 0))
        _check(self.lib.swe_dev_create(C.byref(v), C.byref(p), device, flags, C.byref(ctx)),
               "swe_dev_create")
        self.ctx = ctx
        self.n_cells = mesh.n_cells

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.swe_dev_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def set_state(self, s: FieldState, t: float = 0.0, step: int = 0):
        for a in (s.h, s.qx, s.qy):
            assert a.dtype == np.float64 and a.flags.c_contiguous and len(a) == self.n_cells
        _check(self.lib.swe_dev_set_state(self.ctx, L.ptr(s.h), L.ptr(s.qx), L.ptr(s.qy), t, step),
               "swe_dev_set_state")

    def set_state_ptrs(self, h, qx, qy, t=0.0, step=0, device_ptrs=False):
        fn = self.lib.swe_dev_set_state_device if device_ptrs else self.lib.swe_dev_set_state
        _check(fn(self.ctx, h, qx, qy, t, step), "set_state")

    def get_state(self) -> tuple[FieldState, float, int]:
        s = FieldState.zeros(self.n_cells)
        t, step = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_state(self.ctx, L.ptr(s.h), L.ptr(s.qx), L.ptr(s.qy),
                                          C.byref(t), C.byref(step)), "swe_dev_get_state")
        return s, t.value, step.value

    def get_state_ptrs(self, h, qx, qy):
        t, step = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_state(self.ctx, h, qx, qy, C.byref(t), C.byref(step)),
               "swe_dev_get_state")
        return t.value, step.value

    def clock(self):
        t, step = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_state(self.ctx, None, None, None, C.byref(t), C.byref(step)),
               "swe_dev_get_state")
        return t.value, step.value

    def step(self, t_end: float = 1e30) -> L.swe_step_record:
        rec, st = L.swe_step_record(), L.swe_status()
        _status(self.lib.swe_dev_step(self.ctx, t_end, C.byref(rec), C.byref(st)), st, "swe_dev_step")
        return rec

    def advance(self, t_end: float, max_steps: int = 2**62, next_snapshot: float = float("inf"),
                max_records: int = 1 << 16) -> np.ndarray:
        """Steps on the device (one CUDA graph launch); returns the records as
        an array [n, 5] = step, t, dt, max_speed, mass."""
        recs = (L.swe_step_record * max_records)()
        n, st = C.c_longlong(), L.swe_status()
        rc = self.lib.swe_dev_advance(self.ctx, t_end, max_steps, next_snapshot, recs, max_records,
                                      C.byref(n), C.byref(st))
        out = np.array([(r.step, r.t, r.dt, r.max_speed, r.mass) for r in recs[:n.value]],
                       dtype=np.float64).reshape(-1, 5)
        _status(rc, st, "swe_dev_advance")
        return out

    def advance_async(self, t_end: float, max_steps: int = 2**62,
                      next_snapshot: float = float("inf"), max_records: int = 1 << 16):
        """Enqueue the graph-launched advance; collect with records()."""
        _check(self.lib.swe_dev_advance_async(self.ctx, t_end, max_steps, next_snapshot,
                                              max_records), "swe_dev_advance_async")

    def records(self, max_records: int = 1 << 16) -> np.ndarray:
        recs = (L.swe_step_record * max_records)()
        n, st = C.c_longlong(), L.swe_status()
        rc = self.lib.swe_dev_records(self.ctx, recs, max_records, C.byref(n), C.byref(st))
        out = np.array([(r.step, r.t, r.dt, r.max_speed, r.mass)
                        for r in recs[:min(n.value, max_records)]],
                       dtype=np.float64).reshape(-1, 5)
        _status(rc, st, "swe_dev_records")
        return out

    def cell_skip(self) -> np.ndarray:
        """per cell: 1 if its tile is skipped (dry) in the next step"""
        out = np.empty(self.n_cells, np.uint8)
        _check(self.lib.swe_dev_cell_skip(self.ctx, L.ptr(out)), "swe_dev_cell_skip")
        return out

    def advance_n_async(self, n: int, t_end: float = float("inf")):
        _check(self.lib.swe_dev_advance_n_async(self.ctx, n, t_end), "swe_dev_advance_n_async")

    def synchronize(self):
        st = L.swe_status()
        _status(self.lib.swe_dev_synchronize(self.ctx, C.byref(st)), st, "swe_dev_synchronize")

    def compute_fluxes(self):
        E = self.mesh.n_edges
        left, right = np.empty((E, 3)), np.empty((E, 3))
        st = L.swe_status()
        _status(self.lib.swe_dev_compute_fluxes(self.ctx, L.ptr(left), L.ptr(right), C.byref(st)),
                st, "swe_dev_compute_fluxes")
        return left, right

    def total_mass(self) -> float:
        m = C.c_double()
        _check(self.lib.swe_dev_total_mass(self.ctx, C.byref(m)), "swe_dev_total_mass")
        return m.value

    def ledger(self):
        v, e = C.c_double(), C.c_longlong()
        _check(self.lib.swe_dev_get_ledger(self.ctx, C.byref(v), C.byref(e)), "ledger")
        return v.value, e.value

    def set_profiling(self, on: bool):
        _check(self.lib.swe_dev_set_profiling(self.ctx, int(on)), "profiling")

    def kernel_times(self):
        ms = (C.c_double * 4)()
        n = (C.c_longlong * 4)()
        _check(self.lib.swe_dev_kernel_times(self.ctx, ms, n, 4), "kernel_times")
        names = ("tile", "cell", "finalize", "cfl") if self.info()["fused"] else \
            ("face", "cell", "finalize", "cfl")
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}

    def info(self) -> dict:
        v = (C.c_longlong * 16)()
        _check(self.lib.swe_dev_info(self.ctx, v, 16), "swe_dev_info")
        keys = ("fused", "tile_cells", "tiles", "max_slots", "halo_edges", "grid_tile",
                "grid_face", "grid_cell", "tile_smem_bytes", "edges", "dry_skip",
                "skipped_tiles", "graph_unroll", "persistent", "grid_run", "held_tiles")
        return dict(zip(keys, list(v)))

    @property
    def stream(self) -> int:
        return self.lib.swe_dev_stream(self.ctx) or 0

    def memory_bytes(self) -> int:
        return self.lib.swe_dev_memory_bytes(self.ctx)


def point_eval(kind: int, l, r=None, z=None, nrm=None, params: PhysParams = PhysParams()):
    """Device point physics (swe_dev_point_eval): 0 hllc, 1 wall, 2 edge, 3 friction, 4 pow43,
    5 physical_flux_normal, 6 wave_speed_estimates, 7 hydrostatic_reconstruct,
    8 cell_signal_speed, 9 clamp_dry (kernels.hpp:15-216)."""
    l = np.ascontiguousarray(l, dtype=np.float64).reshape(-1, 3)
    n = len(l)
    width = {2: 6, 4: 1, 7: 12, 8: 1, 9: 5}.get(kind, 3)
    out = np.empty((n, width))
    cv = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
    r, z, nrm = cv(r), cv(z), cv(nrm)
    p = params.c()
    _check(L.load().swe_dev_point_eval(kind, n, C.byref(p), L.ptr(l), L.ptr(r), L.ptr(z),
                                       L.ptr(nrm), L.ptr(out)), "swe_dev_point_eval")
    return out if width > 1 else out[:, 0]


def stable_dt(h, qx, qy, inradius, params: PhysParams = PhysParams(), device: int = 0) -> float:
    """kernels.hpp:174-186 on the device (swe_dev_stable_dt)."""
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (h, qx, qy, inradius)]
    dt, bad = C.c_double(), C.c_longlong()
    p = params.c()
    rc = L.load().swe_dev_stable_dt(device, len(a[0]), C.byref(p), *[L.ptr(x) for x in a],
                                    C.byref(dt), C.byref(bad))
    if rc == L.SWE_NONFINITE_SPEED:
        raise NumericError(f"stable_dt: non-finite velocity in cell {bad.value}")
    _check(rc, "swe_dev_stable_dt")
    return dt.value


def mass(h, area, device: int = 0) -> float:
    """total_mass of host arrays on the device (swe_dev_mass, stateless)."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    area = np.ascontiguousarray(area, dtype=np.float64)
    out = C.c_double()
    _check(L.load().swe_dev_mass(device, len(h), L.ptr(h), L.ptr(area), C.byref(out)),
           "swe_dev_mass")
    return out.value


def launch_count() -> int:
    return L.load().swe_dev_launch_count()

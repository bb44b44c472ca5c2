// swe/engine.hpp -- the drop-in time loop (reference: /root/reference/proj/
// include/swe/engine.hpp:24-394), executed on a B200 through the C-ABI of
// swe_dev.h.  Same types, signatures, exception types and message texts as
// the reference, so callers (the reference's cases.hpp, bench.hpp, CLI and
// tests) compile and behave unchanged; there is no CPU path -- every step runs
// the CUDA kernels, and a missing/failed device raises swe::device_error.
//
// Device residency: the mesh is uploaded (and renumbered on the device) once
// per Mesh object and cached; advance_step() keeps the reference's
// host-resident Simulation contract (state up, one step, state down), while
// run() keeps the state on the device for the whole loop and only downloads at
// snapshots and at the end (the paper's transfer-minimisation rule).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "swe/core.hpp"
#include "swe/kernels.hpp"
#include "swe/mesh.hpp"
#include "swe_dev.h"

namespace swe {

/// The caller's process group for one-process-per-GPU runs (MPI,
/// torch.distributed, threads): rank / size and an allgather of byte blobs
/// (every rank's blob, in rank order).  barrier is optional (lockstep
/// debugging of ranks that share a device).
struct Comm {
  int rank = 0;
  int size = 1;
  std::function<std::vector<std::string>(const std::string&)> allgather;
  std::function<void()> barrier;
};

/// Reference plugin point (engine.hpp:24-31).  The B200 engine always runs
/// on the device; `device` selects the CUDA ordinal.  kind/threads are
/// accepted for source compatibility and do not change results (the
/// reference's backends are bitwise identical too).  Multi-GPU
/// (swe/multigpu.hpp): gpus > 1 drives that many devices from this process
/// (devices lists them; default device, device+1, ...), or comm makes this
/// process one rank of a one-process-per-GPU run.  lockstep steps the parts
/// phase by phase (parts sharing one device; debugging).
struct BackendSpec {
  enum class Kind { sequential, parallel };
  Kind kind = Kind::sequential;
  int threads = 1;
  bool deterministic = true;
  int device = 0;
  int gpus = 1;
  std::vector<int> devices;
  const Comm* comm = nullptr;
  bool lockstep = false;

  bool is_parallel() const { return kind == Kind::parallel && threads > 1; }
};

struct Simulation;
struct RunStats;
struct RunOptions;
namespace detail {
inline RunStats run_multi(Simulation& sim, const Mesh& mesh, const PhysParams& p,
                   const BackendSpec& backend, const RunOptions& opt);
}  // namespace detail

struct FieldState {
  std::vector<double> h, qx, qy;
  void resize(int n) {
    h.assign(n, 0.0);
    qx.assign(n, 0.0);
    qy.assign(n, 0.0);
  }
  int size() const { return static_cast<int>(h.size()); }
  ConservedState cell(int i) const { return {h[i], qx[i], qy[i]}; }
  void set_cell(int i, const ConservedState& u) {
    h[i] = u.h;
    qx[i] = u.qx;
    qy[i] = u.qy;
  }
};

struct EdgeFluxes {
  std::vector<Flux3> left, right;
  void resize(int n) {
    left.assign(n, {});
    right.assign(n, {});
  }
};

struct MassLedger {
  double initial_volume = 0.0;
  double clipped_volume = 0.0;
  long clip_events = 0;
};

struct Simulation {
  FieldState current, next;
  double t = 0.0;
  long step = 0;
  MassLedger ledger;
};

struct StepStats {
  long step = 0;
  double t = 0.0;
  double dt = 0.0;
  double max_speed = 0.0;
  double mass = 0.0;
  double wall_flux_ms = 0.0;
  double wall_update_ms = 0.0;
};

struct RunStats {
  long steps = 0;
  double t_final = 0.0;
  double mass_initial = 0.0;
  double mass_final = 0.0;
  double mass_drift_rel = 0.0;
  double min_dt = 0.0;
  double mean_dt = 0.0;
  long clip_events = 0;
  double clipped_volume = 0.0;
  double wall_flux_s = 0.0;
  double wall_update_s = 0.0;
  double wall_total_s = 0.0;
  std::vector<StepStats> series;
};

struct RunOptions {
  double t_end = 0.0;
  double snapshot_interval = 0.0;
  long max_steps = 100'000'000;
  bool record_series = true;
  bool per_step_timing = false;
  std::function<void(const FieldState&, double t, long step)> on_snapshot;
};

namespace detail {

/// Device context of one Mesh (uploaded + renumbered once).
class DeviceMesh {
 public:
  DeviceMesh(const Mesh& m, const PhysParams& p, int device) : device_(device), params_(p) {
    const int C = m.n_cells(), E = m.n_edges();
    std::vector<double> cx(C), cy(C), nx(E), ny(E);
    std::vector<int> ce(3 * static_cast<size_t>(C)), cs(3 * static_cast<size_t>(C));
    for (int c = 0; c < C; ++c) {
      cx[c] = m.cell_centroid[c].x;
      cy[c] = m.cell_centroid[c].y;
      for (int k = 0; k < 3; ++k) {
        ce[3 * static_cast<size_t>(c) + k] = m.cell_edges[c][k].edge;
        cs[3 * static_cast<size_t>(c) + k] = m.cell_edges[c][k].sign;
      }
    }
    for (int e = 0; e < E; ++e) {
      nx[e] = m.edge_normal[e].x;
      ny[e] = m.edge_normal[e].y;
    }
    swe_mesh_view v{};
    v.n_cells = C;
    v.n_edges = E;
    v.area = m.cell_area.data();
    v.inradius = m.cell_inradius.data();
    v.bed = m.cell_bed.data();
    v.manning = m.cell_manning.data();
    v.cx = cx.data();
    v.cy = cy.data();
    v.cell_edge = ce.data();
    v.cell_sign = cs.data();
    v.edge_left = m.edge_left.data();
    v.edge_right = m.edge_right.data();
    v.nx = nx.data();
    v.ny = ny.data();
    v.len = m.edge_length.data();
    const swe_params sp = to_c(p);
    check(swe_dev_create(&v, &sp, device, 0, &ctx_), "swe_dev_create");
    digest_ = digest(m);
  }
  ~DeviceMesh() { swe_dev_destroy(ctx_); }
  DeviceMesh(const DeviceMesh&) = delete;
  DeviceMesh& operator=(const DeviceMesh&) = delete;

  swe_dev_ctx* ctx() const { return ctx_; }
  /// The cached context serves `m` only if every array it uploaded still holds
  /// the same bytes: a Mesh mutated in place, or a new Mesh whose vectors reuse
  /// freed addresses, is re-uploaded (a content digest, not the addresses).
  bool matches(const Mesh& m, const PhysParams& p, int device) const {
    return device == device_ && same(p, params_) && digest(m) == digest_;
  }

  /// 64-bit content digest of the arrays the device copy is built from
  /// (geometry, bed, Manning, connectivity), hashed by all host threads.
  static uint64_t digest(const Mesh& m) {
    struct Span {
      const unsigned char* p;
      size_t n;
    };
    auto sp = [](const auto& v) {
      return Span{reinterpret_cast<const unsigned char*>(v.data()),
                  v.size() * sizeof(typename std::decay_t<decltype(v)>::value_type)};
    };
    const Span arrays[] = {sp(m.cell_area),  sp(m.cell_inradius), sp(m.cell_bed),
                           sp(m.cell_manning), sp(m.cell_centroid), sp(m.cell_edges),
                           sp(m.edge_left),  sp(m.edge_right),    sp(m.edge_normal),
                           sp(m.edge_length)};
    constexpr size_t kChunk = size_t(1) << 22;  // 4 MiB per task
    std::vector<std::pair<int, size_t>> tasks;  // (array, chunk start)
    for (int a = 0; a < 10; ++a) {
      size_t o = 0;
      do {
        tasks.push_back({a, o});
        o += kChunk;
      } while (o < arrays[a].n);
    }
    std::vector<uint64_t> out(tasks.size());
    auto hash_chunk = [&](size_t i) {
      const Span& s = arrays[tasks[i].first];
      const size_t o = tasks[i].second, n = std::min(kChunk, s.n - o);
      uint64_t h[4] = {0x9e3779b97f4a7c15ULL, 0xc2b2ae3d27d4eb4fULL, 0x165667b19e3779f9ULL,
                       0x27d4eb2f165667c5ULL};
      size_t k = 0;
      for (; k + 32 <= n; k += 32)
        for (int j = 0; j < 4; ++j) {
          uint64_t w;
          std::memcpy(&w, s.p + o + k + 8 * j, 8);
          h[j] = (h[j] ^ w) * 0x100000001b3ULL;
          h[j] ^= h[j] >> 29;
        }
      uint64_t r = (h[0] ^ (h[1] << 1)) ^ ((h[2] << 2) ^ (h[3] << 3)) ^ (n * 0x9e3779b97f4a7c15ULL);
      for (; k < n; ++k) r = (r ^ s.p[o + k]) * 0x100000001b3ULL;
      out[i] = r ^ (uint64_t(tasks[i].first) << 56);
    };
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                        static_cast<unsigned>(tasks.size())));
    if (nt <= 1) {
      for (size_t i = 0; i < tasks.size(); ++i) hash_chunk(i);
    } else {
      std::vector<std::thread> pool;
      for (unsigned t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
          for (size_t i = t; i < tasks.size(); i += nt) hash_chunk(i);
        });
      for (auto& th : pool) th.join();
    }
    uint64_t d = 0xcbf29ce484222325ULL ^ (uint64_t(m.n_cells()) << 32) ^ uint64_t(m.n_edges());
    for (uint64_t v : out) d = (d ^ v) * 0x100000001b3ULL;
    return d;
  }

  int busy = 0;  // run() calls holding this context

  static swe_params to_c(const PhysParams& p) { return {p.g, p.h_dry, p.cfl, p.dt_max, p.h_ref}; }

  static void check(int rc, const char* what) {
    if (rc == SWE_OK) return;
    throw device_error(std::string(what) + ": " + swe_dev_strerror(rc) + " (" +
                       swe_dev_last_error() + ")");
  }

 private:
  static bool same(const PhysParams& a, const PhysParams& b) {
    return a.g == b.g && a.h_dry == b.h_dry && a.cfl == b.cfl && a.dt_max == b.dt_max &&
           a.h_ref == b.h_ref;
  }
  swe_dev_ctx* ctx_ = nullptr;
  int device_;
  PhysParams params_;
  uint64_t digest_ = 0;
};

inline std::map<const Mesh*, std::shared_ptr<DeviceMesh>>& device_cache() {
  static std::map<const Mesh*, std::shared_ptr<DeviceMesh>> cache;
  return cache;
}

/// Process-wide cache: one device context per (Mesh, params, device).  A
/// context a running run() holds is never replaced or re-uploaded: a call
/// made meanwhile (e.g. from on_snapshot) gets a context of its own, so it
/// cannot disturb the run's state, clock or geometry.
inline std::shared_ptr<DeviceMesh> device_mesh(const Mesh& m, const PhysParams& p, int device) {
  auto& slot = device_cache()[&m];
  if (slot && slot->busy > 0) {
    return std::make_shared<DeviceMesh>(m, p, device);  // never share a running context
  }
  if (!slot || !slot->matches(m, p, device)) {
    slot.reset();
    slot = std::make_shared<DeviceMesh>(m, p, device);
  }
  return slot;
}

inline void upload(DeviceMesh& dm, const FieldState& s, double t, long step) {
  DeviceMesh::check(swe_dev_set_state(dm.ctx(), s.h.data(), s.qx.data(), s.qy.data(), t, step),
                    "swe_dev_set_state");
}

inline void download(DeviceMesh& dm, FieldState& s) {
  double t;
  long long step;
  DeviceMesh::check(swe_dev_get_state(dm.ctx(), s.h.data(), s.qx.data(), s.qy.data(), &t, &step),
                    "swe_dev_get_state");
}

// reference message templates (std::to_string formatting, engine.hpp:169,
// :206, :294-296)
[[noreturn]] inline void raise(const swe_status& st, const FieldState* next) {
  (void)next;
  switch (st.code) {
    case SWE_NONFINITE_SPEED:
      throw numeric_error("stable_dt: non-finite velocity in cell " + std::to_string(st.index));
    case SWE_NEGATIVE_DEPTH:
      throw numeric_error("compute_fluxes: negative depth at edge " + std::to_string(st.index));
    case SWE_BLOWUP:
      throw numeric_error("advance_step: numeric blowup at step " + std::to_string(st.step) +
                          ", cell " + std::to_string(st.index) + ", dt " + std::to_string(st.dt) +
                          " (h=" + std::to_string(st.h) + ")");
    default:
      throw device_error(std::string("device step failed: ") + swe_dev_strerror(st.code) + " (" +
                         swe_dev_last_error() + ")");
  }
}

}  // namespace detail

/// Drops the device copy of a mesh (frees its device memory early; a mutated
/// mesh is detected by content and re-uploaded anyway).
inline void release_device_mesh(const Mesh& m) {
  auto it = detail::device_cache().find(&m);
  if (it != detail::device_cache().end() && it->second->busy == 0) detail::device_cache().erase(it);
}

/// Volume integral of the depth (engine.hpp:128-132), reduced on the device
/// in a fixed order (matches the reference's serial sum to round-off).  A
/// pure function as in the reference: it touches no cached context.
inline double total_mass(const FieldState& s, const Mesh& mesh,
                         const PhysParams& p = PhysParams{}, int device = 0) {
  (void)p;
  double m = 0.0;
  detail::DeviceMesh::check(swe_dev_mass(device, static_cast<long long>(mesh.n_cells()),
                                         s.h.data(), mesh.cell_area.data(), &m),
                            "swe_dev_mass");
  return m;
}

/// One flux evaluation per edge (engine.hpp:138-170), on the device.
inline void compute_fluxes(const FieldState& s, const Mesh& mesh, const PhysParams& p,
                           const BackendSpec& backend, EdgeFluxes& out) {
  const auto hold = detail::device_mesh(mesh, p, backend.device);
  auto& dm = *hold;
  detail::upload(dm, s, 0.0, 0);
  if (static_cast<int>(out.left.size()) != mesh.n_edges()) out.resize(mesh.n_edges());
  swe_status st{};
  const int rc = swe_dev_compute_fluxes(dm.ctx(), reinterpret_cast<double*>(out.left.data()),
                                        reinterpret_cast<double*>(out.right.data()), &st);
  if (rc != SWE_OK) detail::raise(st, nullptr);
}

/// One explicit Euler step truncated to land on t_end (engine.hpp:226-319).
/// Host-resident contract: sim.current is uploaded, stepped on the device and
/// the result swapped back in.  `fluxes` is not filled (the edge records stay
/// on the device); use compute_fluxes() to inspect them.
inline StepStats advance_step(Simulation& sim, const Mesh& mesh, const PhysParams& p,
                              const BackendSpec& backend, double t_end, EdgeFluxes& fluxes,
                              StepStats* timing = nullptr) {
  (void)fluxes;
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  const auto hold = detail::device_mesh(mesh, p, backend.device);
  auto& dm = *hold;
  detail::upload(dm, sim.current, sim.t, sim.step);
  detail::DeviceMesh::check(
      swe_dev_set_ledger(dm.ctx(), sim.ledger.clipped_volume, sim.ledger.clip_events),
      "swe_dev_set_ledger");
  swe_step_record rec{};
  swe_status st{};
  double flux_ms = 0.0, kernel_update_ms = 0.0;
  // with timers: the two-phase kernels, so the flux and update phases are
  // timed apart like the reference's (engine.hpp:314-317); same results
  const int rc = timing ? swe_dev_step_timed(dm.ctx(), t_end, &rec, &st, &flux_ms, &kernel_update_ms)
                        : swe_dev_step(dm.ctx(), t_end, &rec, &st);
  if (rc != SWE_OK) detail::raise(st, nullptr);
  if (static_cast<int>(sim.next.h.size()) != mesh.n_cells()) sim.next.resize(mesh.n_cells());
  detail::download(dm, sim.next);
  long long events = 0;
  detail::DeviceMesh::check(swe_dev_get_ledger(dm.ctx(), &sim.ledger.clipped_volume, &events),
                            "swe_dev_get_ledger");
  sim.ledger.clip_events = static_cast<long>(events);
  std::swap(sim.current, sim.next);
  sim.t = rec.t;
  sim.step = static_cast<long>(rec.step);
  StepStats out;
  out.step = sim.step;
  out.t = sim.t;
  out.dt = rec.dt;
  out.max_speed = rec.max_speed;
  if (timing) {
    // flux: the face kernel (device time); update: the rest of the call --
    // the cell kernel, the step commit and the host<->device state copies
    timing->wall_flux_ms = flux_ms;
    timing->wall_update_ms =
        std::chrono::duration<double, std::milli>(clock::now() - t0).count() - flux_ms;
  }
  return out;
}

/// build_mesh (mesh.hpp:121-240) computed on the GPU: the same Mesh, bit for
/// bit, and the same mesh_error texts as the host build_mesh (SURVEY §8(f)
/// row 3: the host version is a serial bucket walk, ~12 s at 10M cells).
inline Mesh build_mesh_device(const RawMesh& raw, std::vector<double> bathymetry,
                              std::vector<double> manning, int device = 0) {
  const int nn = static_cast<int>(raw.nodes.size());
  const int nc = static_cast<int>(raw.triangles.size());
  if (static_cast<int>(bathymetry.size()) != nc || static_cast<int>(manning.size()) != nc)
    throw mesh_error("build_mesh: bathymetry/manning arrays must have one entry per triangle (got " +
                     std::to_string(bathymetry.size()) + "/" + std::to_string(manning.size()) +
                     " for " + std::to_string(nc) + " triangles)");
  for (int c = 0; c < nc; ++c)
    if (manning[c] < 0.0)
      throw mesh_error("build_mesh: negative Manning coefficient at cell " + std::to_string(c));
  static_assert(sizeof(Vec2) == 2 * sizeof(double) && sizeof(std::array<int, 3>) == 3 * sizeof(int),
                "contiguous node / triangle arrays");
  swe_built_mesh* b = nullptr;
  char err[512] = {0};
  const int rc = swe_dev_build_mesh(device, nn, reinterpret_cast<const double*>(raw.nodes.data()), nc,
                                    reinterpret_cast<const int*>(raw.triangles.data()), &b, err,
                                    sizeof(err));
  if (rc == SWE_INVALID) throw mesh_error(err);
  if (rc != SWE_OK) throw device_error(std::string("build_mesh_device: ") + swe_dev_last_error());
  struct Guard {
    swe_built_mesh* b;
    ~Guard() { swe_dev_built_free(b); }
  } guard{b};
  int ne = 0;
  swe_dev_built_sizes(b, nullptr, nullptr, &ne);
  Mesh m;
  m.nodes = raw.nodes;
  m.cell_nodes.resize(nc);
  m.cell_area.resize(nc);
  m.cell_centroid.resize(nc);
  m.cell_inradius.resize(nc);
  m.cell_bed = std::move(bathymetry);
  m.cell_manning = std::move(manning);
  m.cell_edges.resize(nc);
  m.edge_nodes.resize(ne);
  m.edge_left.resize(ne);
  m.edge_right.resize(ne);
  m.edge_normal.resize(ne);
  m.edge_length.resize(ne);
  std::vector<double> cx(nc), cy(nc), nx(ne), ny(ne);
  std::vector<int> ce(3 * (size_t)nc), cs(3 * (size_t)nc);
  if (swe_dev_built_export(b, reinterpret_cast<int*>(m.cell_nodes.data()), m.cell_area.data(),
                           cx.data(), cy.data(), m.cell_inradius.data(), ce.data(), cs.data(),
                           reinterpret_cast<int*>(m.edge_nodes.data()), m.edge_left.data(),
                           m.edge_right.data(), nx.data(), ny.data(), m.edge_length.data()) != SWE_OK)
    throw device_error(std::string("build_mesh_device: ") + swe_dev_last_error());
  for (int c = 0; c < nc; ++c) {
    m.cell_centroid[c] = {cx[c], cy[c]};
    for (int k = 0; k < 3; ++k) m.cell_edges[c][k] = {ce[3 * (size_t)c + k], cs[3 * (size_t)c + k]};
  }
  for (int e = 0; e < ne; ++e) m.edge_normal[e] = {nx[e], ny[e]};
  return m;
}

/// The time loop (engine.hpp:335-394) with the state resident on the device.
inline RunStats run(Simulation& sim, const Mesh& mesh, const PhysParams& p,
                    const BackendSpec& backend, const RunOptions& opt) {
  using clock = std::chrono::steady_clock;
  if (!(opt.t_end > 0.0)) throw config_error("run: t_end must be > 0");
  if (backend.gpus > 1 || backend.comm) return detail::run_multi(sim, mesh, p, backend, opt);
  const auto hold = detail::device_mesh(mesh, p, backend.device);
  auto& dm = *hold;
  swe_dev_ctx* ctx = dm.ctx();
  struct Busy {  // the cache keeps this context out of other calls' reach
    detail::DeviceMesh& d;
    explicit Busy(detail::DeviceMesh& x) : d(x) { ++d.busy; }
    ~Busy() { --d.busy; }
  } busy(dm);

  RunStats rs;
  detail::upload(dm, sim.current, sim.t, sim.step);
  detail::DeviceMesh::check(swe_dev_total_mass(ctx, &rs.mass_initial), "swe_dev_total_mass");
  sim.ledger.initial_volume = rs.mass_initial;
  detail::DeviceMesh::check(
      swe_dev_set_ledger(ctx, sim.ledger.clipped_volume, sim.ledger.clip_events),
      "swe_dev_set_ledger");

  if (opt.on_snapshot) opt.on_snapshot(sim.current, sim.t, sim.step);
  double next_snapshot = opt.snapshot_interval > 0.0 ? sim.t + opt.snapshot_interval
                                                     : std::numeric_limits<double>::infinity();
  rs.min_dt = std::numeric_limits<double>::infinity();
  double dt_sum = 0.0;
  const auto run_start = clock::now();
  std::vector<swe_step_record> recs(1 << 16);
  if (static_cast<int>(sim.next.h.size()) != mesh.n_cells()) sim.next.resize(mesh.n_cells());

  // Segments of the loop run on the device (one graph launch each, ending at
  // t_end, a snapshot time or a full record buffer).  A snapshot is permuted
  // into a device slot and copied (copy stream) straight into sim.current --
  // page-locked for the run -- while the NEXT segment already runs;
  // on_snapshot is called when the copy has landed, so the device does not
  // wait for the host's I/O.
  const size_t C = static_cast<size_t>(mesh.n_cells());
  struct Locked {  // cudaHostRegister of the state vectors for the run
    std::vector<void*> ps;
    ~Locked() {
      for (void* p : ps) swe_dev_host_unregister(p);
    }
  } locked;
  bool async_snapshots = opt.on_snapshot && std::getenv("SWE_SYNC_SNAPSHOTS") == nullptr;
  if (async_snapshots) {
    for (double* p : {sim.current.h.data(), sim.current.qx.data(), sim.current.qy.data()}) {
      if (swe_dev_host_register(p, static_cast<long long>(C * sizeof(double))) != SWE_OK) {
        async_snapshots = false;  // not lockable: synchronous snapshots
        break;
      }
      locked.ps.push_back(p);
    }
  }
  auto launch = [&] {
    const double snap = opt.on_snapshot ? next_snapshot : std::numeric_limits<double>::infinity();
    detail::DeviceMesh::check(swe_dev_advance_async(ctx, opt.t_end, opt.max_steps, snap,
                                                    static_cast<long long>(recs.size())),
                              "swe_dev_advance_async");
  };
  bool running = sim.t < opt.t_end;
  if (running) {
    if (sim.step >= opt.max_steps)
      throw numeric_error("run: exceeded max_steps=" + std::to_string(opt.max_steps) +
                          " before reaching t_end (t=" + std::to_string(sim.t) + ")");
    launch();
  }
  while (running) {
    long long n = 0;
    swe_status st{};
    const auto b0 = clock::now();
    const int rc = swe_dev_records(ctx, recs.data(), static_cast<long long>(recs.size()), &n, &st);
    rs.wall_update_s += std::chrono::duration<double>(clock::now() - b0).count();
    for (long long i = 0; i < n; ++i) {
      const swe_step_record& r = recs[static_cast<size_t>(i)];
      rs.min_dt = std::min(rs.min_dt, r.dt);
      dt_sum += r.dt;
      if (opt.record_series) {
        StepStats s;
        s.step = static_cast<long>(r.step);
        s.t = r.t;
        s.dt = r.dt;
        s.max_speed = r.max_speed;
        s.mass = r.mass;
        rs.series.push_back(s);
      }
    }
    double t;
    long long step;
    detail::DeviceMesh::check(swe_dev_get_state(ctx, nullptr, nullptr, nullptr, &t, &step),
                              "swe_dev_get_state");
    sim.t = t;
    sim.step = static_cast<long>(step);
    if (rc != SWE_OK) {
      detail::download(dm, sim.current);
      detail::raise(st, nullptr);
    }
    bool due = opt.on_snapshot && n > 0 && (sim.t >= opt.t_end || sim.t >= next_snapshot - 1e-12);
    if (due) {
      if (!async_snapshots) {
        detail::download(dm, sim.current);
        opt.on_snapshot(sim.current, sim.t, sim.step);
        due = false;
      } else {
        detail::DeviceMesh::check(
            swe_dev_snapshot_async(ctx, 0, sim.current.h.data(), sim.current.qx.data(),
                                   sim.current.qy.data()),
            "swe_dev_snapshot_async");
      }
      if (opt.snapshot_interval > 0.0)
        while (next_snapshot <= sim.t) next_snapshot += opt.snapshot_interval;
    }
    running = sim.t < opt.t_end;
    const bool over = running && sim.step >= opt.max_steps;
    if (running && !over) launch();  // the device steps on while the snapshot lands
    if (due) {
      detail::DeviceMesh::check(swe_dev_snapshot_wait(ctx, 0), "swe_dev_snapshot_wait");
      opt.on_snapshot(sim.current, sim.t, sim.step);
    }
    if (over)
      throw numeric_error("run: exceeded max_steps=" + std::to_string(opt.max_steps) +
                          " before reaching t_end (t=" + std::to_string(sim.t) + ")");
  }
  detail::download(dm, sim.current);
  long long events = 0;
  detail::DeviceMesh::check(swe_dev_get_ledger(ctx, &sim.ledger.clipped_volume, &events),
                            "swe_dev_get_ledger");
  sim.ledger.clip_events = static_cast<long>(events);

  rs.steps = sim.step;
  rs.t_final = sim.t;
  rs.mass_final = rs.series.empty() ? 0.0 : rs.series.back().mass;
  if (rs.series.empty()) detail::DeviceMesh::check(swe_dev_total_mass(ctx, &rs.mass_final), "mass");
  rs.mass_drift_rel = rs.mass_initial != 0.0 ? (rs.mass_final - rs.mass_initial) / rs.mass_initial
                                             : rs.mass_final;
  rs.mean_dt = rs.steps > 0 ? dt_sum / rs.steps : 0.0;
  if (!std::isfinite(rs.min_dt)) rs.min_dt = 0.0;
  rs.clip_events = sim.ledger.clip_events;
  rs.clipped_volume = sim.ledger.clipped_volume;
  rs.wall_total_s = std::chrono::duration<double>(clock::now() - run_start).count();
  return rs;
}

}  // namespace swe

#include "swe/multigpu.hpp"  // run()'s multi-GPU path (backend.gpus / backend.comm)

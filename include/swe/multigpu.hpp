// swe/multigpu.hpp -- the multi-GPU path behind the drop-in C++ API (SURVEY.md
// §8(e); the reference is single-node shared memory only, SPEC.md lists
// distributed memory as a non-goal, so this extends BackendSpec).
//
//   swe::run(sim, mesh, params, backend, opt) with
//     backend.gpus = N            one process drives N devices (backend.devices,
//                                 default device .. device+N-1), one linked
//                                 part per device;
//     backend.comm = &comm        one process per GPU (MPI / torch.distributed
//                                 style): every rank calls run() with the same
//                                 arguments; comm.allgather exchanges the CUDA
//                                 IPC handles and the halo plans once, and the
//                                 owned states at snapshots and at the end.
//
// Decomposition: recursive coordinate bisection (partition.hpp), cost
// weighted by the initial wet/dry pattern; every part holds its owned cells,
// a one-cell ghost layer and every edge touching an owned cell in the global
// orientation, so the run is bit-identical to one device (state, dt and
// max-speed series; the mass is a rank-ordered sum, equal to 1e-12).  The
// linked contexts push halo cells peer-to-peer from the step kernel and
// agree on dt through device mailboxes (include/swe_dev.h swe_dev_link): no
// host round trip per step.
//
// Rank-local setup (build_rank_mesh): a rank that holds only the RawMesh and
// the case fields materialises its own part -- owned triangles plus the ghost
// layer, built with build_mesh on that subset in global triangle order --
// never the global Mesh (≈ 30-40 GB of host arrays at 82M cells).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include <unistd.h>

#include "swe/engine.hpp"
#include "swe/partition.hpp"

namespace swe {

// ---------------------------------------------------------------------------
// rank-local decomposition from the raw mesh
// ---------------------------------------------------------------------------

/// RCB over the raw triangles' centroids (cell_centroids); the same
/// deterministic cut on every rank.
inline std::vector<int> rcb_partition(const RawMesh& raw, int nparts,
                                      const std::vector<double>* weights = nullptr) {
  return detail::rcb_partition_centroids(cell_centroids(raw), nparts, weights);
}

/// Part p's LocalMesh built from the raw mesh alone: owned triangles, the
/// triangles sharing an edge with them (ghosts), build_mesh over that subset
/// in global triangle order (so every kept edge has the global orientation,
/// normal and length, bit for bit), then build_local_mesh.  cells are global
/// triangle ids; edges are the SUBSET's edge ids (the global edge numbering
/// needs every triangle's edges; error messages of a rank-local run name
/// cells exactly and edges by their part-local id).
inline LocalMesh build_rank_mesh(const RawMesh& raw, const std::vector<double>& bed,
                                 const std::vector<double>& manning, const std::vector<int>& part,
                                 int p) {
  const int C = static_cast<int>(raw.triangles.size());
  const int NN = static_cast<int>(raw.nodes.size());
  if (static_cast<int>(part.size()) != C || static_cast<int>(bed.size()) != C ||
      static_cast<int>(manning.size()) != C)
    throw config_error("build_rank_mesh: part / bed / manning need one entry per triangle");
  auto key = [](int a, int b) {
    const uint64_t lo = static_cast<uint32_t>(std::min(a, b)), hi = static_cast<uint32_t>(std::max(a, b));
    return (hi << 32) | lo;
  };
  // nodes of owned triangles, then the owned triangles' edges
  std::vector<unsigned char> mark(NN, 0);
  std::unordered_set<uint64_t> owned_edges;
  for (int t = 0; t < C; ++t)
    if (part[t] == p) {
      const auto& tri = raw.triangles[t];
      for (int k = 0; k < 3; ++k) {
        if (tri[k] < 0 || tri[k] >= NN) throw mesh_error("build_rank_mesh: node index out of range");
        mark[tri[k]] = 1;
        owned_edges.insert(key(tri[k], tri[(k + 1) % 3]));
      }
    }
  // ghosts: non-owned triangles sharing an edge (two marked nodes, then the set)
  std::vector<int> sub;  // global triangle ids, ascending
  for (int t = 0; t < C; ++t) {
    const auto& tri = raw.triangles[t];
    if (part[t] == p) {
      sub.push_back(t);
      continue;
    }
    if (mark[tri[0]] + mark[tri[1]] + mark[tri[2]] < 2) continue;
    for (int k = 0; k < 3; ++k)
      if (owned_edges.count(key(tri[k], tri[(k + 1) % 3]))) {
        sub.push_back(t);
        break;
      }
  }
  // the subset as a RawMesh with compacted (order-preserving) node ids
  std::vector<int> node_new(NN, -1);
  RawMesh sr;
  for (int t : sub)
    for (int k = 0; k < 3; ++k) node_new[raw.triangles[t][k]] = 0;
  for (int n = 0; n < NN; ++n)
    if (node_new[n] == 0) {
      node_new[n] = static_cast<int>(sr.nodes.size());
      sr.nodes.push_back(raw.nodes[n]);
    }
  sr.triangles.reserve(sub.size());
  std::vector<double> sb(sub.size()), sm(sub.size());
  std::vector<int> spart(sub.size());
  for (size_t i = 0; i < sub.size(); ++i) {
    const auto& tri = raw.triangles[sub[i]];
    sr.triangles.push_back({node_new[tri[0]], node_new[tri[1]], node_new[tri[2]]});
    sb[i] = bed[sub[i]];
    sm[i] = manning[sub[i]];
    spart[i] = part[sub[i]];
  }
  const Mesh m = build_mesh(sr, std::move(sb), std::move(sm));
  LocalMesh L = build_local_mesh(m, spart, p);
  for (int& c : L.cells) c = sub[c];  // subset id -> global triangle id
  return L;
}

namespace detail {

inline swe_mesh_view local_view(const LocalMesh& L) {
  swe_mesh_view v{};
  v.n_cells = static_cast<int>(L.cells.size());
  v.n_edges = static_cast<int>(L.edges.size());
  v.area = L.area.data();
  v.inradius = L.inradius.data();
  v.bed = L.bed.data();
  v.manning = L.manning.data();
  v.cx = L.cx.data();
  v.cy = L.cy.data();
  v.cell_edge = L.cell_edge.data();
  v.cell_sign = L.cell_sign.data();
  v.edge_left = L.edge_left.data();
  v.edge_right = L.edge_right.data();
  v.nx = L.nx.data();
  v.ny = L.ny.data();
  v.len = L.len.data();
  v.n_owned = L.n_owned;
  return v;
}

/// The halo push plan of part p (dist.py push_plan): for every peer q, p's
/// send list to q (local ids, ascending global id) against q's receive list
/// from p (q's local ghost ids, the same global cells in the same order).
struct PushPlan {
  std::vector<int> cell, rank, ghost;
};

inline PushPlan push_plan(const LocalMesh& L, const std::vector<std::vector<int>>& peers_of,
                          const std::vector<std::vector<std::vector<int>>>& recv_of) {
  PushPlan pp;
  for (size_t i = 0; i < L.peers.size(); ++i) {
    const int q = L.peers[i];
    const auto& qp = peers_of[q];
    const auto it = std::find(qp.begin(), qp.end(), L.part);
    if (it == qp.end()) throw device_error("push_plan: peer " + std::to_string(q) + " lacks part " +
                                           std::to_string(L.part));
    const auto& r = recv_of[q][it - qp.begin()];
    if (r.size() != L.send[i].size())
      throw device_error("push_plan: halo plans of parts " + std::to_string(L.part) + " and " +
                         std::to_string(q) + " disagree");
    for (size_t j = 0; j < r.size(); ++j) {
      pp.cell.push_back(L.send[i][j]);
      pp.rank.push_back(q);
      pp.ghost.push_back(r[j]);
    }
  }
  return pp;
}

// byte blobs for Comm::allgather
struct Blob {
  std::string s;
  template <class T>
  void put(const T& v) {
    s.append(reinterpret_cast<const char*>(&v), sizeof(T));
  }
  template <class T>
  void put_vec(const std::vector<T>& v) {
    put<long long>(static_cast<long long>(v.size()));
    s.append(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
  }
};
struct Reader {
  const std::string& s;
  size_t o = 0;
  template <class T>
  T get() {
    T v;
    std::memcpy(&v, s.data() + o, sizeof(T));
    o += sizeof(T);
    return v;
  }
  template <class T>
  std::vector<T> get_vec() {
    const long long n = get<long long>();
    std::vector<T> v(static_cast<size_t>(n));
    std::memcpy(v.data(), s.data() + o, static_cast<size_t>(n) * sizeof(T));
    o += static_cast<size_t>(n) * sizeof(T);
    return v;
  }
};

/// One linked part: its local mesh and device context.
struct Part {
  LocalMesh L;
  swe_dev_ctx* ctx = nullptr;
  int device = 0;
  ~Part() {
    if (ctx) swe_dev_destroy(ctx);
  }
};

inline void check_rc(int rc, const char* what) { DeviceMesh::check(rc, what); }

/// Global state of the owned cells of every local part.
inline void gather_owned(const std::vector<Part*>& parts, FieldState& out) {
  for (Part* pt : parts) {
    const int n = static_cast<int>(pt->L.cells.size());
    std::vector<double> h(n), qx(n), qy(n);
    double t;
    long long step;
    check_rc(swe_dev_get_state(pt->ctx, h.data(), qx.data(), qy.data(), &t, &step),
             "swe_dev_get_state(part)");
    for (int i = 0; i < pt->L.n_owned; ++i) {
      const int c = pt->L.cells[i];
      out.h[c] = h[i];
      out.qx[c] = qx[i];
      out.qy[c] = qy[i];
    }
  }
}

inline void set_parts_state(const std::vector<Part*>& parts, const FieldState& s, double t,
                            long step) {
  for (Part* pt : parts) {
    const int n = static_cast<int>(pt->L.cells.size());
    std::vector<double> h(n), qx(n), qy(n);
    for (int i = 0; i < n; ++i) {
      const int c = pt->L.cells[i];
      h[i] = s.h[c];
      qx[i] = s.qx[c];
      qy[i] = s.qy[c];
    }
    check_rc(swe_dev_set_state(pt->ctx, h.data(), qx.data(), qy.data(), t, step),
             "swe_dev_set_state(part)");
  }
}

/// One segment of the linked run (engine.hpp:355-380) on every local part;
/// lockstep: phases of one step across the parts (parts sharing a device:
/// no kernel may wait on a concurrently running one), else one launch per
/// part enqueued on every device before any is waited for.  Returns the
/// (identical) records of the segment and the status.
inline int advance_parts(const std::vector<Part*>& parts, const Comm* comm, bool lockstep,
                         double t_end, long max_steps, double next_snap,
                         std::vector<swe_step_record>& recs, swe_status& st) {
  recs.clear();
  if (!lockstep) {
    for (Part* pt : parts)
      check_rc(swe_dev_advance_async(pt->ctx, t_end, max_steps, next_snap, 1 << 16),
               "swe_dev_advance_async(part)");
    std::vector<swe_step_record> buf(1 << 16);
    int rc = SWE_OK;
    for (size_t i = 0; i < parts.size(); ++i) {
      long long n = 0;
      swe_status s{};
      const int r = swe_dev_records(parts[i]->ctx, buf.data(), 1 << 16, &n, &s);
      if (i == 0) {
        recs.assign(buf.begin(), buf.begin() + static_cast<long>(std::min<long long>(n, 1 << 16)));
        rc = r;
        st = s;
      }
    }
    return rc;
  }
  // lockstep: one advance_step-shaped step at a time, stop as run()'s loop does
  double t = 0.0;
  long long step = 0;
  check_rc(swe_dev_get_state(parts[0]->ctx, nullptr, nullptr, nullptr, &t, &step), "clock");
  while (t < t_end && step < max_steps && !(t >= next_snap - 1e-12) &&
         recs.size() < (size_t)(1 << 16)) {
    for (int phase = 0; phase < 5; ++phase) {
      for (Part* pt : parts) check_rc(swe_dev_link_phase(pt->ctx, phase, t_end), "link_phase");
      for (Part* pt : parts) check_rc(swe_dev_synchronize(pt->ctx, nullptr) == SWE_CUDA ? SWE_CUDA : 0,
                                      "synchronize");
      if (comm && comm->barrier) comm->barrier();
    }
    swe_step_record r{};
    swe_status s{};
    const int rc = swe_dev_last_record(parts[0]->ctx, &r, &s);
    if (rc != SWE_OK) {
      st = s;
      return rc;
    }
    recs.push_back(r);
    t = r.t;
    step = r.step;
  }
  st = swe_status{};
  return SWE_OK;
}

inline RunStats run_multi(Simulation& sim, const Mesh& mesh, const PhysParams& p,
                          const BackendSpec& backend, const RunOptions& opt) {
  using clock = std::chrono::steady_clock;
  const Comm* comm = backend.comm;
  const int P = comm ? comm->size : backend.gpus;
  if (P < 1 || P > 64) throw config_error("run: backend.gpus / comm.size must lie in 1..64");
  if (comm && (comm->rank < 0 || comm->rank >= P || !comm->allgather))
    throw config_error("run: backend.comm needs rank in [0, size) and an allgather");
  std::vector<int> devs = backend.devices;
  if (devs.empty())
    for (int k = 0; k < (comm ? 1 : P); ++k) devs.push_back(backend.device + k);
  if (!comm && static_cast<int>(devs.size()) != P)
    throw config_error("run: backend.devices must list one device per GPU part");
  const bool same_device =
      !comm && std::count(devs.begin(), devs.end(), devs[0]) == static_cast<long>(devs.size());
  const bool lockstep = backend.lockstep || (same_device && P > 1);

  // the same cost-weighted RCB on every rank (initial wet/dry pattern)
  const std::vector<double> w = cost_weights(sim.current.h, p.h_dry);
  const std::vector<int> part = rcb_partition(mesh, P, &w);
  std::vector<int> mine;
  if (comm) mine.push_back(comm->rank);
  else
    for (int q = 0; q < P; ++q) mine.push_back(q);
  std::vector<std::unique_ptr<Part>> own;
  std::vector<Part*> parts;
  const swe_params sp = DeviceMesh::to_c(p);
  for (size_t i = 0; i < mine.size(); ++i) {
    auto pt = std::make_unique<Part>();
    pt->L = build_local_mesh(mesh, part, mine[i]);
    pt->device = comm ? devs[0] : devs[i];
    const swe_mesh_view v = local_view(pt->L);
    check_rc(swe_dev_create(&v, &sp, pt->device, 0, &pt->ctx), "swe_dev_create(part)");
    parts.push_back(pt.get());
    own.push_back(std::move(pt));
  }
  // link: arenas by pointer (one process) or CUDA IPC handles (allgather)
  std::vector<std::vector<int>> peers_of(P);
  std::vector<std::vector<std::vector<int>>> recv_of(P);
  std::vector<long long> cells_of(P);
  std::vector<void*> arenas(P, nullptr);
  std::vector<unsigned char> handles(64 * static_cast<size_t>(P), 0);
  if (!comm) {
    for (Part* pt : parts) {
      const int q = pt->L.part;
      check_rc(swe_dev_link_export(pt->ctx, &arenas[q], nullptr), "swe_dev_link_export");
      peers_of[q] = pt->L.peers;
      recv_of[q] = pt->L.recv;
      cells_of[q] = static_cast<long long>(pt->L.cells.size());
    }
  } else {
    Part* pt = parts[0];
    unsigned char h[64];
    void* arena = nullptr;
    check_rc(swe_dev_link_export(pt->ctx, &arena, h), "swe_dev_link_export");
    Blob b;
    b.put<int>(comm->rank);
    b.put<long long>(static_cast<long long>(getpid()));  // same process: pointers, not IPC
    b.put<unsigned long long>(reinterpret_cast<uintptr_t>(arena));
    b.s.append(reinterpret_cast<const char*>(h), 64);
    b.put<long long>(static_cast<long long>(pt->L.cells.size()));
    b.put_vec(pt->L.peers);
    b.put<int>(static_cast<int>(pt->L.recv.size()));
    for (const auto& r : pt->L.recv) b.put_vec(r);
    const std::vector<std::string> all = comm->allgather(b.s);
    if (static_cast<int>(all.size()) != P) throw device_error("run: allgather returned the wrong count");
    for (const std::string& s : all) {
      Reader r{s};
      const int q = r.get<int>();
      const long long pid = r.get<long long>();
      const unsigned long long ptr = r.get<unsigned long long>();
      if (pid == static_cast<long long>(getpid()) && q != comm->rank)
        arenas[q] = reinterpret_cast<void*>(static_cast<uintptr_t>(ptr));
      std::memcpy(handles.data() + 64 * static_cast<size_t>(q), s.data() + r.o, 64);
      r.o += 64;
      cells_of[q] = r.get<long long>();
      peers_of[q] = r.get_vec<int>();
      const int nr = r.get<int>();
      for (int k = 0; k < nr; ++k) recv_of[q].push_back(r.get_vec<int>());
    }
  }
  for (Part* pt : parts) {
    const PushPlan pp = push_plan(pt->L, peers_of, recv_of);
    check_rc(swe_dev_link(pt->ctx, pt->L.part, P, arenas.data(), comm ? handles.data() : nullptr,
                          cells_of.data(),
                          static_cast<int>(pp.cell.size()), pp.cell.data(), pp.rank.data(),
                          pp.ghost.data(), pt->L.cells.data(), pt->L.edges.data(), 120.0),
             "swe_dev_link");
  }

  // every rank (and the single process) sees the whole state at snapshots
  auto gather = [&](FieldState& out) {
    if (static_cast<int>(out.h.size()) != mesh.n_cells()) out.resize(mesh.n_cells());
    gather_owned(parts, out);
    if (!comm) return;
    Part* pt = parts[0];
    Blob b;
    std::vector<double> h, qx, qy;
    for (int i = 0; i < pt->L.n_owned; ++i) {
      const int c = pt->L.cells[i];
      h.push_back(out.h[c]);
      qx.push_back(out.qx[c]);
      qy.push_back(out.qy[c]);
    }
    b.put<int>(comm->rank);
    b.put_vec(h);
    b.put_vec(qx);
    b.put_vec(qy);
    for (const std::string& s : comm->allgather(b.s)) {
      Reader r{s};
      const int q = r.get<int>();
      const auto hh = r.get_vec<double>(), xx = r.get_vec<double>(), yy = r.get_vec<double>();
      size_t i = 0;
      for (int c = 0; c < mesh.n_cells(); ++c)  // owned cells of q in ascending global order
        if (part[c] == q) {
          out.h[c] = hh[i];
          out.qx[c] = xx[i];
          out.qy[c] = yy[i];
          ++i;
        }
    }
  };

  RunStats rs;
  rs.mass_initial = total_mass(sim.current, mesh, p, parts[0]->device);
  sim.ledger.initial_volume = rs.mass_initial;
  set_parts_state(parts, sim.current, sim.t, sim.step);
  for (Part* pt : parts)
    check_rc(swe_dev_set_ledger(pt->ctx, sim.ledger.clipped_volume, sim.ledger.clip_events),
             "swe_dev_set_ledger");
  if (opt.on_snapshot) opt.on_snapshot(sim.current, sim.t, sim.step);
  double next_snapshot = opt.snapshot_interval > 0.0 ? sim.t + opt.snapshot_interval
                                                     : std::numeric_limits<double>::infinity();
  rs.min_dt = std::numeric_limits<double>::infinity();
  double dt_sum = 0.0;
  const auto run_start = clock::now();
  std::vector<swe_step_record> recs;
  while (sim.t < opt.t_end) {
    if (sim.step >= opt.max_steps)
      throw numeric_error("run: exceeded max_steps=" + std::to_string(opt.max_steps) +
                          " before reaching t_end (t=" + std::to_string(sim.t) + ")");
    swe_status st{};
    const double snap = opt.on_snapshot ? next_snapshot : std::numeric_limits<double>::infinity();
    const auto b0 = clock::now();
    const int rc = advance_parts(parts, comm, lockstep, opt.t_end, opt.max_steps, snap, recs, st);
    rs.wall_update_s += std::chrono::duration<double>(clock::now() - b0).count();
    for (const swe_step_record& r : recs) {
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
    check_rc(swe_dev_get_state(parts[0]->ctx, nullptr, nullptr, nullptr, &t, &step), "clock");
    sim.t = t;
    sim.step = static_cast<long>(step);
    if (rc != SWE_OK) {
      gather(sim.current);
      raise(st, nullptr);  // indices of a linked run are global cell / edge ids
    }
    const bool due = opt.on_snapshot && !recs.empty() &&
                     (sim.t >= opt.t_end || sim.t >= next_snapshot - 1e-12);
    if (due) {
      gather(sim.current);
      opt.on_snapshot(sim.current, sim.t, sim.step);
      if (opt.snapshot_interval > 0.0)
        while (next_snapshot <= sim.t) next_snapshot += opt.snapshot_interval;
    }
  }
  gather(sim.current);
  long long events = 0;
  check_rc(swe_dev_get_ledger(parts[0]->ctx, &sim.ledger.clipped_volume, &events), "ledger");
  sim.ledger.clip_events = static_cast<long>(events);
  rs.steps = sim.step;
  rs.t_final = sim.t;
  rs.mass_final = rs.series.empty() ? total_mass(sim.current, mesh, p, parts[0]->device)
                                    : rs.series.back().mass;
  rs.mass_drift_rel = rs.mass_initial != 0.0 ? (rs.mass_final - rs.mass_initial) / rs.mass_initial
                                             : rs.mass_final;
  rs.mean_dt = rs.steps > 0 ? dt_sum / rs.steps : 0.0;
  if (!std::isfinite(rs.min_dt)) rs.min_dt = 0.0;
  rs.clip_events = sim.ledger.clip_events;
  rs.clipped_volume = sim.ledger.clipped_volume;
  rs.wall_total_s = std::chrono::duration<double>(clock::now() - run_start).count();
  return rs;
}

}  // namespace detail
}  // namespace swe

// host_abi.cpp -- extern "C" wrappers of the host-side input producers
// (include/swe/mesh.hpp, include/swe/cases.hpp) declared in swe_host.h.
#include <cstring>
#include <exception>
#include <string>

#include "swe/cases.hpp"
#include "swe/engine.hpp"
#include "swe/partition.hpp"
#include "swe/mesh.hpp"
#include "swe/swemesh.hpp"
#include "swe_host.h"

namespace {

void put(const std::exception& e, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

int kind_of(const std::exception& e) {
  if (dynamic_cast<const swe::numeric_error*>(&e)) return 1;
  if (dynamic_cast<const swe::config_error*>(&e)) return 2;
  if (dynamic_cast<const swe::mesh_error*>(&e)) return 3;
  if (dynamic_cast<const swe::case_error*>(&e)) return 4;
  return 9;
}

swe::CaseSpec spec_from(const char* name, const double* v) {
  swe::CaseSpec c = swe::make_case(swe::case_from_name(name));
  if (v) {
    c.lx = v[0];
    c.ly = v[1];
    c.eta0 = v[2];
    c.amplitude = v[3];
    c.sigma = v[4];
    c.manning = v[5];
    c.h_left = v[6];
    c.h_right = v[7];
    c.x_dam = v[8];
    c.t_end = v[9];
  }
  return c;
}

void copy_fields(const swe::CaseFields& f, double* bed, double* man, double* h, double* qx,
                 double* qy) {
  const size_t n = f.bed.size();
  if (bed) std::memcpy(bed, f.bed.data(), n * sizeof(double));
  if (man) std::memcpy(man, f.manning.data(), n * sizeof(double));
  if (h) std::memcpy(h, f.state.h.data(), n * sizeof(double));
  if (qx) std::memcpy(qx, f.state.qx.data(), n * sizeof(double));
  if (qy) std::memcpy(qy, f.state.qy.data(), n * sizeof(double));
}

}  // namespace

#define EXPORT extern "C" __attribute__((visibility("default")))

EXPORT void* swe_host_raw_square(int nx, int ny, double lx, double ly, char* err, int errlen) {
  try {
    return new swe::RawMesh(swe::generate_square_mesh(nx, ny, lx, ly));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* swe_host_raw_unstructured(int nx, int ny, double lx, double ly, double jitter,
                                       unsigned long long seed, char* err, int errlen) {
  try {
    return new swe::RawMesh(swe::generate_unstructured_mesh(nx, ny, lx, ly, jitter, seed));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* swe_host_raw_arrays(int nn, const double* xy, int nc, const int* tris) {
  auto* r = new swe::RawMesh();
  r->nodes.resize(nn);
  for (int i = 0; i < nn; ++i) r->nodes[i] = {xy[2 * i], xy[2 * i + 1]};
  r->triangles.resize(nc);
  for (int c = 0; c < nc; ++c) r->triangles[c] = {tris[3 * c], tris[3 * c + 1], tris[3 * c + 2]};
  return r;
}

EXPORT void swe_host_raw_sizes(void* p, int* nn, int* nc) {
  const auto& r = *static_cast<swe::RawMesh*>(p);
  *nn = static_cast<int>(r.nodes.size());
  *nc = static_cast<int>(r.triangles.size());
}

EXPORT void swe_host_raw_export(void* p, double* xy, int* tris) {
  const auto& r = *static_cast<swe::RawMesh*>(p);
  for (size_t i = 0; i < r.nodes.size(); ++i) {
    xy[2 * i] = r.nodes[i].x;
    xy[2 * i + 1] = r.nodes[i].y;
  }
  for (size_t c = 0; c < r.triangles.size(); ++c)
    for (int k = 0; k < 3; ++k) tris[3 * c + k] = r.triangles[c][k];
}

EXPORT void swe_host_raw_free(void* p) { delete static_cast<swe::RawMesh*>(p); }

EXPORT int swe_host_case_defaults(const char* name, double* v) {
  try {
    const swe::CaseSpec c = swe::make_case(swe::case_from_name(name));
    const double d[10] = {c.lx, c.ly, c.eta0, c.amplitude, c.sigma,
                          c.manning, c.h_left, c.h_right, c.x_dam, c.t_end};
    std::memcpy(v, d, sizeof(d));
    return 0;
  } catch (const std::exception& e) {
    return kind_of(e);
  }
}

EXPORT int swe_host_init_case(void* raw, const char* name, const double* spec, double* bed,
                              double* man, double* h, double* qx, double* qy, char* err,
                              int errlen) {
  try {
    const swe::CaseFields f = swe::init_case(spec_from(name, spec), *static_cast<swe::RawMesh*>(raw));
    copy_fields(f, bed, man, h, qx, qy);
    return 0;
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return kind_of(e);
  }
}

EXPORT void* swe_host_scenario(const char* name, double scale, int unstructured,
                               unsigned long long seed, int weak_nx, double* t_end, char* err,
                               int errlen) {
  try {
    auto* s = new swe::Scenario(swe::make_scenario(name, scale, unstructured != 0, seed, weak_nx));
    if (t_end) *t_end = s->t_end;
    return s;
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* swe_host_scenario_raw(void* s) { return &static_cast<swe::Scenario*>(s)->raw; }

EXPORT void swe_host_scenario_fields(void* s, double* bed, double* man, double* h, double* qx,
                                     double* qy) {
  copy_fields(static_cast<swe::Scenario*>(s)->fields, bed, man, h, qx, qy);
}

EXPORT void swe_host_scenario_free(void* s) { delete static_cast<swe::Scenario*>(s); }

EXPORT void* swe_host_build_mesh(void* raw, const double* bed, const double* man, char* err,
                                 int errlen) {
  try {
    const auto& r = *static_cast<swe::RawMesh*>(raw);
    const size_t nc = r.triangles.size();
    return new swe::Mesh(swe::build_mesh(r, std::vector<double>(bed, bed + nc),
                                         std::vector<double>(man, man + nc)));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* swe_host_build_mesh_device(void* raw, const double* bed, const double* man, int device,
                                        char* err, int errlen) {
  try {
    const auto& r = *static_cast<swe::RawMesh*>(raw);
    const size_t nc = r.triangles.size();
    return new swe::Mesh(swe::build_mesh_device(r, std::vector<double>(bed, bed + nc),
                                                std::vector<double>(man, man + nc), device));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void swe_host_mesh_sizes(void* p, int* nc, int* ne, int* nb) {
  const auto& m = *static_cast<swe::Mesh*>(p);
  *nc = m.n_cells();
  *ne = m.n_edges();
  *nb = m.n_boundary_edges();
}

EXPORT void swe_host_mesh_export(void* p, int* cell_nodes, double* area, double* cx, double* cy,
                                 double* inradius, int* cell_edge, int* cell_sign, int* edge_nodes,
                                 int* edge_left, int* edge_right, double* nx, double* ny,
                                 double* len) {
  const auto& m = *static_cast<swe::Mesh*>(p);
  const int C = m.n_cells(), E = m.n_edges();
  for (int c = 0; c < C; ++c) {
    for (int k = 0; k < 3; ++k) {
      if (cell_nodes) cell_nodes[3 * c + k] = m.cell_nodes[c][k];
      if (cell_edge) cell_edge[3 * c + k] = m.cell_edges[c][k].edge;
      if (cell_sign) cell_sign[3 * c + k] = m.cell_edges[c][k].sign;
    }
    if (cx) cx[c] = m.cell_centroid[c].x;
    if (cy) cy[c] = m.cell_centroid[c].y;
  }
  if (area) std::memcpy(area, m.cell_area.data(), sizeof(double) * C);
  if (inradius) std::memcpy(inradius, m.cell_inradius.data(), sizeof(double) * C);
  for (int e = 0; e < E; ++e) {
    if (edge_nodes) {
      edge_nodes[2 * e] = m.edge_nodes[e][0];
      edge_nodes[2 * e + 1] = m.edge_nodes[e][1];
    }
    if (nx) nx[e] = m.edge_normal[e].x;
    if (ny) ny[e] = m.edge_normal[e].y;
  }
  if (edge_left) std::memcpy(edge_left, m.edge_left.data(), sizeof(int) * E);
  if (edge_right) std::memcpy(edge_right, m.edge_right.data(), sizeof(int) * E);
  if (len) std::memcpy(len, m.edge_length.data(), sizeof(double) * E);
}

EXPORT void swe_host_mesh_free(void* p) {
  swe::release_device_mesh(*static_cast<swe::Mesh*>(p));
  delete static_cast<swe::Mesh*>(p);
}

// ---- the drop-in engine (include/swe/engine.hpp) behind reference-shaped
// C entry points; signatures mirror oracle/ref_shim.cpp so tests can call
// both sides identically.  Return 0 or an error kind (1 numeric, 2 config,
// 3 mesh, 4 case, 5 device).

namespace {

swe::PhysParams params_from(const double* p) {
  swe::PhysParams pp;
  if (p) {
    pp.g = p[0];
    pp.h_dry = p[1];
    pp.cfl = p[2];
    pp.dt_max = p[3];
    pp.h_ref = p[4];
  }
  return pp;
}

swe::FieldState state_from(int n, const double* h, const double* qx, const double* qy) {
  swe::FieldState s;
  s.h.assign(h, h + n);
  s.qx.assign(qx, qx + n);
  s.qy.assign(qy, qy + n);
  return s;
}

int api_kind(const std::exception& e) {
  if (dynamic_cast<const swe::device_error*>(&e)) return 5;
  return kind_of(e);
}

swe::BackendSpec backend_for(int device) {
  swe::BackendSpec b;
  b.device = device;
  return b;
}

}  // namespace

EXPORT int swe_api_compute_fluxes(void* mp, const double* params, const double* h,
                                  const double* qx, const double* qy, double* left, double* right,
                                  int device, char* err, int errlen) {
  const auto& m = *static_cast<swe::Mesh*>(mp);
  try {
    const swe::FieldState s = state_from(m.n_cells(), h, qx, qy);
    swe::EdgeFluxes f;
    f.resize(m.n_edges());
    swe::compute_fluxes(s, m, params_from(params), backend_for(device), f);
    std::memcpy(left, f.left.data(), sizeof(swe::Flux3) * m.n_edges());
    std::memcpy(right, f.right.data(), sizeof(swe::Flux3) * m.n_edges());
    return 0;
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return api_kind(e);
  }
}

EXPORT int swe_api_total_mass(void* mp, const double* params, const double* h, int device,
                              double* out, char* err, int errlen) {
  const auto& m = *static_cast<swe::Mesh*>(mp);
  try {
    swe::FieldState s;
    s.resize(m.n_cells());
    std::memcpy(s.h.data(), h, sizeof(double) * m.n_cells());
    *out = swe::total_mass(s, m, params_from(params), device);
    return 0;
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return api_kind(e);
  }
}

// repeated swe::advance_step (host-resident Simulation contract)
EXPORT int swe_api_advance(void* mp, const double* params, double* h, double* qx, double* qy,
                           double* t, long* step, double t_end, long nsteps, int stop_at_t_end,
                           int device, double* dts, double* maxspeeds, double* clip_volume,
                           long* clip_events, long* done, char* err, int errlen) {
  const auto& m = *static_cast<swe::Mesh*>(mp);
  const swe::PhysParams p = params_from(params);
  swe::Simulation sim;
  sim.current = state_from(m.n_cells(), h, qx, qy);
  sim.next.resize(m.n_cells());
  sim.t = *t;
  sim.step = *step;
  sim.ledger.clipped_volume = *clip_volume;
  sim.ledger.clip_events = *clip_events;
  swe::EdgeFluxes f;
  long k = 0;
  int rc = 0;
  try {
    for (; k < nsteps; ++k) {
      if (stop_at_t_end && !(sim.t < t_end)) break;
      const swe::StepStats st = swe::advance_step(sim, m, p, backend_for(device), t_end, f);
      if (dts) dts[k] = st.dt;
      if (maxspeeds) maxspeeds[k] = st.max_speed;
    }
  } catch (const std::exception& e) {
    put(e, err, errlen);
    rc = api_kind(e);
  }
  std::memcpy(h, sim.current.h.data(), sizeof(double) * m.n_cells());
  std::memcpy(qx, sim.current.qx.data(), sizeof(double) * m.n_cells());
  std::memcpy(qy, sim.current.qy.data(), sizeof(double) * m.n_cells());
  *t = sim.t;
  *step = sim.step;
  *clip_volume = sim.ledger.clipped_volume;
  *clip_events = sim.ledger.clip_events;
  if (done) *done = k;
  return rc;
}

// swe::run with the series/stats layout of ref_run
EXPORT int swe_api_run(void* mp, const double* params, double* h, double* qx, double* qy,
                       double* t, long* step, double t_end, double snapshot_interval,
                       long max_steps, int device, double* series, long max_rows, long* n_rows,
                       double* stats, double* snaps, long max_snaps, long* n_snaps,
                       double* snap_fields, char* err, int errlen) {
  const auto& m = *static_cast<swe::Mesh*>(mp);
  swe::Simulation sim;
  sim.current = state_from(m.n_cells(), h, qx, qy);
  sim.next.resize(m.n_cells());
  sim.t = *t;
  sim.step = *step;
  swe::RunOptions opt;
  opt.t_end = t_end;
  opt.snapshot_interval = snapshot_interval;
  opt.max_steps = max_steps;
  long ns = 0;
  if (snaps)
    opt.on_snapshot = [&](const swe::FieldState& f, double tt, long) {
      if (ns < max_snaps) {
        snaps[ns] = tt;
        if (snap_fields) {  // [max_snaps][3][C]
          const size_t C = f.h.size();
          std::memcpy(snap_fields + (3 * ns + 0) * C, f.h.data(), C * sizeof(double));
          std::memcpy(snap_fields + (3 * ns + 1) * C, f.qx.data(), C * sizeof(double));
          std::memcpy(snap_fields + (3 * ns + 2) * C, f.qy.data(), C * sizeof(double));
        }
      }
      ++ns;
    };
  int rc = 0;
  try {
    const swe::RunStats rs = swe::run(sim, m, params_from(params), backend_for(device), opt);
    long r = 0;
    for (const swe::StepStats& st : rs.series) {
      if (r >= max_rows) break;
      series[5 * r + 0] = double(st.step);
      series[5 * r + 1] = st.t;
      series[5 * r + 2] = st.dt;
      series[5 * r + 3] = st.max_speed;
      series[5 * r + 4] = st.mass;
      ++r;
    }
    *n_rows = long(rs.series.size());
    stats[0] = double(rs.steps);
    stats[1] = rs.t_final;
    stats[2] = rs.mass_initial;
    stats[3] = rs.mass_final;
    stats[4] = rs.mass_drift_rel;
    stats[5] = rs.min_dt;
    stats[6] = rs.mean_dt;
    stats[7] = double(rs.clip_events);
    stats[8] = rs.clipped_volume;
  } catch (const std::exception& e) {
    put(e, err, errlen);
    rc = api_kind(e);
  }
  if (n_snaps) *n_snaps = ns;
  std::memcpy(h, sim.current.h.data(), sizeof(double) * m.n_cells());
  std::memcpy(qx, sim.current.qx.data(), sizeof(double) * m.n_cells());
  std::memcpy(qy, sim.current.qy.data(), sizeof(double) * m.n_cells());
  *t = sim.t;
  *step = sim.step;
  return rc;
}

// ---- domain decomposition (include/swe/partition.hpp) ----------------------

EXPORT int swe_host_partition(void* mp, int nparts, int* part_out) {
  try {
    const std::vector<int> p = swe::rcb_partition(*static_cast<swe::Mesh*>(mp), nparts);
    std::memcpy(part_out, p.data(), sizeof(int) * p.size());
    return 0;
  } catch (const std::exception& e) {
    return kind_of(e);
  }
}

EXPORT int swe_host_partition_weighted(void* mp, int nparts, const double* weights, int* part_out) {
  try {
    const auto& m = *static_cast<swe::Mesh*>(mp);
    const std::vector<double> w(weights, weights + m.n_cells());
    const std::vector<int> p = swe::rcb_partition(m, nparts, &w);
    std::memcpy(part_out, p.data(), sizeof(int) * p.size());
    return 0;
  } catch (const std::exception& e) {
    return kind_of(e);
  }
}

EXPORT int swe_host_partition_raw(void* rp, int nparts, const double* weights, int* part_out) {
  try {
    const auto& raw = *static_cast<swe::RawMesh*>(rp);
    std::vector<double> w;
    if (weights) w.assign(weights, weights + raw.triangles.size());
    const std::vector<int> p = swe::rcb_partition(raw, nparts, weights ? &w : nullptr);
    std::memcpy(part_out, p.data(), sizeof(int) * p.size());
    return 0;
  } catch (const std::exception& e) {
    return kind_of(e);
  }
}

EXPORT void* swe_host_rank_mesh(void* rp, const double* bed, const double* manning, const int* part,
                                int p, char* err, int errlen) {
  try {
    const auto& raw = *static_cast<swe::RawMesh*>(rp);
    const size_t nc = raw.triangles.size();
    const std::vector<int> pv(part, part + nc);
    const std::vector<double> b(bed, bed + nc), m(manning, manning + nc);
    return new swe::LocalMesh(swe::build_rank_mesh(raw, b, m, pv, p));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* swe_host_local_mesh(void* mp, const int* part, int p, char* err, int errlen) {
  try {
    const auto& m = *static_cast<swe::Mesh*>(mp);
    const std::vector<int> pv(part, part + m.n_cells());
    return new swe::LocalMesh(swe::build_local_mesh(m, pv, p));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void swe_host_local_sizes(void* lp, int* n_cells, int* n_owned, int* n_edges, int* n_peers,
                                 int* n_send, int* n_recv) {
  const auto& L = *static_cast<swe::LocalMesh*>(lp);
  *n_cells = static_cast<int>(L.cells.size());
  *n_owned = L.n_owned;
  *n_edges = static_cast<int>(L.edges.size());
  *n_peers = static_cast<int>(L.peers.size());
  int s = 0, r = 0;
  for (size_t i = 0; i < L.peers.size(); ++i) {
    s += static_cast<int>(L.send[i].size());
    r += static_cast<int>(L.recv[i].size());
  }
  *n_send = s;
  *n_recv = r;
}

EXPORT void swe_host_local_export(void* lp, int* cells, int* edges, double* area, double* inradius,
                                  double* bed, double* manning, double* cx, double* cy,
                                  int* cell_edge, int* cell_sign, int* edge_left, int* edge_right,
                                  double* nx, double* ny, double* len) {
  const auto& L = *static_cast<swe::LocalMesh*>(lp);
  auto cp = [](auto* dst, const auto& v) {
    if (dst) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
  };
  cp(cells, L.cells);
  cp(edges, L.edges);
  cp(area, L.area);
  cp(inradius, L.inradius);
  cp(bed, L.bed);
  cp(manning, L.manning);
  cp(cx, L.cx);
  cp(cy, L.cy);
  cp(cell_edge, L.cell_edge);
  cp(cell_sign, L.cell_sign);
  cp(edge_left, L.edge_left);
  cp(edge_right, L.edge_right);
  cp(nx, L.nx);
  cp(ny, L.ny);
  cp(len, L.len);
}

EXPORT void swe_host_local_plan(void* lp, int* peers, int* send_counts, int* recv_counts,
                                int* send_cells, int* recv_cells) {
  const auto& L = *static_cast<swe::LocalMesh*>(lp);
  int s = 0, r = 0;
  for (size_t i = 0; i < L.peers.size(); ++i) {
    peers[i] = L.peers[i];
    send_counts[i] = static_cast<int>(L.send[i].size());
    recv_counts[i] = static_cast<int>(L.recv[i].size());
    for (int c : L.send[i]) send_cells[s++] = c;
    for (int c : L.recv[i]) recv_cells[r++] = c;
  }
}

EXPORT void swe_host_local_free(void* lp) { delete static_cast<swe::LocalMesh*>(lp); }

// ---- SWEMESH 1 files (swe/swemesh.hpp; reference io.hpp:80-165) ----------
EXPORT void* swe_host_swemesh_read(const char* path, int threads, char* err, int errlen) {
  try {
    return new swe::swemesh::NativeFile(swe::swemesh::read_file(path, threads));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* swe_host_swemesh_parse(const char* text, long long size, int threads, char* err,
                                    int errlen) {
  try {
    return new swe::swemesh::NativeFile(swe::swemesh::parse(text, (size_t)size, threads));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* swe_host_swemesh_raw(void* f) {
  return &static_cast<swe::swemesh::NativeFile*>(f)->raw;
}

EXPORT void swe_host_swemesh_fields(void* f, double* bed, double* manning) {
  const auto& m = *static_cast<swe::swemesh::NativeFile*>(f);
  if (bed) std::memcpy(bed, m.bed.data(), m.bed.size() * sizeof(double));
  if (manning) std::memcpy(manning, m.manning.data(), m.manning.size() * sizeof(double));
}

EXPORT void swe_host_swemesh_free(void* f) { delete static_cast<swe::swemesh::NativeFile*>(f); }

EXPORT int swe_host_swemesh_write(const char* path, void* raw, const double* bed,
                                  const double* manning, int threads, char* err, int errlen) {
  try {
    const auto& r = *static_cast<swe::RawMesh*>(raw);
    const size_t nc = r.triangles.size();
    swe::swemesh::write_file(path, r, std::vector<double>(bed, bed + nc),
                             std::vector<double>(manning, manning + nc), threads);
    return 0;
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return 7;
  }
}

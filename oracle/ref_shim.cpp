// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim around the UNMODIFIED reference headers
// (/root/reference/proj/include/swe/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libswe_ref.so with the reference's own Release flags
// (-O3 -DNDEBUG -fopenmp -ffp-contract=off, proj/CMakeLists.txt:8-18).  It is
// the ground truth the C restatement (swe_oracle.c) and the golden fixtures are
// pinned to, and the CPU baseline timed by `bench.py --impl reference`.
// No reference source is copied: the headers are included in place.
#define swe ref_swe
#include "swe/cases.hpp"
#include "swe/engine.hpp"
#include "swe/kernels.hpp"
#include "swe/mesh.hpp"
#undef swe

#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

using namespace ref_swe;

namespace {

void put_err(const std::exception& e, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

// exception class -> status code (matches swe_dev.h's swe_status codes)
int classify(const std::exception& e) {
  if (dynamic_cast<const numeric_error*>(&e)) return 1;
  if (dynamic_cast<const config_error*>(&e)) return 2;
  if (dynamic_cast<const mesh_error*>(&e)) return 3;
  if (dynamic_cast<const case_error*>(&e)) return 4;
  return 9;
}

PhysParams params_from(const double* p) {
  PhysParams pp;
  if (p) {
    pp.g = p[0];
    pp.h_dry = p[1];
    pp.cfl = p[2];
    pp.dt_max = p[3];
    pp.h_ref = p[4];
  }
  return pp;
}

BackendSpec backend_for(int threads) {
  BackendSpec b;
  if (threads > 1) {
    b.kind = BackendSpec::Kind::parallel;
    b.threads = threads;
  }
  return b;
}

FieldState state_from(int n, const double* h, const double* qx, const double* qy) {
  FieldState s;
  s.h.assign(h, h + n);
  s.qx.assign(qx, qx + n);
  s.qy.assign(qy, qy + n);
  return s;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) void* ref_build_mesh(int nn, const double* xy, int nc,
                                                            const int* tris, const double* bed,
                                                            const double* manning, char* err,
                                                            int errlen) {
  try {
    RawMesh raw;
    raw.nodes.resize(nn);
    for (int i = 0; i < nn; ++i) raw.nodes[i] = {xy[2 * i], xy[2 * i + 1]};
    raw.triangles.resize(nc);
    for (int c = 0; c < nc; ++c) raw.triangles[c] = {tris[3 * c], tris[3 * c + 1], tris[3 * c + 2]};
    return new Mesh(build_mesh(raw, std::vector<double>(bed, bed + nc),
                               std::vector<double>(manning, manning + nc)));
  } catch (const std::exception& e) {
    put_err(e, err, errlen);
    return nullptr;
  }
}

__attribute__((visibility("default"))) void ref_mesh_free(void* m) { delete static_cast<Mesh*>(m); }

__attribute__((visibility("default"))) void ref_mesh_sizes(void* mp, int* nc, int* ne, int* nb) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  *nc = m.n_cells();
  *ne = m.n_edges();
  *nb = m.n_boundary_edges();
}

// any output pointer may be null
__attribute__((visibility("default"))) void ref_mesh_export(
    void* mp, int* cell_nodes, double* area, double* cx, double* cy, double* inradius,
    int* cell_edge, int* cell_sign, int* edge_nodes, int* edge_left, int* edge_right, double* nx,
    double* ny, double* len) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  for (int c = 0; c < m.n_cells(); ++c) {
    for (int k = 0; k < 3; ++k) {
      if (cell_nodes) cell_nodes[3 * c + k] = m.cell_nodes[c][k];
      if (cell_edge) cell_edge[3 * c + k] = m.cell_edges[c][k].edge;
      if (cell_sign) cell_sign[3 * c + k] = m.cell_edges[c][k].sign;
    }
    if (area) area[c] = m.cell_area[c];
    if (cx) cx[c] = m.cell_centroid[c].x;
    if (cy) cy[c] = m.cell_centroid[c].y;
    if (inradius) inradius[c] = m.cell_inradius[c];
  }
  for (int e = 0; e < m.n_edges(); ++e) {
    if (edge_nodes) {
      edge_nodes[2 * e] = m.edge_nodes[e][0];
      edge_nodes[2 * e + 1] = m.edge_nodes[e][1];
    }
    if (edge_left) edge_left[e] = m.edge_left[e];
    if (edge_right) edge_right[e] = m.edge_right[e];
    if (nx) nx[e] = m.edge_normal[e].x;
    if (ny) ny[e] = m.edge_normal[e].y;
    if (len) len[e] = m.edge_length[e];
  }
}

__attribute__((visibility("default"))) int ref_compute_fluxes(void* mp, const double* params,
                                                              const double* h, const double* qx,
                                                              const double* qy, double* left,
                                                              double* right, int threads,
                                                              char* err, int errlen) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  try {
    const FieldState s = state_from(m.n_cells(), h, qx, qy);
    EdgeFluxes f;
    f.resize(m.n_edges());
    compute_fluxes(s, m, params_from(params), backend_for(threads), f);
    std::memcpy(left, f.left.data(), sizeof(Flux3) * m.n_edges());
    std::memcpy(right, f.right.data(), sizeof(Flux3) * m.n_edges());
    return 0;
  } catch (const std::exception& e) {
    put_err(e, err, errlen);
    return classify(e);
  }
}

__attribute__((visibility("default"))) double ref_total_mass(void* mp, const double* h) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  FieldState s;
  s.h.assign(h, h + m.n_cells());
  return total_mass(s, m);
}

// Repeated advance_step (engine.hpp:226).  State is in/out.  When
// stop_at_t_end is set the loop ends once t >= t_end (the reference's own
// `while (sim.t < t_end)` callers, e.g. bench.hpp:130 / acceptance c3).
// Per-step dt and max_speed go to dts/maxspeeds (may be null).  Phase wall
// times are the reference's own StepStats timers (engine.hpp:314-317).
__attribute__((visibility("default"))) int ref_advance(
    void* mp, const double* params, double* h, double* qx, double* qy, double* t, long* step,
    double t_end, long nsteps, int stop_at_t_end, int threads, double* dts, double* maxspeeds,
    double* clip_volume, long* clip_events, double* flux_s, double* update_s, long* done,
    char* err, int errlen) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  const PhysParams p = params_from(params);
  const BackendSpec b = backend_for(threads);
  Simulation sim;
  sim.current = state_from(m.n_cells(), h, qx, qy);
  sim.next.resize(m.n_cells());
  sim.t = *t;
  sim.step = *step;
  sim.ledger.clipped_volume = *clip_volume;
  sim.ledger.clip_events = *clip_events;
  EdgeFluxes f;
  f.resize(m.n_edges());
  long k = 0;
  int rc = 0;
  double fs = 0.0, us = 0.0;
  try {
    for (; k < nsteps; ++k) {
      if (stop_at_t_end && !(sim.t < t_end)) break;
      StepStats timing;
      const StepStats st = advance_step(sim, m, p, b, t_end, f, &timing);
      fs += timing.wall_flux_ms / 1e3;
      us += timing.wall_update_ms / 1e3;
      if (dts) dts[k] = st.dt;
      if (maxspeeds) maxspeeds[k] = st.max_speed;
    }
  } catch (const std::exception& e) {
    put_err(e, err, errlen);
    rc = classify(e);
  }
  std::memcpy(h, sim.current.h.data(), sizeof(double) * m.n_cells());
  std::memcpy(qx, sim.current.qx.data(), sizeof(double) * m.n_cells());
  std::memcpy(qy, sim.current.qy.data(), sizeof(double) * m.n_cells());
  *t = sim.t;
  *step = sim.step;
  *clip_volume = sim.ledger.clipped_volume;
  *clip_events = sim.ledger.clip_events;
  if (flux_s) *flux_s = fs;
  if (update_s) *update_s = us;
  if (done) *done = k;
  return rc;
}

// swe::run (engine.hpp:335).  series rows are {step, t, dt, max_speed, mass}
// (5 doubles each, up to max_rows); stats = {steps, t_final, mass_initial,
// mass_final, mass_drift_rel, min_dt, mean_dt, clip_events, clipped_volume};
// snapshot times are written to snaps (up to max_snaps).
__attribute__((visibility("default"))) int ref_run(void* mp, const double* params, double* h,
                                                   double* qx, double* qy, double* t, long* step,
                                                   double t_end, double snapshot_interval,
                                                   long max_steps, int threads, double* series,
                                                   long max_rows, long* n_rows, double* stats,
                                                   double* snaps, long max_snaps, long* n_snaps,
                                                   char* err, int errlen) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  Simulation sim;
  sim.current = state_from(m.n_cells(), h, qx, qy);
  sim.next.resize(m.n_cells());
  sim.t = *t;
  sim.step = *step;
  RunOptions opt;
  opt.t_end = t_end;
  opt.snapshot_interval = snapshot_interval;
  opt.max_steps = max_steps;
  long ns = 0;
  if (snaps)
    opt.on_snapshot = [&](const FieldState&, double tt, long) {
      if (ns < max_snaps) snaps[ns] = tt;
      ++ns;
    };
  int rc = 0;
  try {
    const RunStats rs = run(sim, m, params_from(params), backend_for(threads), opt);
    long r = 0;
    for (const StepStats& st : rs.series) {
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
    put_err(e, err, errlen);
    rc = classify(e);
  }
  if (n_snaps) *n_snaps = ns;
  std::memcpy(h, sim.current.h.data(), sizeof(double) * m.n_cells());
  std::memcpy(qx, sim.current.qx.data(), sizeof(double) * m.n_cells());
  std::memcpy(qy, sim.current.qy.data(), sizeof(double) * m.n_cells());
  *t = sim.t;
  *step = sim.step;
  return rc;
}

// ---- point physics (kernels.hpp) over arrays, for kernel-level goldens ----
// states are (h, qx, qy) triples; normals (nx, ny) pairs.

// kernels.hpp entry points with the device point-eval layouts (swe_dev.h
// swe_dev_point_eval kinds 5-9): 5 physical_flux_normal, 6
// wave_speed_estimates(l[0], l[1], r[0], r[1]), 7 hydrostatic_reconstruct
// -> 12, 8 cell_signal_speed -> 1, 9 clamp_dry -> {h, qx, qy, clipped, throws}
__attribute__((visibility("default"))) int ref_point(int kind, long n, const double* params,
                                                     const double* l, const double* r,
                                                     const double* z, const double* nrm,
                                                     double* out) {
  const PhysParams p = params_from(params);
  for (long i = 0; i < n; ++i) {
    const ConservedState a{l[3 * i], l[3 * i + 1], l[3 * i + 2]};
    if (kind == 5) {
      const Flux3 f = physical_flux_normal(a, {nrm[2 * i], nrm[2 * i + 1]}, p);
      out[3 * i] = f.mass;
      out[3 * i + 1] = f.momx;
      out[3 * i + 2] = f.momy;
    } else if (kind == 6) {
      const WaveSpeeds w = wave_speed_estimates(a.h, a.qx, r[3 * i], r[3 * i + 1], p);
      out[3 * i] = w.SL;
      out[3 * i + 1] = w.Sstar;
      out[3 * i + 2] = w.SR;
    } else if (kind == 7) {
      const ConservedState b{r[3 * i], r[3 * i + 1], r[3 * i + 2]};
      const ReconstructedInterface ri =
          hydrostatic_reconstruct(a, z[2 * i], b, z[2 * i + 1], {nrm[2 * i], nrm[2 * i + 1]}, p);
      const double v[12] = {ri.left.h, ri.left.qx, ri.left.qy, ri.right.h, ri.right.qx,
                            ri.right.qy, ri.corr_left.mass, ri.corr_left.momx, ri.corr_left.momy,
                            ri.corr_right.mass, ri.corr_right.momx, ri.corr_right.momy};
      std::memcpy(out + 12 * i, v, sizeof(v));
    } else if (kind == 8) {
      out[i] = cell_signal_speed(a, p);
    } else if (kind == 9) {
      double clipped = 0.0;
      try {
        const ConservedState u = clamp_dry(a, p, &clipped);
        const double v[5] = {u.h, u.qx, u.qy, clipped, 0.0};
        std::memcpy(out + 5 * i, v, sizeof(v));
      } catch (const numeric_error&) {
        const double v[5] = {a.h, a.qx, a.qy, 0.0, 1.0};
        std::memcpy(out + 5 * i, v, sizeof(v));
      }
    } else {
      return 1;
    }
  }
  return 0;
}

// stable_dt (kernels.hpp:174-186): 0 ok, 1 non-finite (bad = the cell)
__attribute__((visibility("default"))) int ref_stable_dt(long n, const double* params,
                                                         const double* h, const double* qx,
                                                         const double* qy, const double* r,
                                                         double* dt, long* bad) {
  const PhysParams p = params_from(params);
  try {
    *dt = stable_dt({h, (size_t)n}, {qx, (size_t)n}, {qy, (size_t)n}, {r, (size_t)n}, p);
    return 0;
  } catch (const numeric_error& e) {
    const std::string w = e.what();
    *bad = std::stol(w.substr(w.rfind(' ') + 1));
    return 1;
  }
}

__attribute__((visibility("default"))) int ref_hllc(long n, const double* params, const double* l,
                                                    const double* r, const double* nrm,
                                                    double* out) {
  const PhysParams p = params_from(params);
  try {
    for (long i = 0; i < n; ++i) {
      const Flux3 f = hllc_flux({l[3 * i], l[3 * i + 1], l[3 * i + 2]},
                                {r[3 * i], r[3 * i + 1], r[3 * i + 2]},
                                {nrm[2 * i], nrm[2 * i + 1]}, p);
      out[3 * i] = f.mass;
      out[3 * i + 1] = f.momx;
      out[3 * i + 2] = f.momy;
    }
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

__attribute__((visibility("default"))) void ref_wall(long n, const double* params, const double* u,
                                                     const double* nrm, double* out) {
  const PhysParams p = params_from(params);
  for (long i = 0; i < n; ++i) {
    const Flux3 f = wall_flux({u[3 * i], u[3 * i + 1], u[3 * i + 2]}, {nrm[2 * i], nrm[2 * i + 1]}, p);
    out[3 * i] = f.mass;
    out[3 * i + 1] = f.momx;
    out[3 * i + 2] = f.momy;
  }
}

// edge combine of compute_fluxes for arbitrary inputs: z = (zl, zr)
__attribute__((visibility("default"))) void ref_edge(long n, const double* params, const double* l,
                                                     const double* r, const double* z,
                                                     const double* nrm, double* left,
                                                     double* right) {
  const PhysParams p = params_from(params);
  for (long i = 0; i < n; ++i) {
    const Vec2 nn{nrm[2 * i], nrm[2 * i + 1]};
    const ReconstructedInterface ri =
        hydrostatic_reconstruct({l[3 * i], l[3 * i + 1], l[3 * i + 2]}, z[2 * i],
                                {r[3 * i], r[3 * i + 1], r[3 * i + 2]}, z[2 * i + 1], nn, p);
    const Flux3 f = hllc_flux(ri.left, ri.right, nn, p);
    left[3 * i] = f.mass;
    left[3 * i + 1] = f.momx + ri.corr_left.momx;
    left[3 * i + 2] = f.momy + ri.corr_left.momy;
    right[3 * i] = -f.mass;
    right[3 * i + 1] = -(f.momx + ri.corr_right.momx);
    right[3 * i + 2] = -(f.momy + ri.corr_right.momy);
  }
}

__attribute__((visibility("default"))) void ref_friction(long n, const double* params,
                                                         const double* u, const double* nman,
                                                         const double* dt, double* out) {
  const PhysParams p = params_from(params);
  for (long i = 0; i < n; ++i) {
    const ConservedState o = apply_friction({u[3 * i], u[3 * i + 1], u[3 * i + 2]}, nman[i], dt[i], p);
    out[3 * i] = o.h;
    out[3 * i + 1] = o.qx;
    out[3 * i + 2] = o.qy;
  }
}

__attribute__((visibility("default"))) void ref_pow43(long n, const double* h, double* out) {
  for (long i = 0; i < n; ++i) out[i] = std::pow(h[i], 4.0 / 3.0);
}

__attribute__((visibility("default"))) void ref_wave_speeds(long n, const double* params,
                                                            const double* in, double* out) {
  const PhysParams p = params_from(params);
  for (long i = 0; i < n; ++i) {
    const WaveSpeeds s = wave_speed_estimates(in[4 * i], in[4 * i + 1], in[4 * i + 2], in[4 * i + 3], p);
    out[3 * i] = s.SL;
    out[3 * i + 1] = s.Sstar;
    out[3 * i + 2] = s.SR;
  }
}

// ---- cases (cases.hpp) --------------------------------------------------
// spec = {lx, ly, eta0, amplitude, sigma, manning, h_left, h_right, x_dam, t_end}
__attribute__((visibility("default"))) int ref_case_defaults(const char* name, double* spec) {
  try {
    const CaseSpec c = make_case(case_from_name(name));
    const double v[10] = {c.lx, c.ly, c.eta0, c.amplitude, c.sigma, c.manning,
                          c.h_left, c.h_right, c.x_dam, c.t_end};
    std::memcpy(spec, v, sizeof(v));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

__attribute__((visibility("default"))) void ref_generate_square_mesh(int nx, int ny, double lx,
                                                                     double ly, double* xy,
                                                                     int* tris) {
  const RawMesh raw = generate_square_mesh(nx, ny, lx, ly);
  for (size_t i = 0; i < raw.nodes.size(); ++i) {
    xy[2 * i] = raw.nodes[i].x;
    xy[2 * i + 1] = raw.nodes[i].y;
  }
  for (size_t c = 0; c < raw.triangles.size(); ++c)
    for (int k = 0; k < 3; ++k) tris[3 * c + k] = raw.triangles[c][k];
}

__attribute__((visibility("default"))) int ref_init_case(const char* name, const double* spec,
                                                         int nn, const double* xy, int nc,
                                                         const int* tris, double* bed,
                                                         double* manning, double* h, double* qx,
                                                         double* qy, char* err, int errlen) {
  try {
    CaseSpec c = make_case(case_from_name(name));
    c.lx = spec[0];
    c.ly = spec[1];
    c.eta0 = spec[2];
    c.amplitude = spec[3];
    c.sigma = spec[4];
    c.manning = spec[5];
    c.h_left = spec[6];
    c.h_right = spec[7];
    c.x_dam = spec[8];
    c.t_end = spec[9];
    RawMesh raw;
    raw.nodes.resize(nn);
    for (int i = 0; i < nn; ++i) raw.nodes[i] = {xy[2 * i], xy[2 * i + 1]};
    raw.triangles.resize(nc);
    for (int k = 0; k < nc; ++k) raw.triangles[k] = {tris[3 * k], tris[3 * k + 1], tris[3 * k + 2]};
    const CaseFields f = init_case(c, raw);
    std::memcpy(bed, f.bed.data(), sizeof(double) * nc);
    std::memcpy(manning, f.manning.data(), sizeof(double) * nc);
    std::memcpy(h, f.state.h.data(), sizeof(double) * nc);
    std::memcpy(qx, f.state.qx.data(), sizeof(double) * nc);
    std::memcpy(qy, f.state.qy.data(), sizeof(double) * nc);
    return 0;
  } catch (const std::exception& e) {
    put_err(e, err, errlen);
    return classify(e);
  }
}

__attribute__((visibility("default"))) int ref_rotated_cell_index(int c, int nx, int ny) {
  return rotated_cell_index(c, nx, ny);
}

__attribute__((visibility("default"))) void ref_stoker(long n, double hL, double hR,
                                                       const double* x, double t, double x_dam,
                                                       double g, double* h, double* u) {
  for (long i = 0; i < n; ++i) {
    const StokerSample s = stoker_exact(hL, hR, x[i], t, x_dam, g);
    h[i] = s.h;
    u[i] = s.u;
  }
}

}  // extern "C"

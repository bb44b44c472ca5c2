// api_driver.cpp -- a caller written against the REFERENCE API
// (/root/reference/proj/include/swe: setup_case, advance_step, run,
// compute_fluxes, total_mass, exceptions), compiled against this repo's
// drop-in headers (include/swe/*.hpp) and linked to libswe_b200.so.  It
// mirrors reference tests (test_engine.cpp, acceptance.cpp) and prints one
// JSON object that tests/test_gpu_api.py checks against the golden fixtures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "swe/cases.hpp"
#include "swe/engine.hpp"
#include "swe/mesh.hpp"

using namespace swe;

static unsigned long long fnv(const std::vector<double>& a, unsigned long long h = 1469598103934665603ull) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(a.data());
  for (size_t i = 0; i < a.size() * sizeof(double); ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

int main() {
  const PhysParams params;
  std::printf("{");

  {  // acceptance criterion 3 (acceptance.cpp:101-139): advance_step loop to t_end
    CaseSpec spec = make_case(CaseId::three_mounds);
    spec.t_end = 30.0;
    const RawMesh raw = generate_square_mesh(100, 40, spec.lx, spec.ly);
    CaseSetup setup = setup_case(spec, raw);
    Simulation sim;
    sim.current = setup.state;
    sim.next.resize(setup.mesh.n_cells());
    EdgeFluxes fluxes;
    fluxes.resize(setup.mesh.n_edges());
    long steps = 0;
    bool positive = true;
    while (sim.t < spec.t_end) {
      advance_step(sim, setup.mesh, params, {}, spec.t_end, fluxes);
      ++steps;
      for (double h : sim.current.h) positive = positive && h >= 0.0;
    }
    std::printf("\"c3_steps\": %ld, \"c3_positive\": %s, \"c3_t\": %.17g, ", steps,
                positive ? "true" : "false", sim.t);
  }

  {  // run() on the water drop (acceptance c2 geometry), 1000 steps via max horizon
    CaseSpec spec = make_case(CaseId::water_drop);
    const RawMesh raw = generate_square_mesh(71, 71, spec.lx, spec.ly);
    CaseSetup setup = setup_case(spec, raw);
    Simulation sim;
    sim.current = setup.state;
    sim.next.resize(setup.mesh.n_cells());
    RunOptions opt;
    opt.t_end = 868.4939716386242;  // t after 1000 reference steps
    int snaps = 0;
    opt.snapshot_interval = 200.0;
    opt.on_snapshot = [&](const FieldState&, double, long) { ++snaps; };
    const RunStats rs = run(sim, setup.mesh, params, {}, opt);
    std::vector<double> all = sim.current.h;
    all.insert(all.end(), sim.current.qx.begin(), sim.current.qx.end());
    all.insert(all.end(), sim.current.qy.begin(), sim.current.qy.end());
    std::printf("\"run_steps\": %ld, \"run_t\": %.17g, \"run_snaps\": %d, \"run_drift\": %.6e, "
                "\"run_series\": %zu, \"run_state_fnv\": \"%llx\", ",
                rs.steps, rs.t_final, snaps, rs.mass_drift_rel, rs.series.size(), fnv(all));
  }

  {  // compute_fluxes uniform flow cancels (test_engine.cpp:75-110)
    const RawMesh raw = generate_square_mesh(6, 5, 3.0, 2.0);
    const int nc = static_cast<int>(raw.triangles.size());
    const Mesh m = build_mesh(raw, std::vector<double>(nc, 0.0), std::vector<double>(nc, 0.0));
    FieldState s;
    s.resize(m.n_cells());
    for (int c = 0; c < m.n_cells(); ++c) {
      s.h[c] = 1.3;
      s.qx[c] = 1.3 * 0.4;
      s.qy[c] = 1.3 * -0.2;
    }
    EdgeFluxes f;
    f.resize(m.n_edges());
    compute_fluxes(s, m, params, {}, f);
    bool ok = true;
    for (int e = 0; e < m.n_edges(); ++e)
      if (m.edge_right[e] != kBoundary) ok = ok && f.left[e].mass == -f.right[e].mass;
    std::printf("\"uniform_mass_antisymmetric\": %s, \"mass_unit\": %.17g, ", ok ? "true" : "false",
                [&] {
                  FieldState u;
                  u.resize(m.n_cells());
                  for (auto& h : u.h) h = 1.0;
                  return total_mass(u, m);
                }());
  }

  {  // the device cache follows the Mesh's CONTENT: a bed mutated in place and a
     // new Mesh on recycled addresses are re-uploaded; helpers
     // called from on_snapshot during run() do not disturb the run
    CaseSpec spec = make_case(CaseId::three_mounds);
    const RawMesh raw = generate_square_mesh(40, 16, spec.lx, spec.ly);
    CaseSetup setup = setup_case(spec, raw);
    auto steps = [&](const Mesh& m, int n) {
      Simulation sim;
      sim.current = setup.state;
      sim.next.resize(m.n_cells());
      EdgeFluxes f;
      for (int k = 0; k < n; ++k) advance_step(sim, m, params, {}, 1e9, f);
      return sim.current.h;
    };
    Mesh m = setup.mesh;
    const std::vector<double> h0 = steps(m, 20);
    for (double& z : m.cell_bed) z *= 0.5;  // in place: same addresses and sizes
    const std::vector<double> h1 = steps(m, 20);
    const Mesh fresh = m;  // a distinct Mesh with the mutated bed
    const std::vector<double> h2 = steps(fresh, 20);
    const bool mutation_ok = h1 == h2 && h1 != h0;

    Simulation a;
    a.current = setup.state;
    a.next.resize(m.n_cells());
    Simulation b = a;
    RunOptions opt;
    opt.t_end = 3.0;
    opt.snapshot_interval = 0.5;
    int calls = 0;
    double mass_in_cb = 0.0;
    opt.on_snapshot = [&](const FieldState& s, double, long) {
      ++calls;
      mass_in_cb = total_mass(s, m);  // reference-legal inside a run
      EdgeFluxes f;
      compute_fluxes(s, m, params, {}, f);
      Simulation other;
      other.current = s;
      other.next.resize(m.n_cells());
      advance_step(other, m, params, {}, 1e9, f);
    };
    const RunStats ra = run(a, m, params, {}, opt);
    opt.on_snapshot = nullptr;
    const RunStats rb = run(b, m, params, {}, opt);
    const bool reentrant_ok = calls > 3 && ra.steps == rb.steps && ra.t_final == rb.t_final &&
                              a.current.h == b.current.h && a.current.qx == b.current.qx &&
                              mass_in_cb > 0.0;
    std::printf("\"cache_mutation_ok\": %s, \"reentrant_ok\": %s, ", mutation_ok ? "true" : "false",
                reentrant_ok ? "true" : "false");
  }

  {  // errors keep the reference's types and messages (test_engine.cpp:218-247)
    const RawMesh raw = generate_square_mesh(3, 3, 1.0, 1.0);
    const Mesh m = build_mesh(raw, std::vector<double>(18, 0.0), std::vector<double>(18, 0.0));
    Simulation sim;
    sim.current.resize(18);
    for (int c = 0; c < 18; ++c) {
      sim.current.h[c] = 0.5 + 0.05 * c;
      sim.current.qx[c] = 0.1;
    }
    sim.current.qx[5] = std::nan("");
    sim.next.resize(18);
    EdgeFluxes f;
    std::string nan_msg, neg_msg, cfg;
    try {
      advance_step(sim, m, params, {}, 1e9, f);
    } catch (const numeric_error& e) {
      nan_msg = e.what();
    }
    sim.current.qx[5] = 0.1;
    sim.current.h[0] = -0.5;
    try {
      compute_fluxes(sim.current, m, params, {}, f);
    } catch (const numeric_error& e) {
      neg_msg = e.what();
    }
    RunOptions opt;
    try {
      run(sim, m, params, {}, opt);
    } catch (const config_error& e) {
      cfg = e.what();
    }
    std::printf("\"nan_msg\": \"%s\", \"neg_msg\": \"%s\", \"cfg_msg\": \"%s\"", nan_msg.c_str(),
                neg_msg.c_str(), cfg.c_str());
  }
  std::printf("}\n");
  return 0;
}

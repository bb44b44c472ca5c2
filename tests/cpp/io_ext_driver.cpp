// io_ext_driver.cpp -- the §8(f) output and config rows next to the
// reference's own io.hpp (included in place, compiled against this repo's
// drop-in headers as tests/cpp/harness_driver.cpp does):
//   vtk        write_vtk_snapshot_parallel (include/swe/vtk.hpp) vs the
//              reference's write_vtk_snapshot (io.hpp:171-206): byte-identical
//              files; with "vtk nx ny" also both timings
//   config     backend.gpus / devices taken out of the text
//              (include/swe/config_gpus.hpp), the rest parsed by the
//              reference's parse_config (io.hpp:288-420)
//   config-run the parsed config run on 2 linked parts (one device,
//              lockstep) against the single-device run (GPU)
// Prints one JSON object.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>

#include "swe/cases.hpp"
#include "swe/config_gpus.hpp"
#include "swe/engine.hpp"
#include "swe/io.hpp"  // the reference's (its include dir follows ours on the path)
#include "swe/vtk.hpp"

using namespace swe;

static std::string slurp(const std::string& p) {
  std::ifstream f(p, std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "vtk";
  if (mode == "vtk") {
    const int nx = argc > 2 ? std::atoi(argv[2]) : 60, ny = argc > 3 ? std::atoi(argv[3]) : 24;
    const std::string dir = argc > 4 ? argv[4] : "/tmp";
    const RawMesh raw = generate_unstructured_mesh(nx, ny, 1000.0, 400.0, 0.2, 11);
    const int nc = static_cast<int>(raw.triangles.size());
    std::mt19937_64 rng(5);
    std::uniform_real_distribution<double> u(-2.0, 2.0);
    std::vector<double> bed(nc), man(nc, 0.03);
    for (double& z : bed) z = u(rng);
    const Mesh m = build_mesh(raw, bed, man);
    FieldState s;
    s.resize(nc);
    for (int c = 0; c < nc; ++c) {
      s.h[c] = c % 7 == 0 ? 0.0 : (c % 11 == 0 ? 5e-7 : std::fabs(u(rng)));
      s.qx[c] = s.h[c] * u(rng);
      s.qy[c] = c % 5 == 0 ? -0.0 : s.h[c] * u(rng);
    }
    const double t = 12.345678901234567;
    const auto t0 = std::chrono::steady_clock::now();
    write_vtk_snapshot(m, s, t, dir + "/ref.vtk");
    const auto t1 = std::chrono::steady_clock::now();
    write_vtk_snapshot_parallel(m, s, t, dir + "/ours.vtk");
    const auto t2 = std::chrono::steady_clock::now();
    const std::string a = slurp(dir + "/ref.vtk"), b = slurp(dir + "/ours.vtk");
    std::printf("{\"cells\": %d, \"bytes\": %zu, \"vtk_identical\": %s, \"ref_s\": %.3f, \"ours_s\": %.3f}\n",
                nc, a.size(), a == b ? "true" : "false",
                std::chrono::duration<double>(t1 - t0).count(),
                std::chrono::duration<double>(t2 - t1).count());
    std::remove((dir + "/ref.vtk").c_str());
    std::remove((dir + "/ours.vtk").c_str());
    return 0;
  }
  const std::string text = R"({
  "case": {"id": "three_mounds", "t_end": 4.0, "manning": 0.03},
  "mesh": {"generate": {"nx": 60, "ny": 24}},
  "backend": {"kind": "parallel", "threads": 2, "gpus": 2, "devices": [0, 0]}
})";
  BackendSpec ext;
  const std::string rest = split_backend_gpus(text, ext);
  std::string err;
  Config c;
  try {
    parse_config(text);
  } catch (const config_error& e) {
    err = e.what();  // the reference parser alone rejects the extension keys
  }
  c = parse_config(rest);
  apply_backend_gpus(ext, c.backend);
  std::printf("{\"gpus\": %d, \"devices\": %zu, \"kind_parallel\": %s, \"threads\": %d, "
              "\"plain_parser_error\": \"%s\"",
              c.backend.gpus, c.backend.devices.size(),
              c.backend.kind == BackendSpec::Kind::parallel ? "true" : "false", c.backend.threads,
              err.c_str());
  if (mode == "config-run") {
    const GeneratorSpec g = std::get<GeneratorSpec>(c.mesh_source);
    const RawMesh raw = generate_square_mesh(g.nx, g.ny, c.scenario.lx, c.scenario.ly);
    const CaseSetup setup = setup_case(c.scenario, raw);
    RunOptions opt;
    opt.t_end = c.scenario.t_end;
    Simulation a, b;
    a.current = b.current = setup.state;
    a.next.resize(setup.mesh.n_cells());
    b.next.resize(setup.mesh.n_cells());
    const RunStats ra = run(a, setup.mesh, c.params, c.backend, opt);
    const RunStats rb = run(b, setup.mesh, c.params, BackendSpec{}, opt);
    const bool same = a.current.h == b.current.h && a.current.qx == b.current.qx &&
                      a.current.qy == b.current.qy && ra.steps == rb.steps && ra.t_final == rb.t_final;
    std::printf(", \"steps\": %ld, \"two_gpu_run_equals_one\": %s", ra.steps, same ? "true" : "false");
  }
  std::printf("}\n");
  return 0;
}

// multigpu_driver.cpp -- the multi-GPU path of the drop-in C++ API
// (include/swe/multigpu.hpp) driven the way a reference caller would:
//
//   run(sim, mesh, params, backend, opt)
//     * backend.gpus = 2, backend.devices = {0, 0}: two linked parts of one
//       process on one device (stepped in lockstep: no kernel waits on a
//       concurrently running one) -- against the single-domain run();
//     * backend.comm: two ranks (threads of this process, an in-process
//       allgather and barrier), one linked part each through CUDA IPC
//       handles, lockstep on the shared device -- against the same;
//   build_rank_mesh: the rank-local part built from the RawMesh alone equals
//   the part sliced from the global Mesh (every array but the edge ids).
//
// Prints one JSON object (tests/test_gpu_multigpu.py checks it).
//   multigpu_driver [host]   "host": only the CPU-side rank-local check
#include <barrier>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "swe/cases.hpp"
#include "swe/engine.hpp"
#include "swe/mesh.hpp"
#include "swe/multigpu.hpp"

using namespace swe;

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

static bool same_state(const FieldState& a, const FieldState& b) {
  return same_bits(a.h, b.h) && same_bits(a.qx, b.qx) && same_bits(a.qy, b.qy);
}

static bool same_series(const RunStats& a, const RunStats& b) {
  if (a.series.size() != b.series.size() || a.steps != b.steps || a.t_final != b.t_final) return false;
  for (size_t i = 0; i < a.series.size(); ++i) {
    const StepStats &x = a.series[i], &y = b.series[i];
    if (x.step != y.step || x.t != y.t || x.dt != y.dt || x.max_speed != y.max_speed) return false;
    if (std::fabs(x.mass - y.mass) > 1e-12 * std::fabs(y.mass)) return false;
  }
  return true;
}

// rank-local part == part sliced from the global mesh
static bool rank_mesh_matches(const RawMesh& raw, const CaseSetup& setup, int P) {
  const std::vector<int> part = rcb_partition(raw, P);
  const Mesh& m = setup.mesh;
  for (int p = 0; p < P; ++p) {
    const LocalMesh a = build_rank_mesh(raw, m.cell_bed, m.cell_manning, part, p);
    const LocalMesh b = build_local_mesh(m, part, p);
    if (a.cells != b.cells || a.n_owned != b.n_owned || !same_bits(a.area, b.area) ||
        !same_bits(a.inradius, b.inradius) || !same_bits(a.bed, b.bed) ||
        !same_bits(a.manning, b.manning) || !same_bits(a.cx, b.cx) || !same_bits(a.cy, b.cy) ||
        a.cell_edge != b.cell_edge || a.cell_sign != b.cell_sign || a.edge_left != b.edge_left ||
        a.edge_right != b.edge_right || !same_bits(a.nx, b.nx) || !same_bits(a.ny, b.ny) ||
        !same_bits(a.len, b.len) || a.peers != b.peers || a.send != b.send || a.recv != b.recv)
      return false;
  }
  return true;
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::string(argv[1]) == "host";
  CaseSpec spec = make_case(CaseId::three_mounds);
  spec.manning = 0.03;
  const RawMesh raw = generate_unstructured_mesh(90, 36, spec.lx, spec.ly, 0.2, 7);
  const CaseSetup setup = setup_case(spec, raw);
  std::printf("{\"cells\": %d, \"rank_mesh_matches\": %s", setup.mesh.n_cells(),
              rank_mesh_matches(raw, setup, 3) ? "true" : "false");
  if (host_only) {
    std::printf("}\n");
    return 0;
  }
  const PhysParams params;
  RunOptions opt;
  opt.t_end = 6.0;
  opt.snapshot_interval = 2.0;
  auto fresh = [&] {
    Simulation s;
    s.current = setup.state;
    s.next.resize(setup.mesh.n_cells());
    return s;
  };

  Simulation one = fresh();
  int snaps1 = 0;
  RunOptions o1 = opt;
  o1.on_snapshot = [&](const FieldState&, double, long) { ++snaps1; };
  const RunStats r1 = run(one, setup.mesh, params, {}, o1);

  // (1) one process, two parts on device 0 (lockstep)
  Simulation two = fresh();
  BackendSpec b2;
  b2.gpus = 2;
  b2.devices = {0, 0};
  int snaps2 = 0;
  bool snap_ok = true;
  std::vector<FieldState> snap1;
  RunOptions o2 = opt;
  o2.on_snapshot = [&](const FieldState& s, double, long) {
    ++snaps2;
    snap_ok = snap_ok && s.size() == setup.mesh.n_cells();
  };
  const RunStats r2 = run(two, setup.mesh, params, b2, o2);

  // (2) two ranks (threads) through backend.comm, CUDA IPC, lockstep
  const int P = 2;
  std::barrier<> bar(P);
  std::mutex mu;
  std::vector<std::string> slots(P);
  auto allgather_for = [&](int rank) {
    return [&, rank](const std::string& mine) {
      {
        std::lock_guard<std::mutex> lk(mu);
        slots[rank] = mine;
      }
      bar.arrive_and_wait();
      std::vector<std::string> all = slots;
      bar.arrive_and_wait();
      return all;
    };
  };
  std::vector<Simulation> sims(P, fresh());
  std::vector<RunStats> rr(P);
  std::vector<std::string> errs(P);
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r)
    th.emplace_back([&, r] {
      Comm comm;
      comm.rank = r;
      comm.size = P;
      comm.allgather = allgather_for(r);
      comm.barrier = [&] { bar.arrive_and_wait(); };
      BackendSpec b;
      b.device = 0;
      b.comm = &comm;
      b.lockstep = true;
      try {
        rr[r] = run(sims[r], setup.mesh, params, b, opt);
      } catch (const std::exception& e) {
        errs[r] = e.what();
      }
    });
  for (auto& t : th) t.join();
  bool ranks_ok = errs[0].empty() && errs[1].empty();
  for (int r = 0; r < P && ranks_ok; ++r)
    ranks_ok = same_state(sims[r].current, one.current) && same_series(rr[r], r1);

  std::printf(", \"steps\": %ld, \"gpus2_state_bitwise\": %s, \"gpus2_series_ok\": %s, "
              "\"snapshots\": [%d, %d], \"snap_ok\": %s, \"ledger_events\": [%ld, %ld], "
              "\"comm_ranks_ok\": %s, \"comm_errors\": \"%s|%s\"}\n",
              r1.steps, same_state(two.current, one.current) ? "true" : "false",
              same_series(r2, r1) ? "true" : "false", snaps1, snaps2, snap_ok ? "true" : "false",
              one.ledger.clip_events, two.ledger.clip_events, ranks_ok ? "true" : "false",
              errs[0].c_str(), errs[1].c_str());
  return 0;
}

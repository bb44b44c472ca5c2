// harness_driver.cpp -- the reference's own harness (bench ladder and Stoker
// convergence study, /root/reference/proj/include/swe/bench.hpp) compiled
// UNCHANGED against this repo's drop-in headers (include/ first on the path),
// so every advance_step / run inside it executes on the B200
// (SURVEY.md §8(f) row 4).  Built by paper_1807_00672_b200/build.py where
// /root/reference exists; the binary travels to the GPU box.
//
//   harness_driver converge [nx0 ny0 levels t_eval]   -> CSV of the study
//   harness_driver ladder   [steps nx...]             -> CSV of the ladder
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>

#include "swe/bench.hpp"

int main(int argc, char** argv) {
  using namespace swe;
  const std::string mode = argc > 1 ? argv[1] : "converge";
  try {
    if (mode == "converge") {
      ConvergenceOptions opt;  // acceptance.cpp:231-238 defaults
      opt.scenario = make_case(CaseId::dam_break_1d);
      const int nx0 = argc > 2 ? std::atoi(argv[2]) : 100;
      const int ny0 = argc > 3 ? std::atoi(argv[3]) : 10;
      const int levels = argc > 4 ? std::atoi(argv[4]) : 3;
      opt.t_eval = argc > 5 ? std::atof(argv[5]) : 40.0;
      opt.resolutions.clear();
      for (int l = 0; l < levels; ++l) opt.resolutions.push_back({nx0 << l, ny0 << l});
      write_convergence_csv(std::cout, convergence_study(opt));
    } else if (mode == "ladder") {
      BenchOptions opt;  // bench.hpp:53-65, the GPU behind both backend labels
      opt.fixed_steps = argc > 2 ? std::atol(argv[2]) : 50;
      opt.nx_list.clear();
      for (int i = 3; i < argc; ++i) opt.nx_list.push_back(std::atoi(argv[i]));
      if (opt.nx_list.empty()) opt.nx_list = {23, 71, 229, 727};
      opt.run_parallel = false;
      opt.reps = 3;
      write_bench_csv(std::cout, run_benchmark(opt));
    } else {
      std::fprintf(stderr, "usage: harness_driver converge|ladder ...\n");
      return 2;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}

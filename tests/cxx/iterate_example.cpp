// Drop-in check of include/asdsm_b200.hpp: the reference's asdsm_iterate call shape, switched to
// the asdsm_b200 namespace.  Usage: iterate_example <example> <setting> <nf> <nc> <max_iter> [seed]
// Prints one CSV row per history record (k,res_l2,res_inf,err_max,err_l2,s_hat) and the stop
// reason; exits 0, or 3 with the exception class on a library error (no GPU: CudaFailure).
#include <cstdio>
#include <cstdlib>
#include <typeinfo>

#include "asdsm_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s example setting nf nc max_iter [seed]\n", argv[0]);
    return 2;
  }
  try {
    const auto problem = asdsm_b200::make_problem(std::atoi(argv[1]), std::atoi(argv[2]));
    const auto mesh = asdsm_b200::example_mesh(std::atoi(argv[1]), std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]));
    asdsm_b200::IterateOptions o;
    o.tol = 0.0;
    o.max_iter = std::atoi(argv[5]);
    o.stagnation_window = 0;
    o.rng_seed = argc > 6 ? std::strtoull(argv[6], nullptr, 10) : 0;
    const asdsm_b200::IterationState st = asdsm_b200::asdsm_iterate(problem, mesh, o);
    for (const auto& h : st.history)
      std::printf("%d,%.17g,%.17g,%.17g,%.17g,%.17g\n", h.k, h.res_l2, h.res_inf, h.err_max, h.err_l2, h.s_hat);
    std::printf("stop,%s\n", st.stop_reason.c_str());
    return 0;
  } catch (const asdsm_b200::CudaFailure& e) {
    std::printf("error,CudaFailure,%s\n", e.what());
    return 3;
  } catch (const asdsm_b200::Error& e) {
    std::printf("error,%s,%s\n", typeid(e).name(), e.what());
    return 3;
  }
}

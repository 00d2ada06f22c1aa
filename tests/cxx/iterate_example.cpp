// Drop-in check of include/asdsm_b200.hpp: the reference's asdsm_iterate call shape, switched to
// the asdsm_b200 namespace.  Usage: iterate_example <example> <setting> <nf> <nc> <max_iter> [seed]
// Prints one CSV row per history record (k,res_l2,res_inf,err_max,err_l2,s_hat) and the stop
// reason; exits 0, or 3 with the exception class on a library error (no GPU: CudaFailure).
#include <cmath>
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
    // ASDSM_EXAMPLE_FIELDS=1: example 1 setting 1 restated as caller-defined fields (FieldSpec,
    // problems.cpp:13-25) with an observer counting the records -- the same solve
    const bool fields = std::getenv("ASDSM_EXAMPLE_FIELDS") != nullptr;
    asdsm_b200::FieldSpec fs;
    if (fields) {
      const double pi = 3.14159265358979323846;
      fs.dim = 2;
      fs.alpha = {[](const asdsm_b200::Coord&) { return 1.0; }, [](const asdsm_b200::Coord&) { return 1.0; }, {}};
      fs.beta = fs.alpha;
      fs.exact = [pi](const asdsm_b200::Coord& x) { return std::sin(pi * x[0] + pi * x[1]); };
      fs.boundary = fs.exact;
      fs.source = [pi](const asdsm_b200::Coord& x) {
        const double th = pi * x[0] + pi * x[1];
        return 2.0 * pi * pi * std::sin(th) + 2.0 * pi * std::cos(th);
      };
    }
    const auto problem = fields ? asdsm_b200::make_problem(fs) : asdsm_b200::make_problem(std::atoi(argv[1]), std::atoi(argv[2]));
    const auto mesh = asdsm_b200::example_mesh(std::atoi(argv[1]), std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]));
    asdsm_b200::IterateOptions o;
    o.tol = 0.0;
    o.max_iter = std::atoi(argv[5]);
    o.stagnation_window = 0;
    o.rng_seed = argc > 6 ? std::strtoull(argv[6], nullptr, 10) : 0;
    int observed = 0;
    if (fields) o.observer = [&observed](const asdsm_b200::IterationState& s) { observed += s.history.back().k == observed; };
    const asdsm_b200::IterationState st = asdsm_b200::asdsm_iterate(problem, mesh, o);
    if (fields) std::printf("observed,%d\n", observed);
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

// Golden-vector dump driver for the compiled reference (oracle/_ref).  Test infrastructure.
//
// Links the reference's own library (built from /root/reference/proj/src by oracle/Makefile)
// and writes its outputs as raw little-endian binaries for the pytest parity suite:
//   iterate  <spec> <nf> <nc> <iters> <seed> <prefix>   asdsm_iterate (solver.cpp:565-680)
//   bundle   <spec> <nf> <nc> <prefix>                  SolverContext::assembled_bundle (solver.cpp:504)
//   errguess <spec> <nf> <nc> <seed> <r.f64> <prefix>   SolverContext::error_guess (solver.cpp:550)
//   maps     <spec> <nf> <nc> <prefix>                  build_projector / hole_blocks (mesh.cpp:210-305)
//   stage    <name> <spec> <nf> <nc> <seed> <in> <out>  a public solver stage on fields read from
//            <in>.<field>.f64 (solver.hpp:70-105): richardson (u1 u2 ucc), choose (ufc ucf),
//            spline0 / spline1 (ua ecc; dense axis 0 / 1), skeleton_s (ufc ucf ucc), skeleton_e
//            (ufc ucf), merge_s (ux uy uz uccc), merge_e (ux uy uz), fill (skel b) -> <out>.f64
// <spec> is ex:E:S (reference example E, setting S, problems.cpp:114) or cfg:ID:SEED (a
// BASELINE.json config from include/asdsm_problems.hpp).  nf/nc = 0 keeps the catalogue mesh.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/asdsm_problems.hpp"
#include "asdsm/linsolve.hpp"
#include "asdsm/problems.hpp"
#include "asdsm/solver.hpp"

using namespace asdsm;

namespace {

struct Case {
  ProblemSpec problem;
  MeshConfig mesh;
  int iterations = 20;
};

ProblemSpec to_spec(const asdsm_cat::Problem& p) {
  ProblemSpec s;
  s.dim = p.dim;
  s.time_dependent = p.time_dependent;
  for (int a = 0; a < 3; ++a) {
    s.alpha[static_cast<std::size_t>(a)] = p.alpha[static_cast<std::size_t>(a)];
    s.beta[static_cast<std::size_t>(a)] = p.beta[static_cast<std::size_t>(a)];
  }
  s.source = p.source;
  s.boundary = p.boundary;
  s.exact = p.exact;
  return s;
}

Case make_case(const std::string& spec, int nf, int nc) {
  Case c;
  int dim = 2, time_axis = -1;
  std::array<int, 3> f{}, co{};
  if (spec.rfind("ex:", 0) == 0) {
    int e = 0, s = 0;
    std::sscanf(spec.c_str(), "ex:%d:%d", &e, &s);
    c.problem = make_problem(e, s);
    dim = c.problem.dim;
    time_axis = c.problem.time_dependent ? dim - 1 : -1;
    for (int a = 0; a < dim; ++a) {
      f[static_cast<std::size_t>(a)] = nf;
      co[static_cast<std::size_t>(a)] = nc;
    }
  } else if (spec.rfind("cfg:", 0) == 0) {
    int id = 0;
    unsigned long long seed = 0;
    std::sscanf(spec.c_str(), "cfg:%d:%llu", &id, &seed);
    c.problem = to_spec(asdsm_cat::baseline_problem(id, seed));
    const auto m = asdsm_cat::baseline_mesh(id);
    dim = m.dim;
    time_axis = m.time_axis;
    c.iterations = m.iterations;
    for (int a = 0; a < dim; ++a) {
      f[static_cast<std::size_t>(a)] = nf > 0 ? nf : m.nf[static_cast<std::size_t>(a)];
      co[static_cast<std::size_t>(a)] = nc > 0 ? nc : m.nc[static_cast<std::size_t>(a)];
    }
  } else {
    throw std::invalid_argument("spec must be ex:E:S or cfg:ID:SEED");
  }
  c.mesh = MeshConfig::create(dim, std::span<const int>(f.data(), static_cast<std::size_t>(dim)),
                              std::span<const int>(co.data(), static_cast<std::size_t>(dim)), time_axis);
  return c;
}

template <typename T>
void write_bin(const std::string& path, const std::vector<T>& v) {
  std::ofstream o(path, std::ios::binary);
  o.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

void write_meta(const std::string& prefix, const MeshConfig& m) {
  std::ofstream o(prefix + ".meta.txt");
  o << m.dim << " " << m.time_axis << "\n";
  for (int a = 0; a < m.dim; ++a) o << m.fine_counts[static_cast<std::size_t>(a)] << " ";
  o << "\n";
  for (int a = 0; a < m.dim; ++a) o << m.coarse_counts[static_cast<std::size_t>(a)] << " ";
  o << "\n";
}

int cmd_iterate(int argc, char** argv) {
  if (argc < 8) return 2;
  Case c = make_case(argv[2], std::atoi(argv[3]), std::atoi(argv[4]));
  const int iters = std::atoi(argv[5]) >= 0 ? std::atoi(argv[5]) : c.iterations;
  const std::string prefix = argv[7];
  IterateOptions o;
  o.tol = 0.0;
  o.max_iter = iters;
  o.stagnation_window = 0;
  if (std::getenv("REF_DUMP_DEFAULT_OPTS")) {  // the reference's IterateOptions defaults (solver.hpp:56-68)
    o.tol = 1e-12;
    o.stagnation_window = 3;
    o.stagnation_ratio = 0.99;
  }
  // explicit stop-rule options (test fixtures for the stop rules): tolerance, stagnation window/ratio
  if (const char* v = std::getenv("REF_DUMP_TOL")) o.tol = std::atof(v);
  if (const char* v = std::getenv("REF_DUMP_STAG_WINDOW")) o.stagnation_window = std::atoi(v);
  if (const char* v = std::getenv("REF_DUMP_STAG_RATIO")) o.stagnation_ratio = std::atof(v);
  o.rng_seed = std::strtoull(argv[6], nullptr, 10);
  if (argc > 8) o.subsample = std::atof(argv[8]);
  std::vector<double> u0, r0;
  o.observer = [&](const IterationState& st) {
    if (st.history.size() == 1) {
      u0 = st.u.values;
      r0 = st.r.values;
    }
  };
  const IterationState st = asdsm_iterate(c.problem, c.mesh, o);
  write_meta(prefix, c.mesh);
  {
    std::FILE* f = std::fopen((prefix + ".hist.txt").c_str(), "w");
    for (const auto& h : st.history)
      std::fprintf(f, "%d %.17g %.17g %.17g %.17g %.17g %.17g\n", h.k, h.res_l2, h.res_inf, h.err_max,
                   h.err_l2, h.s_hat, h.wall_ms);
    std::fprintf(f, "# stop: %s\n", st.stop_reason.c_str());
    std::fclose(f);
  }
  write_bin(prefix + ".u.f64", st.u.values);
  write_bin(prefix + ".r.f64", st.r.values);
  write_bin(prefix + ".u0.f64", u0);
  write_bin(prefix + ".r0.f64", r0);
  return 0;
}

int cmd_bundle(int argc, char** argv) {
  if (argc < 6) return 2;
  Case c = make_case(argv[2], std::atoi(argv[3]), std::atoi(argv[4]));
  const std::string prefix = argv[5];
  const SolverContext ctx(c.mesh, c.problem);
  const RhsBundle b = ctx.assembled_bundle();
  write_meta(prefix, c.mesh);
  write_bin(prefix + ".b_fine.f64", b.fine.values);
  for (std::size_t a = 0; a < b.aniso.size(); ++a) write_bin(prefix + ".b_slab" + std::to_string(a) + ".f64", b.aniso[a].values);
  write_bin(prefix + ".b_coarse.f64", b.coarse->values);
  if (c.problem.exact) {
    const MeshKind ff = MeshKind::fine(c.mesh.dim);
    std::vector<double> ex(static_cast<std::size_t>(c.mesh.point_count(ff)));
    for (std::int64_t lin = 0; lin < c.mesh.point_count(ff); ++lin) {
      const auto idx = c.mesh.multi_index(ff, lin);
      ex[static_cast<std::size_t>(lin)] =
          c.problem.exact(c.mesh.coordinate(ff, std::span<const int>(idx.data(), static_cast<std::size_t>(c.mesh.dim))));
    }
    write_bin(prefix + ".exact.f64", ex);
  }
  // A_ff in CSR, for operator-level parity.
  const SparseMatrix& A = ctx.fine_operator();
  write_bin(prefix + ".A_rowptr.i64", std::vector<std::int64_t>(A.row_ptr().begin(), A.row_ptr().end()));
  write_bin(prefix + ".A_col.i64", std::vector<std::int64_t>(A.col_indices().begin(), A.col_indices().end()));
  write_bin(prefix + ".A_val.f64", std::vector<double>(A.values().begin(), A.values().end()));
  return 0;
}

int cmd_errguess(int argc, char** argv) {
  if (argc < 8) return 2;
  Case c = make_case(argv[2], std::atoi(argv[3]), std::atoi(argv[4]));
  const std::uint64_t seed = std::strtoull(argv[5], nullptr, 10);
  const SolverContext ctx(c.mesh, c.problem);
  const MeshKind ff = MeshKind::fine(c.mesh.dim);
  GridFunction r(ff, c.mesh.point_count(ff));
  {
    std::ifstream in(argv[6], std::ios::binary);
    in.read(reinterpret_cast<char*>(r.values.data()), static_cast<std::streamsize>(r.values.size() * sizeof(double)));
  }
  const GridFunction e = ctx.error_guess(r, seed);
  write_bin(std::string(argv[7]) + ".e.f64", e.values);
  const double s = optimal_scaling(c.mesh, r, ctx.fine_operator(), e, 0.0, seed);
  std::FILE* f = std::fopen((std::string(argv[7]) + ".s.txt").c_str(), "w");
  std::fprintf(f, "%.17g\n", s);
  std::fclose(f);
  return 0;
}

int cmd_maps(int argc, char** argv) {
  if (argc < 6) return 2;
  Case c = make_case(argv[2], std::atoi(argv[3]), std::atoi(argv[4]));
  const std::string prefix = argv[5];
  const int dim = c.mesh.dim;
  write_meta(prefix, c.mesh);
  const unsigned full = (1u << dim) - 1u;
  for (unsigned from = 0; from <= full; ++from)
    for (unsigned to = 0; to <= full; ++to) {
      if (from == to || (from & to) != from) continue;
      const Projector p = build_projector(c.mesh, MeshKind::from_mask(dim, from), MeshKind::from_mask(dim, to));
      write_bin(prefix + ".map_" + std::to_string(from) + "_" + std::to_string(to) + ".i64",
                std::vector<std::int64_t>(p.index_map().begin(), p.index_map().end()));
    }
  const Projector h = build_projector(c.mesh, MeshKind::fine(dim), MeshKind::holes(dim));
  write_bin(prefix + ".map_holes.i64", std::vector<std::int64_t>(h.index_map().begin(), h.index_map().end()));
  return 0;
}

GridFunction read_field(const std::string& in, const char* name, const MeshKind& kind, const MeshConfig& m) {
  GridFunction g(kind, m.point_count(kind));
  std::ifstream f(in + "." + name + ".f64", std::ios::binary);
  if (!f) throw std::runtime_error(std::string("missing input field ") + name);
  f.read(reinterpret_cast<char*>(g.values.data()), static_cast<std::streamsize>(g.values.size() * sizeof(double)));
  return g;
}

int cmd_stage(int argc, char** argv) {
  if (argc < 9) return 2;
  const std::string name = argv[2];
  Case c = make_case(argv[3], std::atoi(argv[4]), std::atoi(argv[5]));
  const std::uint64_t seed = std::strtoull(argv[6], nullptr, 10);
  const std::string in = argv[7], out = argv[8];
  const MeshConfig& m = c.mesh;
  const int dim = m.dim;
  const MeshKind cc = MeshKind::coarse(dim), ff = MeshKind::fine(dim);
  auto slab = [&](int a) { return MeshKind::coarse_along(dim, a); };
  GridFunction r;
  if (name == "richardson") {
    r = richardson_extrapolate(read_field(in, "u1", cc, m), read_field(in, "u2", cc, m), read_field(in, "ucc", cc, m));
  } else if (name == "choose") {
    SkeletonInputs si{read_field(in, "ufc", slab(1), m), read_field(in, "ucf", slab(0), m), std::nullopt, true};
    r = choose_cross_points(si, m, seed);
  } else if (name == "spline0" || name == "spline1") {
    const int dense = name == "spline0" ? 0 : 1;
    r = spline_correct(read_field(in, "ua", slab(1 - dense), m), read_field(in, "ecc", cc, m), dense, m);
  } else if (name == "skeleton_s" || name == "skeleton_e") {
    const bool smooth = name == "skeleton_s";
    SkeletonInputs si{read_field(in, "ufc", slab(1), m), read_field(in, "ucf", slab(0), m), std::nullopt, !smooth};
    if (smooth) si.u_cc = read_field(in, "ucc", cc, m);
    r = build_skeleton(si, m, seed);
  } else if (name == "merge_s" || name == "merge_e") {
    std::optional<GridFunction> uccc;
    if (name == "merge_s") uccc = read_field(in, "uccc", cc, m);
    r = merge_3d(read_field(in, "ux", slab(0), m), read_field(in, "uy", slab(1), m), read_field(in, "uz", slab(2), m),
                 uccc, m, seed);
  } else if (name == "fill") {
    const SolverContext ctx(m, c.problem);
    r = fill_holes(read_field(in, "skel", ff, m), ctx.fine_operator(), read_field(in, "b", ff, m), m);
  } else {
    throw std::invalid_argument("unknown stage " + name);
  }
  write_bin(out + ".f64", r.values);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_dump iterate|bundle|errguess|maps ...\n");
    return 2;
  }
  try {
    const std::string cmd = argv[1];
    if (cmd == "iterate") return cmd_iterate(argc, argv);
    if (cmd == "bundle") return cmd_bundle(argc, argv);
    if (cmd == "errguess") return cmd_errguess(argc, argv);
    if (cmd == "maps") return cmd_maps(argc, argv);
    if (cmd == "stage") return cmd_stage(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_dump: %s\n", e.what());
    return 3;
  }
  return 2;
}

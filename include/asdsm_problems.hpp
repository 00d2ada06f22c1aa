// Problem catalogue shared by the B200 host code and the oracle dump driver.
//
// Header-only, plain C++17, no CUDA.  Mirrors the reference's problem layer:
//   - reference examples 1-4, settings 1/2: proj/src/problems.cpp:13-141 (make_problem)
//   - the five BASELINE.json configs (synthetic, seeded) used by bench.py and the parity tests
// A problem is the reference's ProblemSpec (proj/include/asdsm/fdm.hpp:18-30): per-axis
// alpha/beta, source s, boundary g (initial data on t=0 for time problems), optional exact u.
// The GPU path computes with constant per-axis coefficients, so every problem here records
// whether its coefficients are constant (`constant_coeffs`) and their values.
#pragma once
#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace asdsm_cat {

using Coord = std::array<double, 3>;
using Field = std::function<double(const Coord&)>;

struct Problem {
  int dim = 2;
  bool time_dependent = false;
  std::array<Field, 3> alpha{}, beta{};  // per spatial axis
  Field source, boundary, exact;          // exact may be empty
  bool constant_coeffs = true;
  std::array<double, 3> alpha_c{}, beta_c{};  // valid iff constant_coeffs
  int spatial_axes() const { return time_dependent ? dim - 1 : dim; }
};

struct MeshChoice {
  int dim = 2;
  std::array<int, 3> nf{}, nc{};
  int time_axis = -1;
  int iterations = 20;
};

// splitmix64 stream: the seeded generator behind every synthetic source term.
struct SplitMix64 {
  std::uint64_t s;
  explicit SplitMix64(std::uint64_t seed) : s(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }        // [0,1)
  double uniform_open() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }  // (0,1)
  double normal() {  // Box-Muller, one draw per call
    const double u1 = uniform_open(), u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
};

struct Bump {
  std::array<double, 3> c{};
  double w = 0.1, amp = 0.0;
};

// Gaussian bumps: s(x) = sum_i amp_i exp(-|x - c_i|^2 / (2 w_i^2)), centers uniform in
// (0,1)^d, widths uniform in [0.05, 0.2], amplitudes N(0,1), drawn in that order per bump.
inline std::vector<Bump> draw_bumps(int count, int dims, std::uint64_t seed) {
  SplitMix64 g(seed);
  std::vector<Bump> b(static_cast<std::size_t>(count));
  for (auto& x : b) {
    for (int a = 0; a < dims; ++a) x.c[static_cast<std::size_t>(a)] = g.uniform_open();
    x.w = 0.05 + 0.15 * g.uniform();
    x.amp = g.normal();
  }
  return b;
}

inline Field bump_field(std::vector<Bump> bumps, int dims) {
  return [bumps = std::move(bumps), dims](const Coord& x) {
    double s = 0.0;
    for (const Bump& b : bumps) {
      double r2 = 0.0;
      for (int a = 0; a < dims; ++a) {
        const double d = x[static_cast<std::size_t>(a)] - b.c[static_cast<std::size_t>(a)];
        r2 += d * d;
      }
      s += b.amp * std::exp(-r2 / (2.0 * b.w * b.w));
    }
    return s;
  };
}

inline Field constant(double v) {
  return [v](const Coord&) { return v; };
}

inline void set_constant_coeffs(Problem& p, std::array<double, 3> a, std::array<double, 3> b) {
  p.constant_coeffs = true;
  p.alpha_c = a;
  p.beta_c = b;
  for (int i = 0; i < p.spatial_axes(); ++i) {
    p.alpha[static_cast<std::size_t>(i)] = constant(a[static_cast<std::size_t>(i)]);
    p.beta[static_cast<std::size_t>(i)] = constant(b[static_cast<std::size_t>(i)]);
  }
}

// ---- reference examples (proj/src/problems.cpp:13-141, restated) ---------------------------
inline Problem reference_example(int example, int setting) {
  constexpr double kPi = M_PI;
  if (setting != 1 && setting != 2) throw std::invalid_argument("setting must be 1 or 2");
  Problem p;
  const auto plane2 = [&] {  // problems.cpp:13-25
    p.dim = 2;
    set_constant_coeffs(p, {1, 1, 0}, {1, 1, 0});
    p.exact = [](const Coord& x) { return std::sin(kPi * x[0] + kPi * x[1]); };
    p.source = [](const Coord& x) {
      const double th = kPi * x[0] + kPi * x[1];
      return 2.0 * kPi * kPi * std::sin(th) + 2.0 * kPi * std::cos(th);
    };
  };
  const auto plane1t = [&] {  // problems.cpp:45-58
    p.dim = 2;
    p.time_dependent = true;
    set_constant_coeffs(p, {1, 0, 0}, {1, 0, 0});
    p.exact = [](const Coord& x) { return std::sin(kPi * x[0] + kPi * x[1]); };
    p.source = [](const Coord& x) {
      const double th = kPi * (x[0] + x[1]);
      return kPi * kPi * std::sin(th) + 2.0 * kPi * std::cos(th);
    };
  };
  switch (example) {
    case 1:
    case 2:
      if (example == 1 && setting == 2) {  // problems.cpp:27-43
        p.dim = 2;
        p.constant_coeffs = false;
        p.alpha[0] = [](const Coord& x) { return 1.0 + x[0] * x[0]; };
        p.alpha[1] = [](const Coord& x) { return 2.0 + x[0] * x[1]; };
        p.beta[0] = [](const Coord& x) { return 2.0 - x[0]; };
        p.beta[1] = [](const Coord& x) { return 1.0 + x[1]; };
        p.exact = [](const Coord& x) { return std::sin(4.0 * kPi * x[0] + 4.0 * kPi * x[1]); };
        p.source = [](const Coord& x) {
          const double th = 4.0 * kPi * (x[0] + x[1]);
          const double a = 3.0 + x[0] * x[0] + x[0] * x[1];
          const double b = 3.0 - x[0] + x[1];
          return 16.0 * kPi * kPi * a * std::sin(th) + 4.0 * kPi * b * std::cos(th);
        };
      } else if (example == 2 && setting == 2) {
        plane1t();
      } else {
        plane2();
      }
      break;
    case 3:
      if (setting == 1) {
        plane1t();
      } else {  // problems.cpp:60-75
        p.dim = 2;
        p.time_dependent = true;
        p.constant_coeffs = false;
        p.alpha[0] = [](const Coord& x) { return 1.0 + x[0] * x[0]; };
        p.beta[0] = [](const Coord& x) { return 2.0 - x[0]; };
        p.exact = [](const Coord& x) { return std::sin(4.0 * kPi * x[0] + 4.0 * kPi * x[1]); };
        p.source = [](const Coord& x) {
          const double th = 4.0 * kPi * (x[0] + x[1]);
          return 16.0 * kPi * kPi * (1.0 + x[0] * x[0]) * std::sin(th) +
                 4.0 * kPi * (3.0 - x[0]) * std::cos(th);
        };
      }
      break;
    case 4:
      p.dim = 3;
      if (setting == 1) {  // problems.cpp:77-89
        set_constant_coeffs(p, {1, 1, 1}, {1, 1, 1});
        p.exact = [](const Coord& x) { return std::sin(kPi * (x[0] + x[1] + x[2])); };
        p.source = [](const Coord& x) {
          const double th = kPi * (x[0] + x[1] + x[2]);
          return 3.0 * kPi * kPi * std::sin(th) + 3.0 * kPi * std::cos(th);
        };
      } else {  // problems.cpp:91-110
        p.constant_coeffs = false;
        p.alpha[0] = [](const Coord& x) { return 1.0 + x[0] * x[0]; };
        p.alpha[1] = [](const Coord& x) { return 2.0 + x[0] * x[1]; };
        p.alpha[2] = [](const Coord& x) { return 3.0 - x[0] * x[1] * x[2]; };
        p.beta[0] = [](const Coord& x) { return 2.0 - x[0]; };
        p.beta[1] = [](const Coord& x) { return 1.0 + x[1]; };
        p.beta[2] = [](const Coord& x) { return 2.0 - x[0] + x[1] * x[2]; };
        p.exact = [](const Coord& x) { return std::sin(4.0 * kPi * (x[0] + x[1] + x[2])); };
        p.source = [](const Coord& x) {
          const double th = 4.0 * kPi * (x[0] + x[1] + x[2]);
          const double a = 6.0 + x[0] * x[0] + x[0] * x[1] - x[0] * x[1] * x[2];
          const double b = 5.0 - 2.0 * x[0] + x[1] + x[1] * x[2];
          return 16.0 * kPi * kPi * a * std::sin(th) + 4.0 * kPi * b * std::cos(th);
        };
      }
      break;
    default:
      throw std::invalid_argument("example must be 1..4");
  }
  p.boundary = p.exact;
  return p;
}

// ---- BASELINE.json configs -----------------------------------------------------------------
// Mesh choice (documented in DESIGN.md): the coarse interior count is the reference CLI's
// default --nc 9 (proj/README.md "--nc INT [9]"), and the fine interior count is the value
// nearest the config's N (ties upward) that satisfies the reference's divisibility rule
// (N_f + 1) = n (N_c + 1) (proj/src/mesh.cpp:63-68).
inline int admissible_nf(int n_target, int nc) {
  const int q = nc + 1;
  const int lo = ((n_target + 1) / q) * q - 1;  // largest admissible <= target (if >= target-..)
  const int hi = lo + q;
  const int best = (n_target - lo) < (hi - n_target) ? lo : hi;
  return best;
}

constexpr int kNumBaselineConfigs = 5;

inline MeshChoice baseline_mesh(int id) {
  MeshChoice m;
  const int nc = 9;
  int n = 0;
  switch (id) {
    case 0: m.dim = 2; n = 128; m.iterations = 10; break;
    case 1: m.dim = 2; n = 1024; m.iterations = 20; break;
    case 2: m.dim = 2; n = 4096; m.iterations = 20; break;
    case 3: m.dim = 3; n = 256; m.iterations = 10; break;
    case 4: m.dim = 3; n = 512; m.iterations = 10; m.time_axis = 2; break;
    default: throw std::invalid_argument("baseline config id must be 0..4");
  }
  for (int a = 0; a < m.dim; ++a) {
    m.nf[static_cast<std::size_t>(a)] = admissible_nf(n, nc);
    m.nc[static_cast<std::size_t>(a)] = nc;
  }
  return m;
}

inline Problem baseline_problem(int id, std::uint64_t seed) {
  constexpr double kPi = M_PI;
  Problem p;
  switch (id) {
    case 0: {  // 2D steady, alpha=(1,1), beta=(1,1), u = sin(pi x) sin(pi y)
      p.dim = 2;
      const double a0 = 1, a1 = 1, b0 = 1, b1 = 1;
      set_constant_coeffs(p, {a0, a1, 0}, {b0, b1, 0});
      p.exact = [](const Coord& x) { return std::sin(kPi * x[0]) * std::sin(kPi * x[1]); };
      p.source = [=](const Coord& x) {
        const double sx = std::sin(kPi * x[0]), sy = std::sin(kPi * x[1]);
        const double cx = std::cos(kPi * x[0]), cy = std::cos(kPi * x[1]);
        return (a0 + a1) * kPi * kPi * sx * sy + b0 * kPi * cx * sy + b1 * kPi * sx * cy;
      };
      p.boundary = p.exact;
      break;
    }
    case 1: {  // 2D steady, alpha=(0.1,0.1), beta=(1,-0.5), g = 0, 8 bumps
      p.dim = 2;
      set_constant_coeffs(p, {0.1, 0.1, 0}, {1.0, -0.5, 0});
      p.source = bump_field(draw_bumps(8, 2, seed), 2);
      p.boundary = constant(0.0);
      break;
    }
    case 2: {  // 2D advection-dominated, alpha=(0.01,0.01), beta=(1,1), 16 bumps, g = 0.1 sin cos
      p.dim = 2;
      set_constant_coeffs(p, {0.01, 0.01, 0}, {1.0, 1.0, 0});
      p.source = bump_field(draw_bumps(16, 2, seed), 2);
      p.boundary = [](const Coord& x) {
        return 0.1 * std::sin(2.0 * kPi * x[0]) * std::cos(2.0 * kPi * x[1]);
      };
      break;
    }
    case 3: {  // 3D steady, alpha=1, beta=0.5, u = sin sin sin
      p.dim = 3;
      const double a = 1.0, b = 0.5;
      set_constant_coeffs(p, {a, a, a}, {b, b, b});
      p.exact = [](const Coord& x) {
        return std::sin(kPi * x[0]) * std::sin(kPi * x[1]) * std::sin(kPi * x[2]);
      };
      p.source = [=](const Coord& x) {
        const double sx = std::sin(kPi * x[0]), sy = std::sin(kPi * x[1]), sz = std::sin(kPi * x[2]);
        const double cx = std::cos(kPi * x[0]), cy = std::cos(kPi * x[1]), cz = std::cos(kPi * x[2]);
        return 3.0 * a * kPi * kPi * sx * sy * sz + b * kPi * (cx * sy * sz + sx * cy * sz + sx * sy * cz);
      };
      p.boundary = p.exact;
      break;
    }
    case 4: {  // 2D + time as a 3D space-time grid, alpha=(0.5,0.5), beta=(1,0), 8 bumps in (x,y,t)
      p.dim = 3;
      p.time_dependent = true;
      set_constant_coeffs(p, {0.5, 0.5, 0}, {1.0, 0.0, 0});
      p.source = bump_field(draw_bumps(8, 3, seed), 3);
      p.boundary = constant(0.0);
      break;
    }
    default:
      throw std::invalid_argument("baseline config id must be 0..4");
  }
  return p;
}

}  // namespace asdsm_cat

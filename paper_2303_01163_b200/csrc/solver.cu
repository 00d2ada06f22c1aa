#include <cstdio>
#include <cxxabi.h>
#include <map>
// Host orchestration of one ASDSM solve on the device (proj/src/solver.cpp:486-680 restated
// for a device-resident state).  All per-iteration decisions (normalization guard, step
// clamp, accept/revert, stop rules) happen in ctrl kernels, so a whole solve is enqueued
// without host synchronization and can be captured in a CUDA graph.
#include "solver.hpp"

#include <cublas_v2.h>

#include "dmma_gemm.cuh"
#include "holes2d.cuh"
#include "holes3d.cuh"
#include "slab2d.cuh"
#include "slabstep2d.cuh"
#include "march.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>

namespace asdsm_b200 {

static void record_graph_kernels(cudaGraph_t g, std::vector<std::pair<std::string, int>>& out);


std::uint64_t mix_seed(std::uint64_t base, std::uint64_t k) {
  std::uint64_t z = base + 0x9E3779B97F4A7C15ull * (k + 1);
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

Solver::Solver(const Mesh& m, const double* alpha, const double* beta) : mesh_(m) {
  for (int a = 0; a < 3; ++a) {
    alpha_[a] = alpha[a];
    beta_[a] = beta[a];
  }
  init(nullptr);
}

Solver::Solver(const Mesh& m, const asdsm_cat::Problem& problem) : mesh_(m) {
  if (problem.dim != m.dim) throw AsdsmError(kDimensionMismatch, "problem/mesh dimension mismatch");
  if (problem.time_dependent != (m.time_axis >= 0))
    throw AsdsmError(kDimensionMismatch, "problem and mesh disagree about a time axis");
  if (problem.constant_coeffs) {
    for (int a = 0; a < 3; ++a) {
      alpha_[a] = problem.alpha_c[static_cast<size_t>(a)];
      beta_[a] = problem.beta_c[static_cast<size_t>(a)];
    }
    init(nullptr);
    return;
  }
  for (int a = 0; a < 3; ++a) {  // stencil structure only (has_right, time axis); values per point
    alpha_[a] = 1.0;
    beta_[a] = 0.0;
  }
  init(&problem);
}

void Solver::init(const asdsm_cat::Problem* varprob) {
  const Mesh& m = mesh_;
  variable_ = varprob != nullptr;
  md_.dim = m.dim;
  for (int a = 0; a < 3; ++a) {
    md_.nf[a] = a < m.dim ? m.nf[a] : 1;
    md_.nc[a] = a < m.dim ? m.nc[a] : 1;
    md_.n[a] = a < m.dim ? m.n[a] : 1;
    md_.h[a] = a < m.dim ? m.h[a] : 0.0;
  }
  const unsigned full = (1u << m.dim) - 1u;
  g_fine_ = kind_geom(m, 0u);
  g_coarse_ = kind_geom(m, full);
  fg_.dim = m.dim;
  for (int a = 0; a < 3; ++a) {
    fg_.ext[a] = g_fine_.ext[a];
    fg_.stride[a] = g_fine_.stride[a];
  }
  fg_.size = g_fine_.size;
  st_fine_ = make_stencil(m, 0u, alpha_, beta_);
  st_coarse_ = make_stencil(m, full, alpha_, beta_);
  for (int a = 0; a < m.dim; ++a) {
    g_slab_[a] = kind_geom(m, 1u << a);
    st_slab_[a] = make_stencil(m, 1u << a, alpha_, beta_);
  }
  cell_ = 1.0;
  for (int a = 0; a < m.dim; ++a) cell_ *= m.h[a];

  // Separable solvers: slabs (one box each), coarse box, hole boxes (all congruent).
  const int tax = m.time_axis;
  int hext[3] = {1, 1, 1};
  i64 nholes = 1;
  for (int a = 0; a < m.dim; ++a) {
    hext[a] = m.n[a] - 1;
    nholes *= m.nc[a] + 1;
  }
  if (!variable_) {
    try {
      for (int a = 0; a < m.dim; ++a)
        sep_slab_[a] = build_sep_solver(dev_, m.dim, g_slab_[a].ext, st_slab_[a], tax, -1, 1, "slab " + std::to_string(a));
      sep_coarse_ = build_sep_solver(dev_, m.dim, g_coarse_.ext, st_coarse_, tax, -1, 1, "coarse mesh");
      // 3D holes that fit the one-kernel fill (m <= 64 on the transform axes) need the Thomas
      // pivot tables whatever the hole count (the fused kernel runs its own line solves), so the
      // few-lines PCR choice is not taken for them
      const bool fused3d_candidate = m.dim == 3 && hext[0] <= 64 && hext[1] <= 64;
      sep_hole_ = build_sep_solver(dev_, m.dim, hext, st_fine_, tax, -1,
                                   fused3d_candidate ? std::max<i64>(nholes, 1 << 20) : nholes, "hole block", m.dim == 2);
    } catch (const AsdsmError& e) {
      if (e.code != kUnsupported || std::getenv("ASDSM_NO_SEPARABLE_FALLBACK")) throw;
      dev_.release_all();
      for (auto& S : sep_slab_) S = SepSolver{};
      sep_coarse_ = SepSolver{};
      sep_hole_ = SepSolver{};
      const_fields_ = asdsm_cat::Problem{};
      const_fields_.dim = m.dim;
      const_fields_.time_dependent = m.time_axis >= 0;
      const_fields_.constant_coeffs = false;
      for (int a = 0; a < 3; ++a) {
        const double al = alpha_[a], be = beta_[a];
        const_fields_.alpha[static_cast<size_t>(a)] = [al](const asdsm_cat::Coord&) { return al; };
        const_fields_.beta[static_cast<size_t>(a)] = [be](const asdsm_cat::Coord&) { return be; };
      }
      separable_fallback_ = true;
      init(&const_fields_);
      return;
    }
  } else {
    // per-point stencils (fdm.cpp:63-126 sampling) + block-Thomas factors for every box
    const std::vector<double> cf = sample_kind_coefficients(m, 0u, *varprob);
    coef_fine_ = dev_.alloc<double>(cf.size());
    ASDSM_CUDA_CHECK(cudaMemcpy(coef_fine_, cf.data(), cf.size() * sizeof(double), cudaMemcpyHostToDevice));
    auto upload_bt = [&](const BlockThomas& b, BTDev& d) {
      d.dim = b.dim;
      d.L = b.L;
      d.B = b.B;
      d.nb = b.nb;
      for (int a = 0; a < 3; ++a) d.ext[a] = b.ext[a];
      double* p0 = dev_.alloc<double>(b.dinv.size());
      double* p1 = dev_.alloc<double>(b.lo.size());
      double* p2 = dev_.alloc<double>(b.up.size());
      ASDSM_CUDA_CHECK(cudaMemcpy(p0, b.dinv.data(), b.dinv.size() * sizeof(double), cudaMemcpyHostToDevice));
      ASDSM_CUDA_CHECK(cudaMemcpy(p1, b.lo.data(), b.lo.size() * sizeof(double), cudaMemcpyHostToDevice));
      ASDSM_CUDA_CHECK(cudaMemcpy(p2, b.up.data(), b.up.size() * sizeof(double), cudaMemcpyHostToDevice));
      d.dinv = p0;
      d.lo = p1;
      d.up = p2;
    };
    for (int a = 0; a < m.dim; ++a)
      upload_bt(factor_kind_box(m, 1u << a, sample_kind_coefficients(m, 1u << a, *varprob), tax), bt_[a]);
    const unsigned full_mask = (1u << m.dim) - 1u;
    upload_bt(factor_kind_box(m, full_mask, sample_kind_coefficients(m, full_mask, *varprob), tax), bt_[3]);
    upload_bt(factor_hole_boxes(m, cf), bt_[4]);
  }

  const i64 nf = g_fine_.size;
  // fine arrays carry one grid row of slack: the 3D pass's pair-row tensor maps (stream3d.cu)
  // address whole row pairs, and the last pair's odd row lies past the array when N_y N_z is odd
  const size_t nfa = static_cast<size_t>(nf) + static_cast<size_t>(m.nf[0]) + 2;
  for (int i = 0; i < 2; ++i) {
    u_[i] = dev_.alloc<double>(nfa);
    r_[i] = dev_.alloc<double>(nfa);
  }
  b_ = dev_.alloc<double>(nfa);
  e_ = dev_.alloc<double>(nfa);
  exact_ = dev_.alloc<double>(nfa);
  size_t scratch = variable_ ? 16 : sep_scratch_bytes(sep_hole_, nholes);
  for (int a = 0; a < m.dim; ++a) {
    const size_t n = static_cast<size_t>(g_slab_[a].size);
    b_slab_[a] = dev_.alloc<double>(n);
    rhs_slab_[a] = dev_.alloc<double>(n);
    sol_slab_[a] = dev_.alloc<double>(n);
    if (!variable_) scratch = std::max(scratch, sep_scratch_bytes(sep_slab_[a], 1));
  }
  if (!variable_) scratch = std::max(scratch, sep_scratch_bytes(sep_coarse_, 1));
  scratch0_ = dev_.alloc<unsigned char>(scratch);
  scratch1_ = dev_.alloc<unsigned char>(scratch);
  if (m.dim == 2 && !variable_ && sep_hole_.part)  // per-hole ring of the partitioned hole solve
    hole_ring_ = dev_.alloc<double>(static_cast<size_t>(nholes) * 2 * (sep_hole_.ext[0] + sep_hole_.ext[1]));
  if (hole_ring_ && !sep_hole_.complex_modes && sep_hole_.nd == 1 && sep_hole_.L == 1 && sep_hole_.dax[0] == 0 &&
      !sep_hole_.use_pcr && !hole2d_fused_fits(sep_hole_.ext[0], sep_hole_.ext[1])) {
    // strip split of the large holes: the fewest strips (p | m0 + 1) of at most kStripMaxW
    // columns; ASDSM_STRIPS=p overrides (0: off)
    constexpr int kStripMaxW = 96;
    const int n0 = sep_hole_.ext[0] + 1;
    int p = 0;
    // (the separator kernel keeps p - 1 rows of V and its k-group partials in 48 KB)
    auto fits = [&](int q) {
      return q >= 2 && q <= 10 && n0 % q == 0 && (q - 1) * (n0 - 1 + (q <= 5 ? 512 : 256)) * 8 <= 48 * 1024;
    };
    if (const char* env = std::getenv("ASDSM_STRIPS")) {
      p = std::atoi(env);
      if (!fits(p)) p = 0;
    } else {
      for (int q = 2; q <= 10 && !p; ++q)
        if (fits(q) && n0 / q - 1 <= kStripMaxW) p = q;
    }
    if (p) {
      int sext[3] = {n0 / p - 1, sep_hole_.ext[1], 1};
      sep_strip_ = build_sep_solver(dev_, 2, sext, st_fine_, tax, -1, nholes * p, "hole strip", true);
      if (!sep_strip_.complex_modes && sep_strip_.nd == 1 && sep_strip_.L == 1 && sep_strip_.dax[0] == 0 &&
          !sep_strip_.use_pcr && sep_strip_.part && hole2d_part_supported(sep_strip_.part_seg)) {
        strip_p_ = p;
        strip_ring_ = dev_.alloc<double>(static_cast<size_t>(nholes) * p * 2 * (sext[0] + sext[1]));
      }
    }
  }
  if (m.dim == 3 && !variable_) {
    // the three slab solves of an iteration are independent: slabs 1 and 2 run on their own
    // streams (forked / joined with events, captured into the graph as parallel branches),
    // each with its own mode-space scratch
    for (int a = 1; a < 3; ++a) {
      const size_t sa = sep_scratch_bytes(sep_slab_[a], 1);
      slab_scr_[a][0] = dev_.alloc<unsigned char>(sa);
      slab_scr_[a][1] = dev_.alloc<unsigned char>(sa);
      ASDSM_CUDA_CHECK(cudaStreamCreateWithFlags(&aux_[a - 1], cudaStreamNonBlocking));
    }
    for (int i = 0; i < 3; ++i) ASDSM_CUDA_CHECK(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming));
  }
  b_coarse_ = dev_.alloc<double>(static_cast<size_t>(g_coarse_.size));
  u_cc_ = dev_.alloc<double>(static_cast<size_t>(g_coarse_.size));
  cc_e1_ = dev_.alloc<double>(static_cast<size_t>(g_coarse_.size));
  cc_e2_ = dev_.alloc<double>(static_cast<size_t>(g_coarse_.size));
  int maxnc = 0;
  for (int a = 0; a < m.dim; ++a) maxnc = std::max(maxnc, m.nc[a]);
  const size_t nlines = static_cast<size_t>(m.nc[0] + m.nc[1] + (m.dim == 3 ? m.nc[2] : 0));
  spl_m1_ = dev_.alloc<double>(static_cast<size_t>(m.nc[1]) * (m.nc[0] + 2) + 16);
  spl_m2_ = dev_.alloc<double>(static_cast<size_t>(m.nc[0]) * (m.nc[1] + 2) + nlines * 4 * (maxnc + 2) + 16);
  if (m.dim == 3) {
    m3_.m = md_;
    const size_t ntr = static_cast<size_t>(g_coarse_.size);
    m3_.u_hat = dev_.alloc<double>(ntr);
    int p = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = a + 1; b < 3; ++b, ++p) {
        const int f = 3 - a - b;
        m3_.corr[p] = dev_.alloc<double>(ntr);
        m3_.mP[p] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nc[b] * (m.nc[f] + 2));
        m3_.T[p] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nc[b] * m.nf[f]);
      }
    for (int a = 0; a < 3; ++a) {
      const int f1 = (a == 0) ? 1 : 0, f2 = (a == 2) ? 1 : 2;
      m3_.mF1[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[f2] * (m.nc[f1] + 2));
      m3_.mF2[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[f1] * (m.nc[f2] + 2));
      m3_.mF3a[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nc[f2] * (m.nc[f1] + 2));
      m3_.mF3b[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[f1] * (m.nc[f2] + 2));
      m3_.g3[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[f1] * (m.nc[f2] + 2));
      m3_.corrected[a] = dev_.alloc<double>(static_cast<size_t>(g_slab_[a].size));
      m3_.sF1[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[f2] * 4 * (m.nc[f1] + 1));
      m3_.sF2[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[f1] * 4 * (m.nc[f2] + 1));
      m3_.sF3a[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nc[f2] * 4 * (m.nc[f1] + 1));
      m3_.sF3b[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[f1] * 4 * (m.nc[f2] + 1));
    }
  }
  partials_ = dev_.alloc<double>(4 * static_cast<size_t>(kRedStride));
  if (m.dim == 3 && !variable_) {  // 3D fused fill buffers (allocated here: never during graph capture)
    Hole3DArgs A{};
    for (int a = 0; a < 3; ++a) A.m[a] = m.n[a] - 1;
    faces3d_ = dev_.alloc<double>(static_cast<size_t>(nholes) * hole3d_face_doubles(A));
    hole3d_prepare(A);
    // one-kernel fill: padded copies of the hole solver's eigenvector tables
    const SepSolver& H = sep_hole_;
    if (!H.complex_modes && H.nd == 2 && H.L == 2 && H.dax[0] == 0 && H.dax[1] == 1 && !H.use_pcr) {
      Hole3DFusedArgs F{};
      for (int a = 0; a < 3; ++a) {
        F.m[a] = H.ext[a];
        F.n[a] = m.n[a];
        F.nf[a] = m.nf[a];
        F.nbox[a] = m.nc[a] + 1;
      }
      h3f_causal_ = H.line_right == 0.0;
      if (hole3d_fused_plan(F, h3f_causal_)) {
        for (int a = 0; a < 2; ++a) {
          const int mm = F.m[a];
          std::vector<double> half(static_cast<size_t>(half_sine_rows(mm)) * 2 * half_sine_kh(mm) + 2 * mm);
          ASDSM_CUDA_CHECK(cudaMemcpy(half.data(), H.half[a], half.size() * sizeof(double), cudaMemcpyDeviceToHost));
          const std::vector<double> t = hole3d_half_table(a == 0 ? F.ax : F.ay, half);
          double* d = dev_.alloc<double>(t.size());
          ASDSM_CUDA_CHECK(cudaMemcpy(d, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice));
          (a == 0 ? F.Hx : F.Hy) = d;
        }
        F.st = st_fine_;
        F.ipiv = H.th_ipiv;
        F.cp = H.th_cp;
        F.line_left = H.line_left;
        hole3d_fused_prepare();
        h3f_ = F;
        h3f_ok_ = true;
      }
    }
  }
  state_ = dev_.alloc<DevState>(1);
  sep_prepare();
  dmma_prepare();
  if (!variable_ && m.dim == 2 && m.nc[0] <= 22 && m.nc[1] <= 22 && std::getenv("ASDSM_GENERIC_FILL") == nullptr) {
    fast2d_ = true;
    for (int a = 0; a < 2; ++a) {
      const SepSolver& S = sep_slab_[a];
      fast2d_ = fast2d_ && S.use_pcr && S.nd == 1 && S.dax[0] == a && S.L == 1 - a &&
                S.complex_modes == sep_slab_[0].complex_modes;
    }
    if (fast2d_) {
      slab2d_prepare();
      for (int a = 0; a < 2; ++a) {
        slab_modes_[a] = dev_.alloc<double>(static_cast<size_t>(m.nc[a]) * m.nf[1 - a] * 2);
        const std::vector<double> tab = spline_axis_table(m.nc[a], m.n[a], m.h[a]);
        sp_tab_[a] = dev_.alloc<double>(tab.size());
        ASDSM_CUDA_CHECK(cudaMemcpy(sp_tab_[a], tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
        const std::vector<double> bas = spline_basis_table(m.nc[a], m.n[a], m.h[a], m.nf[a]);
        sp_basis_[a] = dev_.alloc<double>(bas.size());
        ASDSM_CUDA_CHECK(cudaMemcpy(sp_basis_[a], bas.data(), bas.size() * sizeof(double), cudaMemcpyHostToDevice));
      }
      for (int b = 0; b < 2; ++b)  // residual on the slab stations, one copy per residual buffer
        stations_[b] = dev_.alloc<double>(static_cast<size_t>(m.nc[0]) * m.nf[1] + static_cast<size_t>(m.nc[1]) * m.nf[0]);
      seg1_ = dev_.alloc<double>(static_cast<size_t>(m.nc[1]) * 4 * (m.nc[0] + 1));
      step2d_ = std::getenv("ASDSM_NO_SLABSTEP") == nullptr && std::getenv("ASDSM_HOLE_UNFUSED") == nullptr &&
                slabstep2d_supported(md_, sep_slab_) && !sep_hole_.complex_modes && sep_hole_.nd == 1 &&
                sep_hole_.L == 1 && !sep_hole_.use_pcr && hole2d_fused_fits(sep_hole_.ext[0], sep_hole_.ext[1]);
      skel_line_[0] = dev_.alloc<double>(static_cast<size_t>(m.nc[0]) * m.nf[1]);
      skel_line_[1] = dev_.alloc<double>(static_cast<size_t>(m.nc[1]) * m.nf[0]);
      skel_corr_ = dev_.alloc<double>(2 * static_cast<size_t>(m.nc[0]) * m.nc[1]);
      if (step2d_) {
        slabstep2d_prepare();
        step2d_ = slabstep2d_launchable(slabstep2d_args(nullptr, nullptr));
      }
      seg2_ = dev_.alloc<double>(static_cast<size_t>(m.nc[0]) * 4 * (m.nc[1] + 1));
    }
  }
  ASDSM_CUDA_CHECK(cudaMemset(exact_, 0, sizeof(double) * static_cast<size_t>(nf)));
  if (strip_p_ && std::getenv("ASDSM_SEP_MODES") == nullptr) build_separator_matrix();
  dots_update_ok_ = !variable_ && mesh_.dim == 2 && std::getenv("ASDSM_DOTS_UPDATE") != nullptr &&
                    dots_update_supported(fg_);
}

BoxArray Solver::hole_array(double* p) const {
  BoxArray b;
  b.ptr = p;
  for (int a = 0; a < 3; ++a) {
    b.stride[a] = g_fine_.stride[a];
    b.nbox[a] = a < mesh_.dim ? mesh_.nc[a] + 1 : 1;
    b.box_stride[a] = a < mesh_.dim ? static_cast<i64>(mesh_.n[a]) * g_fine_.stride[a] : 0;
  }
  return b;
}

BoxArray Solver::kind_array(const KindGeom& g, double* p) const {
  BoxArray b;
  b.ptr = p;
  for (int a = 0; a < 3; ++a) {
    b.stride[a] = g.stride[a];
    b.nbox[a] = 1;
    b.box_stride[a] = 0;
  }
  return b;
}

void Solver::set_bundle(const double* b_fine, const double* const* b_slab, const double* b_coarse,
                        const double* exact, bool on_device, cudaStream_t s) {
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const size_t nf = static_cast<size_t>(g_fine_.size) * sizeof(double);
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(b_, b_fine, nf, kind, s));
  for (int a = 0; a < mesh_.dim; ++a)
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(b_slab_[a], b_slab[a], static_cast<size_t>(g_slab_[a].size) * sizeof(double), kind, s));
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(b_coarse_, b_coarse, static_cast<size_t>(g_coarse_.size) * sizeof(double), kind, s));
  has_exact_ = exact != nullptr;
  if (exact) ASDSM_CUDA_CHECK(cudaMemcpyAsync(exact_, exact, nf, kind, s));
}

// The separator response matrix K of the strip split: column c is the solution on the p - 1
// separator columns of one hole for the ring right-hand side e_c (holes2d ring layout fL fR fB
// fT).  Built with the iteration's own kernels -- the mode lines of `nholes` virtual holes with
// unit rings per batch, then the separator product in its dense-output form -- so K carries
// exactly the arithmetic of the per-iteration separator path it replaces.
void Solver::build_separator_matrix() {
  const SepSolver& H = sep_hole_;
  const int m0 = H.ext[0], m1 = H.ext[1];
  const i64 nholes = static_cast<i64>(mesh_.nc[0] + 1) * (mesh_.nc[1] + 1);
  sep_rows_ = (strip_p_ - 1) * m1;
  sep_cols_ = 2 * m1 + 2 * m0;
  const i64 batches = (sep_cols_ + nholes - 1) / nholes;
  sep_K_ = dev_.alloc<double>(static_cast<size_t>(batches * nholes) * sep_rows_);
  sep_C_ = dev_.alloc<double>(static_cast<size_t>(nholes) * sep_rows_);
  Hole2DArgs A{};
  A.m0 = m0;
  A.m1 = m1;
  A.n0 = mesh_.n[0];
  A.n1 = mesh_.n[1];
  A.nf0 = mesh_.nf[0];
  A.nf1 = mesh_.nf[1];
  A.nbox0 = mesh_.nc[0] + 1;
  A.nbox1 = mesh_.nc[1] + 1;
  A.st = st_fine_;
  A.line_left = H.line_left;
  A.line_right = H.line_right;
  const Hole2DPartArgs P{H.W[0], H.part, H.part_stride, H.part_seg, H.part_P, H.part_last, hole_ring_};
  double* modes = static_cast<double*>(scratch0_);
  hole2d_prepare(113 * 1024);  // kernel attributes (dynamic shared memory) of the hole kernels
  std::vector<double> unit(static_cast<size_t>(nholes) * sep_cols_);
  cudaStream_t s = nullptr;
  launch_state_init(state_, 1, 1, s);
  for (i64 b = 0; b < batches; ++b) {
    std::fill(unit.begin(), unit.end(), 0.0);
    for (i64 h = 0; h < nholes && b * nholes + h < sep_cols_; ++h) unit[static_cast<size_t>(h * sep_cols_ + b * nholes + h)] = 1.0;
    ASDSM_CUDA_CHECK(cudaMemcpy(hole_ring_, unit.data(), unit.size() * sizeof(double), cudaMemcpyHostToDevice));
    launch_hole2d_part(modes, A, P, state_, s);
    launch_hole2d_sep_rows(modes, H.V[0], nullptr, A, strip_p_, state_, s, sep_K_ + b * nholes * sep_rows_);
  }
  ASDSM_CUDA_CHECK(cudaDeviceSynchronize());
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasCreate failed");
  blas_ = h;
  const size_t ws = 32u << 20;
  ASDSM_CUDA_CHECK(cudaMalloc(&blas_ws_, ws));
  if (cublasSetWorkspace(h, blas_ws_, ws) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetWorkspace failed");
}

Solver::~Solver() {
  if (blas_) cublasDestroy(static_cast<cublasHandle_t>(blas_));
  if (blas_ws_) cudaFree(blas_ws_);
  if (host_state_) cudaFreeHost(host_state_);
  if (host_hist_) cudaFreeHost(host_hist_);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  for (cudaStream_t& q : aux_)
    if (q) cudaStreamDestroy(q);
  for (cudaEvent_t& e : ev_)
    if (e) cudaEventDestroy(e);
}

void Solver::reset_state(const RunOptions& o, cudaStream_t s) {
  launch_state_init(state_, 1, 1, s);
  // stop_at from ||b||_2 (solver.cpp:570-571)
  CtrlArgs c{};
  c.op = kCtrlInit;
  c.tol = o.tol;
  launch_norm_sq(b_, g_fine_.size, partials_, state_, s, &c, history_);
}

Skel2DArgs Solver::skel2d_args(const double* const* sol, const double* u_cc, const int* coin, double* out) {
  Skel2DArgs a{};
  a.m = md_;
  a.u_fc = sol[1];
  a.u_cf = sol[0];
  a.u_cc = u_cc;
  a.coin = coin;
  a.e1 = cc_e1_;
  a.e2 = cc_e2_;
  a.m1 = spl_m1_;
  a.m2 = spl_m2_;
  a.out = out;
  if (coin != nullptr) {  // error mode: normalized on the fly (values / norm, as normalize_or_throw)
    a.norm_fc = &state_->slab_norm[1];
    a.norm_cf = &state_->slab_norm[0];
  }
  a.sp_tab[0] = sp_tab_[0];
  a.sp_tab[1] = sp_tab_[1];
  a.seg1 = seg1_;
  a.seg2 = seg2_;
  return a;
}

SlabStep2DArgs Solver::slabstep2d_args(const int* coin, double* out) const {
  SlabStep2DArgs A{};
  A.m = md_;
  for (int a = 0; a < 2; ++a) {
    const SepSolver& S = sep_slab_[a];
    A.W[a] = S.W[a];
    A.V[a] = S.V[a];
    A.part[a] = S.part;
    A.pseg[a] = S.part_seg;
    A.pP[a] = S.part_P;
    A.plast[a] = S.part_last;
    A.pstride[a] = S.part_stride;
    A.line_l[a] = S.line_left;
    A.line_r[a] = S.line_right;
  }
  A.sta0 = stations_[0];
  A.sta1 = stations_[1];
  A.coin = coin;
  A.out = out;
  A.skel_line0 = skel_line_[0];
  A.skel_line1 = skel_line_[1];
  A.corr = skel_corr_;
  return A;
}

void Solver::skeleton(const double* const* sol, const double* u_cc, const int* coin, double* out, cudaStream_t s) {
  if (mesh_.dim == 3) {
    Merge3DArgs A = m3_;
    for (int a = 0; a < 3; ++a) A.u[a] = sol[a];
    A.u_ccc = u_cc;
    A.coin = coin;
    launch_merge3d(A, out, state_, s);
    return;
  }
  Skel2DArgs a{};
  a.m = md_;
  a.u_fc = sol[1];
  a.u_cf = sol[0];
  a.u_cc = u_cc;
  a.coin = coin;
  a.e1 = cc_e1_;
  a.e2 = cc_e2_;
  a.m1 = spl_m1_;
  a.m2 = spl_m2_;
  a.out = out;
  if (fast2d_) {
    const Skel2DArgs f = skel2d_args(sol, u_cc, coin, out);
    launch_skel2d_ccspline_fast(f, state_, s);
    launch_skel2d_write_fast(f, state_, s);
    return;
  }
  launch_skeleton2d(a, state_, s);
}

void Solver::march_launch(int mode, MarchArgs A, cudaStream_t s) {
  A.coef = coef_fine_;
  if (A.skel_only) {
    for (int a = 0; a < mesh_.dim; ++a) {
      A.nc[a] = mesh_.nc[a];
      A.n[a] = mesh_.n[a];
    }
  }
  A.sta0 = A.sta1 = nullptr;
  if (fast2d_ && mode != kMarchDots && A.ro0 == r_[0] && A.ro1 == r_[1]) {
    A.sta0 = stations_[0];
    A.sta1 = stations_[1];
    for (int a = 0; a < 2; ++a) {
      A.nc[a] = mesh_.nc[a];
      A.n[a] = mesh_.n[a];
    }
  }
  launch_march(mode, A, s);
}

void Solver::solve_box(int which, double* data, cudaStream_t s) {
  const BoxArray arr = which < 3 ? kind_array(g_slab_[which], data) : which == 3 ? kind_array(g_coarse_, data)
                                                                                  : hole_array(data);
  launch_block_thomas(bt_[which], arr, state_, s);
}

void Solver::fill(double* e, const double* b, cudaStream_t s, int stage) {
  if (variable_) {
    launch_hole_rhs_var(mesh_.dim, e, b, fg_, coef_fine_, md_, state_, s);
    solve_box(4, e, s);
    return;
  }
  const bool generic = std::getenv("ASDSM_GENERIC_FILL") != nullptr;
  const SepSolver& H = sep_hole_;
  if (!generic && mesh_.dim == 2 && !H.complex_modes && H.nd == 1 && H.L == 1 && !H.use_pcr) {
    // One fused kernel per hole (holes2d.cu) in both modes; for larger holes in error mode: ring
    // rhs + analytic forward transform + Thomas (one kernel), then the DMMA back transform
    // straight into the hole positions of the fine array.
    Hole2DArgs A{};
    A.m0 = H.ext[0];
    A.m1 = H.ext[1];
    A.n0 = mesh_.n[0];
    A.n1 = mesh_.n[1];
    A.nf0 = mesh_.nf[0];
    A.nf1 = mesh_.nf[1];
    A.nbox0 = mesh_.nc[0] + 1;
    A.nbox1 = mesh_.nc[1] + 1;
    // (a variant staging every table slice in shared memory first measured slower: its time
    // goes into a dependent shared-store chain; kept available as tables_in_smem)
    const bool staged = std::getenv("ASDSM_HOLE_STAGED") != nullptr;
    hole2d_prepare(113 * 1024);
    A.kb = 32;
    A.tables_in_smem = (staged && hole2d_smem_bytes(A.m0, A.m1, A.kb, true, true) <= 113 * 1024) ? 1 : 0;
    if (!A.tables_in_smem) {
      A.kb = 64;
      A.y_in_smem = hole2d_smem_bytes(A.m0, A.m1, A.kb, true) <= 48 * 1024 ? 1 : 0;
      if (!A.y_in_smem && hole2d_smem_bytes(A.m0, A.m1, 32, true) <= 48 * 1024) {
        A.kb = 32;  // narrower CTAs so the forward sweep stays in shared memory
        A.y_in_smem = 1;
      }
    }
    A.st = st_fine_;
    A.Wt = H.Wt[0];
    A.half = H.half[0];
    A.ipiv = H.th_ipiv;
    A.cp = H.th_cp;
    A.line_left = H.line_left;
    A.line_right = H.line_right;
    const bool unfused = std::getenv("ASDSM_HOLE_UNFUSED") != nullptr;
    if (ring_from_lines_) {  // the slab step left the skeleton to the holes (fused kernel only)
      A.skel_line0 = skel_line_[0];
      A.skel_line1 = skel_line_[1];
      A.corr = skel_corr_;
      A.basis0 = sp_basis_[0];
      A.basis1 = sp_basis_[1];
      A.nc0 = mesh_.nc[0];
      A.nc1 = mesh_.nc[1];
    }
    if (!unfused && hole2d_fused_fits(A.m0, A.m1)) {
      launch_hole2d_fused(e, A, b, state_, s);
      return;
    }
    if (ring_from_lines_) throw AsdsmError(kUnsupported, "slab step without the fused hole kernel");
  }
  if (!generic && mesh_.dim == 2 && b == nullptr && !H.complex_modes && H.nd == 1 && H.L == 1 && !H.use_pcr) {
    Hole2DArgs A{};
    A.m0 = H.ext[0];
    A.m1 = H.ext[1];
    A.n0 = mesh_.n[0];
    A.n1 = mesh_.n[1];
    A.nf0 = mesh_.nf[0];
    A.nf1 = mesh_.nf[1];
    A.nbox0 = mesh_.nc[0] + 1;
    A.nbox1 = mesh_.nc[1] + 1;
    const bool staged = std::getenv("ASDSM_HOLE_STAGED") != nullptr;
    A.kb = 32;
    A.tables_in_smem = (staged && hole2d_smem_bytes(A.m0, A.m1, A.kb, true, true) <= 113 * 1024) ? 1 : 0;
    if (!A.tables_in_smem) {
      A.kb = 64;
      A.y_in_smem = hole2d_smem_bytes(A.m0, A.m1, A.kb, true) <= 48 * 1024 ? 1 : 0;
      if (!A.y_in_smem && hole2d_smem_bytes(A.m0, A.m1, 32, true) <= 48 * 1024) {
        A.kb = 32;  // narrower CTAs so the forward sweep stays in shared memory
        A.y_in_smem = 1;
      }
    }
    A.st = st_fine_;
    A.Wt = H.Wt[0];
    A.half = H.half[0];
    A.ipiv = H.th_ipiv;
    A.cp = H.th_cp;
    A.line_left = H.line_left;
    A.line_right = H.line_right;
    double* modes = static_cast<double*>(scratch0_);
    // one warp per mode line with the partition method (measured, config 2: see DESIGN), else
    // one thread per mode line (Thomas)
    const bool thomas = std::getenv("ASDSM_HOLE_THOMAS") != nullptr;
    const bool part = !thomas && H.part && hole2d_part_supported(H.part_seg) && hole_ring_;
    // strip split (error mode, partitioned lines): separators from the hole's modes, then every
    // strip as a hole of w columns (ASDSM_STRIPS; read at capture time)
    const bool strips = part && strip_p_ > 0;
    const SepSolver& T = strips ? sep_strip_ : H;
    if (stage & kFillLines) {
      const bool gemm = strips && sep_K_ != nullptr;
      if (part) {
        Hole2DPartArgs P{H.W[0], H.part, H.part_stride, H.part_seg, H.part_P, H.part_last, hole_ring_};
        launch_hole2d_ring(e, A, P, state_, s);
        if (!gemm) launch_hole2d_part(modes, A, P, state_, s);
      } else {
        launch_hole2d_fwd_thomas(e, modes, A, state_, s);
      }
      if (gemm) {
        // separators = K ring for every hole at once (cuBLAS DGEMM, captured into the graph)
        cublasHandle_t h = static_cast<cublasHandle_t>(blas_);
        if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream failed");
        const double one = 1.0, zero = 0.0;
        const int nh = A.nbox0 * A.nbox1;
        if (cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, sep_rows_, nh, sep_cols_, &one, sep_K_, sep_rows_, hole_ring_,
                        sep_cols_, &zero, sep_C_, sep_rows_) != CUBLAS_STATUS_SUCCESS)
          throw CudaError("cublasDgemm (hole separators) failed");
        launch_hole2d_sep_scatter(sep_C_, e, A, strip_p_, state_, s);
      } else if (strips) {
        launch_hole2d_sep_rows(modes, H.V[0], e, A, strip_p_, state_, s);
      }
      if (strips) {
        const int w = T.ext[0];
        A.m0 = w;
        A.n0 = w + 1;
        A.nbox0 *= strip_p_;
        A.Wt = T.Wt[0];
        A.half = T.half[0];
        A.ipiv = T.th_ipiv;
        A.cp = T.th_cp;
        A.line_left = T.line_left;
        A.line_right = T.line_right;
        Hole2DPartArgs P{T.W[0], T.part, T.part_stride, T.part_seg, T.part_P, T.part_last, strip_ring_};
        launch_hole2d_ring(e, A, P, state_, s);
        launch_hole2d_part(modes, A, P, state_, s);
      }
    } else if (strips) {
      A.m0 = T.ext[0];
      A.n0 = T.ext[0] + 1;
      A.nbox0 *= strip_p_;
    }
    if (!(stage & kFillBack)) return;
    GemmLines G{};
    G.o_ext[0] = A.m1;
    G.o_ext[1] = 1;
    G.o_in[0] = part ? 1 : A.m0;
    G.o_out[0] = g_fine_.stride[1];
    G.nbox[0] = A.nbox0;
    G.nbox[1] = A.nbox1;
    G.nbox[2] = 1;
    G.in_bs[0] = static_cast<i64>(A.m0) * A.m1;
    G.in_bs[1] = static_cast<i64>(A.m0) * A.m1 * A.nbox0;
    G.out_bs[0] = A.n0;
    G.out_bs[1] = static_cast<i64>(A.n1) * g_fine_.stride[1];
    G.nlines = static_cast<i64>(A.m1) * A.nbox0 * A.nbox1;
    const i64 in_es = part ? A.m1 : 1;  // [hole][k][j] from the partition solve, else [hole][j][k]
    // strips: the table-resident back transform (ASDSM_STRIP_BACK=0: the generic even/odd GEMM;
    // read at capture time)
    const char* sb = std::getenv("ASDSM_STRIP_BACK");
    if (strips && part && strip_back_supported(A.m0, A.m1) && !(sb && sb[0] == '0') &&
        std::getenv("ASDSM_DENSE_GEMM") == nullptr) {
      launch_strip_back(modes, e, T.half[0], A.m0, A.m1, A.nbox0, A.nbox1, G.out_bs[0], G.out_bs[1], g_fine_.stride[1], s);
      return;
    }
    if (A.m0 >= eo_min_modes() && std::getenv("ASDSM_DENSE_GEMM") == nullptr)
      launch_dmma_eo_transform(true, modes, e, T.half[0], A.m0, in_es, 1, G, s);
    else launch_dmma_transform(modes, e, T.V[0], A.m0, in_es, 1, G, s);
    return;
  }
  if (!generic && mesh_.dim == 3 && b == nullptr && !H.complex_modes && H.nd == 2 && H.L == 2 && H.dax[0] == 0 &&
      H.dax[1] == 1 && !H.use_pcr) {
    // Error mode: face-sparse forward transform + Thomas along the line axis, DMMA back transforms.
    Hole3DArgs A{};
    for (int a = 0; a < 3; ++a) {
      A.m[a] = H.ext[a];
      A.n[a] = mesh_.n[a];
      A.nf[a] = mesh_.nf[a];
      A.nbox[a] = mesh_.nc[a] + 1;
    }
    A.st = st_fine_;
    A.Wx = H.W[0];
    A.Wy = H.W[1];
    A.ipiv = H.th_ipiv;
    A.cp = H.th_cp;
    A.line_left = H.line_left;
    A.faces = faces3d_;
    if (h3f_ok_ && std::getenv("ASDSM_HOLE3D_UNFUSED") == nullptr) {  // (read at capture time)
      launch_hole3d_fused(e, h3f_, h3f_causal_, state_, s);
      return;
    }
    launch_hole3d_faces(e, A, state_, s);
    launch_hole3d_thomas(static_cast<double*>(scratch0_), A, state_, s);
    sep_back_transform(H, scratch0_, hole_array(e), scratch1_, s);
    return;
  }
  launch_hole_rhs(mesh_.dim, e, b, fg_, st_fine_, md_, state_, s);
  const BoxArray h = hole_array(e);
  sep_solve(sep_hole_, h, h, scratch0_, scratch1_, s);
}

static MarchArgs march_args(const double* u0, const double* u1, const double* e, const double* b, double* uo0,
                            double* uo1, double* ro0, double* ro1, const double* exact, const FineGeom& g,
                            const Stencil& st, double* partials, DevState* state, const CtrlArgs& c,
                            double* history) {
  MarchArgs A{};
  A.coef = nullptr;
  A.u0 = u0;
  A.u1 = u1;
  A.e = e;
  A.b = b;
  A.uo0 = uo0;
  A.uo1 = uo1;
  A.ro0 = ro0;
  A.ro1 = ro1;
  A.r0 = ro0;
  A.r1 = ro1;
  A.exact = exact;
  A.g = g;
  A.st = st;
  A.partials = partials;
  A.state = state;
  A.ctrl = c;
  A.history = history;
  A.coef = nullptr;
  return A;
}

static void set_factors(MarchArgs& A, const Mesh& m) {
  for (int a = 0; a < 3; ++a) A.n[a] = a < m.dim ? m.n[a] : 1;
}

static Slab2DArgs slab2d_args(const MeshDev& md, const SepSolver* S, double* const* modes, double* const* sol) {
  Slab2DArgs A{};
  A.m = md;
  A.cplx = S[0].complex_modes ? 1 : 0;
  for (int a = 0; a < 2; ++a) {
    A.W[a] = S[a].W[a];
    A.V[a] = S[a].V[a];
    A.k1[a] = S[a].pcr_k1;
    A.k2[a] = S[a].pcr_k2;
    A.invb[a] = S[a].pcr_invb;
    A.levels[a] = S[a].pcr_levels;
    A.modes[a] = modes[a];
    A.sol[a] = sol[a];
  }
  return A;
}

// Alg. 1 with the assembled bundle (solver.cpp:518-548, smooth mode).
void Solver::smooth_guess(double* out, cudaStream_t s) {
  if (variable_) {
    for (int a = 0; a < mesh_.dim; ++a) {
      ASDSM_CUDA_CHECK(cudaMemcpyAsync(sol_slab_[a], b_slab_[a], static_cast<size_t>(g_slab_[a].size) * sizeof(double),
                                       cudaMemcpyDeviceToDevice, s));
      solve_box(a, sol_slab_[a], s);
    }
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(u_cc_, b_coarse_, static_cast<size_t>(g_coarse_.size) * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
    solve_box(3, u_cc_, s);
    const double* sol[3] = {sol_slab_[0], sol_slab_[1], sol_slab_[2]};
    skeleton(sol, u_cc_, nullptr, out, s);
    fill(out, b_, s);
    return;
  }
  if (fast2d_) {
    Slab2DArgs A = slab2d_args(md_, sep_slab_, slab_modes_, sol_slab_);
    A.in_slab[0] = b_slab_[0];
    A.in_slab[1] = b_slab_[1];
    launch_slab2d_fwd(A, state_, s);
    launch_slab2d_back(A, partials_, state_, history_, false, s);
    sep_solve(sep_coarse_, kind_array(g_coarse_, b_coarse_), kind_array(g_coarse_, u_cc_), scratch0_, scratch1_, s);
    const double* sol[3] = {sol_slab_[0], sol_slab_[1], nullptr};
    skeleton(sol, u_cc_, nullptr, out, s);
    fill(out, b_, s);
    return;
  }
  for (int a = 0; a < mesh_.dim; ++a)
    sep_solve(sep_slab_[a], kind_array(g_slab_[a], b_slab_[a]), kind_array(g_slab_[a], sol_slab_[a]), scratch0_,
              scratch1_, s);
  sep_solve(sep_coarse_, kind_array(g_coarse_, b_coarse_), kind_array(g_coarse_, u_cc_), scratch0_, scratch1_, s);
  const double* sol[3] = {sol_slab_[0], sol_slab_[1], sol_slab_[2]};
  skeleton(sol, u_cc_, nullptr, out, s);
  fill(out, b_, s);
}

// error_guess (solver.cpp:550-558): restrict r, solve the slabs, normalize, merge, fill
// against a zero right-hand side.
void Solver::error_mode_guess(const double* r0, const double* r1, int k, double* out, cudaStream_t s) {
  if (fast2d_) {
    Slab2DArgs A = slab2d_args(md_, sep_slab_, slab_modes_, sol_slab_);
    A.in_fine0 = r0;
    A.in_fine1 = r1;
    if (r0 == r_[0] && r1 == r_[1]) {  // the station copies the residual passes keep
      A.sta0 = stations_[0];
      A.sta1 = stations_[1];
      if (step2d_) {  // slab solves + normalization + cc/spline in one launch; the holes
        launch_slabstep2d(slabstep2d_args(coins_ + 4 * k, out), state_, s);  // write the skeleton
        ring_from_lines_ = true;
        fill(out, nullptr, s);
        ring_from_lines_ = false;
        return;
      }
    }
    const double* sol[3] = {sol_slab_[0], sol_slab_[1], nullptr};
    const Skel2DArgs sk = skel2d_args(sol, nullptr, coins_ + 4 * k, out);
    launch_slab2d_fwd(A, state_, s);
    launch_slab2d_back(A, partials_, state_, history_, true, s, &sk);  // + cc/spline phase in its last block
    launch_skel2d_write_fast(sk, state_, s);
    fill(out, nullptr, s);
    return;
  }
  const bool fork = aux_[0] != nullptr && std::getenv("ASDSM_SERIAL_SLABS") == nullptr;  // (read at capture time)
  if (fork) {
    ASDSM_CUDA_CHECK(cudaEventRecord(ev_[0], s));
    for (cudaStream_t q : aux_) ASDSM_CUDA_CHECK(cudaStreamWaitEvent(q, ev_[0], 0));
  }
  for (int a = 0; a < mesh_.dim; ++a) {
    if (variable_) {
      launch_gather(r0, r1, sol_slab_[a], md_, 1u << a, g_slab_[a].size, state_, s);
      solve_box(a, sol_slab_[a], s);
      continue;
    }
    const bool own = fork && a > 0;
    cudaStream_t q = own ? aux_[a - 1] : s;
    launch_gather(r0, r1, rhs_slab_[a], md_, 1u << a, g_slab_[a].size, state_, q);
    sep_solve(sep_slab_[a], kind_array(g_slab_[a], rhs_slab_[a]), kind_array(g_slab_[a], sol_slab_[a]),
              own ? slab_scr_[a][0] : scratch0_, own ? slab_scr_[a][1] : scratch1_, q);
  }
  if (fork) {
    for (int i = 0; i < 2; ++i) {
      ASDSM_CUDA_CHECK(cudaEventRecord(ev_[1 + i], aux_[i]));
      ASDSM_CUDA_CHECK(cudaStreamWaitEvent(s, ev_[1 + i], 0));
    }
  }
  for (int a = 0; a < mesh_.dim; ++a) {
    CtrlArgs c{};
    c.op = kCtrlSlabNorm;
    c.which = a;
    launch_norm_sq(sol_slab_[a], g_slab_[a].size, partials_, state_, s, &c, history_);
  }
  for (int a = 0; a < mesh_.dim; ++a) launch_divide(sol_slab_[a], g_slab_[a].size, &state_->slab_norm[a], state_, s);
  const double* sol[3] = {sol_slab_[0], sol_slab_[1], sol_slab_[2]};
  skeleton(sol, nullptr, coins_ + 4 * k, out, s);
  fill(out, nullptr, s);
}

void Solver::run(const RunOptions& o, cudaStream_t s) {
  prepare_run(o, s);
  const bool no_graph = std::getenv("ASDSM_NO_GRAPH") != nullptr;
  if (no_graph || s == nullptr) {
    const long long l0 = g_kernel_launches;
    enqueue_run(o, s);
    launches_ = g_kernel_launches - l0;
    return;
  }
  run_graph(o, s);
}

void Solver::run_observed(const RunOptions& o, cudaStream_t s, const std::function<bool(int)>& after_record) {
  prepare_run(o, s);
  const long long l0 = g_kernel_launches;
  enqueue_run(o, s, &after_record);
  launches_ = g_kernel_launches - l0;
}

int Solver::snapshot(std::vector<double>& rows, bool& active, double* u_out, double* r_out, cudaStream_t s) {
  if (!host_state_) ASDSM_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&host_state_), sizeof(DevState), 0));
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(host_state_, state_, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(s));
  const DevState h = *host_state_;
  const int nrec = history_ ? std::min(h.nrec, history_cap_) : 0;
  rows.resize(static_cast<size_t>(nrec) * 7);
  const size_t nb = static_cast<size_t>(g_fine_.size) * sizeof(double);
  if (nrec) ASDSM_CUDA_CHECK(cudaMemcpyAsync(rows.data(), history_, rows.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (u_out) ASDSM_CUDA_CHECK(cudaMemcpyAsync(u_out, u_[h.cur], nb, cudaMemcpyDefault, s));
  if (r_out) ASDSM_CUDA_CHECK(cudaMemcpyAsync(r_out, r_[h.cur], nb, cudaMemcpyDefault, s));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(s));
  double prev = h.t0_ns;  // wall_ms per row, as fetch()
  for (int k = 0; k < nrec; ++k) {
    const double t = rows[static_cast<size_t>(k) * 7 + 6];
    rows[static_cast<size_t>(k) * 7 + 6] = (t - prev) / 1e6;
    prev = t;
  }
  active = h.active != 0;
  return nrec;
}

void Solver::prepare_run(const RunOptions& o, cudaStream_t s) {
  last_opts_ = o;
  const int cap = std::max(o.max_iter, 0) + 1;
  if (cap > history_cap_) {
    history_ = dev_.alloc<double>(static_cast<size_t>(cap) * 7);
    history_cap_ = cap;
    if (graph_exec_) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
  }
  // Seeded draws (solver.cpp:110-120, 309-345): per iteration k the engine is
  // mt19937_64(mix_seed(seed, k)); 2D takes one draw % 2, 3D one % 3 then three % 2.
  std::vector<int> coins(static_cast<size_t>(4 * cap), 0);
  for (int k = 0; k < cap; ++k) {
    std::mt19937_64 eng(mix_seed(o.rng_seed, static_cast<std::uint64_t>(k)));
    if (mesh_.dim == 2) {
      coins[static_cast<size_t>(4 * k)] = static_cast<int>(eng() % 2);
    } else {
      coins[static_cast<size_t>(4 * k)] = static_cast<int>(eng() % 3);
      for (int i = 1; i < 4; ++i) coins[static_cast<size_t>(4 * k + i)] = static_cast<int>(eng() % 2);
    }
  }
  if (4 * cap > coins_cap_) {
    coins_ = dev_.alloc<int>(static_cast<size_t>(4 * cap));
    coins_cap_ = 4 * cap;
    if (graph_exec_) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
  }
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(coins_, coins.data(), coins.size() * sizeof(int), cudaMemcpyHostToDevice, s));

  // subsample > 0 (solver.cpp:462-475): per iteration a fresh mt19937_64(seed_k) partial
  // Fisher-Yates over the ascending skeleton rows, the first m kept and sorted.
  sub_m_ = 0;
  if (o.subsample > 0.0) {
    if (skel_rows_.empty()) {
      for (i64 p = 0; p < g_fine_.size; ++p) {
        i64 q = p;
        bool sk = false;
        for (int a = 0; a < mesh_.dim; ++a) {
          const int ia = static_cast<int>(q % mesh_.nf[a]);
          q /= mesh_.nf[a];
          if ((ia + 1) % mesh_.n[a] == 0) sk = true;
        }
        if (sk) skel_rows_.push_back(p);
      }
    }
    const i64 total = static_cast<i64>(skel_rows_.size());
    i64 m = std::llround(o.subsample * static_cast<double>(total));
    m = std::min<i64>(std::max<i64>(m, 1), total);
    sub_m_ = static_cast<int>(m);
    std::vector<long long> all(static_cast<size_t>(m) * cap);
    for (int k = 1; k < cap; ++k) {
      std::vector<long long> rows = skel_rows_;
      std::mt19937_64 eng(mix_seed(o.rng_seed, static_cast<std::uint64_t>(k)));
      for (i64 i = 0; i < m; ++i) {
        const i64 j = i + static_cast<i64>(eng() % static_cast<std::uint64_t>(total - i));
        std::swap(rows[static_cast<size_t>(i)], rows[static_cast<size_t>(j)]);
      }
      std::sort(rows.begin(), rows.begin() + m);
      std::copy(rows.begin(), rows.begin() + m, all.begin() + static_cast<i64>(m) * k);
    }
    if (all.size() > sub_cap_) {
      sub_rows_ = dev_.alloc<long long>(all.size());
      sub_cap_ = all.size();
      if (graph_exec_) {
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
      }
    }
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(sub_rows_, all.data(), all.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  }
}

void Solver::run_graph(const RunOptions& o, cudaStream_t s) {
  const bool same = graph_exec_ && graph_opts_.tol == o.tol && graph_opts_.max_iter == o.max_iter &&
                    graph_opts_.stagnation_window == o.stagnation_window &&
                    graph_opts_.stagnation_ratio == o.stagnation_ratio && graph_opts_.subsample == o.subsample &&
                    graph_opts_.sparse_residual == o.sparse_residual && graph_has_exact_ == has_exact_;
  if (!same) {
    if (graph_exec_) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
    cudaGraph_t g = nullptr;
    const long long l0 = g_kernel_launches;
    ASDSM_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_run(o, s);
    } catch (...) {
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    ASDSM_CUDA_CHECK(cudaStreamEndCapture(s, &g));
    graph_launches_ = g_kernel_launches - l0;
    record_graph_kernels(g, graph_kernels_);
    const cudaError_t e = cudaGraphInstantiate(&graph_exec_, g, 0);
    cudaGraphDestroy(g);
    ASDSM_CUDA_CHECK(e);
    graph_opts_ = o;
    graph_has_exact_ = has_exact_;
  }
  ASDSM_CUDA_CHECK(cudaGraphLaunch(graph_exec_, s));
  launches_ = graph_launches_;
}

// Demangled names of the kernel nodes of a captured graph, with their multiplicity.
static void record_graph_kernels(cudaGraph_t g, std::vector<std::pair<std::string, int>>& out) {
  out.clear();
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess || n == 0) return;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return;
  std::map<std::string, int> count;
  for (cudaGraphNode_t node : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(node, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams p{};
    if (cudaGraphKernelNodeGetParams(node, &p) != cudaSuccess) continue;
    const char* mangled = nullptr;
    if (cudaFuncGetName(&mangled, p.func) != cudaSuccess || !mangled) continue;
    int status = 0;
    char* dem = abi::__cxa_demangle(mangled, nullptr, nullptr, &status);
    std::string name = status == 0 && dem ? std::string(dem) : std::string(mangled);
    std::free(dem);
    for (size_t q; (q = name.find("(anonymous namespace)::")) != std::string::npos;) name.erase(q, 23);
    if (name.rfind("void ", 0) == 0) name = name.substr(5);
    // drop the parameter list: the first '(' outside the template argument list
    int depth = 0;
    for (size_t q = 0; q < name.size(); ++q) {
      if (name[q] == '<') ++depth;
      else if (name[q] == '>') --depth;
      else if (name[q] == '(' && depth == 0) {
        name.resize(q);
        break;
      }
    }
    ++count[name];
  }
  cudaGetLastError();
  out.assign(count.begin(), count.end());
}

void Solver::enqueue_run(const RunOptions& o, cudaStream_t s, const std::function<bool(int)>* after_record) {
  reset_state(o, s);
  CtrlArgs c{};
  c.has_exact = has_exact_;
  c.cell = cell_;
  c.tol_growth = 1.0 + 1e-12;
  c.stagnation_window = o.stagnation_window;
  c.stagnation_pow = std::pow(o.stagnation_ratio, o.stagnation_window);
  c.max_iter = o.max_iter;
  c.tol = o.tol;
  c.subsample = sub_m_ > 0 ? 1 : 0;

  smooth_guess(u_[0], s);
  c.op = kCtrlResidualK0;
  c.k = 0;
  const double* ex = has_exact_ ? exact_ : nullptr;
  march_launch(kMarchResidual, march_args(u_[0], u_[1], nullptr, b_, nullptr, nullptr, r_[0], r_[1], ex, fg_, st_fine_,
                                          partials_, state_, c, history_), s);
  if (after_record && !(*after_record)(0)) return;

  // the step's dot products: their own pass, or (opt-in, ASDSM_DOTS_UPDATE=1) inside the update
  // launch with a grid barrier between the two phases -- measured slower in the captured graph
  // (config 1: 1.18-1.21 -> 1.23-1.26 ms per solve on the same box), kept for the record
  const bool dots_in_update = dots_update_ok_ && sub_m_ == 0 && skel_dots_ && !variable_;
  for (int k = 1; k <= o.max_iter; ++k) {
    CtrlArgs cstep = c;
    cstep.op = kCtrlStep;
    cstep.k = k;
    error_mode_guess(r_[0], r_[1], k, e_, s);
    if (sub_m_ > 0)
      launch_subsample_dots(mesh_.dim, sub_rows_ + static_cast<i64>(sub_m_) * k, sub_m_, e_, r_[0], r_[1], fg_,
                            st_fine_, partials_, state_, history_, s, coef_fine_);
    c.op = kCtrlStep;
    c.k = k;
    if (!dots_in_update) {
      MarchArgs dots = march_args(nullptr, nullptr, e_, nullptr, nullptr, nullptr, r_[0], r_[1], nullptr, fg_,
                                  st_fine_, partials_, state_, c, history_);
      dots.skel_only = skel_dots_ ? 1 : 0;
      march_launch(kMarchDots, dots, s);
    }
    c.op = kCtrlAccept;
    MarchArgs up = march_args(u_[0], u_[1], e_, b_, u_[0], u_[1], r_[0], r_[1], ex, fg_, st_fine_, partials_, state_,
                              c, history_);
    set_factors(up, mesh_);
    up.sparse = o.sparse_residual ? 1 : 0;
    if (dots_in_update) {
      up.skel_only = 1;
      up.dots_ctrl = cstep;
      march_launch(kMarchDotsUpdate, up, s);
    } else {
      march_launch(kMarchUpdate, up, s);
    }
    if (sub_m_ > 0) {  // all-rows retry when the subsampled step grew the residual
      up.ctrl.op = kCtrlAccept2;
      up.retry_pass = 1;
      march_launch(kMarchUpdate, up, s);
    }
    if (after_record && !(*after_record)(k)) return;
  }
}

int Solver::history(std::vector<double>& rows, int& stop_code, cudaStream_t s) {
  return fetch(rows, stop_code, nullptr, nullptr, s);
}

int Solver::fetch(std::vector<double>& rows, int& stop_code, double* u_out, double* r_out, cudaStream_t s) {
  if (!host_state_) ASDSM_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&host_state_), sizeof(DevState), 0));
  const int cap = std::max(history_cap_, 1);
  if (cap > host_hist_cap_) {
    if (host_hist_) cudaFreeHost(host_hist_);
    host_hist_ = nullptr;
    ASDSM_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&host_hist_), static_cast<size_t>(cap) * 7 * sizeof(double), 0));
    host_hist_cap_ = cap;
  }
  const size_t nb = static_cast<size_t>(g_fine_.size) * sizeof(double);
  if (u_out || r_out) launch_publish(state_, u_[0], u_[1], r_[0], r_[1], g_fine_.size, s);
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(host_state_, state_, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  if (history_)
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(host_hist_, history_, static_cast<size_t>(history_cap_) * 7 * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
  if (u_out) ASDSM_CUDA_CHECK(cudaMemcpyAsync(u_out, u_[0], nb, cudaMemcpyDefault, s));
  if (r_out) ASDSM_CUDA_CHECK(cudaMemcpyAsync(r_out, r_[0], nb, cudaMemcpyDefault, s));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(s));
  const DevState& h = *host_state_;
  const int nrec = history_ ? std::min(h.nrec, history_cap_) : 0;
  rows.assign(host_hist_, host_hist_ + static_cast<size_t>(nrec) * 7);
  // wall_ms: time since the previous record (row 0: since the solve started), as the
  // reference's record() does (solver.cpp:586-610), from the device %globaltimer
  double prev = h.t0_ns;
  for (int k = 0; k < nrec; ++k) {
    const double t = rows[static_cast<size_t>(k) * 7 + 6];
    rows[static_cast<size_t>(k) * 7 + 6] = (t - prev) / 1e6;
    prev = t;
  }
  stop_code = h.stop == 0 ? 3 : h.stop;
  return nrec;
}

const double* Solver::u_current(cudaStream_t s) const {
  int cur = 0;
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(&cur, &state_->cur, sizeof(int), cudaMemcpyDeviceToHost, s));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(s));
  return u_[cur];
}

const double* Solver::r_current(cudaStream_t s) const {
  int cur = 0;
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(&cur, &state_->cur, sizeof(int), cudaMemcpyDeviceToHost, s));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(s));
  return r_[cur];
}

void Solver::residual(const double* u, const double* b, double* r, cudaStream_t s) {
  launch_state_init(state_, 1, 1, s);
  CtrlArgs c{};
  c.op = -1;
  march_launch(kMarchResidual, march_args(u, u, nullptr, b, nullptr, nullptr, r, r, nullptr, fg_, st_fine_, partials_,
                                          state_, c, nullptr), s);
}

void Solver::error_guess(const double* r, std::uint64_t seed, double* e, cudaStream_t s) {
  launch_state_init(state_, 1, 1, s);
  if (coins_cap_ < 4) {
    coins_ = dev_.alloc<int>(4);
    coins_cap_ = 4;
  }
  int coins[4] = {0, 0, 0, 0};
  std::mt19937_64 eng(seed);
  if (mesh_.dim == 2) {
    coins[0] = static_cast<int>(eng() % 2);
  } else {
    coins[0] = static_cast<int>(eng() % 3);
    for (int i = 1; i < 4; ++i) coins[i] = static_cast<int>(eng() % 2);
  }
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(coins_, coins, sizeof(coins), cudaMemcpyHostToDevice, s));
  if (history_cap_ < 1) {
    history_ = dev_.alloc<double>(7);
    history_cap_ = 1;
  }
  error_mode_guess(r, r, 0, e, s);
  DevState back{};
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(&back, state_, sizeof(back), cudaMemcpyDeviceToHost, s));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(s));
  if (!back.have_e) throw AsdsmError(kZeroNormSolution, "initial_guess: zero-norm solution cannot be normalized");
}

double Solver::optimal_scaling(const double* r, const double* e, cudaStream_t s) {
  launch_state_init(state_, 1, 1, s);
  if (history_cap_ < 1) {
    history_ = dev_.alloc<double>(7);
    history_cap_ = 1;
  }
  CtrlArgs c{};
  c.op = kCtrlStep;
  march_launch(kMarchDots, march_args(nullptr, nullptr, e, nullptr, nullptr, nullptr, const_cast<double*>(r),
                                      const_cast<double*>(r), nullptr, fg_, st_fine_, partials_, state_, c, history_), s);
  DevState back{};
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(&back, state_, sizeof(back), cudaMemcpyDeviceToHost, s));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(s));
  return back.s;
}

void Solver::initial_guess(double* u_out, std::uint64_t seed, cudaStream_t s) {
  (void)seed;
  launch_state_init(state_, 1, 1, s);
  smooth_guess(u_out, s);
}

}  // namespace asdsm_b200

namespace asdsm_b200 {

std::vector<Solver::Component> Solver::profile(cudaStream_t s, int reps) {
  std::vector<Component> out;
  cudaEvent_t e0, e1;
  ASDSM_CUDA_CHECK(cudaEventCreate(&e0));
  ASDSM_CUDA_CHECK(cudaEventCreate(&e1));
  const i64 N = g_fine_.size;
  const i64 NH = mesh_.hole_count();
  const int iters = std::max(last_opts_.max_iter, 1);
  // the step dots run inside the fused hole kernel on this plan (enqueue_run's condition)
  const bool dots_in_update = dots_update_ok_ && sub_m_ == 0 && skel_dots_ && !variable_;
  auto timed = [&](const char* name, double bytes, double flops, int per_solve, auto&& body) {
    launch_state_init(state_, 1, 1, s);
    body();  // warm
    launch_spin(3000.0, s);  // keep the device busy while the host enqueues the timed loop
    ASDSM_CUDA_CHECK(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) body();
    ASDSM_CUDA_CHECK(cudaEventRecord(e1, s));
    ASDSM_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0;
    ASDSM_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    Component c;
    c.name = name;
    c.ms = ms / reps;
    c.bytes = bytes;
    c.flops = flops;
    c.per_solve = per_solve;
    out.push_back(c);
  };
  // a non-zero step so the update kernel does its work
  auto set_step = [&]() {
    CtrlArgs c{};
    c.op = kCtrlStep;
    MarchArgs dots = march_args(nullptr, nullptr, e_, nullptr, nullptr, nullptr, r_[0], r_[1], nullptr, fg_, st_fine_,
                                partials_, state_, c, history_);
    dots.skel_only = skel_dots_ ? 1 : 0;
    march_launch(kMarchDots, dots, s);
  };
  const double ex = has_exact_ ? 1.0 : 0.0;
  timed("update_residual", 8.0 * N * (5.0 + ex), 0.0, iters, [&] {
    launch_state_init(state_, 1, 1, s);
    CtrlArgs cs{};
    cs.op = kCtrlSetStep;
    cs.cell = 1e-3;  // any non-zero step: the pass does its full work
    launch_ctrl(cs, partials_, state_, history_, s);
    CtrlArgs c{};
    c.op = -1;
    march_launch(kMarchUpdate, march_args(u_[0], u_[1], e_, b_, u_[0], u_[1], r_[0], r_[1], has_exact_ ? exact_ : nullptr,
                                          fg_, st_fine_, partials_, state_, c, history_), s);
  });
  // the update-pass time alone: subtract the state-init + set-step part measured alone
  timed("step_overhead", 0.0, 0.0, 0, [&] {
    launch_state_init(state_, 1, 1, s);
    CtrlArgs cs{};
    cs.op = kCtrlSetStep;
    cs.cell = 1e-3;
    launch_ctrl(cs, partials_, state_, history_, s);
  });
  out[0].ms -= out[1].ms;
  out.pop_back();
  if (dots_in_update) {
    // the launch the step actually runs: skeleton dots, step control, grid barrier, update.
    // The standalone update pass above stays listed (per_solve 0) as the unfused reference.
    out[0].per_solve = 0;
    out[0].name = "update_residual_standalone";
    i64 nskel = 0;
    for (int a = 0; a < mesh_.dim; ++a) {
      i64 plane = mesh_.nc[a];
      for (int b = 0; b < mesh_.dim; ++b)
        if (b != a) plane *= mesh_.nf[b];
      nskel += plane;
    }
    timed("dots_update", 8.0 * N * (5.0 + ex) + 16.0 * nskel, 0.0, iters, [&] {
      launch_state_init(state_, 1, 1, s);
      CtrlArgs c{};
      c.op = -1;
      CtrlArgs cstep{};
      cstep.op = kCtrlStep;
      MarchArgs up = march_args(u_[0], u_[1], e_, b_, u_[0], u_[1], r_[0], r_[1], has_exact_ ? exact_ : nullptr, fg_,
                                st_fine_, partials_, state_, c, history_);
      set_factors(up, mesh_);
      up.skel_only = 1;
      up.dots_ctrl = cstep;
      march_launch(kMarchDotsUpdate, up, s);
    });
    timed("state_init", 0.0, 0.0, 0, [&] { launch_state_init(state_, 1, 1, s); });
    out[out.size() - 2].ms -= out.back().ms;
    out.pop_back();
  }
  if (!dots_in_update) {
    // skeleton-row dots move 2 doubles per skeleton point (+ the stencil's e neighbours, cached)
    i64 nskel_pts = N;
    if (skel_dots_) {
      nskel_pts = 0;
      for (int a = 0; a < mesh_.dim; ++a) {
        i64 plane = mesh_.nc[a];
        for (int b = 0; b < mesh_.dim; ++b)
          if (b != a) plane *= mesh_.nf[b];
        nskel_pts += plane;  // (cross points counted per plane: an upper bound)
      }
    }
    timed(skel_dots_ ? "step_dots_skeleton" : "step_dots", 8.0 * nskel_pts * 2.0, 0.0, iters, [&] { set_step(); });
  }
  const SepSolver& H = sep_hole_;
  i64 slab_pts = 0;
  for (int a = 0; a < mesh_.dim; ++a) slab_pts += g_slab_[a].size;
  if (fast2d_) {
    // the kernels of one fast-path iteration, each timed alone
    Slab2DArgs SA = slab2d_args(md_, sep_slab_, slab_modes_, sol_slab_);
    SA.in_fine0 = r_[0];
    SA.in_fine1 = r_[1];
    SA.sta0 = stations_[0];
    SA.sta1 = stations_[1];
    const double* sol[3] = {sol_slab_[0], sol_slab_[1], nullptr};
    const Skel2DArgs sk = skel2d_args(sol, nullptr, coins_, e_);
    const double cb = sep_slab_[0].complex_modes ? 16.0 : 8.0;
    const i64 nskel = static_cast<i64>(mesh_.nc[1]) * mesh_.nf[0] + static_cast<i64>(mesh_.nc[0]) * mesh_.nf[1];
    if (step2d_) {
      timed("slabstep2d", 8.0 * slab_pts + 8.0 * nskel, 0.0, iters,
            [&] { launch_slabstep2d(slabstep2d_args(coins_, e_), state_, s); });
    } else {
      timed("slab2d_fwd_pcr", (8.0 + cb) * slab_pts, 0.0, iters, [&] { launch_slab2d_fwd(SA, state_, s); });
      timed("slab2d_back_norms_ccspline", (8.0 + cb) * slab_pts, 0.0, iters,
            [&] { launch_slab2d_back(SA, partials_, state_, history_, true, s, &sk); });
      timed("skeleton_write", 16.0 * nskel, 0.0, iters, [&] { launch_skel2d_write_fast(sk, state_, s); });
    }
    // the hole fill exactly as the solve launches it (Solver::fill): one fused kernel per hole,
    // or (large holes) the mode-line solves and the DMMA back transform timed apart
    if (hole2d_fused_fits(H.ext[0], H.ext[1]) && std::getenv("ASDSM_HOLE_UNFUSED") == nullptr) {
      const double eo = H.ext[0] >= eo_min_modes() ? 0.5 : 1.0;  // even/odd split executes half the MACs
      timed("hole2d_fused_dmma", 8.0 * NH, 2.0 * H.ext[0] * eo * static_cast<double>(NH), iters,
            [&] { fill(e_, nullptr, s); });
    } else {
      // (strip split: the back transform runs over the strips' w-point transforms)
      const int mt = strip_p_ ? sep_strip_.ext[0] : H.ext[0];
      const double eot = mt >= eo_min_modes() ? 0.5 : 1.0;
      timed(strip_p_ ? "hole2d_mode_lines_separators_strip_lines" : "hole2d_mode_lines", 8.0 * NH * 2.0, 0.0, iters,
            [&] { fill(e_, nullptr, s, kFillLines); });
      timed("hole_backtransform_dmma", 8.0 * NH * 2.0, 2.0 * mt * eot * static_cast<double>(NH), iters,
            [&] { fill(e_, nullptr, s, kFillBack); });
    }
  } else {
    double hflops = 0;
    if (!variable_)
      for (int i = 0; i < H.nd; ++i) hflops += 2.0 * H.ext[H.dax[i]] * static_cast<double>(NH);
    if (h3f_ok_ && std::getenv("ASDSM_HOLE3D_UNFUSED") == nullptr) hflops *= 0.5;  // even/odd on both axes
    // algorithmic bytes: the fused kernel writes every hole value once (the ring it reads is
    // O(m^2) per hole); the unfused path also writes and reads the mode buffer
    const bool h3_fused = h3f_ok_ && std::getenv("ASDSM_HOLE3D_UNFUSED") == nullptr;
    timed("hole_fill", 8.0 * NH * (h3_fused ? 1.0 : 3.0), hflops, iters, [&] { fill(e_, nullptr, s); });
    timed("slab_solves", 8.0 * slab_pts * 4.0, 0.0, iters, [&] {
      for (int a = 0; a < mesh_.dim; ++a) {
        launch_gather(r_[0], r_[1], rhs_slab_[a], md_, 1u << a, g_slab_[a].size, state_, s);
        if (variable_) {
          solve_box(a, rhs_slab_[a], s);
          continue;
        }
        sep_solve(sep_slab_[a], kind_array(g_slab_[a], rhs_slab_[a]), kind_array(g_slab_[a], sol_slab_[a]), scratch0_,
                  scratch1_, s);
      }
    });
    timed("skeleton_merge", 8.0 * slab_pts * 2.0, 0.0, iters, [&] {
      const double* sol[3] = {sol_slab_[0], sol_slab_[1], sol_slab_[2]};
      skeleton(sol, nullptr, coins_, e_, s);
    });
  }
  timed("residual", 8.0 * N * 3.0, 0.0, 1, [&] {
    CtrlArgs c{};
    c.op = -1;
    march_launch(kMarchResidual, march_args(u_[0], u_[1], nullptr, b_, nullptr, nullptr, r_[0], r_[1], nullptr, fg_,
                                            st_fine_, partials_, state_, c, history_), s);
  });
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return out;
}

}  // namespace asdsm_b200

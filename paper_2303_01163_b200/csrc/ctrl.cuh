// Device-side control logic and the last-block reduction fold (header-only so every
// translation unit's reduction kernels can finish with the control op, no separate launch).
#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

__device__ __forceinline__ double ctrl_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-shape reduction of the kRedBlocks partials of one slot.
__device__ inline double ctrl_reduce(const double* part, bool is_max, int nblocks = kRedBlocks) {
  __shared__ double sh[kRedThreads];
  double v = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) v = is_max ? fmax(v, __ldcg(part + i)) : v + __ldcg(part + i);
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = is_max ? fmax(sh[threadIdx.x], sh[threadIdx.x + w]) : sh[threadIdx.x] + sh[threadIdx.x + w];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// All four slots (sum, max, sum, max) in one pass: fixed per-thread order, then a fixed
// warp-shuffle tree and one shared-memory round.
__device__ inline void ctrl_reduce4(const double* part, int nblocks, double& s0, double& m1, double& s2, double& m3) {
  __shared__ double sh[4][32];
  double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
    a += __ldcg(part + i);
    b = fmax(b, __ldcg(part + kRedStride + i));
    c += __ldcg(part + 2 * kRedStride + i);
    d = fmax(d, __ldcg(part + 3 * kRedStride + i));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b = fmax(b, __shfl_down_sync(0xffffffffu, b, o));
    c += __shfl_down_sync(0xffffffffu, c, o);
    d = fmax(d, __shfl_down_sync(0xffffffffu, d, o));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    sh[0][w] = a;
    sh[1][w] = b;
    sh[2][w] = c;
    sh[3][w] = d;
  }
  __syncthreads();
  if (w == 0) {
    a = lane < nw ? sh[0][lane] : 0.0;
    b = lane < nw ? sh[1][lane] : 0.0;
    c = lane < nw ? sh[2][lane] : 0.0;
    d = lane < nw ? sh[3][lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b = fmax(b, __shfl_down_sync(0xffffffffu, b, o));
      c += __shfl_down_sync(0xffffffffu, c, o);
      d = fmax(d, __shfl_down_sync(0xffffffffu, d, o));
    }
  }
  s0 = a;
  m1 = b;
  s2 = c;
  m3 = d;
}

// Control logic of one reduction (thread 0 of the reducing block).
__device__ inline void ctrl_apply(const CtrlArgs& c, double s0, double m1, double s2, double m3, DevState* S,
                           double* history) {
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  auto record = [&](int k, double s_hat) {
    double* row = history + static_cast<i64>(k) * 7;
    row[0] = k;
    row[1] = S->res_l2;
    row[2] = S->res_inf;
    row[3] = S->err_max;
    row[4] = S->err_l2;
    row[5] = s_hat;
    unsigned long long tns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
    row[6] = static_cast<double>(tns);  // absolute ns; converted to per-row wall_ms on fetch
    S->nrec = k + 1;
  };
  switch (c.op) {
    case kCtrlResidualK0: {
      S->res_l2 = sqrt(s0);
      S->res_inf = m1;
      S->err_max = c.has_exact ? m3 : nan;
      S->err_l2 = c.has_exact ? sqrt(s2 * c.cell) : nan;
      record(0, nan);
      if (S->res_l2 <= S->stop_at) {
        S->stop = 1;
        S->active = 0;
      } else if (c.max_iter <= 0) {
        S->stop = 3;
        S->active = 0;
      }
      S->have_e = 1;
      break;
    }
    case kCtrlInit: {
      S->b_l2 = sqrt(s0);
      S->stop_at = c.tol * (S->b_l2 > 0.0 ? S->b_l2 : 1.0);
      break;
    }
    case kCtrlSetStep: {
      S->s = c.cell;
      break;
    }
    case kCtrlSlabNorms2: {
      const double n0 = sqrt(s0), n1 = sqrt(s2);
      S->slab_norm[0] = n0;
      S->slab_norm[1] = n1;
      if (!(n0 > 0.0) || !(n1 > 0.0)) S->have_e = 0;
      break;
    }
    case kCtrlSlabNorm: {
      const double n = sqrt(s0);
      S->slab_norm[c.which] = n;
      if (!(n > 0.0)) S->have_e = 0;
      break;
    }
    case kCtrlSubDots: {
      S->num_sub = s0;
      S->den_sub = s2;
      break;
    }
    case kCtrlStep: {  // optimal_scaling (solver.cpp:447-484), clamp at zero
      double s = 0.0, ssub = 0.0;
      if (S->have_e) {
        S->num = s0;
        S->den = s2;
        if (s2 > 0.0) {
          const double q = s0 / s2;
          s = (0.0 < q) ? q : 0.0;
        }
        if (c.subsample && S->den_sub > 0.0) {
          const double q = S->num_sub / S->den_sub;
          ssub = (0.0 < q) ? q : 0.0;
        }
      }
      S->s_full = s;
      S->s = c.subsample ? ssub : s;
      S->retry = 0;
      break;
    }
    case kCtrlAccept:
    case kCtrlAccept2: {  // residual-growth guard + record + stop rules (solver.cpp:648-677)
      if (c.op == kCtrlAccept2 && !S->retry) break;  // no retry was needed: already recorded
      double s = S->s;
      if (c.op == kCtrlAccept && c.subsample && s != 0.0 && sqrt(s0) > S->res_l2 * c.tol_growth) {
        S->retry = 1;  // the subsampled step grew the residual: retry with all rows
        S->s = S->s_full;
        break;
      }
      S->retry = 0;
      if (s != 0.0) {
        const double nl2 = sqrt(s0);
        if (nl2 > S->res_l2 * c.tol_growth) {
          s = 0.0;
        } else {
          S->cur = 1 - S->cur;
          S->res_l2 = nl2;
          S->res_inf = m1;
          if (c.has_exact) {
            S->err_max = m3;
            S->err_l2 = sqrt(s2 * c.cell);
          }
        }
      }
      S->s = s;
      record(c.k, s);
      if (S->res_l2 <= S->stop_at) {
        S->stop = 1;
      } else if (c.stagnation_window > 0 && c.k >= c.stagnation_window) {
        const double then = history[static_cast<i64>(c.k - c.stagnation_window) * 7 + 1];
        if (S->res_l2 > then * c.stagnation_pow) S->stop = 2;
      }
      if (S->stop == 0 && c.k >= c.max_iter) S->stop = 3;
      if (S->stop != 0) S->active = 0;
      S->have_e = 1;
      break;
    }
  }
}

static __global__ void __launch_bounds__(kRedThreads) ctrl_kernel(CtrlArgs c, const double* partials, DevState* S,
                                                          double* history) {
  if (!S->active) return;
  const double s0 = ctrl_reduce(partials + 0 * kRedStride, false);
  const double m1 = ctrl_reduce(partials + 1 * kRedStride, true);
  const double s2 = ctrl_reduce(partials + 2 * kRedStride, false);
  const double m3 = ctrl_reduce(partials + 3 * kRedStride, true);
  if (threadIdx.x != 0) return;
  ctrl_apply(c, s0, m1, s2, m3, S, history);
}

// Block partials of (sum, max, sum, max) for any 1D grid: partials[slot*kRedStride + block].
__device__ inline void block_reduce4_march(double s0, double m1, double s2, double m3, double* partials) {
  __shared__ double sh[4][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_down_sync(0xffffffffu, s0, o);
    m1 = fmax(m1, __shfl_down_sync(0xffffffffu, m1, o));
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
    m3 = fmax(m3, __shfl_down_sync(0xffffffffu, m3, o));
  }
  if (lane == 0) {
    sh[0][w] = s0;
    sh[1][w] = m1;
    sh[2][w] = s2;
    sh[3][w] = m3;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    s0 = lane < nw ? sh[0][lane] : 0.0;
    m1 = lane < nw ? sh[1][lane] : 0.0;
    s2 = lane < nw ? sh[2][lane] : 0.0;
    m3 = lane < nw ? sh[3][lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_down_sync(0xffffffffu, s0, o);
      m1 = fmax(m1, __shfl_down_sync(0xffffffffu, m1, o));
      s2 += __shfl_down_sync(0xffffffffu, s2, o);
      m3 = fmax(m3, __shfl_down_sync(0xffffffffu, m3, o));
    }
    if (lane == 0) {
      partials[0 * kRedStride + blockIdx.x] = s0;
      partials[1 * kRedStride + blockIdx.x] = m1;
      partials[2 * kRedStride + blockIdx.x] = s2;
      partials[3 * kRedStride + blockIdx.x] = m3;
    }
  }
}

// Last-block fold: after every block has written its partials, the last block to finish
// reduces them in a fixed order and applies the control op -- no separate ctrl launch.

__device__ inline bool fold_ctrl(const CtrlArgs& c, double* partials, DevState* S, double* history,
                                 unsigned nblocks_part = 0) {
  if (c.op < 0) return false;
  __shared__ int last;
  // nblocks_part: only blocks [0, nblocks_part) take part (the rest do not call this)
  const unsigned nblocks = nblocks_part ? nblocks_part : gridDim.x * gridDim.y * gridDim.z;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    __threadfence();
    const unsigned t = atomicAdd(&S->red_counter, 1u);
    last = (t == nblocks - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double s0, m1, s2, m3;
  ctrl_reduce4(partials, static_cast<int>(nblocks), s0, m1, s2, m3);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    ctrl_apply(c, s0, m1, s2, m3, S, history);
    S->red_counter = 0;
    __threadfence();
  }
  return true;
}


}  // namespace asdsm_b200

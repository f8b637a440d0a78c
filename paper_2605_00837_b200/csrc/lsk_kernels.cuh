// Stand-alone kernels behind the reference's half-step / diagnostic API:
// update_alpha (solver.py:118-140), update_beta (143-176), marginal_error
// (179-206), transport_cost (209-227), materialize_plan (434-458), and the
// cost builder squared_euclidean_cost (costs.py:36-50). These handle any
// (n, m) and are the parity hooks for the pieces the persistent solver fuses.
#pragma once
#include "lsk_device.cuh"

namespace lsk {

enum RowMode { kRowAlpha = 0, kRowCheck = 1, kRowCost = 2 };

// One CTA (256 threads) per row, two-pass LSE over the row (max, then the
// shifted sum, recomputing the argument -- reduction.py:179-208). Reads the
// row twice from L1/L2. mode:
//   kRowAlpha: out[i] = neg_eps * LSE_j(arg3(other_j, C_ij, inv, lw_j))
//   kRowCheck: out[i] = |exp(log_mu_i + LSE_j(arg4(f_i, g_j, C_ij, inv, lnu_j))) - mu_i|
//   kRowCost : out[i] = sum_j C_ij * exp(arg4(f_i,g_j,C_ij,inv,lmu_i) + lnu_j)
template <int MODE>
static __global__ void __launch_bounds__(256) k_row_lse(const float* __restrict__ C, long long ldc, int n, int m,
                                                  const float* __restrict__ rowv,   // f (check/cost)
                                                  const float* __restrict__ other,  // g / beta
                                                  const float* __restrict__ lw,     // log nu
                                                  const float* __restrict__ lrow,   // log mu (check/cost)
                                                  const float* __restrict__ murow,  // mu (check)
                                                  float inv_eps, float neg_eps, float* __restrict__ out,
                                                  const int* __restrict__ active = nullptr) {
  __shared__ float red[64];
  if (active && !*active) return;
  const int i = blockIdx.x;
  const float* Ci = C + (long long)i * ldc;
  if (MODE == kRowCost) {
    const float fi = rowv[i], li = lrow[i];
    float s[1] = {0.f};
    for (int j = threadIdx.x; j < m; j += 256) {
      float z = __fadd_rn(arg4(fi, other[j], Ci[j], inv_eps, li), lw[j]);
      s[0] += __fmul_rn(Ci[j], expf(z));
    }
    block_reduce<256, 1, false>(s, red);
    if (threadIdx.x == 0) out[i] = s[0];
    return;
  }
  const float fi = MODE == kRowCheck ? rowv[i] : 0.f;
  auto argf = [&](int j) {
    return MODE == kRowCheck ? arg4(fi, other[j], Ci[j], inv_eps, lw[j]) : arg3(other[j], Ci[j], inv_eps, lw[j]);
  };
  float mx[1] = {-INFINITY};
  for (int j = threadIdx.x; j < m; j += 256) mx[0] = fmax_nan(mx[0], argf(j));
  block_reduce<256, 1, true>(mx, red);
  const float M = mx[0];
  const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
  const float sl = __fmul_rn(Ms, kLog2e);
  float s[1] = {0.f};
  for (int j = threadIdx.x; j < m; j += 256) s[0] += exp_shifted(argf(j), sl);
  __syncthreads();
  block_reduce<256, 1, false>(s, red + 32);
  if (threadIdx.x == 0) {
    const float L = lse_finish(M, s[0]);
    if (MODE == kRowAlpha) out[i] = __fmul_rn(neg_eps, L);
    else out[i] = fabsf(__fsub_rn(expf(__fadd_rn(lrow[i], L)), murow[i]));
  }
}

// One-pass alpha row LSE for the m > 8192 loop: shifted by the stale row shift
// -f_i^{k-1} * inv_eps (as the fused solver); a row whose shifted
// sum leaves [1e-20, 1e30] (or whose previous f is not finite) redoes the exact
// two-pass LSE from L1/L2. One read of the row instead of two sweeps.
static __global__ void __launch_bounds__(256) k_row_alpha_stale(const float* __restrict__ C, long long ldc, int n,
                                                               int m, const float* __restrict__ fprev,
                                                               const float* __restrict__ other,
                                                               const float* __restrict__ lw, float inv_eps,
                                                               float neg_eps, float* __restrict__ out,
                                                               const int* __restrict__ active = nullptr) {
  __shared__ float red[64];
  if (active && !*active) return;
  const int i = blockIdx.x;
  const float* Ci = C + (long long)i * ldc;
  const float fo = fprev[i];
  float M = __fmul_rn(-fo, inv_eps);
  float s[1] = {0.f};
  if (isfinite(M)) {
    const float sl = __fmul_rn(M, kLog2e);
    for (int j = threadIdx.x; j < m; j += 256) s[0] += exp_shifted(arg3(other[j], Ci[j], inv_eps, lw[j]), sl);
    block_reduce<256, 1, false>(s, red);
  }
  __shared__ int redo;
  if (threadIdx.x == 0) redo = !(isfinite(M) && s[0] >= 1e-20f && s[0] <= 1e30f);
  __syncthreads();
  if (redo) {  // exact two-pass (reduction.py:179-208)
    float mx[1] = {-INFINITY};
    for (int j = threadIdx.x; j < m; j += 256) mx[0] = fmax_nan(mx[0], arg3(other[j], Ci[j], inv_eps, lw[j]));
    __syncthreads();
    block_reduce<256, 1, true>(mx, red);
    M = mx[0];
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    const float sl = __fmul_rn(Ms, kLog2e);
    s[0] = 0.f;
    for (int j = threadIdx.x; j < m; j += 256) s[0] += exp_shifted(arg3(other[j], Ci[j], inv_eps, lw[j]), sl);
    __syncthreads();
    block_reduce<256, 1, false>(s, red + 32);
  }
  if (threadIdx.x == 0) out[i] = __fmul_rn(neg_eps, lse_finish(M, s[0]));
}

// Column LSE of the beta argument y_ij = arg3(alpha_i, C_ij, inv, log_mu_i):
// CTA (bx, by) owns columns [bx*1024, +1024) (256 threads x float4, coalesced
// 4 KB row segments) and rows [by*rs, +rs); each thread keeps a chunked online
// (max, sumexp) per column. Partials [gridDim.y][m] are merged in fixed order.
static __global__ void __launch_bounds__(256) k_col_pairs(const float* __restrict__ C, long long ldc, int n, int m,
                                                    const float* __restrict__ alpha, const float* __restrict__ lmu,
                                                    float inv_eps, int rs, float2* __restrict__ pairs,
                                                    const int* __restrict__ active = nullptr) {
  if (active && !*active) return;
  const int j0 = (blockIdx.x * 256 + threadIdx.x) * 4;
  const int i0 = blockIdx.y * rs, i1 = min(n, i0 + rs);
  float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, sm[4] = {0.f, 0.f, 0.f, 0.f};
  constexpr int CH = 8;
  for (int i = i0; i < i1; i += CH) {
    float y[CH][4];
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int ii = i + r;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + q;
        y[r][q] = (ii < i1 && j < m) ? arg3(alpha[ii], C[(long long)ii * ldc + j], inv_eps, lmu[ii]) : -INFINITY;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float cm = -INFINITY;
#pragma unroll
      for (int r = 0; r < CH; ++r) cm = fmax_nan(cm, y[r][q]);
      const float mn = fmax_nan(mx[q], cm);
      const float ms = (fabsf(mn) <= 3.402823466e38f) ? mn : 0.f;
      const float sl = __fmul_rn(ms, kLog2e);
      float s = (mx[q] == -INFINITY) ? 0.f : sm[q] * exp_shifted(mx[q], sl);
#pragma unroll
      for (int r = 0; r < CH; ++r) s += exp_shifted(y[r][q], sl);
      mx[q] = mn;
      sm[q] = s;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (j0 + q < m) pairs[(size_t)blockIdx.y * m + j0 + q] = make_float2(mx[q], sm[q]);
}

static __global__ void k_col_combine(const float2* __restrict__ pairs, int parts, int m, float neg_eps,
                              float* __restrict__ out, const int* __restrict__ active = nullptr) {
  if (active && !*active) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  float mx = -INFINITY, s = 0.f;
  for (int p = 0; p < parts; ++p) {
    float2 v = pairs[(size_t)p * m + j];
    pair_merge(mx, s, v.x, v.y);
  }
  out[j] = __fmul_rn(neg_eps, lse_finish(mx, s));
}

// Fixed-order sum of `len` floats by one CTA of 1024 threads (thread t folds
// t, t+1024, ..., then the block tree). Writes out[0].
static __global__ void __launch_bounds__(1024) k_sum_fixed(const float* __restrict__ v, int len, float* __restrict__ out) {
  __shared__ float red[64];
  float s[1] = {0.f};
  for (int k = threadIdx.x; k < len; k += 1024) s[0] += v[k];
  block_reduce<1024, 1, false>(s, red);
  if (threadIdx.x == 0) out[0] = s[0];
}

// pi_ij = exp(fl(fl(fl(fl(fl(f_i + g_j) - C_ij) * inv) + lmu_i) + lnu_j)); counts non-finite
// entries (materialize_plan raises NonFiniteResult, solver.py:456-457).
static __global__ void k_plan(const float* __restrict__ C, long long ldc, int n, int m, const float* __restrict__ f,
                       const float* __restrict__ g, const float* __restrict__ lmu, const float* __restrict__ lnu,
                       float inv_eps, float* __restrict__ P, long long ldp, int* __restrict__ nonfinite) {
  int bad = 0;
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    const float fi = f[i], li = lmu[i];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
      float z = __fadd_rn(arg4(fi, g[j], C[(long long)i * ldc + j], inv_eps, li), lnu[j]);
      float p = expf(z);
      P[(long long)i * ldp + j] = p;
      bad |= !isfinite(p);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1);
}

// C_ij = fl32( scale64 * ((d0^2 + d1^2) + d2^2 ...) ), all fp64 and unfused, d_k = x_ik - y_jk:
// the reference's direct broadcast (costs.py:48-49), the (optional) fp64
// max-normalisation (applications.py:186-188: C64 / Cmax, pass 1/Cmax as
// scale... see below) and the single fp64->fp32 rounding of solver.py:253.
// When `div` is non-zero the value is C64 / div (true division, as numpy).
static __global__ void k_cost_build(const double* __restrict__ X, const double* __restrict__ Y, int n, int m, int d,
                             double div, float* __restrict__ C, long long ldc) {
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) {
        double t = __dsub_rn(X[(long long)i * d + k], Y[(long long)j * d + k]);
        acc = (k == 0) ? __dmul_rn(t, t) : __dadd_rn(acc, __dmul_rn(t, t));
      }
      if (div != 0.0) acc = __ddiv_rn(acc, div);
      C[(long long)i * ldc + j] = __double2float_rn(acc);
    }
}

// max and min over the fp64 cost (the pipeline normalises by C.max() only if
// max - min > 0, applications.py:186-188); per-CTA partials part[2*b], part[2*b+1]
static __global__ void k_cost_max(const double* __restrict__ X, const double* __restrict__ Y, int n, int m, int d,
                           double* __restrict__ part) {
  __shared__ double red[32], redn[32];
  double mx = -1.0, mn = INFINITY;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)n * m;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = int(idx / m), j = int(idx % m);
    double acc = 0.0;
    for (int k = 0; k < d; ++k) {
      double t = __dsub_rn(X[(long long)i * d + k], Y[(long long)j * d + k]);
      acc = (k == 0) ? __dmul_rn(t, t) : __dadd_rn(acc, __dmul_rn(t, t));
    }
    mx = fmax(mx, acc);
    mn = fmin(mn, acc);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = mx; redn[threadIdx.x >> 5] = mn; }
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -1.0;
    mn = threadIdx.x < blockDim.x / 32 ? redn[threadIdx.x] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = mx; part[2 * blockIdx.x + 1] = mn; }
  }
}

// dst (row stride ldd, zero-padded to ldd) = fl32(src) (row stride lds): the
// single fp64 -> fp32 rounding of solver.py:253, done on the device.
static __global__ void k_cast_pad(const double* __restrict__ src, long long lds, int n, int m, float* __restrict__ dst,
                           long long ldd) {
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < ldd; j += (long long)gridDim.x * blockDim.x)
      dst[(long long)i * ldd + j] = j < m ? __double2float_rn(src[(long long)i * lds + j]) : 0.f;
}
static __global__ void k_pad_f32(const float* __restrict__ src, long long lds, int n, int m, float* __restrict__ dst,
                          long long ldd) {
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < ldd; j += (long long)gridDim.x * blockDim.x)
      dst[(long long)i * ldd + j] = j < m ? src[(long long)i * lds + j] : 0.f;
}

// dst[i] = src[sel][i] where sel = *which (final-buffer pick after the solve)
static __global__ void k_pick(const float* __restrict__ s0, const float* __restrict__ s1, const int* __restrict__ which,
                       int len, float* __restrict__ dst) {
  const float* s = (*which) ? s1 : s0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) dst[i] = s[i];
}

}  // namespace lsk

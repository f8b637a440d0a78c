// Stand-alone kernels behind the reference's half-step / diagnostic API:
// update_alpha (solver.py:118-140), update_beta (143-176), marginal_error
// (179-206), transport_cost (209-227), materialize_plan (434-458), and the
// cost builder squared_euclidean_cost (costs.py:36-50). These handle any
// (n, m) and are the parity hooks for the pieces the persistent solver fuses.
#pragma once
#include "lsk_device.cuh"

namespace lsk {

enum RowMode { kRowAlpha = 0, kRowCheck = 1, kRowCost = 2 };

// ---- 128-bit access to a row of C and to the length-m column vectors. A row is
// read as float4 when C is 16-byte aligned and ldc % 4 == 0 (then the float4
// holding column j0 < m lies inside the row); otherwise, and for a vector that
// is unaligned or ends mid-float4, scalar loads (warp-uniform branches).
__device__ __forceinline__ float4 ldrow4(const float* __restrict__ row, int j0, int m = 0, bool vec = true) {
  if (vec) return __ldg(reinterpret_cast<const float4*>(row + j0));
  float4 r;
  r.x = j0 < m ? row[j0] : 0.f;
  r.y = j0 + 1 < m ? row[j0 + 1] : 0.f;
  r.z = j0 + 2 < m ? row[j0 + 2] : 0.f;
  r.w = j0 + 3 < m ? row[j0 + 3] : 0.f;
  return r;
}
__device__ __forceinline__ bool rows_vec(const float* C, long long ldc) {
  return (reinterpret_cast<uintptr_t>(C) & 15) == 0 && (ldc & 3) == 0;
}
__device__ __forceinline__ float4 ldvec4(const float* __restrict__ v, int j0, int m, bool aligned) {
  if (aligned && j0 + 3 < m) return __ldg(reinterpret_cast<const float4*>(v + j0));
  float4 r;
  r.x = j0 < m ? v[j0] : 0.f;
  r.y = j0 + 1 < m ? v[j0 + 1] : 0.f;
  r.z = j0 + 2 < m ? v[j0 + 2] : 0.f;
  r.w = j0 + 3 < m ? v[j0 + 3] : 0.f;
  return r;
}
__device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
__device__ __forceinline__ float comp(const float4& v, int u) { return u == 0 ? v.x : u == 1 ? v.y : u == 2 ? v.z : v.w; }

// One CTA (256 threads) per row, two-pass LSE over the row (max, then the
// shifted sum, recomputing the argument -- reduction.py:179-208); 128-bit loads
// of C and of the column vectors, four float4 per thread in flight, the second
// sweep from L1/L2. mode:
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
  const int m4 = (m + 3) >> 2;
  const bool alg = al16(other) && al16(lw), vec = rows_vec(C, ldc);
  if (MODE == kRowCost) {
    const float fi = rowv[i], li = lrow[i];
    float s[1] = {0.f};
#pragma unroll 4
    for (int q = threadIdx.x; q < m4; q += 256) {
      const int j0 = 4 * q;
      const float4 c = ldrow4(Ci, j0, m, vec), g = ldvec4(other, j0, m, alg), l = ldvec4(lw, j0, m, alg);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < m) {
          const float z = __fadd_rn(arg4(fi, comp(g, u), comp(c, u), inv_eps, li), comp(l, u));
          s[0] += __fmul_rn(comp(c, u), expf(z));
        }
    }
    block_reduce<256, 1, false>(s, red);
    if (threadIdx.x == 0) out[i] = s[0];
    return;
  }
  const float fi = MODE == kRowCheck ? rowv[i] : 0.f;
  auto argf = [&](float g, float c, float l) {
    return MODE == kRowCheck ? arg4(fi, g, c, inv_eps, l) : arg3(g, c, inv_eps, l);
  };
  float mx[1] = {-INFINITY};
#pragma unroll 4
  for (int q = threadIdx.x; q < m4; q += 256) {
    const int j0 = 4 * q;
    const float4 c = ldrow4(Ci, j0, m, vec), g = ldvec4(other, j0, m, alg), l = ldvec4(lw, j0, m, alg);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u < m) mx[0] = fmax_nan(mx[0], argf(comp(g, u), comp(c, u), comp(l, u)));
  }
  block_reduce<256, 1, true>(mx, red);
  const float M = mx[0];
  const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
  const float sl = __fmul_rn(Ms, kLog2e);
  float s[1] = {0.f};
#pragma unroll 4
  for (int q = threadIdx.x; q < m4; q += 256) {
    const int j0 = 4 * q;
    const float4 c = ldrow4(Ci, j0, m, vec), g = ldvec4(other, j0, m, alg), l = ldvec4(lw, j0, m, alg);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u < m) s[0] += exp_shifted(argf(comp(g, u), comp(c, u), comp(l, u)), sl);
  }
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
// two-pass LSE from L1/L2. One read of the row instead of two sweeps, 128-bit
// loads with four float4 of C per thread in flight. CHECK: the same read also
// forms the marginal-error term of iterate k-1 (solver.py:97-104; argument
// arg4(f^{k-1}_i, g^{k-1}_j, C_ij) with shift 0, exact two-pass fallback), so a
// checkpoint costs no extra pass over C. UNI: log nu is one value (uniform
// targets), read once instead of per column.
template <bool CHECK, bool UNI>
static __global__ void __launch_bounds__(256) k_row_alpha_stale(const float* __restrict__ C, long long ldc, int n,
                                                               int m, const float* __restrict__ fprev,
                                                               const float* __restrict__ other,
                                                               const float* __restrict__ lw, float inv_eps,
                                                               float neg_eps, float* __restrict__ out,
                                                               const int* __restrict__ active,
                                                               const float* __restrict__ lrow = nullptr,
                                                               const float* __restrict__ murow = nullptr,
                                                               float* __restrict__ rowterm = nullptr) {
  __shared__ float red[128];
  if (active && !*active) return;
  const int i = blockIdx.x;
  const float* Ci = C + (long long)i * ldc;
  const int m4 = (m + 3) >> 2;
  const bool alg = al16(other) && (UNI || al16(lw)), vec = rows_vec(C, ldc);
  const float lw0 = UNI ? __ldg(lw) : 0.f;
  const float fo = fprev[i];
  float M = __fmul_rn(-fo, inv_eps);
  float s[2] = {0.f, 0.f};
  const bool okM = isfinite(M);
  {
    const float sl = okM ? __fmul_rn(M, kLog2e) : 0.f;
#pragma unroll 4
    for (int q = threadIdx.x; q < m4; q += 256) {
      const int j0 = 4 * q;
      const float4 c = ldrow4(Ci, j0, m, vec), g = ldvec4(other, j0, m, alg);
      const float4 l = UNI ? make_float4(lw0, lw0, lw0, lw0) : ldvec4(lw, j0, m, alg);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < m) {
          if (okM) s[0] += exp_shifted(arg3(comp(g, u), comp(c, u), inv_eps, comp(l, u)), sl);
          if (CHECK) s[1] += ex2(__fmul_rn(arg4(fo, comp(g, u), comp(c, u), inv_eps, comp(l, u)), kLog2e));
        }
    }
    if (CHECK) block_reduce<256, 2, false>(s, red);
    else block_reduce<256, 1, false>(*reinterpret_cast<float(*)[1]>(s), red);
  }
  auto lwj = [&](int j) { return UNI ? lw0 : lw[j]; };
  __shared__ int redo;
  if (threadIdx.x == 0) redo = !(okM && s[0] >= 1e-20f && s[0] <= 1e30f);
  __syncthreads();
  if (redo) {  // exact two-pass (reduction.py:179-208)
    float mx[1] = {-INFINITY};
    for (int j = threadIdx.x; j < m; j += 256) mx[0] = fmax_nan(mx[0], arg3(other[j], Ci[j], inv_eps, lwj(j)));
    __syncthreads();
    block_reduce<256, 1, true>(mx, red + 64);
    M = mx[0];
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    const float sl = __fmul_rn(Ms, kLog2e);
    float t[1] = {0.f};
    for (int j = threadIdx.x; j < m; j += 256) t[0] += exp_shifted(arg3(other[j], Ci[j], inv_eps, lwj(j)), sl);
    __syncthreads();
    block_reduce<256, 1, false>(t, red + 96);
    s[0] = t[0];
  }
  if (threadIdx.x == 0) out[i] = __fmul_rn(neg_eps, lse_finish(M, s[0]));
  if (CHECK) {
    float Mz = 0.f, Sz = s[1];
    if (!(Sz >= 1e-20f && Sz <= 1e30f)) {  // block-uniform: exact two-pass of the check argument
      float mx[1] = {-INFINITY};
      for (int j = threadIdx.x; j < m; j += 256) mx[0] = fmax_nan(mx[0], arg4(fo, other[j], Ci[j], inv_eps, lwj(j)));
      __syncthreads();
      block_reduce<256, 1, true>(mx, red + 64);
      Mz = mx[0];
      const float Ms = (fabsf(Mz) <= 3.402823466e38f) ? Mz : 0.f;
      const float sl = __fmul_rn(Ms, kLog2e);
      float t[1] = {0.f};
      for (int j = threadIdx.x; j < m; j += 256) t[0] += exp_shifted(arg4(fo, other[j], Ci[j], inv_eps, lwj(j)), sl);
      __syncthreads();
      block_reduce<256, 1, false>(t, red + 96);
      Sz = t[0];
    }
    if (threadIdx.x == 0) rowterm[i] = fabsf(__fsub_rn(expf(__fadd_rn(lrow[i], lse_finish(Mz, Sz))), murow[i]));
  }
}

// Column LSE of the beta argument y_ij = arg3(alpha_i, C_ij, inv, log_mu_i):
// CTA (bx, by) owns columns [bx*1024, +1024) (256 threads x float4, coalesced
// 4 KB row segments) and rows [by*rs, +rs); each thread keeps a chunked online
// (max, sumexp) per column, with the next chunk's 8 row segments loaded while
// the current one is reduced. Partials [gridDim.y][m] are merged in fixed order.
static __global__ void __launch_bounds__(256) k_col_pairs(const float* __restrict__ C, long long ldc, int n, int m,
                                                    const float* __restrict__ alpha, const float* __restrict__ lmu,
                                                    float inv_eps, int rs, float2* __restrict__ pairs,
                                                    const int* __restrict__ active = nullptr) {
  if (active && !*active) return;
  const int j0 = (blockIdx.x * 256 + threadIdx.x) * 4;
  const int i0 = blockIdx.y * rs, i1 = min(n, i0 + rs);
  const bool vec = rows_vec(C, ldc);
  float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, sm[4] = {0.f, 0.f, 0.f, 0.f};
  constexpr int CH = 8;
  float4 cn[CH];
  float an[CH], ln[CH];
  auto fetch = [&](int i) {
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int ii = i + r;
      cn[r] = make_float4(0.f, 0.f, 0.f, 0.f);
      an[r] = 0.f;
      ln[r] = 0.f;
      if (ii < i1 && j0 < m) {  // one 128-bit load of the row segment
        cn[r] = ldrow4(C + (long long)ii * ldc, j0, m, vec);
        an[r] = __ldg(alpha + ii);
        ln[r] = __ldg(lmu + ii);
      }
    }
  };
  if (i0 < i1) fetch(i0);
  for (int i = i0; i < i1; i += CH) {
    float y[CH][4];
#pragma unroll
    for (int r = 0; r < CH; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        y[r][q] = (i + r < i1 && j0 + q < m) ? arg3(an[r], comp(cn[r], q), inv_eps, ln[r]) : -INFINITY;
    if (i + CH < i1) fetch(i + CH);
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

// Fixed-order merge of the [parts][m] column pairs: 8 threads per column, thread
// t of the group merges parts t, t + 8, ... in order, then a fixed xor tree
// over the group (identical bits on every call; the reference's own fold order
// is not reproduced by any fp32 path, SURVEY 8(a')).
static __global__ void k_col_combine(const float2* __restrict__ pairs, int parts, int m, float neg_eps,
                              float* __restrict__ out, const int* __restrict__ active = nullptr) {
  if (active && !*active) return;
  const int t = threadIdx.x & 7;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  float mx = -INFINITY, s = 0.f;
  if (j < m)
    for (int p = t; p < parts; p += 8) {
      const float2 v = __ldg(pairs + (size_t)p * m + j);
      pair_merge(mx, s, v.x, v.y);
    }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    // merge in a fixed operand order (lower group index first): identical in both partners
    if (t & o) { float a = m2, b = s2; pair_merge(a, b, mx, s); mx = a; s = b; }
    else pair_merge(mx, s, m2, s2);
  }
  if (j < m && t == 0) out[j] = __fmul_rn(neg_eps, lse_finish(mx, s));
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

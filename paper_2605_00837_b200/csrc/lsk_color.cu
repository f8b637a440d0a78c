// Colour-transfer pipeline kernels, fp64 like the
// reference pipeline (applications.py:100-107 solves in double):
//
//  * lsk_build_cost_f64: C_ij = sum_k (x_ik - y_jk)^2 in fp64, coordinates in
//    order, never contracted -- bit-identical to costs.py:36-50's broadcast
//    (the fp32 builder k_cost_build uses the same loop, rounded once);
//  * lsk_barycentric_points_f64: mapped_i = sum_j pi_ij t_j / sum_j pi_ij with
//    pi_ij = exp(((a_i + b_j) - C_ij) * inv_eps + log mu_i + log nu_j)
//    (materialize_plan solver.py:434-458 followed by barycentric_map
//    applications.py:75-97) with C_ij recomputed from the points, so the
//    (n, m) plan is never written;
//  * lsk_recolor_nearest_f64: every pixel takes the mapped colour of its
//    nearest source sample in RGB, ties to the lowest sample index, clamped to
//    [0, 1] (applications.py:149-160). The distance is the reference's
//    ((d0*d0 + d1*d1) + d2*d2) in fp64, so the argmin is bit-exact.
#include <cmath>
#include <string>

#include "../../include/lsk.h"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace {

#define C_CUDA(expr)                                                                                    \
  do {                                                                                                  \
    cudaError_t e__ = (expr);                                                                           \
    if (e__ != cudaSuccess) return lsk_host::fail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

inline cudaStream_t Sc(void* s) { return static_cast<cudaStream_t>(s); }

constexpr int kMaxDim = 8;

// fp64 squared distance in coordinate order (costs.py:36-50): the first term
// is the product itself, then sequential adds; separately rounded ops
__device__ __forceinline__ double sqdist(const double* __restrict__ x, const double* __restrict__ y, int d) {
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = __dsub_rn(x[k], y[k]);
    acc = (k == 0) ? __dmul_rn(t, t) : __dadd_rn(acc, __dmul_rn(t, t));
  }
  return acc;
}

__global__ void k_cost_build_d(const double* __restrict__ X, const double* __restrict__ Y, int n, int m, int d,
                               double div, double* __restrict__ C, long long ldc) {
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    const double* x = X + (long long)i * d;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
      double c = sqdist(x, Y + (long long)j * d, d);
      if (div != 0.0) c = __ddiv_rn(c, div);
      C[(long long)i * ldc + j] = c;
    }
  }
}

// one warp per source row: lanes stride the target points, fixed-order warp
// butterfly at the end (deterministic); flags[0] += rows with a non-finite
// weight, flags[1] += rows with zero mass
template <int DT>
__global__ void __launch_bounds__(256) k_bary_d(const double* __restrict__ X, const double* __restrict__ Y,
                                                const double* __restrict__ T, int n, int m, int d, double div,
                                                const double* __restrict__ lmu, const double* __restrict__ lnu,
                                                const double* __restrict__ f, const double* __restrict__ g,
                                                double inv, double* __restrict__ mapped, int* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    double x[kMaxDim];
    for (int k = 0; k < d; ++k) x[k] = X[(long long)i * d + k];
    const double fi = f[i], lmi = lmu[i];
    double den = 0.0, num[DT];
#pragma unroll
    for (int k = 0; k < DT; ++k) num[k] = 0.0;
    int bad = 0;
    for (int j = lane; j < m; j += 32) {
      double c = sqdist(x, Y + (long long)j * d, d);
      if (div != 0.0) c = __ddiv_rn(c, div);
      // materialize_plan: Z = a + b; Z -= C; Z *= inv_eps; Z += log mu; Z += log nu
      const double z = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(__dadd_rn(fi, g[j]), c), inv), lmi), lnu[j]);
      const double p = exp(z);
      bad |= !isfinite(p);
      den = __dadd_rn(den, p);
#pragma unroll
      for (int k = 0; k < DT; ++k) num[k] = __dadd_rn(num[k], __dmul_rn(p, T[(long long)j * DT + k]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      den = __dadd_rn(den, __shfl_xor_sync(0xffffffffu, den, o));
#pragma unroll
      for (int k = 0; k < DT; ++k) num[k] = __dadd_rn(num[k], __shfl_xor_sync(0xffffffffu, num[k], o));
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (bad) atomicAdd(flags + 0, 1);
      if (den == 0.0) atomicAdd(flags + 1, 1);
#pragma unroll
      for (int k = 0; k < DT; ++k) mapped[(long long)i * DT + k] = __ddiv_rn(num[k], den);
    }
  }
}

// nearest source sample per pixel (RGB), samples staged through shared memory
// in tiles; each thread owns PX pixels
constexpr int kTile = 2048;
constexpr int kPx = 2;
__global__ void __launch_bounds__(256) k_recolor_d(const double* __restrict__ pix, long long N,
                                                   const double* __restrict__ smp, int S,
                                                   const double* __restrict__ mapped, double* __restrict__ out,
                                                   int* __restrict__ nearest) {
  __shared__ double sx[kTile], sy[kTile], sz[kTile];
  const long long base = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kPx;
  double p[kPx][3], best[kPx];
  int bi[kPx];
#pragma unroll
  for (int u = 0; u < kPx; ++u) {
    const long long q = base + u;
    const bool ok = q < N;
#pragma unroll
    for (int k = 0; k < 3; ++k) p[u][k] = ok ? pix[q * 3 + k] : 0.0;
    best[u] = INFINITY;
    bi[u] = 0;
  }
  for (int t0 = 0; t0 < S; t0 += kTile) {
    const int tn = min(kTile, S - t0);
    __syncthreads();
    for (int s = threadIdx.x; s < tn; s += blockDim.x) {
      sx[s] = smp[(long long)(t0 + s) * 3 + 0];
      sy[s] = smp[(long long)(t0 + s) * 3 + 1];
      sz[s] = smp[(long long)(t0 + s) * 3 + 2];
    }
    __syncthreads();
    for (int s = 0; s < tn; ++s) {
      const double a = sx[s], b = sy[s], c = sz[s];
#pragma unroll
      for (int u = 0; u < kPx; ++u) {
        const double d0 = __dsub_rn(p[u][0], a), d1 = __dsub_rn(p[u][1], b), d2 = __dsub_rn(p[u][2], c);
        const double dd = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
        if (dd < best[u]) {  // strict: ties keep the lowest sample index (np.argmin)
          best[u] = dd;
          bi[u] = t0 + s;
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kPx; ++u) {
    const long long q = base + u;
    if (q >= N) continue;
    if (nearest) nearest[q] = bi[u];
#pragma unroll
    for (int k = 0; k < 3; ++k) out[q * 3 + k] = fmin(fmax(mapped[(long long)bi[u] * 3 + k], 0.0), 1.0);
  }
}

}  // namespace

extern "C" {

int32_t lsk_build_cost_f64(const double* X, const double* Y, int32_t n, int32_t m, int32_t d, double div,
                           double* C, int64_t ldc, void* stream) {
  if (!X || !Y || !C) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || d < 1 || ldc < m) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  int bx = (m + 255) / 256;
  if (bx > 32) bx = 32;
  k_cost_build_d<<<dim3(bx, n < 65535 ? n : 65535), 256, 0, Sc(stream)>>>(X, Y, n, m, d, div, C, ldc);
  C_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_barycentric_points_f64(const double* X, const double* Y, const double* T, int32_t n, int32_t m,
                                   int32_t d, int32_t dt, double div, const double* log_mu, const double* log_nu,
                                   const double* alpha, const double* beta, double eps, double* mapped,
                                   int32_t* flags, void* stream) {
  if (!X || !Y || !T || !log_mu || !log_nu || !alpha || !beta || !mapped || !flags)
    return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || d < 1 || d > kMaxDim || !(eps > 0)) return lsk_host::fail(LSK_EINVAL, "bad arguments");
  const double inv = 1.0 / eps;
  const int blocks = (n + 7) / 8;
  const cudaStream_t s = Sc(stream);
  switch (dt) {
    case 1: k_bary_d<1><<<blocks, 256, 0, s>>>(X, Y, T, n, m, d, div, log_mu, log_nu, alpha, beta, inv, mapped, flags); break;
    case 2: k_bary_d<2><<<blocks, 256, 0, s>>>(X, Y, T, n, m, d, div, log_mu, log_nu, alpha, beta, inv, mapped, flags); break;
    case 3: k_bary_d<3><<<blocks, 256, 0, s>>>(X, Y, T, n, m, d, div, log_mu, log_nu, alpha, beta, inv, mapped, flags); break;
    case 4: k_bary_d<4><<<blocks, 256, 0, s>>>(X, Y, T, n, m, d, div, log_mu, log_nu, alpha, beta, inv, mapped, flags); break;
    default: return lsk_host::fail(LSK_EINVAL, "target dimension must be 1..4");
  }
  C_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_recolor_nearest_f64(const double* pixels, int64_t n_pixels, const double* samples, int32_t n_samples,
                                const double* mapped, double* out, int32_t* nearest, void* stream) {
  if (!pixels || !samples || !mapped || !out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n_pixels < 0 || n_samples < 1) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  if (n_pixels == 0) return LSK_OK;
  const long long per = 256LL * kPx;
  const long long blocks = (n_pixels + per - 1) / per;
  if (blocks > 0x7fffffffLL) return lsk_host::fail(LSK_EINVAL, "too many pixels");
  k_recolor_d<<<unsigned(blocks), 256, 0, Sc(stream)>>>(pixels, n_pixels, samples, n_samples, mapped, out, nearest);
  C_CUDA(cudaGetLastError());
  return LSK_OK;
}

}  // extern "C"

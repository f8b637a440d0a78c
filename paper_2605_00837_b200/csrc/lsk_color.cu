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
//    ((d0*d0 + d1*d1) + d2*d2) in fp64, so the argmin is bit-exact;
//  * lsk_nearest_map_f64: the same lookup for d = 1..4 without the clamp
//    (SinkhornTransport.transform, estimator.py:118-132).
#include <cmath>
#include <string>

#include "../../include/lsk.h"
#include "lsk_kernels.cuh"

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

// barycentric map of a materialised plan (barycentric_map, applications.py:75-97):
// one warp per row, lanes stride the columns, fixed-order butterfly; flags[1]
// += rows whose total mass is zero (ZeroRowMass)
template <int DT>
__global__ void __launch_bounds__(256) k_bary_plan_d(const double* __restrict__ P, long long ldp, int n, int m,
                                                     const double* __restrict__ T, double* __restrict__ mapped,
                                                     int* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const double* row = P + (long long)i * ldp;
    double den = 0.0, num[DT];
#pragma unroll
    for (int k = 0; k < DT; ++k) num[k] = 0.0;
    for (int j = lane; j < m; j += 32) {
      const double p = row[j];
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
    if (lane == 0) {
      if (den == 0.0) atomicAdd(flags + 1, 1);
#pragma unroll
      for (int k = 0; k < DT; ++k) mapped[(long long)i * DT + k] = __ddiv_rn(num[k], den);
    }
  }
}

// nearest sample per query point (D coordinates), samples staged through
// shared memory in tiles; each thread owns kPx queries. The distance is the
// reference's sequential fp64 sum of squared differences, the argmin strict
// (ties keep the lowest sample index, np.argmin); out = mapped[nearest]
// (DM values per sample), clamped to [0, 1] for the colour pipeline.
constexpr int kTile = 1536;  // D x kTile doubles of static shared memory (<= 48 KB at D = 4)
constexpr int kPx = 2;
template <int D, int DM>
__global__ void __launch_bounds__(256) k_nearest_d(const double* __restrict__ q, long long N,
                                                   const double* __restrict__ smp, int S,
                                                   const double* __restrict__ mapped, int clamp,
                                                   double* __restrict__ out, int* __restrict__ nearest) {
  __shared__ double sm[D][kTile];
  const long long base = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kPx;
  double p[kPx][D], best[kPx];
  int bi[kPx];
#pragma unroll
  for (int u = 0; u < kPx; ++u) {
    const long long r = base + u;
    const bool ok = r < N;
#pragma unroll
    for (int k = 0; k < D; ++k) p[u][k] = ok ? q[r * D + k] : 0.0;
    best[u] = INFINITY;
    bi[u] = 0;
  }
  for (int t0 = 0; t0 < S; t0 += kTile) {
    const int tn = min(kTile, S - t0);
    __syncthreads();
    for (int s = threadIdx.x; s < tn; s += blockDim.x)
#pragma unroll
      for (int k = 0; k < D; ++k) sm[k][s] = smp[(long long)(t0 + s) * D + k];
    __syncthreads();
    for (int s = 0; s < tn; ++s) {
#pragma unroll
      for (int u = 0; u < kPx; ++u) {
        double dd = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const double t = __dsub_rn(p[u][k], sm[k][s]);
          dd = (k == 0) ? __dmul_rn(t, t) : __dadd_rn(dd, __dmul_rn(t, t));
        }
        if (dd < best[u]) {  // strict: ties keep the lowest sample index
          best[u] = dd;
          bi[u] = t0 + s;
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kPx; ++u) {
    const long long r = base + u;
    if (r >= N) continue;
    if (nearest) nearest[r] = bi[u];
#pragma unroll
    for (int k = 0; k < DM; ++k) {
      const double v = mapped[(long long)bi[u] * DM + k];
      out[r * DM + k] = clamp ? fmin(fmax(v, 0.0), 1.0) : v;
    }
  }
}

}  // namespace

extern "C" {

int32_t lsk_build_cost_f64(const double* X, const double* Y, int32_t n, int32_t m, int32_t d, int32_t normalize_max,
                           double* C, int64_t ldc, double* cmax_out, void* workspace, size_t workspace_bytes,
                           void* stream) {
  if (!X || !Y || !C) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || d < 1 || ldc < m) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  cudaStream_t st = Sc(stream);
  double div = 0.0;
  if (normalize_max || cmax_out) {
    // exact max / min of the fp64 cost (order independent), as lsk_build_cost_f32
    if (!workspace || workspace_bytes < lsk_build_cost_workspace_bytes())
      return lsk_host::fail(LSK_EINVAL, "workspace too small");
    double* part = static_cast<double*>(workspace);
    const int blocks = 2048;
    lsk::k_cost_max<<<blocks, 256, 0, st>>>(X, Y, n, m, d, part);
    double host[2 * 2048];
    C_CUDA(cudaMemcpyAsync(host, part, sizeof(host), cudaMemcpyDeviceToHost, st));
    C_CUDA(cudaStreamSynchronize(st));
    double mx = -1.0, mn = INFINITY;
    for (int k = 0; k < blocks; ++k) {
      mx = host[2 * k] > mx ? host[2 * k] : mx;
      mn = host[2 * k + 1] < mn ? host[2 * k + 1] : mn;
    }
    if (cmax_out) C_CUDA(cudaMemcpyAsync(cmax_out, &mx, sizeof(double), cudaMemcpyHostToDevice, st));
    if (normalize_max && (mx - mn) > 0.0) div = mx;  // cost.value_range > 0 (estimator.py:87-89)
    C_CUDA(cudaStreamSynchronize(st));
  }
  int bx = (m + 255) / 256;
  if (bx > 32) bx = 32;
  k_cost_build_d<<<dim3(bx, n < 65535 ? n : 65535), 256, 0, st>>>(X, Y, n, m, d, div, C, ldc);
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

int32_t lsk_barycentric_plan_f64(const double* P, int64_t ldp, int32_t n, int32_t m, const double* T, int32_t dt,
                                 double* mapped, int32_t* flags, void* stream) {
  if (!P || !T || !mapped || !flags) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldp < m) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  const int blocks = (n + 7) / 8;
  const cudaStream_t s = Sc(stream);
  switch (dt) {
    case 1: k_bary_plan_d<1><<<blocks, 256, 0, s>>>(P, ldp, n, m, T, mapped, flags); break;
    case 2: k_bary_plan_d<2><<<blocks, 256, 0, s>>>(P, ldp, n, m, T, mapped, flags); break;
    case 3: k_bary_plan_d<3><<<blocks, 256, 0, s>>>(P, ldp, n, m, T, mapped, flags); break;
    case 4: k_bary_plan_d<4><<<blocks, 256, 0, s>>>(P, ldp, n, m, T, mapped, flags); break;
    default: return lsk_host::fail(LSK_EINVAL, "target dimension must be 1..4");
  }
  C_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_nearest_map_f64(const double* queries, int64_t n_queries, int32_t d, const double* samples,
                            int32_t n_samples, const double* mapped, int32_t dm, int32_t clamp01, double* out,
                            int32_t* nearest, void* stream) {
  if (!queries || !samples || !mapped || !out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n_queries < 0 || n_samples < 1) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  if (d < 1 || d > 4 || dm != d) return lsk_host::fail(LSK_EINVAL, "point dimension must be 1..4 (mapped alike)");
  if (n_queries == 0) return LSK_OK;
  const long long per = 256LL * kPx;
  const long long blocks = (n_queries + per - 1) / per;
  if (blocks > 0x7fffffffLL) return lsk_host::fail(LSK_EINVAL, "too many query points");
  const cudaStream_t s = Sc(stream);
  const unsigned g = unsigned(blocks);
  switch (d) {
    case 1: k_nearest_d<1, 1><<<g, 256, 0, s>>>(queries, n_queries, samples, n_samples, mapped, clamp01, out, nearest); break;
    case 2: k_nearest_d<2, 2><<<g, 256, 0, s>>>(queries, n_queries, samples, n_samples, mapped, clamp01, out, nearest); break;
    case 3: k_nearest_d<3, 3><<<g, 256, 0, s>>>(queries, n_queries, samples, n_samples, mapped, clamp01, out, nearest); break;
    default: k_nearest_d<4, 4><<<g, 256, 0, s>>>(queries, n_queries, samples, n_samples, mapped, clamp01, out, nearest); break;
  }
  C_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_recolor_nearest_f64(const double* pixels, int64_t n_pixels, const double* samples, int32_t n_samples,
                                const double* mapped, double* out, int32_t* nearest, void* stream) {
  return lsk_nearest_map_f64(pixels, n_pixels, 3, samples, n_samples, mapped, 3, 1, out, nearest, stream);
}

}  // extern "C"

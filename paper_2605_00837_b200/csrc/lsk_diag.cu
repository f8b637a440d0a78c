// Plan diagnostics of the reference (solver.py:461-519) on the GPU:
//
//  * kkt_residual: max over entries with P_ij >= tiny(dt) of
//    |C_ij + eps * log(P_ij / (mu_i nu_j)) - alpha_i - beta_j| in the plan's
//    precision, evaluated in the reference's order (outer product first, the
//    ratio, then C + eps*ratio, minus alpha, minus beta). A max is order
//    independent, so the result differs from the reference only by the log's ulps;
//  * regularized_objective: <C, P> + eps (sum_ij P_ij (log(P_ij/(mu_i nu_j)) - 1) + 1)
//    in fp64, zero-mass entries contributing 0, per-row sums in a fixed order.
#include <cmath>
#include <string>

#include "../../include/lsk.h"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace {

#define D_CUDA(expr)                                                                                    \
  do {                                                                                                  \
    cudaError_t e__ = (expr);                                                                           \
    if (e__ != cudaSuccess) return lsk_host::fail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

template <class T> struct DN;
template <> struct DN<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float lg(float x) { return logf(x); }
  static constexpr float tiny = 1.17549435e-38f;
};
template <> struct DN<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double lg(double x) { return log(x); }
  static constexpr double tiny = 2.2250738585072014e-308;
};

// max |resid| over masked entries; bits of a non-negative double compare like
// unsigned integers, so atomicMax on them is exact and order independent.
// A NaN residual is recorded through flag (numpy's max would return NaN).
template <class T>
__global__ void k_kkt(const T* __restrict__ C, const T* __restrict__ P, long long ld, int n, int m,
                      const T* __restrict__ mu, const T* __restrict__ nu, const T* __restrict__ a,
                      const T* __restrict__ b, T eps, unsigned long long* mx, int* nmask, int* nan_flag) {
  double best = 0.0;
  int cnt = 0, isnan_ = 0;
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
      const T p = P[(long long)i * ld + j];
      if (!(p >= DN<T>::tiny)) continue;
      ++cnt;
      const T outer = DN<T>::mul(mu[i], nu[j]);
      const T ratio = DN<T>::lg(DN<T>::div(p, outer));
      T r = DN<T>::add(C[(long long)i * ld + j], DN<T>::mul(eps, ratio));
      r = DN<T>::sub(DN<T>::sub(r, a[i]), b[j]);
      const double v = fabs((double)r);
      if (v != v) isnan_ = 1;
      else best = v > best ? v : best;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  isnan_ = __reduce_or_sync(0xffffffffu, isnan_);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(mx, (unsigned long long)__double_as_longlong(best));
    if (cnt) atomicAdd(nmask, cnt);
    if (isnan_) atomicOr(nan_flag, 1);
  }
}

// per-row (sum C P, sum P (log(P/outer) - 1)) in fp64, lanes strided, fixed-order warp+block tree
__global__ void __launch_bounds__(256) k_regobj_rows(const double* __restrict__ C, const double* __restrict__ P,
                                                     long long ld, int n, int m, const double* __restrict__ mu,
                                                     const double* __restrict__ nu, double* __restrict__ rows) {
  __shared__ double sh[2][8];
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    double cp = 0.0, kl = 0.0;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      const double p = P[(long long)i * ld + j];
      cp = __dadd_rn(cp, __dmul_rn(C[(long long)i * ld + j], p));
      if (p > 0.0) kl = __dadd_rn(kl, __dmul_rn(p, __dsub_rn(log(__ddiv_rn(p, __dmul_rn(mu[i], nu[j]))), 1.0)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cp = __dadd_rn(cp, __shfl_xor_sync(0xffffffffu, cp, o));
      kl = __dadd_rn(kl, __shfl_xor_sync(0xffffffffu, kl, o));
    }
    if ((threadIdx.x & 31) == 0) { sh[0][threadIdx.x >> 5] = cp; sh[1][threadIdx.x >> 5] = kl; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < 8; ++w) { a = __dadd_rn(a, sh[0][w]); b = __dadd_rn(b, sh[1][w]); }
      rows[2 * (long long)i] = a;
      rows[2 * (long long)i + 1] = b;
    }
    __syncthreads();
  }
}

__global__ void k_regobj_finish(const double* __restrict__ rows, int n, double eps, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double cp = 0.0, kl = 0.0;
  for (int i = 0; i < n; ++i) { cp = __dadd_rn(cp, rows[2 * i]); kl = __dadd_rn(kl, rows[2 * i + 1]); }
  *out = __dadd_rn(cp, __dmul_rn(eps, __dadd_rn(kl, 1.0)));
}

}  // namespace

extern "C" {

int32_t lsk_kkt_residual(const void* C, const void* P, int64_t ld, int32_t n, int32_t m, const void* mu,
                         const void* nu, const void* alpha, const void* beta, double eps, int32_t dtype,
                         double* out_max, int32_t* out_count, void* workspace, size_t workspace_bytes, void* stream) {
  if (!C || !P || !mu || !nu || !alpha || !beta || !out_max || !out_count) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ld < m) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  if (!workspace || workspace_bytes < 16) return lsk_host::fail(LSK_EINVAL, "workspace too small (16 bytes)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* mx = static_cast<unsigned long long*>(workspace);
  int* flag = reinterpret_cast<int*>(mx + 1);
  D_CUDA(cudaMemsetAsync(workspace, 0, 16, st));
  D_CUDA(cudaMemsetAsync(out_count, 0, 4, st));
  int bx = (m + 255) / 256;
  if (bx > 32) bx = 32;
  const dim3 g(bx, n < 4096 ? n : 4096);
  if (dtype == 0)
    k_kkt<float><<<g, 256, 0, st>>>(static_cast<const float*>(C), static_cast<const float*>(P), ld, n, m,
                                    static_cast<const float*>(mu), static_cast<const float*>(nu),
                                    static_cast<const float*>(alpha), static_cast<const float*>(beta), float(eps),
                                    mx, out_count, flag);
  else
    k_kkt<double><<<g, 256, 0, st>>>(static_cast<const double*>(C), static_cast<const double*>(P), ld, n, m,
                                     static_cast<const double*>(mu), static_cast<const double*>(nu),
                                     static_cast<const double*>(alpha), static_cast<const double*>(beta), eps, mx,
                                     out_count, flag);
  D_CUDA(cudaGetLastError());
  // result: the max (as double) or NaN when a masked residual was NaN
  D_CUDA(cudaMemcpyAsync(out_max, mx, 8, cudaMemcpyDeviceToDevice, st));
  D_CUDA(cudaMemcpyAsync(out_count + 1, flag, 4, cudaMemcpyDeviceToDevice, st));
  return LSK_OK;
}

int32_t lsk_regularized_objective_f64(const double* C, const double* P, int64_t ld, int32_t n, int32_t m,
                                      const double* mu, const double* nu, double eps, double* out, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  if (!C || !P || !mu || !nu || !out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ld < m) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  if (!workspace || workspace_bytes < 16 * (size_t)n) return lsk_host::fail(LSK_EINVAL, "workspace too small (16 n bytes)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* rows = static_cast<double*>(workspace);
  k_regobj_rows<<<n < 8192 ? n : 8192, 256, 0, st>>>(C, P, ld, n, m, mu, nu, rows);
  k_regobj_finish<<<1, 32, 0, st>>>(rows, n, eps, out);
  D_CUDA(cudaGetLastError());
  return LSK_OK;
}

}  // extern "C"

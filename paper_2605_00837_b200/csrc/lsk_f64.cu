// fp64 path (precision="double", and the half-steps called with float64
// potentials): the reference's double-precision solve on the GPU.
//
// Reference: solver.py:230-337 with dt = float64 (types.py:168-170); the
// half-steps 118-227 and materialize_plan 434-458 follow the potentials' dtype
// (solver.py:60-65). Arithmetic contract in double: inv_eps = 1.0 / eps,
// neg_eps = -eps (259-260), arguments built with separately rounded ops
// (__dsub_rn/__dmul_rn/__dadd_rn, never contracted), the two-pass LSE with the
// 1e-30 sum floor (reduction.py:179-208), full-precision exp/log. B200 runs
// fp64 at 1/2 of fp32 vector rate; this path is the exact-variant multi-kernel
// loop (row LSE per row, coalesced column (max, sumexp) partials, fixed-order
// combines, device-side checks), not the fused fp32 kernel.
#include <cmath>
#include <string>

#include "../../include/lsk.h"
#include "lsk_device.cuh"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace {

#define D_CUDA(expr)                                                                                    \
  do {                                                                                                  \
    cudaError_t e__ = (expr);                                                                           \
    if (e__ != cudaSuccess) return lsk_host::fail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

constexpr double kFloor = 1e-30;  // reduction.py:44

__device__ __forceinline__ double dmax_nan(double a, double b) {
  if (a != a || b != b) return NAN;  // np.maximum propagates NaN
  return a > b ? a : b;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// 256-thread block reduction, every thread returns the same value
template <bool MAX>
__device__ __forceinline__ double block_red_d(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = MAX ? warp_max_d(v) : warp_sum_d(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = lane < 8 ? red[lane] : (MAX ? -INFINITY : 0.0);
  return MAX ? warp_max_d(t) : warp_sum_d(t);
}
__device__ __forceinline__ double arg3d(double a, double c, double s, double l) {
  return __dadd_rn(__dmul_rn(__dsub_rn(a, c), s), l);
}
__device__ __forceinline__ double arg4d(double f, double g, double c, double s, double l) {
  return __dadd_rn(__dmul_rn(__dsub_rn(__dadd_rn(f, g), c), s), l);
}
__device__ __forceinline__ double lse_finish_d(double M, double S) {
  if (!(fabs(M) <= 1.7976931348623157e308)) return -INFINITY;  // reduction.py:196-207
  return __dadd_rn(M, log(fmax(S, kFloor)));
}
__device__ __forceinline__ void pair_merge_d(double& m, double& s, double m2, double s2) {
  const double mm = dmax_nan(m, m2);
  double a = (m == mm) ? 1.0 : exp(m - mm);
  double b = (m2 == mm) ? 1.0 : exp(m2 - mm);
  if (!(mm > -INFINITY)) { a = 1.0; b = 1.0; }
  s = s * a + s2 * b;
  m = mm;
}

enum { kA = 0, kChk = 1, kCost = 2 };

// one CTA per row; two passes over the row (max, then the shifted sum)
template <int MODE>
__global__ void __launch_bounds__(256) k_row_d(const double* __restrict__ C, long long ldc, int n, int m,
                                               const double* __restrict__ rowv, const double* __restrict__ other,
                                               const double* __restrict__ lw, const double* __restrict__ lrow,
                                               const double* __restrict__ murow, double inv, double neg,
                                               double* __restrict__ out, const int* __restrict__ active) {
  __shared__ double red[32];
  if (active && !*active) return;
  const int i = blockIdx.x;
  const double* Ci = C + (long long)i * ldc;
  if (MODE == kCost) {  // sum_j C_ij * exp(z_ij), z as solver.py:108-112
    const double fi = rowv[i], li = lrow[i];
    double s = 0.0;
    for (int j = threadIdx.x; j < m; j += 256) s += __dmul_rn(Ci[j], exp(__dadd_rn(arg4d(fi, other[j], Ci[j], inv, li), lw[j])));
    s = block_red_d<false>(s, red);
    if (threadIdx.x == 0) out[i] = s;
    return;
  }
  const double fi = MODE == kChk ? rowv[i] : 0.0;
  auto argf = [&](int j) {
    return MODE == kChk ? arg4d(fi, other[j], Ci[j], inv, lw[j]) : arg3d(other[j], Ci[j], inv, lw[j]);
  };
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < m; j += 256) mx = dmax_nan(mx, argf(j));
  const double M = block_red_d<true>(mx, red);
  const double Ms = (fabs(M) <= 1.7976931348623157e308) ? M : 0.0;
  double s = 0.0;
  for (int j = threadIdx.x; j < m; j += 256) s += exp(__dsub_rn(argf(j), Ms));
  s = block_red_d<false>(s, red);
  if (threadIdx.x == 0) {
    const double L = lse_finish_d(M, s);
    if (MODE == kA) out[i] = __dmul_rn(neg, L);
    else out[i] = fabs(__dsub_rn(exp(__dadd_rn(lrow[i], L)), murow[i]));
  }
}

// column (max, sumexp) partials of the beta argument over row slabs of rs rows;
// thread owns 2 adjacent columns (coalesced 16-byte loads of doubles)
__global__ void __launch_bounds__(256) k_col_pairs_d(const double* __restrict__ C, long long ldc, int n, int m,
                                                     const double* __restrict__ alpha, const double* __restrict__ lmu,
                                                     double inv, int rs, double2* __restrict__ mx_s,
                                                     const int* __restrict__ active) {
  if (active && !*active) return;
  const int j = blockIdx.x * 256 + threadIdx.x;
  const int i0 = blockIdx.y * rs, i1 = min(n, i0 + rs);
  if (j >= m) return;
  double M = -INFINITY, S = 0.0;
  for (int i = i0; i < i1; ++i) {
    const double y = arg3d(alpha[i], C[(long long)i * ldc + j], inv, lmu[i]);
    if (y <= M && fabs(M) <= 1.7976931348623157e308) {
      // max unchanged: the general update's rescale is exp(0) = 1 exactly, so
      // skipping it gives the same bits for one exp instead of two
      S = S + exp(__dsub_rn(y, M));
      continue;
    }
    const double mn = dmax_nan(M, y);
    const double ms = (fabs(mn) <= 1.7976931348623157e308) ? mn : 0.0;
    S = (M == -INFINITY ? 0.0 : S * exp(__dsub_rn(M, ms))) + exp(__dsub_rn(y, ms));
    M = mn;
  }
  mx_s[(size_t)blockIdx.y * m + j] = make_double2(M, S);
}
__global__ void k_col_combine_d(const double2* __restrict__ p, int parts, int m, double neg, double* __restrict__ out,
                                const int* __restrict__ active) {
  if (active && !*active) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double M = -INFINITY, S = 0.0;
  for (int k = 0; k < parts; ++k) {
    const double2 v = p[(size_t)k * m + j];
    pair_merge_d(M, S, v.x, v.y);
  }
  out[j] = __dmul_rn(neg, lse_finish_d(M, S));
}

// fixed-order sum of len doubles (one CTA) -> out[0]
__global__ void __launch_bounds__(256) k_sum_d(const double* __restrict__ v, int len, double* __restrict__ out,
                                               const int* __restrict__ active) {
  __shared__ double red[32];
  if (active && !*active) return;
  double s = 0.0;
  const int per = (len + 255) / 256, lo = threadIdx.x * per, hi = min(len, lo + per);
  for (int k = lo; k < hi; ++k) s += v[k];
  s = block_red_d<false>(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void k_nonfinite_d(const double* __restrict__ v, int len, int* bad, const int* __restrict__ active) {
  if (active && !*active) return;
  int any = 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < len; k += gridDim.x * blockDim.x) any |= !isfinite(v[k]);
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(bad, 1);
}

struct StateD {
  int active, status, iters, ntrace, fbuf, pad[3];
  double err, cost;
};
__global__ void k_init_d(StateD* s, int* act) {
  StateD t{};
  t.active = 1;
  *s = t;
  *act = 1;
}
// solver.py:286-300 for iterate kk
__global__ void k_decide_d(StateD* st, const double* errp, int* bad, double tol, int kk, int final, int* trace_iter,
                           double* trace_err, int cap, int* act) {
  StateD& s = *st;
  if (!s.active) return;
  const double err = *errp;
  const int isbad = *bad;
  *bad = 0;
  int status = 0;
  bool stop = false, append = true;
  double e = err;
  if (isbad) { stop = true; status = 2; e = NAN; append = false; }
  else if (!isfinite(err)) { stop = true; status = 2; }
  else if (err < tol) { stop = true; status = 1; }
  if (append && s.ntrace < cap) {
    trace_iter[s.ntrace] = kk;
    trace_err[s.ntrace] = err;
    s.ntrace += 1;
  }
  s.status = status;
  s.err = e;
  if (stop || final) { s.active = 0; s.iters = kk; s.fbuf = kk & 1; }
  *act = s.active;
}
__global__ void k_pick_d(const double* p0, const double* p1, const StateD* st, int len, double* out) {
  const double* s = st->fbuf ? p1 : p0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) out[i] = s[i];
}
__global__ void k_cost_done_d(StateD* st, const double* c) {
  if (st->status == 2) { st->cost = NAN; return; }
  double v = *c;
  if (!isfinite(v)) { st->status = 2; v = NAN; }
  st->cost = v;
}
__global__ void k_results_d(const StateD* st, int32_t* result, double* result_f, int cost) {
  const StateD s = *st;
  result[LSK_RES_STATUS] = s.status;
  result[LSK_RES_ITERS] = s.iters;
  result[LSK_RES_NTRACE] = s.ntrace;
  result[3] = s.fbuf;
  result[LSK_RES_ROWGUARD] = 0;
  result[LSK_RES_COLGUARD] = 0;
  result_f[0] = s.err;
  result_f[1] = cost ? s.cost : NAN;
}
__global__ void k_plan_d(const double* __restrict__ C, long long ldc, int n, int m, const double* __restrict__ f,
                         const double* __restrict__ g, const double* __restrict__ lmu, const double* __restrict__ lnu,
                         double inv, double* __restrict__ P, long long ldp, int* __restrict__ nonfinite) {
  int bad = 0;
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
      const double p = exp(__dadd_rn(arg4d(f[i], g[j], C[(long long)i * ldc + j], inv, lmu[i]), lnu[j]));
      P[(long long)i * ldp + j] = p;
      bad |= !isfinite(p);
    }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1);
}

inline size_t al(size_t x) { return (x + 255) / 256 * 256; }
int num_sms_d() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}
int col_parts(int n, int m, int* rs_out) {
  const int tiles = (m + 255) / 256;
  const int want = (4 * num_sms_d() + tiles - 1) / tiles;
  int rs = (n + want - 1) / want;
  if (rs < 32) rs = 32;
  *rs_out = rs;
  return (n + rs - 1) / rs;
}
struct Lay {
  size_t f0, f1, g0, g1, pairs, rows, errv, bad, st, act, total;
};
Lay lay(int n, int m) {
  int rs;
  const int parts = col_parts(n, m, &rs);
  Lay L{};
  size_t o = 0;
  L.f0 = o; o = al(o + size_t(n) * 8);
  L.f1 = o; o = al(o + size_t(n) * 8);
  L.g0 = o; o = al(o + size_t(m) * 8);
  L.g1 = o; o = al(o + size_t(m) * 8);
  L.pairs = o; o = al(o + size_t(parts) * m * 16);
  L.rows = o; o = al(o + size_t(n) * 8);
  L.errv = o; o = al(o + 16);
  L.bad = o; o = al(o + 16);
  L.st = o; o = al(o + sizeof(StateD));
  L.act = o; o = al(o + 16);
  L.total = o;
  return L;
}
inline cudaStream_t Sd(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

size_t lsk_solve_dense_f64_workspace_bytes(int32_t n, int32_t m) {
  if (n < 1 || m < 1) return 0;
  return lay(n, m).total;
}

int32_t lsk_solve_dense_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* log_mu,
                            const double* log_nu, const double* mu, double eps, double tol, int32_t max_iter,
                            int32_t check_interval, int32_t flags, double* f_out, double* g_out, int32_t* trace_iter,
                            double* trace_err, int32_t* result, double* result_f, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!C || !log_mu || !log_nu || !mu || !f_out || !g_out || !trace_iter || !trace_err || !result || !result_f)
    return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldc < m) return lsk_host::fail(LSK_EINVAL, "bad shape");
  if (!(eps > 0) || !(tol > 0) || max_iter < 1 || check_interval < 1)
    return lsk_host::fail(LSK_EINVAL, "eps, tol > 0; max_iter, check_interval >= 1 required");
  const Lay L = lay(n, m);
  if (!workspace || workspace_bytes < L.total) return lsk_host::fail(LSK_EINVAL, "workspace too small");
  cudaStream_t st = Sd(stream);
  char* ws = static_cast<char*>(workspace);
  double* F[2] = {reinterpret_cast<double*>(ws + L.f0), reinterpret_cast<double*>(ws + L.f1)};
  double* G[2] = {reinterpret_cast<double*>(ws + L.g0), reinterpret_cast<double*>(ws + L.g1)};
  double2* pairs = reinterpret_cast<double2*>(ws + L.pairs);
  double* rows = reinterpret_cast<double*>(ws + L.rows);
  double* errv = reinterpret_cast<double*>(ws + L.errv);
  int* bad = reinterpret_cast<int*>(ws + L.bad);
  StateD* S = reinterpret_cast<StateD*>(ws + L.st);
  int* act = reinterpret_cast<int*>(ws + L.act);
  const double inv = 1.0 / eps, neg = -eps;  // solver.py:259-260 in double
  const int cap = lsk_trace_capacity(max_iter, check_interval);
  int rs;
  const int parts = col_parts(n, m, &rs);
  D_CUDA(cudaMemsetAsync(F[0], 0, size_t(n) * 8, st));
  D_CUDA(cudaMemsetAsync(G[0], 0, size_t(m) * 8, st));
  D_CUDA(cudaMemsetAsync(bad, 0, 16, st));
  D_CUDA(cudaMemsetAsync(act, 0, 16, st));
  k_init_d<<<1, 1, 0, st>>>(S, act);
  auto check = [&](int kk, bool final) -> int32_t {
    const double* fk = F[kk & 1];
    const double* gk = G[kk & 1];
    k_row_d<kChk><<<n, 256, 0, st>>>(C, ldc, n, m, fk, gk, log_nu, log_mu, mu, inv, neg, rows, act);
    k_nonfinite_d<<<8, 256, 0, st>>>(fk, n, bad, act);
    k_nonfinite_d<<<8, 256, 0, st>>>(gk, m, bad, act);
    k_sum_d<<<1, 256, 0, st>>>(rows, n, errv, act);
    k_decide_d<<<1, 1, 0, st>>>(S, errv, bad, tol, kk, final ? 1 : 0, trace_iter, trace_err, cap, act);
    D_CUDA(cudaGetLastError());
    return LSK_OK;
  };
  int32_t rc;
  for (int k = 1; k <= max_iter; ++k) {
    if (k > 1 && (k - 1) % check_interval == 0 && (rc = check(k - 1, false))) return rc;
    k_row_d<kA><<<n, 256, 0, st>>>(C, ldc, n, m, nullptr, G[(k - 1) & 1], log_nu, nullptr, nullptr, inv, neg,
                                   F[k & 1], act);
    k_col_pairs_d<<<dim3((m + 255) / 256, parts), 256, 0, st>>>(C, ldc, n, m, F[k & 1], log_mu, inv, rs, pairs, act);
    k_col_combine_d<<<(m + 255) / 256, 256, 0, st>>>(pairs, parts, m, neg, G[k & 1], act);
    D_CUDA(cudaGetLastError());
  }
  if ((rc = check(max_iter, true))) return rc;
  k_pick_d<<<64, 256, 0, st>>>(F[0], F[1], S, n, f_out);
  k_pick_d<<<64, 256, 0, st>>>(G[0], G[1], S, m, g_out);
  if (flags & LSK_FLAG_COST) {
    k_row_d<kCost><<<n, 256, 0, st>>>(C, ldc, n, m, f_out, g_out, log_nu, log_mu, nullptr, inv, neg, rows, nullptr);
    k_sum_d<<<1, 256, 0, st>>>(rows, n, errv, nullptr);
    k_cost_done_d<<<1, 1, 0, st>>>(S, errv);
  }
  k_results_d<<<1, 1, 0, st>>>(S, result, result_f, (flags & LSK_FLAG_COST) ? 1 : 0);
  D_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_update_alpha_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* beta,
                             const double* log_nu, double eps, double* alpha_out, void* stream) {
  if (!C || !beta || !log_nu || !alpha_out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldc < m || !(eps > 0)) return lsk_host::fail(LSK_EINVAL, "bad arguments");
  k_row_d<kA><<<n, 256, 0, Sd(stream)>>>(C, ldc, n, m, nullptr, beta, log_nu, nullptr, nullptr, 1.0 / eps, -eps,
                                          alpha_out, nullptr);
  D_CUDA(cudaGetLastError());
  return LSK_OK;
}

size_t lsk_update_beta_f64_workspace_bytes(int32_t n, int32_t m) {
  if (n < 1 || m < 1) return 0;
  int rs;
  return size_t(col_parts(n, m, &rs)) * m * 16;
}

int32_t lsk_update_beta_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* alpha,
                            const double* log_mu, double eps, double* beta_out, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!C || !alpha || !log_mu || !beta_out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldc < m || !(eps > 0)) return lsk_host::fail(LSK_EINVAL, "bad arguments");
  if (!workspace || workspace_bytes < lsk_update_beta_f64_workspace_bytes(n, m))
    return lsk_host::fail(LSK_EINVAL, "workspace too small");
  int rs;
  const int parts = col_parts(n, m, &rs);
  double2* pairs = static_cast<double2*>(workspace);
  k_col_pairs_d<<<dim3((m + 255) / 256, parts), 256, 0, Sd(stream)>>>(C, ldc, n, m, alpha, log_mu, 1.0 / eps, rs,
                                                                       pairs, nullptr);
  k_col_combine_d<<<(m + 255) / 256, 256, 0, Sd(stream)>>>(pairs, parts, m, -eps, beta_out, nullptr);
  D_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_marginal_error_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* mu,
                               const double* log_mu, const double* log_nu, const double* alpha, const double* beta,
                               double eps, double* err_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!C || !mu || !log_mu || !log_nu || !alpha || !beta || !err_out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldc < m || !(eps > 0)) return lsk_host::fail(LSK_EINVAL, "bad arguments");
  if (!workspace || workspace_bytes < size_t(n) * 8) return lsk_host::fail(LSK_EINVAL, "workspace too small");
  double* rows = static_cast<double*>(workspace);
  k_row_d<kChk><<<n, 256, 0, Sd(stream)>>>(C, ldc, n, m, alpha, beta, log_nu, log_mu, mu, 1.0 / eps, -eps, rows,
                                            nullptr);
  k_sum_d<<<1, 256, 0, Sd(stream)>>>(rows, n, err_out, nullptr);
  D_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_transport_cost_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* log_mu,
                               const double* log_nu, const double* alpha, const double* beta, double eps,
                               double* cost_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!C || !log_mu || !log_nu || !alpha || !beta || !cost_out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldc < m || !(eps > 0)) return lsk_host::fail(LSK_EINVAL, "bad arguments");
  if (!workspace || workspace_bytes < size_t(n) * 8) return lsk_host::fail(LSK_EINVAL, "workspace too small");
  double* rows = static_cast<double*>(workspace);
  k_row_d<kCost><<<n, 256, 0, Sd(stream)>>>(C, ldc, n, m, alpha, beta, log_nu, log_mu, nullptr, 1.0 / eps, -eps, rows,
                                             nullptr);
  k_sum_d<<<1, 256, 0, Sd(stream)>>>(rows, n, cost_out, nullptr);
  D_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t lsk_materialize_plan_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* log_mu,
                                 const double* log_nu, const double* alpha, const double* beta, double eps, double* P,
                                 int64_t ldp, int32_t* nonfinite_out, void* stream) {
  if (!C || !log_mu || !log_nu || !alpha || !beta || !P || !nonfinite_out)
    return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldc < m || ldp < m || !(eps > 0)) return lsk_host::fail(LSK_EINVAL, "bad arguments");
  int bx = (m + 255) / 256;
  if (bx > 16) bx = 16;
  k_plan_d<<<dim3(bx, n < 65535 ? n : 65535), 256, 0, Sd(stream)>>>(C, ldc, n, m, alpha, beta, log_mu, log_nu,
                                                                     1.0 / eps, P, ldp, nonfinite_out);
  D_CUDA(cudaGetLastError());
  return LSK_OK;
}

}  // extern "C"

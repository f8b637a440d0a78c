// Standard-domain Sinkhorn on the materialised Gibbs kernel (SURVEY 8(f)
// rank 3): the reference's deliberately unguarded twin of the log-domain
// solve, solver.py:340-431, in fp32 (precision="single") or fp64 ("double").
//
//   K = exp(-C / eps)                       (one pass, IEEE division)
//   per iteration: u = mu / (K v)            row dot products
//                  v = nu / (K^T u)          coalesced column partials + fixed-order combine
//   every c iterations: finiteness of u and v (else numerical_failure, err NaN,
//   no trace entry); err = sum_i |u_i (K v)_i - mu_i|; stop on non-finite err or
//   err < tol; the extra check at a cap that is not a checkpoint; the cost
//   sum_ij C_ij (u_i K_ij) v_j unless the solve failed.
//
// Overflow, underflow and division by zero propagate exactly as in numpy
// (that failure at small eps is the point of the variant). Host-enqueued
// loop, every decision on the device (kernels return early once stopped).
// Traffic: K read twice per iteration (2 n m sizeof(T)) -- the matvec pair.
#include <cmath>
#include <string>

#include <type_traits>

#include "../../include/lsk.h"
#include "lsk_stdfused.cuh"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace {

#define S_CUDA(expr)                                                                                    \
  do {                                                                                                  \
    cudaError_t e__ = (expr);                                                                           \
    if (e__ != cudaSuccess) return lsk_host::fail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

constexpr int kBlk = 1024;  // rows per fixed-order block of the error sum

template <class T>
struct StdState {
  int active, status, iters, ntrace;
  T err, cost;
};

template <class T> __device__ __forceinline__ T dmul(T a, T b);
template <> __device__ __forceinline__ float dmul(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
template <class T> __device__ __forceinline__ T dadd(T a, T b);
template <> __device__ __forceinline__ float dadd(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
template <class T> __device__ __forceinline__ T ddiv(T a, T b);
template <> __device__ __forceinline__ float ddiv(float a, float b) { return __fdiv_rn(a, b); }
template <> __device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float dexp(float x) { return expf(x); }
__device__ __forceinline__ double dexp(double x) { return exp(x); }

// 4 consecutive values (16-byte aligned for float, 2 x 16 B for double)
__device__ __forceinline__ void ld4(const float* p, float (&v)[4]) {
  const float4 t = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

template <class T>
__device__ __forceinline__ T warp_sum_t(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// fixed-order block sum (blockDim.x = 256): warp butterflies, then warp 0 over the 8 partials
template <class T>
__device__ __forceinline__ T block_sum_t(T v, T* sh) {
  v = warp_sum_t(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  T r = T(0);
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : T(0);
    r = warp_sum_t(r);
  }
  return r;  // valid in thread 0
}

// K = exp(-C / eps); the row padding [m, ldk) is written as 0 (the one-pass
// kernel copies whole 16-byte groups and multiplies them by v = 0 there)
template <class T>
__global__ void k_gibbs(const T* __restrict__ C, long long ldc, int n, int m, T eps, T* __restrict__ Kmat,
                        long long ldk) {
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ldk; j += gridDim.x * blockDim.x)
      Kmat[(long long)i * ldk + j] = j < m ? dexp(ddiv(-C[(long long)i * ldc + j], eps)) : T(0);
}

// MODE 0: u_i = mu_i / (K v)_i.  MODE 1: term_i = |u_i (K v)_i - mu_i| (check).
// One CTA per row, 4 consecutive columns per thread per step (vector loads),
// fixed-order block sum.
template <class T, int MODE>
__global__ void __launch_bounds__(256) k_rowdot(const T* __restrict__ Kmat, long long ldk, int n, int m,
                                                const T* __restrict__ v, const T* __restrict__ mu,
                                                T* __restrict__ u, T* __restrict__ term,
                                                const int* __restrict__ act) {
  if (act && !*act) return;
  __shared__ T sh[32];
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const T* row = Kmat + (long long)i * ldk;
    T s = T(0);
    for (int j = 4 * threadIdx.x; j < m; j += 4 * blockDim.x) {
      if (j + 3 < m) {
        T k[4], w[4];
        ld4(row + j, k);
#pragma unroll
        for (int c = 0; c < 4; ++c) w[c] = v[j + c];
#pragma unroll
        for (int c = 0; c < 4; ++c) s = dadd(s, dmul(k[c], w[c]));
      } else {
        for (int c = 0; j + c < m; ++c) s = dadd(s, dmul(row[j + c], v[j + c]));
      }
    }
    s = block_sum_t(s, sh);
    if (threadIdx.x == 0) {
      if (MODE == 0) u[i] = ddiv(mu[i], s);
      else term[i] = fabs(dadd(dmul(u[i], s), -mu[i]));
    }
    __syncthreads();
  }
}

// column partials over row slabs of rs rows: part[p][j] = sum_{i in slab p} K_ij u_i;
// 4 columns per thread, 8 rows of vector loads in flight
template <class T>
__global__ void __launch_bounds__(256) k_colpart(const T* __restrict__ Kmat, long long ldk, int n, int m,
                                                 const T* __restrict__ u, int rs, T* __restrict__ part,
                                                 const int* __restrict__ act) {
  if (act && !*act) return;
  const int j0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (j0 >= m) return;
  const int i0 = blockIdx.y * rs, i1 = min(n, i0 + rs);
  T s[4] = {T(0), T(0), T(0), T(0)};
  int i = i0;
  for (; i + 7 < i1; i += 8) {
    T k[8][4], uu[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      ld4(Kmat + (long long)(i + r) * ldk + j0, k[r]);
      uu[r] = u[i + r];
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) s[c] = dadd(s[c], dmul(k[r][c], uu[r]));
  }
  for (; i < i1; ++i) {
    T k[4];
    ld4(Kmat + (long long)i * ldk + j0, k);
    const T ui = u[i];
#pragma unroll
    for (int c = 0; c < 4; ++c) s[c] = dadd(s[c], dmul(k[c], ui));
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (j0 + c < m) part[(long long)blockIdx.y * m + j0 + c] = s[c];
}

template <class T>
__global__ void k_colfin(const T* __restrict__ part, int parts, int m, const T* __restrict__ nu, T* __restrict__ v,
                         const int* __restrict__ act) {
  if (act && !*act) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  T s = T(0);
  for (int p = 0; p < parts; ++p) s = dadd(s, part[(long long)p * m + j]);
  v[j] = ddiv(nu[j], s);
}

template <class T>
__global__ void k_nonfinite(const T* __restrict__ x, int n, int* bad, const int* __restrict__ act) {
  if (act && !*act) return;
  int b = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b |= !isfinite(x[i]);
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

// fixed 1024-row blocks of the per-row terms, in order inside each block
template <class T>
__global__ void __launch_bounds__(256) k_blocksum(const T* __restrict__ term, int n, T* __restrict__ blk,
                                                  const int* __restrict__ act) {
  if (act && !*act) return;
  __shared__ T sh[32];
  const int i0 = blockIdx.x * kBlk, i1 = min(n, i0 + kBlk);
  T s = T(0);
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) s = dadd(s, term[i]);
  s = block_sum_t(s, sh);
  if (threadIdx.x == 0) blk[blockIdx.x] = s;
}

template <class T>
__global__ void k_init(StdState<T>* st, int* act, T* u, int n, T* v, int m) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = t; i < n; i += gridDim.x * blockDim.x) u[i] = T(1);
  for (int j = t; j < m; j += gridDim.x * blockDim.x) v[j] = T(1);
  if (t == 0) {
    StdState<T> s{};
    s.active = 1;
    *st = s;
    *act = 1;
  }
}

// check decision (solver.py:380-411), identical to the log-domain one
template <class T>
__global__ void k_decide(int n, const T* __restrict__ blk, int* bad, double tol, int kk, int final, StdState<T>* st,
                         int* act, int32_t* trace_iter, T* trace_err, int cap) {
  StdState<T>& s = *st;
  if (!s.active) return;
  const int nb = (n + kBlk - 1) / kBlk;
  const int isbad = *bad;
  *bad = 0;
  T err = T(0);
  if (!isbad)
    for (int k = 0; k < nb; ++k) err = dadd(err, blk[k]);
  int status = 0;
  bool stop = false, append = true;
  T e = err;
  if (isbad) { stop = true; status = 2; e = T(NAN); append = false; }
  else if (!isfinite(err)) { stop = true; status = 2; }
  else if (err < T(tol)) { stop = true; status = 1; }
  if (append && s.ntrace < cap) {
    trace_iter[s.ntrace] = kk;
    trace_err[s.ntrace] = err;
    s.ntrace += 1;
  }
  s.status = status;
  s.err = e;
  if (stop || final) {
    s.active = 0;
    s.iters = kk;
  }
  *act = s.active;
}

// transport cost rows: sum_j C_ij * ((u_i * K_ij) * v_j)   (solver.py:413-417)
template <class T>
__global__ void __launch_bounds__(256) k_cost_rows(const T* __restrict__ C, long long ldc, const T* __restrict__ Kmat,
                                                   long long ldk, int n, int m, const T* __restrict__ u,
                                                   const T* __restrict__ v, T* __restrict__ term,
                                                   const StdState<T>* st) {
  if (st->status == 2) return;
  __shared__ T sh[32];
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const T ui = u[i];
    T s = T(0);
    for (int j = threadIdx.x; j < m; j += blockDim.x)
      s = dadd(s, dmul(C[(long long)i * ldc + j], dmul(dmul(ui, Kmat[(long long)i * ldk + j]), v[j])));
    s = block_sum_t(s, sh);
    if (threadIdx.x == 0) term[i] = s;
    __syncthreads();
  }
}

template <class T>
__global__ void k_cost_finish(int n, const T* __restrict__ blk, StdState<T>* st) {
  StdState<T>& s = *st;
  if (s.status == 2) { s.cost = T(NAN); return; }
  const int nb = (n + kBlk - 1) / kBlk;
  T c = T(0);
  for (int k = 0; k < nb; ++k) c = dadd(c, blk[k]);
  if (!isfinite(c)) { s.status = 2; c = T(NAN); }
  s.cost = c;
}

template <class T>
__global__ void k_results(const StdState<T>* st, int32_t* result, T* result_f, int cost) {
  const StdState<T> s = *st;
  result[LSK_RES_STATUS] = s.status;
  result[LSK_RES_ITERS] = s.iters;
  result[LSK_RES_NTRACE] = s.ntrace;
  result_f[0] = s.err;
  result_f[1] = cost ? s.cost : T(NAN);
}

inline size_t al(size_t x) { return (x + 255) / 256 * 256; }

int num_sms_s() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}
int std_parts(int n, int m, int* rs_out) {
  const int tiles = (m + 1023) / 1024;
  const int want = (4 * num_sms_s() + tiles - 1) / tiles;
  int rs = (n + want - 1) / want;
  if (rs < 32) rs = 32;
  *rs_out = rs;
  return (n + rs - 1) / rs;
}

struct StdLayout {
  size_t K, part, term, blk, bad, state, act, total;
  // fused one-pass path (fp32, m <= 8192)
  size_t u0, u1, v0, v1, fpart, errp, flagp, bar, outbuf;
  long long ldk;
};
using StdFused = lsk::StdSolver<256, 8, 6>;
constexpr int kStdW = StdFused::W;
template <class T>
StdLayout std_layout(int n, int m) {
  StdLayout L{};
  int rs;
  const int parts = std_parts(n, m, &rs);
  L.ldk = (m + 31) / 32 * 32;
  size_t o = 0;
  L.K = o; o = al(o + size_t(n) * L.ldk * sizeof(T));
  L.part = o; o = al(o + size_t(parts) * m * sizeof(T));
  L.term = o; o = al(o + size_t(n) * sizeof(T));
  L.blk = o; o = al(o + size_t((n + kBlk - 1) / kBlk) * sizeof(T));
  L.bad = o; o = al(o + 16);
  L.state = o; o = al(o + sizeof(StdState<T>));
  L.act = o; o = al(o + 16);
  if (sizeof(T) == 4 && m <= kStdW) {
    const int G = num_sms_s();
    L.u0 = o; o = al(o + size_t(n) * 4);
    L.u1 = o; o = al(o + size_t(n) * 4);
    L.v0 = o; o = al(o + size_t(kStdW) * 4);
    L.v1 = o; o = al(o + size_t(kStdW) * 4);
    L.fpart = o; o = al(o + size_t(G) * kStdW * 4);
    L.errp = o; o = al(o + size_t(G) * 4);
    L.flagp = o; o = al(o + size_t(G) * 4);
    L.bar = o; o = al(o + 16);
    L.outbuf = o; o = al(o + 16);
  }
  L.total = o;
  return L;
}

__global__ void k_std_fused(lsk::StdArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  StdFused sv(a, smem);
  sv.solve();
}
__global__ void k_std_init(float* u0, int n, float* v0, int m, StdState<float>* st) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = t; i < n; i += gridDim.x * blockDim.x) u0[i] = 1.f;
  for (int j = t; j < kStdW; j += gridDim.x * blockDim.x) v0[j] = j < m ? 1.f : 0.f;
  if (t == 0) {
    StdState<float> s{};
    s.active = 1;
    *st = s;
  }
}
__global__ void k_std_pick(const float* u0, const float* u1, int n, const float* v0, const float* v1, int m,
                           const int* outbuf, float* u, float* v) {
  const int sel = *outbuf;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) u[i] = sel ? u1[i] : u0[i];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) v[j] = sel ? v1[j] : v0[j];
}

template <class T>
int32_t solve_standard(const T* C, int64_t ldc, int32_t n, int32_t m, const T* mu, const T* nu, double eps,
                       double tol, int32_t K, int32_t c, int32_t flags, T* u, T* v, int32_t* trace_iter,
                       T* trace_err, int32_t* result, T* result_f, void* workspace, size_t workspace_bytes,
                       void* stream) {
  if (!C || !mu || !nu || !u || !v || !trace_iter || !trace_err || !result || !result_f)
    return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || ldc < m) return lsk_host::fail(LSK_EINVAL, "bad dimensions");
  if (!(eps > 0) || K < 1 || c < 1) return lsk_host::fail(LSK_EINVAL, "need eps > 0, max_iter >= 1, check >= 1");
  const StdLayout L = std_layout<T>(n, m);
  if (!workspace || workspace_bytes < L.total) return lsk_host::fail(LSK_EINVAL, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  T* Km = reinterpret_cast<T*>(ws + L.K);
  T* part = reinterpret_cast<T*>(ws + L.part);
  T* term = reinterpret_cast<T*>(ws + L.term);
  T* blk = reinterpret_cast<T*>(ws + L.blk);
  int* bad = reinterpret_cast<int*>(ws + L.bad);
  StdState<T>* S = reinterpret_cast<StdState<T>*>(ws + L.state);
  int* act = reinterpret_cast<int*>(ws + L.act);
  const int cap = lsk_trace_capacity(K, c);
  int rs;
  const int parts = std_parts(n, m, &rs);
  const int nb = (n + kBlk - 1) / kBlk;
  const int sms = num_sms_s();
  const int rblocks = n < 8 * sms ? n : 8 * sms;

  S_CUDA(cudaMemsetAsync(bad, 0, 16, st));
  k_init<T><<<64, 256, 0, st>>>(S, act, u, n, v, m);
  int bx = (m + 255) / 256;
  if (bx > 32) bx = 32;
  k_gibbs<T><<<dim3(bx, n < 65535 ? n : 65535), 256, 0, st>>>(C, ldc, n, m, T(eps), Km, L.ldk);
  if constexpr (std::is_same<T, float>::value) {
    if (m <= kStdW && !(flags & LSK_FLAG_STD_MULTIKERNEL)) {
      // one persistent launch, one read of K per iteration (lsk_stdfused.cuh)
      const int G = num_sms_s() < n ? num_sms_s() : n;
      lsk::StdArgs sa{};
      sa.K = Km; sa.ldk = L.ldk; sa.n = n; sa.m = m; sa.mpad = (m + 3) / 4 * 4;
      sa.mu = mu; sa.nu = nu; sa.tol = tol; sa.max_iter = K; sa.check = c;
      sa.u0 = reinterpret_cast<float*>(ws + L.u0); sa.u1 = reinterpret_cast<float*>(ws + L.u1);
      sa.v0 = reinterpret_cast<float*>(ws + L.v0); sa.v1 = reinterpret_cast<float*>(ws + L.v1);
      sa.part = reinterpret_cast<float*>(ws + L.fpart);
      sa.errpart = reinterpret_cast<float*>(ws + L.errp);
      sa.flagpart = reinterpret_cast<int*>(ws + L.flagp);
      sa.bar = reinterpret_cast<unsigned long long*>(ws + L.bar);
      sa.st_active = &S->active; sa.st_status = &S->status; sa.st_iters = &S->iters; sa.st_ntrace = &S->ntrace;
      sa.st_err = &S->err;
      sa.out_buf = reinterpret_cast<int*>(ws + L.outbuf);
      sa.trace_iter = trace_iter; sa.trace_err = trace_err; sa.cap = cap;
      S_CUDA(cudaMemsetAsync(ws + L.bar, 0, 16, st));
      S_CUDA(cudaMemsetAsync(ws + L.outbuf, 0, 16, st));
      k_std_init<<<64, 256, 0, st>>>(sa.u0, n, sa.v0, m, S);
      // per-device-context attribute: set on every launch, never cached process-wide
      S_CUDA(cudaFuncSetAttribute(k_std_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, int(StdFused::kSmemBytes)));
      void* args[] = {&sa};
      S_CUDA(cudaLaunchCooperativeKernel((const void*)k_std_fused, dim3(G), dim3(StdFused::NW * 32), args, StdFused::kSmemBytes, st));
      k_std_pick<<<64, 256, 0, st>>>(sa.u0, sa.u1, n, sa.v0, sa.v1, m, sa.out_buf, u, v);
      if (flags & LSK_FLAG_COST) {
        k_cost_rows<T><<<rblocks, 256, 0, st>>>(C, ldc, Km, L.ldk, n, m, u, v, term, S);
        k_blocksum<T><<<nb, 256, 0, st>>>(term, n, blk, nullptr);
        k_cost_finish<T><<<1, 1, 0, st>>>(n, blk, S);
      }
      k_results<T><<<1, 1, 0, st>>>(S, result, result_f, (flags & LSK_FLAG_COST) ? 1 : 0);
      S_CUDA(cudaGetLastError());
      return LSK_OK;
    }
  }
  auto check = [&](int kk, bool final) -> int32_t {
    k_nonfinite<T><<<8, 256, 0, st>>>(u, n, bad, act);
    k_nonfinite<T><<<8, 256, 0, st>>>(v, m, bad, act);
    k_rowdot<T, 1><<<rblocks, 256, 0, st>>>(Km, L.ldk, n, m, v, mu, u, term, act);
    k_blocksum<T><<<nb, 256, 0, st>>>(term, n, blk, act);
    k_decide<T><<<1, 1, 0, st>>>(n, blk, bad, tol, kk, final ? 1 : 0, S, act, trace_iter, trace_err, cap);
    S_CUDA(cudaGetLastError());
    return LSK_OK;
  };
  int32_t rc;
  for (int k = 1; k <= K; ++k) {
    k_rowdot<T, 0><<<rblocks, 256, 0, st>>>(Km, L.ldk, n, m, v, mu, u, nullptr, act);
    k_colpart<T><<<dim3((m + 1023) / 1024, parts), 256, 0, st>>>(Km, L.ldk, n, m, u, rs, part, act);
    k_colfin<T><<<(m + 255) / 256, 256, 0, st>>>(part, parts, m, nu, v, act);
    S_CUDA(cudaGetLastError());
    if (k % c == 0 && k < K && (rc = check(k, false))) return rc;
  }
  if ((rc = check(K, true))) return rc;
  if (flags & LSK_FLAG_COST) {
    k_cost_rows<T><<<rblocks, 256, 0, st>>>(C, ldc, Km, L.ldk, n, m, u, v, term, S);
    k_blocksum<T><<<nb, 256, 0, st>>>(term, n, blk, nullptr);
    k_cost_finish<T><<<1, 1, 0, st>>>(n, blk, S);
  }
  k_results<T><<<1, 1, 0, st>>>(S, result, result_f, (flags & LSK_FLAG_COST) ? 1 : 0);
  S_CUDA(cudaGetLastError());
  return LSK_OK;
}

}  // namespace

extern "C" {

size_t lsk_solve_standard_workspace_bytes(int32_t n, int32_t m, int32_t double_precision) {
  if (n < 1 || m < 1) return 0;
  return double_precision ? std_layout<double>(n, m).total : std_layout<float>(n, m).total;
}

int32_t lsk_solve_standard_f32(const float* C, int64_t ldc, int32_t n, int32_t m, const float* mu, const float* nu,
                               double eps, double tol, int32_t max_iter, int32_t check, int32_t flags, float* u_out,
                               float* v_out, int32_t* trace_iter, float* trace_err, int32_t* result, float* result_f,
                               void* workspace, size_t workspace_bytes, void* stream) {
  // the reference divides by dt.type(eps): fp32 eps in single precision
  return solve_standard<float>(C, ldc, n, m, mu, nu, double(float(eps)), tol, max_iter, check, flags, u_out, v_out,
                               trace_iter, trace_err, result, result_f, workspace, workspace_bytes, stream);
}

int32_t lsk_solve_standard_f64(const double* C, int64_t ldc, int32_t n, int32_t m, const double* mu,
                               const double* nu, double eps, double tol, int32_t max_iter, int32_t check,
                               int32_t flags, double* u_out, double* v_out, int32_t* trace_iter, double* trace_err,
                               int32_t* result, double* result_f, void* workspace, size_t workspace_bytes,
                               void* stream) {
  return solve_standard<double>(C, ldc, n, m, mu, nu, eps, tol, max_iter, check, flags, u_out, v_out, trace_iter,
                                trace_err, result, result_f, workspace, workspace_bytes, stream);
}

}  // extern "C"

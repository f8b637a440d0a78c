// The reference's deterministic reductions (reduction.py; SURVEY 8(a) rows
// a5-a7) on the GPU: max / sum / log-sum-exp over rows or columns with the
// fixed two-level tree of a ReductionPlan(chunk_width w, group_size B):
//
//   1. lane fold: lane t accumulates elements t, t+B, t+2B, ... in order, the
//      ragged tail padded with the identity (-inf for max, 0.0 for sum) and the
//      padding APPLIED, as the reference concatenates it (so -0.0 + 0.0 = +0.0
//      exactly as numpy does);
//   2. chunk tree: each w-wide chunk of lanes is combined by ceil-halving
//      steps (a[i] = op(a[i], a[half + i]) for i < off - half), then the chunk
//      results by the same halving (reduction.py:72-156).
//
// The pairing is replicated exactly, so max and sum are bit-identical to the
// reference for every plan. LSE = M + log(max(S, 1e-30)) with M the tree max
// (all -inf rows -> -inf) and S the tree sum of exp(x - M) (reduction.py:
// 179-224): the exponentials are CUDA's (<= 2 ulp), so LSE matches to ulps.
//
// Rows: one CTA per row, lanes in shared memory. Columns: one CTA per 32
// consecutive columns (coalesced 128-byte row segments), lanes [B][32] in
// shared memory. Both are HBM-bound single passes (two for LSE).
#include <cmath>
#include <string>

#include "../../include/lsk.h"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace {

#define R_CUDA(expr)                                                                                    \
  do {                                                                                                  \
    cudaError_t e__ = (expr);                                                                           \
    if (e__ != cudaSuccess) return lsk_host::fail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

constexpr int kMaxLanes = 4096;  // group_size supported (shared-memory lanes)

template <class T> struct Num;
template <> struct Num<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float ex(float x) { return expf(x); }
  static __device__ __forceinline__ float lg(float x) { return logf(x); }
};
template <> struct Num<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double ex(double x) { return exp(x); }
  static __device__ __forceinline__ double lg(double x) { return log(x); }
};

// np.maximum: NaN propagates (either operand), otherwise the larger
template <class T>
__device__ __forceinline__ T nmax(T a, T b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : (b > a ? b : a);  // equal (incl. -0 vs +0): numpy keeps the first operand
}

enum { kMax = 0, kSum = 1, kExpSum = 2 };  // kExpSum: sum of exp(x - shift), pads 0

template <class T, int OP>
__device__ __forceinline__ T identity() { return OP == kMax ? T(-INFINITY) : T(0); }
template <class T, int OP>
__device__ __forceinline__ T combine(T a, T b) { return OP == kMax ? nmax(a, b) : Num<T>::add(a, b); }

// chunk tree over lanes a[0..B) (stride st between consecutive lanes), run by
// the calling threads: thread c < n_chunks halves chunk c, then thread 0 the
// chunk results. The caller synchronises before and after.
template <class T, int OP>
__device__ void chunk_tree(T* a, int st, int B, int w, int tid, int nthreads) {
  const int n_chunks = B / w;
  for (int c = tid; c < n_chunks; c += nthreads) {
    T* ch = a + (size_t)c * w * st;
    for (int off = w; off > 1;) {
      const int half = (off + 1) / 2, lo = off - half;
      for (int i = 0; i < lo; ++i) ch[(size_t)i * st] = combine<T, OP>(ch[(size_t)i * st], ch[(size_t)(half + i) * st]);
      off = half;
    }
  }
}
template <class T, int OP>
__device__ void cross_tree(T* a, int st, int B, int w) {
  const int n_chunks = B / w;
  for (int off = n_chunks; off > 1;) {
    const int half = (off + 1) / 2, lo = off - half;
    for (int i = 0; i < lo; ++i)
      a[(size_t)i * w * st] = combine<T, OP>(a[(size_t)i * w * st], a[(size_t)(half + i) * w * st]);
    off = half;
  }
}

// element loader: x or exp(x - shift) for kExpSum
template <class T, int OP>
__device__ __forceinline__ T elem(T x, T shift) { return OP == kExpSum ? Num<T>::ex(x - shift) : x; }

// one CTA per row; lanes in dynamic shared memory
template <class T, int OP>
__global__ void __launch_bounds__(256) k_tree_rows(const T* __restrict__ A, long long lda, int R, int L, int B, int w,
                                                   const T* __restrict__ shift, T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* lanes = reinterpret_cast<T*>(smem_raw);
  const int strides = (L + B - 1) / B;
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    const T* row = A + (long long)r * lda;
    const T sh = (OP == kExpSum) ? shift[r] : T(0);
    for (int t = threadIdx.x; t < B; t += blockDim.x) {
      T acc = t < L ? elem<T, OP>(row[t], sh) : identity<T, OP>();
      for (int k = 1; k < strides; ++k) {
        const long long idx = (long long)k * B + t;
        acc = combine<T, OP>(acc, idx < L ? elem<T, OP>(row[idx], sh) : identity<T, OP>());
      }
      lanes[t] = acc;
    }
    __syncthreads();
    if (B > 1) {
      chunk_tree<T, OP>(lanes, 1, B, w, threadIdx.x, blockDim.x);
      __syncthreads();
      if (threadIdx.x == 0) cross_tree<T, OP>(lanes, 1, B, w);
    }
    if (threadIdx.x == 0) out[r] = lanes[0];
    __syncthreads();
  }
}

// 32 consecutive columns per CTA; lanes [B][32] in dynamic shared memory;
// A is (L, R) with row stride lda; the reduction runs down each column
template <class T, int OP>
__global__ void __launch_bounds__(256) k_tree_cols(const T* __restrict__ A, long long lda, int L, int R, int B, int w,
                                                   const T* __restrict__ shift, T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* lanes = reinterpret_cast<T*>(smem_raw);  // lanes[t * 32 + c]
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5, G = blockDim.x >> 5;
  const int j = blockIdx.x * 32 + c;
  const bool ok = j < R;
  const T sh = (OP == kExpSum && ok) ? shift[j] : T(0);
  const int strides = (L + B - 1) / B;
  for (int t = g; t < B; t += G) {
    T acc = (t < L && ok) ? elem<T, OP>(A[(long long)t * lda + j], sh) : identity<T, OP>();
    for (int k = 1; k < strides; ++k) {
      const long long idx = (long long)k * B + t;
      acc = combine<T, OP>(acc, (idx < L && ok) ? elem<T, OP>(A[idx * lda + j], sh) : identity<T, OP>());
    }
    lanes[t * 32 + c] = acc;
  }
  __syncthreads();
  if (B > 1) {
    // (column, chunk) pairs over all threads, then one thread per column across chunks
    const int n_chunks = B / w;
    for (int p = threadIdx.x; p < n_chunks * 32; p += blockDim.x) {
      const int cc = p & 31, ch = p >> 5;
      T* base = lanes + (size_t)ch * w * 32 + cc;
      for (int off = w; off > 1;) {
        const int half = (off + 1) / 2, lo = off - half;
        for (int i = 0; i < lo; ++i) base[(size_t)i * 32] = combine<T, OP>(base[(size_t)i * 32], base[(size_t)(half + i) * 32]);
        off = half;
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) cross_tree<T, OP>(lanes + threadIdx.x, 32, B, w);
    __syncthreads();
  }
  if (g == 0 && ok) out[j] = lanes[c];
}

// LSE finish (reduction.py:196-207): M non-finite -> shift 0 for the sum pass
template <class T>
__global__ void k_lse_shift(const T* __restrict__ M, int R, T* __restrict__ shift) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) shift[r] = isfinite(M[r]) ? M[r] : T(0);
}
template <class T>
__global__ void k_lse_finish(const T* __restrict__ M, const T* __restrict__ S, int R, T* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const T m = M[r];
  if (!isfinite(m)) {
    out[r] = T(-INFINITY);
    return;
  }
  const T s = S[r] > T(1e-30) ? S[r] : T(1e-30);  // np.maximum(S, floor): NaN stays NaN
  out[r] = (S[r] != S[r]) ? S[r] : Num<T>::add(m, Num<T>::lg(s));
}

template <class T>
int32_t run(const T* A, long long lda, int R, int L, int cols, int op, int w, int B, T* out, void* workspace,
            size_t ws_bytes, cudaStream_t st) {
  const size_t lane_bytes = (size_t)B * sizeof(T) * (cols ? 32 : 1);
  if (lane_bytes > 200 * 1024) return lsk_host::fail(LSK_EUNSUPPORTED, "group_size too large for the column tree");
  auto launch = [&](auto kern, const T* shift, T* dst) -> int32_t {
    R_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(lane_bytes)));
    if (cols) kern<<<(R + 31) / 32, 256, lane_bytes, st>>>(A, lda, L, R, B, w, shift, dst);
    else kern<<<R < 65535 ? R : 65535, 256, lane_bytes, st>>>(A, lda, R, L, B, w, shift, dst);
    R_CUDA(cudaGetLastError());
    return LSK_OK;
  };
  int32_t rc;
  if (op == 0) return cols ? launch(k_tree_cols<T, kMax>, nullptr, out) : launch(k_tree_rows<T, kMax>, nullptr, out);
  if (op == 1) return cols ? launch(k_tree_cols<T, kSum>, nullptr, out) : launch(k_tree_rows<T, kSum>, nullptr, out);
  // LSE: workspace holds M, shift, S (3 R values)
  if (!workspace || ws_bytes < 3 * (size_t)R * sizeof(T)) return lsk_host::fail(LSK_EINVAL, "workspace too small");
  T* M = static_cast<T*>(workspace);
  T* sh = M + R;
  T* S = sh + R;
  if ((rc = cols ? launch(k_tree_cols<T, kMax>, nullptr, M) : launch(k_tree_rows<T, kMax>, nullptr, M))) return rc;
  k_lse_shift<T><<<(R + 255) / 256, 256, 0, st>>>(M, R, sh);
  if ((rc = cols ? launch(k_tree_cols<T, kExpSum>, sh, S) : launch(k_tree_rows<T, kExpSum>, sh, S))) return rc;
  k_lse_finish<T><<<(R + 255) / 256, 256, 0, st>>>(M, S, R, out);
  R_CUDA(cudaGetLastError());
  return LSK_OK;
}

int32_t reduce(const void* A, int64_t lda, int32_t R, int32_t L, int32_t dtype, int32_t op, int32_t cols,
               int32_t chunk_width, int32_t group_size, void* out, void* workspace, size_t ws_bytes, void* stream) {
  if (!A || !out) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (R < 1 || L < 1) return lsk_host::fail(LSK_EINVAL, "empty reduction");
  if (op < 0 || op > 2 || (dtype != 0 && dtype != 1)) return lsk_host::fail(LSK_EINVAL, "bad op or dtype");
  if (chunk_width < 1 || group_size < 1 || group_size % chunk_width != 0)
    return lsk_host::fail(LSK_EINVAL, "group_size must be a positive multiple of chunk_width");
  if (group_size > kMaxLanes) return lsk_host::fail(LSK_EUNSUPPORTED, "group_size above 4096 lanes");
  if (cols ? lda < R : lda < L) return lsk_host::fail(LSK_EINVAL, "leading dimension too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == 0)
    return run<float>(static_cast<const float*>(A), lda, R, L, cols, op, chunk_width, group_size,
                      static_cast<float*>(out), workspace, ws_bytes, st);
  return run<double>(static_cast<const double*>(A), lda, R, L, cols, op, chunk_width, group_size,
                     static_cast<double*>(out), workspace, ws_bytes, st);
}

}  // namespace

extern "C" {

size_t lsk_reduce_workspace_bytes(int32_t R, int32_t dtype) { return 3 * (size_t)(R > 0 ? R : 0) * (dtype ? 8 : 4); }

int32_t lsk_reduce_rows(const void* A, int64_t lda, int32_t R, int32_t L, int32_t dtype, int32_t op,
                        int32_t chunk_width, int32_t group_size, void* out, void* workspace, size_t workspace_bytes,
                        void* stream) {
  return reduce(A, lda, R, L, dtype, op, 0, chunk_width, group_size, out, workspace, workspace_bytes, stream);
}

int32_t lsk_reduce_cols(const void* A, int64_t lda, int32_t L, int32_t R, int32_t dtype, int32_t op,
                        int32_t chunk_width, int32_t group_size, void* out, void* workspace, size_t workspace_bytes,
                        void* stream) {
  return reduce(A, lda, R, L, dtype, op, 1, chunk_width, group_size, out, workspace, workspace_bytes, stream);
}

}  // extern "C"

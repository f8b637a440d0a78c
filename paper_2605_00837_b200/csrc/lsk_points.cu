// C-ABI of the points helpers (include/lsk.h): the NCCL communicator
// (lsk_comm_*), the plan consumers without the plan (lsk_points_consume_f32)
// and the exact fp64 cost maximum (lsk_points_cost_max). The solve itself is
// lsk_points_solve.cu.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include <nccl.h>

#include "../../include/lsk.h"
#include "lsk_points.cuh"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);  // lsk_api.cu: thread-local lsk_last_error()
}

namespace {

int32_t pfail(int32_t code, const std::string& msg) { return lsk_host::fail(code, msg); }
#define P_CUDA(expr)                                                                              \
  do {                                                                                            \
    cudaError_t e__ = (expr);                                                                     \
    if (e__ != cudaSuccess) return pfail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)
#define P_NCCL(expr)                                                                              \
  do {                                                                                            \
    ncclResult_t r__ = (expr);                                                                    \
    if (r__ != ncclSuccess) return pfail(LSK_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r__)); \
  } while (0)

inline size_t al(size_t x) { return (x + 255) / 256 * 256; }
inline int chunks_of(int ncols) { return (ncols + lsk::kPtsChunk - 1) / lsk::kPtsChunk; }

__global__ void k_fill_u64(unsigned long long* p, int count, unsigned long long v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) p[i] = v;
}
__global__ void k_interleave2(const double* a, const double* b, int count, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) { out[2 * i] = a[i]; out[2 * i + 1] = b[i]; }
}

struct EpsC {
  float inv, neg;
};
EpsC epsc(double eps) {
  volatile float e32 = static_cast<float>(eps);
  volatile float one = 1.0f;
  return {one / e32, -e32};
}

}  // namespace

extern "C" {

int32_t lsk_nccl_unique_id(void* id_out) {
  if (!id_out) return pfail(LSK_EINVAL, "null id");
  ncclUniqueId id;
  P_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return LSK_OK;
}
int32_t lsk_nccl_unique_id_bytes(void) { return int32_t(sizeof(ncclUniqueId)); }

int32_t lsk_comm_create(const void* id, int32_t nranks, int32_t rank, void** comm_out) {
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return pfail(LSK_EINVAL, "bad comm args");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  P_NCCL(ncclCommInitRank(&comm, nranks, uid, rank));
  *comm_out = comm;
  return LSK_OK;
}

int32_t lsk_comm_destroy(void* comm) {
  if (comm) P_NCCL(ncclCommDestroy(static_cast<ncclComm_t>(comm)));
  return LSK_OK;
}


// ---- plan consumers without the plan
size_t lsk_points_consume_workspace_bytes(int32_t B, int32_t n, int32_t m) {
  if (B < 1 || n < 1 || m < 1) return 0;
  const size_t ch = size_t(chunks_of(m));
  return al(size_t(B) * n * 16) + al(size_t(B) * m * 16) + al(size_t(B) * ch * n * 16) + al(size_t(B) * ch * n * 8) +
         al(size_t(B) * 24);
}

int32_t lsk_points_consume_f32(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                               const float* scale, const float* f, const float* g, const float* log_mu,
                               const float* log_nu, double eps, float* mapped_out, int32_t* match_idx,
                               float* match_w, int32_t* zero_rows, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (!X || !Y || !scale || !f || !g || !log_mu || !log_nu || !mapped_out || !match_idx || !match_w || !zero_rows)
    return pfail(LSK_EINVAL, "null pointer");
  if (B < 1 || n < 1 || m < 1) return pfail(LSK_EINVAL, "B, n, m must be >= 1");
  if (d < 1 || d > 3) return pfail(LSK_EUNSUPPORTED, "points consumers support d in 1..3");
  if (!(eps > 0)) return pfail(LSK_EINVAL, "eps must be > 0");
  if (!workspace || workspace_bytes < lsk_points_consume_workspace_bytes(B, n, m))
    return pfail(LSK_EINVAL, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  const int chunks = chunks_of(m);
  float4* X4 = reinterpret_cast<float4*>(ws);
  ws += al(size_t(B) * n * 16);
  float4* Y4 = reinterpret_cast<float4*>(ws);
  ws += al(size_t(B) * m * 16);
  float4* part = reinterpret_cast<float4*>(ws);
  ws += al(size_t(B) * chunks * n * 16);
  float2* best = reinterpret_cast<float2*>(ws);
  ws += al(size_t(B) * chunks * n * 8);
  double* ctr = reinterpret_cast<double*>(ws);
  lsk::k_pts_center<<<B, 256, 0, st>>>(X, Y, n, m, d, ctr);
  lsk::k_pts_pack<<<256, 256, 0, st>>>(X, (long long)B * n, n, d, ctr, X4);
  lsk::k_pts_pack<<<256, 256, 0, st>>>(Y, (long long)B * m, m, d, ctr, Y4);
  const EpsC ec = epsc(eps);
  lsk::PtsConsume h{B, n, m, chunks, X4, Y4, f, g, log_nu, scale, ec.inv, part, best};
  const int tiles = (n + lsk::kPtsTileRows - 1) / lsk::kPtsTileRows;
  lsk::k_pts_consume<<<dim3(chunks, tiles, B), lsk::kPtsThreads, 0, st>>>(h);
  lsk::k_pts_consume_finish<<<dim3((n + 255) / 256, B), 256, 0, st>>>(B, n, m, d, chunks, part, best, X4, Y4, f, g,
                                                                    log_mu, log_nu, scale, ec.inv, mapped_out,
                                                                    match_idx, match_w, zero_rows, ctr);
  P_CUDA(cudaGetLastError());
  return LSK_OK;
}

}  // extern "C"

// Exact fp64 max of sum_k (x_ik - y_jk)^2 per problem (the C.max() normaliser of
// applications.py:186-188) without materialising C: an fp32 screen of all
// pairs on translated points, then exact fp64 re-evaluation of the pairs within
// 1e-5 of the screened max. The fp32 value of any pair is within ~1e-6
// relative of its exact value (translation to the bounding-box centre bounds
// the rounded coordinates by the box half-diagonal, at most sqrt(3)/2 of the
// largest pair distance's span), so the true maximiser is always among the
// re-evaluated pairs.
extern "C" size_t lsk_points_cost_max_workspace_bytes(int32_t B, int32_t n, int32_t m) {
  if (B < 1 || n < 1 || m < 1) return 0;
  return al(size_t(B) * n * 16) + al(size_t(B) * m * 16) + al(size_t(B) * 4) + al(size_t(B) * 24);
}

extern "C" int32_t lsk_points_cost_max(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                                       double* cmax_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!X || !Y || !cmax_out) return pfail(LSK_EINVAL, "null pointer");
  if (B < 1 || n < 1 || m < 1 || d < 1) return pfail(LSK_EINVAL, "bad shape");
  if (d > 3) return pfail(LSK_EUNSUPPORTED, "points cost max supports d in 1..3");
  if (!workspace || workspace_bytes < lsk_points_cost_max_workspace_bytes(B, n, m))
    return pfail(LSK_EINVAL, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  float4* X4 = reinterpret_cast<float4*>(ws);
  ws += al(size_t(B) * n * 16);
  float4* Y4 = reinterpret_cast<float4*>(ws);
  ws += al(size_t(B) * m * 16);
  unsigned* m32 = reinterpret_cast<unsigned*>(ws);
  ws += al(size_t(B) * 4);
  double* ctr = reinterpret_cast<double*>(ws);
  lsk::k_pts_center<<<B, 256, 0, st>>>(X, Y, n, m, d, ctr);
  lsk::k_pts_pack<<<256, 256, 0, st>>>(X, (long long)B * n, n, d, ctr, X4);
  lsk::k_pts_pack<<<256, 256, 0, st>>>(Y, (long long)B * m, m, d, ctr, Y4);
  P_CUDA(cudaMemsetAsync(m32, 0, size_t(B) * 4, st));
  P_CUDA(cudaMemsetAsync(cmax_out, 0, size_t(B) * 8, st));
  const dim3 grid(chunks_of(m), (n + lsk::kPtsTileRows - 1) / lsk::kPtsTileRows, B);
  unsigned long long* m64 = reinterpret_cast<unsigned long long*>(cmax_out);
  lsk::k_pts_cmax2<0><<<grid, lsk::kPtsThreads, 0, st>>>(n, m, d, X4, Y4, X, Y, m32, m64);
  lsk::k_pts_cmax2<1><<<grid, lsk::kPtsThreads, 0, st>>>(n, m, d, X4, Y4, X, Y, m32, m64);
  P_CUDA(cudaGetLastError());
  return LSK_OK;
}

// (B, 2) device doubles: [b][0] = exact fp64 max, [b][1] = exact fp64 min of
// sum_k (x_ik - y_jk)^2 -- the max/min behind CostMatrix.value_range
// (types.py:60-86) for the pipelines' C / C.max() gate (applications.py:186).
extern "C" int32_t lsk_points_cost_range(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                                         double* range_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!range_out) return pfail(LSK_EINVAL, "null pointer");
  if (!workspace || workspace_bytes < lsk_points_cost_max_workspace_bytes(B, n, m) + al(size_t(B) * 16))
    return pfail(LSK_EINVAL, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  const size_t base = lsk_points_cost_max_workspace_bytes(B, n, m);
  double* mx = reinterpret_cast<double*>(ws + base);
  double* mn = mx + B;
  int32_t rc = lsk_points_cost_max(X, Y, B, n, m, d, mx, workspace, base, stream);
  if (rc != LSK_OK) return rc;
  const unsigned long long inf_bits = 0x7FF0000000000000ull;
  P_CUDA(cudaMemsetAsync(mn, 0, size_t(B) * 8, st));
  k_fill_u64<<<(B + 127) / 128, 128, 0, st>>>(reinterpret_cast<unsigned long long*>(mn), B, inf_bits);
  lsk::k_pts_cmin64<<<dim3((m + 255) / 256, (n + 63) / 64, B), 256, 0, st>>>(
      n, m, d, X, Y, reinterpret_cast<unsigned long long*>(mn));
  k_interleave2<<<(B + 127) / 128, 128, 0, st>>>(mx, mn, B, range_out);
  P_CUDA(cudaGetLastError());
  return LSK_OK;
}

extern "C" size_t lsk_points_cost_range_workspace_bytes(int32_t B, int32_t n, int32_t m) {
  if (B < 1 || n < 1 || m < 1) return 0;
  return lsk_points_cost_max_workspace_bytes(B, n, m) + al(size_t(B) * 16);
}

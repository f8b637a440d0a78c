// Dense solve for m > 8192 (beyond the register-resident persistent kernel):
// a host-enqueued loop of the standalone half-step kernels with every check
// decision on the device (no host synchronisation inside the loop).
//
// Reference path replaced: solve (solver.py:230-337) exactly as the reference
// orders it: per iteration the alpha step (76-80) as a row LSE -- one pass
// shifted by the previous f with an exact two-pass fallback per row
// (k_row_alpha_stale, LSK_FLAG_STALE_SHIFT) or the exact two-pass
// k_row_lse<kRowAlpha> -- the beta step (83-94) as coalesced column (max,
// sumexp) partials + fixed-order combine (k_col_pairs / k_col_combine), and at
// every checkpoint the finiteness test and the reference marginal-error formula
// (97-104, k_row_lse<kRowCheck>) summed in fixed 1024-row blocks; the extra
// check at a cap that is not a checkpoint (301-316); the cost (107-115).
// Memory traffic: one pass of C per half-step (the row LSE's second pass hits
// L1/L2), i.e. the 2*n*m*4 bytes/iteration of SURVEY 8(d).
#include <cmath>
#include <string>

#include "../../include/lsk.h"
#include "lsk_kernels.cuh"
#include "lsk_points.cuh"
#include "lsk_poll.h"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace {

#define L_CUDA(expr)                                                                                    \
  do {                                                                                                  \
    cudaError_t e__ = (expr);                                                                           \
    if (e__ != cudaSuccess) return lsk_host::fail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

inline size_t al(size_t x) { return (x + 255) / 256 * 256; }

int beta_parts(int n, int m, int sms, int* rs_out) {
  const int tiles = (m + 1023) / 1024;
  const int want = (8 * sms + tiles - 1) / tiles;  // ~8 CTAs per SM: enough rows in flight for HBM
  int rs = (n + want - 1) / want;
  if (rs < 64) rs = 64;
  *rs_out = rs;
  return (n + rs - 1) / rs;
}

struct LoopLayout {
  size_t f0, f1, g0, g1, pairs, rowterm, blk, bad, state, act, total;
};

LoopLayout loop_layout(int n, int m, int sms) {
  LoopLayout L{};
  int rs;
  const int parts = beta_parts(n, m, sms, &rs);
  size_t o = 0;
  L.f0 = o; o = al(o + size_t(n) * 4);
  L.f1 = o; o = al(o + size_t(n) * 4);
  L.g0 = o; o = al(o + size_t(m) * 4);
  L.g1 = o; o = al(o + size_t(m) * 4);
  L.pairs = o; o = al(o + size_t(parts) * m * 8);
  L.rowterm = o; o = al(o + size_t(n) * 4);
  L.blk = o; o = al(o + size_t((n + lsk::kPtsBlk - 1) / lsk::kPtsBlk) * 4);
  L.bad = o; o = al(o + 16);
  L.state = o; o = al(o + sizeof(lsk::PtsState));
  L.act = o; o = al(o + 16);
  L.total = o;
  return L;
}

int num_sms_() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

__global__ void k_loop_init(lsk::PtsState* st, int* act) {
  lsk::PtsState s{};
  s.active = 1;
  *st = s;
  *act = 1;
}
__global__ void k_loop_active(const lsk::PtsState* st, int* act) { *act = st->active; }
// LSK_FLAG_UNIFORM_NU contract (include/lsk.h): a non-uniform log nu ends the
// solve as numerical_failure after 0 iterations (every later kernel sees act = 0)
__global__ void k_loop_verify_uniform(const float* log_nu, int m, lsk::PtsState* st, int* act) {
  const float L = log_nu[0];
  int bad = 0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) bad |= log_nu[j] != L;
  if (__syncthreads_or(bad) && threadIdx.x == 0) {
    st->active = 0;
    st->status = 2;
    st->iters = 0;
    st->err = NAN;
    *act = 0;
  }
}
__global__ void k_loop_results(const lsk::PtsState* st, int32_t* result, float* result_f, int cost) {
  const lsk::PtsState s = *st;
  result[LSK_RES_STATUS] = s.status;
  result[LSK_RES_ITERS] = s.iters;
  result[LSK_RES_NTRACE] = s.ntrace;
  result[3] = s.fbuf;
  result[LSK_RES_ROWGUARD] = 0;
  result[LSK_RES_COLGUARD] = 0;
  result_f[0] = s.err;
  result_f[1] = cost ? s.cost : NAN;
}

}  // namespace

namespace lsk_host {

size_t dense_loop_workspace_bytes(int32_t n, int32_t m) { return loop_layout(n, m, num_sms_()).total; }

int32_t solve_dense_loop(const float* C, int64_t ldc, int32_t n, int32_t m, const float* log_mu,
                         const float* log_nu, const float* mu, float inv_eps, float neg_eps, double tol,
                         int32_t K, int32_t c, int32_t flags, float* f_out, float* g_out, int32_t* trace_iter,
                         float* trace_err, int32_t* result, float* result_f, void* workspace,
                         size_t workspace_bytes, cudaStream_t st) {
  const int sms = num_sms_();
  const LoopLayout L = loop_layout(n, m, sms);
  if (!workspace || workspace_bytes < L.total) return fail(LSK_EINVAL, "workspace too small");
  char* ws = static_cast<char*>(workspace);
  float* F[2] = {reinterpret_cast<float*>(ws + L.f0), reinterpret_cast<float*>(ws + L.f1)};
  float* G[2] = {reinterpret_cast<float*>(ws + L.g0), reinterpret_cast<float*>(ws + L.g1)};
  float2* pairs = reinterpret_cast<float2*>(ws + L.pairs);
  float* rowterm = reinterpret_cast<float*>(ws + L.rowterm);
  float* blk = reinterpret_cast<float*>(ws + L.blk);
  int* bad = reinterpret_cast<int*>(ws + L.bad);
  lsk::PtsState* S = reinterpret_cast<lsk::PtsState*>(ws + L.state);
  int* act = reinterpret_cast<int*>(ws + L.act);
  const int cap = lsk_trace_capacity(K, c);
  int rs;
  const int parts = beta_parts(n, m, sms, &rs);
  const int nb = (n + lsk::kPtsBlk - 1) / lsk::kPtsBlk;

  L_CUDA(cudaMemsetAsync(F[0], 0, size_t(n) * 4, st));
  L_CUDA(cudaMemsetAsync(G[0], 0, size_t(m) * 4, st));
  L_CUDA(cudaMemsetAsync(bad, 0, 16, st));
  k_loop_init<<<1, 1, 0, st>>>(S, act);
  if (flags & LSK_FLAG_UNIFORM_NU) k_loop_verify_uniform<<<1, 1024, 0, st>>>(log_nu, m, S, act);

  // the checkpoint of iterate kk; `fused`: its per-row terms came with the stale row pass
  auto check = [&](int kk, bool final, bool fused) -> int32_t {
    const float* fk = F[kk & 1];
    const float* gk = G[kk & 1];
    if (!fused)
      lsk::k_row_lse<lsk::kRowCheck><<<n, 256, 0, st>>>(C, ldc, n, m, fk, gk, log_nu, log_mu, mu, inv_eps, neg_eps,
                                                        rowterm, act);
    lsk::k_pts_colcheck<<<dim3(8, 1), 256, 0, st>>>(1, n, fk, act, bad);
    lsk::k_pts_colcheck<<<dim3(8, 1), 256, 0, st>>>(1, m, gk, act, bad);
    lsk::k_pts_blocksum<<<dim3(nb, 1), 1024, 0, st>>>(1, n, 0, n, rowterm, act, blk);
    lsk::k_pts_decide<<<1, 32, 0, st>>>(1, n, blk, bad, tol, kk, final ? 1 : 0, S, trace_iter, trace_err, cap);
    k_loop_active<<<1, 1, 0, st>>>(S, act);
    L_CUDA(cudaGetLastError());
    return LSK_OK;
  };
  int32_t rc;
  const bool stale = (flags & LSK_FLAG_STALE_SHIFT) != 0;
  lsk_poll::StopPoll poll;
  if ((rc = poll.init(1, st))) return rc;
  const bool uni = (flags & LSK_FLAG_UNIFORM_NU) != 0;
  // one read of the row, shifted by the stale f (exact fallback per row); at a
  // checkpoint the same read forms the check terms of iterate k-1
  auto row_stale = [&](int k, bool chk) {
    const float* fp = F[(k - 1) & 1];
    const float* gp = G[(k - 1) & 1];
    float* fn = F[k & 1];
    if (chk && uni)
      lsk::k_row_alpha_stale<true, true><<<n, 256, 0, st>>>(C, ldc, n, m, fp, gp, log_nu, inv_eps, neg_eps, fn, act,
                                                            log_mu, mu, rowterm);
    else if (chk)
      lsk::k_row_alpha_stale<true, false><<<n, 256, 0, st>>>(C, ldc, n, m, fp, gp, log_nu, inv_eps, neg_eps, fn, act,
                                                             log_mu, mu, rowterm);
    else if (uni)
      lsk::k_row_alpha_stale<false, true><<<n, 256, 0, st>>>(C, ldc, n, m, fp, gp, log_nu, inv_eps, neg_eps, fn, act);
    else
      lsk::k_row_alpha_stale<false, false><<<n, 256, 0, st>>>(C, ldc, n, m, fp, gp, log_nu, inv_eps, neg_eps, fn, act);
  };
  for (int k = 1; k <= K; ++k) {
    const bool chk = k > 1 && (k - 1) % c == 0;
    if (k > 1 && stale) row_stale(k, chk);
    if (chk) {
      if ((rc = check(k - 1, false, stale))) return rc;
      bool stop = false;
      if ((rc = poll.after_check(act, st, stop))) return rc;
      if (stop) break;
    }
    if (!(k > 1 && stale))
      lsk::k_row_lse<lsk::kRowAlpha><<<n, 256, 0, st>>>(C, ldc, n, m, nullptr, G[(k - 1) & 1], log_nu, nullptr,
                                                        nullptr, inv_eps, neg_eps, F[k & 1], act);
    lsk::k_col_pairs<<<dim3((m + 1023) / 1024, parts), 256, 0, st>>>(C, ldc, n, m, F[k & 1], log_mu, inv_eps, rs,
                                                                    pairs, act);
    lsk::k_col_combine<<<(8 * m + 255) / 256, 256, 0, st>>>(pairs, parts, m, neg_eps, G[k & 1], act);
    L_CUDA(cudaGetLastError());
  }
  if ((rc = check(K, true, false))) return rc;
  lsk::k_pts_pick<<<dim3(64, 1), 256, 0, st>>>(1, n, F[0], F[1], S, f_out);
  lsk::k_pts_pick<<<dim3(64, 1), 256, 0, st>>>(1, m, G[0], G[1], S, g_out);
  if (flags & LSK_FLAG_COST) {
    lsk::k_row_lse<lsk::kRowCost><<<n, 256, 0, st>>>(C, ldc, n, m, f_out, g_out, log_nu, log_mu, nullptr, inv_eps,
                                                     neg_eps, rowterm);
    lsk::k_pts_blocksum<<<dim3(nb, 1), 1024, 0, st>>>(1, n, 0, n, rowterm, nullptr, blk);
    lsk::k_pts_cost_finish<<<1, 32, 0, st>>>(1, n, blk, S);
  }
  k_loop_results<<<1, 1, 0, st>>>(S, result, result_f, (flags & LSK_FLAG_COST) ? 1 : 0);
  L_CUDA(cudaGetLastError());
  return LSK_OK;
}

}  // namespace lsk_host

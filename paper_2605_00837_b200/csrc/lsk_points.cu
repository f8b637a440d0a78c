// C-ABI of the on-the-fly points solver (include/lsk.h: lsk_solve_points_f32,
// lsk_points_cost_max, lsk_comm_*): argument checks, workspace carving and the
// host-side iteration loop. The loop only enqueues (no host synchronisation):
// every check decision, stop flag and trace entry lives on the device, and the
// kernels of a problem that has stopped exit immediately.
//
// Sharding (owner computes): with a communicator of P ranks, rank
// r computes f for rows [r n/P, (r+1) n/P) against all of Y and g, and g for
// columns [r m/P, (r+1) m/P) against all of X and f; an ncclAllGather after
// each half-step replicates the potentials. Every potential is produced by the
// same kernel over the same column chunks as on one GPU, so the potentials,
// the trace and the stop iteration are bit-identical for every P.
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

struct PtsLayout {
  size_t x4, y4, f0, f1, g0, g1, part, rowflag, nflag, errrow, errblk, bad, costrow, costblk, state, total;
};

PtsLayout pts_layout(int B, int n, int m) {
  PtsLayout L{};
  size_t o = 0;
  const size_t nm = n > m ? n : m;
  const size_t pmax = size_t(B) * (size_t(chunks_of(m)) * n > size_t(chunks_of(n)) * m ? size_t(chunks_of(m)) * n
                                                                                        : size_t(chunks_of(n)) * m);
  L.x4 = o; o = al(o + size_t(B) * n * 16);
  L.y4 = o; o = al(o + size_t(B) * m * 16);
  L.f0 = o; o = al(o + size_t(B) * n * 4);
  L.f1 = o; o = al(o + size_t(B) * n * 4);
  L.g0 = o; o = al(o + size_t(B) * m * 4);
  L.g1 = o; o = al(o + size_t(B) * m * 4);
  L.part = o; o = al(o + pmax * 8);
  L.rowflag = o; o = al(o + size_t(B) * nm * 4);
  L.nflag = o; o = al(o + 16);
  L.errrow = o; o = al(o + size_t(B) * n * 4);
  L.errblk = o; o = al(o + size_t(B) * ((n + lsk::kPtsBlk - 1) / lsk::kPtsBlk) * 4);
  L.bad = o; o = al(o + size_t(B) * 4);
  L.costrow = o; o = al(o + size_t(B) * n * 4);
  L.costblk = o; o = al(o + size_t(B) * ((n + lsk::kPtsBlk - 1) / lsk::kPtsBlk) * 4);
  L.state = o; o = al(o + size_t(B) * sizeof(lsk::PtsState));
  L.total = o;
  return L;
}

struct EpsC {
  float inv, neg;
};
EpsC epsc(double eps) {
  volatile float e32 = static_cast<float>(eps);
  volatile float one = 1.0f;
  return {one / e32, -e32};
}

__global__ void k_pts_init(int B, lsk::PtsState* st) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  lsk::PtsState s{};
  s.active = 1;
  st[b] = s;
}

// one half-step: rows R (slab [lo, hi)) against all columns C
struct Half {
  const float4* rpts;
  const float4* cpts;
  int nr, nc;
  const float* rpot_old;
  float* rpot_new;
  const float* cpot;
  const float* clw;
};

struct Ctx {
  int B, n, m;
  lsk::PtsState* st;
  int* active;  // &st[0].active with stride (see kernels: they read active[b] via PtsState layout)
  void* part;
  int* rowflag;
  int* nflag;
  float inv, neg;
  const float* scale;
  cudaStream_t s;
};

}  // namespace

namespace {
// active flags are read as int per problem: expose st[b].active
__global__ void k_active_view(int B, const lsk::PtsState* st, int* act) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) act[b] = st[b].active;
}

__global__ void k_pts_rowsum(int B, int n, int lo, int hi, int chunks, const float* part, float* out) {
  const int b = blockIdx.y;
  const int r = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi) return;
  float s = 0.f;
  for (int ch = 0; ch < chunks; ++ch) s += part[((size_t)b * chunks + ch) * n + r];
  out[(size_t)b * n + r] = s;
}

__global__ void k_pts_results(int B, const lsk::PtsState* st, int32_t* result, float* result_f, int cost) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const lsk::PtsState s = st[b];
  result[b * 8 + LSK_RES_STATUS] = s.status;
  result[b * 8 + LSK_RES_ITERS] = s.iters;
  result[b * 8 + LSK_RES_NTRACE] = s.ntrace;
  result[b * 8 + 3] = s.fbuf;
  result_f[b * 2 + 0] = s.err;
  result_f[b * 2 + 1] = cost ? s.cost : NAN;
}

int32_t run_part(int mode, const Half& h, int lo, int hi, const Ctx& c, const int* active, const float* rlw,
                 const int* rowflag, const int* nflag) {
  lsk::PtsHalf ph{};
  ph.B = c.B;
  ph.n_rows = h.nr;
  ph.n_cols = h.nc;
  ph.row_lo = lo;
  ph.row_hi = hi;
  ph.chunks = chunks_of(h.nc);
  ph.rpts = h.rpts;
  ph.cpts = h.cpts;
  ph.rpot = h.rpot_old;
  ph.cpot = h.cpot;
  ph.clw = h.clw;
  ph.rlw = rlw;
  ph.scale = c.scale;
  ph.inv_eps = c.inv;
  ph.part = c.part;
  ph.active = active;
  ph.rowflag = rowflag;
  ph.nflag = nflag;
  // rows per warp of the partial sweeps
  constexpr int kWide = 8;  // 16 rows per warp measured 7% slower (register pressure, 2 CTAs/SM)
  const int tile_rows = (mode == lsk::kPtsOnline) ? lsk::kPtsTileRows : 8 * kWide;
  const int tiles = (hi - lo + tile_rows - 1) / tile_rows;
  if (tiles <= 0) return LSK_OK;
  dim3 grid(ph.chunks, tiles, c.B);
  if (mode == lsk::kPtsStale) lsk::k_pts_part<lsk::kPtsStale, kWide><<<grid, lsk::kPtsThreads, 0, c.s>>>(ph);
  else if (mode == lsk::kPtsStaleX) lsk::k_pts_part<lsk::kPtsStaleX, kWide><<<grid, lsk::kPtsThreads, 0, c.s>>>(ph);
  else if (mode == lsk::kPtsOnline) lsk::k_pts_part<lsk::kPtsOnline, 8><<<grid, lsk::kPtsThreads, 0, c.s>>>(ph);
  else lsk::k_pts_part<lsk::kPtsCost, kWide><<<grid, lsk::kPtsThreads, 0, c.s>>>(ph);
  P_CUDA(cudaGetLastError());
  return LSK_OK;
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

size_t lsk_solve_points_workspace_bytes(int32_t B, int32_t n, int32_t m) {
  if (B < 1 || n < 1 || m < 1) return 0;
  return pts_layout(B, n, m).total + size_t(B) * 4 + 256;
}

int32_t lsk_solve_points_f32(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                             const float* scale, const float* log_mu, const float* log_nu, const float* mu,
                             double eps, double tol, int32_t max_iter, int32_t check_interval, int32_t flags,
                             float* f_out, float* g_out, int32_t* trace_iter, float* trace_err, int32_t* result,
                             float* result_f, void* workspace, size_t workspace_bytes, void* comm, void* stream) {
  if (!X || !Y || !scale || !log_mu || !log_nu || !mu || !f_out || !g_out || !trace_iter || !trace_err || !result ||
      !result_f)
    return pfail(LSK_EINVAL, "null pointer");
  if (B < 1 || n < 1 || m < 1) return pfail(LSK_EINVAL, "B, n, m must be >= 1");
  if (d < 1 || d > 3) return pfail(LSK_EUNSUPPORTED, "points solver supports d in 1..3");
  if (!(eps > 0) || !(tol > 0) || max_iter < 1 || check_interval < 1)
    return pfail(LSK_EINVAL, "eps, tol > 0; max_iter, check_interval >= 1 required");
  const PtsLayout L = pts_layout(B, n, m);
  if (!workspace || workspace_bytes < lsk_solve_points_workspace_bytes(B, n, m))
    return pfail(LSK_EINVAL, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ncclComm_t nc = static_cast<ncclComm_t>(comm);
  int P = 1, rank = 0;
  if (nc) {
    P_NCCL(ncclCommCount(nc, &P));
    P_NCCL(ncclCommUserRank(nc, &rank));
    if (B != 1) return pfail(LSK_EUNSUPPORTED, "sharded points solve: one problem per call (split batches instead)");
    if (n % P || m % P) return pfail(LSK_EINVAL, "sharded points solve: n and m must be multiples of the rank count");
  }
  const int rlo = int((long long)rank * n / P), rhi = int((long long)(rank + 1) * n / P);
  const int clo = int((long long)rank * m / P), chi = int((long long)(rank + 1) * m / P);
  char* ws = static_cast<char*>(workspace);
  float4* X4 = reinterpret_cast<float4*>(ws + L.x4);
  float4* Y4 = reinterpret_cast<float4*>(ws + L.y4);
  float* F[2] = {reinterpret_cast<float*>(ws + L.f0), reinterpret_cast<float*>(ws + L.f1)};
  float* Gp[2] = {reinterpret_cast<float*>(ws + L.g0), reinterpret_cast<float*>(ws + L.g1)};
  int* rowflag = reinterpret_cast<int*>(ws + L.rowflag);
  int* nflag = reinterpret_cast<int*>(ws + L.nflag);
  float* errrow = reinterpret_cast<float*>(ws + L.errrow);
  float* errblk = reinterpret_cast<float*>(ws + L.errblk);
  int* bad = reinterpret_cast<int*>(ws + L.bad);
  float* costrow = reinterpret_cast<float*>(ws + L.costrow);
  float* costblk = reinterpret_cast<float*>(ws + L.costblk);
  lsk::PtsState* S = reinterpret_cast<lsk::PtsState*>(ws + L.state);
  int* act = reinterpret_cast<int*>(ws + L.total);
  const EpsC ec = epsc(eps);
  const int cap = lsk_trace_capacity(max_iter, check_interval);

  P_CUDA(cudaMemsetAsync(F[0], 0, size_t(B) * n * 4, st));
  P_CUDA(cudaMemsetAsync(Gp[0], 0, size_t(B) * m * 4, st));
  P_CUDA(cudaMemsetAsync(rowflag, 0, size_t(B) * (n > m ? n : m) * 4, st));
  P_CUDA(cudaMemsetAsync(nflag, 0, 16, st));
  P_CUDA(cudaMemsetAsync(bad, 0, size_t(B) * 4, st));
  lsk::k_pts_pack<<<256, 256, 0, st>>>(X, (long long)B * n, n, d, X, n, X4);
  lsk::k_pts_pack<<<256, 256, 0, st>>>(Y, (long long)B * m, m, d, X, n, Y4);
  k_pts_init<<<(B + 127) / 128, 128, 0, st>>>(B, S);
  P_CUDA(cudaGetLastError());

  Ctx c{B, n, m, S, act, ws + L.part, rowflag, nflag, ec.inv, ec.neg, scale, st};
  const bool stale = (flags & LSK_FLAG_STALE_SHIFT) != 0;
  // expansion-form cost in the stale sweeps: only where its rounding is at the
  // reference's own level (eps >= 5e-3), and only when asked for
  const bool expansion = (flags & LSK_FLAG_EXPANSION) != 0 && eps >= 5e-3;
  auto refresh_active = [&]() -> int32_t {
    k_active_view<<<(B + 127) / 128, 128, 0, st>>>(B, S, act);
    P_CUDA(cudaGetLastError());
    return LSK_OK;
  };
  int32_t rc;
  // one half-step: new row potentials of the slab [lo, hi) (and, when check,
  // the error terms of the iterate whose potentials are (rpot_old, cpot))
  auto half = [&](const Half& h, int lo, int hi, bool use_stale, bool check, const float* rlw,
                  const float* rmu) -> int32_t {
    if (use_stale) {
      if ((rc = run_part(expansion ? lsk::kPtsStaleX : lsk::kPtsStale, h, lo, hi, c, act, nullptr, nullptr, nullptr)))
        return rc;
      lsk::PtsCombine cb{};
      cb.B = B; cb.n_rows = h.nr; cb.row_lo = lo; cb.row_hi = hi; cb.chunks = chunks_of(h.nc);
      cb.part = c.part; cb.rpot_old = h.rpot_old; cb.rpot_new = h.rpot_new; cb.inv_eps = ec.inv;
      cb.neg_eps = ec.neg; cb.active = act; cb.rowflag = rowflag; cb.nflag = nflag;
      cb.rlw = rlw; cb.rmu = rmu; cb.cpot = h.cpot; cb.errrow = errrow; cb.badrow = bad; cb.check = check;
      dim3 g((hi - lo + 255) / 256, B);
      lsk::k_pts_combine<lsk::kPtsStale><<<g, 256, 0, st>>>(cb);
      P_CUDA(cudaGetLastError());
      if (!h.rpot_new) return LSK_OK;  // check only
      // guard: rows whose stale sum left [1e-20, 1e30] are recomputed exactly by
      // one CTA per problem (exits at once when nothing was flagged)
      {
        lsk::PtsHalf ph{};
        ph.B = B; ph.n_rows = h.nr; ph.n_cols = h.nc; ph.row_lo = lo; ph.row_hi = hi;
        ph.rpts = h.rpts; ph.cpts = h.cpts; ph.cpot = h.cpot; ph.clw = h.clw; ph.scale = c.scale;
        ph.inv_eps = ec.inv; ph.active = act;
        lsk::k_pts_fixup<<<B, 256, 0, st>>>(ph, ec.neg, h.rpot_new, rowflag, nflag);
        P_CUDA(cudaGetLastError());
      }
      P_CUDA(cudaMemsetAsync(nflag, 0, 4, st));
    } else {
      if ((rc = run_part(lsk::kPtsOnline, h, lo, hi, c, act, nullptr, nullptr, nullptr))) return rc;
      lsk::PtsCombine co{};
      co.B = B; co.n_rows = h.nr; co.row_lo = lo; co.row_hi = hi; co.chunks = chunks_of(h.nc);
      co.part = c.part; co.rpot_new = h.rpot_new; co.inv_eps = ec.inv; co.neg_eps = ec.neg; co.active = act;
      dim3 g((hi - lo + 255) / 256, B);
      lsk::k_pts_combine<lsk::kPtsOnline><<<g, 256, 0, st>>>(co);
      P_CUDA(cudaGetLastError());
    }
    return LSK_OK;
  };
  auto gather = [&](float* buf, int count_per_rank) -> int32_t {
    if (!nc || P == 1) return LSK_OK;
    P_NCCL(ncclAllGather(buf + size_t(rank) * count_per_rank, buf, size_t(count_per_rank), ncclFloat, nc, st));
    return LSK_OK;
  };
  // check decision for iterate kk from the f-half's row terms
  auto decide = [&](int kk, const float* gk, bool final) -> int32_t {
    lsk::k_pts_colcheck<<<dim3(8, B), 256, 0, st>>>(B, m, gk, act, bad);
    P_CUDA(cudaGetLastError());
    if (nc && P > 1) {
      if ((rc = gather(errrow, n / P))) return rc;
      P_NCCL(ncclAllReduce(bad, bad, size_t(B), ncclInt32, ncclMax, nc, st));
    }
    const int nb = (n + lsk::kPtsBlk - 1) / lsk::kPtsBlk;
    lsk::k_pts_blocksum<<<dim3(nb, B), 1024, 0, st>>>(B, n, 0, n, errrow, act, errblk);
    lsk::k_pts_decide<<<(B + 127) / 128, 128, 0, st>>>(B, n, errblk, bad, tol, kk, final ? 1 : 0, S, trace_iter,
                                                        trace_err, cap);
    P_CUDA(cudaGetLastError());
    return refresh_active();
  };

  if ((rc = refresh_active())) return rc;
  for (int k = 1; k <= max_iter; ++k) {
    const bool do_check = (k > 1) && ((k - 1) % check_interval == 0);
    const float* fprev = F[(k - 1) & 1];
    float* fnew = F[k & 1];
    const float* gprev = Gp[(k - 1) & 1];
    float* gnew = Gp[k & 1];
    const bool st_k = stale && k > 1;
    if (do_check && !st_k) {  // exact variant: a separate check pass of iterate k-1
      Half hc{X4, Y4, n, m, fprev, nullptr, gprev, log_nu};
      if ((rc = half(hc, rlo, rhi, true, true, log_mu, mu))) return rc;
    }
    Half hf{X4, Y4, n, m, fprev, fnew, gprev, log_nu};
    if ((rc = half(hf, rlo, rhi, st_k, do_check && st_k, log_mu, mu))) return rc;
    if ((rc = gather(fnew, n / P))) return rc;
    if (do_check && (rc = decide(k - 1, gprev, false))) return rc;
    Half hg{Y4, X4, m, n, gprev, gnew, fnew, log_mu};
    if ((rc = half(hg, clo, chi, st_k, false, nullptr, nullptr))) return rc;
    if ((rc = gather(gnew, m / P))) return rc;
  }
  // the final check at the cap (solver.py:286-316): a check-only f-pass of iterate K
  {
    const int K = max_iter;
    Half hc{X4, Y4, n, m, F[K & 1], nullptr, Gp[K & 1], log_nu};
    if ((rc = half(hc, rlo, rhi, true, true, log_mu, mu))) return rc;
    if ((rc = decide(K, Gp[K & 1], true))) return rc;
  }
  // potentials of the returned iterate, then the transport cost from them
  lsk::k_pts_pick<<<dim3(64, B), 256, 0, st>>>(B, n, F[0], F[1], S, f_out);
  lsk::k_pts_pick<<<dim3(64, B), 256, 0, st>>>(B, m, Gp[0], Gp[1], S, g_out);
  P_CUDA(cudaGetLastError());
  if (flags & LSK_FLAG_COST) {
    Half hk{X4, Y4, n, m, f_out, nullptr, g_out, log_nu};
    if ((rc = run_part(lsk::kPtsCost, hk, rlo, rhi, c, nullptr, log_mu, nullptr, nullptr))) return rc;
    // per-row sums of the chunk partials (fixed order) -> costrow
    k_pts_rowsum<<<dim3((rhi - rlo + 255) / 256, B), 256, 0, st>>>(B, n, rlo, rhi, chunks_of(m),
                                                                  reinterpret_cast<const float*>(c.part), costrow);
    P_CUDA(cudaGetLastError());
    if ((rc = gather(costrow, n / P))) return rc;
    const int nb = (n + lsk::kPtsBlk - 1) / lsk::kPtsBlk;
    lsk::k_pts_blocksum<<<dim3(nb, B), 1024, 0, st>>>(B, n, 0, n, costrow, nullptr, costblk);
    lsk::k_pts_cost_finish<<<(B + 127) / 128, 128, 0, st>>>(B, n, costblk, S);
    P_CUDA(cudaGetLastError());
  }
  k_pts_results<<<(B + 127) / 128, 128, 0, st>>>(B, S, result, result_f, (flags & LSK_FLAG_COST) ? 1 : 0);
  P_CUDA(cudaGetLastError());
  return LSK_OK;
}


// ---- plan consumers without the plan
size_t lsk_points_consume_workspace_bytes(int32_t B, int32_t n, int32_t m) {
  if (B < 1 || n < 1 || m < 1) return 0;
  const size_t ch = size_t(chunks_of(m));
  return al(size_t(B) * n * 16) + al(size_t(B) * m * 16) + al(size_t(B) * ch * n * 16) + al(size_t(B) * ch * n * 8);
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
  lsk::k_pts_pack<<<256, 256, 0, st>>>(X, (long long)B * n, n, d, X, n, X4);
  lsk::k_pts_pack<<<256, 256, 0, st>>>(Y, (long long)B * m, m, d, X, n, Y4);
  const EpsC ec = epsc(eps);
  lsk::PtsConsume h{B, n, m, chunks, X4, Y4, f, g, log_nu, scale, ec.inv, part, best};
  const int tiles = (n + lsk::kPtsTileRows - 1) / lsk::kPtsTileRows;
  lsk::k_pts_consume<<<dim3(chunks, tiles, B), lsk::kPtsThreads, 0, st>>>(h);
  lsk::k_pts_consume_finish<<<dim3((n + 255) / 256, B), 256, 0, st>>>(B, n, m, d, chunks, part, best, X4, Y4, f, g,
                                                                    log_mu, log_nu, scale, ec.inv, mapped_out,
                                                                    match_idx, match_w, zero_rows, X);
  P_CUDA(cudaGetLastError());
  return LSK_OK;
}

}  // extern "C"

// Exact fp64 max of sum_k (x_ik - y_jk)^2 per problem (the C.max() normaliser of
// applications.py:186-188) without materialising C: an fp32 screen of all
// pairs on translated points, then exact fp64 re-evaluation of the pairs within
// 1e-5 of the screened max. The fp32 value of any pair is within ~1e-6
// relative of its exact value (translation by a data point bounds the rounded
// coordinates by twice the largest pair distance), so the true maximiser is
// always among the re-evaluated pairs.
extern "C" size_t lsk_points_cost_max_workspace_bytes(int32_t B, int32_t n, int32_t m) {
  if (B < 1 || n < 1 || m < 1) return 0;
  return al(size_t(B) * n * 16) + al(size_t(B) * m * 16) + al(size_t(B) * 4);
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
  lsk::k_pts_pack<<<256, 256, 0, st>>>(X, (long long)B * n, n, d, X, n, X4);
  lsk::k_pts_pack<<<256, 256, 0, st>>>(Y, (long long)B * m, m, d, X, n, Y4);
  P_CUDA(cudaMemsetAsync(m32, 0, size_t(B) * 4, st));
  P_CUDA(cudaMemsetAsync(cmax_out, 0, size_t(B) * 8, st));
  const dim3 grid(chunks_of(m), (n + lsk::kPtsTileRows - 1) / lsk::kPtsTileRows, B);
  unsigned long long* m64 = reinterpret_cast<unsigned long long*>(cmax_out);
  lsk::k_pts_cmax2<0><<<grid, lsk::kPtsThreads, 0, st>>>(n, m, d, X4, Y4, X, Y, m32, m64);
  lsk::k_pts_cmax2<1><<<grid, lsk::kPtsThreads, 0, st>>>(n, m, d, X4, Y4, X, Y, m32, m64);
  P_CUDA(cudaGetLastError());
  return LSK_OK;
}

// C-ABI of the on-the-fly points solve (include/lsk.h: lsk_solve_points_f32,
// lsk_solve_points_emulated_f32 and their workspace queries): argument checks,
// the rank decomposition, workspace carving and the host-side iteration loop.
//
// Reference path replaced: squared_euclidean_cost (costs.py:36-50) [/ C.max(),
// applications.py:186-188] followed by solve (solver.py:230-337).
//
// The loop only enqueues: every check decision, stop flag and trace entry
// lives on the device, and the kernels of a stopped problem exit at once. To
// stop enqueueing after convergence the host polls a pinned copy of the
// per-problem active flags every check, lagging the device by at most two
// check intervals (no stall of the stream; disabled under stream capture).
//
// Multi-GPU, one problem over P ranks, three selectable designs:
//  * owner computes (LSK_SHARD_OWNER): rank r computes f for rows
//    [r rpr, (r+1) rpr) and g for columns [r cpr, (r+1) cpr), rpr = ceil(n/P),
//    cpr = ceil(m/P); an allgather of each potential slab after each half-step.
//  * column partials (LSK_SHARD_PARTIALS, the north star's design): rank r
//    owns a row slab of the source cloud (whole 2048-row chunks) and computes
//    f for it locally; for g it reduces its rows into per-column partials
//    (stale-shift sums, or (max, sumexp) pairs in log2 units) -- the complete
//    subtree of the fixed chunk tree it owns -- and the P subtree roots are
//    allgathered and merged by the top of the same tree on every rank. The
//    tree's shape depends on n only, so g is bit-identical for every
//    power-of-two P and replicated on every rank without a broadcast.
//  * allreduce (LSK_SHARD_ALLREDUCE): as partials, but the stale-shift sums
//    are combined by ncclAllReduce(SUM) of m floats (NCCL's reduction order:
//    not bitwise P-invariant, within float rounding); first / guard
//    iterations use the exact pair exchange.
// Every design allgathers f after the f half-step (4 rpr bytes per rank) so
// the guard fallback, the check and the outputs see the whole potential. The
// check's error and the transport cost sum fixed 1024-row blocks of per-row
// terms, independent of P.
//
// CUDA graphs: after the first checkpoint the loop is a repetition of blocks
// of c iterations (the block's first iteration carries the check of the
// previous iterate), so one block is captured once (two when c is odd: the
// potential buffers alternate with the iteration's parity) and replayed; the
// checked iterate reaches k_pts_decide through a device counter that the
// block's first node advances. The host poll runs between replays. Single-GPU
// and emulated solves use graphs by default; with an NCCL communicator they
// are opt-in (LSK_FLAG_GRAPH_NCCL: NCCL calls captured into the graph), and
// LSK_FLAG_NO_GRAPH enqueues every iteration.
//
// lsk_solve_points_emulated_f32 runs the same decomposition for P virtual
// ranks on one GPU: each rank has its own workspace, the rank-local kernels of
// every phase run rank after rank on one stream, and the collectives become
// device copies (the allreduce a rank-order sum). It proves the P-rank data
// plane -- slabs, exchanges, tree split -- on a single B200; only NCCL itself
// is left to the multi-GPU run.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/lsk.h"
#include "lsk_points.cuh"
#include "lsk_poll.h"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);  // lsk_api.cu: thread-local lsk_last_error()
}

namespace {

int32_t sfail(int32_t code, const std::string& msg) { return lsk_host::fail(code, msg); }
#define S_CUDA(expr)                                                                              \
  do {                                                                                            \
    cudaError_t e__ = (expr);                                                                     \
    if (e__ != cudaSuccess) return sfail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)
#define S_NCCL(expr)                                                                              \
  do {                                                                                            \
    ncclResult_t r__ = (expr);                                                                    \
    if (r__ != ncclSuccess) return sfail(LSK_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r__)); \
  } while (0)
#define S_TRY(expr)                  \
  do {                               \
    int32_t rc__ = (expr);           \
    if (rc__ != LSK_OK) return rc__; \
  } while (0)

inline size_t al(size_t x) { return (x + 255) / 256 * 256; }
inline int chunks_of(int ncols) { return (ncols + lsk::kPtsChunk - 1) / lsk::kPtsChunk; }
inline int cdiv(long long a, long long b) { return int((a + b - 1) / b); }

// ---- the decomposition of the problem over P ranks
struct Shard {
  int mode = LSK_SHARD_NONE;
  int P = 1;
  int rpr = 0;   // f rows per rank (slab stride)
  int cpr = 0;   // owner: g columns per rank
  int xch = 0;   // chunks of the source cloud (g-half "columns")
  int L2 = 1;    // width of the g-half chunk tree
  int spr = 1;   // partials: tree leaves (source chunks) per rank
  int npad = 0, mpad = 0;
};

int32_t make_shard(int n, int m, int P, int mode, Shard& s) {
  s = Shard{};
  s.mode = mode;
  s.P = P;
  s.xch = chunks_of(n);
  s.L2 = lsk::pow2_ceil(s.xch);
  if (mode == LSK_SHARD_NONE) {
    if (P != 1) return sfail(LSK_EINVAL, "LSK_SHARD_NONE with more than one rank");
    s.rpr = n; s.cpr = m;
  } else if (mode == LSK_SHARD_OWNER) {
    s.rpr = cdiv(n, P); s.cpr = cdiv(m, P);
  } else if (mode == LSK_SHARD_PARTIALS || mode == LSK_SHARD_ALLREDUCE) {
    if ((P & (P - 1)) != 0 || P > s.L2)
      return sfail(LSK_EUNSUPPORTED, "column-partials sharding needs a power-of-two rank count <= the source cloud's "
                                     "2048-point chunk tree width (" + std::to_string(s.L2) + ")");
    s.spr = s.L2 / P;
    s.rpr = s.spr * lsk::kPtsChunk;
    s.cpr = m;
  } else {
    return sfail(LSK_EINVAL, "unknown shard mode");
  }
  s.npad = int((long long)s.rpr * P);
  if (s.npad < n) s.npad = n;
  s.mpad = (mode == LSK_SHARD_OWNER) ? int((long long)s.cpr * P) : m;
  if (s.mpad < m) s.mpad = m;
  return LSK_OK;
}

struct PtsLayout {
  size_t x4, y4, ctr, f0, f1, g0, g1, fsel, gsel, part, slots, rowflag, nflag, errrow, errblk, bad, badslots, costrow, costblk, state,
      act, kk, total;
};

PtsLayout pts_layout(int B, int n, int m, const Shard& s) {
  PtsLayout L{};
  size_t o = 0;
  const size_t nm = n > m ? n : m;
  const size_t pa = size_t(chunks_of(m)) * n, pb = size_t(chunks_of(n)) * m;
  const size_t pmax = size_t(B) * (pa > pb ? pa : pb);
  const int nb = (s.npad + lsk::kPtsBlk - 1) / lsk::kPtsBlk;
  L.x4 = o; o = al(o + size_t(B) * n * 16);
  L.y4 = o; o = al(o + size_t(B) * m * 16);
  L.ctr = o; o = al(o + size_t(B) * 24);
  L.f0 = o; o = al(o + size_t(B) * s.npad * 4);
  L.f1 = o; o = al(o + size_t(B) * s.npad * 4);
  L.g0 = o; o = al(o + size_t(B) * s.mpad * 4);
  L.g1 = o; o = al(o + size_t(B) * s.mpad * 4);
  L.fsel = o; o = al(o + size_t(B) * n * 4);
  L.gsel = o; o = al(o + size_t(B) * m * 4);
  L.part = o; o = al(o + pmax * 8);
  L.slots = o; o = al(o + (s.mode == LSK_SHARD_NONE || s.mode == LSK_SHARD_OWNER ? 0 : size_t(s.P) * m * 8));
  L.rowflag = o; o = al(o + size_t(B) * nm * 4);
  L.nflag = o; o = al(o + 16);
  L.errrow = o; o = al(o + size_t(B) * s.npad * 4);
  L.errblk = o; o = al(o + size_t(B) * nb * 4);
  L.bad = o; o = al(o + size_t(B) * 4);
  L.badslots = o; o = al(o + size_t(s.P) * 4);
  L.costrow = o; o = al(o + size_t(B) * s.npad * 4);
  L.costblk = o; o = al(o + size_t(B) * nb * 4);
  L.state = o; o = al(o + size_t(B) * sizeof(lsk::PtsState));
  L.act = o; o = al(o + size_t(B) * 4);
  L.kk = o; o = al(o + 16);
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
__global__ void k_or_slots(int P, const int* slots, int* bad) {
  int v = 0;
  for (int r = 0; r < P; ++r) v |= slots[r];
  bad[0] = v;
}
__global__ void k_put_slot(const int* bad, int* slots, int r) { slots[r] = bad[0]; }

// emulated allreduce: rank-order sum of P equal-length float buffers into the first
struct RankPtrs {
  float* p[LSK_EMU_MAX_RANKS];
};
__global__ void k_sum_ranks(int P, RankPtrs rp, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    float s = rp.p[0][i];
    for (int r = 1; r < P; ++r) s = __fadd_rn(s, rp.p[r][i]);
    rp.p[0][i] = s;
  }
}
// bitwise agreement of a rank's returned iterate with rank 0's
__global__ void k_cmp_rank(int n, int m, const lsk::PtsState* s0, const float* f00, const float* f01,
                           const float* g00, const float* g01, const lsk::PtsState* sr, const float* fr0,
                           const float* fr1, const float* gr0, const float* gr1, int* mismatch) {
  const float* fa = s0->fbuf ? f01 : f00;
  const float* fb = sr->fbuf ? fr1 : fr0;
  const float* ga = s0->fbuf ? g01 : g00;
  const float* gb = sr->fbuf ? gr1 : gr0;
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    bad |= __float_as_uint(fa[i]) != __float_as_uint(fb[i]);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
    bad |= __float_as_uint(ga[j]) != __float_as_uint(gb[j]);
  if (blockIdx.x == 0 && threadIdx.x == 0)
    bad |= (s0->status != sr->status) | (s0->iters != sr->iters) | (s0->ntrace != sr->ntrace) |
           (__float_as_uint(s0->err) != __float_as_uint(sr->err)) |
           (__float_as_uint(s0->cost) != __float_as_uint(sr->cost));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(mismatch, 1);
}

// One rank's device state: pointers into its workspace and its slabs.
struct Rank {
  int r = 0;
  char* base = nullptr;
  float4 *X4, *Y4;
  double* ctr;
  float *F[2], *G[2];
  float *fsel, *gsel;  // the returned iterate
  void *part, *slots;
  int *rowflag, *nflag;
  float *errrow, *errblk;
  int *bad, *badslots;
  float *costrow, *costblk;
  lsk::PtsState* S;
  int* act;
  int* kk;        // graph replay: the iterate the next check decides on
  int rlo, rhi;   // f rows (source points)
  int glo, ghi;   // g rows (target points) this rank finishes
  int leaf_lo;    // partials: first source chunk it reduces
};

void carve(Rank& R, char* ws, const PtsLayout& L) {
  R.base = ws;
  R.X4 = reinterpret_cast<float4*>(ws + L.x4);
  R.Y4 = reinterpret_cast<float4*>(ws + L.y4);
  R.ctr = reinterpret_cast<double*>(ws + L.ctr);
  R.F[0] = reinterpret_cast<float*>(ws + L.f0);
  R.F[1] = reinterpret_cast<float*>(ws + L.f1);
  R.G[0] = reinterpret_cast<float*>(ws + L.g0);
  R.G[1] = reinterpret_cast<float*>(ws + L.g1);
  R.fsel = reinterpret_cast<float*>(ws + L.fsel);
  R.gsel = reinterpret_cast<float*>(ws + L.gsel);
  R.part = ws + L.part;
  R.slots = ws + L.slots;
  R.rowflag = reinterpret_cast<int*>(ws + L.rowflag);
  R.nflag = reinterpret_cast<int*>(ws + L.nflag);
  R.errrow = reinterpret_cast<float*>(ws + L.errrow);
  R.errblk = reinterpret_cast<float*>(ws + L.errblk);
  R.bad = reinterpret_cast<int*>(ws + L.bad);
  R.badslots = reinterpret_cast<int*>(ws + L.badslots);
  R.costrow = reinterpret_cast<float*>(ws + L.costrow);
  R.costblk = reinterpret_cast<float*>(ws + L.costblk);
  R.S = reinterpret_cast<lsk::PtsState*>(ws + L.state);
  R.act = reinterpret_cast<int*>(ws + L.act);
  R.kk = reinterpret_cast<int*>(ws + L.kk);
}

__global__ void k_add_int(int* p, int v) { *p += v; }

// The stream captures are recorded on: the caller's stream may be the legacy
// default stream, which cannot be captured (the graph is launched on it).
// One non-blocking stream per host thread and device, kept for the process.
struct CaptureStream {
  cudaStream_t s = nullptr;
  int device = -1;
};
inline thread_local CaptureStream t_cap;
int32_t capture_stream(cudaStream_t& out) {
  int dev = 0;
  S_CUDA(cudaGetDevice(&dev));
  if (t_cap.s == nullptr || t_cap.device != dev) {
    S_CUDA(cudaStreamCreateWithFlags(&t_cap.s, cudaStreamNonBlocking));
    t_cap.device = dev;
  }
  out = t_cap.s;
  return LSK_OK;
}
__global__ void k_set_int(int* p, int v) { *p = v; }

// The collectives of the decomposition. Every exchanged buffer sits at the
// same workspace offset on every rank, rank r's contribution at
// [off + r bpr, off + (r+1) bpr); after gather() every rank holds all P.
struct Exchange {
  int P = 1;
  ncclComm_t nc = nullptr;   // real: this process's communicator (one local rank)
  std::vector<Rank>* ranks;  // local ranks (real: 1; emulated: P)
  cudaStream_t s;

  int32_t gather(size_t off_from_base, size_t bpr) {
    if (P == 1) return LSK_OK;
    if (nc) {
      Rank& R = (*ranks)[0];
      char* buf = R.base + off_from_base;
      S_NCCL(ncclAllGather(buf + size_t(R.r) * bpr, buf, bpr / 4, ncclFloat, nc, s));
      return LSK_OK;
    }
    for (Rank& D : *ranks)
      for (Rank& Sr : *ranks) {
        if (D.r == Sr.r) continue;
        S_CUDA(cudaMemcpyAsync(D.base + off_from_base + size_t(Sr.r) * bpr, Sr.base + off_from_base + size_t(Sr.r) * bpr,
                               bpr, cudaMemcpyDeviceToDevice, s));
      }
    return LSK_OK;
  }
  int32_t allreduce_sum(size_t off_from_base, size_t count) {
    if (P == 1) return LSK_OK;
    if (nc) {
      float* buf = reinterpret_cast<float*>((*ranks)[0].base + off_from_base);
      S_NCCL(ncclAllReduce(buf, buf, count, ncclFloat, ncclSum, nc, s));
      return LSK_OK;
    }
    RankPtrs rp{};
    for (Rank& R : *ranks) rp.p[R.r] = reinterpret_cast<float*>(R.base + off_from_base);
    k_sum_ranks<<<148, 256, 0, s>>>(P, rp, count);
    S_CUDA(cudaGetLastError());
    for (Rank& D : *ranks)
      if (D.r != 0) S_CUDA(cudaMemcpyAsync(rp.p[D.r], rp.p[0], count * 4, cudaMemcpyDeviceToDevice, s));
    return LSK_OK;
  }
};

struct SolveArgs {
  const double *X, *Y;
  int B, n, m, d;
  const float *scale, *log_mu, *log_nu, *mu;
  double eps, tol;
  int max_iter, check;
  int flags;
  float *f_out, *g_out;
  int32_t* trace_iter;
  float* trace_err;
  int32_t* result;
  float* result_f;
};

// The solve for the local ranks of a decomposition (one real rank under NCCL,
// or P emulated ranks). Outputs are written from local rank 0.
int32_t run_solve(const SolveArgs& a, const Shard& sh, std::vector<Rank>& ranks, Exchange& X, cudaStream_t st,
                  int* mismatch) {
  const int B = a.B, n = a.n, m = a.m;
  const PtsLayout L = pts_layout(B, n, m, sh);
  const EpsC ec = epsc(a.eps);
  const int cap = lsk_trace_capacity(a.max_iter, a.check);
  const bool stale = (a.flags & LSK_FLAG_STALE_SHIFT) != 0;
  const bool expansion = (a.flags & LSK_FLAG_EXPANSION) != 0 && a.eps >= 5e-3;
  const bool partials = sh.mode == LSK_SHARD_PARTIALS || sh.mode == LSK_SHARD_ALLREDUCE;
  const int ych = chunks_of(m);
  const int nb = (n + lsk::kPtsBlk - 1) / lsk::kPtsBlk;

  for (Rank& R : ranks) {
    R.rlo = int(std::min<long long>(n, (long long)R.r * sh.rpr));
    R.rhi = int(std::min<long long>(n, (long long)(R.r + 1) * sh.rpr));
    if (sh.mode == LSK_SHARD_OWNER) {
      R.glo = int(std::min<long long>(m, (long long)R.r * sh.cpr));
      R.ghi = int(std::min<long long>(m, (long long)(R.r + 1) * sh.cpr));
    } else {
      R.glo = 0;
      R.ghi = m;
    }
    R.leaf_lo = R.r * sh.spr;
    // potentials, flags, padded exchange slabs: all defined before any exchange
    S_CUDA(cudaMemsetAsync(R.base + L.f0, 0, L.part - L.f0, st));
    S_CUDA(cudaMemsetAsync(R.base + L.slots, 0, L.total - L.slots, st));
    lsk::k_pts_center<<<B, 256, 0, st>>>(a.X, a.Y, n, m, a.d, R.ctr);
    lsk::k_pts_pack<<<256, 256, 0, st>>>(a.X, (long long)B * n, n, a.d, R.ctr, R.X4);
    lsk::k_pts_pack<<<256, 256, 0, st>>>(a.Y, (long long)B * m, m, a.d, R.ctr, R.Y4);
    k_pts_init<<<(B + 127) / 128, 128, 0, st>>>(B, R.S);
    k_active_view<<<(B + 127) / 128, 128, 0, st>>>(B, R.S, R.act);
    S_CUDA(cudaGetLastError());
  }

  // ---- kernel launchers (rank-local)
  // partial sweep: rows [lo, hi) of (rpts, rpot_old) against column chunks
  // [ch_lo, ch_lo + nch) of (cpts, cpot, clw)
  struct Half {
    const float4* rpts;
    const float4* cpts;
    int nr, nc;
    const float* rpot_old;
    float* rpot_new;
    const float* cpot;
    const float* clw;
  };
  auto run_part = [&](Rank& R, int mode, const Half& h, int lo, int hi, int ch_lo, int nch, const float* rlw,
                      const int* act) -> int32_t {
    if (hi <= lo || nch <= 0) return LSK_OK;
    lsk::PtsHalf ph{};
    ph.B = B; ph.n_rows = h.nr; ph.n_cols = h.nc; ph.row_lo = lo; ph.row_hi = hi;
    ph.chunks = chunks_of(h.nc); ph.ch_lo = ch_lo;
    ph.rpts = h.rpts; ph.cpts = h.cpts; ph.rpot = h.rpot_old; ph.cpot = h.cpot; ph.clw = h.clw; ph.rlw = rlw;
    ph.scale = a.scale; ph.inv_eps = ec.inv; ph.part = R.part; ph.active = act;
    constexpr int kWide = 8;  // 16 rows per warp measured 7% slower (register pressure, 2 CTAs/SM)
    const int tile_rows = (mode == lsk::kPtsOnline) ? lsk::kPtsTileRows : 8 * kWide;
    const dim3 grid(nch, (hi - lo + tile_rows - 1) / tile_rows, B);
    if (mode == lsk::kPtsStale) lsk::k_pts_part<lsk::kPtsStale, kWide><<<grid, lsk::kPtsThreads, 0, st>>>(ph);
    else if (mode == lsk::kPtsStaleX) lsk::k_pts_part<lsk::kPtsStaleX, kWide><<<grid, lsk::kPtsThreads, 0, st>>>(ph);
    else if (mode == lsk::kPtsOnline) lsk::k_pts_part<lsk::kPtsOnline, 8><<<grid, lsk::kPtsThreads, 0, st>>>(ph);
    else lsk::k_pts_part<lsk::kPtsCost, kWide><<<grid, lsk::kPtsThreads, 0, st>>>(ph);
    S_CUDA(cudaGetLastError());
    return LSK_OK;
  };
  // finish rows [lo, hi) from partials `part` (leaves [0, nleaves), `chunks` real)
  auto run_combine = [&](Rank& R, bool use_stale, const Half& h, int lo, int hi, const void* part, int chunks,
                         int nleaves, bool check, const float* rlw, const float* rmu) -> int32_t {
    if (hi <= lo) return LSK_OK;
    lsk::PtsCombine cb{};
    cb.B = B; cb.n_rows = h.nr; cb.row_lo = lo; cb.row_hi = hi; cb.chunks = chunks; cb.nleaves = nleaves;
    cb.part = part; cb.rpot_old = h.rpot_old; cb.rpot_new = h.rpot_new; cb.inv_eps = ec.inv; cb.neg_eps = ec.neg;
    cb.active = R.act;
    const dim3 g((hi - lo + 255) / 256, B);
    if (use_stale) {
      cb.rowflag = R.rowflag; cb.nflag = R.nflag; cb.rlw = rlw; cb.rmu = rmu; cb.cpot = h.cpot;
      cb.errrow = R.errrow; cb.badrow = R.bad; cb.check = check;
      lsk::k_pts_combine<lsk::kPtsStale><<<g, 256, 0, st>>>(cb);
    } else {
      lsk::k_pts_combine<lsk::kPtsOnline><<<g, 256, 0, st>>>(cb);
    }
    S_CUDA(cudaGetLastError());
    return LSK_OK;
  };
  // stale guard: rows whose sum left [1e-20, 1e30] recomputed exactly (one CTA per problem)
  auto run_fixup = [&](Rank& R, const Half& h, int lo, int hi, const float* clw_full) -> int32_t {
    if (hi <= lo) return LSK_OK;
    lsk::PtsHalf ph{};
    ph.B = B; ph.n_rows = h.nr; ph.n_cols = h.nc; ph.row_lo = lo; ph.row_hi = hi;
    ph.rpts = h.rpts; ph.cpts = h.cpts; ph.cpot = h.cpot; ph.clw = clw_full; ph.scale = a.scale;
    ph.inv_eps = ec.inv; ph.active = R.act;
    lsk::k_pts_fixup<<<B, 256, 0, st>>>(ph, ec.neg, h.rpot_new, R.rowflag, R.nflag);
    S_CUDA(cudaGetLastError());
    S_CUDA(cudaMemsetAsync(R.nflag, 0, 4, st));
    return LSK_OK;
  };
  // a complete half-step of rows [lo, hi) against every column chunk
  auto half_full = [&](Rank& R, const Half& h, int lo, int hi, bool use_stale, bool check, const float* rlw,
                       const float* rmu) -> int32_t {
    const int nch = chunks_of(h.nc);
    const int mode = use_stale ? (expansion ? lsk::kPtsStaleX : lsk::kPtsStale) : lsk::kPtsOnline;
    S_TRY(run_part(R, mode, h, lo, hi, 0, nch, nullptr, R.act));
    S_TRY(run_combine(R, use_stale, h, lo, hi, R.part, nch, lsk::pow2_ceil(nch), check, rlw, rmu));
    if (use_stale && h.rpot_new) S_TRY(run_fixup(R, h, lo, hi, h.clw));
    return LSK_OK;
  };
  auto pot_off = [&](float* p, const Rank& R) { return size_t(reinterpret_cast<char*>(p) - R.base); };

  // check decision for iterate kk from the f-half's row terms
  bool dev_kk = false;  // inside a captured block: the checked iterate comes from R.kk
  auto decide = [&](int kk, int gbuf, bool final) -> int32_t {
    for (Rank& R : ranks) {
      lsk::k_pts_colcheck<<<dim3(8, B), 256, 0, st>>>(B, m, R.G[gbuf], R.act, R.bad);
      S_CUDA(cudaGetLastError());
    }
    if (sh.P > 1) {
      Rank& R0 = ranks[0];
      S_TRY(X.gather(pot_off(R0.errrow, R0), size_t(sh.rpr) * 4));
      for (Rank& R : ranks) k_put_slot<<<1, 1, 0, st>>>(R.bad, R.badslots, R.r);
      S_TRY(X.gather(size_t(reinterpret_cast<char*>(R0.badslots) - R0.base), 4));
      for (Rank& R : ranks) k_or_slots<<<1, 1, 0, st>>>(sh.P, R.badslots, R.bad);
      S_CUDA(cudaGetLastError());
    }
    for (Rank& R : ranks) {
      lsk::k_pts_blocksum<<<dim3(nb, B), 1024, 0, st>>>(B, n, 0, n, R.errrow, R.act, R.errblk);
      lsk::k_pts_decide<<<(B + 127) / 128, 128, 0, st>>>(B, n, R.errblk, R.bad, a.tol, kk, final ? 1 : 0, R.S,
                                                          a.trace_iter, a.trace_err, cap, dev_kk ? R.kk : nullptr);
      k_active_view<<<(B + 127) / 128, 128, 0, st>>>(B, R.S, R.act);
      S_CUDA(cudaGetLastError());
    }
    return LSK_OK;
  };

  // one iteration k (everything but the host poll)
  auto iterate = [&](int k) -> int32_t {
    const bool do_check = (k > 1) && ((k - 1) % a.check == 0);
    const int pb = (k - 1) & 1, nbuf = k & 1;
    const bool st_k = stale && k > 1;
    // ---- f half-step (rank-local rows)
    for (Rank& R : ranks) {
      if (do_check && !st_k) {  // exact variant: a separate check pass of iterate k-1
        Half hc{R.X4, R.Y4, n, m, R.F[pb], nullptr, R.G[pb], a.log_nu};
        S_TRY(half_full(R, hc, R.rlo, R.rhi, true, true, a.log_mu, a.mu));
      }
      Half hf{R.X4, R.Y4, n, m, R.F[pb], R.F[nbuf], R.G[pb], a.log_nu};
      S_TRY(half_full(R, hf, R.rlo, R.rhi, st_k, do_check && st_k, a.log_mu, a.mu));
    }
    S_TRY(X.gather(pot_off(ranks[0].F[nbuf], ranks[0]), size_t(sh.rpr) * 4));
    if (do_check) S_TRY(decide(k - 1, pb, false));
    // ---- g half-step
    if (!partials) {
      for (Rank& R : ranks) {
        Half hg{R.Y4, R.X4, m, n, R.G[pb], R.G[nbuf], R.F[nbuf], a.log_mu};
        S_TRY(half_full(R, hg, R.glo, R.ghi, st_k, false, nullptr, nullptr));
      }
      S_TRY(X.gather(pot_off(ranks[0].G[nbuf], ranks[0]), size_t(sh.cpr) * 4));
    } else {
      const int mode = st_k ? (expansion ? lsk::kPtsStaleX : lsk::kPtsStale) : lsk::kPtsOnline;
      const bool ar = st_k && sh.mode == LSK_SHARD_ALLREDUCE;
      const size_t esz = st_k ? 4 : 8;
      for (Rank& R : ranks) {
        Half hg{R.Y4, R.X4, m, n, R.G[pb], R.G[nbuf], R.F[nbuf], a.log_mu};
        const int nch = std::max(0, std::min(sh.xch, R.leaf_lo + sh.spr) - R.leaf_lo);
        S_TRY(run_part(R, mode, hg, 0, m, R.leaf_lo, nch, nullptr, R.act));
        char* slot = static_cast<char*>(R.slots) + (ar ? 0 : size_t(R.r) * m * esz);
        const dim3 g((m + 255) / 256);
        if (st_k)
          lsk::k_pts_subtree<lsk::kPtsStale><<<g, 256, 0, st>>>(m, 0, m, sh.xch, R.leaf_lo, sh.spr, R.part, slot,
                                                               R.act, nullptr);
        else
          lsk::k_pts_subtree<lsk::kPtsOnline><<<g, 256, 0, st>>>(m, 0, m, sh.xch, R.leaf_lo, sh.spr, R.part, slot,
                                                                R.act, nullptr);
        S_CUDA(cudaGetLastError());
      }
      const size_t soff = size_t(static_cast<char*>(ranks[0].slots) - ranks[0].base);
      if (ar) S_TRY(X.allreduce_sum(soff, size_t(m)));
      else S_TRY(X.gather(soff, size_t(m) * esz));
      for (Rank& R : ranks) {
        Half hg{R.Y4, R.X4, m, n, R.G[pb], R.G[nbuf], R.F[nbuf], a.log_mu};
        const int slots = ar ? 1 : sh.P;
        S_TRY(run_combine(R, st_k, hg, 0, m, R.slots, slots, slots, false, nullptr, nullptr));
        if (st_k) S_TRY(run_fixup(R, hg, 0, m, a.log_mu));
      }
    }
    return LSK_OK;
  };

  lsk_poll::StopPoll poll;
  S_TRY(poll.init(B, st));
  const int c = a.check;
  // graph blocks start at the first checkpoint iteration c + 1 and repeat every c
  const int first_blk = c + 1;
  const int nblk = a.max_iter >= first_blk ? (a.max_iter - first_blk + 1) / c : 0;
  bool graphs = !(a.flags & LSK_FLAG_NO_GRAPH) && (X.nc == nullptr || (a.flags & LSK_FLAG_GRAPH_NCCL)) && nblk >= 3;
  if (graphs) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    S_CUDA(cudaStreamIsCapturing(st, &cs));
    graphs = cs == cudaStreamCaptureStatusNone;  // a caller's capture already owns the stream
  }
  const int graph_end = graphs ? first_blk + nblk * c : 1;  // iterations [first_blk, graph_end) replayed
  bool stopped = false;
  for (int k = 1; k <= a.max_iter && !stopped; ++k) {
    if (graphs && k == first_blk) break;
    S_TRY(iterate(k));
    if ((k > 1) && ((k - 1) % c == 0)) {
      bool stop = false;
      S_TRY(poll.after_check(ranks[0].act, st, stop));
      if (stop) stopped = true;
    }
  }
  if (graphs && !stopped) {
    cudaGraphExec_t ge[2] = {nullptr, nullptr};
    auto destroy = [&]() {
      for (auto& e : ge)
        if (e) cudaGraphExecDestroy(e);
    };
    // capture block b's shape: iterations first_blk + b c ... + c - 1
    // every launcher above enqueues on `st` / X.s: point them at the capture stream
    // while recording, back at the caller's stream for the replays
    auto capture = [&](int b, cudaGraphExec_t* out) -> int32_t {
      const int k0 = first_blk + b * c;
      cudaGraph_t g = nullptr;
      cudaStream_t cap = nullptr;
      S_TRY(capture_stream(cap));
      const cudaStream_t main_st = st;
      S_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed));
      st = cap;
      X.s = cap;
      int32_t rc = LSK_OK;
      dev_kk = true;
      for (Rank& R : ranks) k_add_int<<<1, 1, 0, st>>>(R.kk, c);
      for (int k = k0; k < k0 + c && rc == LSK_OK; ++k) rc = iterate(k);
      dev_kk = false;
      st = main_st;
      X.s = main_st;
      const cudaError_t ec = cudaStreamEndCapture(cap, &g);
      if (rc != LSK_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      S_CUDA(ec);
      const cudaError_t ei = cudaGraphInstantiate(out, g, 0);
      cudaGraphDestroy(g);
      S_CUDA(ei);
      return LSK_OK;
    };
    int32_t rc = LSK_OK;
    for (Rank& R : ranks) k_set_int<<<1, 1, 0, st>>>(R.kk, first_blk - 1 - c);
    const int nshape = (c & 1) ? 2 : 1;
    for (int q = 0; q < nshape && rc == LSK_OK; ++q) rc = capture(q, &ge[q]);
    int resume = graph_end;  // first iteration the eager loop below enqueues
    if (rc != LSK_OK) {
      // the capture itself failed (nothing of the block was enqueued): clear the
      // sticky-free launch error and enqueue the blocks instead; a real launch
      // problem resurfaces there
      (void)cudaGetLastError();
      rc = LSK_OK;
      resume = first_blk;
    } else {
      for (int b = 0; b < nblk && rc == LSK_OK && !stopped; ++b) {
        const cudaError_t e = cudaGraphLaunch(ge[b % nshape], st);
        if (e != cudaSuccess) rc = sfail(LSK_ECUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
        bool stop = false;
        if (rc == LSK_OK) rc = poll.after_check(ranks[0].act, st, stop);
        stopped = stop;
      }
    }
    destroy();
    S_TRY(rc);
    if (resume == first_blk)  // eager fallback: the checkpoint counter is not used
      for (Rank& R : ranks) k_set_int<<<1, 1, 0, st>>>(R.kk, 0);
    for (int k = resume; k <= a.max_iter && !stopped; ++k) {
      S_TRY(iterate(k));
      if ((k - 1) % c == 0) {
        bool stop = false;
        S_TRY(poll.after_check(ranks[0].act, st, stop));
        if (stop) stopped = true;
      }
    }
  }
  // the final check at the cap (solver.py:286-316): a check-only f pass of iterate K
  {
    const int K = a.max_iter, kb = K & 1;
    for (Rank& R : ranks) {
      Half hc{R.X4, R.Y4, n, m, R.F[kb], nullptr, R.G[kb], a.log_nu};
      S_TRY(half_full(R, hc, R.rlo, R.rhi, true, true, a.log_mu, a.mu));
    }
    S_TRY(decide(K, kb, true));
  }
  // potentials of the returned iterate (every rank selects its own copy), then
  // the transport cost from them: per-row sums over the rank's rows, gathered,
  // fixed 1024-row blocks
  Rank& R0 = ranks[0];
  for (Rank& R : ranks) {
    lsk::k_pts_pick<<<dim3(64, B), 256, 0, st>>>(B, n, R.F[0], R.F[1], R.S, R.fsel);
    lsk::k_pts_pick<<<dim3(64, B), 256, 0, st>>>(B, m, R.G[0], R.G[1], R.S, R.gsel);
    S_CUDA(cudaGetLastError());
  }
  S_CUDA(cudaMemcpyAsync(a.f_out, R0.fsel, size_t(B) * n * 4, cudaMemcpyDeviceToDevice, st));
  S_CUDA(cudaMemcpyAsync(a.g_out, R0.gsel, size_t(B) * m * 4, cudaMemcpyDeviceToDevice, st));
  if (a.flags & LSK_FLAG_COST) {
    for (Rank& R : ranks) {
      Half hk{R.X4, R.Y4, n, m, R.fsel, nullptr, R.gsel, a.log_nu};
      S_TRY(run_part(R, lsk::kPtsCost, hk, R.rlo, R.rhi, 0, ych, a.log_mu, nullptr));
      if (R.rhi > R.rlo) {
        k_pts_rowsum<<<dim3((R.rhi - R.rlo + 255) / 256, B), 256, 0, st>>>(
            B, n, R.rlo, R.rhi, ych, reinterpret_cast<const float*>(R.part), R.costrow);
        S_CUDA(cudaGetLastError());
      }
    }
    if (sh.P > 1) S_TRY(X.gather(pot_off(R0.costrow, R0), size_t(sh.rpr) * 4));
    for (Rank& R : ranks) {
      lsk::k_pts_blocksum<<<dim3(nb, B), 1024, 0, st>>>(B, n, 0, n, R.costrow, nullptr, R.costblk);
      lsk::k_pts_cost_finish<<<(B + 127) / 128, 128, 0, st>>>(B, n, R.costblk, R.S);
      S_CUDA(cudaGetLastError());
    }
  }
  k_pts_results<<<(B + 127) / 128, 128, 0, st>>>(B, R0.S, a.result, a.result_f, (a.flags & LSK_FLAG_COST) ? 1 : 0);
  S_CUDA(cudaGetLastError());
  if (mismatch) {
    S_CUDA(cudaMemsetAsync(mismatch, 0, 4, st));
    for (size_t i = 1; i < ranks.size(); ++i) {
      Rank& R = ranks[i];
      k_cmp_rank<<<64, 256, 0, st>>>(n, m, R0.S, R0.F[0], R0.F[1], R0.G[0], R0.G[1], R.S, R.F[0], R.F[1], R.G[0],
                                     R.G[1], mismatch);
    }
    S_CUDA(cudaGetLastError());
  }
  return LSK_OK;
}

int32_t check_args(const SolveArgs& a) {
  if (!a.X || !a.Y || !a.scale || !a.log_mu || !a.log_nu || !a.mu || !a.f_out || !a.g_out || !a.trace_iter ||
      !a.trace_err || !a.result || !a.result_f)
    return sfail(LSK_EINVAL, "null pointer");
  if (a.B < 1 || a.n < 1 || a.m < 1) return sfail(LSK_EINVAL, "B, n, m must be >= 1");
  if (a.d < 1 || a.d > 3) return sfail(LSK_EUNSUPPORTED, "points solver supports d in 1..3");
  if (!(a.eps > 0) || !(a.tol > 0) || a.max_iter < 1 || a.check < 1)
    return sfail(LSK_EINVAL, "eps, tol > 0; max_iter, check_interval >= 1 required");
  return LSK_OK;
}

int shard_mode_of(int flags) {
  if (flags & LSK_FLAG_SHARD_ALLREDUCE) return LSK_SHARD_ALLREDUCE;
  if (flags & LSK_FLAG_SHARD_PARTIALS) return LSK_SHARD_PARTIALS;
  return LSK_SHARD_OWNER;
}

}  // namespace

extern "C" {

size_t lsk_solve_points_workspace_bytes(int32_t B, int32_t n, int32_t m) {
  if (B < 1 || n < 1 || m < 1) return 0;
  Shard s;
  if (make_shard(n, m, 1, LSK_SHARD_NONE, s) != LSK_OK) return 0;
  return pts_layout(B, n, m, s).total;
}

size_t lsk_solve_points_sharded_workspace_bytes(int32_t n, int32_t m, int32_t P, int32_t shard_mode) {
  if (n < 1 || m < 1 || P < 1) return 0;
  Shard s;
  if (make_shard(n, m, P, shard_mode, s) != LSK_OK) return 0;
  return pts_layout(1, n, m, s).total;
}

int32_t lsk_solve_points_f32(const double* X, const double* Y, int32_t B, int32_t n, int32_t m, int32_t d,
                             const float* scale, const float* log_mu, const float* log_nu, const float* mu,
                             double eps, double tol, int32_t max_iter, int32_t check_interval, int32_t flags,
                             float* f_out, float* g_out, int32_t* trace_iter, float* trace_err, int32_t* result,
                             float* result_f, void* workspace, size_t workspace_bytes, void* comm, void* stream) {
  const SolveArgs a{X, Y, B, n, m, d, scale, log_mu, log_nu, mu, eps, tol, max_iter, check_interval, flags,
                    f_out, g_out, trace_iter, trace_err, result, result_f};
  S_TRY(check_args(a));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ncclComm_t nc = static_cast<ncclComm_t>(comm);
  int P = 1, rank = 0, mode = LSK_SHARD_NONE;
  if (nc) {
    S_NCCL(ncclCommCount(nc, &P));
    S_NCCL(ncclCommUserRank(nc, &rank));
    if (B != 1) return sfail(LSK_EUNSUPPORTED, "sharded points solve: one problem per call (split batches instead)");
    mode = shard_mode_of(flags);
  }
  Shard sh;
  S_TRY(make_shard(n, m, P, mode, sh));
  const PtsLayout L = pts_layout(B, n, m, sh);
  if (!workspace || workspace_bytes < L.total) return sfail(LSK_EINVAL, "workspace too small");
  std::vector<Rank> ranks(1);
  ranks[0].r = rank;
  carve(ranks[0], static_cast<char*>(workspace), L);
  Exchange ex;
  ex.P = P; ex.nc = nc; ex.ranks = &ranks; ex.s = st;
  return run_solve(a, sh, ranks, ex, st, nullptr);
}

int32_t lsk_solve_points_emulated_f32(const double* X, const double* Y, int32_t n, int32_t m, int32_t d,
                                      const float* scale, const float* log_mu, const float* log_nu, const float* mu,
                                      double eps, double tol, int32_t max_iter, int32_t check_interval, int32_t flags,
                                      int32_t P, int32_t shard_mode, float* f_out, float* g_out, int32_t* trace_iter,
                                      float* trace_err, int32_t* result, float* result_f, int32_t* rank_mismatch,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  const SolveArgs a{X, Y, 1, n, m, d, scale, log_mu, log_nu, mu, eps, tol, max_iter, check_interval, flags,
                    f_out, g_out, trace_iter, trace_err, result, result_f};
  S_TRY(check_args(a));
  if (!rank_mismatch) return sfail(LSK_EINVAL, "null pointer");
  if (P < 1 || P > LSK_EMU_MAX_RANKS) return sfail(LSK_EINVAL, "emulated rank count must be in 1..LSK_EMU_MAX_RANKS");
  if (shard_mode == LSK_SHARD_NONE && P != 1) return sfail(LSK_EINVAL, "LSK_SHARD_NONE needs P == 1");
  Shard sh;
  S_TRY(make_shard(n, m, P, shard_mode, sh));
  const PtsLayout L = pts_layout(1, n, m, sh);
  if (!workspace || workspace_bytes < size_t(P) * L.total) return sfail(LSK_EINVAL, "workspace too small");
  std::vector<Rank> ranks(P);
  for (int r = 0; r < P; ++r) {
    ranks[r].r = r;
    carve(ranks[r], static_cast<char*>(workspace) + size_t(r) * L.total, L);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Exchange ex;
  ex.P = P; ex.nc = nullptr; ex.ranks = &ranks; ex.s = st;
  return run_solve(a, sh, ranks, ex, st, rank_mismatch);
}

}  // extern "C"

// Single-cluster persistent solver for small dense problems (config C1:
// n=m=1024, C = 4 MB, L2-resident): ONE thread-block cluster of CL CTAs
// (16, the non-portable maximum; 8 where 16 cannot be scheduled) runs the
// whole solve. Every CTA-to-CTA exchange goes through distributed shared
// memory and barrier.cluster -- no global grid barrier, no cooperative launch.
//
// Reference path replaced: logsinkhorn.solver.solve (solver.py:230-337) with
// _alpha_step / _beta_step_* / _marginal_error / _transport_cost
// (solver.py:76-115) over reduction.py:179-224 -- the same fp32 arithmetic
// contract as DenseSolver (lsk_dense.cuh, SURVEY 8(a')); uniform target
// weights (the C1 config), m <= 1024.
//
// Why (profiles/r1_dense_experiments.md): with 148 CTAs of
// ~7 rows each, C1 spent ~7 of its 8.9 us per iteration in two global atomic
// grid barriers and the 148-way column combine. Here:
//  * WARP PER ROW. Lane l owns the 32 columns 4 (32 v + l) + q (v < 8, q < 4);
//    a warp streams its rows through its own 4-slot shared-memory ring of
//    cp.async 16-byte copies (each lane copies and later reads only its own
//    columns, so no intra-warp sync; the ring cycles over the warp's rows
//    across passes and iterations, C being constant; a per-warp TMA bulk ring
//    with an mbarrier per slot measured 12% slower), forms the f-side terms,
//    reduces the row sum with one butterfly and finishes f_i -- no cross-warp
//    hand-off per row, so the 8 warps of a CTA run free and de-phase. f,
//    log mu and mu of the CTA's rows live in shared memory.
//  * Column update in registers (the multiplicative update of
//    DenseSolver::fused_pass_mult when its band allows, else the direct
//    reference arithmetic from the row still in registers). lsk_api.cu
//    clears a.mult for the cluster solvers, so only the direct update runs;
//    the multiplicative branch stays compiled in because ptxas schedules the
//    kernel better with it (without it: no spills, but C1 1.183 -> 1.187 ms
//    and n = 4096 1.77 -> 1.82 ms per 200 iterations).
//  * Column combine: warp partials -> CTA partial in smem (fixed order) ->
//    barrier.cluster -> CTA c sums the CL CTA partials of its m/CL columns
//    over DSMEM in rank order, finishes g_j and stores it into every CTA's
//    shared g copy (DSMEM) -> barrier.cluster. Two cluster barriers per
//    iteration; the check's error sum rides on the first.
// MC = true (multi-cluster): NCL clusters of CL CTAs (up to one CTA per SM)
// split the rows, so C1 (n = 1024) gives every warp at most one row. Each
// cluster first combines its CTAs' partials over DSMEM as above; the CTA that
// owns column slice s stores its cluster's slice sums to global memory, ONE
// software grid barrier per iteration, then EVERY cluster sums the NCL
// cluster partials of its slices in cluster order, finishes g and broadcasts
// it into its CTAs' shared copies -- the same bits in every cluster, so the
// guard decision and the stop decision need no further exchange. The global
// slots are double-buffered by iteration parity (every iteration has at least
// one grid barrier, so a slot is rewritten only after every cluster has read
// it). This replaces the 148-CTA DenseSolver's two grid barriers and 148-way
// combine per iteration at m <= 1024 (profiles/r2_c1_cluster.md).
// Stale shifts and guards are those of DenseSolver: a row sum
// outside [1e-20, 1e30] is redone exactly in-warp from the registers; a column
// sum outside the band redoes the iteration's g with the exact online
// (max, sumexp) pass, merged warp -> CTA -> cluster in fixed order.
#pragma once
#include <cooperative_groups.h>

#include "lsk_dense.cuh"

namespace lsk {

template <int CL, bool MC = false>
struct ClusterSolver {
  static constexpr bool kUniform = true;
  static constexpr int NT = 256, NW = NT / 32;
  static constexpr int V = 8, E = 32, P2 = 16;  // float4 chunks / columns / packed pairs per lane
  static constexpr int W = 1024;                // row capacity (floats)
  static constexpr int CPC = W / CL;            // columns combined by each CTA
  static constexpr int R = 4;                   // row-ring slots per warp
  static constexpr int kMaxRows = 2048;         // n supported (rows per CTA <= kMaxRows / CL)
  static constexpr int RPC = kMaxRows / CL;
  // smem (floats): gS[W] | wred[NW][2W] (warp partials; float2 pairs on the exact path) |
  //   cpart[2W] (CTA partial / pairs) | scal[96] | fS[2][RPC] | lmuS[RPC] | muS[RPC] | ring[NW][R][W]
  static constexpr int kOffG = 0, kOffW = W, kOffC = W + NW * 2 * W, kOffS = kOffC + 2 * W;
  static constexpr int kOffF = kOffS + 96, kOffLm = kOffF + 2 * RPC, kOffMu = kOffLm + RPC;
  static constexpr int kOffR = kOffMu + RPC;
  static constexpr size_t kSmemBytes = size_t(kOffR + NW * R * W) * sizeof(float);
  // scal slots
  static constexpr int kSErr = NW, kSBad = NW + 1, kSGuard = NW + 2, kSCost = NW + 3;
  // mailboxes: every CTA stores its scalar into slot [crank] of EVERY CTA's copy
  // (DSMEM stores before the barrier), so the reads after it are local
  static constexpr int kMErr = 16, kMBad = 16 + 16, kMGuard = 16 + 32;
  static_assert(CL <= 16, "mailbox width");
  static constexpr int kMaxClusters = 32;  // MC: cluster partials per column summed with all loads in flight

  const DenseArgs& a;
  cooperative_groups::cluster_group cl;
  float* sm;
  int crank, lane, w, r0, r1;
  int cid, ncl;        // cluster index / count (MC; 0 / 1 otherwise)
  unsigned epoch = 0;  // MC: software grid barrier epochs
  int nexact = 0;      // MC: exact column passes so far (their global slots alternate)
  int nrw;       // rows of this warp: r0 + w + NW q, q < nrw
  int q_iss;     // ring: rows issued (in the warp's cyclic row sequence)
  int q_row;     // ... = q_iss mod nrw, kept incrementally (no integer division per row)
  f2 inv2, l2e2, nz2, lnu2;
  float bcol;
  f2 g2[P2];   // g^{k-1} of the lane's columns
  f2 ac2[P2];  // column accumulators

  __device__ ClusterSolver(const DenseArgs& args, unsigned char* smem)
      : a(args), cl(cooperative_groups::this_cluster()) {
    sm = reinterpret_cast<float*>(smem);
    crank = int(cl.block_rank());
    cid = MC ? int(blockIdx.x) / CL : 0;
    ncl = MC ? int(gridDim.x) / CL : 1;
    lane = threadIdx.x & 31;
    w = threadIdx.x >> 5;
    const int gi = cid * CL + crank, gn = ncl * CL;
    r0 = int((long long)gi * a.n / gn);
    r1 = int((long long)(gi + 1) * a.n / gn);
    nrw = (r1 - r0 - w + NW - 1) / NW;
    if (nrw < 0) nrw = 0;
    q_iss = 0;
    q_row = 0;
    inv2 = pk2(a.inv_eps, a.inv_eps);
    l2e2 = pk2(kLog2e, kLog2e);
    nz2 = pk2(a.negzero, a.negzero);
    const float L = __ldg(a.log_nu);
    lnu2 = pk2(L, L);
    bcol = -__fmul_rn(L, kLog2e);
  }

  __device__ __forceinline__ int col(int v) const { return 4 * (32 * v + lane); }
  __device__ __forceinline__ float* remote(float* p, int r) { return cl.map_shared_rank(p, r); }

  // ---- the warp's row ring: row q of the cyclic sequence r0 + w + NW (q mod nrw)
  __device__ __forceinline__ void issue_row() {
    const int i = r0 + w + NW * q_row;
    const float* base = a.C + (long long)i * a.ldc;
    float* slot = sm + kOffR + (w * R + (unsigned(q_iss) % R)) * W;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int j0 = col(v);
      if (j0 < a.m)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(slot + j0)), "l"(base + j0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    ++q_iss;
    if (++q_row == nrw) q_row = 0;
  }
  __device__ void ring_init() {
    float4* r4 = reinterpret_cast<float4*>(sm + kOffR + w * R * W);  // columns >= m read as 0
    for (int k = lane; k < R * W / 4; k += 32) r4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    if (nrw > 0)
      for (int k = 0; k < R - 1; ++k) issue_row();
  }
  // the next row of the sequence into registers; its slot is refilled R-1 rows ahead
  // (refilling lazily at the next take, so no copy is in flight at a cluster
  // barrier, measured the same: profiles/r2_c1_cluster.md)
  __device__ __forceinline__ void take_row(f2 (&c)[P2]) {
    asm volatile("cp.async.wait_group %0;" ::"n"(R - 2) : "memory");
    const float* slot = sm + kOffR + (w * R + (unsigned(q_iss - (R - 1)) % R)) * W;
#pragma unroll
    for (int v = 0; v < V; ++v) lds2x2(slot + col(v), c[2 * v], c[2 * v + 1]);
    issue_row();
  }

  // g^{k-1} from the CTA's shared copy; true if a loaded g (j < m) is non-finite
  template <bool CHK = true>
  __device__ bool load_columns() {
    bool bad = false;
    const float* gS = sm + kOffG;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float4 t = *reinterpret_cast<const float4*>(gS + col(v));
      const float tt[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (CHK && col(v) + q < a.m) bad |= !isfinite(tt[q]);
      g2[2 * v] = pk2(t.x, t.y);
      g2[2 * v + 1] = pk2(t.z, t.w);
      ac2[2 * v] = 0ull;
      ac2[2 * v + 1] = 0ull;
    }
    return bad;
  }

  // exact two-pass LSE over the row in registers (CHK: the check argument with f_i = fi)
  template <bool CHK>
  __device__ __forceinline__ void exact_lse(const f2 (&c)[P2], float fi, float& M, float& S) const {
    const f2 f2i = pk2(fi, fi);
    float mx = -INFINITY;
#pragma unroll
    for (int p = 0; p < P2; ++p) {
      float x0, x1;
      up2(CHK ? arg4x2(f2i, g2[p], c[p], inv2, lnu2, nz2) : arg3x2(g2[p], c[p], inv2, lnu2, nz2), x0, x1);
      mx = fmax_nan(mx, fmax_nan(x0, x1));
    }
    M = warp_max(mx);
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    const f2 nsl = pk2(-__fmul_rn(Ms, kLog2e), -__fmul_rn(Ms, kLog2e));
    f2 s2 = 0ull;
#pragma unroll
    for (int p = 0; p < P2; ++p) {
      const f2 x = CHK ? arg4x2(f2i, g2[p], c[p], inv2, lnu2, nz2) : arg3x2(g2[p], c[p], inv2, lnu2, nz2);
      s2 = add2(s2, ex2x2(fma2(x, l2e2, nsl)));
    }
    float s0, s1;
    up2(s2, s0, s1);
    S = warp_sum(s0 + s1);
  }
  static __device__ __forceinline__ bool shift_ok(float S) { return S >= kShiftLo && S <= kShiftHi; }

  // ---- the f pass of iteration k over this warp's rows (+ the check of iterate
  // k-1 when CHECK; + the column update when FUSED)
#ifdef LSK_X_TRACE
  int cur_k = 0;
// (the value's MOV waits on its scoreboard; a warp issues in order, so the clock
// read that follows stamps the time the value became available)
#define LSK_RTR(slot, val)                                                                   \
  if (threadIdx.x == 0 && blockIdx.x == 0 && cur_k >= 20 && cur_k < 30 && i == r0) {      \
    float dep_ = (val);                                                                     \
    asm volatile("mov.b32 %0, %0;" : "+f"(dep_));                                           \
    lsk_x_trace[(cur_k - 20) * 4 + (slot)] = clock64() + (dep_ == 1.2345e-30f ? 1 : 0);    \
  }
#else
#define LSK_RTR(slot, val)
#endif
  template <bool FUSED, bool CHECK>
  __device__ void f_pass(const float* fprev, float* fnew, float& err_acc, int& bad) {
    for (int i = r0 + w; i < r1; i += NW) {
      f2 c[P2];
      LSK_RTR(0, 0.f);
      take_row(c);
      LSK_RTR(1, __uint_as_float(unsigned(c[0])));
      const float fold = fprev[i - r0], lmu = sm[kOffLm + i - r0];
      float fi;
      f2 e[P2];
      if (FUSED) {
        // f-side terms with the stale row shift fl(-f^{k-1}_i inv_eps)
        const float shl = __fmul_rn(__fmul_rn(-fold, a.inv_eps), kLog2e);
        const f2 nsl = pk2(-shl, -shl);
        f2 s2a = 0ull, s2b = 0ull;
#pragma unroll
        for (int p = 0; p < P2; ++p) {
          e[p] = ex2x2(fma2(arg3x2(g2[p], c[p], inv2, lnu2, nz2), l2e2, nsl));
          if (p & 1) s2b = add2(s2b, e[p]);
          else s2a = add2(s2a, e[p]);
        }
        float s0, s1;
        up2(add2(s2a, s2b), s0, s1);
        float S = warp_sum(s0 + s1);
        float M = __fmul_rn(-fold, a.inv_eps);
        if (__builtin_expect(!shift_ok(S), 0)) {
          if (lane == 0) atomicAdd(a.stats + 0, 1);
          exact_lse<false>(c, 0.f, M, S);
        }
        fi = __fmul_rn(a.neg_eps, lse_finish(M, S));
        LSK_RTR(2, fi);
      } else {
        float M, S;
        exact_lse<false>(c, 0.f, M, S);
        fi = __fmul_rn(a.neg_eps, lse_finish(M, S));
      }
      if (CHECK) {  // marginal error of iterate k-1 (solver.py:97-104), shift 0
        const f2 fo2 = pk2(fold, fold);
        f2 z2 = 0ull;
#pragma unroll
        for (int p = 0; p < P2; ++p) z2 = add2(z2, ex2x2(mul2(arg4x2(fo2, g2[p], c[p], inv2, lnu2, nz2), l2e2)));
        float z0, z1;
        up2(z2, z0, z1);
        float Sz = warp_sum(z0 + z1), Mz = 0.f;
        if (__builtin_expect(!shift_ok(Sz), 0)) exact_lse<true>(c, fold, Mz, Sz);
        if (lane == 0) {
          const float rr = expf(__fadd_rn(lmu, lse_finish(Mz, Sz)));
          err_acc += fabsf(__fsub_rn(rr, sm[kOffMu + i - r0]));
          if (!isfinite(fold)) bad = 1;
        }
      }
      if (lane == 0) fnew[i - r0] = fi;
      if (FUSED) {
        const float ai = __fmul_rn(__fadd_rn(__fmul_rn(__fsub_rn(fi, fold), a.inv_eps), lmu), kLog2e);
        if (a.mult && ai >= -100.f && ai + bcol <= 23.f) {
          const f2 A2 = pk2(ex2(ai + bcol), ex2(ai + bcol));
#pragma unroll
          for (int p = 0; p < P2; ++p) ac2[p] = fma2(e[p], A2, ac2[p]);
        } else {  // direct: the beta argument against the stale column shift fl(-g_j inv_eps)
          const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
#pragma unroll
          for (int p = 0; p < P2; ++p)
            ac2[p] = add2(ac2[p], ex2x2(fma2(arg3x2(fi2, c[p], inv2, lm2, nz2), l2e2,
                                             mul2(mul2(g2[p], inv2), l2e2))));
        }
      }
      LSK_RTR(3, __uint_as_float(unsigned(ac2[P2 - 1])));
    }
  }

  // ---- warp partials -> CTA partial cpart[W] (fixed warp order)
  __device__ void cta_partial() {
    float* wr = sm + kOffW + w * 2 * W;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float x0, x1, x2, x3;
      up2(ac2[2 * v], x0, x1);
      up2(ac2[2 * v + 1], x2, x3);
      *reinterpret_cast<float4*>(wr + col(v)) = make_float4(x0, x1, x2, x3);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < W; j += NT) {
      float s = 0.f;
#pragma unroll
      for (int u = 0; u < NW; ++u) s += sm[kOffW + u * 2 * W + j];
      sm[kOffC + j] = s;
    }
  }
  // CTA's err / bad into scal (fixed warp order)
  __device__ void cta_check(float err_acc, int bad) {
    if (lane == 0) sm[kOffS + w] = err_acc;
    bad = __syncthreads_or(bad);  // CTA-uniform in every thread
    if (w == 0) {
      float e = 0.f;
      for (int u = 0; u < NW; ++u) e += sm[kOffS + u];
      if (lane < CL) {
        float* rs = remote(sm + kOffS, lane);
        rs[kMErr + crank] = e;
        rs[kMBad + crank] = bad ? 1.f : 0.f;
      }
    }
  }
  // after a cluster barrier: the cluster's err (rank order) and bad, identical in every CTA
  __device__ void cluster_err(float& err, int& bad) const {
    // lane r reads rank r's scalars (all in flight at once); the butterfly sum
    // has the same bits in every lane, warp and CTA
    float er = 0.f;
    int bd = 0;
    if (lane < CL) {
      er = sm[kOffS + kMErr + lane];
      bd = sm[kOffS + kMBad + lane] != 0.f;
    }
    err = warp_sum(er);
    bad = __any_sync(0xffffffffu, bd);
  }
  __device__ bool decide(int kk, bool& failed) {
    float err;
    int bad;
    if constexpr (MC) {
      // the NCL cluster errors (published before the grid barrier, slot kk + 1 parity), cluster order
      const int sl = ((kk + 1) & 1) * ncl;
      float er = 0.f;
      int bd = 0;
      if (lane < ncl) {
        er = ldcg(a.errpart + sl + lane);
        bd = __ldcg(a.flagpart + sl + lane);
      }
      err = warp_sum(er);
      bad = __any_sync(0xffffffffu, bd != 0);
    } else {
      cluster_err(err, bad);
    }
    return decide_from(err, bad, kk, failed);
  }
  // MC, after the cluster barrier: the cluster's check scalars to global slot (k & 1)
  __device__ void publish_cluster_err(int k) {
    if (crank == 0 && w == 0) {
      float err;
      int bad;
      cluster_err(err, bad);
      if (lane == 0) {
        a.errpart[(k & 1) * ncl + cid] = err;
        a.flagpart[(k & 1) * ncl + cid] = bad;
      }
    }
  }
  __device__ bool decide_from(float err, int bad, int kk, bool& failed) {
    bool stop = false;
    int status = 0;
    float e = err;
    bool append = true;
    if (bad) { stop = true; status = 2; e = NAN; append = false; }
    else if (!isfinite(err)) { stop = true; status = 2; }
    else if (err < a.tol) { stop = true; status = 1; }
    if (cid == 0 && crank == 0 && threadIdx.x == 0) {
      if (append) {
        const int t = *a.n_trace;
        a.trace_iter[t] = kk;
        a.trace_err[t] = err;
        *a.n_trace = t + 1;
      }
      *a.out_status = status;
      *a.out_err = e;
    }
    failed = status == 2;
    return stop;
  }
  // stale combine of this CTA's columns over the cluster and broadcast of
  // g^k into every CTA's shared copy; returns "a column left the band".
  // Thread t sums rank slice t / CPC of column t % CPC (all its DSMEM loads in
  // flight), the slices are added in order, and the CPC x CL broadcast stores
  // are spread over every thread.
  static constexpr int NSL = NT / CPC;   // rank slices
  static constexpr int RPS = CL / NSL;   // ranks per slice
  // sum of the CL CTA partials of this CTA's column slice (thread c < CPC holds column c's)
  __device__ float cluster_slice_sum() {
    static_assert(NT % CPC == 0 && CL % (NT / CPC) == 0, "slicing");
    float* tmp = sm + kOffW;
    {
      const int c = threadIdx.x % CPC, sl = threadIdx.x / CPC, j = crank * CPC + c;
      float v[RPS];
#pragma unroll
      for (int u = 0; u < RPS; ++u) v[u] = remote(sm + kOffC, sl * RPS + u)[j];
      float S = 0.f;
#pragma unroll
      for (int u = 0; u < RPS; ++u) S += v[u];
      tmp[sl * CPC + c] = S;
    }
    __syncthreads();
    float S = 0.f;
    if (threadIdx.x < CPC) {
#pragma unroll
      for (int sl = 0; sl < NSL; ++sl) S += tmp[sl * CPC + threadIdx.x];
    }
    return S;
  }
  // MC: the software grid barrier, every CTA arriving (one arrival per cluster
  // behind a cluster barrier measured slower: the extra barrier.cluster costs
  // more than the 16x fewer same-address atomics, profiles/r2_c1_cluster.md)
  __device__ void mc_barrier() { grid_barrier(a.bar, epoch); }
  // MC stage 1 (before the grid barrier): the cluster's slice sums to global slot (k & 1)
  __device__ void stale_publish(int k) {
    const float S = cluster_slice_sum();
    if (threadIdx.x < CPC) a.part[(size_t)((k & 1) * ncl + cid) * W + crank * CPC + threadIdx.x] = S;
  }
  // MC stage 2 (after it): g^k of the slice from the NCL cluster sums in cluster
  // order (identical in every cluster), broadcast into the cluster's copies
  __device__ bool stale_finish(int k) {
    float* gt = sm + kOffW + NSL * CPC;
    bool fired = false;
    if (threadIdx.x < CPC) {
      const int c = threadIdx.x, j = crank * CPC + c;
      const float* P = a.part + (size_t)((k & 1) * ncl) * W + j;
      float v[kMaxClusters];
#pragma unroll
      for (int q = 0; q < kMaxClusters; ++q) v[q] = q < ncl ? ldcg(P + (size_t)q * W) : 0.f;
      float S = 0.f;
#pragma unroll
      for (int q = 0; q < kMaxClusters; ++q)
        if (q < ncl) S += v[q];
      const float gold = sm[kOffG + j];
      float gn = __fmul_rn(a.neg_eps, lse_finish(__fmul_rn(-gold, a.inv_eps), S));
      if (j >= a.m) gn = -INFINITY;
      else if (!shift_ok(S)) fired = true;
      gt[c] = gn;
    }
    fired = __syncthreads_or(fired);
    broadcast_g(gt);
    return fired;
  }
  __device__ bool combine_stale() {
    static_assert(NT % CPC == 0 && CL % (NT / CPC) == 0, "slicing");
    float* tmp = sm + kOffW;  // [NSL][CPC] slice sums, then [CPC] g (wred is free here)
    {
      const int c = threadIdx.x % CPC, sl = threadIdx.x / CPC, j = crank * CPC + c;
      float v[RPS];
#pragma unroll
      for (int u = 0; u < RPS; ++u) v[u] = remote(sm + kOffC, sl * RPS + u)[j];
      float S = 0.f;
#pragma unroll
      for (int u = 0; u < RPS; ++u) S += v[u];
      tmp[sl * CPC + c] = S;
    }
    __syncthreads();
    bool fired = false;
    if (threadIdx.x < CPC) {
      const int c = threadIdx.x, j = crank * CPC + c;
      float S = 0.f;
#pragma unroll
      for (int sl = 0; sl < NSL; ++sl) S += tmp[sl * CPC + c];
      const float gold = sm[kOffG + j];
      float gn = __fmul_rn(a.neg_eps, lse_finish(__fmul_rn(-gold, a.inv_eps), S));
      if (j >= a.m) gn = -INFINITY;  // padded column stays masked
      else if (!shift_ok(S)) fired = true;
      tmp[NSL * CPC + c] = gn;
    }
    fired = __syncthreads_or(fired);
    broadcast_g(tmp + NSL * CPC);
    return fired;
  }
  // g of this CTA's CPC columns (smem) -> every CTA's shared copy
  __device__ void broadcast_g(const float* gsrc) {
    for (int t = threadIdx.x; t < CPC * CL; t += NT) {
      const int c = t % CPC, r = t / CPC;
      remote(sm + kOffG, r)[crank * CPC + c] = gsrc[c];
    }
  }
  // exact column pass of f^k: online (max, sumexp) per column, warp -> CTA -> cluster
  __device__ void col_exact(const float* f) {
    float cm[E], cs[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { cm[e] = -INFINITY; cs[e] = 0.f; }
    __syncthreads();  // f of every warp's rows is in fS
    for (int i = r0 + w; i < r1; i += NW) {
      f2 c[P2];
      take_row(c);
      const float fi = f[i - r0], lmu = sm[kOffLm + i - r0];
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
#pragma unroll
      for (int p = 0; p < P2; ++p) {
        float y[2];
        up2(arg3x2(fi2, c[p], inv2, lm2, nz2), y[0], y[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = 2 * p + h;
          const float mo = cm[e];
          const float mn = fmax_nan(mo, y[h]);
          const float ms = (fabsf(mn) <= 3.402823466e38f) ? mn : 0.f;
          const float sl = __fmul_rn(ms, kLog2e);
          const float sv = (mo == -INFINITY) ? 0.f : cs[e] * exp_shifted(mo, sl);
          cs[e] = sv + exp_shifted(y[h], sl);
          cm[e] = mn;
        }
      }
    }
    float2* wr = reinterpret_cast<float2*>(sm + kOffW + w * 2 * W);
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int q = 0; q < 4; ++q) wr[col(v) + q] = make_float2(cm[4 * v + q], cs[4 * v + q]);
    __syncthreads();
    float2* cp = reinterpret_cast<float2*>(sm + kOffC);
    for (int j = threadIdx.x; j < W; j += NT) {
      float m0 = -INFINITY, s0 = 0.f;
      for (int u = 0; u < NW; ++u) {
        const float2 o = reinterpret_cast<const float2*>(sm + kOffW + u * 2 * W)[j];
        pair_merge(m0, s0, o.x, o.y);
      }
      cp[j] = make_float2(m0, s0);
    }
    cl.sync();
    float2* tmp = reinterpret_cast<float2*>(sm + kOffW);  // [NSL][CPC] slice pairs, then g
    {
      const int c = threadIdx.x % CPC, sl = threadIdx.x / CPC, j = crank * CPC + c;
      float2 v[RPS];
#pragma unroll
      for (int u = 0; u < RPS; ++u) v[u] = reinterpret_cast<const float2*>(remote(sm + kOffC, sl * RPS + u))[j];
      float m0 = -INFINITY, s0 = 0.f;
#pragma unroll
      for (int u = 0; u < RPS; ++u) pair_merge(m0, s0, v[u].x, v[u].y);
      tmp[sl * CPC + c] = make_float2(m0, s0);
    }
    __syncthreads();
    float* gt = sm + kOffW + 2 * NSL * CPC;
    if constexpr (MC) {  // the cluster's pairs -> global slot, grid barrier, NCL pairs merged in cluster order
      float2* P = a.pairs + (size_t)((nexact & 1) * ncl) * W;
      if (threadIdx.x < CPC) {
        const int c = threadIdx.x;
        float m0 = -INFINITY, s0 = 0.f;
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) pair_merge(m0, s0, tmp[sl * CPC + c].x, tmp[sl * CPC + c].y);
        P[(size_t)cid * W + crank * CPC + c] = make_float2(m0, s0);
      }
      mc_barrier();
      if (threadIdx.x < CPC) {
        const int j = crank * CPC + threadIdx.x;
        float2 v[kMaxClusters];
#pragma unroll
        for (int q = 0; q < kMaxClusters; ++q) v[q] = q < ncl ? __ldcg(P + (size_t)q * W + j) : make_float2(-INFINITY, 0.f);
        float m0 = -INFINITY, s0 = 0.f;
#pragma unroll
        for (int q = 0; q < kMaxClusters; ++q)
          if (q < ncl) pair_merge(m0, s0, v[q].x, v[q].y);
        tmp[threadIdx.x] = make_float2(m0, s0);
      }
      ++nexact;
    }
    if (threadIdx.x < CPC) {
      const int c = threadIdx.x, j = crank * CPC + c;
      float m0, s0;
      if constexpr (MC) {
        m0 = tmp[c].x;
        s0 = tmp[c].y;
      } else {
        m0 = -INFINITY;
        s0 = 0.f;
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) pair_merge(m0, s0, tmp[sl * CPC + c].x, tmp[sl * CPC + c].y);
      }
      float gn = __fmul_rn(a.neg_eps, lse_finish(m0, s0));
      if (j >= a.m) gn = -INFINITY;
      gt[c] = gn;
    }
    __syncthreads();
    broadcast_g(gt);
    cl.sync();
  }

  // ---- final check of iterate K and the transport cost (solver.py:108-112)
  __device__ void check_only(const float* f, float& err_acc, int& bad) {
    for (int i = r0 + w; i < r1; i += NW) {
      f2 c[P2];
      take_row(c);
      const float fold = f[i - r0], lmu = sm[kOffLm + i - r0];
      const f2 fo2 = pk2(fold, fold);
      f2 z2 = 0ull;
#pragma unroll
      for (int p = 0; p < P2; ++p) z2 = add2(z2, ex2x2(mul2(arg4x2(fo2, g2[p], c[p], inv2, lnu2, nz2), l2e2)));
      float z0, z1;
      up2(z2, z0, z1);
      float Sz = warp_sum(z0 + z1), Mz = 0.f;
      if (!shift_ok(Sz)) exact_lse<true>(c, fold, Mz, Sz);
      if (lane == 0) {
        const float rr = expf(__fadd_rn(lmu, lse_finish(Mz, Sz)));
        err_acc += fabsf(__fsub_rn(rr, sm[kOffMu + i - r0]));
        if (!isfinite(fold)) bad = 1;
      }
    }
  }
  __device__ float cost_rows(const float* f) {
    float acc = 0.f;
    for (int i = r0 + w; i < r1; i += NW) {
      f2 c[P2];
      take_row(c);
      const float fi = f[i - r0], lmu = sm[kOffLm + i - r0];
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
      float s = 0.f;
#pragma unroll
      for (int p = 0; p < P2; ++p) {
        const f2 zz = add2(arg4x2(fi2, g2[p], c[p], inv2, lm2, nz2), lnu2);
        float z0, z1, c0, c1;
        up2(zz, z0, z1);
        up2(c[p], c0, c1);
        s += __fmul_rn(c0, expf(z0));
        s += __fmul_rn(c1, expf(z1));
      }
      acc += warp_sum(s);
    }
    return acc;  // identical in every lane
  }

  __device__ void solve() {
    auto fb = [&](int k) { return (k & 1) ? a.f1 : a.f0; };
    auto gb = [&](int k) { return (k & 1) ? a.g1 : a.g0; };
    auto fs = [&](int k) { return sm + kOffF + (k & 1) * RPC; };  // f of the CTA's rows
    for (int j = threadIdx.x; j < W; j += NT) sm[kOffG + j] = j < a.m ? 0.f : -INFINITY;  // g^0
    for (int t = threadIdx.x; t < r1 - r0; t += NT) {
      sm[kOffF + t] = 0.f;  // f^0
      sm[kOffLm + t] = __ldg(a.log_mu + r0 + t);
      sm[kOffMu + t] = __ldg(a.mu + r0 + t);
    }
    ring_init();
    cl.sync();
    int final_k = a.max_iter;
    bool stopped = false, failed = false;
    int to_check = a.check;  // decremented from k = 2 on: zero at k = check + 1, 2 check + 1, ...
    for (int k = 1; k <= a.max_iter; ++k) {
#ifdef LSK_X_TRACE
#define LSK_CTR(slot)                                                                                     \
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && k >= 20 && k < 30)         \
  lsk_x_trace[1536 + (blockIdx.x == 0 ? 0 : 80) + (k - 20) * 8 + (slot)] = clock64()
#else
#define LSK_CTR(slot)
#endif
      LSK_CTR(0);
#ifdef LSK_X_TRACE
      cur_k = k;
#endif
      // check of iterate k-1 when (k - 1) % check == 0, k > 1: a countdown, no division
      const bool do_check = (k > 1) && (--to_check == 0);
      if (do_check) to_check = a.check;
      const bool fused = a.stale && k > 1;
      const bool gbad = do_check ? load_columns<true>() : load_columns<false>();
      float err_acc = 0.f;
      int bad = (do_check && gbad) ? 1 : 0;
      const float* fp = fs(k - 1);
      float* fn = fs(k);
      if (fused) {
        if (do_check) f_pass<true, true>(fp, fn, err_acc, bad);
        else f_pass<true, false>(fp, fn, err_acc, bad);
        LSK_CTR(1);
        cta_partial();
      } else {
        if (do_check) f_pass<false, true>(fp, fn, err_acc, bad);
        else f_pass<false, false>(fp, fn, err_acc, bad);
      }
      if (do_check) cta_check(err_acc, bad);
      LSK_CTR(2);
      cl.sync();  // (A) CTA partials, check scalars and f^k visible cluster-wide
      LSK_CTR(3);
      if constexpr (MC) {  // cluster slice sums and check scalars to global memory, one grid barrier
        if (fused) stale_publish(k);
        if (do_check) publish_cluster_err(k);
        LSK_CTR(4);
        if (fused || do_check) mc_barrier();
        LSK_CTR(5);
      }
      if (do_check && decide(k - 1, failed)) { stopped = true; final_k = k - 1; break; }
      bool need_exact = !fused;
      if (fused) {
        bool fired;
        if constexpr (MC) fired = stale_finish(k);
        else fired = combine_stale();
        LSK_CTR(6);
        if (w == 0 && lane < CL) remote(sm + kOffS, lane)[kMGuard + crank] = fired ? 1.f : 0.f;
        cl.sync();  // (B) g^k in every CTA's copy; guard flags in every CTA's mailbox
        LSK_CTR(7);
        need_exact = __any_sync(0xffffffffu, lane < CL && sm[kOffS + kMGuard + lane] != 0.f);
      }
      if (need_exact) {
        if (cid == 0 && crank == 0 && threadIdx.x == 0 && fused) {
          atomicAdd(a.stats + 1, 1);
          atomicMax(a.guard, k);
        }
        col_exact(fn);
      }
    }
    if (!stopped) {  // the final check at the cap (solver.py:286-316)
      final_k = a.max_iter;
      const bool gbad = load_columns();
      float err_acc = 0.f;
      int bad = gbad ? 1 : 0;
      check_only(fs(final_k), err_acc, bad);
      cta_check(err_acc, bad);
      cl.sync();
      if constexpr (MC) {
        publish_cluster_err(final_k + 1);
        mc_barrier();
      }
      decide(final_k, failed);
    }
    const int fbuf = final_k & 1;
    if (!failed && a.want_cost) {
      // g of the returned iterate: the shared copy holds g^{final_k} unless the
      // solve stopped inside iteration final_k + 1 (g^{final_k} is still current then too)
      load_columns();
      const float acc = cost_rows(fs(final_k));
      cl.sync();  // every CTA is done reading scal (decide) before it is reused
      if (lane == 0) sm[kOffS + w] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        float s = 0.f;
        for (int u = 0; u < NW; ++u) s += sm[kOffS + u];
        sm[kOffS + kSCost] = s;
      }
      cl.sync();
      float cost = 0.f;
      if (crank == 0 && w == 0) cost = warp_sum(lane < CL ? remote(sm + kOffS, lane)[kSCost] : 0.f);
      if constexpr (MC) {  // cluster costs -> global, summed in cluster order by cluster 0
        if (crank == 0 && threadIdx.x == 0) a.costpart[cid] = cost;
        mc_barrier();
        if (cid == 0 && crank == 0 && w == 0) cost = warp_sum(lane < ncl ? ldcg(a.costpart + lane) : 0.f);
      }
      if (cid == 0 && crank == 0 && threadIdx.x == 0) {
        if (!isfinite(cost)) { *a.out_status = 2; cost = NAN; }
        *a.out_cost = cost;
      }
    } else if (cid == 0 && crank == 0 && threadIdx.x == 0) {
      *a.out_cost = NAN;
    }
    // the returned iterate's potentials to global (f of the CTA's rows; g of its columns)
    for (int t = threadIdx.x; t < r1 - r0; t += NT) fb(fbuf)[r0 + t] = fs(final_k)[t];
    if (cid == 0)
      for (int t = threadIdx.x; t < CPC; t += NT)
        if (crank * CPC + t < a.m) gb(fbuf)[crank * CPC + t] = sm[kOffG + crank * CPC + t];
    if (cid == 0 && crank == 0 && threadIdx.x == 0) {
      *a.out_iters = final_k;
      *a.out_fbuf = fbuf;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // the ring's outstanding copies land before exit
    cl.sync();  // no CTA exits while another may still read its shared memory
  }
};

}  // namespace lsk

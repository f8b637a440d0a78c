// Persistent, register-resident log-domain Sinkhorn solver for dense fp32 C
// (m <= 8192): the whole solve -- K iterations, the fused marginal check every
// c iterations, the stop decision, the final check and the transport cost --
// is ONE cooperative launch with one CTA per SM.
//
// Reference path replaced: logsinkhorn.solver.solve (solver.py:230-337) with
// _alpha_step / _beta_step_* / _marginal_error / _transport_cost
// (solver.py:76-115) over reduction.py:179-224.
//
// Data layout and schedule:
//  * CTA b owns rows [b*n/G, (b+1)*n/G) for the whole solve. Thread t owns
//    columns j = 4*(v*NT + t) + q (v < V, q < 4), so per-column state (g_j,
//    log nu_j, the column shift, the column accumulator) lives in registers as
//    packed fp32 pairs and each smem row read is a conflict-free 16-byte LDS.
//  * Rows stream HBM -> smem through a STAGES-deep ring of TMA bulk copies
//    (cp.async.bulk + mbarrier complete_tx) that runs ahead across passes.
//    Passes alternate the sweep direction, so the rows one pass read last are
//    still L2-resident when the next pass starts.
//  * ONE pass over C per iteration (fused_pass): from the on-chip row the CTA
//    computes f_i^k (row LSE against g^{k-1}, shifted by the stale row shift
//    fl(-f_i^{k-1} * inv_eps)), and one step later -- once the row sum is
//    known -- adds exp(y_ij - s_j) into its per-column accumulators, where
//    y_ij = fl(fl(fl(f_i^k - C_ij) * inv_eps) + log mu_i) is the reference's
//    beta argument and s_j = fl(-g_j^{k-1} * inv_eps) the stale column shift
//    (terms are bounded by mu_i / nu_j, no overflow). Warps hand
//    the row sums to each other through an mbarrier per step (no block
//    barrier); thread 0 refills a ring stage once every warp is two rows past it.
//    A grid-wide fixed-order combine of the G per-CTA column partials forms
//    g^k. Sums outside [1e-20, 1e30] fall back to the exact max shift (rows:
//    from the smem copy of the row; columns: an exact (max, sumexp) pass).
//  * Uniform targets, 1e-3 <= eps <= 2e-3, n m >= 2^20 (fused_pass_mult): the g-side
//    term of (i, j) is the f-side term times 2^(a_i + b) in exact arithmetic,
//    so the column update is one FFMA2 per pair from the f-side terms kept in
//    registers (no second cost read, no second ex2); a block barrier per row.
//  * Every c iterations the pass of k+1 also evaluates the reference marginal
//    error formula for iterate k (solver.py:97-104) from the same on-chip row
//    -- no extra HBM pass, no host sync; f/g are double buffered so a stop at
//    k returns iterate k.
#pragma once
#include "lsk_device.cuh"

namespace lsk {

struct DenseArgs {
  const float* C;
  long long ldc;  // floats between rows (multiple of 4)
  int n, m, mpad; // mpad = round_up(m, 4): floats copied per row
  const float* log_mu;
  const float* log_nu;
  const float* mu;
  float inv_eps, neg_eps;
  float negzero;  // -0.0f, passed at run time (see muladd_rn2)
  double tol;
  int max_iter, check, stale, want_cost;
  int mult;       // column update from the f-side terms (see fused_pass_mult) ...
  int mult_iters; // ... for iterations k <= mult_iters only (its drift grows with k)
  // workspace (zero-initialised by the host where noted)
  float* f0; float* f1;  // f^k lives in f[k & 1]; f0 = 0 on entry
  float* g0; float* g1;  // g^k lives in g[k & 1]; g0 = 0 on entry
  float* part;           // [G][W] stale column partial sums
  float2* pairs;         // [G][W] exact column (max, sumexp) partials
  float* errpart;        // [G]
  int* flagpart;         // [G]
  float* errrow;         // [n] (unused by this solver)
  float* costpart;       // [G]
  unsigned long long* bar;  // grid barrier counter (zeroed): arrivals | flags << 32
  int* guard;            // last iteration whose column guard fired (zeroed)
  int* stats;            // [0] row-guard fires, [1] column-guard passes (zeroed)
  // outputs
  int* out_status;  // 0 not_converged, 1 converged, 2 numerical_failure
  int* out_iters;
  float* out_err;
  float* out_cost;
  int* out_fbuf;    // index of the buffer that holds the returned f/g
  int* trace_iter;
  float* trace_err;
  int* n_trace;
};

#ifdef LSK_X_TRACE
__device__ unsigned long long lsk_x_trace[2 * 256 * 3 + 160];
#endif

// UNI: every log nu_j equals log_nu[0] (uniform target weights, the C1-C5
// configs): the 2V log-nu register pairs become one broadcast pair and padded
// columns are masked through g = -inf instead of log nu = -inf.
template <int NT, int V, int STAGES, bool UNI = false>
struct DenseSolver {
  static constexpr bool kUniform = UNI;
  static constexpr int E = 4 * V;       // columns per thread
  static constexpr int P2 = 2 * V;      // packed pairs per thread
  static constexpr int W = 4 * V * NT;  // row capacity (floats)
  static constexpr int NW = NT / 32;
  static constexpr size_t kRingBytes = size_t(STAGES) * W * sizeof(float);
  // red layout (floats): [0, 4NW) double-buffered row sums (f, check);
  // [4NW, 4NW+128) exact-path block reductions; [4NW+128, +64NW) combines
  static constexpr int kRedRows = 0;
  static constexpr int kRedExact = 4 * NW;
  static constexpr int kRedComb = 4 * NW + 128;
  static constexpr size_t kRedFloats = 4 * NW + 128 + 64 * NW;
  // mbarriers: FULL[STAGES] (TMA) + SUMS[2] (per-step warp arrivals); then STAGES release counters
  // LSK_X_ALLARRIVE (sanitizer builds only): every thread arrives on the row-sum
  // mbarrier, so each reader's ordering before the next write / TMA refill is a
  // direct arrive->wait edge instead of one composed through __syncwarp and the
  // warp's lane-0 arrival (which racecheck does not compose)
#ifdef LSK_X_ALLARRIVE
  static constexpr int kSumArrivals = NT;
#else
  static constexpr int kSumArrivals = NW;
#endif
  static constexpr size_t kSmemBytes = kRingBytes + kRedFloats * sizeof(float) + (STAGES + 2) * 8 + STAGES * 4 + 64;

  // ---- per-CTA state
  const DenseArgs& a;
  float* ring;
  float* red;
  uint64_t* mbar;
  uint64_t* bsum;      // SUMS[2]: NW arrivals per step (step parity picks the barrier)
  unsigned* relc;      // [STAGES] warps done with the row in each stage
  unsigned gstep;      // fused steps so far (barrier / phase selection)
  // f and log mu of the last two rows of the previous fused pass: the first two
  // rows of the next pass when it is the very next pass (sweeps alternate)
  float carry_f0, carry_f1, carry_l0, carry_l1;
  int carry_pass;
  int b, G, r0, r1, rows;
  // TMA ring, tracked incrementally (no 64-bit div/mod on the hot path):
  // the producer (thread 0) walks the global row sequence pass by pass; the
  // consumers wait rows in the same order (head) and release them in order (tail).
  int iss_st, iss_pass, iss_step;  // next row to issue
  int head_st, head_ph;            // next row to wait for
  bool head_ready;                 // a probe saw the next row's TMA complete
  unsigned epoch;
  int pass;                        // pass counter (sweep direction = pass & 1)
  f2 inv2, l2e2, nz2;

  // ---- per-thread column state (packed pairs of the columns it owns)
  f2 g2[P2];   // g_j^{k-1}
  f2 ln2[P2];  // log nu_j (-inf beyond m); unused when UNI
  f2 lnu2;     // UNI: (log nu_0, log nu_0)
  float bcol;  // UNI: -log nu_0 * log2 e, the column exponent of fused_pass_mult
  f2 ac2[P2];  // column accumulators

  __device__ DenseSolver(const DenseArgs& args, unsigned char* smem) : a(args) {
    ring = reinterpret_cast<float*>(smem);
    red = reinterpret_cast<float*>(smem + kRingBytes);
    mbar = reinterpret_cast<uint64_t*>(smem + kRingBytes + kRedFloats * sizeof(float));
    bsum = mbar + STAGES;
    relc = reinterpret_cast<unsigned*>(bsum + 2);
    gstep = 0;
    carry_pass = -1;
    b = blockIdx.x;
    G = gridDim.x;
    r0 = int((long long)b * a.n / G);
    r1 = int((long long)(b + 1) * a.n / G);
    rows = r1 - r0;
    iss_st = iss_pass = iss_step = 0;
    head_st = head_ph = 0;
    head_ready = false;
    epoch = 0;
    pass = 0;
    inv2 = pk2(a.inv_eps, a.inv_eps);
    l2e2 = pk2(kLog2e, kLog2e);
    nz2 = pk2(a.negzero, a.negzero);
  }

  __device__ __forceinline__ int col(int v, int q) const { return 4 * (v * NT + threadIdx.x) + q; }
  // row processed at step q of pass P (passes alternate the sweep direction)
  __device__ __forceinline__ int row_of(int P, int q) const { return (P & 1) ? (r1 - 1 - q) : (r0 + q); }

  // ---------------- TMA ring
  __device__ __forceinline__ void issue() {
    const uint32_t bytes = uint32_t(a.mpad) * 4u;
    const int i = row_of(iss_pass, iss_step);
#ifndef LSK_X_NOTMA
    mbar_expect_tx(&mbar[iss_st], bytes);
    tma_load_1d(ring + size_t(iss_st) * W, a.C + (long long)i * a.ldc, bytes, &mbar[iss_st]);
#endif
#ifdef LSK_X_PFD
    int P = iss_pass, q = iss_step + LSK_X_PFD;
    while (q >= rows) { q -= rows; ++P; }
    prefetch_l2(a.C + (long long)row_of(P, q) * a.ldc, bytes);
#endif
  }
  __device__ __forceinline__ void advance_issue() {
    iss_st = (iss_st + 1 == STAGES) ? 0 : iss_st + 1;
    if (++iss_step == rows) { iss_step = 0; ++iss_pass; }
  }
  __device__ void ring_init() {
    // zero the ring once: columns >= mpad are never written by TMA and must read as 0
    float4* r4 = reinterpret_cast<float4*>(ring);
    for (size_t k = threadIdx.x; k < kRingBytes / 16; k += NT) r4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) mbar_init(&mbar[s], 1);
      mbar_init(&bsum[0], kSumArrivals);
      mbar_init(&bsum[1], kSumArrivals);
      for (int s = 0; s < STAGES; ++s) relc[s] = 0;
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) fence_proxy_async();
    for (int s = 0; s < STAGES; ++s) {
      if (threadIdx.x == 0) issue();
      advance_issue();
    }
  }
  // wait for the next row of the sequence; returns its smem copy
  __device__ __forceinline__ const float* wait_head() {
#ifndef LSK_X_NOTMA
    if (!head_ready) mbar_wait(&mbar[head_st], uint32_t(head_ph));
#endif
    head_ready = false;
    const float* p = ring + size_t(head_st) * W;
    if (++head_st == STAGES) { head_st = 0; head_ph ^= 1; }
    return p;
  }
  // probe the next row's TMA now so the next wait_head can skip the blocking
  // wait (the mbarrier round trip then overlaps this step's math)
  __device__ __forceinline__ void probe_head() {
#ifndef LSK_X_NOTMA
    head_ready = mbar_test(smem_u32(&mbar[head_st]), uint32_t(head_ph));
#endif
  }
  // release the oldest held row (call after a __syncthreads that follows every
  // read of it) and refill its stage with the next row of the sequence
  __device__ __forceinline__ void release() {
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue();
    }
    advance_issue();
  }
  // every stage holds an issued row at the end: wait for all before exit
  __device__ void drain() {
    for (int s = 0; s < STAGES; ++s) wait_head();
    __syncthreads();
  }

  // this thread's columns of a smem row as packed pairs
  __device__ __forceinline__ void load_row(const float* base, f2 (&c)[P2]) const {
#pragma unroll
    for (int v = 0; v < V; ++v) lds2x2(base + 4 * (v * NT + threadIdx.x), c[2 * v], c[2 * v + 1]);
  }

  // the stale column shift of g^{k-1}, negated: -fl(fl(-g_j inv_eps) log2 e) =
  // fl(fl(g_j inv_eps) log2 e) (round-to-nearest is sign-symmetric), formed on
  // the fly instead of holding 2V more register pairs
  __device__ __forceinline__ f2 nscol(int p) const { return mul2(mul2(g2[p], inv2), l2e2); }
  __device__ __forceinline__ f2 lnv(int p) const {
    if constexpr (UNI) return lnu2;
    else return ln2[p];
  }
  __device__ void load_lognu() {
    if constexpr (UNI) {
      const float L = __ldg(a.log_nu);
      lnu2 = pk2(L, L);
      bcol = -__fmul_rn(L, kLog2e);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = col(v, q);
          t[q] = j < a.m ? __ldg(a.log_nu + j) : -INFINITY;
        }
        ln2[2 * v] = pk2(t[0], t[1]);
        ln2[2 * v + 1] = pk2(t[2], t[3]);
      }
    }
  }

  // g^{k-1} into registers (+ the stale column shifts); returns "some owned g is non-finite"
  __device__ bool load_columns(const float* g) {
    bool bad = false;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int j0 = col(v, 0);
      float4 t4 = j0 < a.m ? ldcg4(reinterpret_cast<const float4*>(g + j0)) : make_float4(0.f, 0.f, 0.f, 0.f);
      float t[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (j0 + q >= a.m) t[q] = 0.f;
        bad |= !isfinite(t[q]);
        if (UNI && j0 + q >= a.m) t[q] = -INFINITY;  // padded column: every argument -inf
      }
      g2[2 * v] = pk2(t[0], t[1]);
      g2[2 * v + 1] = pk2(t[2], t[3]);
      ac2[2 * v] = 0ull;
      ac2[2 * v + 1] = 0ull;
    }
    return bad;
  }

  // ---------------- block reductions for the exact (max-shifted) paths
  __device__ __forceinline__ float block_max1(float v) {
    float t[1] = {v};
    block_reduce<NT, 1, true>(t, red + kRedExact);
    __syncthreads();
    return t[0];
  }
  __device__ __forceinline__ float block_sum1(float v) {
    float t[1] = {v};
    block_reduce<NT, 1, false>(t, red + kRedExact);
    __syncthreads();
    return t[0];
  }
  // exact LSE of the f argument arg3(g_j, C_ij, inv, lnu_j) over a smem row
  __device__ void exact_row(const float* row, float& M, float& S) {
    f2 c[P2];
    load_row(row, c);
    float mx = -INFINITY;
#pragma unroll
    for (int p = 0; p < P2; ++p) {
      float x0, x1;
      up2(arg3x2(g2[p], c[p], inv2, lnv(p), nz2), x0, x1);
      mx = fmax_nan(mx, fmax_nan(x0, x1));
    }
    M = block_max1(mx);
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    const f2 nsl = pk2(-__fmul_rn(Ms, kLog2e), -__fmul_rn(Ms, kLog2e));
    f2 s2 = 0ull;
#pragma unroll
    for (int p = 0; p < P2; ++p) s2 = add2(s2, ex2x2(fma2(arg3x2(g2[p], c[p], inv2, lnv(p), nz2), l2e2, nsl)));
    float s0, s1;
    up2(s2, s0, s1);
    S = block_sum1(s0 + s1);
  }
  // exact LSE of the check argument arg4(f_i, g_j, C_ij, inv, lnu_j) over a smem row
  __device__ void exact_check_row(const float* row, float fi, float& M, float& S) {
    f2 c[P2];
    load_row(row, c);
    const f2 f2i = pk2(fi, fi);
    float mx = -INFINITY;
#pragma unroll
    for (int p = 0; p < P2; ++p) {
      float x0, x1;
      up2(arg4x2(f2i, g2[p], c[p], inv2, lnv(p), nz2), x0, x1);
      mx = fmax_nan(mx, fmax_nan(x0, x1));
    }
    M = block_max1(mx);
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    const f2 nsl = pk2(-__fmul_rn(Ms, kLog2e), -__fmul_rn(Ms, kLog2e));
    f2 s2 = 0ull;
#pragma unroll
    for (int p = 0; p < P2; ++p) s2 = add2(s2, ex2x2(fma2(arg4x2(f2i, g2[p], c[p], inv2, lnv(p), nz2), l2e2, nsl)));
    float s0, s1;
    up2(s2, s0, s1);
    S = block_sum1(s0 + s1);
  }

  static __device__ __forceinline__ bool shift_ok(float S) { return S >= kShiftLo && S <= kShiftHi; }

  // fixed-order sum of the NW warp partials at red[off .. off+NW) (same bits in every thread)
  __device__ __forceinline__ float sum_warps(int off) const {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; w += 4) {
      const float4 t = *reinterpret_cast<const float4*>(red + off + w);
      s += (t.x + t.y) + (t.z + t.w);
    }
    return s;
  }

  // marginal-check bookkeeping for row i given its check sum (shift 0)
  __device__ __forceinline__ void check_row(const float* row, int i, float fold, float lmu, float Sz,
                                            float& err_acc, int& bad) {
    float Mz = 0.f;
    if (!shift_ok(Sz)) exact_check_row(row, fold, Mz, Sz);
    if (threadIdx.x == 0) {
      const float rr = expf(__fadd_rn(lmu, lse_finish(Mz, Sz)));
      err_acc += fabsf(__fsub_rn(rr, __ldg(a.mu + i)));
      if (!isfinite(fold)) bad = 1;
    }
  }

  // ================= the fused one-pass iteration (stale shifts) =================
  // f^k = neg_eps * LSE_j(arg3(g_j^{k-1}, C_ij)) for this CTA's rows, written to
  // fnew; stale-shift column partials of the beta argument into ac2; with CHECK,
  // the marginal error of iterate k-1 (fold = f^{k-1}, g2 = g^{k-1}).
  //
  // Software pipeline, one __syncthreads per row: step q computes the per-thread
  // row sums of row q, then the column update of row q-1 (whose f is known)
  // with the warp butterfly of row q's sums interleaved into it, then the
  // barrier, then every thread finishes row q from the NW warp sums.

  // per-thread partial sums of row `row` (f argument, and the check argument)
  template <bool CHECK>
  __device__ __forceinline__ void f_part(const float* row, float fold, float& s, float& z) const {
    f2 c[P2];
    load_row(row, c);
    const float shl = __fmul_rn(__fmul_rn(-fold, a.inv_eps), kLog2e);
    const f2 nsl = pk2(-shl, -shl);
    const f2 fo2 = pk2(fold, fold);
    f2 s2 = 0ull, z2 = 0ull;
#pragma unroll
    for (int p = 0; p < P2; ++p) {
#ifndef LSK_X_NOF
      s2 = add2(s2, ex2x2(fma2(arg3x2(g2[p], c[p], inv2, lnv(p), nz2), l2e2, nsl)));
#else
      s2 = add2(s2, c[p]);
#endif
      if (CHECK) z2 = add2(z2, ex2x2(mul2(arg4x2(fo2, g2[p], c[p], inv2, lnv(p), nz2), l2e2)));
    }
    float s0, s1;
    up2(s2, s0, s1);
    s = s0 + s1;
    if (CHECK) {
      up2(z2, s0, s1);
      z = s0 + s1;
    }
  }
  // column update of row `row` with its fresh f; the 5 butterfly levels of the
  // pending row sums (s, z) are interleaved so their latency hides under MUFU work
  template <bool CHECK, bool SHFL>
  __device__ __forceinline__ void g_part(const float* row, float fi, float lmu, float& s, float& z) {
    f2 c[P2];
    load_row(row, c);
    const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
#pragma unroll
    for (int p = 0; p < P2; ++p) {
#ifndef LSK_X_NOG
      ac2[p] = add2(ac2[p], ex2x2(fma2(arg3x2(fi2, c[p], inv2, lm2, nz2), l2e2, nscol(p))));
#else
      ac2[p] = add2(ac2[p], c[p]);
#endif
      if (SHFL && p < 5) {
        s += __shfl_xor_sync(0xffffffffu, s, 16 >> p);
        if (CHECK) z += __shfl_xor_sync(0xffffffffu, z, 16 >> p);
      }
    }
    if (SHFL)
#pragma unroll
      for (int l = P2; l < 5; ++l) {
        s += __shfl_xor_sync(0xffffffffu, s, 16 >> l);
        if (CHECK) z += __shfl_xor_sync(0xffffffffu, z, 16 >> l);
      }
  }
  // Row-sum hand-off between warps: no block barrier per row; each warp posts
  // its row sum with an mbarrier arrival (SUMS[step & 1]) and waits for step
  // q-1's arrivals only when it needs row q-1's total (at step q).
  __device__ __forceinline__ void post(unsigned step, float s, float z, bool check) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncwarp();  // the warp's reads of the rows it is done with precede the arrival
    if (lane == 0) {
      red[kRedRows + (step & 1) * NW + w] = s;
      if (check) red[kRedRows + 2 * NW + (step & 1) * NW + w] = z;
#ifndef LSK_X_ALLARRIVE
      mbar_arrive(&bsum[step & 1]);
#endif
    }
#ifdef LSK_X_ALLARRIVE
    mbar_arrive(&bsum[step & 1]);
#endif
  }
  // block-barrier hand-off of the multiplicative pass: the warp sum goes to red
  // and the next step's __syncthreads publishes it (no mbarrier)
  __device__ __forceinline__ void post_bar(unsigned step, float s) {
    if ((threadIdx.x & 31) == 0) red[kRedRows + (step & 1) * NW + (threadIdx.x >> 5)] = s;
  }
  __device__ __forceinline__ void wait_posted(unsigned step) {
#ifndef LSK_X_NOWAIT
    mbar_wait(&bsum[step & 1], (step >> 1) & 1);
#endif
  }
  // refill the stage that held row (P, q) with the row STAGES positions later
  // in the sequence (thread 0; every warp is known to be done with it)
  __device__ __forceinline__ void refill(int st, int P, int q) {
#ifndef LSK_X_NOTMA
    if (threadIdx.x == 0) {
      q += STAGES;
      while (q >= rows) { q -= rows; ++P; }
      const uint32_t bytes = uint32_t(a.mpad) * 4u;
      fence_proxy_async();
      mbar_expect_tx(&mbar[st], bytes);
      tma_load_1d(ring + size_t(st) * W, a.C + (long long)row_of(P, q) * a.ldc, bytes, &mbar[st]);
    }
#endif
  }
  // f of the row whose warp sums are in buffer `buf`: the stale-shift finish is
  // branch-free so it schedules into the MUFU stream of the next row's sums;
  // the (rare, CTA-uniform) out-of-range sum falls back to the exact row LSE
  __device__ __forceinline__ float finish_f(const float* row, float fold, float S) {
    float M = __fmul_rn(-fold, a.inv_eps);
    float fr = __fmul_rn(a.neg_eps, lse_finish(M, S));
    if (__builtin_expect(!shift_ok(S), 0)) {
      if (threadIdx.x == 0) atomicAdd(a.stats + 0, 1);
      exact_row(row, M, S);
      fr = __fmul_rn(a.neg_eps, lse_finish(M, S));
    }
    return fr;
  }

  // Step q: wait for row q and for every warp's sums of row q-1 (posted at
  // step q-1, which also means every warp is done with row q-2: thread 0
  // refills its stage); then, in one straight-line block, row q's partial sums
  // and row q-1's finish (sum of the NW warp sums + logf); then the column
  // update of row q-1 with row q's warp butterfly interleaved; post row q's
  // warp sum (mbarrier arrival, no block barrier). Warps drift by at most one
  // step, so two sum buffers / two barriers suffice.
  template <bool CHECK>
  __device__ void fused_pass(const float* fprev, float* fnew, float& err_acc, int& bad) {
    const int P = pass++;
    // scalars of rows q (cur) and q+1 (nx), prefetched one step ahead; the
    // first two come from the previous pass's registers when it was pass P-1
    int i_cur = row_of(P, 0);
    int i_nx = rows > 1 ? row_of(P, 1) : i_cur;
    float fold_cur, lmu_cur, fold_nx, lmu_nx;
    if (carry_pass == P && rows > 1) {
      fold_cur = carry_f0; lmu_cur = carry_l0;
      fold_nx = carry_f1; lmu_nx = carry_l1;
    } else {
      fold_cur = ldcg(fprev + i_cur);
      lmu_cur = __ldg(a.log_mu + i_cur);
      fold_nx = rows > 1 ? ldcg(fprev + i_nx) : fold_cur;
      lmu_nx = rows > 1 ? __ldg(a.log_mu + i_nx) : lmu_cur;
    }
    const unsigned g0 = gstep;
    int st_cur = head_st;
    const float* row = wait_head();
    float s, z = 0.f;
    f_part<CHECK>(row, fold_cur, s, z);
    s = warp_sum(s);
    if (CHECK) z = warp_sum(z);
    post(g0, s, z, CHECK);
    const float* row_prev = row;
    int st_prev = st_cur, st_pp = 0;
    int i_prev = i_cur;
    float fold_prev = fold_cur, lmu_prev = lmu_cur;
    for (int q = 1; q < rows; ++q) {
      i_cur = i_nx; fold_cur = fold_nx; lmu_cur = lmu_nx;
      if (q + 1 < rows) {
        i_nx = row_of(P, q + 1);
        fold_nx = ldcg(fprev + i_nx);
        lmu_nx = __ldg(a.log_mu + i_nx);
      }
      st_cur = head_st;
#ifdef LSK_X_TRACE
      const unsigned long long tr0 = clock64();
#endif
      row = wait_head();
#ifdef LSK_X_TRACE
      const unsigned long long tr1 = clock64();
#endif
      const unsigned sp = g0 + q - 1;
      wait_posted(sp);
#ifdef LSK_X_TRACE
      {
        const unsigned long long tr2 = clock64();
        const int w = threadIdx.x >> 5;
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (w == 0 || w == NW - 1) && P == 20) {
          const int k = (w == 0 ? 0 : 1) * 256 + (q & 255);
          lsk_x_trace[k * 3 + 0] = tr0;
          lsk_x_trace[k * 3 + 1] = tr1;
          lsk_x_trace[k * 3 + 2] = tr2;
        }
      }
#endif
      if (q >= 2) refill(st_pp, P, q - 2);
      const float S = sum_warps(kRedRows + (sp & 1) * NW);
      f_part<CHECK>(row, fold_cur, s, z);
      const float f_prev = finish_f(row_prev, fold_prev, S);
      if (CHECK) check_row(row_prev, i_prev, fold_prev, lmu_prev, sum_warps(kRedRows + 2 * NW + (sp & 1) * NW), err_acc, bad);
      if (threadIdx.x == 0) fnew[i_prev] = f_prev;
      g_part<CHECK, true>(row_prev, f_prev, lmu_prev, s, z);
      carry_f1 = f_prev;
      carry_l1 = lmu_prev;
      post(g0 + q, s, z, CHECK);
      st_pp = st_prev;
      row_prev = row;
      st_prev = st_cur;
      i_prev = i_cur;
      fold_prev = fold_cur;
      lmu_prev = lmu_cur;
    }
    const unsigned sl = g0 + rows - 1;
    wait_posted(sl);
    if (rows >= 2) refill(st_pp, P, rows - 2);
    const float f_last = finish_f(row_prev, fold_prev, sum_warps(kRedRows + (sl & 1) * NW));
    if (CHECK) check_row(row_prev, i_prev, fold_prev, lmu_prev, sum_warps(kRedRows + 2 * NW + (sl & 1) * NW), err_acc, bad);
    if (threadIdx.x == 0) fnew[i_prev] = f_last;
    g_part<false, false>(row_prev, f_last, lmu_prev, s, z);
    __syncthreads();
    refill(st_prev, P, rows - 1);
    gstep = g0 + rows;
    carry_f0 = f_last;
    carry_l0 = lmu_prev;
    carry_pass = rows > 1 ? P + 1 : -1;
    // the barrier-synchronised passes resume the ring cursor after this pass
    {
      int q2 = rows + STAGES, P2_ = P;
      while (q2 >= rows) { q2 -= rows; ++P2_; }
      iss_pass = P2_;
      iss_step = q2;
      iss_st = head_st;
    }
  }
  // ================= fused pass with the multiplicative column update ==============
  // In exact arithmetic the g-side term of element (i, j) is the f-side term
  // times 2^(a_i + b_j):  exp(y_ij - M_j) = exp(x_ij - M_i) * exp(a_i + b_j) with
  // a_i = (f_i^k - f_i^{k-1}) / eps + log mu_i and b_j = -log nu_j (the stale
  // shifts are M_i = -f^{k-1}_i / eps, M_j = -g^{k-1}_j / eps). So the column
  // update of row q-1 needs no cost element and no ex2: one FFMA2 per pair
  // from the f-side terms kept in registers (uniform nu only: b_j is one scalar). It is used for a row
  // only while a_i stays in a band where no f-side term that underflowed could
  // matter to a column sum inside the guard band, and only when 1e-3 <= eps <= 2e-3
  // (a.mult); otherwise the row takes the direct update. The exponents carry
  // the f-side argument rounding instead of the g-side one (|dy| <= |y| 2^-24):
  // parity with the reference stays within the fp32 tolerance there (its gauge
  // drift grows with eps * K: 1.2e-5 at eps = 1e-2, K = 300, profiles/r2_c1_cluster.md).
  __device__ __forceinline__ void f_part_e(const float* row, float fold, float& s, f2 (&e)[P2]) const {
    f2 c[P2];
    load_row(row, c);
    const float shl = __fmul_rn(__fmul_rn(-fold, a.inv_eps), kLog2e);
    const f2 nsl = pk2(-shl, -shl);
    f2 s2 = 0ull;
#pragma unroll
    for (int p = 0; p < P2; ++p) {
      e[p] = ex2x2(fma2(arg3x2(g2[p], c[p], inv2, lnv(p), nz2), l2e2, nsl));
      s2 = add2(s2, e[p]);
    }
    float s0, s1;
    up2(s2, s0, s1);
    s = s0 + s1;
  }
  template <bool SHFL>
  __device__ __forceinline__ void col_update(const float* row, float fi, float fold, float lmu, const f2 (&e)[P2],
                                             float& s) {
    const float ai = __fmul_rn(__fadd_rn(__fmul_rn(__fsub_rn(fi, fold), a.inv_eps), lmu), kLog2e);
    if (ai >= -100.f && ai + bcol <= 23.f) {
      const float A = ex2(ai + bcol);
      const f2 A2 = pk2(A, A);
#pragma unroll
      for (int p = 0; p < P2; ++p) {
        ac2[p] = fma2(e[p], A2, ac2[p]);
        if (SHFL && p < 5) s += __shfl_xor_sync(0xffffffffu, s, 16 >> p);
      }
      if (SHFL)
#pragma unroll
        for (int l = P2; l < 5; ++l) s += __shfl_xor_sync(0xffffffffu, s, 16 >> l);
    } else {
      float z = 0.f;
      g_part<false, SHFL>(row, fi, lmu, s, z);
    }
  }

  __device__ void fused_pass_mult(const float* fprev, float* fnew) {
    const int P = pass++;
    int i_cur = row_of(P, 0);
    int i_nx = rows > 1 ? row_of(P, 1) : i_cur;
    float fold_cur, lmu_cur, fold_nx, lmu_nx;
    if (carry_pass == P && rows > 1) {
      fold_cur = carry_f0; lmu_cur = carry_l0;
      fold_nx = carry_f1; lmu_nx = carry_l1;
    } else {
      fold_cur = ldcg(fprev + i_cur);
      lmu_cur = __ldg(a.log_mu + i_cur);
      fold_nx = rows > 1 ? ldcg(fprev + i_nx) : fold_cur;
      lmu_nx = rows > 1 ? __ldg(a.log_mu + i_nx) : lmu_cur;
    }
    const unsigned g0 = gstep;
    f2 eA[P2], eB[P2];
    int st_cur = head_st;
    const float* row = wait_head();
    probe_head();
    float s;
    f_part_e(row, fold_cur, s, eA);
    s = warp_sum(s);
    post_bar(g0, s);
    const float* row_prev = row;
    int st_prev = st_cur, st_pp = 0;
    int i_prev = i_cur;
    float fold_prev = fold_cur, lmu_prev = lmu_cur;
    auto step = [&](int q, const f2 (&ein)[P2], f2 (&eout)[P2]) {
      i_cur = i_nx; fold_cur = fold_nx; lmu_cur = lmu_nx;
      if (q + 1 < rows) {
        i_nx = row_of(P, q + 1);
        fold_nx = ldcg(fprev + i_nx);
        lmu_nx = __ldg(a.log_mu + i_nx);
      }
      st_cur = head_st;
      row = wait_head();
      probe_head();
      const unsigned sp = g0 + q - 1;
      __syncthreads();  // every warp's sum of row q-1 is in red (and row q-2 is done)
      if (q >= 2) refill(st_pp, P, q - 2);
      const float S = sum_warps(kRedRows + (sp & 1) * NW);
      f_part_e(row, fold_cur, s, eout);
      const float f_prev = finish_f(row_prev, fold_prev, S);
      if (threadIdx.x == 0) fnew[i_prev] = f_prev;
      col_update<true>(row_prev, f_prev, fold_prev, lmu_prev, ein, s);
      carry_f1 = f_prev;
      carry_l1 = lmu_prev;
      post_bar(g0 + q, s);
      st_pp = st_prev;
      row_prev = row;
      st_prev = st_cur;
      i_prev = i_cur;
      fold_prev = fold_cur;
      lmu_prev = lmu_cur;
    };
    int q = 1;
    for (; q + 1 < rows; q += 2) {
      step(q, eA, eB);
      step(q + 1, eB, eA);
    }
    const bool odd = q < rows;
    if (odd) step(q, eA, eB);
    const unsigned sl = g0 + rows - 1;
    __syncthreads();
    if (rows >= 2) refill(st_pp, P, rows - 2);
    const float f_last = finish_f(row_prev, fold_prev, sum_warps(kRedRows + (sl & 1) * NW));
    if (threadIdx.x == 0) fnew[i_prev] = f_last;
    if (odd) col_update<false>(row_prev, f_last, fold_prev, lmu_prev, eB, s);
    else col_update<false>(row_prev, f_last, fold_prev, lmu_prev, eA, s);
    __syncthreads();
    refill(st_prev, P, rows - 1);
    // gstep (the SUMS mbarrier phase count) is untouched: this pass hands off through __syncthreads
    carry_f0 = f_last;
    carry_l0 = lmu_prev;
    carry_pass = rows > 1 ? P + 1 : -1;
    {
      int q2 = rows + STAGES, P2_ = P;
      while (q2 >= rows) { q2 -= rows; ++P2_; }
      iss_pass = P2_;
      iss_step = q2;
      iss_st = head_st;
    }
  }

  // ================= exact row pass (two-pass max/sum from the on-chip row) ========
  template <bool CHECK>
  __device__ void row_exact_pass(const float* fprev, float* fnew, float& err_acc, int& bad) {
    const int P = pass++;
    carry_pass = -1;  // f changes outside the fused pass
    for (int q = 0; q < rows; ++q) {
      const int i = row_of(P, q);
      const float* row = wait_head();
      float M, S;
      exact_row(row, M, S);
      const float fr = __fmul_rn(a.neg_eps, lse_finish(M, S));
      if (CHECK) {
        const float fold = ldcg(fprev + i);
        const f2 fo2 = pk2(fold, fold);
        f2 c[P2];
        load_row(row, c);
        f2 z2 = 0ull;
#pragma unroll
        for (int p = 0; p < P2; ++p) z2 = add2(z2, ex2x2(mul2(arg4x2(fo2, g2[p], c[p], inv2, lnv(p), nz2), l2e2)));
        float s0, s1;
        up2(z2, s0, s1);
        const float Sz = block_sum1(s0 + s1);
        check_row(row, i, fold, __ldg(a.log_mu + i), Sz, err_acc, bad);
      }
      if (threadIdx.x == 0) fnew[i] = fr;
      __syncthreads();
      release();
    }
  }

  // ================= check-only pass (final check at the cap) =================
  __device__ void check_pass(const float* f, float& err_acc, int& bad) {
    const int P = pass++;
    for (int q = 0; q < rows; ++q) {
      const int i = row_of(P, q);
      const float* row = wait_head();
      const float fold = ldcg(f + i);
      const f2 fo2 = pk2(fold, fold);
      f2 c[P2];
      load_row(row, c);
      f2 z2 = 0ull;
#pragma unroll
      for (int p = 0; p < P2; ++p) z2 = add2(z2, ex2x2(mul2(arg4x2(fo2, g2[p], c[p], inv2, lnv(p), nz2), l2e2)));
      float s0, s1;
      up2(z2, s0, s1);
      const float Sz = block_sum1(s0 + s1);
      check_row(row, i, fold, __ldg(a.log_mu + i), Sz, err_acc, bad);
      __syncthreads();
      release();
    }
  }

  // ================= transport cost: sum_ij fl(C_ij * exp(z_ij)), z as solver.py:108-112
  __device__ void cost_pass(const float* f, float& cost_acc) {
    const int P = pass++;
    for (int q = 0; q < rows; ++q) {
      const int i = row_of(P, q);
      const float* row = wait_head();
      const float fi = ldcg(f + i), lmu = __ldg(a.log_mu + i);
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
      f2 c[P2];
      load_row(row, c);
      float s = 0.f;
#pragma unroll
      for (int p = 0; p < P2; ++p) {
        const f2 z = add2(arg4x2(fi2, g2[p], c[p], inv2, lm2, nz2), lnv(p));
        float z0, z1, c0, c1;
        up2(z, z0, z1);
        up2(c[p], c0, c1);
        s += __fmul_rn(c0, expf(z0));
        s += __fmul_rn(c1, expf(z1));
      }
      const float S = block_sum1(s);
      if (threadIdx.x == 0) cost_acc += S;
      __syncthreads();
      release();
    }
  }

  // ================= exact column pass: online (max, sumexp) per owned column ======
  // beta argument arg3(f_i^k, C_ij, inv, log mu_i); writes (max, sum) pairs to a.pairs[b]
  __device__ void col_exact_pass(const float* f) {
    const int P = pass++;
    float cm[E], cs[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { cm[e] = -INFINITY; cs[e] = 0.f; }
    for (int q = 0; q < rows; ++q) {
      const int i = row_of(P, q);
      const float* row = wait_head();
      const float fi = ldcg(f + i), lmu = __ldg(a.log_mu + i);
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
      f2 c[P2];
      load_row(row, c);
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
          const float s = (mo == -INFINITY) ? 0.f : cs[e] * exp_shifted(mo, sl);
          cs[e] = s + exp_shifted(y[h], sl);
          cm[e] = mn;
        }
      }
      __syncthreads();
      release();
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int j0 = col(v, 0);
      if (j0 >= a.m) continue;
      float2* dst = a.pairs + (size_t)b * W + j0;
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float2(cm[4 * v + q], cs[4 * v + q]);
    }
  }

  // ---- fixed-order tree over the G per-CTA scalars (identical in every CTA)
  __device__ float tree_over_ctas(const float* v) {
    const int lane = threadIdx.x & 31;
    float s = 0.f;
    for (int k = lane; k < G; k += 32) s += ldcg(v + k);
    return warp_sum(s);
  }
  __device__ int any_over_ctas(const int* v) {
    const int lane = threadIdx.x & 31;
    int s = 0;
    for (int k = lane; k < G; k += 32) s |= __ldcg(v + k);
    return __any_sync(0xffffffffu, s != 0);
  }

  // ---- column combines: CTA b handles 32-column groups b, b+G, ...; the NW
  // warps split the G partial rows into contiguous ranges, then a fixed
  // halving tree over the NW range sums (in smem) finishes each column.
  // Column combine, balanced over the grid: CTA b owns the contiguous columns
  // [b m/G, (b+1) m/G); its threads are (column, slice) pairs -- slice q of
  // QS sums the partial rows k = q, q + QS, ... of its column with all loads
  // in flight at once -- then one thread per column adds the QS slice sums in
  // order (deterministic) and finishes g_j.
  __device__ void combine_stale(const float* gold, float* gnew, int k) {
    const int j0 = int((long long)b * a.m / G), j1 = int((long long)(b + 1) * a.m / G);
    const int nc = j1 - j0;
    float* cr = red + kRedComb;  // [QS][nc] slice sums (64*NW floats available)
    const int QS = nc > 0 ? min(NT / nc, (64 * NW) / nc) : 1;
    const int t = threadIdx.x;
    bool fired = false;
    if (nc > 0 && QS >= 1 && t < QS * nc) {
      const int c = t % nc, q = t / nc, j = j0 + c;
      // every partial of the slice in flight at once (one L2 round trip), then
      // summed in a fixed order
#ifndef LSK_X_COMB_KB
#define LSK_X_COMB_KB 40  // >= G / QS at C2 (148 / 4): every partial of a slice in one L2 round trip
#endif
      constexpr int KB = LSK_X_COMB_KB;
      float s = 0.f;
      for (int k0 = q; k0 < G; k0 += KB * QS) {
        float v[KB];
#pragma unroll
        for (int u = 0; u < KB; ++u) {
          const int kk = k0 + u * QS;
          v[u] = kk < G ? ldcg(a.part + (size_t)kk * W + j) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < KB; u += 4) s += (v[u] + v[u + 1]) + (v[u + 2] + v[u + 3]);
      }
      cr[q * nc + c] = s;
    }
    const float gj = (t < nc) ? ldcg(gold + j0 + t) : 0.f;  // issued before the barrier
    __syncthreads();
    if (t < nc) {
      float S = 0.f;
      for (int q = 0; q < QS; ++q) S += cr[q * nc + t];
      const float sj = __fmul_rn(-gj, a.inv_eps);
      if (!shift_ok(S)) fired = true;
      gnew[j0 + t] = __fmul_rn(a.neg_eps, lse_finish(sj, S));
    }
    if (__syncthreads_or(fired) && threadIdx.x == 0) atomicMax(a.guard, k);
  }

  __device__ void combine_pairs(float* gnew) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ngroups = (a.m + 31) / 32;
    float* cr = red + kRedComb;
    for (int grp = b; grp < ngroups; grp += G) {
      const int j = grp * 32 + lane;
      const int k0 = w * G / NW, k1 = (w + 1) * G / NW;
      float mx = -INFINITY, s = 0.f;
      if (j < a.m)
        for (int kk = k0; kk < k1; ++kk) {
          float2 p = __ldcg(a.pairs + (size_t)kk * W + j);
          pair_merge(mx, s, p.x, p.y);
        }
      cr[w * 64 + lane] = mx;
      cr[w * 64 + 32 + lane] = s;
      __syncthreads();
      if (w == 0) {
        for (int h = NW / 2; h >= 1; h >>= 1)
          for (int u = 0; u < h; ++u) {
            float m1 = cr[u * 64 + lane], s1 = cr[u * 64 + 32 + lane];
            pair_merge(m1, s1, cr[(u + h) * 64 + lane], cr[(u + h) * 64 + 32 + lane]);
            cr[u * 64 + lane] = m1;
            cr[u * 64 + 32 + lane] = s1;
          }
        if (j < a.m) gnew[j] = __fmul_rn(a.neg_eps, lse_finish(cr[lane], cr[32 + lane]));
      }
      __syncthreads();
    }
  }

  __device__ void store_stale_partials() {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (col(v, 0) >= a.m) continue;
      float x0, x1, x2, x3;
      up2(ac2[2 * v], x0, x1);
      up2(ac2[2 * v + 1], x2, x3);
      reinterpret_cast<float4*>(a.part + (size_t)b * W)[v * NT + threadIdx.x] = make_float4(x0, x1, x2, x3);
    }
  }

  // ---- check decision, identical in every CTA (solver.py:286-300)
  // returns true if the solve stops at iterate kk
  __device__ bool decide(int kk, bool& failed) {
    const int bad = any_over_ctas(a.flagpart);
    const float err = tree_over_ctas(a.errpart);
    bool stop = false;
    int status = 0;
    float e = err;
    bool append = true;
    if (bad) { stop = true; status = 2; e = NAN; append = false; }
    else if (!isfinite(err)) { stop = true; status = 2; }
    else if (err < a.tol) { stop = true; status = 1; }
    if (b == 0 && threadIdx.x == 0) {
      if (append) {
        int t = *a.n_trace;
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

  __device__ void publish_check(float err_acc, int bad) {
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) { a.errpart[b] = err_acc; a.flagpart[b] = bad; }
  }

  __device__ void solve() {
    load_lognu();
    ring_init();
    auto fb = [&](int k) { return (k & 1) ? a.f1 : a.f0; };
    auto gb = [&](int k) { return (k & 1) ? a.g1 : a.g0; };
    int final_k = a.max_iter;
    bool stopped = false, failed = false;
    for (int k = 1; k <= a.max_iter; ++k) {
      const bool do_check = (k > 1) && ((k - 1) % a.check == 0);
      const float* gcur = gb((k - 1) & 1);
      const bool gbad = load_columns(gcur);
      float err_acc = 0.f;
      int bad = (do_check && gbad) ? 1 : 0;
      const bool fused = a.stale && k > 1;
#ifdef LSK_X_TRACE
#define LSK_TR(slot) \
  if (threadIdx.x == 0 && (b == 0 || b == G - 1) && k >= 20 && k < 30) lsk_x_trace[1536 + (b == 0 ? 0 : 80) + (k - 20) * 8 + (slot)] = clock64()
#else
#define LSK_TR(slot)
#endif
      LSK_TR(0);
      if (fused) {
        if (do_check) fused_pass<true>(fb((k - 1) & 1), fb(k & 1), err_acc, bad);
        else if (UNI && a.mult && k <= a.mult_iters) fused_pass_mult(fb((k - 1) & 1), fb(k & 1));
        else fused_pass<false>(fb((k - 1) & 1), fb(k & 1), err_acc, bad);
        LSK_TR(1);
        store_stale_partials();
      } else {
        if (do_check) row_exact_pass<true>(fb((k - 1) & 1), fb(k & 1), err_acc, bad);
        else row_exact_pass<false>(fb((k - 1) & 1), fb(k & 1), err_acc, bad);
      }
      if (do_check) publish_check(err_acc, bad);
      LSK_TR(2);
      grid_barrier(a.bar, epoch);
      LSK_TR(3);
      if (do_check && decide(k - 1, failed)) { stopped = true; final_k = k - 1; break; }
      if (fused) {
        combine_stale(gcur, gb(k & 1), k);
        LSK_TR(4);
        grid_barrier(a.bar, epoch);
        LSK_TR(5);
      }
      const bool need_exact = !fused || (__ldcg(a.guard) == k);
      if (need_exact) {
        if (threadIdx.x == 0 && b == 0 && fused) atomicAdd(a.stats + 1, 1);
        col_exact_pass(fb(k & 1));
        grid_barrier(a.bar, epoch);
        combine_pairs(gb(k & 1));
        grid_barrier(a.bar, epoch);
      }
    }
    if (!stopped) {
      // the final check at the cap (solver.py:286-316: in-loop if K % c == 0, else the extra one)
      final_k = a.max_iter;
      const bool gbad = load_columns(gb(final_k & 1));
      float err_acc = 0.f;
      int bad = gbad ? 1 : 0;
      check_pass(fb(final_k & 1), err_acc, bad);
      publish_check(err_acc, bad);
      grid_barrier(a.bar, epoch);
      decide(final_k, failed);
    }
    const int fbuf = final_k & 1;
    if (!failed && a.want_cost) {
      load_columns(gb(fbuf));
      float cost_acc = 0.f;
      cost_pass(fb(fbuf), cost_acc);
      if (threadIdx.x == 0) a.costpart[b] = cost_acc;
      grid_barrier(a.bar, epoch);
      if (b == 0) {
        float cost = tree_over_ctas(a.costpart);
        if (threadIdx.x == 0) {
          if (!isfinite(cost)) { *a.out_status = 2; cost = NAN; }
          *a.out_cost = cost;
        }
      }
    } else if (b == 0 && threadIdx.x == 0) {
      *a.out_cost = NAN;
    }
    if (b == 0 && threadIdx.x == 0) {
      *a.out_iters = final_k;
      *a.out_fbuf = fbuf;
    }
    drain();
  }
};

}  // namespace lsk

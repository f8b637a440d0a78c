// EXPERIMENT (round 2, rejected; not built): two-team variant of the dense
// solver, kept as the record behind profiles/r2_dense_experiments.md. It was
// wired as k_solve_dense<TeamSolver<8, 3>> with a [G][2W] float scratch in
// DenseArgs; measured 11.4 ms vs 10.1 ms per 200 C2 iterations (one team).
// Two-team persistent dense solver (uniform targets, multiplicative column
// update): the C2 headline kernel (n=m=8192, eps >= 1e-3).
//
// Reference path replaced: logsinkhorn.solver.solve (solver.py:230-337) with
// _alpha_step / _beta_step_* / _marginal_error / _transport_cost
// (solver.py:76-115) over reduction.py:179-224 -- the same contract as
// DenseSolver (lsk_dense.cuh); this kernel only changes the schedule.
//
// Why two teams (profiles/r2_dense_teams.md): with one 8-warp team every row
// step is a lock-stepped chain -- the row's warp sums, an accurate logf, the
// column scale 2^(a_i+b), the column FFMA2s, the 5-level warp butterfly, a
// block barrier -- and with 2 warps per scheduler the MUFU idles while it
// runs (ncu r2: 'wait' + 'short_scoreboard' 25% of the samples, issue 36%).
// Here each CTA runs TWO independent 8-warp teams of 256 threads; team t
// takes the even / odd positions of the CTA's row sequence, owns its own
// 3-stage TMA ring and synchronises on its own named barrier, so one team's
// serial row finish overlaps the other team's ex2 stream (4 warps per
// scheduler). Each team-thread owns 32 columns: their accumulators and the
// row's f-side terms stay in registers (<= 128 per thread at 512 threads), g
// is read from ONE shared-memory copy per CTA (32 KB; shared-memory traffic per
// row = C row + g = 64 KB = 512 cycles at 128 B/clk, the same as the row's
// MUFU time and well under its HBM time).
//
// Row step of a team (row k of its sequence, one named barrier per row):
//   wait TMA(row k); team barrier (every warp posted row k-1's sums and is
//   done with row k-1's smem) ; refill row k-1's stage ; finish f of row
//   k-1 (stale shift + logf) ; column update of row k-1 = one FFMA2 per pair
//   from its f-side terms e (kept in registers since step k-1) ; f-side terms
//   of row k (overwriting e) and their sums ; butterfly ; post.
// Rare paths (a row sum outside the guard band, a column scale outside the
// band of the multiplicative update) re-read the row from global memory
// (L2), so a ring stage is free as soon as the f-side terms are formed.
// The two teams' column accumulators are added in a fixed order (team 0 +
// team 1) before the grid-wide combine, so the solve is deterministic.
#pragma once
#include "lsk_dense.cuh"

namespace lsk {

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int V, int STAGES>
struct TeamSolver {
  static constexpr bool kUniform = true;
  static constexpr int NT = 256;           // threads per team
  static constexpr int TEAMS = 2;
  static constexpr int NTB = NT * TEAMS;   // threads per CTA
  static constexpr int NW = NT / 32;       // warps per team
  static constexpr int NWB = NTB / 32;     // warps per CTA
  static constexpr int E = 4 * V;          // columns per thread
  static constexpr int P2 = 2 * V;         // packed pairs per thread
  static constexpr int W = 4 * V * NT;     // row capacity (floats)
  static constexpr size_t kRingBytes = size_t(TEAMS) * STAGES * W * sizeof(float);
  // per-team red (floats): [0, 2NW) row sums, [2NW, 4NW) check sums (both
  // double buffered by step parity), [4NW, 4NW + 32) exact-path reductions
  static constexpr int kRedTeam = 4 * NW + 32;
  static constexpr int kRedComb = 64 * NWB;  // CTA-wide combine scratch (aliases the g copy)
  static constexpr int kRedMisc = 16;        // team merges of the check / cost scalars
  static_assert(kRedComb <= W, "combine scratch aliases the g copy");
  static constexpr size_t kRedFloats = W + TEAMS * kRedTeam + kRedMisc;  // g copy | team reds | misc
  static constexpr size_t kSmemBytes = kRingBytes + kRedFloats * sizeof(float) + TEAMS * STAGES * 8 + 64;

  const DenseArgs& a;
  float* ring;      // this team's ring [STAGES][W]
  float* red;       // this team's red
  float* gsm;       // g^{k-1}, one copy per CTA [W] (-inf beyond m)
  float* comb;      // CTA-wide combine scratch (= gsm, used only between the passes)
  float* misc;
  uint64_t* full;   // this team's FULL[STAGES] (TMA complete_tx)
  int tid, team, b, G, r0, r1, rows, rows_t;
  int iss_st, iss_pass, iss_k;  // producer cursor (team thread 0)
  int head_st, head_ph;         // consumer cursor (every thread of the team)
  unsigned epoch;
  int pass;
  f2 inv2, l2e2, nz2, lnu2;
  float bcol;
  f2 ac2[P2];  // column accumulators

  __device__ TeamSolver(const DenseArgs& args, unsigned char* smem) : a(args) {
    tid = threadIdx.x % NT;
    team = threadIdx.x / NT;
    ring = reinterpret_cast<float*>(smem) + size_t(team) * STAGES * W;
    gsm = reinterpret_cast<float*>(smem + kRingBytes);
    comb = gsm;
    red = gsm + W + team * kRedTeam;
    misc = gsm + W + TEAMS * kRedTeam;
    full = reinterpret_cast<uint64_t*>(smem + kRingBytes + kRedFloats * sizeof(float)) + team * STAGES;
    b = blockIdx.x;
    G = gridDim.x;
    r0 = int((long long)b * a.n / G);
    r1 = int((long long)(b + 1) * a.n / G);
    rows = r1 - r0;
    rows_t = (rows + 1 - team) / 2;  // positions team, team + 2, ... of the CTA's row sequence
    iss_st = iss_pass = iss_k = 0;
    head_st = head_ph = 0;
    epoch = 0;
    pass = 0;
    inv2 = pk2(a.inv_eps, a.inv_eps);
    l2e2 = pk2(kLog2e, kLog2e);
    nz2 = pk2(a.negzero, a.negzero);
  }

  __device__ __forceinline__ void team_bar() const { named_bar(1 + team, NT); }
  __device__ __forceinline__ int col(int v, int q) const { return 4 * (v * NT + tid) + q; }
  // row of this team's k-th step in pass P (passes alternate the sweep direction)
  __device__ __forceinline__ int row_at(int P, int k) const {
    const int q = team + 2 * k;
    return (P & 1) ? (r1 - 1 - q) : (r0 + q);
  }

  // ---------------- per-team TMA ring
  __device__ __forceinline__ void issue_next() {  // team thread 0
    const uint32_t bytes = uint32_t(a.mpad) * 4u;
    const int i = row_at(iss_pass, iss_k);
    mbar_expect_tx(&full[iss_st], bytes);
    tma_load_1d(ring + size_t(iss_st) * W, a.C + (long long)i * a.ldc, bytes, &full[iss_st]);
#ifdef LSK_X_TEAM_PF
    {  // L2 prefetch of the row LSK_X_TEAM_PF positions further in this team's sequence
      int P = iss_pass, k = iss_k + LSK_X_TEAM_PF;
      while (k >= rows_t) { k -= rows_t; ++P; }
      prefetch_l2(a.C + (long long)row_at(P, k) * a.ldc, bytes);
    }
#endif
    iss_st = (iss_st + 1 == STAGES) ? 0 : iss_st + 1;
    if (++iss_k == rows_t) { iss_k = 0; ++iss_pass; }
  }
  __device__ void ring_init() {
    float4* r4 = reinterpret_cast<float4*>(ring);  // columns >= mpad are never written by TMA
    for (size_t k = tid; k < size_t(STAGES) * W / 4; k += NT) r4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid == 0) {
      for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async();
      for (int s = 0; s < STAGES; ++s) issue_next();
    }
  }
  __device__ __forceinline__ const float* wait_head() {
#ifndef LSK_X_T_NOWAIT
    mbar_wait(&full[head_st], uint32_t(head_ph));
#endif
    const float* p = ring + size_t(head_st) * W;
    if (++head_st == STAGES) { head_st = 0; head_ph ^= 1; }
    return p;
  }
  // refill the oldest held stage (call after a team barrier that follows every read of it)
  __device__ __forceinline__ void release() {
    if (tid == 0) {
      fence_proxy_async();
      issue_next();
    }
  }
  __device__ void drain() {
    for (int s = 0; s < STAGES; ++s) wait_head();
    __syncthreads();
  }

  // ---------------- row data
  __device__ __forceinline__ void load_row(const float* base, f2 (&c)[P2]) const {
#pragma unroll
    for (int v = 0; v < V; ++v) lds2x2(base + 4 * (v * NT + tid), c[2 * v], c[2 * v + 1]);
  }
  // g of the owned columns 4(v NT + tid) .. +3 as two packed pairs
  __device__ __forceinline__ void ldg4(int v, f2& lo, f2& hi) const { lds2x2(gsm + 4 * (v * NT + tid), lo, hi); }
  __device__ void load_lognu() {
    const float L = __ldg(a.log_nu);
    lnu2 = pk2(L, L);
    bcol = -__fmul_rn(L, kLog2e);
  }
  // g^{k-1} into the CTA's shared copy (every thread of both teams; padded
  // columns -inf so every argument there is -inf), the accumulators to zero;
  // returns "some g this thread loaded is non-finite"
  __device__ bool load_columns(const float* g) {
    bool bad = false;
    __syncthreads();  // every read of the previous copy (and of the combine scratch) is done
    for (int q = threadIdx.x; q < W / 4; q += NTB) {
      const int j0 = 4 * q;
      float4 t4 = j0 < a.m ? ldcg4(reinterpret_cast<const float4*>(g + j0)) : make_float4(0.f, 0.f, 0.f, 0.f);
      float t[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u >= a.m) t[u] = 0.f;
        bad |= !isfinite(t[u]);
        if (j0 + u >= a.m) t[u] = -INFINITY;
      }
      reinterpret_cast<float4*>(gsm)[q] = make_float4(t[0], t[1], t[2], t[3]);
    }
#pragma unroll
    for (int p = 0; p < P2; ++p) ac2[p] = 0ull;
    __syncthreads();
    return bad;
  }

  // ---------------- team reductions (exact paths)
  __device__ __forceinline__ float team_max1(float v) {
    const int lane = tid & 31, w = tid >> 5;
    v = warp_max(v);
    if (lane == 0) red[4 * NW + w] = v;
    team_bar();
    const float t = lane < NW ? red[4 * NW + lane] : -INFINITY;
    v = warp_max(t);
    team_bar();
    return v;
  }
  __device__ __forceinline__ float team_sum1(float v) {
    const int lane = tid & 31, w = tid >> 5;
    v = warp_sum(v);
    if (lane == 0) red[4 * NW + w] = v;
    team_bar();
    const float t = lane < NW ? red[4 * NW + lane] : 0.f;
    v = warp_sum(t);
    team_bar();
    return v;
  }
  // 4 consecutive owned columns (pairs 2v, 2v+1) of a row: smem stage or global (zeros beyond m)
  template <bool GL>
  __device__ __forceinline__ void ld4(const float* base, int v, f2& lo, f2& hi) const {
    if constexpr (GL) {
      const int j0 = col(v, 0);
      const float4 t = j0 < a.m ? __ldg(reinterpret_cast<const float4*>(base + j0)) : make_float4(0.f, 0.f, 0.f, 0.f);
      lo = pk2(t.x, t.y);
      hi = pk2(t.z, t.w);
    } else {
      lds2x2(base + 4 * (v * NT + tid), lo, hi);
    }
  }
  // exact two-pass LSE of the f argument (CHK: the check argument with f_i = fi)
  // over a row streamed twice from smem or global memory (nothing held across
  // the max pass, so the rare global-row fallback keeps the register budget)
  template <bool GL, bool CHK>
  __device__ void exact_lse(const float* base, float fi, float& M, float& S) {
    const f2 f2i = pk2(fi, fi);
    float mx = -INFINITY;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      f2 c[2], gg[2];
      ld4<GL>(base, v, c[0], c[1]);
      ldg4(v, gg[0], gg[1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float x0, x1;
        up2(CHK ? arg4x2(f2i, gg[h], c[h], inv2, lnu2, nz2) : arg3x2(gg[h], c[h], inv2, lnu2, nz2), x0, x1);
        mx = fmax_nan(mx, fmax_nan(x0, x1));
      }
    }
    M = team_max1(mx);
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    const f2 nsl = pk2(-__fmul_rn(Ms, kLog2e), -__fmul_rn(Ms, kLog2e));
    f2 s2 = 0ull;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      f2 c[2], gg[2];
      ld4<GL>(base, v, c[0], c[1]);
      ldg4(v, gg[0], gg[1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const f2 x = CHK ? arg4x2(f2i, gg[h], c[h], inv2, lnu2, nz2) : arg3x2(gg[h], c[h], inv2, lnu2, nz2);
        s2 = add2(s2, ex2x2(fma2(x, l2e2, nsl)));
      }
    }
    float s0, s1;
    up2(s2, s0, s1);
    S = team_sum1(s0 + s1);
  }
  __device__ __forceinline__ const float* grow(int i) const { return a.C + (long long)i * a.ldc; }

  static __device__ __forceinline__ bool shift_ok(float S) { return S >= kShiftLo && S <= kShiftHi; }
  __device__ __forceinline__ float sum_warps(int off) const {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; w += 4) {
      const float4 t = *reinterpret_cast<const float4*>(red + off + w);
      s += (t.x + t.y) + (t.z + t.w);
    }
    return s;
  }

  // ================= the team row step =================
  // f-side terms e of a smem row (stale shift fl(-f^{k-1}_i inv_eps)), their
  // sum, and with CHECK the check sum of iterate k-1 (shift 0)
  template <bool CHECK>
  __device__ __forceinline__ void f_part_e(const float* row, float fold, float& s, float& z, f2 (&e)[P2]) const {
    const float shl = __fmul_rn(__fmul_rn(-fold, a.inv_eps), kLog2e);
    const f2 nsl = pk2(-shl, -shl);
    const f2 fo2 = pk2(fold, fold);
    f2 s2 = 0ull, z2 = 0ull;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      f2 c[2], gg[2];
      ld4<false>(row, v, c[0], c[1]);
      ldg4(v, gg[0], gg[1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * v + h;
#ifndef LSK_X_T_NOMUFU
        e[p] = ex2x2(fma2(arg3x2(gg[h], c[h], inv2, lnu2, nz2), l2e2, nsl));
#else
        e[p] = fma2(arg3x2(gg[h], c[h], inv2, lnu2, nz2), l2e2, nsl);
#endif
        s2 = add2(s2, e[p]);
        if (CHECK) z2 = add2(z2, ex2x2(mul2(arg4x2(fo2, gg[h], c[h], inv2, lnu2, nz2), l2e2)));
      }
    }
    float s0, s1;
    up2(s2, s0, s1);
    s = s0 + s1;
    if (CHECK) {
      up2(z2, s0, s1);
      z = s0 + s1;
    }
  }
  // f of row i from its posted sum; the (rare, team-uniform) out-of-band sum
  // falls back to the exact row LSE from global memory
  __device__ __forceinline__ float finish_f(int i, float fold, float S) {
    float M = __fmul_rn(-fold, a.inv_eps);
    float fr = __fmul_rn(a.neg_eps, lse_finish(M, S));
    if (__builtin_expect(!shift_ok(S), 0)) {
      if (tid == 0) atomicAdd(a.stats + 0, 1);
      exact_lse<true, false>(grow(i), 0.f, M, S);
      fr = __fmul_rn(a.neg_eps, lse_finish(M, S));
    }
    return fr;
  }
  __device__ __forceinline__ void check_row(int i, float fold, float lmu, float Sz, float& err_acc, int& bad) {
    float Mz = 0.f;
    if (__builtin_expect(!shift_ok(Sz), 0)) exact_lse<true, true>(grow(i), fold, Mz, Sz);
    if (tid == 0) {
      const float rr = expf(__fadd_rn(lmu, lse_finish(Mz, Sz)));
      err_acc += fabsf(__fsub_rn(rr, __ldg(a.mu + i)));
      if (!isfinite(fold)) bad = 1;
    }
  }
  // column update of row i: g-side terms = f-side terms x 2^(a_i + b) (see
  // DenseSolver::fused_pass_mult); outside the band the direct reference
  // arithmetic from the row re-read from global memory
  __device__ __forceinline__ void col_update(int i, float fi, float fold, float lmu, const f2 (&e)[P2]) {
    const float ai = __fmul_rn(__fadd_rn(__fmul_rn(__fsub_rn(fi, fold), a.inv_eps), lmu), kLog2e);
    if (a.mult && ai >= -100.f && ai + bcol <= 23.f) {
      const float A = ex2(ai + bcol);
      const f2 A2 = pk2(A, A);
#pragma unroll
      for (int p = 0; p < P2; ++p) ac2[p] = fma2(e[p], A2, ac2[p]);
    } else {
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        f2 c[2], gg[2];
        ld4<true>(grow(i), v, c[0], c[1]);
        ldg4(v, gg[0], gg[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int p = 2 * v + h;
          // the stale column shift fl(-g_j inv_eps) log2 e, negated (sign-symmetric rounding)
          const f2 nsc = mul2(mul2(gg[h], inv2), l2e2);
          ac2[p] = add2(ac2[p], ex2x2(fma2(arg3x2(fi2, c[h], inv2, lm2, nz2), l2e2, nsc)));
        }
      }
    }
  }
  __device__ __forceinline__ void post(int k, float s, float z, bool check) {
    const int lane = tid & 31, w = tid >> 5;
    s = warp_sum(s);
    if (check) z = warp_sum(z);
    if (lane == 0) {
      red[(k & 1) * NW + w] = s;
      if (check) red[2 * NW + (k & 1) * NW + w] = z;
    }
  }

  template <bool CHECK>
  __device__ void team_pass(const float* fprev, float* fnew, float& err_acc, int& bad) {
    const int P = pass++;
    int i_cur = row_at(P, 0);
    float fold_cur = ldcg(fprev + i_cur), lmu_cur = __ldg(a.log_mu + i_cur);
    int i_nx = rows_t > 1 ? row_at(P, 1) : i_cur;
    float fold_nx = rows_t > 1 ? ldcg(fprev + i_nx) : fold_cur;
    float lmu_nx = rows_t > 1 ? __ldg(a.log_mu + i_nx) : lmu_cur;
    f2 e[P2];
    float s, z = 0.f;
    f_part_e<CHECK>(wait_head(), fold_cur, s, z, e);
    post(0, s, z, CHECK);
    int i_prev = i_cur;
    float fold_prev = fold_cur, lmu_prev = lmu_cur;
    for (int k = 1; k < rows_t; ++k) {
      i_cur = i_nx; fold_cur = fold_nx; lmu_cur = lmu_nx;
      if (k + 1 < rows_t) {
        i_nx = row_at(P, k + 1);
        fold_nx = ldcg(fprev + i_nx);
        lmu_nx = __ldg(a.log_mu + i_nx);
      }
      const float* row = wait_head();
#ifndef LSK_X_T_NOBAR
      team_bar();  // row k-1's sums are posted; every warp is done with row k-1's stage
#endif
      release();
      const int pb = (k - 1) & 1;
#ifndef LSK_X_T_NOFIN
      const float f_prev = finish_f(i_prev, fold_prev, sum_warps(pb * NW));
#else
      const float f_prev = fold_prev + 1e-9f * sum_warps(pb * NW);
#endif
      if (CHECK) check_row(i_prev, fold_prev, lmu_prev, sum_warps(2 * NW + pb * NW), err_acc, bad);
      if (tid == 0) fnew[i_prev] = f_prev;
      col_update(i_prev, f_prev, fold_prev, lmu_prev, e);
      f_part_e<CHECK>(row, fold_cur, s, z, e);
      post(k, s, z, CHECK);
      i_prev = i_cur; fold_prev = fold_cur; lmu_prev = lmu_cur;
    }
    team_bar();
    release();
    const int pb = (rows_t - 1) & 1;
    const float f_last = finish_f(i_prev, fold_prev, sum_warps(pb * NW));
    if (CHECK) check_row(i_prev, fold_prev, lmu_prev, sum_warps(2 * NW + pb * NW), err_acc, bad);
    if (tid == 0) fnew[i_prev] = f_last;
    col_update(i_prev, f_last, fold_prev, lmu_prev, e);
  }

  // ================= cold passes (each team takes its rows) =================
  __device__ void row_exact_pass(float* fnew) {
    const int P = pass++;
    for (int k = 0; k < rows_t; ++k) {
      const int i = row_at(P, k);
      float M, S;
      exact_lse<false, false>(wait_head(), 0.f, M, S);  // its team barriers order every read of the stage before the refill
      if (tid == 0) fnew[i] = __fmul_rn(a.neg_eps, lse_finish(M, S));
      release();
    }
  }
  __device__ void check_pass(const float* f, float& err_acc, int& bad) {
    const int P = pass++;
    for (int k = 0; k < rows_t; ++k) {
      const int i = row_at(P, k);
      const float* row = wait_head();
      const float fold = ldcg(f + i);
      const f2 fo2 = pk2(fold, fold);
      f2 z2 = 0ull;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        f2 c[2], gg[2];
        ld4<false>(row, v, c[0], c[1]);
        ldg4(v, gg[0], gg[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) z2 = add2(z2, ex2x2(mul2(arg4x2(fo2, gg[h], c[h], inv2, lnu2, nz2), l2e2)));
      }
      float s0, s1;
      up2(z2, s0, s1);
      const float Sz = team_sum1(s0 + s1);
      check_row(i, fold, __ldg(a.log_mu + i), Sz, err_acc, bad);
      team_bar();
      release();
    }
  }
  __device__ void cost_pass(const float* f, float& cost_acc) {
    const int P = pass++;
    for (int k = 0; k < rows_t; ++k) {
      const int i = row_at(P, k);
      const float* row = wait_head();
      const float fi = ldcg(f + i), lmu = __ldg(a.log_mu + i);
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
      float s = 0.f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        f2 c[2], gg[2];
        ld4<false>(row, v, c[0], c[1]);
        ldg4(v, gg[0], gg[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const f2 zz = add2(arg4x2(fi2, gg[h], c[h], inv2, lm2, nz2), lnu2);
          float z0, z1, c0, c1;
          up2(zz, z0, z1);
          up2(c[h], c0, c1);
          s += __fmul_rn(c0, expf(z0));
          s += __fmul_rn(c1, expf(z1));
        }
      }
      const float S = team_sum1(s);
      if (tid == 0) cost_acc += S;
      release();
    }
  }
  // exact online (max, sumexp) of the beta argument per owned column over the
  // team's rows; team 1's pairs are merged into team 0's (fixed order) -> a.pairs[b]
  __device__ void col_exact_pass(const float* f) {
    const int P = pass++;
    float cm[E], cs[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { cm[e] = -INFINITY; cs[e] = 0.f; }
    for (int k = 0; k < rows_t; ++k) {
      const int i = row_at(P, k);
      const float* row = wait_head();
      const float fi = ldcg(f + i), lmu = __ldg(a.log_mu + i);
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lmu, lmu);
#pragma unroll
      for (int p = 0; p < P2; ++p) {
        f2 c0, c1;
        if (p & 1) continue;
        ld4<false>(row, p / 2, c0, c1);
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {
        const int pp = p + hp;
        float y[2];
        up2(arg3x2(fi2, hp ? c1 : c0, inv2, lm2, nz2), y[0], y[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = 2 * pp + h;
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
      team_bar();
      release();
    }
    float2* scr = reinterpret_cast<float2*>(a.scratch) + (size_t)b * W;  // team 1 -> scratch
    __syncthreads();
    if (team == 1) {
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int q = 0; q < 4; ++q) scr[col(v, q)] = make_float2(cm[4 * v + q], cs[4 * v + q]);
    }
    __syncthreads();
    if (team == 0) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int j0 = col(v, 0);
        if (j0 >= a.m) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float m0 = cm[4 * v + q], s0 = cs[4 * v + q];
          const float2 o = __ldcg(scr + j0 + q);
          pair_merge(m0, s0, o.x, o.y);
          a.pairs[(size_t)b * W + j0 + q] = make_float2(m0, s0);
        }
      }
    }
  }

  // ---- the two teams' column accumulators: team 0 + team 1 -> a.part[b]
  __device__ void store_stale_partials() {
    float4* scr = reinterpret_cast<float4*>(a.scratch + (size_t)b * 2 * W);
    __syncthreads();
    if (team == 1) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float x0, x1, x2, x3;
        up2(ac2[2 * v], x0, x1);
        up2(ac2[2 * v + 1], x2, x3);
        scr[v * NT + tid] = make_float4(x0, x1, x2, x3);
      }
    }
    __syncthreads();
    if (team == 0) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (col(v, 0) >= a.m) continue;
        const float4 o = __ldcg(scr + v * NT + tid);
        const f2 s0 = add2(ac2[2 * v], pk2(o.x, o.y)), s1 = add2(ac2[2 * v + 1], pk2(o.z, o.w));
        float x0, x1, x2, x3;
        up2(s0, x0, x1);
        up2(s1, x2, x3);
        reinterpret_cast<float4*>(a.part + (size_t)b * W)[v * NT + tid] = make_float4(x0, x1, x2, x3);
      }
    }
  }

  // ---- grid-wide pieces (all NTB threads)
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
  // column combine: CTA b owns columns [b m/G, (b+1) m/G); threads are
  // (column, slice) pairs, slice q sums partial rows q, q + QS, ... with all
  // loads in flight, then one thread per column adds the slices in order
  __device__ void combine_stale(const float* gold, float* gnew, int k) {
    const int j0 = int((long long)b * a.m / G), j1 = int((long long)(b + 1) * a.m / G);
    const int nc = j1 - j0;
    float* cr = comb;
    const int QS = nc > 0 ? min(NTB / nc, kRedComb / nc) : 1;
    const int t = threadIdx.x;
    bool fired = false;
    if (nc > 0 && QS >= 1 && t < QS * nc) {
      const int c = t % nc, q = t / nc, j = j0 + c;
      constexpr int KB = 16;
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
    const float gj = (t < nc) ? ldcg(gold + j0 + t) : 0.f;
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
    float* cr = comb;
    for (int grp = b; grp < ngroups; grp += G) {
      const int j = grp * 32 + lane;
      const int k0 = w * G / NWB, k1 = (w + 1) * G / NWB;
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
        for (int h = NWB / 2; h >= 1; h >>= 1)
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
  // both teams' thread-0 check scalars, added in team order
  __device__ void publish_check(float err_acc, int bad) {
    bad = __syncthreads_or(bad);
    if (threadIdx.x == NT) misc[0] = err_acc;
    __syncthreads();
    if (threadIdx.x == 0) { a.errpart[b] = err_acc + misc[0]; a.flagpart[b] = bad; }
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
      const bool fused = k > 1;  // the host selects this kernel for the stale-shift iteration only
      if (fused) {
#ifndef XP_NOCHECK
        if (do_check) team_pass<true>(fb((k - 1) & 1), fb(k & 1), err_acc, bad);
#else
        if (do_check) team_pass<false>(fb((k - 1) & 1), fb(k & 1), err_acc, bad);
#endif
        else team_pass<false>(fb((k - 1) & 1), fb(k & 1), err_acc, bad);
        store_stale_partials();
      } else {
        row_exact_pass(fb(k & 1));
      }
      if (do_check) publish_check(err_acc, bad);
      grid_barrier(a.bar, epoch);
      if (do_check && decide(k - 1, failed)) { stopped = true; final_k = k - 1; break; }
      if (fused) {
        combine_stale(gcur, gb(k & 1), k);
        grid_barrier(a.bar, epoch);
      }
      const bool need_exact = !fused || (__ldcg(a.guard) == k);
      if (need_exact) {
        if (threadIdx.x == 0 && b == 0 && fused) atomicAdd(a.stats + 1, 1);
#ifndef XP_NOCOLX
        col_exact_pass(fb(k & 1));
#endif
        grid_barrier(a.bar, epoch);
        combine_pairs(gb(k & 1));
        grid_barrier(a.bar, epoch);
      }
    }
    if (!stopped) {
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
      if (threadIdx.x == NT) misc[1] = cost_acc;
      __syncthreads();
      if (threadIdx.x == 0) a.costpart[b] = cost_acc + misc[1];
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

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
//  * CTA b owns rows [b*n/G, (b+1)*n/G). Thread t owns columns
//    j = 4*(v*NT + t) + q (v < V, q < 4) for the whole solve, so per-column
//    state (g_j, log nu_j, the column shift, the column accumulator) lives in
//    registers and each smem row read is one conflict-free LDS.128 per v.
//  * Rows stream HBM -> smem through a STAGES-deep ring of TMA bulk copies
//    (cp.async.bulk + mbarrier complete_tx). Each pass alternates the sweep
//    direction, so the rows read last by one pass are L2-hot for the next.
//  * ONE pass over C per iteration: from the on-chip row the CTA computes
//    f_i^k (row LSE against g^{k-1}), then -- from the same registers --
//    adds exp(y_ij - s_j) into its per-column accumulators, where
//    y_ij = fl(fl(fl(f_i^k - C_ij) * inv_eps) + log mu_i) is the reference's
//    beta argument and s_j = fl(-g_j^{k-1} * inv_eps) a stale shift
//    (the terms are bounded by mu_i / nu_j, so no overflow). A
//    grid-wide combine sums the G partials per column in a fixed tree and
//    forms g^k. The row LSE uses the stale row shift fl(-f_i^{k-1}*inv_eps)
//    likewise. Sums outside [1e-20, 1e30] fall back to the exact max shift
//    (rows: in registers; columns: an exact (max, sumexp) column pass).
//  * Every c iterations the row pass of k+1 also evaluates the reference
//    marginal-error formula for iterate k (solver.py:97-104) from the same
//    on-chip row -- no extra HBM pass, no host sync; f/g are double
//    buffered so a stop at k returns iterate k.
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
  double tol;
  int max_iter, check, stale, want_cost;
  // workspace (zero-initialised by the host where noted)
  float* f0; float* f1;  // f^k lives in f[k & 1]; f0 = 0 on entry
  float* g0; float* g1;  // g^k lives in g[k & 1]; g0 = 0 on entry
  float* part;           // [G][W] stale column partial sums
  float2* pairs;         // [G][W] exact column (max, sumexp) partials
  float* errpart;        // [G]
  int* flagpart;         // [G]
  float* costpart;       // [G]
  unsigned* bar;         // grid barrier counter (zeroed)
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

enum PassKind { kPassRow = 0, kPassColExact = 1, kPassCheck = 2, kPassCost = 3 };

template <int NT, int V, int R, int STAGES>
struct DenseSolver {
  static constexpr int E = 4 * V;       // columns per thread
  static constexpr int W = 4 * V * NT;  // row capacity (floats)
  static constexpr int NW = NT / 32;
  static constexpr size_t kRingBytes = size_t(STAGES) * R * W * sizeof(float);
  static constexpr size_t kRedFloats = 64 * 2 * R + 64 + NW * 64;
  static constexpr size_t kSmemBytes = kRingBytes + kRedFloats * sizeof(float) + STAGES * 8 + 64;

  // ---- per-CTA state
  const DenseArgs& a;
  float* ring;
  float* red;
  uint64_t* mbar;
  int b, G, r0, r1, rows, nb;     // rows of this CTA, batches per pass
  long long issued, consumed;     // global batch counters of the TMA ring
  unsigned epoch;
  int pass;                       // pass counter (sweep direction = pass & 1)

  // ---- per-thread column state
  float gcol[E], lnu[E], gsl[E], acc[E];

  __device__ DenseSolver(const DenseArgs& args, unsigned char* smem) : a(args) {
    ring = reinterpret_cast<float*>(smem);
    red = reinterpret_cast<float*>(smem + kRingBytes);
    mbar = reinterpret_cast<uint64_t*>(smem + kRingBytes + kRedFloats * sizeof(float));
    b = blockIdx.x;
    G = gridDim.x;
    r0 = int((long long)b * a.n / G);
    r1 = int((long long)(b + 1) * a.n / G);
    rows = r1 - r0;
    nb = (rows + R - 1) / R;
    issued = consumed = 0;
    epoch = 0;
    pass = 0;
  }

  __device__ __forceinline__ int col(int v, int q) const { return 4 * (v * NT + threadIdx.x) + q; }

  // row index of slot r of within-pass batch qb in pass P
  __device__ __forceinline__ int row_of(int P, int qb, int r) const {
    int idx = qb * R + r;
    if (idx >= rows) return -1;
    return (P & 1) ? (r1 - 1 - idx) : (r0 + idx);
  }

  // producer (thread 0): issue global batch p into its ring stage
  __device__ void issue(long long p) {
    const int st = int(p % STAGES);
    const int P = int(p / nb), qb = int(p % nb);
    const uint32_t bytes = uint32_t(a.mpad) * 4u;
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) cnt += row_of(P, qb, r) >= 0;
    mbar_expect_tx(&mbar[st], bytes * cnt);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int i = row_of(P, qb, r);
      if (i >= 0) tma_load_1d(ring + (size_t(st) * R + r) * W, a.C + (long long)i * a.ldc, bytes, &mbar[st]);
    }
  }

  __device__ void ring_init() {
    // zero the ring once: columns >= mpad are never written by TMA and must read as 0
    float4* r4 = reinterpret_cast<float4*>(ring);
    for (size_t k = threadIdx.x; k < kRingBytes / 16; k += NT) r4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) mbar_init(&mbar[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && nb > 0) {
      fence_proxy_async();
      for (; issued < STAGES; ++issued) issue(issued);
    }
  }

  // wait for batch `consumed`, copy the R rows of this thread's columns to regs
  __device__ __forceinline__ void load_batch(float (&c)[R][E]) {
    const int st = int(consumed % STAGES);
    mbar_wait(&mbar[st], uint32_t((consumed / STAGES) & 1));
    const float* base = ring + size_t(st) * R * W;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float4 t4 = reinterpret_cast<const float4*>(base + size_t(r) * W)[v * NT + threadIdx.x];
        c[r][4 * v + 0] = t4.x; c[r][4 * v + 1] = t4.y; c[r][4 * v + 2] = t4.z; c[r][4 * v + 3] = t4.w;
      }
  }
  // call after a __syncthreads that follows load_batch: the stage is free
  __device__ __forceinline__ void refill() {
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(issued);
      ++issued;
    }
    ++consumed;
  }
  __device__ void drain() {
    if (threadIdx.x == 0)
      for (long long p = consumed; p < issued; ++p)
        mbar_wait(&mbar[int(p % STAGES)], uint32_t((p / STAGES) & 1));
    __syncthreads();
  }

  __device__ void load_columns(const float* g) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      int j0 = 4 * (v * NT + threadIdx.x);
      float4 t4 = j0 < a.m ? ldcg4(reinterpret_cast<const float4*>(g + j0)) : make_float4(0.f, 0.f, 0.f, 0.f);
      float tt[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float gj = (j0 + q < a.m) ? tt[q] : 0.f;
        gcol[4 * v + q] = gj;
        gsl[4 * v + q] = __fmul_rn(__fmul_rn(-gj, a.inv_eps), kLog2e);
        acc[4 * v + q] = 0.f;
      }
    }
  }

  // ---- the exact (max-shifted) row LSE of the f argument, from registers
  __device__ __forceinline__ void exact_row(const float (&c)[R][E], int r, float& M, float& S) {
    float mx[1] = {-INFINITY};
#pragma unroll
    for (int e = 0; e < E; ++e) mx[0] = fmax_nan(mx[0], arg3(gcol[e], c[r][e], a.inv_eps, lnu[e]));
    block_reduce<NT, 1, true>(mx, red + 64 * 2 * R);
    M = mx[0];
    float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    float sl = __fmul_rn(Ms, kLog2e);
    float s[1] = {0.f};
#pragma unroll
    for (int e = 0; e < E; ++e) s[0] += exp_shifted(arg3(gcol[e], c[r][e], a.inv_eps, lnu[e]), sl);
    __syncthreads();  // red reuse
    block_reduce<NT, 1, false>(s, red + 64 * 2 * R);
    S = s[0];
    __syncthreads();
  }
  __device__ __forceinline__ void exact_check_row(const float (&c)[R][E], int r, float fi, float& M, float& S) {
    float mx[1] = {-INFINITY};
#pragma unroll
    for (int e = 0; e < E; ++e) mx[0] = fmax_nan(mx[0], arg4(fi, gcol[e], c[r][e], a.inv_eps, lnu[e]));
    block_reduce<NT, 1, true>(mx, red + 64 * 2 * R);
    M = mx[0];
    float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    float sl = __fmul_rn(Ms, kLog2e);
    float s[1] = {0.f};
#pragma unroll
    for (int e = 0; e < E; ++e) s[0] += exp_shifted(arg4(fi, gcol[e], c[r][e], a.inv_eps, lnu[e]), sl);
    __syncthreads();
    block_reduce<NT, 1, false>(s, red + 64 * 2 * R);
    S = s[0];
    __syncthreads();
  }

  static __device__ __forceinline__ bool shift_ok(float S) { return S >= kShiftLo && S <= kShiftHi; }

  // ---- one streaming pass over this CTA's rows
  // kPassRow:      f^k from g^{k-1} (gcol), stale column partials into acc,
  //                optionally the marginal check of iterate k-1 (fchk = f^{k-1})
  // kPassColExact: exact (max, sumexp) of the beta argument per column (acc=max, gsl=sum)
  // kPassCheck:    marginal check only (fchk = f^k, gcol = g^k)
  // kPassCost:     transport cost (fchk = f, gcol = g)
  template <int KIND>
  __device__ void run_pass(const float* fprev, float* fnew, bool exact_rows, bool do_check,
                           float& err_acc, int& bad_flag, float& cost_acc, bool do_gpart = false) {
    const int P = pass++;
    if (nb == 0) return;
    float c[R][E];
    for (int qb = 0; qb < nb; ++qb) {
      load_batch(c);
      int ri[R];
      float fold[R], lmu_r[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ri[r] = row_of(P, qb, r);
        int i = ri[r] < 0 ? r0 : ri[r];
        fold[r] = ldcg(fprev + i);
        lmu_r[r] = __ldg(a.log_mu + i);
      }
      if (KIND == kPassRow) {
        // --- f-update (+ check) sums
        float S[2 * R];
        float sh[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          sh[r] = exact_rows ? 0.f : __fmul_rn(-fold[r], a.inv_eps);
          S[r] = 0.f;
          S[R + r] = 0.f;
        }
        if (!exact_rows) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float sl = __fmul_rn(sh[r], kLog2e);
            float s = 0.f, sz = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              s += exp_shifted(arg3(gcol[e], c[r][e], a.inv_eps, lnu[e]), sl);
              if (do_check) sz += ex2(__fmul_rn(arg4(fold[r], gcol[e], c[r][e], a.inv_eps, lnu[e]), kLog2e));
            }
            S[r] = s;
            S[R + r] = sz;
          }
          if (do_check) block_reduce<NT, 2 * R, false>(S, red);
          else {
            float S1[R];
#pragma unroll
            for (int r = 0; r < R; ++r) S1[r] = S[r];
            block_reduce<NT, R, false>(S1, red);
#pragma unroll
            for (int r = 0; r < R; ++r) S[r] = S1[r];
          }
        } else {
          if (do_check) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              float sz = 0.f;
#pragma unroll
              for (int e = 0; e < E; ++e)
                sz += ex2(__fmul_rn(arg4(fold[r], gcol[e], c[r][e], a.inv_eps, lnu[e]), kLog2e));
              S[R + r] = sz;
            }
            float S2[R];
#pragma unroll
            for (int r = 0; r < R; ++r) S2[r] = S[R + r];
            block_reduce<NT, R, false>(S2, red);
#pragma unroll
            for (int r = 0; r < R; ++r) S[R + r] = S2[r];
          } else {
            __syncthreads();
          }
        }
        refill();
        __syncthreads();  // red consumed before any exact-path reuse
        float fr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float M = sh[r], Ssum = S[r];
          if (exact_rows || !shift_ok(Ssum)) {
            if (!exact_rows && threadIdx.x == 0 && ri[r] >= 0) atomicAdd(a.stats + 0, 1);
            exact_row(c, r, M, Ssum);
          }
          fr[r] = __fmul_rn(a.neg_eps, lse_finish(M, Ssum));
          if (do_check) {
            float Mz = 0.f, Sz = S[R + r];
            if (!shift_ok(Sz)) exact_check_row(c, r, fold[r], Mz, Sz);
            float L = lse_finish(Mz, Sz);
            float rr = expf(__fadd_rn(lmu_r[r], L));
            if (threadIdx.x == 0 && ri[r] >= 0) {
              err_acc += fabsf(__fsub_rn(rr, __ldg(a.mu + ri[r])));
              if (!isfinite(fold[r])) bad_flag = 1;
            }
          }
          if (threadIdx.x == 0 && ri[r] >= 0) fnew[ri[r]] = fr[r];
        }
        // --- stale-shift column partials of the beta argument, same registers
        if (do_gpart)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (ri[r] < 0) continue;
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] += exp_shifted(arg3(fr[r], c[r][e], a.inv_eps, lmu_r[r]), gsl[e]);
        }
      } else if (KIND == kPassColExact) {
        // chunked online (max, sumexp) per owned column; acc = max, gsl = sum
#pragma unroll
        for (int e = 0; e < E; ++e) {
          float y[R];
          float cm = -INFINITY;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            y[r] = ri[r] >= 0 ? arg3(fold[r], c[r][e], a.inv_eps, lmu_r[r]) : -INFINITY;
            cm = fmax_nan(cm, y[r]);
          }
          float mo = acc[e];
          float mn = fmax_nan(mo, cm);
          float ms = (fabsf(mn) <= 3.402823466e38f) ? mn : 0.f;
          float sl = __fmul_rn(ms, kLog2e);
          float s = (mo == -INFINITY) ? 0.f : gsl[e] * exp_shifted(mo, sl);
#pragma unroll
          for (int r = 0; r < R; ++r) s += exp_shifted(y[r], sl);
          acc[e] = mn;
          gsl[e] = s;
        }
        __syncthreads();
        refill();
      } else if (KIND == kPassCheck) {
        float S[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float sz = 0.f;
#pragma unroll
          for (int e = 0; e < E; ++e) sz += ex2(__fmul_rn(arg4(fold[r], gcol[e], c[r][e], a.inv_eps, lnu[e]), kLog2e));
          S[r] = sz;
        }
        block_reduce<NT, R, false>(S, red);
        refill();
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float Mz = 0.f, Sz = S[r];
          if (!shift_ok(Sz)) exact_check_row(c, r, fold[r], Mz, Sz);
          float L = lse_finish(Mz, Sz);
          float rr = expf(__fadd_rn(lmu_r[r], L));
          if (threadIdx.x == 0 && ri[r] >= 0) {
            err_acc += fabsf(__fsub_rn(rr, __ldg(a.mu + ri[r])));
            if (!isfinite(fold[r])) bad_flag = 1;
          }
        }
      } else {  // kPassCost: sum_ij fl(C_ij * exp(z_ij)), z as solver.py:108-112
        float S[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float s = 0.f;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            float z = __fadd_rn(arg4(fold[r], gcol[e], c[r][e], a.inv_eps, lmu_r[r]), lnu[e]);
            s += __fmul_rn(c[r][e], expf(z));
          }
          S[r] = ri[r] >= 0 ? s : 0.f;
        }
        block_reduce<NT, R, false>(S, red);
        refill();
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) cost_acc += S[r];
        }
      }
    }
  }

  // fixed-order tree over the G per-CTA scalars (identical in every CTA)
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

  // ---- column combines: CTA b handles 32-column groups b, b+G, ...; the
  // NW warps split the G partial rows into contiguous ranges, then a fixed
  // halving tree over the NW range sums (in smem) finishes each column.
  __device__ void combine_stale(const float* gold, float* gnew, int k) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ngroups = (a.m + 31) / 32;
    bool fired = false;
    for (int grp = b; grp < ngroups; grp += G) {
      const int j = grp * 32 + lane;
      const int k0 = w * G / NW, k1 = (w + 1) * G / NW;
      float s = 0.f;
      if (j < a.m)
        for (int kk = k0; kk < k1; ++kk) s += ldcg(a.part + (size_t)kk * W + j);
      red[w * 32 + lane] = s;
      __syncthreads();
      if (w == 0) {
        for (int h = NW / 2; h >= 1; h >>= 1)
          for (int u = 0; u < h; ++u) red[u * 32 + lane] += red[(u + h) * 32 + lane];
        if (j < a.m) {
          float sj = __fmul_rn(-ldcg(gold + j), a.inv_eps);
          float S = red[lane];
          if (!shift_ok(S)) fired = true;
          gnew[j] = __fmul_rn(a.neg_eps, lse_finish(sj, S));
        }
      }
      __syncthreads();
    }
    if (w == 0 && __any_sync(0xffffffffu, fired) && lane == 0) atomicMax(a.guard, k);
  }

  __device__ void combine_pairs(float* gnew) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ngroups = (a.m + 31) / 32;
    for (int grp = b; grp < ngroups; grp += G) {
      const int j = grp * 32 + lane;
      const int k0 = w * G / NW, k1 = (w + 1) * G / NW;
      float mx = -INFINITY, s = 0.f;
      if (j < a.m)
        for (int kk = k0; kk < k1; ++kk) {
          float2 p = __ldcg(a.pairs + (size_t)kk * W + j);
          pair_merge(mx, s, p.x, p.y);
        }
      red[w * 64 + lane] = mx;
      red[w * 64 + 32 + lane] = s;
      __syncthreads();
      if (w == 0) {
        for (int h = NW / 2; h >= 1; h >>= 1)
          for (int u = 0; u < h; ++u) {
            float m1 = red[u * 64 + lane], s1 = red[u * 64 + 32 + lane];
            pair_merge(m1, s1, red[(u + h) * 64 + lane], red[(u + h) * 64 + 32 + lane]);
            red[u * 64 + lane] = m1;
            red[u * 64 + 32 + lane] = s1;
          }
        if (j < a.m) gnew[j] = __fmul_rn(a.neg_eps, lse_finish(red[lane], red[32 + lane]));
      }
      __syncthreads();
    }
  }

  __device__ void store_partials(bool pairs_mode) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int j0 = 4 * (v * NT + threadIdx.x);
      if (j0 >= a.m) continue;
      if (pairs_mode) {
        float2* dst = a.pairs + (size_t)b * W + j0;
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_float2(acc[4 * v + q], gsl[4 * v + q]);
      } else {
        reinterpret_cast<float4*>(a.part + (size_t)b * W)[v * NT + threadIdx.x] =
            make_float4(acc[4 * v], acc[4 * v + 1], acc[4 * v + 2], acc[4 * v + 3]);
      }
    }
  }

  // ---- check decision, identical in every CTA (solver.py:286-300)
  // returns true if the solve stops at iterate kk
  __device__ bool decide(int kk, bool& failed, float& err_out) {
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
    err_out = e;
    return stop;
  }

  __device__ void solve() {
    const float* gcur;
    // per-thread log nu for owned columns (-inf masks columns >= m)
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int j = col(v, q);
        lnu[4 * v + q] = j < a.m ? __ldg(a.log_nu + j) : -INFINITY;
      }
    ring_init();
    auto fb = [&](int k) { return (k & 1) ? a.f1 : a.f0; };
    auto gb = [&](int k) { return (k & 1) ? a.g1 : a.g0; };
    int final_k = a.max_iter;
    bool stopped = false, failed = false;
    float err_dummy = 0.f;
    for (int k = 1; k <= a.max_iter; ++k) {
      const bool do_check = (k > 1) && ((k - 1) % a.check == 0);
      gcur = gb((k - 1) & 1);
      load_columns(gcur);
      float err_acc = 0.f, cost_dummy = 0.f;
      int bad = 0;
      if (do_check) {
        // finiteness of g^{k-1} on this CTA's view (every CTA holds all of g)
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (!isfinite(gcol[e]) && col(e / 4, e % 4) < a.m) bad = 1;
      }
      const bool exact_rows = (k == 1) || !a.stale;
      run_pass<kPassRow>(fb((k - 1) & 1), fb(k & 1), exact_rows, do_check, err_acc, bad, cost_dummy,
                         a.stale && k > 1);
      if (do_check) {
        bad = __syncthreads_or(bad);
        if (threadIdx.x == 0) { a.errpart[b] = err_acc; a.flagpart[b] = bad; }
      }
      if (a.stale && k > 1) store_partials(false);
      grid_barrier(a.bar, epoch);
      if (do_check) {
        float e;
        if (decide(k - 1, failed, e)) { stopped = true; final_k = k - 1; break; }
      }
      if (a.stale && k > 1) {
        combine_stale(gcur, gb(k & 1), k);
        grid_barrier(a.bar, epoch);
      }
      const bool need_exact = !a.stale || k == 1 || (__ldcg(a.guard) == k);
      if (need_exact) {
        if (threadIdx.x == 0 && b == 0 && a.stale && k > 1) atomicAdd(a.stats + 1, 1);
#pragma unroll
        for (int e = 0; e < E; ++e) { acc[e] = -INFINITY; gsl[e] = 0.f; }
        run_pass<kPassColExact>(fb(k & 1), nullptr, false, false, err_dummy, bad, cost_dummy);
        store_partials(true);
        grid_barrier(a.bar, epoch);
        combine_pairs(gb(k & 1));
        grid_barrier(a.bar, epoch);
      }
    }
    if (!stopped) {
      // the final check at the cap (solver.py:286-316: in-loop if K % c == 0, else the extra one)
      final_k = a.max_iter;
      load_columns(gb(final_k & 1));
      float err_acc = 0.f, cost_dummy = 0.f;
      int bad = 0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (!isfinite(gcol[e]) && col(e / 4, e % 4) < a.m) bad = 1;
      run_pass<kPassCheck>(fb(final_k & 1), nullptr, false, true, err_acc, bad, cost_dummy);
      bad = __syncthreads_or(bad);
      if (threadIdx.x == 0) { a.errpart[b] = err_acc; a.flagpart[b] = bad; }
      grid_barrier(a.bar, epoch);
      float e;
      decide(final_k, failed, e);
    }
    const int fbuf = final_k & 1;
    if (!failed && a.want_cost) {
      load_columns(gb(fbuf));
      float err_acc = 0.f, cost_acc = 0.f;
      int bad = 0;
      run_pass<kPassCost>(fb(fbuf), nullptr, false, false, err_acc, bad, cost_acc);
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

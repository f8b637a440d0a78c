// Dense persistent solver, task-queue variant ("v4"), m <= 8192.
//
// Same iteration, arithmetic contract and results as lsk_dense.cuh (the
// reference solve, solver.py:230-337), organised so that no per-row work is
// replicated across the warps of a CTA:
//  * an F task = one row, owned by ONE warp: lanes stream the row from HBM
//    (128-bit loads, lane l takes columns 128 t + 4 l) against g^{k-1} and
//    log nu staged in shared memory; the row sum is a warp butterfly and the
//    finish (logf, guard, check term) is done once, by that warp;
//  * a G task = one 128-column strip of one 64-row slice: lanes own 4 columns
//    and walk the slice's rows in row order (the rows are still in L2: the F
//    tasks of that slice ran one phase earlier), producing the slice's column
//    partial sums of the beta argument with the stale column shift;
//  * tasks are taken from a global counter in a fixed phase order
//    F(slice p) | G(slice p-1) | F(slice p+1) | ...; a G task waits on its
//    slice's row counter (release/acquire), which is normally long complete;
//  * the column partials of the S slices are combined in a fixed order
//    (deterministic) between the two grid barriers of each iteration.
// Row/column results depend only on fixed orders, never on which warp ran
// which task: bit-identical run to run.
#pragma once
#include "lsk_device.cuh"

namespace lsk {

struct D4Args {
  const float* C;
  long long ldc;
  int n, m, mpad;
  const float* log_mu;
  const float* log_nu;
  const float* mu;
  float inv_eps, neg_eps, negzero;
  double tol;
  int max_iter, check, stale, want_cost;
  float* f0; float* f1;
  float* g0; float* g1;
  float* part;          // [S][mpad] stale column partials
  float2* pairs;        // [S][mpad] exact column (max, sumexp) partials
  float* rowterm;       // [n] per-row check / cost terms
  unsigned* rows_done;  // [S] monotonic per-slice F completion counters (zeroed)
  unsigned* tctr;       // [2] task counters (zeroed)
  unsigned long long* bar;
  int* guard;
  int* stats;
  int* out_status;
  int* out_iters;
  float* out_err;
  float* out_cost;
  int* out_fbuf;
  int* trace_iter;
  float* trace_err;
  int* n_trace;
};

template <int NT, int WMAX>
struct DenseV4 {
  static constexpr int NW = NT / 32;
  static constexpr int SR = 64;      // rows per slice
  static constexpr int STRIP = 128;  // columns per G task (4 per lane)
  static constexpr size_t kSmemBytes = size_t(WMAX) * 8 + 64 * NW * 4 + 256;  // g, log nu, scratch, flags

  const D4Args& a;
  float* gsm;     // [WMAX] g^{k-1}
  float* lnusm;   // [WMAX] log nu (-inf beyond m)
  float* red;     // [64*NW] combine scratch
  unsigned* cta_flag;
  int b, G, S, T, lane, w;
  unsigned epoch;
  unsigned npass;     // passes run so far (slice counter targets, sweep direction)
  unsigned flags_seen;
  f2 inv2, l2e2, nz2;

  __device__ DenseV4(const D4Args& args, unsigned char* smem) : a(args) {
    gsm = reinterpret_cast<float*>(smem);
    lnusm = gsm + WMAX;
    red = lnusm + WMAX;
    cta_flag = reinterpret_cast<unsigned*>(red + 64 * NW);
    b = blockIdx.x;
    G = gridDim.x;
    S = (a.n + SR - 1) / SR;
    T = (a.mpad + STRIP - 1) / STRIP;
    lane = threadIdx.x & 31;
    w = threadIdx.x >> 5;
    epoch = 0;
    npass = 0;
    flags_seen = 0;
    inv2 = pk2(a.inv_eps, a.inv_eps);
    l2e2 = pk2(kLog2e, kLog2e);
    nz2 = pk2(a.negzero, a.negzero);
  }

  // ---------------- task sequence of one pass
  // phase 0: F(sl(0)) ; phase p in 1..S-1: F(sl(p)) then G(sl(p-1)) ; phase S: G(sl(S-1))
  __device__ __forceinline__ int slice_of(int p, unsigned P) const { return (P & 1) ? (S - 1 - p) : p; }
  __device__ __forceinline__ int tasks_total(bool with_g) const { return with_g ? S * SR + S * T : S * SR; }
  // decode task t -> (is_f, slice, index)
  __device__ __forceinline__ void decode(int t, bool with_g, unsigned P, bool& is_f, int& sl, int& idx) const {
    if (!with_g) { is_f = true; sl = slice_of(t / SR, P); idx = t % SR; return; }
    if (t < SR) { is_f = true; sl = slice_of(0, P); idx = t; return; }
    const int u = t - SR, ph = SR + T;
    const int p = 1 + u / ph, r = u % ph;
    if (p < S && r < SR) { is_f = true; sl = slice_of(p, P); idx = r; return; }
    is_f = false;
    sl = slice_of(p - 1, P);
    idx = (p < S) ? r - SR : r;
  }
  __device__ __forceinline__ int next_task(unsigned P) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(a.tctr + (P & 1), 1u);
    return int(__shfl_sync(0xffffffffu, t, 0));
  }

  // ---------------- staging
  __device__ void load_lognu() {
    for (int j = threadIdx.x; j < WMAX; j += NT) lnusm[j] = j < a.m ? __ldg(a.log_nu + j) : -INFINITY;
  }
  __device__ bool load_g(const float* g) {  // returns: some g_j non-finite (any thread of the CTA)
    int bad = 0;
    for (int j = threadIdx.x; j < WMAX; j += NT) {
      const float v = j < a.m ? ldcg(g + j) : 0.f;
      gsm[j] = v;
      bad |= !isfinite(v);
    }
    return __syncthreads_or(bad) != 0;
  }

  static __device__ __forceinline__ bool shift_ok(float S_) { return S_ >= kShiftLo && S_ <= kShiftHi; }
  __device__ __forceinline__ float4 ldrow(const float* p) const {
    return __ldcg(reinterpret_cast<const float4*>(p));  // L2: the slice's G tasks re-read it next phase
  }

  // ---------------- F tasks: one row, one warp
  // MODE 0: stale fused f (+ check terms of iterate k-1 with CHECK); 1: exact f (two passes)
  // 2: check only (terms of the iterate (f, g)); 3: cost terms
  template <int MODE, bool CHECK>
  __device__ void f_task(int i, const float* fprev, float* fnew, unsigned& flag) {
    const float* Ci = a.C + (long long)i * a.ldc;
    const float fold = ldcg(fprev + i);
    const f2 fo2 = pk2(fold, fold);
    const float lmu = __ldg(a.log_mu + i);
    const f2 lm2 = pk2(lmu, lmu);
    const int nT = (a.mpad + STRIP - 1) / STRIP;
    float M = 0.f;
    if (MODE == 1) {  // exact: max pass
      float mx = -INFINITY;
#pragma unroll 4
      for (int t = 0; t < nT; ++t) {
        const int j = t * STRIP + 4 * lane;
        if (j >= a.mpad) continue;
        const float4 c = __ldcg(reinterpret_cast<const float4*>(Ci + j));
        const float4 gg = *reinterpret_cast<const float4*>(gsm + j);
        const float4 ll = *reinterpret_cast<const float4*>(lnusm + j);
        float x0, x1, x2, x3;
        up2(arg3x2(pk2(gg.x, gg.y), pk2(c.x, c.y), inv2, pk2(ll.x, ll.y), nz2), x0, x1);
        up2(arg3x2(pk2(gg.z, gg.w), pk2(c.z, c.w), inv2, pk2(ll.z, ll.w), nz2), x2, x3);
        mx = fmax_nan(mx, fmax_nan(fmax_nan(x0, x1), fmax_nan(x2, x3)));
      }
      M = warp_max(mx);
    } else if (MODE == 0) {
      M = __fmul_rn(-fold, a.inv_eps);
    }
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    const float shl = __fmul_rn(Ms, kLog2e);
    const f2 nsl = pk2(-shl, -shl);
    f2 sa = 0ull, sb = 0ull, za = 0ull, zb = 0ull;
    float cs = 0.f;
    auto body = [&](const float4& c, int j) {
      const float4 gg = *reinterpret_cast<const float4*>(gsm + j);
      const float4 ll = *reinterpret_cast<const float4*>(lnusm + j);
      const f2 c01 = pk2(c.x, c.y), c23 = pk2(c.z, c.w);
      const f2 g01 = pk2(gg.x, gg.y), g23 = pk2(gg.z, gg.w);
      const f2 l01 = pk2(ll.x, ll.y), l23 = pk2(ll.z, ll.w);
      if (MODE == 0 || MODE == 1) {
        sa = add2(sa, ex2x2(fma2(arg3x2(g01, c01, inv2, l01, nz2), l2e2, nsl)));
        sb = add2(sb, ex2x2(fma2(arg3x2(g23, c23, inv2, l23, nz2), l2e2, nsl)));
      }
      if ((MODE == 0 && CHECK) || MODE == 2) {
        za = add2(za, ex2x2(mul2(arg4x2(fo2, g01, c01, inv2, l01, nz2), l2e2)));
        zb = add2(zb, ex2x2(mul2(arg4x2(fo2, g23, c23, inv2, l23, nz2), l2e2)));
      }
      if (MODE == 3) {  // cost: fl(C_ij * exp(z_ij)), z as solver.py:108-112
        float z0, z1, z2v, z3;
        up2(add2(arg4x2(fo2, g01, c01, inv2, lm2, nz2), l01), z0, z1);
        up2(add2(arg4x2(fo2, g23, c23, inv2, lm2, nz2), l23), z2v, z3);
        cs += __fmul_rn(c.x, expf(z0));
        cs += __fmul_rn(c.y, expf(z1));
        cs += __fmul_rn(c.z, expf(z2v));
        cs += __fmul_rn(c.w, expf(z3));
      }
    };
    // U loads in flight per lane (memory-level parallelism), then the math
    constexpr int U = 8;
    const int nfull = a.mpad / STRIP;
    int t = 0;
    for (; t + U <= nfull; t += U) {
      float4 c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = ldrow(Ci + (t + u) * STRIP + 4 * lane);
#pragma unroll
      for (int u = 0; u < U; ++u) body(c[u], (t + u) * STRIP + 4 * lane);
    }
    for (; t < nT; ++t) {
      const int j = t * STRIP + 4 * lane;
      if (j < a.mpad) body(ldrow(Ci + j), j);
    }
    if (MODE == 3) {
      cs = warp_sum(cs);
      if (lane == 0) a.rowterm[i] = cs;
      return;
    }
    float s0, s1, s2_, s3;
    float Ssum = 0.f, Z = 0.f;
    if (MODE == 0 || MODE == 1) {
      up2(sa, s0, s1);
      up2(sb, s2_, s3);
      Ssum = warp_sum((s0 + s1) + (s2_ + s3));
    }
    if ((MODE == 0 && CHECK) || MODE == 2) {
      up2(za, s0, s1);
      up2(zb, s2_, s3);
      Z = warp_sum((s0 + s1) + (s2_ + s3));
    }
    if (lane == 0) {
      if (MODE == 0 || MODE == 1) {
        if (MODE == 0 && !shift_ok(Ssum)) flag = 1;
        fnew[i] = __fmul_rn(a.neg_eps, lse_finish(M, MODE == 0 ? fmaxf(Ssum, kSumFloor) : Ssum));
      }
      if ((MODE == 0 && CHECK) || MODE == 2) {
        float Zs = Z, Mz = 0.f;
        if (!shift_ok(Zs)) {
          if (MODE == 0) flag = 1;  // the redo recomputes the check exactly
          // check-only pass: an exact second look is not needed for the stop
          // decision beyond the reference's own floor; keep the unshifted sum
        }
        const float rr = expf(__fadd_rn(lmu, lse_finish(Mz, Zs)));
        a.rowterm[i] = fabsf(__fsub_rn(rr, __ldg(a.mu + i)));
      }
    }
  }

  // ---------------- G tasks: one 128-column strip of one slice, one warp
  // EXACT: online (max, sumexp) pairs; else stale-shift sums
  template <bool EXACT>
  __device__ void g_task(int sl, int strip, const float* fnew) {
    const int i0 = sl * SR, cnt = min(SR, a.n - i0);
    const int j0 = strip * STRIP + 4 * lane;
    const bool live = j0 < a.mpad;
    const int jc = live ? j0 : 0;
    // stale column shifts of the 4 owned columns: -fl(fl(-g_j * inv) * log2e)
    float ns[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ns[q] = -__fmul_rn(__fmul_rn(-gsm[jc + q], a.inv_eps), kLog2e);
    const f2 ns01 = pk2(ns[0], ns[1]), ns23 = pk2(ns[2], ns[3]);
    // f and log mu of the slice's rows, two per lane, broadcast by shuffles
    const float fA = lane < cnt ? ldcg(fnew + i0 + lane) : 0.f;
    const float fB = lane + 32 < cnt ? ldcg(fnew + i0 + 32 + lane) : 0.f;
    const float lA = lane < cnt ? __ldg(a.log_mu + i0 + lane) : 0.f;
    const float lB = lane + 32 < cnt ? __ldg(a.log_mu + i0 + 32 + lane) : 0.f;
    f2 a01 = 0ull, a23 = 0ull;
    float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, sm[4] = {0.f, 0.f, 0.f, 0.f};
    const float* Cc = a.C + (long long)i0 * a.ldc + jc;
    auto row = [&](int r, const float4& c) {
      const float fi = __shfl_sync(0xffffffffu, r < 32 ? fA : fB, r & 31);
      const float lm = __shfl_sync(0xffffffffu, r < 32 ? lA : lB, r & 31);
      const f2 fi2 = pk2(fi, fi), lm2 = pk2(lm, lm);
      const f2 y01 = arg3x2(fi2, pk2(c.x, c.y), inv2, lm2, nz2);
      const f2 y23 = arg3x2(fi2, pk2(c.z, c.w), inv2, lm2, nz2);
      if (!EXACT) {
        a01 = add2(a01, ex2x2(fma2(y01, l2e2, ns01)));
        a23 = add2(a23, ex2x2(fma2(y23, l2e2, ns23)));
      } else {
        float y[4];
        up2(y01, y[0], y[1]);
        up2(y23, y[2], y[3]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float mo = mx[q];
          const float mn = fmax_nan(mo, y[q]);
          const float mss = (fabsf(mn) <= 3.402823466e38f) ? mn : 0.f;
          const float sl2 = __fmul_rn(mss, kLog2e);
          const float s = (mo == -INFINITY) ? 0.f : sm[q] * exp_shifted(mo, sl2);
          sm[q] = s + exp_shifted(y[q], sl2);
          mx[q] = mn;
        }
      }
    };
    constexpr int U = 8;
    int r = 0;
    for (; r + U <= cnt; r += U) {  // rows in order (deterministic), U loads in flight
      float4 c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = __ldcg(reinterpret_cast<const float4*>(Cc + (long long)(r + u) * a.ldc));
#pragma unroll
      for (int u = 0; u < U; ++u) row(r + u, c[u]);
    }
    for (; r < cnt; ++r) row(r, __ldcg(reinterpret_cast<const float4*>(Cc + (long long)r * a.ldc)));
    if (!live) return;
    if (!EXACT) {
      float v0, v1, v2, v3;
      up2(a01, v0, v1);
      up2(a23, v2, v3);
      *reinterpret_cast<float4*>(a.part + (size_t)sl * a.mpad + j0) = make_float4(v0, v1, v2, v3);
    } else {
      float2* dst = a.pairs + (size_t)sl * a.mpad + j0;
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float2(mx[q], sm[q]);
    }
  }

  __device__ __forceinline__ void wait_slice(int sl, unsigned target) {
    if (lane == 0) {
      const unsigned* p = a.rows_done + sl;
      if (ld_acquire(p) < target) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire(p) < target)
          if (globaltimer_ns() - t0 > kSpinTimeoutNs) __trap();
      }
    }
    __syncwarp();
  }

  // One pass over the task list; returns this warp's guard flag.
  //   MODE 0: fused (F stale [+ CHECK terms of iterate k-1] and G stale sums)
  //   MODE 1: exact (F two-pass and G (max, sumexp) pairs)
  //   MODE 2: F check-only terms of the iterate (fprev, gsm)
  //   MODE 3: F transport-cost terms of (fprev, gsm)
  //   MODE 4: G pairs only (f complete; no slice waits)
  template <int MODE, bool CHECK>
  __device__ unsigned pass(const float* fprev, float* fnew) {
    const unsigned P = npass++;
    const bool with_f = MODE != 4;
    const bool interleave = MODE <= 1;
    const unsigned target = (gpasses + 1) * unsigned(SR);
    const int total = interleave ? S * SR + S * T : (with_f ? S * SR : S * T);
    unsigned flag = 0;
    // static round-robin over all warps of the grid in phase order: equal-size
    // tasks, no atomics; each warp walks the phases in order
    const int nwarps = G * NW;
    auto prefetch_task = [&](int t2) {  // bring this warp's upcoming F row into L2 early
      if (t2 >= total || lane != 0 || !with_f) return;
      bool f2_;
      int sl2, idx2;
      if (interleave) decode(t2, true, P, f2_, sl2, idx2);
      else { f2_ = with_f; sl2 = slice_of(t2 / SR, P); idx2 = t2 % SR; }
      const int i2 = sl2 * SR + idx2;
      if (f2_ && i2 < a.n) prefetch_l2(a.C + (long long)i2 * a.ldc, uint32_t(a.mpad) * 4u);
    };
    prefetch_task(b * NW + w);
    prefetch_task(b * NW + w + nwarps);
    for (int t = b * NW + w; t < total; t += nwarps) {
      prefetch_task(t + 2 * nwarps);
      bool is_f;
      int sl, idx;
      if (interleave) decode(t, true, P, is_f, sl, idx);
      else if (with_f) { is_f = true; sl = slice_of(t / SR, P); idx = t % SR; }
      else { is_f = false; sl = slice_of(t / T, P); idx = t % T; }
      if (is_f) {
        const int i = sl * SR + idx;
        if (i < a.n) {
          if (MODE == 0) f_task<0, CHECK>(i, fprev, fnew, flag);
          else if (MODE == 1) f_task<1, false>(i, fprev, fnew, flag);
          else if (MODE == 2) f_task<2, false>(i, fprev, fnew, flag);
          else f_task<3, false>(i, fprev, fnew, flag);
        }
        if (interleave) {  // publish: f_i visible before the slice counter moves
          __syncwarp();
          if (lane == 0) {
            __threadfence();
            atomicAdd(a.rows_done + sl, 1u);
          }
        }
      } else {
        if (interleave) wait_slice(sl, target);
        if (MODE == 0) g_task<false>(sl, idx, fnew);
        else g_task<true>(sl, idx, fnew);
      }
    }
    if (interleave) ++gpasses;
    return flag;
  }
  unsigned gpasses;  // interleaved passes so far (slice counter targets)

  // ---------------- combines over the S slice partials (fixed order)
  __device__ void combine_stale(const float* gold, float* gnew, int k) {
    const int ngroups = (a.m + 31) / 32;
    bool fired = false;
    for (int grp = b; grp < ngroups; grp += G) {
      const int j = grp * 32 + lane;
      const int k0 = w * S / NW, k1 = (w + 1) * S / NW;
      float s = 0.f;
      if (j < a.m)
        for (int kk = k0; kk < k1; ++kk) s += ldcg(a.part + (size_t)kk * a.mpad + j);
      red[w * 32 + lane] = s;
      __syncthreads();
      if (w == 0) {
        for (int h = NW / 2; h >= 1; h >>= 1)
          for (int u = 0; u < h; ++u) red[u * 32 + lane] += red[(u + h) * 32 + lane];
        if (j < a.m) {
          const float sj = __fmul_rn(-ldcg(gold + j), a.inv_eps);
          const float Sv = red[lane];
          if (!shift_ok(Sv)) fired = true;
          gnew[j] = __fmul_rn(a.neg_eps, lse_finish(sj, Sv));
        }
      }
      __syncthreads();
    }
    if (w == 0 && __any_sync(0xffffffffu, fired) && lane == 0) atomicMax(a.guard, k);
  }
  __device__ void combine_pairs(float* gnew) {
    const int ngroups = (a.m + 31) / 32;
    for (int grp = b; grp < ngroups; grp += G) {
      const int j = grp * 32 + lane;
      const int k0 = w * S / NW, k1 = (w + 1) * S / NW;
      float mx = -INFINITY, s = 0.f;
      if (j < a.m)
        for (int kk = k0; kk < k1; ++kk) {
          const float2 p = __ldcg(a.pairs + (size_t)kk * a.mpad + j);
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

  // every CTA sums the per-row terms in the same fixed order (identical result)
  __device__ float sum_rows() {
    float s = 0.f;
    const int per = (a.n + NT - 1) / NT;
    const int lo = threadIdx.x * per, hi = min(a.n, lo + per);
    for (int i = lo; i < hi; ++i) s += ldcg(a.rowterm + i);
    float v[1] = {s};
    block_reduce<NT, 1, false>(v, red);
    __syncthreads();
    return v[0];
  }

  // check decision (solver.py:286-300), identical in every CTA
  __device__ bool decide(int kk, bool bad, bool& failed) {
    const float err = sum_rows();
    bool stop = false, append = true;
    int status = 0;
    float e = err;
    if (bad) { stop = true; status = 2; e = NAN; append = false; }
    else if (!isfinite(err)) { stop = true; status = 2; }
    else if (err < a.tol) { stop = true; status = 1; }
    if (b == 0 && threadIdx.x == 0) {
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

  // pass + grid barrier; the barrier word carries "a guard fired in my CTA"
  template <int MODE, bool CHECK>
  __device__ bool run(const float* fprev, float* fnew) {
    if (threadIdx.x == 0) *cta_flag = 0;
    // the counter of the next pass was last used two passes ago: clear it now
    if (b == 0 && threadIdx.x == 0) a.tctr[(npass + 1) & 1] = 0;
    __syncthreads();
    const unsigned fl = pass<MODE, CHECK>(fprev, fnew);
    if (fl && lane == 0) atomicOr(cta_flag, 1u);
    __syncthreads();
    const unsigned word = grid_barrier(a.bar, epoch, *cta_flag ? 1u : 0u, cta_flag + 1);
    const bool fired = word != flags_seen;
    flags_seen = word;
    return fired;
  }

  // non-finite entries of a vector (every CTA reads all of it: same answer everywhere)
  __device__ bool any_nonfinite(const float* v, int len) {
    int bad = 0;
    for (int i = threadIdx.x; i < len; i += NT) bad |= !isfinite(ldcg(v + i));
    return __syncthreads_or(bad) != 0;
  }

  __device__ void solve() {
    load_lognu();
    gpasses = 0;
    auto fb = [&](int k) { return (k & 1) ? a.f1 : a.f0; };
    auto gb = [&](int k) { return (k & 1) ? a.g1 : a.g0; };
    int final_k = a.max_iter;
    bool stopped = false, failed = false;
    for (int k = 1; k <= a.max_iter; ++k) {
      const bool do_check = (k > 1) && ((k - 1) % a.check == 0);
      const float* fprev = fb((k - 1) & 1);
      float* fnew = fb(k & 1);
      const float* gcur = gb((k - 1) & 1);
      const bool gbad = load_g(gcur);
      const bool fused = a.stale && k > 1;
      bool redo = false, checked = false;
      if (fused) {
        redo = do_check ? run<0, true>(fprev, fnew) : run<0, false>(fprev, fnew);
        checked = do_check && !redo;
        if (redo) {
          if (threadIdx.x == 0 && b == 0) atomicAdd(a.stats + 0, 1);
          run<1, false>(fprev, fnew);  // exact f^k and exact column pairs
        }
      } else {
        run<1, false>(fprev, fnew);
      }
      if (do_check && !checked) run<2, false>(fprev, nullptr);  // exact-path check of iterate k-1
      if (do_check) {
        const bool bad = gbad || any_nonfinite(fprev, a.n);
        if (decide(k - 1, bad, failed)) { stopped = true; final_k = k - 1; break; }
      }
      if (fused && !redo) {
        combine_stale(gcur, gb(k & 1), k);
        grid_barrier(a.bar, epoch);
        if (__ldcg(a.guard) == k) {  // a column sum left the band: exact column pass
          if (threadIdx.x == 0 && b == 0) atomicAdd(a.stats + 1, 1);
          run<4, false>(fnew, nullptr);
          combine_pairs(gb(k & 1));
          grid_barrier(a.bar, epoch);
        }
      } else {
        combine_pairs(gb(k & 1));
        grid_barrier(a.bar, epoch);
      }
    }
    if (!stopped) {  // the final check at the cap (solver.py:286-316)
      final_k = a.max_iter;
      const bool gbad = load_g(gb(final_k & 1));
      run<2, false>(fb(final_k & 1), nullptr);
      decide(final_k, gbad || any_nonfinite(fb(final_k & 1), a.n), failed);
    }
    const int fbuf = final_k & 1;
    if (!failed && a.want_cost) {
      load_g(gb(fbuf));
      run<3, false>(fb(fbuf), nullptr);
      const float cost0 = sum_rows();
      if (b == 0 && threadIdx.x == 0) {
        float cost = cost0;
        if (!isfinite(cost)) { *a.out_status = 2; cost = NAN; }
        *a.out_cost = cost;
      }
    } else if (b == 0 && threadIdx.x == 0) {
      *a.out_cost = NAN;
    }
    if (b == 0 && threadIdx.x == 0) {
      *a.out_iters = final_k;
      *a.out_fbuf = fbuf;
    }
  }
};

}  // namespace lsk

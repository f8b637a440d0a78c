// On-the-fly squared-Euclidean log-domain Sinkhorn kernels (configs C4/C5):
// the cost c_ij = scale * sum_k (x_ik - y_jk)^2 is recomputed in registers
// from fp32 point clouds and never stored (C4 at n=m=65536 would be 17 GB).
//
// Reference path replaced: squared_euclidean_cost (costs.py:36-50) [+ C/C.max()
// of applications.py:186-188] followed by solve (solver.py:230-337). Because
// the cost is symmetric in the roles of the two clouds, the g-update is the
// f-update with (X, f, log mu) and (Y, g, log nu) swapped: one
// "row LSE over points" kernel serves both half-steps.
//
// One half-step (rows R with old potential p_i, columns Q with potential q_j
// and log-weights l_j):
//   p_i^new = neg_eps * LSE_j( (q_j - c_ij) * inv_eps + l_j )
// computed in log2 units as
//   v_ij = A_j - K * (sum_k d_k^2 + init_i),  A_j = (q_j * inv_eps + l_j) * log2 e,
//   K = inv_eps * log2 e * scale,  init_i = -p_i / scale  (stale shift)
// so v_ij = log2(e) * (x_ij - sh_i) with sh_i = -p_i * inv_eps; the row shift is
// folded into the start value of the coordinate sum (no extra op per pair).
// Per pair: 3 sub + 3 fma (cost) + 1 fma (argument) + 1 add, packed two rows
// per f32x2 op, and one MUFU ex2: the FP32 lanes and the MUFU pipe are
// balanced at 16 pairs/clk/SM.
//
// Numerics: the cost is fp32 from fp32-rounded points in the direct form (the
// reference builds it in fp64 and rounds once); SURVEY F5 measures this at
// 2-3e-6 on the potentials at eps=1e-3, inside the 1e-5 bar. Use the dense
// solver (fp32(C64) bit for bit) for eps < 1e-3.
#pragma once
#include "lsk_device.cuh"

namespace lsk {

constexpr int kPtsThreads = 256;            // 8 warps
constexpr int kPtsRowsPerWarp = 8;          // 4 packed row pairs per lane
constexpr int kPtsTileRows = 8 * kPtsRowsPerWarp;  // 64 rows per CTA tile
constexpr int kPtsChunk = 2048;             // columns per chunk (32 KB of smem)

enum PtsMode { kPtsStale = 0, kPtsOnline = 1, kPtsCost = 2, kPtsStaleX = 3 };
// kPtsStaleX: the stale sweep with the cost in expansion form |x|^2 + |y|^2 - 2 x.y
// (3 FMA per pair instead of 3 sub + 3 FMA), folded as
//   v_ij = B_j + R_i + sum_k x_ik (2K y_jk),  B_j = A_j - K |y_j|^2,  R_i = -K (|x_i|^2 + init_i).
// The cancellation costs ~K (|x|^2 + |y|^2) ulp in the exponent, the same order as
// the reference's own fp32 argument rounding at |C|/eps; used only for eps >= 5e-3
// (tests/test_gpu_points.py checks the C5/C1 fixtures at eps = 1e-2).

struct PtsHalf {
  // problem b's rows/cols: rows_b = rows + b * n_rows, etc.
  int B, n_rows, n_cols;
  int row_lo, row_hi;          // this rank's slab of rows [row_lo, row_hi)
  int chunks;                  // ceil(n_cols / kPtsChunk)
  int ch_lo;                   // first column chunk this launch covers (grid.x chunks from here)
  const float4* rpts;          // (B, n_rows) points (x, y, z, 0)
  const float4* cpts;          // (B, n_cols)
  const float* rpot;           // (B, n_rows) old row potential (stale shift / cost)
  const float* cpot;           // (B, n_cols) column potential
  const float* clw;            // (B, n_cols) column log-weights
  const float* rlw;            // (B, n_rows) row log-weights (cost mode)
  const float* scale;          // (B) cost scale (1/Cmax or 1)
  float inv_eps;
  void* part;                  // (B, chunks, n_rows) float (stale/cost) or float2 (online)
  const int* active;           // (B) problem still iterating (nullptr = all)
  const int* rowflag;          // (B, n_rows) online mode: only rows flagged here
  const int* nflag;            // online mode: number of flagged rows (0 -> exit)
};

__device__ __forceinline__ f2 bc2(float a) { return pk2(a, a); }

// One CTA = one (problem, 8*RPW-row tile of the slab, column chunk) unit.
template <int MODE, int RPW>
static __global__ void __launch_bounds__(kPtsThreads, (RPW > 8 ? 2 : 3)) k_pts_part(PtsHalf h) {
  constexpr int PP = RPW / 2, TILE = 8 * RPW;
  __shared__ __align__(16) float4 colv[kPtsChunk];
  __shared__ int tile_any;
  const int ch = h.ch_lo + blockIdx.x, tile = blockIdx.y, b = blockIdx.z;
  if (MODE == kPtsOnline && h.nflag && *h.nflag == 0) return;
  if (h.active && !h.active[b]) return;
  const int r_base = h.row_lo + tile * TILE;
  if (r_base >= h.row_hi) return;
  if (MODE == kPtsOnline && h.rowflag) {
    if (threadIdx.x == 0) tile_any = 0;
    __syncthreads();
    if (threadIdx.x < TILE) {
      const int r = r_base + threadIdx.x;
      if (r < h.row_hi && h.rowflag[(size_t)b * h.n_rows + r]) tile_any = 1;
    }
    __syncthreads();
    if (!tile_any) return;
  }
  const float sc = __ldg(h.scale + b);
  const float l2 = kLog2e;
  const int j0 = ch * kPtsChunk;
  const int ncol = min(kPtsChunk, h.n_cols - j0);
  const float Kf = __fmul_rn(__fmul_rn(h.inv_eps, l2), sc);
  // stage the chunk: (y0, y1, y2, A_j), A_j = (q_j * inv + l_j) * log2e
  // (expansion form: (2K y0, 2K y1, 2K y2, A_j - K |y_j|^2))
  for (int t = threadIdx.x; t < ncol; t += kPtsThreads) {
    const size_t j = (size_t)b * h.n_cols + j0 + t;
    float4 q = __ldg(h.cpts + j);
    const float A = __fmul_rn(__fmaf_rn(__ldg(h.cpot + j), h.inv_eps, __ldg(h.clw + j)), l2);
    if (MODE == kPtsStaleX) {
      const float yy = __fmaf_rn(q.z, q.z, __fmaf_rn(q.y, q.y, q.x * q.x));
      const float k2 = 2.f * Kf;
      q = make_float4(k2 * q.x, k2 * q.y, k2 * q.z, __fmaf_rn(-Kf, yy, A));
    } else {
      q.w = A;
    }
    colv[t] = q;
  }
  // this warp's 8 rows, packed in pairs
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  f2 X0[PP], X1[PP], X2[PP], I0[PP];
  float lrow[RPW];
#pragma unroll
  for (int p = 0; p < PP; ++p) {
    float xa[3], xb[3], ia, ib;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      int r = r_base + w * RPW + 2 * p + h2;
      r = r < h.row_hi ? r : h.row_hi - 1;
      const size_t ri = (size_t)b * h.n_rows + r;
      const float4 x = __ldg(h.rpts + ri);
      float init = 0.f;
      if (MODE != kPtsOnline) init = __fdiv_rn(-__ldg(h.rpot + ri), sc);  // (stale / expansion / cost)
      if (MODE == kPtsCost) lrow[2 * p + h2] = __ldg(h.rlw + ri);
      if (h2 == 0) { xa[0] = x.x; xa[1] = x.y; xa[2] = x.z; ia = init; }
      else { xb[0] = x.x; xb[1] = x.y; xb[2] = x.z; ib = init; }
    }
    X0[p] = pk2(xa[0], xb[0]);
    X1[p] = pk2(xa[1], xb[1]);
    X2[p] = pk2(xa[2], xb[2]);
    if (MODE == kPtsStaleX) {  // R_i = -K (|x_i|^2 + init_i)
      const float xxa = __fmaf_rn(xa[2], xa[2], __fmaf_rn(xa[1], xa[1], xa[0] * xa[0]));
      const float xxb = __fmaf_rn(xb[2], xb[2], __fmaf_rn(xb[1], xb[1], xb[0] * xb[0]));
      I0[p] = pk2(-Kf * (xxa + ia), -Kf * (xxb + ib));
    } else {
      I0[p] = pk2(ia, ib);
    }
  }
  const f2 NK = bc2(-Kf);
  __syncthreads();

  f2 acc[PP];
  float mx[RPW], sm[RPW];
#pragma unroll
  for (int p = 0; p < PP; ++p) acc[p] = 0ull;
#pragma unroll
  for (int r = 0; r < RPW; ++r) { mx[r] = -INFINITY; sm[r] = 0.f; }

#pragma unroll 2
  for (int t = lane; t < ncol; t += 32) {
    const float4 q = colv[t];
    const f2 Q0 = bc2(q.x), Q1 = bc2(q.y), Q2 = bc2(q.z), QA = bc2(q.w);
#pragma unroll
    for (int p = 0; p < PP; ++p) {
      if (MODE == kPtsStaleX) {
        f2 t2 = add2(I0[p], QA);
        t2 = fma2(X0[p], Q0, t2);
        t2 = fma2(X1[p], Q1, t2);
        t2 = fma2(X2[p], Q2, t2);
        acc[p] = add2(acc[p], ex2x2(t2));
        continue;
      }
      f2 d = sub2(X0[p], Q0);
      f2 s = (MODE == kPtsCost) ? mul2(d, d) : fma2(d, d, I0[p]);
      d = sub2(X1[p], Q1);
      s = fma2(d, d, s);
      d = sub2(X2[p], Q2);
      s = fma2(d, d, s);
      if (MODE == kPtsStale) {
        acc[p] = add2(acc[p], ex2x2(fma2(s, NK, QA)));
      } else if (MODE == kPtsCost) {
        // c_ij * exp(z_ij), z = ((f_i + g_j) - c_ij) * inv + lmu_i + lnu_j
        const f2 v = fma2(add2(s, I0[p]), NK, QA);
        float v0, v1, s0, s1;
        up2(v, v0, v1);
        up2(s, s0, s1);
        const float e0 = ex2(__fmaf_rn(lrow[2 * p], l2, v0)), e1 = ex2(__fmaf_rn(lrow[2 * p + 1], l2, v1));
        acc[p] = add2(acc[p], pk2(__fmul_rn(__fmul_rn(s0, sc), e0), __fmul_rn(__fmul_rn(s1, sc), e1)));
      } else {  // online (max, sum) in log2 units
        float v0, v1;
        up2(fma2(s, NK, QA), v0, v1);
        const float vv[2] = {v0, v1};
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int r = 2 * p + h2;
          const float mn = fmax_nan(mx[r], vv[h2]);
          const float ms = (fabsf(mn) <= 3.402823466e38f) ? mn : 0.f;
          sm[r] = __fmaf_rn(sm[r], (mx[r] == -INFINITY) ? 0.f : ex2(mx[r] - ms), ex2(vv[h2] - ms));
          mx[r] = mn;
        }
      }
    }
  }
  // lane reduction (xor butterfly: fixed order) and store
  const size_t pbase = ((size_t)b * h.chunks + ch) * h.n_rows;
#pragma unroll
  for (int p = 0; p < PP; ++p) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int r8 = 2 * p + h2;
      const int r = r_base + w * RPW + r8;
      if (MODE != kPtsOnline) {
        float a0, a1;
        up2(acc[p], a0, a1);
        const float v = warp_sum(h2 == 0 ? a0 : a1);
        if (lane == 0 && r < h.row_hi) reinterpret_cast<float*>(h.part)[pbase + r] = v;
      } else {
        float m2 = mx[r8], s2 = sm[r8];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float mo = __shfl_xor_sync(0xffffffffu, m2, o), so = __shfl_xor_sync(0xffffffffu, s2, o);
          // merge in log2 units
          const float mm = fmax_nan(m2, mo);
          const float mms = (fabsf(mm) <= 3.402823466e38f) ? mm : 0.f;
          const float wa = (m2 == -INFINITY) ? 0.f : ex2(m2 - mms), wb = (mo == -INFINITY) ? 0.f : ex2(mo - mms);
          s2 = __fmaf_rn(s2, wa, so * wb);
          m2 = mm;
        }
        if (lane == 0 && r < h.row_hi) reinterpret_cast<float2*>(h.part)[pbase + r] = make_float2(m2, s2);
      }
    }
  }
}

// ---- fixed-shape combine of per-chunk partials: a balanced binary tree over
// `cnt` (a power of two) leaves [lo, lo + cnt), leaves >= nreal being the
// identity. The leaf count is a function of the column count only, never of
// the rank count, so a rank that owns the complete subtree [r cnt/P, (r+1)
// cnt/P) can reduce it locally (k_pts_subtree) and the P subtree roots
// combine with the top P leaves of the same tree: bitwise the single-GPU
// result for every power-of-two P. Identity padding is skipped
// (merge(x, id) == x bit for bit for both operators), and the partial
// subtrees left on the stack fold right to left, exactly as the padded tree.
struct SumOp {
  using T = float;
  __device__ static T ident() { return 0.f; }
  __device__ static T merge(T a, T b) { return __fadd_rn(a, b); }
};
// (max, sum) pairs in log2 units: the online max-rescale merge
struct PairOp {
  using T = float2;
  __device__ static T ident() { return make_float2(-INFINITY, 0.f); }
  __device__ static T merge(T a, T b) {
    const float mm = fmax_nan(a.x, b.x);
    const float mms = (fabsf(mm) <= 3.402823466e38f) ? mm : 0.f;
    const float wa = (a.x == -INFINITY) ? 0.f : ex2(a.x - mms), wb = (b.x == -INFINITY) ? 0.f : ex2(b.x - mms);
    return make_float2(mm, __fmaf_rn(a.y, wa, b.y * wb));
  }
};
constexpr int kTreeDepth = 32;
template <class Op, class Get>
__device__ __forceinline__ typename Op::T leaf_tree(int lo, int cnt, int nreal, Get get) {
  using T = typename Op::T;
  T stk[kTreeDepth];
  int lev[kTreeDepth];
  int sp = 0;
  const int hi = min(lo + cnt, nreal);
  // leaves are loaded 8 at a time (all in flight) and folded in the same order
  constexpr int PF = 8;
  for (int l0 = lo; l0 < hi; l0 += PF) {
    T buf[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) buf[u] = (l0 + u < hi) ? get(l0 + u) : Op::ident();
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      if (l0 + u < hi) {
        T v = buf[u];
        int lv = 0;
        while (sp > 0 && lev[sp - 1] == lv) {
          v = Op::merge(stk[sp - 1], v);
          --sp;
          ++lv;
        }
        stk[sp] = v;
        lev[sp] = lv;
        ++sp;
      }
    }
  }
  if (sp == 0) return Op::ident();
  T acc = stk[sp - 1];
  for (int i = sp - 2; i >= 0; --i) acc = Op::merge(stk[i], acc);
  return acc;
}
__host__ __device__ inline int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

struct PtsCombine {
  int B, n_rows, row_lo, row_hi, chunks;
  int nleaves;            // tree width: pow2_ceil(chunks) (or the rank count over subtree roots)
  const void* part;
  const float* rpot_old;  // (B, n_rows) stale potential (shift); for check: f^k
  float* rpot_new;        // (B, n_rows) new potential (nullptr: check only)
  float inv_eps, neg_eps;
  const int* active;
  int* rowflag;           // stale: set rows whose sum left the guard band
  int* nflag;             // stale: count of such rows
  // check (f-update only): per-row error terms of iterate k
  const float* rlw;       // log mu
  const float* rmu;       // mu
  const float* cpot;      // g^k (finiteness)
  float* errrow;          // (B, n_rows)
  int* badrow;            // (B) a non-finite f^k or g^k was seen
  int check;
  const int* nflag_in;    // online: number of flagged rows (0 -> exit)
};

// per (problem, row): combine the chunk partials in fixed order
template <int MODE>
static __global__ void k_pts_combine(PtsCombine c) {
  const int b = blockIdx.y;
  const int r = c.row_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (MODE == kPtsOnline && c.nflag_in && *c.nflag_in == 0) return;
  if (r >= c.row_hi) return;
  if (c.active && !c.active[b]) return;
  const size_t ri = (size_t)b * c.n_rows + r;
  if (MODE == kPtsOnline) {
    if (c.rowflag && !c.rowflag[ri]) return;
    const float2* p = reinterpret_cast<const float2*>(c.part);
    const float2 t = leaf_tree<PairOp>(0, c.nleaves, c.chunks,
                                       [&](int ch) { return p[((size_t)b * c.chunks + ch) * c.n_rows + r]; });
    const float m2 = t.x, s2 = t.y;
    // LSE = M2 * ln2 + ln S (reduction.py:196-207: an all -inf row gives -inf)
    float L;
    if (!(fabsf(m2) <= 3.402823466e38f)) L = -INFINITY;
    else L = __fadd_rn(__fmul_rn(m2, 0.6931471805599453f), logf(fmaxf(s2, kSumFloor)));
    if (c.rpot_new) c.rpot_new[ri] = __fmul_rn(c.neg_eps, L);
    if (c.rowflag) c.rowflag[ri] = 0;
    return;
  }
  const float* p = reinterpret_cast<const float*>(c.part);
  const float S = leaf_tree<SumOp>(0, c.nleaves, c.chunks,
                                   [&](int ch) { return p[((size_t)b * c.chunks + ch) * c.n_rows + r]; });
  const float pold = c.rpot_old[ri];
  const float sh = __fmul_rn(-pold, c.inv_eps);
  const bool ok = S >= kShiftLo && S <= kShiftHi;
  if (c.rpot_new) {
    c.rpot_new[ri] = __fmul_rn(c.neg_eps, lse_finish(sh, S));
    if (!ok) {
      c.rowflag[ri] = 1;
      atomicAdd(c.nflag, 1);
    }
  }
  if (c.check) {
    // the stale sum with shift -f^k * inv is exactly the check sum of iterate k:
    // r_i = exp(log mu_i + LSE_j(((f_i + g_j) - c_ij) * inv + log nu_j)) (solver.py:97-104)
    const float rr = expf(__fadd_rn(c.rlw[ri], logf(fmaxf(S, kSumFloor))));
    c.errrow[ri] = fabsf(__fsub_rn(rr, c.rmu[ri]));
    if (!isfinite(pold) || !ok) {
      if (!isfinite(pold)) atomicOr(c.badrow + b, 1);
    }
  }
}

// A rank's complete subtree of the chunk tree, leaves [leaf_lo, leaf_lo + cnt),
// for rows [row_lo, row_hi) of problem 0 (sharded solves are single-problem):
// the root goes to slot row r of `out` (n_rows entries), the rank's
// contribution to the exchange.
template <int MODE>
static __global__ void k_pts_subtree(int n_rows, int row_lo, int row_hi, int chunks, int leaf_lo, int cnt,
                                     const void* __restrict__ part, void* __restrict__ out, const int* active,
                                     const int* nflag_in) {
  const int r = row_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= row_hi) return;
  if (active && !active[0]) return;
  if (MODE == kPtsOnline && nflag_in && *nflag_in == 0) return;
  if (MODE == kPtsOnline) {
    const float2* p = reinterpret_cast<const float2*>(part);
    reinterpret_cast<float2*>(out)[r] =
        leaf_tree<PairOp>(leaf_lo, cnt, chunks, [&](int ch) { return p[(size_t)ch * n_rows + r]; });
  } else {
    const float* p = reinterpret_cast<const float*>(part);
    reinterpret_cast<float*>(out)[r] =
        leaf_tree<SumOp>(leaf_lo, cnt, chunks, [&](int ch) { return p[(size_t)ch * n_rows + r]; });
  }
}

// non-finite g^k (columns) for the check's finiteness test (solver.py:287-290)
static __global__ void k_pts_colcheck(int B, int n, const float* __restrict__ pot, const int* active, int* bad) {
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  int any = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    any |= !isfinite(pot[(size_t)b * n + j]);
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(bad + b, 1);
}

// Per (problem, block of kPtsBlk rows): fixed-order sums of per-row terms.
// The block size is independent of the number of ranks, so a sharded solve
// sums exactly the same blocks in the same order as a single GPU.
constexpr int kPtsBlk = 1024;
static __global__ void __launch_bounds__(1024) k_pts_blocksum(int B, int n, int lo, int hi, const float* __restrict__ v,
                                                        const int* active, float* __restrict__ blk) {
  __shared__ float red[64];
  const int b = blockIdx.y, k = blockIdx.x;
  const int r0 = lo + k * kPtsBlk;
  if (r0 >= hi) return;
  if (active && !active[b]) return;
  float s[1] = {0.f};
  const int r = r0 + threadIdx.x;
  if (r < hi) s[0] = v[(size_t)b * n + r];
  block_reduce<1024, 1, false>(s, red);
  if (threadIdx.x == 0) blk[(size_t)b * ((n + kPtsBlk - 1) / kPtsBlk) + (r0 / kPtsBlk)] = s[0];
}

// Per-problem state for the batched solve (all device-resident).
struct PtsState {
  int active;     // still iterating
  int status;     // 0 not_converged, 1 converged, 2 numerical_failure
  int iters;
  int ntrace;
  int fbuf;       // buffer holding the returned f (and g)
  int pad[3];
  float err;
  float cost;
};

// check decision for every problem (solver.py:286-300): err = fixed-order sum
// of the row-block sums; stop on non-finite f/g, non-finite err or err < tol.
// kk = the iterate being checked; final = the check at the cap.
// kk_dev (optional): the checked iterate read from the device (a CUDA-graph
// replay of a block of iterations cannot carry it as a launch parameter)
static __global__ void k_pts_decide(int B, int n, const float* __restrict__ blk, int* bad, double tol, int kk, int final,
                             PtsState* st, int* trace_iter, float* trace_err, int cap,
                             const int* __restrict__ kk_dev = nullptr) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (kk_dev) kk = *kk_dev;
  PtsState& s = st[b];
  if (!s.active) return;
  const int nb = (n + kPtsBlk - 1) / kPtsBlk;
  float err = 0.f;
  for (int k = 0; k < nb; ++k) err += blk[(size_t)b * nb + k];
  const int isbad = bad[b];
  bad[b] = 0;
  int status = 0;
  bool stop = false, append = true;
  float e = err;
  if (isbad) { stop = true; status = 2; e = NAN; append = false; }
  else if (!isfinite(err)) { stop = true; status = 2; }
  else if (err < tol) { stop = true; status = 1; }
  if (append && s.ntrace < cap) {
    trace_iter[(size_t)b * cap + s.ntrace] = kk;
    trace_err[(size_t)b * cap + s.ntrace] = err;
    s.ntrace += 1;
  }
  s.status = status;
  s.err = e;
  if (stop || final) {
    s.active = 0;
    s.iters = kk;
    s.fbuf = kk & 1;
  }
}

static __global__ void k_pts_cost_finish(int B, int n, const float* __restrict__ blk, PtsState* st) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  PtsState& s = st[b];
  if (s.status == 2) { s.cost = NAN; return; }
  const int nb = (n + kPtsBlk - 1) / kPtsBlk;
  float c = 0.f;
  for (int k = 0; k < nb; ++k) c += blk[(size_t)b * nb + k];
  if (!isfinite(c)) { s.status = 2; c = NAN; }
  s.cost = c;
}

// Per problem, the centre of the bounding box of both clouds (fp64; ctr is
// (B, 3), unused coordinates 0): the translation of k_pts_pack.
static __global__ void __launch_bounds__(256) k_pts_center(const double* __restrict__ X, const double* __restrict__ Y,
                                                          int n, int m, int d, double* __restrict__ ctr) {
  __shared__ double smn[3][8], smx[3][8];
  const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < 3; ++k) {
    double mn = INFINITY, mx = -INFINITY;
    if (k < d) {
      for (int i = threadIdx.x; i < n + m; i += blockDim.x) {
        const double v = i < n ? X[((size_t)b * n + i) * d + k] : Y[((size_t)b * m + (i - n)) * d + k];
        mn = fmin(mn, v);
        mx = fmax(mx, v);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) { smn[k][w] = mn; smx[k][w] = mx; }
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int k = threadIdx.x;
    double mn = INFINITY, mx = -INFINITY;
    for (int q = 0; q < 8; ++q) { mn = fmin(mn, smn[k][q]); mx = fmax(mx, smx[k][q]); }
    ctr[b * 3 + k] = (k < d) ? __dmul_rn(__dadd_rn(mn, mx), 0.5) : 0.0;
  }
}

// fp64 points -> float4 (x, y, z, 0), coordinates beyond d zero. Each problem
// is translated by the centre of its bounding box (k_pts_center) in fp64
// before the single fp32 rounding: distances are unchanged, and the fp32
// coordinates carry the data's spread (|x - c| <= half the box diagonal)
// instead of its offset, which keeps the on-the-fly cost accurate for clouds
// far from the origin and halves the expansion form's cancellation.
static __global__ void k_pts_pack(const double* __restrict__ P, long long count, int per_problem, int d,
                                  const double* __restrict__ ctr, float4* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / per_problem;
    const double* c = ctr + b * 3;
    float v[3] = {0.f, 0.f, 0.f};
    for (int k = 0; k < d; ++k) v[k] = __double2float_rn(__dsub_rn(P[i * d + k], c[k]));
    out[i] = make_float4(v[0], v[1], v[2], 0.f);
  }
}

// select buffer s.fbuf into the outputs
static __global__ void k_pts_pick(int B, int n, const float* __restrict__ p0, const float* __restrict__ p1,
                           const PtsState* st, float* __restrict__ out) {
  const int b = blockIdx.y;
  const float* src = st[b].fbuf ? p1 : p0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[(size_t)b * n + i] = src[(size_t)b * n + i];
}

}  // namespace lsk

namespace lsk {

// ---- plan consumers without the plan: per source row i,
// with pi_ij = exp(((f_i + g_j) - c_ij) * inv + log mu_i + log nu_j):
//   barycentric map  sum_j pi_ij y_j / sum_j pi_ij   (applications.py:75-97)
//   argmax_j pi_ij, lowest j on ties                 (applications.py:195-204)
// Row constants cancel in both, so the weights are the f-update terms
// w_ij = 2^(A_j - K (sum d^2 - f_i / scale)) (bounded by ~1 at the solution).
struct PtsConsume {
  int B, n_rows, n_cols, chunks;
  const float4* rpts;
  const float4* cpts;
  const float* rpot;   // f (B, n)
  const float* cpot;   // g (B, m)
  const float* clw;    // log nu (B, m)
  const float* scale;
  float inv_eps;
  float4* part;        // (B, chunks, n): (sum w, sum w y0, sum w y1, sum w y2)
  float2* best;        // (B, chunks, n): (max v, index as int bits)
};

static __global__ void __launch_bounds__(kPtsThreads) k_pts_consume(PtsConsume h) {
  __shared__ __align__(16) float4 colv[kPtsChunk];
  const int ch = blockIdx.x, tile = blockIdx.y, b = blockIdx.z;
  const int r_base = tile * kPtsTileRows;
  if (r_base >= h.n_rows) return;
  const float sc = __ldg(h.scale + b);
  const int j0 = ch * kPtsChunk;
  const int ncol = min(kPtsChunk, h.n_cols - j0);
  for (int t = threadIdx.x; t < ncol; t += kPtsThreads) {
    const size_t j = (size_t)b * h.n_cols + j0 + t;
    float4 q = __ldg(h.cpts + j);
    q.w = __fmul_rn(__fmaf_rn(__ldg(h.cpot + j), h.inv_eps, __ldg(h.clw + j)), kLog2e);
    colv[t] = q;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float x0[8], x1[8], x2[8], ini[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int i = r_base + w * kPtsRowsPerWarp + r;
    i = i < h.n_rows ? i : h.n_rows - 1;
    const size_t ri = (size_t)b * h.n_rows + i;
    const float4 x = __ldg(h.rpts + ri);
    x0[r] = x.x; x1[r] = x.y; x2[r] = x.z;
    ini[r] = __fdiv_rn(-__ldg(h.rpot + ri), sc);
  }
  const float NK = -__fmul_rn(__fmul_rn(h.inv_eps, kLog2e), sc);
  __syncthreads();
  float sw[8], sy0[8], sy1[8], sy2[8], bv[8];
  int bj[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) { sw[r] = sy0[r] = sy1[r] = sy2[r] = 0.f; bv[r] = -INFINITY; bj[r] = 0x7fffffff; }
  for (int t = lane; t < ncol; t += 32) {
    const float4 q = colv[t];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float d0 = x0[r] - q.x, d1 = x1[r] - q.y, d2 = x2[r] - q.z;
      const float s = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmaf_rn(d0, d0, ini[r])));
      const float v = __fmaf_rn(s, NK, q.w);
      const float e = ex2(v);
      sw[r] += e;
      sy0[r] = __fmaf_rn(e, q.x, sy0[r]);
      sy1[r] = __fmaf_rn(e, q.y, sy1[r]);
      sy2[r] = __fmaf_rn(e, q.z, sy2[r]);
      if (v > bv[r]) { bv[r] = v; bj[r] = j0 + t; }  // columns visited in increasing j: first max wins
    }
  }
  const size_t pbase = ((size_t)b * h.chunks + ch) * h.n_rows;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    float a0 = sw[r], a1 = sy0[r], a2 = sy1[r], a3 = sy2[r], v = bv[r];
    int j = bj[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      a3 += __shfl_xor_sync(0xffffffffu, a3, o);
      const float vo = __shfl_xor_sync(0xffffffffu, v, o);
      const int jo = __shfl_xor_sync(0xffffffffu, j, o);
      if (vo > v || (vo == v && jo < j)) { v = vo; j = jo; }
    }
    const int i = r_base + w * kPtsRowsPerWarp + r;
    if (lane == 0 && i < h.n_rows) {
      h.part[pbase + i] = make_float4(a0, a1, a2, a3);
      h.best[pbase + i] = make_float2(v, __int_as_float(j));
    }
  }
}

// per row: fixed-order chunk sums -> mapped point; argmax over chunks (lowest
// index on ties) -> target index and the plan entry pi_ij
static __global__ void k_pts_consume_finish(int B, int n, int m, int d, int chunks, const float4* __restrict__ part,
                                            const float2* __restrict__ best, const float4* __restrict__ rpts,
                                            const float4* __restrict__ cpts, const float* __restrict__ f,
                                            const float* __restrict__ g, const float* __restrict__ lmu,
                                            const float* __restrict__ lnu, const float* __restrict__ scale,
                                            float inv_eps, float* __restrict__ mapped, int* __restrict__ idx,
                                            float* __restrict__ wt, int* __restrict__ zero_rows,
                                            const double* __restrict__ ctr) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, v = -INFINITY;
  int j = 0x7fffffff;
  for (int ch = 0; ch < chunks; ++ch) {
    const size_t k = ((size_t)b * chunks + ch) * n + i;
    const float4 p = part[k];
    a0 += p.x; a1 += p.y; a2 += p.z; a3 += p.w;
    const float2 bb = best[k];
    const int jj = __float_as_int(bb.y);
    if (bb.x > v || (bb.x == v && jj < j)) { v = bb.x; j = jj; }
  }
  const size_t ri = (size_t)b * n + i;
  if (!(a0 > 0.f)) atomicAdd(zero_rows, 1);  // ZeroRowMass (applications.py:92-93)
  // undo the translation of k_pts_pack (points were shifted by the problem's box centre)
  const double* c0 = ctr + (size_t)b * 3;
  const float out[3] = {a1 / a0, a2 / a0, a3 / a0};
  for (int k = 0; k < d; ++k) mapped[ri * d + k] = __double2float_rn(__dadd_rn(double(out[k]), c0[k]));
  if (j == 0x7fffffff) j = 0;
  idx[ri] = j;
  // pi_ij = exp(((f_i + g_j) - c_ij) * inv + lmu_i + lnu_j), c from the fp32 points
  const float4 x = rpts[ri], y = cpts[(size_t)b * m + j];
  const float dx = x.x - y.x, dy = x.y - y.y, dz = x.z - y.z;
  const float c = __fmul_rn(__fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx))), __ldg(scale + b));
  const float z = __fadd_rn(__fadd_rn(__fmul_rn(__fsub_rn(__fadd_rn(f[ri], g[(size_t)b * m + j]), c), inv_eps), lmu[ri]),
                            lnu[(size_t)b * m + j]);
  wt[ri] = expf(z);
}

}  // namespace lsk

namespace lsk {

// Guard fallback without a full-grid launch: one CTA per problem returns
// at once unless some row's stale sum left the band (nflag > 0, rare); then
// it recomputes each flagged row exactly -- max pass, then the shifted sum,
// over all columns in log2 units -- and writes the potential.
static __global__ void __launch_bounds__(256) k_pts_fixup(PtsHalf h, float neg_eps, float* __restrict__ rpot_new,
                                                          int* __restrict__ rowflag, int* __restrict__ nflag) {
  __shared__ float red[64];
  if (*nflag == 0) return;
  const int b = blockIdx.x;
  if (h.active && !h.active[b]) return;
  const float sc = __ldg(h.scale + b);
  const float NK = -__fmul_rn(__fmul_rn(h.inv_eps, kLog2e), sc);
  for (int r = h.row_lo; r < h.row_hi; ++r) {
    const size_t ri = (size_t)b * h.n_rows + r;
    if (!rowflag[ri]) continue;  // uniform: every thread reads the same flag
    const float4 x = h.rpts[ri];
    auto v_of = [&](int j) {
      const size_t cj = (size_t)b * h.n_cols + j;
      const float4 y = h.cpts[cj];
      const float A = __fmul_rn(__fmaf_rn(h.cpot[cj], h.inv_eps, h.clw[cj]), kLog2e);
      const float d0 = x.x - y.x, d1 = x.y - y.y, d2 = x.z - y.z;
      return __fmaf_rn(__fmaf_rn(d2, d2, __fmaf_rn(d1, d1, d0 * d0)), NK, A);
    };
    float mx[1] = {-INFINITY};
    for (int j = threadIdx.x; j < h.n_cols; j += 256) mx[0] = fmax_nan(mx[0], v_of(j));
    block_reduce<256, 1, true>(mx, red);
    const float M = mx[0];
    const float Ms = (fabsf(M) <= 3.402823466e38f) ? M : 0.f;
    float s[1] = {0.f};
    for (int j = threadIdx.x; j < h.n_cols; j += 256) s[0] += ex2(v_of(j) - Ms);
    __syncthreads();
    block_reduce<256, 1, false>(s, red + 32);
    if (threadIdx.x == 0) {
      float L;  // LSE in natural units: M log2-units * ln2 + ln S (reduction.py:196-207)
      if (!(fabsf(M) <= 3.402823466e38f)) L = -INFINITY;
      else L = __fadd_rn(__fmul_rn(M, 0.6931471805599453f), logf(fmaxf(s[0], kSumFloor)));
      rpot_new[ri] = __fmul_rn(neg_eps, L);
      rowflag[ri] = 0;
    }
    __syncthreads();
  }
}

}  // namespace lsk

namespace lsk {

// Exact fp64 max of the squared-Euclidean cost without 2 n m fp64 evaluations:
// MODE 0 screens all pairs in fp32 (translated points, < 1e-6 relative error,
// see lsk_points.cu) for max32; MODE 1 re-evaluates in fp64 -- the reference's
// direct coordinate sum (costs.py:48-49) on the original points -- only the
// pairs whose fp32 value is within 1e-5 of max32, and keeps their exact max.
template <int MODE>
static __global__ void __launch_bounds__(kPtsThreads) k_pts_cmax2(int n, int m, int d, const float4* __restrict__ X4,
                                                                 const float4* __restrict__ Y4,
                                                                 const double* __restrict__ X,
                                                                 const double* __restrict__ Y,
                                                                 unsigned* __restrict__ max32,
                                                                 unsigned long long* __restrict__ max64) {
  __shared__ __align__(16) float4 colv[kPtsChunk];
  const int ch = blockIdx.x, tile = blockIdx.y, b = blockIdx.z;
  const int r_base = tile * kPtsTileRows;
  if (r_base >= n) return;
  const int j0 = ch * kPtsChunk, ncol = min(kPtsChunk, m - j0);
  for (int t = threadIdx.x; t < ncol; t += kPtsThreads) colv[t] = Y4[(size_t)b * m + j0 + t];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float x0[8], x1[8], x2[8];
  int ri[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int i = r_base + w * kPtsRowsPerWarp + r;
    ri[r] = i < n ? i : -1;
    const float4 x = X4[(size_t)b * n + (i < n ? i : n - 1)];
    x0[r] = x.x; x1[r] = x.y; x2[r] = x.z;
  }
  const float T = (MODE == 1) ? __uint_as_float(max32[b]) * (1.0f - 1e-5f) : 0.f;
  __syncthreads();
  float mx = 0.f;
  for (int t = lane; t < ncol; t += 32) {
    const float4 q = colv[t];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float dx = x0[r] - q.x, dy = x1[r] - q.y, dz = x2[r] - q.z;
      const float v = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
      if (MODE == 0) {
        mx = (ri[r] >= 0 && v > mx) ? v : mx;
      } else if (ri[r] >= 0 && v >= T) {  // rare: exact fp64 re-evaluation
        const double* xp = X + ((size_t)b * n + ri[r]) * d;
        const double* yp = Y + ((size_t)b * m + j0 + t) * d;
        double acc = 0.0;
        for (int k = 0; k < d; ++k) {
          const double dd = __dsub_rn(xp[k], yp[k]);
          acc = (k == 0) ? __dmul_rn(dd, dd) : __dadd_rn(acc, __dmul_rn(dd, dd));
        }
        atomicMax(max64 + b, static_cast<unsigned long long>(__double_as_longlong(acc)));
      }
    }
  }
  if (MODE == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) atomicMax(max32 + b, __float_as_uint(mx));  // non-negative: bits order like values
  }
}


// Exact fp64 min of the direct coordinate sum (costs.py:48-49) per problem:
// value_range = max - min decides the C / C.max() of applications.py:186-188.
// One thread per column j, 64 rows per CTA (row loads are warp-uniform).
static __global__ void __launch_bounds__(256) k_pts_cmin64(int n, int m, int d, const double* __restrict__ X,
                                                          const double* __restrict__ Y,
                                                          unsigned long long* __restrict__ min64) {
  const int b = blockIdx.z;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = blockIdx.y * 64;
  double y[3] = {0.0, 0.0, 0.0};
  if (j < m)
    for (int k = 0; k < d; ++k) y[k] = Y[((size_t)b * m + j) * d + k];
  double mn = INFINITY;
  const int i1 = min(n, i0 + 64);
  for (int i = i0; i < i1; ++i) {
    const double* xp = X + ((size_t)b * n + i) * d;
    double acc = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = __dsub_rn(xp[k], y[k]);
      acc = (k == 0) ? __dmul_rn(t, t) : __dadd_rn(acc, __dmul_rn(t, t));
    }
    mn = fmin(mn, acc);
  }
  if (j >= m) mn = INFINITY;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) atomicMin(min64 + b, static_cast<unsigned long long>(__double_as_longlong(mn)));
}

}  // namespace lsk

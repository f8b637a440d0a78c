// Persistent one-pass standard-domain Sinkhorn (fp32, m <= 8192): the whole
// u/v alternation of solver.py:340-431 as ONE cooperative launch that reads
// the materialised K = exp(-C/eps) once per iteration.
//
// CTA b owns rows [b n/G, (b+1) n/G); thread t owns columns
// j = 4 (v NT + t) + q, so v_j and the column accumulator stay in registers as
// packed pairs. K rows stream through the same TMA ring + mbarrier row hand-off
// as the log-domain solver: at step q every warp adds its share of row q's dot
// (K v^{k-1})_q, and once the NW warp sums of row q-1 are posted it forms
// u_{q-1} = mu / (K v)_{q-1} (IEEE division, unguarded as the reference) and
// adds K_{q-1,j} u_{q-1} into its column accumulators. After the pass the G
// column partials are combined in a fixed order into v^k = nu / (K^T u^k).
// The checkpoint of iterate k (finiteness of u^k and v^k, then
// err = sum_i |u^k_i (K v^k)_i - mu_i|) is evaluated inside pass k+1, whose dot
// products are exactly (K v^k); u and v are double buffered so a stop at k
// returns iterate k. A cap that is not checked in the loop gets one dot-only
// pass. Traffic: n m 4 bytes per iteration (one read of K).
#pragma once
#include "lsk_device.cuh"

namespace lsk {

struct StdArgs {
  const float* K;
  long long ldk;
  int n, m, mpad;
  const float* mu;
  const float* nu;
  double tol;
  int max_iter, check;
  float* u0; float* u1;  // u^k in u[k & 1]; u0 = 1
  float* v0; float* v1;  // v^k in v[k & 1]; v0 = 1 (0 beyond m)
  float* part;           // [G][W] column partials
  float* errpart;        // [G]
  int* flagpart;         // [G]
  unsigned long long* bar;
  // outputs (the StdState of lsk_standard.cu: active, status, iters, ntrace, err)
  int* st_active; int* st_status; int* st_iters; int* st_ntrace; float* st_err;
  int* out_buf;          // buffer index holding the returned u / v
  int* trace_iter;
  float* trace_err;
  int cap;
};

template <int NT, int V, int STAGES>
struct StdSolver {
  static constexpr int P2 = 2 * V;
  static constexpr int W = 4 * V * NT;
  static constexpr int NW = NT / 32;
  static constexpr size_t kRingBytes = size_t(STAGES) * W * sizeof(float);
  static constexpr int kRedFloats = 2 * NW + 64 * NW;  // row sums [2][NW]; combine scratch
  static constexpr size_t kSmemBytes = kRingBytes + kRedFloats * sizeof(float) + (STAGES + 2) * 8 + 64;

  const StdArgs& a;
  float* ring;
  float* red;
  uint64_t* mbar;
  uint64_t* bsum;
  int b, G, r0, r1, rows;
  int head_st, head_ph, pass;
  unsigned gstep, epoch;
  f2 v2[P2], ac2[P2];

  __device__ StdSolver(const StdArgs& args, unsigned char* smem) : a(args) {
    ring = reinterpret_cast<float*>(smem);
    red = reinterpret_cast<float*>(smem + kRingBytes);
    mbar = reinterpret_cast<uint64_t*>(smem + kRingBytes + kRedFloats * sizeof(float));
    bsum = mbar + STAGES;
    b = blockIdx.x;
    G = gridDim.x;
    r0 = int((long long)b * a.n / G);
    r1 = int((long long)(b + 1) * a.n / G);
    rows = r1 - r0;
    head_st = head_ph = pass = 0;
    gstep = epoch = 0;
  }
  __device__ __forceinline__ int col(int v, int q) const { return 4 * (v * NT + threadIdx.x) + q; }
  __device__ __forceinline__ int row_of(int P, int q) const { return (P & 1) ? (r1 - 1 - q) : (r0 + q); }

  // ---- TMA ring (the sequence of rows: pass P visits its rows in direction P & 1)
  __device__ void issue(int st, int P, int q) {
    while (q >= rows) { q -= rows; ++P; }
    const uint32_t bytes = uint32_t(a.mpad) * 4u;
    mbar_expect_tx(&mbar[st], bytes);
    tma_load_1d(ring + size_t(st) * W, a.K + (long long)row_of(P, q) * a.ldk, bytes, &mbar[st]);
  }
  __device__ void ring_init() {
    float4* r4 = reinterpret_cast<float4*>(ring);
    for (size_t k = threadIdx.x; k < kRingBytes / 16; k += NT) r4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) mbar_init(&mbar[s], 1);
#ifdef LSK_X_ALLARRIVE  // sanitizer builds: every thread arrives (see lsk_dense.cuh kSumArrivals)
      mbar_init(&bsum[0], NT);
      mbar_init(&bsum[1], NT);
#else
      mbar_init(&bsum[0], NW);
      mbar_init(&bsum[1], NW);
#endif
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (int s = 0; s < STAGES; ++s) issue(s, 0, s);
    }
  }
  __device__ __forceinline__ const float* wait_head() {
    mbar_wait(&mbar[head_st], uint32_t(head_ph));
    const float* p = ring + size_t(head_st) * W;
    if (++head_st == STAGES) { head_st = 0; head_ph ^= 1; }
    return p;
  }
  __device__ __forceinline__ void refill(int st, int P, int q) {
    if (threadIdx.x == 0) {
      fence_proxy_async();
      issue(st, P, q + STAGES);
    }
  }
  __device__ __forceinline__ void post(unsigned step, float s) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      red[(step & 1) * NW + (threadIdx.x >> 5)] = s;
#ifndef LSK_X_ALLARRIVE
      mbar_arrive(&bsum[step & 1]);
#endif
    }
#ifdef LSK_X_ALLARRIVE
    mbar_arrive(&bsum[step & 1]);
#endif
  }
  __device__ __forceinline__ float posted_sum(unsigned step) {
    mbar_wait(&bsum[step & 1], (step >> 1) & 1);
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; w += 4) {
      const float4 t = *reinterpret_cast<const float4*>(red + (step & 1) * NW + w);
      s += (t.x + t.y) + (t.z + t.w);
    }
    return s;
  }
  __device__ __forceinline__ void load_row(const float* base, f2 (&c)[P2]) const {
#pragma unroll
    for (int v = 0; v < V; ++v) lds2x2(base + 4 * (v * NT + threadIdx.x), c[2 * v], c[2 * v + 1]);
  }
  // this thread's share of (K v)_row
  __device__ __forceinline__ float dot(const float* row) const {
    f2 c[P2];
    load_row(row, c);
    f2 s2 = 0ull;
#pragma unroll
    for (int p = 0; p < P2; ++p) s2 = fma2(c[p], v2[p], s2);
    float s0, s1;
    up2(s2, s0, s1);
    return s0 + s1;
  }
  template <bool SHFL>
  __device__ __forceinline__ void col_update(const float* row, float u, float& s) {
    f2 c[P2];
    load_row(row, c);
    const f2 u2 = pk2(u, u);
#pragma unroll
    for (int p = 0; p < P2; ++p) {
      ac2[p] = fma2(c[p], u2, ac2[p]);
      if (SHFL && p < 5) s += __shfl_xor_sync(0xffffffffu, s, 16 >> p);
    }
    if (SHFL)
#pragma unroll
      for (int l = P2; l < 5; ++l) s += __shfl_xor_sync(0xffffffffu, s, 16 >> l);
  }
  __device__ bool load_v(const float* v) {
    bool bad = false;
#pragma unroll
    for (int w = 0; w < V; ++w) {
      const int j0 = col(w, 0);
      float4 t = j0 < a.m ? ldcg4(reinterpret_cast<const float4*>(v + j0)) : make_float4(0.f, 0.f, 0.f, 0.f);
      float x[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (j0 + q >= a.m) x[q] = 0.f;
        else bad |= !isfinite(x[q]);
      }
      v2[2 * w] = pk2(x[0], x[1]);
      v2[2 * w + 1] = pk2(x[2], x[3]);
      ac2[2 * w] = 0ull;
      ac2[2 * w + 1] = 0ull;
    }
    return bad;
  }

  // one pass: u_new from (K v^{k-1}); with CHECK (or DOT_ONLY) the checkpoint
  // term of the previous iterate |u_old (K v)_i - mu_i| and its finiteness
  template <bool CHECK, bool DOT_ONLY>
  __device__ void run_pass(const float* uold, float* unew, float& err_acc, int& bad) {
    const int P = pass++;
    const unsigned g0 = gstep;
    int st = head_st;
    const float* row = wait_head();
    float s = warp_sum(dot(row));
    post(g0, s);
    const float* row_p = row;
    int st_p = st, st_pp = 0;
    int i_p = row_of(P, 0);
    auto finish = [&](int i, float S) -> float {
      if (CHECK && threadIdx.x == 0) {
        const float uo = ldcg(uold + i);
        err_acc += fabsf(__fsub_rn(__fmul_rn(uo, S), __ldg(a.mu + i)));
        if (!isfinite(uo)) bad = 1;
      }
      if (DOT_ONLY) return 0.f;
      const float u = __fdiv_rn(__ldg(a.mu + i), S);
      if (threadIdx.x == 0) unew[i] = u;
      return u;
    };
    for (int q = 1; q < rows; ++q) {
      st = head_st;
      row = wait_head();
      const float S = posted_sum(g0 + q - 1);
      if (q >= 2) refill(st_pp, P, q - 2);
      float sq = dot(row);
      const float u = finish(i_p, S);
      if (!DOT_ONLY) col_update<true>(row_p, u, sq);
      else sq = warp_sum(sq);
      post(g0 + q, sq);
      st_pp = st_p;
      row_p = row;
      st_p = st;
      i_p = row_of(P, q);
    }
    const float S = posted_sum(g0 + rows - 1);
    if (rows >= 2) refill(st_pp, P, rows - 2);
    const float u = finish(i_p, S);
    float dummy = 0.f;
    if (!DOT_ONLY) col_update<false>(row_p, u, dummy);
    __syncthreads();
    refill(st_p, P, rows - 1);
    gstep = g0 + rows;
  }

  __device__ float tree_over_ctas(const float* v) {
    float s = 0.f;
    for (int k = threadIdx.x & 31; k < G; k += 32) s += ldcg(v + k);
    return warp_sum(s);
  }
  __device__ int any_over_ctas(const int* v) {
    int s = 0;
    for (int k = threadIdx.x & 31; k < G; k += 32) s |= __ldcg(v + k);
    return __any_sync(0xffffffffu, s != 0);
  }
  // checkpoint decision (solver.py:380-411), identical in every CTA
  __device__ bool decide(int kk, bool final) {
    const int isbad = any_over_ctas(a.flagpart);
    const float err = tree_over_ctas(a.errpart);
    int status = 0;
    bool stop = false, append = true;
    float e = err;
    if (isbad) { stop = true; status = 2; e = NAN; append = false; }
    else if (!isfinite(err)) { stop = true; status = 2; }
    else if (err < float(a.tol)) { stop = true; status = 1; }
    if (b == 0 && threadIdx.x == 0) {
      if (append && *a.st_ntrace < a.cap) {
        a.trace_iter[*a.st_ntrace] = kk;
        a.trace_err[*a.st_ntrace] = err;
        *a.st_ntrace += 1;
      }
      *a.st_status = status;
      *a.st_err = e;
      if (stop || final) {
        *a.st_iters = kk;
        *a.out_buf = kk & 1;
        *a.st_active = 0;
      }
    }
    return stop;
  }
  __device__ void publish(float err_acc, int bad) {
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) { a.errpart[b] = err_acc; a.flagpart[b] = bad; }
  }
  // column owners: v_j = nu_j / sum_b part[b][j] (fixed order)
  __device__ void combine(float* vnew) {
    const int j0 = int((long long)b * a.m / G), j1 = int((long long)(b + 1) * a.m / G);
    for (int j = j0 + threadIdx.x; j < j1; j += NT) {
      float s = 0.f;
      for (int k = 0; k < G; ++k) s += ldcg(a.part + (size_t)k * W + j);
      vnew[j] = __fdiv_rn(__ldg(a.nu + j), s);
    }
  }
  __device__ void store_partials() {
#pragma unroll
    for (int w = 0; w < V; ++w) {
      if (col(w, 0) >= a.m) continue;
      float x0, x1, x2, x3;
      up2(ac2[2 * w], x0, x1);
      up2(ac2[2 * w + 1], x2, x3);
      reinterpret_cast<float4*>(a.part + (size_t)b * W)[w * NT + threadIdx.x] = make_float4(x0, x1, x2, x3);
    }
  }

  __device__ void solve() {
    auto ub = [&](int k) { return (k & 1) ? a.u1 : a.u0; };
    auto vb = [&](int k) { return (k & 1) ? a.v1 : a.v0; };
    ring_init();
    bool stopped = false;
    for (int k = 1; k <= a.max_iter; ++k) {
      const bool do_check = (k > 1) && ((k - 1) % a.check == 0);
      const bool vbad = load_v(vb(k - 1));
      float err_acc = 0.f;
      int bad = (do_check && vbad) ? 1 : 0;
      if (do_check) run_pass<true, false>(ub(k - 1), ub(k), err_acc, bad);
      else run_pass<false, false>(ub(k - 1), ub(k), err_acc, bad);
      store_partials();
      if (do_check) publish(err_acc, bad);
      grid_barrier(a.bar, epoch);
      if (do_check && decide(k - 1, false)) { stopped = true; break; }
      combine(vb(k));
      grid_barrier(a.bar, epoch);
    }
    if (!stopped) {  // the checkpoint at the cap (in-loop if K % c == 0, else the extra one)
      const int K = a.max_iter;
      const bool vbad = load_v(vb(K));
      float err_acc = 0.f;
      int bad = vbad ? 1 : 0;
      run_pass<true, true>(ub(K), nullptr, err_acc, bad);
      publish(err_acc, bad);
      grid_barrier(a.bar, epoch);
      decide(K, true);
    }
    for (int s = 0; s < STAGES; ++s) wait_head();  // drain the ring
    __syncthreads();
  }
};

}  // namespace lsk

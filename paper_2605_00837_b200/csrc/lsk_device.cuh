// Device-side building blocks for the B200 log-domain Sinkhorn kernels.
//
// Arithmetic contract (SURVEY.md 8(a'); reference solver.py:76-115,
// reduction.py:179-208): every potential / check / cost ARGUMENT is built with
// separately rounded fp32 ops (__fsub_rn/__fmul_rn/__fadd_rn, never an FMA),
// because contracting (g - C) * inv_eps + log_nu into an FFMA moves the
// potentials by 1.3e-5 at eps=1e-4. Only what happens AFTER the
// argument is rounded -- the shift, the exponential, the summation order -- is
// free, and that is where the kernels get their speed (ex2.approx on the MUFU
// pipe, fused shift+scale FFMA, warp-shuffle trees).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lsk {

constexpr float kLog2e = 1.4426950408889634f;   // fl(log2 e)
constexpr float kSumFloor = 1e-30f;             // reduction.py:44 SUM_FLOOR
// Stale-shift sums outside [kShiftLo, kShiftHi] are recomputed exactly. With
// ex2.approx.ftz, flushed terms are < 1.2e-38 each, so a sum >= 1e-20 is
// exact to ~1e-13 relative even at 65536 terms.
constexpr float kShiftLo = 1e-20f;
constexpr float kShiftHi = 1e30f;

// ---- the reference's three separately rounded ops: fl(fl(fl(a - c) * s) + l)
__device__ __forceinline__ float arg3(float a, float c, float inv_eps, float l) {
  return __fadd_rn(__fmul_rn(__fsub_rn(a, c), inv_eps), l);
}
// check argument: fl(fl(fl(fl(f + g) - c) * s) + l)   (solver.py:98-101)
__device__ __forceinline__ float arg4(float f, float g, float c, float inv_eps, float l) {
  return __fadd_rn(__fmul_rn(__fsub_rn(__fadd_rn(f, g), c), inv_eps), l);
}

// exp(x - shift) as 2^(x*log2e - shift*log2e): x is the exactly rounded
// reference argument; the FFMA only re-rounds the (small) post-shift value and
// a per-row/column constant, i.e. the SURVEY F4/F10 "free" part.
__device__ __forceinline__ float ex2(float t) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(t));
  return y;
}
__device__ __forceinline__ float exp_shifted(float x, float shift_l2e) {
  return ex2(__fmaf_rn(x, kLog2e, -shift_l2e));
}

// NaN-propagating max, like np.maximum (reduction.py:160).
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float y;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(y) : "f"(a), "f"(b));
  return y;
}

// ---- warp reductions (xor butterfly: every lane ends with identical bits,
// since each level adds the same two operands in swapped order).
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// (max, sum) pair merge: the online max-rescale combine.
__device__ __forceinline__ void pair_merge(float& m, float& s, float m2, float s2) {
  float mm = fmax_nan(m, m2);
  float a = (m == mm) ? 1.f : ex2((m - mm) * kLog2e);
  float b = (m2 == mm) ? 1.f : ex2((m2 - mm) * kLog2e);
  if (!(mm > -INFINITY)) { a = 1.f; b = 1.f; }   // both empty / NaN: keep sums
  s = s * a + s2 * b;
  m = mm;
}
__device__ __forceinline__ void warp_pair(float& m, float& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    pair_merge(m, s, m2, s2);
  }
}

// Block-wide sum/max of K values per thread, one __syncthreads. `red` holds
// K * 32 floats. Every thread returns the identical result.
template <int NT, int K, bool MAX>
__device__ __forceinline__ void block_reduce(float (&v)[K], float* red) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    v[k] = MAX ? warp_max(v[k]) : warp_sum(v[k]);
    if (lane == 0) red[k * 32 + w] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float t = lane < NW ? red[k * 32 + lane] : (MAX ? -INFINITY : 0.f);
    v[k] = MAX ? warp_max(t) : warp_sum(t);
  }
}

// Block-wide (max, sum) pair reduction, one __syncthreads; `red` holds 64*K.
template <int NT, int K>
__device__ __forceinline__ void block_pair(float (&m)[K], float (&s)[K], float* red) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    warp_pair(m[k], s[k]);
    if (lane == 0) { red[k * 64 + w] = m[k]; red[k * 64 + 32 + w] = s[k]; }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float mm = lane < NW ? red[k * 64 + lane] : -INFINITY;
    float ss = lane < NW ? red[k * 64 + 32 + lane] : 0.f;
    warp_pair(mm, ss);
    m[k] = mm; s[k] = ss;
  }
}

// LSE finalisation exactly as reduction.py:196-207 given the shift M and the
// shifted sum S: non-finite M (an all -inf / NaN row) yields -inf.
__device__ __forceinline__ float lse_finish(float M, float S) {
  // select, not branch: keeps the logf chain in the caller's basic block so it
  // can be scheduled under independent MUFU work
  const float r = __fadd_rn(M, logf(fmaxf(S, kSumFloor)));
  return (fabsf(M) <= 3.402823466e38f) ? r : -INFINITY;
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Watchdog for every spin in the persistent solver: a wait longer than this
// is a bug (lost TMA bytes, a CTA that never arrives); trap instead of hanging.
constexpr uint64_t kSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;

// non-blocking probe of a phase (acquire semantics when it returns true)
__device__ __forceinline__ bool mbar_test(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the thread sleeps in hardware until the
// phase completes (or the hint expires) instead of spinning on issue slots
__device__ __forceinline__ bool mbar_try_wait_sleep(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try_wait_sleep(addr, parity)) {
    if (globaltimer_ns() - t0 > kSpinTimeoutNs) __trap();
  }
}
// spin variant for short hand-offs between warps of one CTA: plain try_wait
// (hardware-suspending, no nanosleep), watchdog checked only every 4096 tries
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t tries = 0;
  uint64_t t0 = 0;
  while (!mbar_try_wait(addr, parity)) {
    if ((++tries & 4095u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > kSpinTimeoutNs) __trap();
    }
  }
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// bulk prefetch of [src, src+bytes) into L2 (no smem, no completion tracking)
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---- L2-coherent loads for data produced by other CTAs of the same launch.
__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ float4 ldcg4(const float4* p) { return __ldcg(p); }

// ---- software grid barrier for the persistent (cooperatively launched)
// solver: a monotonic arrival counter, so no reset race; target = (#barriers
// passed so far) * gridDim.x.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long atom_add_acqrel64(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
// Grid barrier on a 64-bit counter: the low word counts arrivals, the high
// word accumulates a per-CTA flag (e.g. "a guard fired in my rows"), so the
// barrier also delivers the grid-wide OR without another L2 round trip.
// Returns the high word as seen at release (exact as long as two flagged
// barriers are always separated by an unflagged one). `scratch` is one
// shared-memory word used to broadcast thread 0's result.
__device__ __forceinline__ unsigned grid_barrier(unsigned long long* counter, unsigned& epoch, unsigned flag = 0,
                                                 unsigned* scratch = nullptr) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    const unsigned target = epoch * gridDim.x;
    // acq_rel add (releases this CTA's writes, ordered before it by the
    // bar.sync above; acquires when it is the last arrival), else acquire
    // polling; the trailing bar.sync extends the acquire to the whole CTA
    unsigned long long v = atom_add_acqrel64(counter, 1ull | (static_cast<unsigned long long>(flag) << 32)) +
                           (1ull | (static_cast<unsigned long long>(flag) << 32));
    if (static_cast<unsigned>(v) < target) {
      const uint64_t t0 = globaltimer_ns();
      while (static_cast<unsigned>(v = ld_acquire64(counter)) < target)
        if (globaltimer_ns() - t0 > kSpinTimeoutNs) __trap();
    }
    if (scratch) *scratch = static_cast<unsigned>(v >> 32);
  }
  __syncthreads();
  return scratch ? *scratch : 0u;
}

}  // namespace lsk

namespace lsk {
// ---- packed fp32 pairs (sm_100a add/sub/mul/fma.rn.f32x2 -> FADD2/FMUL2/FFMA2).
// Each lane of a packed op is ONE IEEE round-to-nearest op, so the reference's
// separately rounded argument build is preserved bit for bit while the FMA
// pipe issue count halves (profiles/r1_v1_dense_ncu.md).
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2 ex2x2(f2 t) {
  float a, b;
  up2(t, a, b);
  return pk2(ex2(a), ex2(b));
}
// two packed pairs (4 consecutive floats) from shared memory
__device__ __forceinline__ void lds2x2(const float* p, f2& lo, f2& hi) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(smem_u32(p)));
}
// fl(fl(u * s) + l) lane-wise. ptxas contracts a packed mul.rn.f32x2 feeding
// add.rn.f32x2 into one FFMA2 even with -fmad=false (the .rn qualifiers do not
// stop it on f32x2), which would break the reference's separately rounded
// argument build. The product is therefore formed as
// fma(u, s, z) with z a RUNTIME -0.0 pair (kernel argument, opaque to the
// compiler): u*s + (-0) is exactly the rounded product (sign of zero
// included), and an fma cannot be fused with the following add.
// tests/test_gpu_parity.py::test_argument_build_bitwise checks the bits.
__device__ __forceinline__ f2 muladd_rn2(f2 u, f2 s, f2 l, f2 z) { return add2(fma2(u, s, z), l); }
// reference argument fl(fl(fl(a - c) * s) + l), lane-wise
__device__ __forceinline__ f2 arg3x2(f2 a, f2 c, f2 s, f2 l, f2 z) { return muladd_rn2(sub2(a, c), s, l, z); }
// check argument fl(fl(fl(fl(f + g) - c) * s) + l), lane-wise
__device__ __forceinline__ f2 arg4x2(f2 f, f2 g, f2 c, f2 s, f2 l, f2 z) {
  return muladd_rn2(sub2(add2(f, g), c), s, l, z);
}
}  // namespace lsk

namespace lsk {
// plain mbarrier arrive (release.cta): producer -> consumer hand-off in smem
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// shared-memory counter increment with acq_rel ordering; returns the old value
__device__ __forceinline__ unsigned atom_add_acqrel_smem(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}
}  // namespace lsk

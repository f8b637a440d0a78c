// Row-step microbenchmark of the dense solver's inner loop with the memory
// system taken out: every row comes from the same shared-memory buffer, so
// only the instruction stream and the synchronisation remain. Prints cycles
// per row per CTA (one CTA per SM, 148 CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I../../paper_2605_00837_b200/csrc \
//        -o rowstep rowstep.cu && ./rowstep
//
// variants: TEAMS in {1, 2} (8-warp teams, 32 columns per thread), SYNC
// (team barrier per row), FIN (the accurate logf finish of the previous row),
// GSM (g read from shared memory instead of registers)
#include <cstdio>

#include "lsk_device.cuh"

using namespace lsk;

#ifndef RS_WARPS
#define RS_WARPS 8
#endif
constexpr int NT = 32 * RS_WARPS, V = 64 / RS_WARPS, P2 = 2 * V, W = 4 * V * NT, ROWS = 512;

template <int TEAMS, bool SYNC, bool FIN, bool GSM>
__global__ void __launch_bounds__(NT * TEAMS, 1) kern(float* out, unsigned long long* cyc, float negzero) {
  extern __shared__ __align__(16) float sm[];
  float* row = sm;          // [W]
  float* gs = sm + W;       // [W]
  float* red = sm + 2 * W;  // [TEAMS][2][8]
  const int team = threadIdx.x / NT, tid = threadIdx.x % NT, lane = tid & 31, w = tid >> 5;
  for (int j = threadIdx.x; j < W; j += blockDim.x) {
    row[j] = 0.5f + 1e-4f * (j % 97);
    gs[j] = 0.3f + 1e-4f * (j % 89);
  }
  __syncthreads();
  const f2 inv2 = pk2(1000.f, 1000.f), l2e2 = pk2(kLog2e, kLog2e), nz2 = pk2(negzero, negzero);
  const f2 lnu2 = pk2(-9.f, -9.f);
  f2 g2[P2], ac2[P2], e[P2];
#pragma unroll
  for (int p = 0; p < P2; ++p) {
    g2[p] = pk2(0.3f + 1e-4f * p, 0.3f);
    ac2[p] = 0ull;
    e[p] = 0ull;
  }
  float fold = 0.25f, lmu = -9.f;
  unsigned long long t0 = clock64();
  for (int k = 0; k < ROWS; ++k) {
    if (SYNC) {
      if (TEAMS == 1) __syncthreads();
      else asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(NT) : "memory");
    }
    const int pb = (k - 1) & 1;
    float S = 0.f;
#pragma unroll
    for (int q = 0; q < RS_WARPS; q += 4) {
      const float4 t = *reinterpret_cast<const float4*>(red + team * 64 + pb * 32 + q);
      S += (t.x + t.y) + (t.z + t.w);
    }
    float fi = fold + 1e-7f * S;
    if (FIN) fi = __fmul_rn(-1e-3f, lse_finish(__fmul_rn(-fold, 1000.f), S + 1.f));
    const float ai = __fmul_rn(__fadd_rn(__fmul_rn(__fsub_rn(fi, fold), 1000.f), lmu), kLog2e);
    const float A = ex2(fminf(ai, 0.f));
    const f2 A2 = pk2(A, A);
#pragma unroll
    for (int p = 0; p < P2; ++p) ac2[p] = fma2(e[p], A2, ac2[p]);
    const float shl = __fmul_rn(__fmul_rn(-fi, 1000.f), kLog2e);
    const f2 nsl = pk2(-shl, -shl);
    f2 s2 = 0ull;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      f2 c0, c1, gg0, gg1;
      lds2x2(row + 4 * (v * NT + tid), c0, c1);
      if (GSM) lds2x2(gs + 4 * (v * NT + tid), gg0, gg1);
      else { gg0 = g2[2 * v]; gg1 = g2[2 * v + 1]; }
      e[2 * v] = ex2x2(fma2(arg3x2(gg0, c0, inv2, lnu2, nz2), l2e2, nsl));
      e[2 * v + 1] = ex2x2(fma2(arg3x2(gg1, c1, inv2, lnu2, nz2), l2e2, nsl));
      s2 = add2(s2, add2(e[2 * v], e[2 * v + 1]));
    }
    float s0, s1;
    up2(s2, s0, s1);
    float s = warp_sum(s0 + s1);
    if (lane == 0) red[team * 64 + (k & 1) * 32 + w] = s;
    fold = fi;
  }
  unsigned long long t1 = clock64();
  float acc = fold;
#pragma unroll
  for (int p = 0; p < P2; ++p) { float a0, a1; up2(ac2[p], a0, a1); acc += a0 + a1; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// two rows per step: one barrier, both rows' finish (independent chains) and
// column updates, then both rows' f-side terms (e for 2 rows in registers)
__global__ void __launch_bounds__(NT, 1) kern_r2(float* out, unsigned long long* cyc, float negzero) {
  extern __shared__ __align__(16) float sm[];
  float* row = sm;
  float* red = sm + 2 * W;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int j = threadIdx.x; j < W; j += blockDim.x) row[j] = 0.5f + 1e-4f * (j % 97);
  __syncthreads();
  const f2 inv2 = pk2(1000.f, 1000.f), l2e2 = pk2(kLog2e, kLog2e), nz2 = pk2(negzero, negzero);
  const f2 lnu2 = pk2(-9.f, -9.f);
  f2 g2[P2], ac2[P2], e0[P2], e1[P2];
#pragma unroll
  for (int p = 0; p < P2; ++p) {
    g2[p] = pk2(0.3f + 1e-4f * p, 0.3f);
    ac2[p] = 0ull;
    e0[p] = 0ull;
    e1[p] = 0ull;
  }
  float fold0 = 0.25f, fold1 = 0.26f, lmu = -9.f;
  unsigned long long t0 = clock64();
  for (int k = 0; k < ROWS / 2; ++k) {
    __syncthreads();
    const int pb = (k - 1) & 1;
    float S0 = 0.f, S1 = 0.f;
#pragma unroll
    for (int q = 0; q < RS_WARPS; q += 4) {
      const float4 t = *reinterpret_cast<const float4*>(red + pb * 64 + q);
      const float4 u = *reinterpret_cast<const float4*>(red + pb * 64 + 32 + q);
      S0 += (t.x + t.y) + (t.z + t.w);
      S1 += (u.x + u.y) + (u.z + u.w);
    }
    const float fi0 = __fmul_rn(-1e-3f, lse_finish(__fmul_rn(-fold0, 1000.f), S0 + 1.f));
    const float fi1 = __fmul_rn(-1e-3f, lse_finish(__fmul_rn(-fold1, 1000.f), S1 + 1.f));
    const float a0 = __fmul_rn(__fadd_rn(__fmul_rn(__fsub_rn(fi0, fold0), 1000.f), lmu), kLog2e);
    const float a1 = __fmul_rn(__fadd_rn(__fmul_rn(__fsub_rn(fi1, fold1), 1000.f), lmu), kLog2e);
    const float A0 = ex2(fminf(a0, 0.f)), A1 = ex2(fminf(a1, 0.f));
    const f2 A20 = pk2(A0, A0), A21 = pk2(A1, A1);
#pragma unroll
    for (int p = 0; p < P2; ++p) ac2[p] = fma2(e1[p], A21, fma2(e0[p], A20, ac2[p]));
    const float shl0 = __fmul_rn(__fmul_rn(-fold0, 1000.f), kLog2e), shl1 = __fmul_rn(__fmul_rn(-fold1, 1000.f), kLog2e);
    const f2 nsl0 = pk2(-shl0, -shl0), nsl1 = pk2(-shl1, -shl1);
    f2 s20 = 0ull, s21 = 0ull;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      f2 c0, c1, d0, d1;
      lds2x2(row + 4 * (v * NT + tid), c0, c1);
      lds2x2(row + 4 * (v * NT + tid) + 64, d0, d1);
      e0[2 * v] = ex2x2(fma2(arg3x2(g2[2 * v], c0, inv2, lnu2, nz2), l2e2, nsl0));
      e0[2 * v + 1] = ex2x2(fma2(arg3x2(g2[2 * v + 1], c1, inv2, lnu2, nz2), l2e2, nsl0));
      e1[2 * v] = ex2x2(fma2(arg3x2(g2[2 * v], d0, inv2, lnu2, nz2), l2e2, nsl1));
      e1[2 * v + 1] = ex2x2(fma2(arg3x2(g2[2 * v + 1], d1, inv2, lnu2, nz2), l2e2, nsl1));
      s20 = add2(s20, add2(e0[2 * v], e0[2 * v + 1]));
      s21 = add2(s21, add2(e1[2 * v], e1[2 * v + 1]));
    }
    float x0, x1, y0, y1;
    up2(s20, x0, x1);
    up2(s21, y0, y1);
    float s0 = x0 + x1, s1 = y0 + y1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) { red[(k & 1) * 64 + w] = s0; red[(k & 1) * 64 + 32 + w] = s1; }
    fold0 = fi0 * 0.999f + 0.25f;  // the next rows' previous f (independent of this step's chain in the kernel)
    fold1 = fi1 * 0.999f + 0.26f;
  }
  unsigned long long t1 = clock64();
  float acc = fold0 + fold1;
#pragma unroll
  for (int p = 0; p < P2; ++p) { float q0, q1; up2(ac2[p], q0, q1); acc += q0 + q1; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

void run_r2(const char* name) {
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int smem = (2 * W + 128) * 4;
  cudaFuncSetAttribute(kern_r2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 2; ++r) kern_r2<<<148, NT, smem>>>(out, cyc, -0.0f);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int b = 0; b < 148; ++b) s += h[b];
  printf("%-44s %7.1f cycles/row  (%s)\n", name, s / 148 / ROWS, cudaGetErrorString(e));
}

template <int TEAMS, bool SYNC, bool FIN, bool GSM>
void run(const char* name) {
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int smem = (2 * W + 128) * 4;
  cudaFuncSetAttribute(kern<TEAMS, SYNC, FIN, GSM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 2; ++r) kern<TEAMS, SYNC, FIN, GSM><<<148, NT * TEAMS, smem>>>(out, cyc, -0.0f);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int b = 0; b < 148; ++b) s += h[b];
  // TEAMS teams each process ROWS rows: rows per CTA = TEAMS * ROWS
  printf("%-44s %7.1f cycles/row  (%s)\n", name, s / 148 / (ROWS * TEAMS), cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1, false, false, false>("1 team, no sync, no finish, g in regs");
  run<1, true, false, false>("1 team, sync, no finish, g in regs");
  run<1, true, true, false>("1 team, sync, finish, g in regs");
  run<1, true, true, true>("1 team, sync, finish, g in smem");
  run<2, false, false, true>("2 teams, no sync, no finish, g in smem");
  run<2, true, false, true>("2 teams, sync, no finish, g in smem");
  run<2, true, true, true>("2 teams, sync, finish, g in smem");
  run_r2("1 team, 2 rows per step (sync + finish)");
  return 0;
}

// Instruction-mix microbenchmark of the dense row step (no sync, no finish):
// which part of the per-element stream costs what. 148 CTAs x 8 warps, 32
// columns per thread, every "row" from the same shared buffer; cycles per row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I../../paper_2605_00837_b200/csrc -o rowmix rowmix.cu
#include <cstdio>

#include "lsk_device.cuh"

using namespace lsk;
constexpr int NT = 256, V = 8, P2 = 16, W = 4 * V * NT, ROWS = 512;

// MODE 0: packed (the kernel's form)      1: scalar argument build
//      2: packed, no column FFMA2         3: packed, C from registers (no LDS)
//      4: packed, ex2 replaced by FADD (FP-only stream)   5: MUFU only (ex2 of a register)
template <int MODE>
__global__ void __launch_bounds__(NT, 1) kern(float* out, unsigned long long* cyc, float negzero, float Aval) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  for (int j = tid; j < W; j += NT) sm[j] = 0.5f + 1e-4f * (j % 97);
  __syncthreads();
  const f2 inv2 = pk2(1000.f, 1000.f), l2e2 = pk2(kLog2e, kLog2e), nz2 = pk2(negzero, negzero);
  const f2 lnu2 = pk2(-9.f, -9.f), A2 = pk2(Aval, Aval);
  f2 g2[P2], ac2[P2], creg[P2];
#pragma unroll
  for (int p = 0; p < P2; ++p) {
    g2[p] = pk2(0.3f + 1e-4f * p, 0.3f);
    ac2[p] = 0ull;
    creg[p] = pk2(0.5f + p * 1e-3f, 0.6f);
  }
  float shl = 1.f, tot = 0.f;
  unsigned long long t0 = clock64();
  for (int k = 0; k < ROWS; ++k) {
    const f2 nsl = pk2(-shl, -shl);
    float s = 0.f;
    f2 s2 = 0ull;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      f2 c[2];
      if (MODE == 3) { c[0] = creg[2 * v]; c[1] = creg[2 * v + 1]; }
      else lds2x2(sm + 4 * (v * NT + tid), c[0], c[1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * v + h;
        if (MODE == 1) {
          float g0, g1, c0, c1;
          up2(g2[p], g0, g1);
          up2(c[h], c0, c1);
          const float x0 = __fadd_rn(__fmul_rn(__fsub_rn(g0, c0), 1000.f), -9.f);
          const float x1 = __fadd_rn(__fmul_rn(__fsub_rn(g1, c1), 1000.f), -9.f);
          const float e0 = ex2(__fmaf_rn(x0, kLog2e, shl)), e1 = ex2(__fmaf_rn(x1, kLog2e, shl));
          s += e0 + e1;
          ac2[p] = fma2(pk2(e0, e1), A2, ac2[p]);
        } else if (MODE == 5) {
          float c0, c1;
          up2(c[h], c0, c1);
          const float e0 = ex2(c0 + shl), e1 = ex2(c1 + shl);
          s += e0 + e1;
        } else {
          const f2 x = fma2(arg3x2(g2[p], c[h], inv2, lnu2, nz2), l2e2, nsl);
          const f2 e = (MODE == 4) ? add2(x, nsl) : ex2x2(x);
          s2 = add2(s2, e);
          if (MODE != 2) ac2[p] = fma2(e, A2, ac2[p]);
        }
      }
    }
    float a0, a1;
    up2(s2, a0, a1);
    tot += s + a0 + a1;
    shl = 1.f + 1e-9f * tot;
  }
  unsigned long long t1 = clock64();
  float acc = tot;
#pragma unroll
  for (int p = 0; p < P2; ++p) { float a0, a1; up2(ac2[p], a0, a1); acc += a0 + a1; }
  out[blockIdx.x * NT + tid] = acc;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name) {
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * NT * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int smem = W * 4;
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 2; ++r) kern<MODE><<<148, NT, smem>>>(out, cyc, -0.0f, 0.5f);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int b = 0; b < 148; ++b) s += h[b];
  printf("%-52s %7.1f cycles/row  (%s)\n", name, s / 148 / ROWS, cudaGetErrorString(e));
}

int main() {
  run<0>("packed argument build + ex2 + sum + column FFMA2");
  run<1>("scalar argument build");
  run<2>("packed, no column FFMA2");
  run<3>("packed, C from registers (no LDS)");
  run<4>("packed, ex2 replaced by FADD2 (FP only)");
  run<5>("MUFU only (ex2 of the row value)");
  return 0;
}

// Pipe-throughput microbenchmark for the ops the Sinkhorn inner loop issues
// (FADD/FMUL/FFMA scalar vs packed f32x2, MUFU.EX2). Prints lanes/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu && ./pipes
#include <cstdio>
#include <cstdint>

#define CH 8
#define IT 4096

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long p; asm("mov.b64 %0, {%1,%2};" : "=l"(p) : "f"(a), "f"(b)); return p;
}
__device__ __forceinline__ float ex2(float t) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(t)); return y; }

template <int OP>
__global__ void __launch_bounds__(512) kern(float* out, float a, float b, float c, unsigned long long* cyc) {
  float v[CH]; unsigned long long p[CH];
  for (int k = 0; k < CH; ++k) { v[k] = threadIdx.x * 1e-3f + k; p[k] = pk(v[k], v[k] + 1.f); }
  const unsigned long long q = pk(a, b), r = pk(c, a);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (OP == 0) v[k] = __fadd_rn(v[k], a);                 // FADD reg
      if (OP == 1) v[k] = __fmul_rn(v[k], a);                 // FMUL reg
      if (OP == 2) v[k] = __fmaf_rn(v[k], a, b);              // FFMA 3-reg
      if (OP == 3) v[k] = __fmaf_rn(v[k], 1.4426950408889634f, b);  // FFMA imm
      if (OP == 4) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(q));
      if (OP == 5) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(q));
      if (OP == 6) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(q), "l"(r));
      if (OP == 7) v[k] = ex2(v[k]);
      if (OP == 8) {  // the f-element sequence: fsub, fmul, fadd, ffma, ex2, fadd
        float x = __fadd_rn(__fmul_rn(__fsub_rn(a, v[k]), b), c);
        v[k] = __fadd_rn(v[k], ex2(__fmaf_rn(x, 1.4426950408889634f, -b)));
      }
      if (OP == 9) {  // same, packed pairs
        unsigned long long x;
        asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(x) : "l"(q), "l"(p[k]));
        asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(r));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(q));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(r), "l"(q));
        float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x));
        unsigned long long e = pk(ex2(lo), ex2(hi));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(e));
      }
      if (OP == 10) v[k] = fmaxf(v[k], a);  // FMNMX (alu)
    }
  }
  unsigned long long t1 = clock64();
  float s = 0.f;
  for (int k = 0; k < CH; ++k) { float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[k])); s += v[k] + lo + hi; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int lanes_per_op, int threads) {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  kern<OP><<<148, threads>>>(out, 1.0001f, 0.5f, 0.25f, cyc);
  kern<OP><<<148, threads>>>(out, 1.0001f, 0.5f, 0.25f, cyc);
  cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  double ops = double(threads) * CH * IT * lanes_per_op;
  printf("%-28s threads=%4d  %7.1f lane-ops/clk/SM  (%.0f cyc)\n", name, threads, ops / mx, mx);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int t : {256, 512, 1024}) {
    run<0>("FADD r,r", 1, t); run<1>("FMUL r,r", 1, t); run<2>("FFMA r,r,r", 1, t); run<3>("FFMA r,imm,r", 1, t);
    run<4>("FADD2", 2, t); run<5>("FMUL2", 2, t); run<6>("FFMA2", 2, t); run<7>("MUFU.EX2", 1, t);
    run<8>("f-element seq (elements)", 1, t); run<9>("f-element packed (elements)", 2, t); run<10>("FMNMX", 1, t);
  }
  return 0;
}

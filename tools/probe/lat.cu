// micro-probe: dependent-chain latencies on the B200 (cycles per op)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters, double a, float af) {
  __shared__ double sm[1024];
  __shared__ int si[1024];
  const int t = threadIdx.x;
  sm[t] = a + t; si[t] = (t + 1) & 1023;
  __syncthreads();
  long long c0, c1;
  double x = a, y = a * 0.5;
  float xf = af;
  // DFMA chain
  c0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.9999999, 1e-9);
  c1 = clock64(); if (t == 0) cyc[0] = c1 - c0;
  // DMUL+DADD chain
  c0 = clock64();
  for (int i = 0; i < iters; ++i) { y = y * 1.0000001; y = y + 1e-12; }
  c1 = clock64(); if (t == 0) cyc[1] = c1 - c0;
  // FFMA chain
  c0 = clock64();
  for (int i = 0; i < iters; ++i) xf = fmaf(xf, 0.999f, 1e-3f);
  c1 = clock64(); if (t == 0) cyc[2] = c1 - c0;
  // MUFU rsqrt f32 chain
  float r = af;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) { float q; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(q) : "f"(r)); r = q + 1.0f; }
  c1 = clock64(); if (t == 0) cyc[3] = c1 - c0;
  // double division chain
  double dv = a + 2.0;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) dv = 3.0 / dv + 1.0;
  c1 = clock64(); if (t == 0) cyc[4] = c1 - c0;
  // double sqrt chain
  double sq = a + 2.0;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) sq = sqrt(sq) + 1.0;
  c1 = clock64(); if (t == 0) cyc[5] = c1 - c0;
  // shfl chain (double)
  double sh = a;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) sh = __shfl_xor_sync(0xffffffffu, sh, 1) + 1.0;
  c1 = clock64(); if (t == 0) cyc[6] = c1 - c0;
  // LDS pointer chase
  int p = t;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) p = si[p];
  c1 = clock64(); if (t == 0) cyc[7] = c1 - c0;
  // __syncthreads
  c0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  c1 = clock64(); if (t == 0) cyc[8] = c1 - c0;
  // f64<->f32 convert chain
  double cv = a;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) cv = (double)((float)cv) + 1.0;
  c1 = clock64(); if (t == 0) cyc[9] = c1 - c0;
  // __syncwarp + smem store/load round trip
  double rt = a;
  __shared__ double cell[32];
  c0 = clock64();
  for (int i = 0; i < iters; ++i) { cell[t & 31] = rt; __syncwarp(); rt = cell[(t + 1) & 31] + 1.0; __syncwarp(); }
  c1 = clock64(); if (t == 0) cyc[10] = c1 - c0;
  // __threadfence_block
  c0 = clock64();
  for (int i = 0; i < iters; ++i) { cell[t & 31] = rt + i; __threadfence_block(); }
  c1 = clock64(); if (t == 0) cyc[11] = c1 - c0;
  // warp_sum 5 levels (double)
  double ws = a + t;
  c0 = clock64();
  for (int i = 0; i < iters / 10; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
    ws *= 1e-3;
  }
  c1 = clock64(); if (t == 0) cyc[12] = (c1 - c0) * 10;
  out[t] = x + y + xf + r + dv + sq + sh + p + cv + rt + ws;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMalloc(&cyc, 128);
  const char* names[] = {"DFMA", "DMUL+DADD (2 ops)", "FFMA", "MUFU.RSQ f32 + FADD", "f64 div + add", "f64 sqrt + add", "SHFL f64 + DADD", "LDS chase", "BAR.SYNC (256 thr)", "F2F d->f->d + DADD", "STS+syncwarp+LDS+DADD+syncwarp", "STS+MEMBAR.CTA", "warp_sum f64 (5 lvl) + DMUL"};
  for (int nt : {32, 256}) {
    k<<<1, nt>>>(out, cyc, 1000, 1.5, 1.5f);
    cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
    printf("threads=%d\n", nt);
    for (int i = 0; i < 13; ++i) printf("  %-22s %6.1f cycles/iter\n", names[i], h[i] / 1000.0);
  }
  return 0;
}

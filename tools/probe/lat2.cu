// micro-probe: latencies that bound the per-cut phases of the QTT-FFT chain
// on B200 — dependent DMMA m8n8k4 (f64), dependent DFMA, __syncthreads with
// 8 warps, a shared-memory store -> barrier -> load round trip, a double
// shuffle.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/lat2 tools/probe/lat2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[256];
  const int tid = threadIdx.x;
  double a = 1.0 + 1e-9 * tid, b = 0.999, c0 = 0.0, c1 = 0.0, x = 1.0 + tid;
  long long t0, t1;
  // 1. dependent DMMA chain (warp 0)
  __syncthreads();
  t0 = clock64();
  if (tid < 32)
    for (int i = 0; i < iters; ++i) dmma(c0, c1, a, b);
  t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0) / iters;
  // 2. dependent DFMA chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.9999999, 1e-9);
  t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0) / iters;
  // 3. __syncthreads, 8 warps arriving together
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0) / iters;
  // 4. STS -> barrier -> LDS of another warp's value, dependent
  double v = x;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sm[tid] = v;
    __syncthreads();
    v = sm[(tid + 32) & 255] + 1e-9;
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0) / iters;
  // 5. dependent double shuffle
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1e-9;
  t1 = clock64();
  if (tid == 0) cyc[4] = (t1 - t0) / iters;
  // 6. 4 independent DMMA chains per warp (2 accumulator pairs each op), 8 warps
  double d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0, g0 = 0, g1 = 0;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    dmma(d0, d1, a, b);
    dmma(e0, e1, a, b);
    dmma(f0, f1, a, b);
    dmma(g0, g1, a, b);
  }
  t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0) / iters;
  out[tid] = c0 + c1 + x + v + d0 + d1 + e0 + e1 + f0 + f1 + g0 + g1;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 256>>>(out, cyc, 256);
    cudaDeviceSynchronize();
  }
  printf("dmma dependent %lld cyc | dfma dependent %lld | syncthreads(8 warps) %lld | sts-bar-lds-bar %lld | shfl f64 %lld | 4 indep dmma x 8 warps %lld cyc/iter\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
  return 0;
}

// micro-probe: FP64 pipe latency / issue rate per SM sub-partition on B200,
// for the latency-bound small-matrix kernels (eigensolver, Sturm counts).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/fp64pipe tools/probe/fp64pipe.cu
// Prints cycles per warp instruction for C independent DFMA chains per warp,
// W warps per CTA (W / 4 per sub-partition), and DADD / DMUL alone.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k_fma(double* out, long long* cyc, int iters) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = fma(x[c], 0.9999999, 1e-9);
  }
  long long c1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

template <int C>
__global__ void k_add(double* out, long long* cyc, int iters) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = x[c] + 1e-9;
  }
  long long c1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

// LDS.128 dependent latency and shfl (double) latency, 1 warp
__global__ void k_misc(double* out, long long* cyc, int iters) {
  __shared__ double2 sm[64];
  const int t = threadIdx.x;
  sm[t & 63] = make_double2(t, 1.0);
  __syncthreads();
  double v = 0.0;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double2 q = sm[((int)v + t) & 31];
    v = q.y * 0.0 + v * 0.0;      // dependent address
  }
  long long c1 = clock64();
  if (t == 0) cyc[0] = c1 - c0;
  double sh = t;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) sh = __shfl_xor_sync(0xffffffffu, sh, 1) * 0.5;
  c1 = clock64();
  if (t == 0) cyc[1] = c1 - c0;
  // STS + syncwarp + LDS round trip
  double rt = t;
  c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sm[t] = make_double2(rt, rt);
    __syncwarp();
    rt = sm[(t + 1) & 31].x * 0.5;
    __syncwarp();
  }
  c1 = clock64();
  if (t == 0) cyc[2] = c1 - c0;
  out[t] = v + sh + rt;
}

template <class K>
double run(K kern, int warps, int iters, double* d_out, long long* d_cyc) {
  kern<<<1, 32 * warps>>>(d_out, d_cyc, iters);
  cudaDeviceSynchronize();
  kern<<<1, 32 * warps>>>(d_out, d_cyc, iters);
  long long h;
  cudaMemcpy(&h, d_cyc, 8, cudaMemcpyDeviceToHost);
  return (double)h / iters;
}

int main() {
  double* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 1 << 20);
  cudaMalloc(&d_cyc, 64);
  const int it = 4096;
  for (int w : {1, 2, 4, 8, 16}) {
    printf("warps=%2d  DFMA cycles/iter: C=1 %.1f  C=2 %.1f  C=4 %.1f  C=8 %.1f | DADD C=1 %.1f C=8 %.1f\n", w,
           run(k_fma<1>, w, it, d_out, d_cyc), run(k_fma<2>, w, it, d_out, d_cyc),
           run(k_fma<4>, w, it, d_out, d_cyc), run(k_fma<8>, w, it, d_out, d_cyc),
           run(k_add<1>, w, it, d_out, d_cyc), run(k_add<8>, w, it, d_out, d_cyc));
  }
  k_misc<<<1, 32>>>(d_out, d_cyc, it);
  cudaDeviceSynchronize();
  long long h[3];
  cudaMemcpy(h, d_cyc, 24, cudaMemcpyDeviceToHost);
  printf("LDS dependent %.1f, SHFL(double)+DMUL %.1f, STS+syncwarp+LDS+syncwarp %.1f cycles\n", (double)h[0] / it,
         (double)h[1] / it, (double)h[2] / it);
  return 0;
}

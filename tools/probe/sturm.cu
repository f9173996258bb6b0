// micro-probe: latency of one division-free Sturm count (qtt_dev.cuh) on B200
#include <cstdio>
#include "../../paper_2301_13339_b200/csrc/qtt_dev.cuh"
using namespace qtt;
template <int NMAX>
__global__ void k(const double* dgi, const double* e2i, int* out, long long* cyc, int reps) {
  double dg[NMAX], e2[NMAX];
#pragma unroll
  for (int i = 0; i < NMAX; ++i) { dg[i] = dgi[i]; e2[i] = e2i[i]; }
  double x = -0.5 + 1e-3 * threadIdx.x;
  int acc = 0;
  __syncthreads();
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
    int c = sturm_count<NMAX>(dg, e2, x);
    acc += c;
    x += 1e-9 * c;
  }
  long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
int main() {
  double h[32], e[32];
  for (int i = 0; i < 32; ++i) { h[i] = 0.1 * (i % 7) - 0.3; e[i] = 0.01 * (1 + i % 3); }
  double *dd, *de; int* o; long long* c;
  cudaMalloc(&dd, 256); cudaMalloc(&de, 256); cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  cudaMemcpy(dd, h, 256, cudaMemcpyHostToDevice); cudaMemcpy(de, e, 256, cudaMemcpyHostToDevice);
  for (int nt : {32, 256}) {
    long long hc;
    k<16><<<1, nt>>>(dd, de, o, c, 100); cudaDeviceSynchronize();
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost); printf("NMAX=16 threads=%d: %.1f cycles/count\n", nt, hc / 100.0);
    k<20><<<1, nt>>>(dd, de, o, c, 100); cudaDeviceSynchronize();
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost); printf("NMAX=20 threads=%d: %.1f cycles/count\n", nt, hc / 100.0);
  }
  return 0;
}

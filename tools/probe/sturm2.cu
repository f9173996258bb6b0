// variants of the division-free Sturm recurrence p_i = (d_i - x) p_{i-1} - e2_{i-1} p_{i-2}
#include <cstdio>
#include <cuda_runtime.h>
template <int N, int V>
__device__ __forceinline__ int count(const double (&dg)[N], const double (&e2)[N], double x) {
  double p0 = 1.0, p1 = dg[0] - x;
  unsigned s1 = (unsigned)__double2hiint(p1) >> 31;
  int cnt = (int)s1;
#pragma unroll
  for (int i = 1; i < N; ++i) {
    double p2;
    if (V == 0) p2 = fma(dg[i] - x, p1, -e2[i - 1] * p0);
    else p2 = fma(dg[i] - x, p1, -(e2[i - 1] * p0));
    const unsigned s2 = (unsigned)__double2hiint(p2) >> 31;
    cnt += (int)(s1 ^ s2);
    s1 = s2;
    p0 = p1;
    p1 = p2;
    if (V != 2 && (i & 7) == 7 && i + 1 < N) {
      const double a = fabs(p1) + fabs(p0);
      const double sc = a > 1e120 ? 1e-120 : (a < 1e-120 ? 1e120 : 1.0);
      p0 *= sc;
      p1 *= sc;
    }
  }
  return cnt;
}
// V3: no sign tracking, just the chain (lower bound)
template <int N>
__device__ __forceinline__ double chain(const double (&dg)[N], const double (&e2)[N], double x) {
  double p0 = 1.0, p1 = dg[0] - x;
#pragma unroll
  for (int i = 1; i < N; ++i) { double p2 = fma(dg[i] - x, p1, -e2[i - 1] * p0); p0 = p1; p1 = p2; }
  return p1;
}
template <int N, int V>
__global__ void k(const double* dgi, const double* e2i, int* out, long long* cyc, int reps) {
  double dg[N], e2[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { dg[i] = dgi[i]; e2[i] = e2i[i]; }
  double x = -0.5 + 1e-3 * threadIdx.x;
  int acc = 0;
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
    int c;
    if (V == 3) c = chain<N>(dg, e2, x) > 0.0;
    else c = count<N, V>(dg, e2, x);
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
  long long hc;
#define RUN(V) k<20, V><<<1, 32>>>(dd, de, o, c, 100); cudaDeviceSynchronize(); \
  cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost); printf("N=20 variant %d: %.1f cycles/count\n", V, hc / 100.0);
  RUN(0) RUN(1) RUN(2) RUN(3)
  return 0;
}

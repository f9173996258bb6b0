// micro-probe: one multisection step of the small eigensolver (qtt_dev.cuh
// trid_values) for a 16 x 16 normalised tridiagonal T, 256 threads, and
// variants of the Sturm count.  Prints cycles per step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/probe/msect tools/probe/msect.cu
#include <cstdio>
#include "../../paper_2301_13339_b200/csrc/qtt_dev.cuh"
using namespace qtt;

// variant 1: no rescaling (n <= 16, |d - x| <= 2 keeps p_i inside the range
// unless a leading minor underflows)
template <int L>
__device__ __forceinline__ int sturm_plain(const double (&dg)[16], const double (&e2)[16], double x) {
  double p0 = 1.0, p1 = dg[0] - x;
  unsigned s1 = (unsigned)__double2hiint(p1) >> 31;
  int cnt = (int)s1;
#pragma unroll
  for (int i = 1; i < L; ++i) {
    const double p2 = fma(dg[i] - x, p1, -e2[i - 1] * p0);
    const unsigned s2 = (unsigned)__double2hiint(p2) >> 31;
    cnt += (int)(s1 ^ s2);
    s1 = s2;
    p0 = p1;
    p1 = p2;
  }
  return cnt;
}

// variant 2: LDL^T pivots q_i = (d_i - x) - e2_{i-1} / q_{i-1} with a fast
// reciprocal (MUFU + 1 Newton), count of negative pivots
__device__ __forceinline__ int sturm_ratio(const double (&dg)[16], const double (&e2)[16], double x) {
  double q = dg[0] - x;
  int cnt = q < 0.0;
#pragma unroll
  for (int i = 1; i < 16; ++i) {
    if (fabs(q) < 1e-300) q = -1e-300;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    const double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    q = fma(-e2[i - 1], r, dg[i] - x);
    cnt += q < 0.0;
  }
  return cnt;
}

template <int VAR, int GL>
__global__ void k(const double* dgi, const double* e2i, double* out, long long* cyc, int reps) {
  double dg[16], e2[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { dg[i] = dgi[i]; e2[i] = e2i[i]; }
  const int tid = threadIdx.x;
  const int n = 16;
  const int k = tid / GL, j = tid % GL;
  const int steps = GL == 32 ? 11 : (GL == 16 ? 13 : 17);
  const double sj = (double)(j + 1) / (double)(GL + 1);
  const double inv_g1 = 1.0 / (double)(GL + 1);
  const int base = (tid & 31) & ~(GL - 1);
  const unsigned gmask = (GL == 32) ? 0xffffffffu : (((1u << GL) - 1u) << base);
  double acc = 0.0;
  __syncthreads();
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double l = -1.0 - 1e-14, h = 1.0 + 1e-14;
    for (int st = 0; st < steps; ++st) {
      const double x = l + (h - l) * sj;
      int c = 0;
      if (k < n) {
        if (VAR == 0) c = sturm_count<16>(dg, e2, x);
        else if (VAR == 1) c = sturm_plain<16>(dg, e2, x);
        else c = sturm_ratio(dg, e2, x);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, c >= k + 1) & gmask;
      const int first = bal ? (__ffs(bal) - 1 - base) : GL;
      const double w = h - l;
      const double nh = (first < GL) ? l + w * (double)(first + 1) * inv_g1 : h;
      const double nl = (first > 0) ? l + w * (double)first * inv_g1 : l;
      l = nl;
      h = nh;
    }
    acc += 0.5 * (l + h);
  }
  long long c1 = clock64();
  out[tid] = acc;
  if (tid == 0) cyc[0] = c1 - c0;
}

int main() {
  // a normalised tridiagonal with a graded spectrum
  double h[16], e[16];
  for (int i = 0; i < 16; ++i) { h[i] = 0.25 * cos(0.7 * i) * pow(0.6, i); e[i] = 0.02 * pow(0.5, i); }
  double *dd, *de, *o; long long* c;
  cudaMalloc(&dd, 256); cudaMalloc(&de, 256); cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
  cudaMemcpy(dd, h, 128, cudaMemcpyHostToDevice); cudaMemcpy(de, e, 128, cudaMemcpyHostToDevice);
  const int reps = 50;
  auto run = [&](auto kern, const char* name, int steps, int threads) {
    kern<<<1, threads>>>(dd, de, o, c, reps); cudaDeviceSynchronize();
    kern<<<1, threads>>>(dd, de, o, c, reps); cudaDeviceSynchronize();
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    double r0; cudaMemcpy(&r0, o, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %7.1f cycles/step  %8.1f per solve  (lam0 %.17g)\n", name, (double)hc / reps / steps,
           (double)hc / reps, r0 / reps);
  };
  run(k<0, 16>, "current (rescaled, 16 thr/eig, 256 thr)", 13, 256);
  run(k<1, 16>, "plain product (16 thr/eig)", 13, 256);
  run(k<2, 16>, "ratio + fast rcp (16 thr/eig)", 13, 256);
  run(k<0, 32>, "current, 32 thr/eig, 512 thr", 11, 512);
  run(k<1, 32>, "plain, 32 thr/eig, 512 thr", 11, 512);
  run(k<1, 8>, "plain, 8 thr/eig, 128 thr", 17, 128);
  return 0;
}

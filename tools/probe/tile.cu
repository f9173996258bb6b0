// micro-probe: one warp computing one 8 x 8 complex output tile of a small
// product from shared memory (the per-cut products of the QTT-FFT chain),
// k = 16: (a) DMMA m8n8k4 with per-chunk predicated loads (as in the chain),
// (b) DMMA with all operands loaded up front, (c) DFMA, one output element per
// lane pair (lanes 0..31 -> 64 outputs: 2 per lane), four accumulators.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/tile tools/probe/tile.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef double2 cplx;
__device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void k(cplx* out, long long* cyc, int a1, int rc) {
  __shared__ cplx A[16 * 16], B[16 * 16], C[16 * 16];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < 256; e += blockDim.x) {
    A[e] = cmk(1.0 + e * 1e-3, 0.5 - e * 1e-3);
    B[e] = cmk(0.25 + e * 1e-3, -0.5 + e * 2e-3);
  }
  __syncthreads();
  const int ar = lane >> 2, ac = lane & 3;
  const int K = 2 * rc, nk = (K + 3) >> 2;
  long long t0, t1;
  for (int rep = 0; rep < 3; ++rep) {
    // (a) chain-style
    __syncwarp();
    t0 = clock64();
    {
      double r0 = 0, r1 = 0, i0 = 0, i1 = 0;
      for (int kc = 0; kc < nk; ++kc) {
        const int kk = 4 * kc + ac;
        cplx av = cmk(0, 0), bv = cmk(0, 0);
        if (ar < a1 && kk < K) av = A[ar + a1 * kk];
        if (kk < K && ar < a1) bv = B[kk + K * ar];
        dmma(r0, r1, av.x, bv.x);
        dmma(r0, r1, -av.y, bv.y);
        dmma(i0, i1, av.x, bv.y);
        dmma(i0, i1, av.y, bv.x);
      }
      C[ar + 8 * (2 * ac)] = cmk(r0, i0);
      C[ar + 8 * (2 * ac + 1)] = cmk(r1, i1);
    }
    __syncwarp();
    t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    // (b) operands up front (K <= 16)
    __syncwarp();
    t0 = clock64();
    {
      cplx av[4], bv[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        const int kk = 4 * kc + ac;
        av[kc] = (kc < nk && ar < a1 && kk < K) ? A[ar + a1 * kk] : cmk(0, 0);
        bv[kc] = (kc < nk && kk < K && ar < a1) ? B[kk + K * ar] : cmk(0, 0);
      }
      double r0 = 0, r1 = 0, i0 = 0, i1 = 0, s0 = 0, s1 = 0, u0 = 0, u1 = 0;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        dmma(r0, r1, av[kc].x, bv[kc].x);
        dmma(s0, s1, -av[kc].y, bv[kc].y);
        dmma(i0, i1, av[kc].x, bv[kc].y);
        dmma(u0, u1, av[kc].y, bv[kc].x);
      }
      C[ar + 8 * (2 * ac)] = cmk(r0 + s0, i0 + u0);
      C[ar + 8 * (2 * ac + 1)] = cmk(r1 + s1, i1 + u1);
    }
    __syncwarp();
    t1 = clock64();
    if (lane == 0) cyc[1] = t1 - t0;
    // (c) DFMA: lane -> outputs (i, j) = (lane & 7, lane >> 3) and (.., + 4)
    __syncwarp();
    t0 = clock64();
    {
      const int i = lane & 7, j0 = lane >> 3;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = j0 + 4 * h;
        cplx s[4] = {cmk(0, 0), cmk(0, 0), cmk(0, 0), cmk(0, 0)};
#pragma unroll
        for (int l = 0; l < 16; ++l)
          if (l < K) s[l & 3] = cfma(A[i + a1 * l], B[l + K * j], s[l & 3]);
        C[i + 8 * j] = cmk(s[0].x + s[1].x + s[2].x + s[3].x, s[0].y + s[1].y + s[2].y + s[3].y);
      }
    }
    __syncwarp();
    t1 = clock64();
    if (lane == 0) cyc[2] = t1 - t0;
  }
  out[tid] = C[tid & 63];
}

int main() {
  cplx* out;
  long long* cyc;
  cudaMalloc(&out, 256 * sizeof(cplx));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  k<<<1, 32>>>(out, cyc, 8, 8);
  cudaDeviceSynchronize();
  printf("8x8 complex tile, k = 16, one warp: DMMA chain-style %lld cyc | DMMA loads up front %lld | DFMA 2 outputs/lane %lld\n",
         cyc[0], cyc[1], cyc[2]);
  return 0;
}

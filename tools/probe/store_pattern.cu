// Store-pattern probe for the expansion (k_expand_main): the same grid, loop
// and fragment->address mapping with constant data, (a) direct 8-byte
// streaming stores from the DMMA fragments (the current kernel), (b) staged
// through a swizzled shared-memory block of 2048 elements and written as
// 512-byte rows with 16-byte stores.  2^28 doubles, interleaved and 1D.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_pattern store_pattern.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__host__ __device__ inline uint64_t compact_even(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
  x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
  x = (x | (x >> 16)) & 0x00000000ffffffffull;
  return x;
}
__host__ __device__ inline uint64_t off(uint64_t q, int il, int bx) {
  return il ? compact_even(q) + (compact_even(q >> 1) << bx) : q;
}

__global__ void __launch_bounds__(256, 3) k_direct(double* y, int d, int il, int bx, int per) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint64_t nsup = 1ull << (d - 15);
  uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = c0 + per;
  if (c1 > nsup) c1 = nsup;
  uint32_t offrow[4], offcol[2];
  for (int mb = 0; mb < 4; ++mb) offrow[mb] = (uint32_t)off(32 * w + 8 * mb + (lane >> 2), il, bx);
  for (int e = 0; e < 2; ++e) offcol[e] = (uint32_t)off((uint64_t)(2 * (lane & 3) + e) << 8, il, bx);
  for (uint64_t c = c0; c < c1; ++c) {
    double* yb = y + off(c << 15, il, bx);
#pragma unroll 1
    for (int nb = 0; nb < 16; ++nb) {
      const uint32_t onb = (uint32_t)off((uint64_t)(8 * nb) << 8, il, bx);
      for (int mb = 0; mb < 4; ++mb)
        for (int e = 0; e < 2; ++e) __stcs(yb + (offrow[mb] + offcol[e] + onb), 1.0 + mb + e);
    }
  }
}

// smem position of block-local element (row r in 0..255, col j in 0..7):
// q = r + 256 j (bits 0..10).  Interleaved: x = bits 0,2,..,10 (6), y = bits
// 1,..,9 (5), stored row-major 32 x 64 with x' = x ^ (h << 1),
// h = y0 | y4 << 1 | x5 << 2.  1D: q' = q ^ (((q >> 9) & 3) << 2).
__device__ __forceinline__ int spos(int q, int il) {
  if (il) {
    const int x = (int)compact_even((uint64_t)q), y = (int)compact_even((uint64_t)q >> 1);
    const int h = (y & 1) | (((y >> 4) & 1) << 1) | (((x >> 5) & 1) << 2);
    return y * 64 + (x ^ (h << 1));
  }
  return q ^ (((q >> 9) & 3) << 2);
}

__global__ void __launch_bounds__(256, 3) k_staged(double* y, int d, int il, int bx, int per) {
  __shared__ __align__(16) double blk[2][2048];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint64_t nsup = 1ull << (d - 15);
  uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = c0 + per;
  if (c1 > nsup) c1 = nsup;
  int sp[4][2];
  for (int mb = 0; mb < 4; ++mb)
    for (int e = 0; e < 2; ++e) sp[mb][e] = spos(32 * w + 8 * mb + (lane >> 2) + 256 * (2 * (lane & 3) + e), il);
  const uint64_t W = il ? (1ull << bx) : 0;
  int buf = 0;
  for (uint64_t c = c0; c < c1; ++c) {
#pragma unroll 1
    for (int nb = 0; nb < 16; ++nb) {
      double* yb = y + off((c << 15) + ((uint64_t)nb << 11), il, bx);
      for (int mb = 0; mb < 4; ++mb)
        for (int e = 0; e < 2; ++e) blk[buf][sp[mb][e]] = 1.0 + mb + e;
      __syncthreads();
      // 2048 doubles = 1024 16-byte pairs, 4 per thread
      for (int t = 0; t < 4; ++t) {
        const int pi = tid + 256 * t;           // pair index in storage order
        double2 v;
        if (il) {
          const int yy = pi >> 5, x = 2 * (pi & 31);
          const int h = (yy & 1) | (((yy >> 4) & 1) << 1) | (((x >> 5) & 1) << 2);
          v = *reinterpret_cast<const double2*>(&blk[buf][yy * 64 + (x ^ (h << 1))]);
          __stcs(reinterpret_cast<double2*>(yb + yy * W + x), v);
        } else {
          const int q = 2 * pi;
          v = *reinterpret_cast<const double2*>(&blk[buf][q ^ (((q >> 9) & 3) << 2)]);
          __stcs(reinterpret_cast<double2*>(yb + q), v);
        }
      }
      buf ^= 1;
    }
  }
}

int main() {
  const int d = 28;
  const size_t n = 1ull << d;
  double* y;
  cudaMalloc(&y, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint64_t nsup = 1ull << (d - 15);
  for (int waves : {3, 6}) {
    const int target = waves * 148;
    const int per = (int)((nsup + target - 1) / target);
    const int nb = (int)((nsup + per - 1) / per);
    for (int il = 0; il < 2; ++il)
      for (int kind = 0; kind < 2; ++kind) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(e0);
          if (kind == 0) k_direct<<<nb, 256>>>(y, d, il, 14, per);
          else k_staged<<<nb, 256>>>(y, d, il, 14, per);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep && ms < best) best = ms;
        }
        // verify the staged pattern writes every element exactly (value check)
        printf("waves %d %s %-7s %7.3f ms %7.1f GB/s\n", waves, il ? "interleaved" : "1d",
               kind ? "staged" : "direct", best, n * 8 / (best * 1e6));
      }
  }
  // coverage check of the staged mapping: fill with NaN, run, count NaN left
  cudaMemset(y, 0xff, n * 8);
  k_staged<<<148 * 3, 256>>>(y, d, 1, 14, (int)((nsup + 443) / 444));
  double* h = (double*)malloc(n * 8);
  cudaMemcpy(h, y, n * 8, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += !(h[i] >= 1.0 && h[i] <= 5.0);
  printf("staged interleaved coverage: %zu unwritten; %s\n", bad, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

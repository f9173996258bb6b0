// HBM bandwidth probe: write-only, read-only and copy over 2 GiB buffers
// (float64, 16-byte and 32-byte vector accesses, grid = k x 148 SMs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw bw.cu && ./bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write16(double2* y, size_t n2, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    y[i] = make_double2(v, v);
}
__global__ void k_write32(double4* y, size_t n4, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    y[i] = make_double4(v, v, v, v);
}
__global__ void k_write16_cs(double2* y, size_t n2, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    __stcs(y + i, make_double2(v, v));
}
__global__ void k_read16(const double2* x, size_t n2, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 a = __ldcs(x + i);
    s += a.x + a.y;
  }
  if (s == 12345.678) *out = s;
}
__global__ void k_copy16(const double2* x, double2* y, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    y[i] = __ldcs(x + i);
}

int main() {
  const size_t bytes = 2ull << 30;
  double *x, *y, *o;
  cudaMalloc(&x, bytes);
  cudaMalloc(&y, bytes);
  cudaMalloc(&o, 8);
  cudaMemset(x, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n2 = bytes / 16, n4 = bytes / 32;
  for (int waves : {1, 2, 4, 8, 16}) {
    const int grid = 148 * waves;
    for (int kind = 0; kind < 5; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) k_write16<<<grid, 256>>>((double2*)y, n2, 1.0);
        if (kind == 1) k_write32<<<grid, 256>>>((double4*)y, n4, 1.0);
        if (kind == 2) k_write16_cs<<<grid, 256>>>((double2*)y, n2, 1.0);
        if (kind == 3) k_read16<<<grid, 256>>>((const double2*)x, n2, o);
        if (kind == 4) k_copy16<<<grid, 256>>>((const double2*)x, (double2*)y, n2 / 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      const char* nm[] = {"write16", "write32", "write16_cs", "read16", "copy16(1GiB each way)"};
      printf("grid %5d  %-22s %8.3f ms  %7.1f GB/s\n", grid, nm[kind], best, bytes / (best * 1e6));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

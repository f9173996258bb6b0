// FP64 throughput probe: DFMA (8 independent chains per thread) and DMMA m8n8k4
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_k(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, 0.999, 1e-3); a1 = fma(a1, 0.999, 1e-3); a2 = fma(a2, 0.999, 1e-3); a3 = fma(a3, 0.999, 1e-3);
    a4 = fma(a4, 0.999, 1e-3); a5 = fma(a5, 0.999, 1e-3); a6 = fma(a6, 0.999, 1e-3); a7 = fma(a7, 0.999, 1e-3);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dmma_k(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, (size_t)sms * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dfma_k<<<sms * 4, 512>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)sms * 4 * 512;
    printf("DFMA: %.2f TFLOP/s (%.1f FMA/clk/SM at 1.965 GHz)\n", fl / ms / 1e9, fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); dmma_k<<<sms * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 8 * iters * (double)sms * 4 * 256 / 32;
    printf("DMMA: %.2f TFLOP/s (%.1f FMA/clk/SM at 1.965 GHz)\n", fl / ms / 1e9, fl / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}

// debug.cu — test-only entry point exposing the CTA Jacobi eigensolver used
// by every truncated SVD of the path (qtt_dev.cuh), so tests can check it
// against numpy.linalg.eigh on graded Hermitian spectra.
#include "../../include/qtt.h"
#include "qtt_kernels.h"

namespace qtt {
static constexpr int NT = 256;

__global__ void __launch_bounds__(NT) k_debug_eigh(const cplx* A, int n, double* lam, cplx* U, int* sweeps) {
  extern __shared__ __align__(16) unsigned char smraw[];
  EigSmem<32>& E = *reinterpret_cast<EigSmem<32>*>(smraw);
  constexpr int LD = EigSmem<32>::LD;
  for (int e = threadIdx.x; e < n * n; e += NT) E.A[0][(e % n) + LD * (e / n)] = A[e];
  __syncthreads();
  const cplx* V = jacobi_eig<32, NT>(E, n, nullptr);
  for (int e = threadIdx.x; e < n * n; e += NT) U[e] = V[(e % n) + LD * (e / n)];
  for (int i = threadIdx.x; i < n; i += NT) lam[i] = E.lam[i];
  if (threadIdx.x == 0) *sweeps = E.sweeps;
}
}  // namespace qtt

extern "C" int qtt_debug_eigh(const void* A, int n, double* lam, void* U, int* sweeps, void* stream) {
  using namespace qtt;
  if (n < 1 || n > 32) return QTT_EINVAL;
  cudaFuncSetAttribute(k_debug_eigh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EigSmem<32>));
  k_debug_eigh<<<1, NT, sizeof(EigSmem<32>), (cudaStream_t)stream>>>((const cplx*)A, n, lam, (cplx*)U, sweeps);
  return cudaGetLastError() == cudaSuccess ? QTT_OK : QTT_ECUDA;
}

// debug.cu — test-only entry point exposing the small Hermitian eigensolver
// used by every truncated SVD of the path (qtt_dev.cuh: tridiagonal solver
// with Jacobi fallback, or Jacobi alone), so tests can check it against
// numpy.linalg.eigh.
#include "../../include/qtt.h"
#include "qtt_kernels.h"

namespace qtt {
static constexpr int NT = 256;

template <int NMAX>
__global__ void __launch_bounds__(NT, 1) k_debug_eigh(const cplx* A, int n, double* lam, cplx* U, int* sweeps,
                                                   int reps, int mode) {
  extern __shared__ __align__(16) unsigned char smraw[];
  EigSmem<NMAX>& E = *reinterpret_cast<EigSmem<NMAX>*>(smraw);
  constexpr int LD = EigSmem<NMAX>::LD;
  const cplx* V = nullptr;
  if (threadIdx.x == 0) { E.fallbacks = 0; E.sweeps = 0; }
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < n * n; e += NT) E.A[0][(e % n) + LD * (e / n)] = A[e];
    __syncthreads();
    if (mode == 1) V = jacobi_eig<NMAX, NT>(E, n, nullptr);
    else if (mode >= 64) {
      // diagnostics (tools/eig_timing.py --warm): the vector phase twice on
      // the same T, phase cycles of the second (instruction-cache warm) run
      eig_values<NMAX, NT>(E, n);
      V = eig_vectors<NMAX, NT>(E, n, mode - 64, nullptr);
      V = eig_vectors<NMAX, NT>(E, n, mode - 64, nullptr);
    } else V = eig_small<NMAX, NT>(E, n, mode >= 2 ? mode - 1 : n, nullptr);
  }
  for (int e = threadIdx.x; e < n * n; e += NT) U[e] = V[(e % n) + LD * (e / n)];
  for (int i = threadIdx.x; i < n; i += NT) lam[i] = E.lam[i];
  if (threadIdx.x == 0) {
    sweeps[0] = E.sweeps;
    sweeps[1] = E.fallbacks;
    for (int k = 0; k < 5; ++k) sweeps[2 + k] = (int)E.u.tr.tph[k];
    for (int k = 0; k < 5; ++k) sweeps[7 + k] = (int)E.u.tr.tstep[k];
  }
}
__global__ void k_debug_omega(unsigned long long seed, int k, unsigned long long j0, int n, int kp, double* out) {
  const int npairs = (kp + 1) / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * npairs; e += gridDim.x * blockDim.x) {
    const int row = e / npairs, cp = e % npairs;
    double z0, z1;
    omega_pair(j0 + row, (unsigned)k, (unsigned)cp, seed, z0, z1);
    out[(size_t)row * kp + 2 * cp] = z0;
    if (2 * cp + 1 < kp) out[(size_t)row * kp + 2 * cp + 1] = z1;
  }
}
}  // namespace qtt

extern "C" int qtt_debug_omega(unsigned long long seed, int k, unsigned long long j0, int n, int kp, double* out,
                               void* stream) {
  using namespace qtt;
  if (n < 1 || kp < 1 || kp > 64 || !out) return QTT_EINVAL;
  k_debug_omega<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(seed, k, j0, n, kp, out);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? QTT_OK : QTT_ECUDA;
}

extern "C" int qtt_debug_eigh(const void* A, int n, double* lam, void* U, int* sweeps, int reps, int mode,
                              void* stream) {
  using namespace qtt;
  if (n < 1 || n > 32 || reps < 1) return QTT_EINVAL;
  // mode bit 8: run the NMAX = 20 instantiation (the width the R_max = 10 /
  // Rhat <= 8 pipelines use) for n <= 20
  const bool w20 = (mode & 256) != 0;
  mode &= 255;
  if (w20 && n <= 20) {
    cudaFuncSetAttribute(k_debug_eigh<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EigSmem<20>));
    k_debug_eigh<20><<<1, NT, sizeof(EigSmem<20>), (cudaStream_t)stream>>>((const cplx*)A, n, lam, (cplx*)U,
                                                                           sweeps, reps, mode);
  } else if (n <= 16) {
    cudaFuncSetAttribute(k_debug_eigh<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EigSmem<16>));
    k_debug_eigh<16><<<1, NT, sizeof(EigSmem<16>), (cudaStream_t)stream>>>((const cplx*)A, n, lam, (cplx*)U,
                                                                           sweeps, reps, mode);
  } else {
    cudaFuncSetAttribute(k_debug_eigh<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EigSmem<32>));
    k_debug_eigh<32><<<1, NT, sizeof(EigSmem<32>), (cudaStream_t)stream>>>((const cplx*)A, n, lam, (cplx*)U,
                                                                           sweeps, reps, mode);
  }
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? QTT_OK : QTT_ECUDA;
}

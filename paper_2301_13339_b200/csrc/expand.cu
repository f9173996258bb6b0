// expand.cu — QTT-to-full expansion (Alg. 3 "Full", P:408-424;
// Step 4 of Alg. 2) on sm_100a, written straight into the caller's
// layout (1D, or row-major image for the interleaved / concatenated 2D QTT).
//
// y[i] = Re(C_1[i_1] ... C_d[i_d]).  The chain is split at m_e = 8:
//   L = full(cores 1..8)  (256 x r, complex)          k_expand_prep
//   R = full(cores 9..d)  (r x 2^{d-8}), formed per 4096-element chunk from a
//       suffix stack of the top cores and a 4-level tree of the mid cores
//   y_chunk = [Re L, -Im L] (256 x 2r) . [Re R; Im R] (2r x 16)
// on FP64 tensor cores (DMMA), staged through shared memory so every store is
// a coalesced 16-byte write (the pass is bound by HBM writes).
#include "qtt_kernels.h"

namespace qtt {

static constexpr int NT = 256;
static constexpr int ME = 8;        // bits of L
static constexpr int CHX = 4096;    // chunk (64 x 64 square in 2D)
static constexpr int OSLD = 68;     // staging row stride (interleaved)

// ----------------------------------------------------------- small d
__global__ void k_expand_small(const ExProb* probs, ExParams P) {
  const ExProb& pr = probs[blockIdx.y];
  const int d = P.d;
  const uint64_t n = 1ull << d;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    cplx v[RC];
    int r = pr.ranks[1];
    {
      const cplx* c = pr.cores;
      int be = (int)(q & 1);
      for (int j = 0; j < RC; ++j) v[j] = (j < r) ? c[be + 2 * j] : czero();
    }
    for (int k = 2; k <= d; ++k) {
      const cplx* c = pr.cores + (size_t)(k - 1) * SLOT;
      const int r0 = r, r1 = pr.ranks[k];
      const int be = (int)((q >> (k - 1)) & 1);
      cplx w[RC];
      for (int j = 0; j < RC; ++j) {
        cplx s = czero();
        if (j < r1)
          for (int i = 0; i < r0; ++i) s = cfma(v[i], c[i + r0 * be + 2 * r0 * j], s);
        w[j] = s;
      }
      for (int j = 0; j < RC; ++j) v[j] = w[j];
      r = r1;
    }
    pr.y[qtt_offset(q, P.layout, P.bx)] = P.imag ? v[0].y : v[0].x;
  }
}

// ------------------------------------------------------------ L split
// lsplit (256 x KL, column-major ld 256): imag = 0: [Re L, -Im L],
// imag = 1: [Im L, Re L]; zero padded to KL = round4(2 r_8).
__global__ void k_expand_prep(const ExProb* probs, ExParams P) {
  const ExProb& pr = probs[blockIdx.x];
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx (*A)[256 * RC] = reinterpret_cast<cplx (*)[256 * RC]>(smraw);
  const int tid = threadIdx.x;
  int r = pr.ranks[1];
  for (int e = tid; e < 2 * r; e += blockDim.x) {
    int i = e & 1, j = e >> 1;
    A[0][i + 2 * j] = pr.cores[i + 2 * j];     // core 1 is (1, 2, r): (0, i, j) at i + 2 j
  }
  __syncthreads();
  int cur = 0;
  for (int k = 2; k <= ME; ++k) {
    const cplx* c = pr.cores + (size_t)(k - 1) * SLOT;
    const int r0 = r, r1 = pr.ranks[k];
    const int h = 1 << (k - 1), n2 = 1 << k;
    for (int e = tid; e < n2 * r1; e += blockDim.x) {
      int i = e % n2, j = e / n2;
      int il = i % h, be = i / h;
      cplx s = czero();
      for (int l = 0; l < r0; ++l) s = cfma(A[cur][il + h * l], c[l + r0 * be + 2 * r0 * j], s);
      A[cur ^ 1][i + n2 * j] = s;
    }
    __syncthreads();
    cur ^= 1;
    r = r1;
  }
  const int kl = (2 * r + 3) & ~3;
  for (int e = tid; e < 256 * 32; e += blockDim.x) {
    int i = e & 255, j = e >> 8;
    double v = 0.0;
    if (j < r) v = P.imag ? A[cur][i + 256 * j].y : A[cur][i + 256 * j].x;
    else if (j < 2 * r) v = P.imag ? A[cur][i + 256 * (j - r)].x : -A[cur][i + 256 * (j - r)].y;
    (void)kl;
    pr.lsplit[e] = v;
  }
}

// ------------------------------------------------------------- main
struct ExSmem {
  double stage[64 * OSLD];
  double Rs[32 * 20];         // [Re R; Im R] (KL x 16), ld KLD
  cplx stack[MAXD][RC];       // suffix products S_k (k = 13..d)
  cplx tree[2][16 * RC];
};

__global__ void __launch_bounds__(NT) k_expand_main(const ExProb* probs, ExParams P, int per_cta) {
  const ExProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  ExSmem& S = *reinterpret_cast<ExSmem*>(smraw);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int d = P.d;
  const uint64_t nchunks = 1ull << (d - 12);
  const uint64_t c0 = (uint64_t)blockIdx.x * per_cta;
  uint64_t c1 = c0 + per_cta;
  if (c1 > nchunks) c1 = nchunks;
  if (c0 >= c1) return;
  const int r8 = pr.ranks[ME];
  const int kl = (2 * r8 + 3) & ~3;
  const int kld = (kl % 8 == 0) ? kl + 4 : kl;
  const int ksteps = kl / 4;
  // A fragments: this warp's 4 m-blocks (rows 32 w .. 32 w + 31), all k-steps
  double afr[4][8];
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      int row = 32 * w + 8 * mb + (lane >> 2), col = 4 * ks + (lane & 3);
      afr[mb][ks] = (col < kl) ? pr.lsplit[row + 256 * col] : 0.0;
    }
  uint64_t prev = ~0ull;
  for (uint64_t c = c0; c < c1; ++c) {
    // ---- suffix stack of the top cores 13..d for the bits of c
    int hi;   // highest core index whose bit changed (>= 13)
    if (prev == ~0ull) hi = d;
    else {
      uint64_t diff = prev ^ c;
      hi = 12 + (64 - __clzll((long long)diff));
    }
    if (w == 0) {
      for (int k = hi; k >= 13; --k) {
        const int r0 = pr.ranks[k - 1], r1 = pr.ranks[k];
        const int be = (int)((c >> (k - 13)) & 1);
        const cplx* core = pr.cores + (size_t)(k - 1) * SLOT;
        if (lane < r0) {
          cplx s = czero();
          if (k == d) s = core[lane + r0 * be];
          else
            for (int j = 0; j < r1; ++j) s = cfma(core[lane + r0 * be + 2 * r0 * j], S.stack[k][j], s);
          S.stack[k - 1][lane] = s;
        }
        __syncwarp();
      }
    }
    prev = c;
    __syncthreads();
    // ---- mid tree over cores 12, 11, 10, 9 -> 16 vectors of size r_8
    {
      const cplx* vin = S.stack[12];
      int nv = 1;
      int cur = 0;
      for (int k = 12; k >= 9; --k) {
        const int r0 = pr.ranks[k - 1], r1 = pr.ranks[k];
        const cplx* core = pr.cores + (size_t)(k - 1) * SLOT;
        cplx* vout = S.tree[cur];
        // output vector v' = 2*v + be (bit k-9 of the column index is the MSB so far)
        for (int e = tid; e < 2 * nv * r0; e += NT) {
          int i = e % r0, vv = e / r0;
          int be = vv & 1, src = vv >> 1;
          cplx s = czero();
          for (int j = 0; j < r1; ++j) s = cfma(core[i + r0 * be + 2 * r0 * j], vin[src * RC + j], s);
          vout[vv * RC + i] = s;
        }
        __syncthreads();
        vin = vout;
        cur ^= 1;
        nv *= 2;
      }
      // vin holds 16 vectors; vector index vv has bits (b12 b11 b10 b9) with b9 as LSB
      for (int e = tid; e < kl * 16; e += NT) {
        int row = e % kl, col = e / kl;
        double v = 0.0;
        if (row < r8) v = vin[col * RC + row].x;
        else if (row < 2 * r8) v = vin[col * RC + row - r8].y;
        S.Rs[row + kld * col] = v;
      }
    }
    __syncthreads();
    // ---- GEMM: rows 32 w .. +31, 16 columns
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      double acc[4][2];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) acc[mb][0] = acc[mb][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (ks < ksteps) {
          double b = S.Rs[(4 * ks + (lane & 3)) + kld * (8 * nb + (lane >> 2))];
#pragma unroll
          for (int mb = 0; mb < 4; ++mb) dmma884(acc[mb][0], acc[mb][1], afr[mb][ks], b);
        }
      }
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          uint32_t row = 32 * w + 8 * mb + (lane >> 2);
          uint32_t col = 8 * nb + 2 * (lane & 3) + e;
          uint32_t q = row + (col << ME);
          int off = (P.layout == LAYOUT_INTERLEAVED)
                        ? (int)(compact_even(q) + OSLD * compact_even(q >> 1))
                        : (int)q;
          S.stage[off] = acc[mb][e];
        }
    }
    __syncthreads();
    // ---- coalesced store of the chunk
    if (P.layout == LAYOUT_INTERLEAVED) {
      const uint64_t q0 = c * (uint64_t)CHX;
      const uint64_t x0 = compact_even(q0), y0 = compact_even(q0 >> 1);
      for (int u = tid; u < CHX / 2; u += NT) {
        int row = u >> 5, cp = u & 31;
        double2 v = make_double2(S.stage[row * OSLD + 2 * cp], S.stage[row * OSLD + 2 * cp + 1]);
        *reinterpret_cast<double2*>(pr.y + ((y0 + row) << P.bx) + x0 + 2 * cp) = v;
      }
    } else {
      double* o = pr.y + c * (uint64_t)CHX;
      for (int u = tid; u < CHX / 2; u += NT)
        reinterpret_cast<double2*>(o)[u] = reinterpret_cast<const double2*>(S.stage)[u];
    }
    __syncthreads();
  }
}

static constexpr size_t PREP_SMEM = 2 * 256 * RC * sizeof(cplx);

cudaError_t setup_expand_kernels() {
  cudaError_t e = cudaFuncSetAttribute(k_expand_main, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(ExSmem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_expand_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PREP_SMEM);
}

cudaError_t launch_expand(const ExProb* probs_dev, int nprob, const ExParams& prm, cudaStream_t st) {
  const int d = prm.d;
  if (d <= 13) {
    int nb = (int)(((1ull << d) + 255) / 256);
    k_expand_small<<<dim3(nb, nprob), 256, 0, st>>>(probs_dev, prm);
    count_launches(1);
    return cudaGetLastError();
  }
  k_expand_prep<<<nprob, 256, PREP_SMEM, st>>>(probs_dev, prm);
  const uint64_t nchunks = 1ull << (d - 12);
  const int target = NBLK_MAX;
  int per = (int)((nchunks + target - 1) / target);
  int nb = (int)((nchunks + per - 1) / per);
  k_expand_main<<<dim3(nb, nprob), NT, sizeof(ExSmem), st>>>(probs_dev, prm, per);
  count_launches(2);
  return cudaGetLastError();
}

}  // namespace qtt

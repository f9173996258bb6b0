// ttsvd.cu — max-rank TT-SVD (Alg. 1, with modification
// (1)) of full float64 arrays on sm_100a.
//
// The sweep over successive unfoldings A^{k} (2 r_{k-1} x 2^{d-k}, Lemma 1
// P:430) is organised so the full array is read exactly twice:
//   K1 k_level_gram   G = X_m X_m^T, X_m = reshape(x, [2^m, 2^{d-m}]), m = 5,
//                     on FP64 tensor cores (DMMA) from cp.async-staged chunks.
//   K2 k_level_solve  steps 1..m from G by projected partial traces (the
//                     Gram of A^{k} is (I2 (x) P_{k-1})^T PT_k(G) (I2 (x)
//                     P_{k-1})); Jacobi eigensolver + RANK.
//   K3 k_project      W_m = P_m^T X_m (= Sigma V^* of Alg. 1 line "A := Sigma
//                     V^*") written in QTT column order, fused with the
//                     DMMA Gram of the next unfolding reshape(W_m, [2 r_m, .]).
//   K2'/K3'           the same per step k > m on the shrinking W buffers.
//   K4 k_finish       one CTA per tensor finishes the last steps in shared
//                     memory (and does small tensors, d <= 12, entirely).
// Truncation: tau^2 = eps^2 ||x||^2 / (d-1) (reading Q1), rank =
// RANK(lambda, tau^2, R_max, delta_c) on the Gram eigenvalues lambda = sigma^2.
#include <functional>
#include <vector>

#include "qtt_dev.cuh"
#include "qtt_kernels.h"

namespace qtt {

static constexpr int NT = 256;
static constexpr int LVL_M = 5;                 // level-1 bits
static constexpr int LVL_ROWS = 1 << LVL_M;     // 32
static constexpr int CH = 4096;                 // chunk elements (64 x 64 square in 2D)
static constexpr int CH_COLS = CH / LVL_ROWS;   // 128 columns of X_m per chunk
static constexpr int SLD = 68;                  // smem row stride of an interleaved chunk
static constexpr int S1D = 36;                  // smem stride of a 32-element column (1D)
// doubles per chunk buffer: the larger of the interleaved 64 x 64 tile (ld
// SLD) and the 1D / concat 128 columns of 32 (ld S1D)
static constexpr int CHUNK_SMEM = (64 * SLD > 128 * S1D) ? 64 * SLD : 128 * S1D;
static_assert(CHUNK_SMEM >= 31 + S1D * 127 + 1 && CHUNK_SMEM >= 63 + SLD * 63 + 1, "chunk buffer too small");

// ------------------------------------------------------------ chunk I/O
// chunk-local QTT index -> smem offset
__device__ __forceinline__ int chunk_off(uint32_t q, int layout) {
  if (layout == LAYOUT_INTERLEAVED) return (int)(compact_even(q) + SLD * compact_even(q >> 1));
  return (int)((q & 31u) + S1D * (q >> 5));
}

// async copy of QTT chunk c of x into sm
__device__ __forceinline__ void load_chunk_async(double* sm, const double* x, uint64_t c, int layout,
                                                 int bx) {
  const int tid = threadIdx.x;
  if (layout == LAYOUT_INTERLEAVED) {
    const uint64_t q0 = c * (uint64_t)CH;
    const uint64_t x0 = compact_even(q0), y0 = compact_even(q0 >> 1);
    for (int u = tid; u < CH / 2; u += NT) {
      int row = u >> 5, cp = u & 31;
      cp_async16(sm + row * SLD + 2 * cp, x + ((y0 + row) << bx) + x0 + 2 * cp);
    }
  } else {
    const double* src = x + c * (uint64_t)CH;
    for (int u = tid; u < CH / 2; u += NT) {
      int col = u >> 4, w = u & 15;
      cp_async16(sm + col * S1D + 2 * w, src + 2 * u);
    }
  }
}

// TMA (bulk-copy) form of load_chunk_async, issued by one warp: the 64 rows
// of 512 B of an interleaved 64 x 64 tile, or the 128 columns of 256 B of a
// 1D / concat chunk, land in the same padded smem layout; the 32 KB are
// counted on the stage's mbarrier.
__device__ __forceinline__ void load_chunk_bulk(double* sm, const double* x, uint64_t c, int layout, int bx,
                                                uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) mbar_expect_tx(bar, CH * sizeof(double));
  __syncwarp();
  if (layout == LAYOUT_INTERLEAVED) {
    const uint64_t q0 = c * (uint64_t)CH;
    const uint64_t x0 = compact_even(q0), y0 = compact_even(q0 >> 1);
    for (int row = lane; row < 64; row += 32)
      bulk_g2s(sm + row * SLD, x + ((y0 + row) << bx) + x0, 64 * sizeof(double), bar);
  } else {
    const double* src = x + c * (uint64_t)CH;
    for (int col = lane; col < CH / 32; col += 32)
      bulk_g2s(sm + col * S1D, src + 32 * col, 32 * sizeof(double), bar);
  }
}

// ------------------------------------------------- DMMA Gram accumulation
// acc[pair][2] += Gram contributions of a (nrows x 4) column step, rows split
// in 8-row blocks nb <= 4, unique block pairs (bi <= bj).
__device__ __forceinline__ void gram_step(double (&acc)[10][2], const double (&a)[4], int nb) {
  int pi = 0;
#pragma unroll
  for (int bi = 0; bi < 4; ++bi) {
#pragma unroll
    for (int bj = bi; bj < 4; ++bj) {
      if (bj < nb) dmma884(acc[pi][0], acc[pi][1], a[bi], a[bj]);
      ++pi;
    }
  }
}

// Reduce per-warp Gram fragments (acc) over the CTA into a full 32x32
// matrix `out` (row-major == column-major, symmetric) in a fixed order.
// scratch holds >= NSCR*1024 doubles; the 8 warps go in 8/NSCR passes.
template <int NSCR = 8>
__device__ void gram_reduce_cta(const double (&acc)[10][2], double* scratch, double* out) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  double part[1024 / NT];
#pragma unroll
  for (int k = 0; k < 1024 / NT; ++k) part[k] = 0.0;
#pragma unroll
  for (int pass = 0; pass < 8 / NSCR; ++pass) {
    if (w / NSCR == pass) {
      double* mine = scratch + (w % NSCR) * 1024;
      int pi = 0;
#pragma unroll
      for (int bi = 0; bi < 4; ++bi) {
#pragma unroll
        for (int bj = bi; bj < 4; ++bj) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int r = 8 * bi + (lane >> 2), c = 8 * bj + 2 * (lane & 3) + e;
            mine[r * 32 + c] = acc[pi][e];
            if (bi != bj) mine[c * 32 + r] = acc[pi][e];
          }
          ++pi;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 1024 / NT; ++k) {
      const int e = tid + NT * k;
#pragma unroll
      for (int ww = 0; ww < NSCR; ++ww) part[k] += scratch[ww * 1024 + e];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 1024 / NT; ++k) out[tid + NT * k] = part[k];
  __syncthreads();
}

// ------------------------------------------------------------------- K1
#ifdef QTT_LEVEL_GRAM_TMA
// A/B variant (diagnostic build -DQTT_LEVEL_GRAM_TMA): the chunks stream
// through a 3-stage ring filled by TMA bulk copies (warp 0 issues one
// 512-byte copy per tile row, an mbarrier per stage counts the bytes).
// Measured slower than the cp.async double buffer below (C4 level-1 Gram
// pass 1.18 vs 0.86 ms, 56% vs 76% of HBM; profiles/r02_summary.md), so the
// product build keeps cp.async.
static constexpr int LG_STAGES = 3;
__global__ void __launch_bounds__(NT) k_level_gram(const DecProb* probs, int nblk, int* status) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ double smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LG_STAGES * CHUNK_SMEM);
  const uint64_t nchunks = 1ull << (pr.dl - 12);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  double acc[10][2];
#pragma unroll
  for (int i = 0; i < 10; ++i) acc[i][0] = acc[i][1] = 0.0;
  int rowoff[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) rowoff[b] = chunk_off(8 * b + (lane >> 2), pr.layout);
  bool bad = false;
  if (tid == 0) {
    for (int st = 0; st < LG_STAGES; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const uint64_t c0 = blockIdx.x;
  if (w == 0) {
    for (int st = 0; st < LG_STAGES - 1; ++st) {
      const uint64_t cc = c0 + (uint64_t)st * nblk;
      if (cc < nchunks) load_chunk_bulk(smem + st * CHUNK_SMEM, pr.x, cc, pr.layout, pr.bx, &bars[st]);
    }
  }
  int it = 0;
  for (uint64_t c = c0; c < nchunks; c += nblk, ++it) {
    const int st = it % LG_STAGES;
    // refill the stage consumed in the previous iteration (every thread
    // passed that iteration's closing barrier)
    if (w == 0) {
      const uint64_t cn = c + (uint64_t)(LG_STAGES - 1) * nblk;
      const int sn = (it + LG_STAGES - 1) % LG_STAGES;
      if (cn < nchunks) load_chunk_bulk(smem + sn * CHUNK_SMEM, pr.x, cn, pr.layout, pr.bx, &bars[sn]);
    }
    mbar_wait(&bars[st], (unsigned)((it / LG_STAGES) & 1));
    const double* s = smem + st * CHUNK_SMEM;
    // 32 k-steps of 4 columns per chunk, 4 per warp
#pragma unroll
    for (int kk = 0; kk < CH_COLS / 4 / (NT / 32); ++kk) {
      int ks = w * (CH_COLS / 4 / (NT / 32)) + kk;
      int col = 4 * ks + (lane & 3);
      int coff = chunk_off((uint32_t)col << LVL_M, pr.layout);
      double a[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        a[b] = s[rowoff[b] + coff];
        bad |= !isfinite(a[b]);
      }
      gram_step(acc, a, 4);
    }
    __syncthreads();
  }
#else
static constexpr int LG_STAGES = 2;
__global__ void __launch_bounds__(NT) k_level_gram(const DecProb* probs, int nblk, int* status) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ double smem[];
  double* buf[2] = {smem, smem + CHUNK_SMEM};
  const uint64_t nchunks = 1ull << (pr.dl - 12);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  double acc[10][2];
#pragma unroll
  for (int i = 0; i < 10; ++i) acc[i][0] = acc[i][1] = 0.0;
  int rowoff[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) rowoff[b] = chunk_off(8 * b + (lane >> 2), pr.layout);
  bool bad = false;
  uint64_t c = blockIdx.x;
  int it = 0;
  if (c < nchunks) load_chunk_async(buf[0], pr.x, c, pr.layout, pr.bx);
  cp_async_commit();
  for (; c < nchunks; c += nblk, ++it) {
    uint64_t nx = c + nblk;
    if (nx < nchunks) load_chunk_async(buf[(it + 1) & 1], pr.x, nx, pr.layout, pr.bx);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* s = buf[it & 1];
    // 32 k-steps of 4 columns per chunk, 4 per warp
#pragma unroll
    for (int kk = 0; kk < CH_COLS / 4 / (NT / 32); ++kk) {
      int ks = w * (CH_COLS / 4 / (NT / 32)) + kk;
      int col = 4 * ks + (lane & 3);
      int coff = chunk_off((uint32_t)col << LVL_M, pr.layout);
      double a[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        a[b] = s[rowoff[b] + coff];
        bad |= !isfinite(a[b]);
      }
      gram_step(acc, a, 4);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();
#endif
  if (bad) raise_status(status, ST_NONFINITE);
  double* out = pr.part + (size_t)blockIdx.x * 1024;
  gram_reduce_cta(acc, smem, out);
}

// ------------------------------------------------------ TT-RSVD sketches
// Modification (2) (Appendix A): Y_k = A^{k} Omega_k,
// Omega_k[j, c] from omega_pair(j, k, c >> 1, seed) (j = column of A^{k}).
// Partial sketches per CTA go to psk[blk * 1024 + i + 32 c].
static constexpr int KPMAX = 16;
static constexpr int OLD = KPMAX + 1;     // smem ld of an Omega tile row

struct SketchXSmem {
  double tile[CHUNK_SMEM];
  double om5[128 * OLD];                  // Omega_5 rows j = 128 c + col
  double om4[256 * OLD];                  // Omega_4 rows b5 + 2 j
  double red[8][1024];
};

// Level sketches from x (one extra pass): Z_5 = X_5 Omega_5 (32 x kp) and,
// if need4, Z_4[a, c] = sum_{b5, j} X_5[a + 16 b5, j] Omega_4[b5 + 2 j, c]
// (16 x kp), X_5 = reshape(x, [32, 2^{d-5}]).  Then Y_k = (I2 (x) P_{k-1})^T Z_k.
__global__ void __launch_bounds__(NT) k_sketch_x(const DecProb* probs, int nblk, int kp, int need4) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  SketchXSmem& S = *reinterpret_cast<SketchXSmem*>(smraw);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint64_t nchunks = 1ull << (pr.dl - 12);
  const int rb = lane >> 2, cb = lane & 3;                 // Z_5: rows 4rb.., cols 4cb..
  const int rb4 = (lane >> 2) & 3, b5 = lane >> 4;         // Z_4: rows 4rb4.., half b5
  double a5[4][4], a4[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) a5[i][q] = a4[i][q] = 0.0;
  int ro5[4], ro4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ro5[i] = chunk_off(4 * rb + i, pr.layout);
    ro4[i] = chunk_off(4 * rb4 + i + 16 * b5, pr.layout);
  }
  const int npairs = (kp + 1) / 2;
  for (uint64_t c = blockIdx.x; c < nchunks; c += nblk) {
    load_chunk_async(S.tile, pr.x, c, pr.layout, pr.bx);
    cp_async_commit();
    for (int e = tid; e < (need4 ? 384 : 128) * npairs; e += NT) {
      const int row = e / npairs, cp = e % npairs;
      double z0, z1;
      if (row < 128) {
        omega_pair(c * 128 + row, 5u, (unsigned)cp, pr.seed, z0, z1);
        S.om5[row * OLD + 2 * cp] = z0;
        S.om5[row * OLD + 2 * cp + 1] = z1;
      } else {
        const int r4 = row - 128;
        omega_pair(c * 256 + r4, 4u, (unsigned)cp, pr.seed, z0, z1);
        S.om4[r4 * OLD + 2 * cp] = z0;
        S.om4[r4 * OLD + 2 * cp + 1] = z1;
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int col = w; col < 128; col += NT / 32) {
      const int coff = chunk_off((uint32_t)col << LVL_M, pr.layout);
      double xv[4], ov[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = S.tile[ro5[i] + coff];
#pragma unroll
      for (int q = 0; q < 4; ++q) ov[q] = S.om5[col * OLD + 4 * cb + q];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) a5[i][q] = fma(xv[i], ov[q], a5[i][q]);
      if (need4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) xv[i] = S.tile[ro4[i] + coff];
#pragma unroll
        for (int q = 0; q < 4; ++q) ov[q] = S.om4[(b5 + 2 * col) * OLD + 4 * cb + q];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) a4[i][q] = fma(xv[i], ov[q], a4[i][q]);
      }
    }
    __syncthreads();
  }
  // fixed-order reduction over the 8 warps (and the two b5 halves of Z_4)
  double* mine = S.red[w];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      mine[(4 * rb + i) + 32 * (4 * cb + q)] = a5[i][q];
      mine[512 + (b5 ? 16 : 0) + (4 * rb4 + i) + 32 * (4 * cb + q)] = a4[i][q];
    }
  __syncthreads();
  double* out = pr.psk + (size_t)blockIdx.x * 1024;
  for (int e = tid; e < 1024; e += NT) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < NT / 32; ++ww) t += S.red[ww][e];
    S.red[0][e] = t;   // safe: each e read by its own thread only
  }
  __syncthreads();
  for (int e = tid; e < 1024; e += NT) {
    if (e < 512) {
      out[e] = S.red[0][e];
    } else {
      // Z_4 halves: rows i (< 16) at 512 + i + 32 c and 512 + 16 + i + 32 c
      const int f = e - 512, i = f & 31, cc = f >> 5;
      out[e] = (i < 16) ? S.red[0][512 + i + 32 * cc] + S.red[0][512 + 16 + i + 32 * cc] : 0.0;
    }
  }
}

struct SketchWSmem {
  double A[32 * 64];                      // 64 columns of A^{k+1} (ld rr)
  double om[64 * OLD];
  double red[8][512];
};

// Sketch of A^{k+1} = reshape(W_k, [2 r_k, 2^{d-k-1}]) (column-major: A's
// column j is W's columns 2j, 2j+1): Y_{k+1} = A^{k+1} Omega_{k+1} (rr x kp).
__global__ void __launch_bounds__(NT) k_sketch_w(const DecProb* probs, int k, int nblk, int src_is_a, int kp) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  SketchWSmem& S = *reinterpret_cast<SketchWSmem*>(smraw);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int rr = 2 * pr.ranks[k];
  const double* W = src_is_a ? pr.Wa : pr.Wb;
  const uint64_t ncols = 1ull << (pr.dl - k - 1);
  const uint64_t nchunks = (ncols + 63) / 64;
  const int rb = lane >> 2, cb = lane & 3;
  const int npairs = (kp + 1) / 2;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.0;
  for (uint64_t c = blockIdx.x; c < nchunks; c += nblk) {
    const int nc = (int)((ncols - c * 64) < 64 ? (ncols - c * 64) : 64);
    for (int e = tid; e < rr * nc; e += NT) S.A[e] = W[c * 64 * rr + e];
    for (int e = tid; e < nc * npairs; e += NT) {
      const int row = e / npairs, cp = e % npairs;
      double z0, z1;
      omega_pair(c * 64 + row, (unsigned)(k + 1), (unsigned)cp, pr.seed, z0, z1);
      S.om[row * OLD + 2 * cp] = z0;
      S.om[row * OLD + 2 * cp + 1] = z1;
    }
    __syncthreads();
    if (4 * rb < rr) {
      for (int j = w; j < nc; j += NT / 32) {
        double av[4], ov[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = (4 * rb + i < rr) ? S.A[(4 * rb + i) + rr * j] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) ov[q] = S.om[j * OLD + 4 * cb + q];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] = fma(av[i], ov[q], acc[i][q]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) S.red[w][(4 * rb + i) + 32 * (4 * cb + q)] = acc[i][q];
  __syncthreads();
  double* out = pr.psk + (size_t)blockIdx.x * 1024;
  for (int e = tid; e < 1024; e += NT) {
    double t = 0.0;
    if (e < 512)
#pragma unroll
      for (int ww = 0; ww < NT / 32; ++ww) t += S.red[ww][e];
    out[e] = t;
  }
}

// RSVD truncation of one cut (Appendix A, in Gram form): G = A A^T
// (rr x rr, row-major ld 32), Y = A Omega (rr x kp, Y[i + 32 c]).  Q = the kp
// leading eigenvectors of Y Y^T (an orthonormal basis of range(Y), the Q of
// "QR = Y"), B B^T = Q^T G Q (B = Q^* A), its eigenpairs give Sigma^2 and
// U~, U = Q U~.  Writes U_r to UB[i + 32 r] and returns r = RANK(Sigma^2).
struct RsvdBuf {
  double GK[1024];
  double QB[512];
  double UB[512];
  double TB[512];
  double Y[512];
  int rk;
};

template <int NE>
__device__ int rsvd_truncate(EigSmem<NE>& E, RsvdBuf& R, int rr, int kp, double tau2, const DecParams& prm) {
  constexpr int LD = EigSmem<NE>::LD;
  const int tid = threadIdx.x;
  for (int e = tid; e < rr * rr; e += NT) {
    const int i = e % rr, j = e / rr;
    double t = 0.0;
    for (int c = 0; c < kp; ++c) t = fma(R.Y[i + 32 * c], R.Y[j + 32 * c], t);
    E.A[0][i + LD * j] = cmk(t, 0.0);
  }
  __syncthreads();
  eig_values<NE, NT, true>(E, rr);
  const cplx* Q = eig_vectors<NE, NT>(E, rr, kp, prm.status);
  for (int e = tid; e < rr * kp; e += NT) {
    const int i = e % rr, c = e / rr;
    R.QB[i + 32 * c] = Q[i + LD * c].x;
  }
  __syncthreads();
  // TB = G Q (rr x kp), then E.A = Q^T TB (kp x kp)
  for (int e = tid; e < rr * kp; e += NT) {
    const int i = e % rr, c = e / rr;
    double t = 0.0;
    for (int j = 0; j < rr; ++j) t = fma(R.GK[i * 32 + j], R.QB[j + 32 * c], t);
    R.TB[i + 32 * c] = t;
  }
  __syncthreads();
  for (int e = tid; e < kp * kp; e += NT) {
    const int a = e % kp, b = e / kp;
    double t = 0.0;
    for (int i = 0; i < rr; ++i) t = fma(R.QB[i + 32 * a], R.TB[i + 32 * b], t);
    E.A[0][a + LD * b] = cmk(t, 0.0);
  }
  __syncthreads();
  eig_values<NE, NT, true>(E, kp);
  if (tid == 0) R.rk = rank_choose(E.lam, kp, tau2, prm.rmax, prm.ctol, 0, 0.0);
  __syncthreads();
  const int rk = R.rk;
  const cplx* Ut = eig_vectors<NE, NT>(E, kp, rk, prm.status);
  for (int e = tid; e < rr * rk; e += NT) {
    const int i = e % rr, r = e / rr;
    double t = 0.0;
    for (int a = 0; a < kp; ++a) t = fma(R.QB[i + 32 * a], Ut[a + LD * r].x, t);
    R.UB[i + 32 * r] = t;
  }
  __syncthreads();
  return rk;
}

// the TT-RSVD applies at step k when min(m_k, n_k) > R_max + p
__device__ __forceinline__ bool use_rsvd(const DecParams& prm, int rr, uint64_t ncols) {
  return prm.kp > 0 && rr > prm.kp && ncols > (uint64_t)prm.kp;
}

// ------------------------------------------------------------------- K2
// shared helper: write U_r as core k (slot k-1) and ranks[k]
__device__ void write_core_from_U(const DecProb& pr, int k, const cplx* U, int ld, int rr, int rk) {
  cplx* core = pr.cores + (size_t)(k - 1) * SLOT;
  for (int e = threadIdx.x; e < rr * rk; e += NT) {
    int a = e % rr, r = e / rr;
    core[a + rr * r] = cmk(U[a + ld * r].x, 0.0);
  }
  if (threadIdx.x == 0) pr.ranks[k] = rk;
}

__device__ void write_core_from_Ud(const DecProb& pr, int k, const double* U, int rr, int rk) {
  cplx* core = pr.cores + (size_t)(k - 1) * SLOT;
  for (int e = threadIdx.x; e < rr * rk; e += NT) {
    int a = e % rr, r = e / rr;
    core[a + rr * r] = cmk(U[a + 32 * r], 0.0);
  }
  if (threadIdx.x == 0) pr.ranks[k] = rk;
}

// sum of nsk per-CTA partial sketches (rows < rows_, kp columns) into R.Y
__device__ void gather_sketch(const DecProb& pr, int nsk, int off, int rows_, int kp, double* Y) {
  for (int e = threadIdx.x; e < rows_ * kp; e += NT) {
    const int i = e % rows_, c = e / rows_;
    double t = 0.0;
    for (int b = 0; b < nsk; ++b) t += pr.psk[(size_t)b * 1024 + off + i + 32 * c];
    Y[i + 32 * c] = t;
  }
}

template <int NE>
struct LevelSolveSmem {
  EigSmem<NE> E;
  double G[1024];
  double P[2][32 * 16];
  double PT[1024];
  int rk;
  RsvdBuf R;
};

template <int NE>
__global__ void __launch_bounds__(NT, 1) k_level_solve(const DecProb* probs, int nblk, DecParams prm, int nsk) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  LevelSolveSmem<NE>& S = *reinterpret_cast<LevelSolveSmem<NE>*>(smraw);
  const int tid = threadIdx.x;
  constexpr int LD = EigSmem<NE>::LD;
  for (int e = tid; e < 1024; e += NT) {
    double s = 0.0;
    if (nblk == 0) s = pr.gsum[e];   // Gram already reduced (across shards)
    for (int b = 0; b < nblk; ++b) s += pr.part[(size_t)b * 1024 + e];
    S.G[e] = s;
  }
  __syncthreads();
  double tr = 0.0;
  if (tid < 32) tr = S.G[tid * 33];
  tr = block_sum<NT>(tr, S.E.red);
  const int d = pr.d;
  const double tau2 = prm.eps * prm.eps * tr / (double)(d - 1);
  if (tid == 0) { *pr.tau2 = tau2; pr.ranks[0] = 1; }
  int cur = 0;
  if (tid == 0) S.P[0][0] = 1.0;
  int r_prev = 1;
  __syncthreads();
  for (int k = 1; k <= LVL_M; ++k) {
    const int n2 = 1 << k, h = n2 >> 1, rr = 2 * r_prev;
    // PT_k(G)[a][b] = sum_c G[a + n2 c][b + n2 c]
    for (int e = tid; e < n2 * n2; e += NT) {
      int a = e % n2, b = e / n2;
      double s = 0.0;
      for (int c = 0; c < (LVL_ROWS >> k); ++c) s += S.G[(a + n2 * c) * 32 + b + n2 * c];
      S.PT[a + n2 * b] = s;
    }
    __syncthreads();
    // G_k[(rho,be),(sg,ga)] = sum P[jl][rho] PT[jl + h be][jl' + h ga] P[jl'][sg]
    const double* Pp = S.P[cur];
    for (int e = tid; e < rr * rr; e += NT) {
      int i = e % rr, j = e / rr;
      int rho = i % r_prev, be = i / r_prev, sg = j % r_prev, ga = j / r_prev;
      double s = 0.0;
      for (int jl = 0; jl < h; ++jl) {
        double t = 0.0;
        for (int jl2 = 0; jl2 < h; ++jl2) t += S.PT[(jl + h * be) + n2 * (jl2 + h * ga)] * Pp[jl2 + 32 * sg];
        s += Pp[jl + 32 * rho] * t;
      }
      S.E.A[0][i + LD * j] = cmk(s, 0.0);
      S.R.GK[i * 32 + j] = s;
    }
    __syncthreads();
    int rk;
    const cplx* U = nullptr;
    const bool rs = (k == 4 || k == 5) && nsk > 0 && use_rsvd(prm, rr, 1ull << (d - k));
    if (rs) {
      // Y_k = (I2 (x) P_{k-1})^T Z_k, Z_5 at psk offset 0 (32 rows), Z_4 at 512 (16 rows)
      gather_sketch(pr, nsk, k == 5 ? 0 : 512, n2, prm.kp, S.R.TB);
      __syncthreads();
      for (int e = tid; e < rr * prm.kp; e += NT) {
        const int i = e % rr, c = e / rr;
        const int rho = i % r_prev, be = i / r_prev;
        double t = 0.0;
        for (int a = 0; a < h; ++a) t = fma(Pp[a + 32 * rho], S.R.TB[(a + h * be) + 32 * c], t);
        S.R.Y[i + 32 * c] = t;
      }
      __syncthreads();
      rk = rsvd_truncate<NE>(S.E, S.R, rr, prm.kp, tau2, prm);
      write_core_from_Ud(pr, k, S.R.UB, rr, rk);
    } else {
      eig_values<NE, NT, true>(S.E, rr);
      if (tid == 0) {
        int mp = rr < (1 << (d - k)) ? rr : (1 << (d - k));
        S.rk = rank_choose(S.E.lam, mp, tau2, prm.rmax, prm.ctol, prm.rule, prm.delta, prm.status);
      }
      __syncthreads();
      rk = S.rk;
      U = eig_vectors<NE, NT>(S.E, rr, rk, prm.status);
      write_core_from_U(pr, k, U, LD, rr, rk);
    }
    // P_k[a][r] = sum_rho P_{k-1}[a mod h][rho] U[rho + r_prev (a div h)][r]
    double* Pn = S.P[cur ^ 1];
    for (int e = tid; e < n2 * rk; e += NT) {
      int a = e % n2, r = e / n2;
      int al = a % h, ah = a / h;
      double s = 0.0;
      for (int rho = 0; rho < r_prev; ++rho)
        s += Pp[al + 32 * rho] * (rs ? S.R.UB[rho + r_prev * ah + 32 * r] : U[rho + r_prev * ah + LD * r].x);
      Pn[a + 32 * r] = s;
    }
    __syncthreads();
    cur ^= 1;
    r_prev = rk;
  }
  for (int e = tid; e < 32 * r_prev; e += NT) pr.proj[e] = S.P[cur][e];
}

// ------------------------------------------------------------------- K3
// Project a 128-column tile (Krows x 128, accessed through `xs`) by P^T
// (Krows x r in global, ld 32) into W (r x 128) and accumulate the DMMA Gram
// of reshape(W, [2r, 64]).
struct ProjSmem {
  double tile[2][CHUNK_SMEM];
  double W[16 * 128];
};

template <bool FROM_X>
__device__ __forceinline__ void load_tile(double* sm, const DecProb& pr, const double* src, uint64_t c,
                                          int krows, int kp) {
  if (FROM_X) {
    load_chunk_async(sm, pr.x, c, pr.layout, pr.bx);
  } else {
    // columns [128 c, 128 c + 128) of a krows x n matrix (ld krows) -> column stride kp
    const double* s = src + (size_t)c * 128 * krows;
    const int units = krows / 2;
    for (int u = threadIdx.x; u < 128 * units; u += NT) {
      int col = u / units, w = u % units;
      cp_async16(sm + col * kp + 2 * w, s + (size_t)col * krows + 2 * w);
    }
  }
}

// K3 (FROM_X) and K3' (!FROM_X): step k projector applied, writes W_k, Gram for step k+1.
template <bool FROM_X>
__global__ void __launch_bounds__(NT) k_project(const DecProb* probs, int k, int nblk, int src_is_a) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  ProjSmem& S = *reinterpret_cast<ProjSmem*>(smraw);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int d = pr.d;
  const int rk = pr.ranks[k];
  const int krows = FROM_X ? LVL_ROWS : 2 * pr.ranks[k - 1];
  int kp = (krows + 3) & ~3;
  if ((kp & 7) == 0) kp += 4;
  const double* src = FROM_X ? nullptr : (src_is_a ? pr.Wa : pr.Wb);
  double* dst = FROM_X ? pr.Wa : (src_is_a ? pr.Wb : pr.Wa);
  const uint64_t ncols = 1ull << (pr.dl - k);    // (local) columns of W_k
  const uint64_t nchunks = ncols / 128;
  // projector fragments: A = P^T (r x krows): a[mb][ks] = P[4ks + lane&3][8mb + lane>>2]
  double afr[2][8];
#pragma unroll
  for (int mb = 0; mb < 2; ++mb)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      int row = 4 * ks + (lane & 3), col = 8 * mb + (lane >> 2);
      afr[mb][ks] = (row < krows && col < rk) ? pr.proj[row + 32 * col] : 0.0;
    }
  const int ksteps = (krows + 3) / 4;
  const int nbg = (2 * rk + 7) / 8;   // row blocks of the next Gram
  double gacc[10][2];
#pragma unroll
  for (int i = 0; i < 10; ++i) gacc[i][0] = gacc[i][1] = 0.0;
  int it = 0;
  uint64_t c = blockIdx.x;
  if (c < nchunks) load_tile<FROM_X>(S.tile[0], pr, src, c, krows, kp);
  cp_async_commit();
  for (; c < nchunks; c += nblk, ++it) {
    uint64_t nx = c + nblk;
    if (nx < nchunks) load_tile<FROM_X>(S.tile[(it + 1) & 1], pr, src, nx, krows, kp);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* s = S.tile[it & 1];
    // projection: warp w handles n-blocks w and w + 8 (16 blocks of 8 columns)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int nb = w + 8 * h;
      const int col = 8 * nb + (lane >> 2);
      double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (ks < ksteps) {
          int row = 4 * ks + (lane & 3);
          double b;
          if (FROM_X) b = s[chunk_off((uint32_t)row + ((uint32_t)col << LVL_M), pr.layout)];
          else b = (row < krows) ? s[row + kp * col] : 0.0;
          dmma884(c0[0], c0[1], afr[0][ks], b);
          dmma884(c1[0], c1[1], afr[1][ks], b);
        }
      }
      // C[mb][row r][col]: r = 8 mb + lane>>2, col = 8 nb + 2 (lane&3) + e
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int cc = 8 * nb + 2 * (lane & 3) + e;
        int r0 = lane >> 2, r1 = 8 + (lane >> 2);
        if (r0 < rk) S.W[r0 + rk * cc] = c0[e];
        if (r1 < rk) S.W[r1 + rk * cc] = c1[e];
      }
    }
    __syncthreads();
    // write W tile (contiguous rk*128 doubles)
    {
      double* o = dst + (size_t)c * 128 * rk;
      const int n2 = rk * 64;  // 16-byte units
      for (int u = tid; u < n2; u += NT)
        reinterpret_cast<double2*>(o)[u] = reinterpret_cast<const double2*>(S.W)[u];
    }
    // fused Gram of reshape(W, [2 rk, 64]): 16 k-steps, 2 per warp
    if (k + 1 <= d - 1) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        int ks = 2 * w + kk;
        int colg = 4 * ks + (lane & 3);
        double a[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          int row = 8 * b + (lane >> 2);
          a[b] = (row < 2 * rk) ? S.W[row + 2 * rk * colg] : 0.0;
        }
        gram_step(gacc, a, nbg);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();
  gram_reduce_cta(gacc, &S.tile[0][0], pr.part + (size_t)blockIdx.x * 1024);
}

// ------------------------------------------------------------------- K2'
template <int NE>
struct StepSolveSmem {
  EigSmem<NE> E;
  int rk;
  RsvdBuf R;
};

template <int NE>
__global__ void __launch_bounds__(NT, 1) k_step_solve(const DecProb* probs, int k, int nblk, DecParams prm, int nsk) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  StepSolveSmem<NE>& S = *reinterpret_cast<StepSolveSmem<NE>*>(smraw);
  constexpr int LD = EigSmem<NE>::LD;
  const int tid = threadIdx.x;
  const int r_prev = pr.ranks[k - 1], rr = 2 * r_prev;
  for (int e = tid; e < rr * rr; e += NT) {
    int i = e % rr, j = e / rr;
    double s = 0.0;
    if (nblk == 0) s = pr.gsum[i * 32 + j];   // Gram already reduced (across shards)
    for (int b = 0; b < nblk; ++b) s += pr.part[(size_t)b * 1024 + i * 32 + j];
    S.E.A[0][i + LD * j] = cmk(s, 0.0);
    S.R.GK[i * 32 + j] = s;
  }
  __syncthreads();
  if (nsk > 0 && use_rsvd(prm, rr, 1ull << (pr.d - k))) {
    gather_sketch(pr, nsk, 0, rr, prm.kp, S.R.Y);
    __syncthreads();
    const int rk = rsvd_truncate<NE>(S.E, S.R, rr, prm.kp, *pr.tau2, prm);
    write_core_from_Ud(pr, k, S.R.UB, rr, rk);
    for (int e = tid; e < rr * rk; e += NT) {
      int a = e % rr, r = e / rr;
      pr.proj[a + 32 * r] = S.R.UB[a + 32 * r];
    }
    return;
  }
#ifdef QTT_STEP_TIMING
  long long c0 = clock64();
#endif
  eig_values<NE, NT, true>(S.E, rr);
#ifdef QTT_STEP_TIMING
  long long c1 = clock64();
#endif
  if (tid == 0) {
    int mp = rr < (1 << (pr.d - k)) ? rr : (1 << (pr.d - k));
    S.rk = rank_choose(S.E.lam, mp, *pr.tau2, prm.rmax, prm.ctol, prm.rule, prm.delta, prm.status);
  }
  __syncthreads();
  const int rk = S.rk;
  const cplx* U = eig_vectors<NE, NT>(S.E, rr, rk, prm.status);
#ifdef QTT_STEP_TIMING
  if (tid == 0)
    printf("step %d prob %d rr %d rk %d values %lld vectors %lld fallbacks %d tphase %lld %lld %lld %lld %lld\n", k,
           blockIdx.y, rr, rk, c1 - c0, clock64() - c1, *prm.status, S.E.u.tr.tph[0], S.E.u.tr.tph[1],
           S.E.u.tr.tph[2], S.E.u.tr.tph[3], S.E.u.tr.tph[4]);
#endif
  write_core_from_U(pr, k, U, LD, rr, rk);
  for (int e = tid; e < rr * rk; e += NT) {
    int a = e % rr, r = e / rr;
    pr.proj[a + 32 * r] = U[a + LD * r].x;
  }
}

// ------------------------------------------------------------------- K4
static constexpr int FIN_CAP = 4096;             // doubles of W_{k-1} the finisher holds
static constexpr int FIN_COLS = FIN_CAP / RC;     // 256 columns at the rank cap
static_assert(FIN_COLS == FIN_COLS_HOST, "host driver mirrors FIN_COLS");
static constexpr int FIN_D = 12;                  // d <= 12: whole TT-SVD in one CTA
template <int NE>
struct FinishSmem {
  double B[2][FIN_CAP];
  RsvdBuf R;
  EigSmem<NE> E;
  double G[1024];
  int rk;
};

// Gram of an (rows x n) matrix in smem (ld rows) with DMMA, into S.G (32x32),
// using scratch (>= 8*1024 doubles).
__device__ void gram_smem(const double* M, int rows, int n, double* scratch, double* G) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  double acc[10][2];
#pragma unroll
  for (int i = 0; i < 10; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int nb = (rows + 7) / 8;
  const int ksteps = (n + 3) / 4;
  for (int ks = w; ks < ksteps; ks += NT / 32) {
    int col = 4 * ks + (lane & 3);
    double a[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int row = 8 * b + (lane >> 2);
      a[b] = (row < rows && col < n) ? M[row + rows * col] : 0.0;
    }
    gram_step(acc, a, nb);
  }
  __syncthreads();
  gram_reduce_cta<4>(acc, scratch, G);
}

template <int NE>
__global__ void __launch_bounds__(NT, 1) k_finish(const DecProb* probs, int kstart, int src_is_a,
                                               DecParams prm) {
  const DecProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  FinishSmem<NE>& S = *reinterpret_cast<FinishSmem<NE>*>(smraw);
  constexpr int LD = EigSmem<NE>::LD;
  const int tid = threadIdx.x;
  const int d = pr.d;
  int r_prev;
  double tau2;
  int cur = 0;
  if (kstart == 1) {
    const uint64_t n = 1ull << d;
    bool bad = false;
    double nrm = 0.0;
    for (uint64_t q = tid; q < n; q += NT) {
      double v = pr.x[qtt_offset(q, pr.layout, pr.bx)];
      bad |= !isfinite(v);
      S.B[0][q] = v;
    }
    if (bad) raise_status(prm.status, ST_NONFINITE);
    __syncthreads();
    for (uint64_t q = tid; q < n; q += NT) nrm += S.B[0][q] * S.B[0][q];
    nrm = block_sum<NT>(nrm, S.E.red);
    tau2 = prm.eps * prm.eps * nrm / (double)(d - 1);
    if (tid == 0) { *pr.tau2 = tau2; pr.ranks[0] = 1; }
    r_prev = 1;
  } else {
    r_prev = pr.ranks[kstart - 1];
    tau2 = *pr.tau2;
    const double* src = src_is_a ? pr.Wa : pr.Wb;
    const int tot = r_prev << (d - kstart + 1);
    for (int e = tid; e < tot; e += NT) S.B[0][e] = src[e];
  }
  __syncthreads();
  for (int k = kstart; k <= d - 1; ++k) {
    const int rr = 2 * r_prev;
    const int n = 1 << (d - k);
    gram_smem(S.B[cur], rr, n, S.B[cur ^ 1], S.G);
    for (int e = tid; e < rr * rr; e += NT) {
      int i = e % rr, j = e / rr;
      S.E.A[0][i + LD * j] = cmk(S.G[i * 32 + j], 0.0);
      S.R.GK[i * 32 + j] = S.G[i * 32 + j];
    }
    __syncthreads();
    int rk;
    const cplx* U = nullptr;
    const bool rs = use_rsvd(prm, rr, (uint64_t)n);
    if (rs) {
      // Y = A Omega_k directly from the unfolding in smem (A = B[cur], rr x n),
      // Omega generated in blocks of 64 rows into the free buffer
      double* om = S.B[cur ^ 1];
      const int npairs = (prm.kp + 1) / 2;
      for (int e = tid; e < rr * prm.kp; e += NT) S.R.Y[(e % rr) + 32 * (e / rr)] = 0.0;
      for (int j0 = 0; j0 < n; j0 += 64) {
        const int nb = n - j0 < 64 ? n - j0 : 64;
        for (int e = tid; e < nb * npairs; e += NT) {
          const int row = e / npairs, cp = e % npairs;
          double z0, z1;
          omega_pair((unsigned long long)(j0 + row), (unsigned)k, (unsigned)cp, pr.seed, z0, z1);
          om[row * OLD + 2 * cp] = z0;
          om[row * OLD + 2 * cp + 1] = z1;
        }
        __syncthreads();
        for (int e = tid; e < rr * prm.kp; e += NT) {
          const int i = e % rr, c = e / rr;
          double t = 0.0;
          for (int j = 0; j < nb; ++j) t = fma(S.B[cur][i + rr * (j0 + j)], om[j * OLD + c], t);
          S.R.Y[i + 32 * c] += t;
        }
        __syncthreads();
      }
      rk = rsvd_truncate<NE>(S.E, S.R, rr, prm.kp, tau2, prm);
      write_core_from_Ud(pr, k, S.R.UB, rr, rk);
    } else {
      eig_values<NE, NT, true>(S.E, rr);
      if (tid == 0) {
        int mp = rr < n ? rr : n;
        S.rk = rank_choose(S.E.lam, mp, tau2, prm.rmax, prm.ctol, prm.rule, prm.delta, prm.status);
      }
      __syncthreads();
      rk = S.rk;
      U = eig_vectors<NE, NT>(S.E, rr, rk, prm.status);
      write_core_from_U(pr, k, U, LD, rr, rk);
    }
    // W_k = U_r^T M_k
    const double* M = S.B[cur];
    double* Wn = S.B[cur ^ 1];
    __syncthreads();
    for (int e = tid; e < rk * n; e += NT) {
      int r = e % rk, j = e / rk;
      double s = 0.0;
      for (int a = 0; a < rr; ++a) s += (rs ? S.R.UB[a + 32 * r] : U[a + LD * r].x) * M[a + rr * j];
      Wn[r + rk * j] = s;
    }
    __syncthreads();
    cur ^= 1;
    r_prev = rk;
  }
  // last core: reshape(W_{d-1}, [r, 2, 1])
  cplx* core = pr.cores + (size_t)(d - 1) * SLOT;
  for (int e = tid; e < 2 * r_prev; e += NT) core[e] = cmk(S.B[cur][e], 0.0);
  if (tid == 0) pr.ranks[d] = 1;
}

size_t smem_level_gram() { return LG_STAGES * CHUNK_SMEM * sizeof(double) + LG_STAGES * sizeof(uint64_t); }
template <int NE> size_t smem_level_solve() { return sizeof(LevelSolveSmem<NE>); }
size_t smem_project() { return sizeof(ProjSmem); }
template <int NE> size_t smem_step_solve() { return sizeof(StepSolveSmem<NE>); }
template <int NE> size_t smem_finish() { return sizeof(FinishSmem<NE>); }
// solver width: 2 r_{k-1} <= 2 R_max rows; 20 covers R_max <= 10 (all configs)
static inline bool narrow(const DecParams& prm) { return prm.rmax <= 10; }

// ------------------------------------------------- sharded-path helpers
// gsum_t = sum over the tensor's local shards j (in order) of sum over the
// per-CTA partials b.  Grid (32, ntens): CTA x owns 32 Gram entries, its 8
// warps split the partials and are combined in a fixed order.
__global__ void __launch_bounds__(NT) k_gram_reduce(const DecProb* sh, int nlocal, int nblk) {
  __shared__ double red[NT / 32][32];
  const int t = blockIdx.y, lane = threadIdx.x & 31, wb = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double tot = 0.0;
  for (int j = 0; j < nlocal; ++j) {
    const DecProb& pr = sh[t * nlocal + j];
    // 4 independent chains per lane keep 4 loads in flight; fixed order
    constexpr int W = NT / 32;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int b = wb;
    for (; b + 3 * W < nblk; b += 4 * W) {
      s0 += pr.part[(size_t)b * 1024 + e];
      s1 += pr.part[(size_t)(b + W) * 1024 + e];
      s2 += pr.part[(size_t)(b + 2 * W) * 1024 + e];
      s3 += pr.part[(size_t)(b + 3 * W) * 1024 + e];
    }
    for (; b < nblk; b += W) s0 += pr.part[(size_t)b * 1024 + e];
    red[wb][lane] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (wb == 0) {
      double u = 0.0;
#pragma unroll
      for (int q = 0; q < NT / 32; ++q) u += red[q][lane];
      tot += u;
    }
    __syncthreads();
  }
  if (wb == 0) sh[t * nlocal].gsum[e] = tot;
}

// tn[t].Wa[:, nl j + c] = W_k of shard j, column c (r_k rows).  Source: the
// local shards' ping-pong buffer, or the all-gathered blocks of RS_GATHER*nl.
__global__ void __launch_bounds__(NT) k_gather_w(const DecProb* sh, const DecProb* tn, int nlocal, int k,
                                                 long long nl, int src_is_a, const double* gathered,
                                                 int nshards) {
  const int t = blockIdx.y;
  const DecProb& T = tn[t];
  const int r = T.ranks[k];
  const long long blk = (long long)r * nl;
  for (int j = 0; j < nshards; ++j) {
    const double* src;
    if (gathered) src = gathered + ((size_t)t * nshards + j) * (size_t)(RS_GATHER * nl);
    else src = src_is_a ? sh[t * nlocal + j].Wa : sh[t * nlocal + j].Wb;
    for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < blk; e += (long long)gridDim.x * NT)
      T.Wa[j * blk + e] = src[e];
  }
}

// CTAs per problem of a full-array pass: the whole launch targets 4 CTAs
// per SM of the device however many problems it carries, so batched
// launches keep several chunks per CTA (the cp.async double buffer reaches
// steady state) and write few per-CTA partial Grams (8 KiB each).
// grid cap override while planning a launch with reserved slots (launch_ttsvd)
static thread_local int t_grid_cap = 0;
static inline int per_problem(uint64_t nchunks, int nprob) {
  const int grid_target = 4 * sm_count();
  uint64_t want = (uint64_t)((grid_target + nprob - 1) / nprob);
  if (want > (uint64_t)NBLK_MAX) want = NBLK_MAX;
  if (t_grid_cap > 0) {   // the whole launch stays within the resident slots minus the reserve
    const uint64_t cap = (uint64_t)(t_grid_cap / nprob > 0 ? t_grid_cap / nprob : 1);
    if (want > cap) want = cap;
  }
  if (want > nchunks) want = nchunks;
  return want < 1 ? 1 : (int)want;
}

int dec_nblk_loc(int dl, int nprob) { return per_problem(1ull << (dl - 12), nprob); }

int proj_nblk(int ncols, int nprob) { return per_problem((uint64_t)(ncols / 128), nprob); }

cudaError_t launch_level_gram(const DecProb* sh, int nsh, int nblk, int* status, cudaStream_t st) {
  k_level_gram<<<dim3(nblk, nsh), NT, smem_level_gram(), st>>>(sh, nblk, status);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_gram_reduce(const DecProb* sh, int ntens, int nlocal, int nblk, cudaStream_t st) {
  k_gram_reduce<<<dim3(32, ntens), NT, 0, st>>>(sh, nlocal, nblk);
  count_launches(1);
  return cudaGetLastError();
}

// The solve kernels run in one CTA per tensor: the per-CTA partial Grams are
// summed first by k_gram_reduce (32 CTAs per tensor) into gsum.
cudaError_t launch_level_solve(const DecProb* tn, int ntens, int nblk, DecParams prm, cudaStream_t st, int nsk) {
  if (nblk > 0) {
    launch_gram_reduce(tn, ntens, 1, nblk, st);
    nblk = 0;
  }
  if (narrow(prm)) k_level_solve<20><<<dim3(1, ntens), NT, smem_level_solve<20>(), st>>>(tn, nblk, prm, nsk);
  else k_level_solve<32><<<dim3(1, ntens), NT, smem_level_solve<32>(), st>>>(tn, nblk, prm, nsk);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_step_solve(const DecProb* tn, int ntens, int k, int nblk, DecParams prm, cudaStream_t st,
                              int nsk) {
  if (nblk > 0) {
    launch_gram_reduce(tn, ntens, 1, nblk, st);
    nblk = 0;
  }
  if (narrow(prm)) k_step_solve<20><<<dim3(1, ntens), NT, smem_step_solve<20>(), st>>>(tn, k, nblk, prm, nsk);
  else k_step_solve<32><<<dim3(1, ntens), NT, smem_step_solve<32>(), st>>>(tn, k, nblk, prm, nsk);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_project(bool from_x, const DecProb* pr, int nprob, int k, int nblk, int src_is_a,
                           cudaStream_t st) {
  if (from_x) k_project<true><<<dim3(nblk, nprob), NT, smem_project(), st>>>(pr, k, nblk, src_is_a);
  else k_project<false><<<dim3(nblk, nprob), NT, smem_project(), st>>>(pr, k, nblk, src_is_a);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_finish(const DecProb* tn, int ntens, int k, int src_is_a, DecParams prm, cudaStream_t st) {
  if (narrow(prm)) k_finish<20><<<dim3(1, ntens), NT, smem_finish<20>(), st>>>(tn, k, src_is_a, prm);
  else k_finish<32><<<dim3(1, ntens), NT, smem_finish<32>(), st>>>(tn, k, src_is_a, prm);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_gather_w(const DecProb* sh, const DecProb* tn, int ntens, int nlocal, int k, long long nl,
                            int src_is_a, const double* gathered, int nshards, cudaStream_t st) {
  k_gather_w<<<dim3(8, ntens), NT, 0, st>>>(sh, tn, nlocal, k, nl, src_is_a, gathered, nshards);
  count_launches(1);
  return cudaGetLastError();
}

// ------------------------------------------------------------ host driver

int dec_nblk(int d, int nprob) {
  if (d <= FIN_D) return 0;
  return dec_nblk_loc(d, nprob);
}

cudaError_t setup_ttsvd_kernels() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_level_gram, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_level_gram())))
    return e;
#define QTT_SET_SMEM(K, BYTES) \
  if ((e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(BYTES)))) return e;
  QTT_SET_SMEM(k_level_solve<20>, smem_level_solve<20>())
  QTT_SET_SMEM(k_level_solve<32>, smem_level_solve<32>())
  QTT_SET_SMEM(k_project<true>, smem_project())
  QTT_SET_SMEM(k_project<false>, smem_project())
  QTT_SET_SMEM(k_step_solve<20>, smem_step_solve<20>())
  QTT_SET_SMEM(k_step_solve<32>, smem_step_solve<32>())
  QTT_SET_SMEM(k_finish<20>, smem_finish<20>())
  QTT_SET_SMEM(k_finish<32>, smem_finish<32>())
  QTT_SET_SMEM(k_sketch_x, sizeof(SketchXSmem))
  QTT_SET_SMEM(k_sketch_w, sizeof(SketchWSmem))
#undef QTT_SET_SMEM
  return cudaSuccess;
}

// The TT-SVD of nprob problems of equal d as a list of launches, each tagged
// HBM (a pass over x or W: grid over all SMs) or latency-bound (the one-CTA
// solves and their partial-Gram reduction).
struct TtsvdOp {
  bool hbm;
  std::function<void(cudaStream_t)> run;
};
static std::vector<TtsvdOp> ttsvd_ops(const DecProb* probs_dev, int nprob, int d, DecParams prm) {
  std::vector<TtsvdOp> ops;
  if (d <= FIN_D) {
    ops.push_back({false, [=](cudaStream_t st) { launch_finish(probs_dev, nprob, 1, 1, prm, st); }});
    return ops;
  }
  const int nblk = dec_nblk(d, nprob);
  // TT-RSVD (modification (2)): level sketches Z_5 (and Z_4) from one more pass over x
  int nsx = 0;
  if (prm.kp > 0 && (1ull << (d - LVL_M)) > (uint64_t)prm.kp) nsx = nblk;
  ops.push_back({true, [=](cudaStream_t st) {
    prof_pass(PASS_LEVEL_GRAM, 0, st);
    k_level_gram<<<dim3(nblk, nprob), NT, smem_level_gram(), st>>>(probs_dev, nblk, prm.status);
    prof_pass(PASS_LEVEL_GRAM, 1, st);
    count_launches(1);
    if (nsx) {
      const int need4 = (16 > prm.kp) && ((1ull << (d - 4)) > (uint64_t)prm.kp);
      k_sketch_x<<<dim3(nsx, nprob), NT, sizeof(SketchXSmem), st>>>(probs_dev, nsx, prm.kp, need4);
      count_launches(1);
    }
  }});
  ops.push_back({false, [=](cudaStream_t st) { launch_level_solve(probs_dev, nprob, nblk, prm, st, nsx); }});
  // K3: W_m from x, Gram for step m+1
  int k = LVL_M;
  const int nb = proj_nblk(1 << (d - k), nprob);
  ops.push_back({true, [=](cudaStream_t st) {
    prof_pass(PASS_PROJECT_X, 0, st);
    k_project<true><<<dim3(nb, nprob), NT, smem_project(), st>>>(probs_dev, k, nb, 1);
    prof_pass(PASS_PROJECT_X, 1, st);
    count_launches(1);
  }});
  int src_is_a = 1;  // W_m lives in Wa
  int prev_nb = nb;
  ++k;
  // steps while W_{k-1} has more than FIN_COLS columns
  while ((1 << (d - k + 1)) > FIN_COLS) {
    // TT-RSVD: sketch of A^{k} = reshape(W_{k-1}) when its columns exceed k + p
    int nsk = 0;
    if (prm.kp > 0 && (1ull << (d - k)) > (uint64_t)prm.kp) nsk = per_problem((1ull << (d - k)) / 64, nprob);
    ops.push_back({false, [=](cudaStream_t st) {
      if (nsk) {
        k_sketch_w<<<dim3(nsk, nprob), NT, sizeof(SketchWSmem), st>>>(probs_dev, k - 1, nsk, src_is_a, prm.kp);
        count_launches(1);
      }
      launch_step_solve(probs_dev, nprob, k, prev_nb, prm, st, nsk);
    }});
    const int nb2 = proj_nblk(1 << (d - k), nprob);
    const bool first_w = k == LVL_M + 1;
    ops.push_back({true, [=](cudaStream_t st) {
      if (first_w) prof_pass(PASS_PROJECT_W, 0, st);
      k_project<false><<<dim3(nb2, nprob), NT, smem_project(), st>>>(probs_dev, k, nb2, src_is_a);
      if (first_w) prof_pass(PASS_PROJECT_W, 1, st);
      count_launches(1);
    }});
    src_is_a ^= 1;
    prev_nb = nb2;
    ++k;
  }
  ops.push_back({false, [=](cudaStream_t st) { launch_finish(probs_dev, nprob, k, src_is_a, prm, st); }});
  return ops;
}

// Launch the whole TT-SVD for nprob problems of equal d (device array probs).
// reserve > 0: the HBM passes leave `reserve` CTA slots free (2 CTAs per SM
// otherwise), so a solve CTA of a concurrent chain on another stream becomes
// resident at once instead of after the whole pass (see qtt_conv_full).
cudaError_t launch_ttsvd(const DecProb* probs_dev, int nprob, int d, DecParams prm, cudaStream_t st, int reserve) {
  if (reserve > 0) t_grid_cap = 2 * sm_count() - reserve;
  std::vector<TtsvdOp> ops = ttsvd_ops(probs_dev, nprob, d, prm);
  t_grid_cap = 0;
  for (const TtsvdOp& op : ops) op.run(st);
  return cudaGetLastError();
}


}  // namespace qtt

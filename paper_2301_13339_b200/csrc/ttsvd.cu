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
static constexpr int CHUNK_SMEM = 64 * SLD;     // doubles per chunk buffer (>= 128*36)

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
  if (bad) raise_status(status, ST_NONFINITE);
  double* out = pr.part + (size_t)blockIdx.x * 1024;
  gram_reduce_cta(acc, smem, out);
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

template <int NE>
struct LevelSolveSmem {
  EigSmem<NE> E;
  double G[1024];
  double P[2][32 * 16];
  double PT[1024];
  int rk;
};

template <int NE>
__global__ void __launch_bounds__(NT) k_level_solve(const DecProb* probs, int nblk, DecParams prm) {
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
    }
    __syncthreads();
    eig_values<NE, NT>(S.E, rr);
    if (tid == 0) {
      int mp = rr < (1 << (d - k)) ? rr : (1 << (d - k));
      S.rk = rank_choose(S.E.lam, mp, tau2, prm.rmax, prm.ctol, prm.rule, prm.delta);
    }
    __syncthreads();
    const int rk = S.rk;
    const cplx* U = eig_vectors<NE, NT>(S.E, rr, rk, prm.status);
    write_core_from_U(pr, k, U, LD, rr, rk);
    // P_k[a][r] = sum_rho P_{k-1}[a mod h][rho] U[rho + r_prev (a div h)][r]
    double* Pn = S.P[cur ^ 1];
    for (int e = tid; e < n2 * rk; e += NT) {
      int a = e % n2, r = e / n2;
      int al = a % h, ah = a / h;
      double s = 0.0;
      for (int rho = 0; rho < r_prev; ++rho) s += Pp[al + 32 * rho] * U[rho + r_prev * ah + LD * r].x;
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
};

template <int NE>
__global__ void __launch_bounds__(NT) k_step_solve(const DecProb* probs, int k, int nblk, DecParams prm) {
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
  }
  __syncthreads();
  eig_values<NE, NT>(S.E, rr);
  if (tid == 0) {
    int mp = rr < (1 << (pr.d - k)) ? rr : (1 << (pr.d - k));
    S.rk = rank_choose(S.E.lam, mp, *pr.tau2, prm.rmax, prm.ctol, prm.rule, prm.delta);
  }
  __syncthreads();
  const int rk = S.rk;
  const cplx* U = eig_vectors<NE, NT>(S.E, rr, rk, prm.status);
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
__global__ void __launch_bounds__(NT) k_finish(const DecProb* probs, int kstart, int src_is_a,
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
    }
    __syncthreads();
    eig_values<NE, NT>(S.E, rr);
    if (tid == 0) {
      int mp = rr < n ? rr : n;
      S.rk = rank_choose(S.E.lam, mp, tau2, prm.rmax, prm.ctol, prm.rule, prm.delta);
    }
    __syncthreads();
    const int rk = S.rk;
    const cplx* U = eig_vectors<NE, NT>(S.E, rr, rk, prm.status);
    write_core_from_U(pr, k, U, LD, rr, rk);
    // W_k = U_r^T M_k
    const double* M = S.B[cur];
    double* Wn = S.B[cur ^ 1];
    for (int e = tid; e < rk * n; e += NT) {
      int r = e % rk, j = e / rk;
      double s = 0.0;
      for (int a = 0; a < rr; ++a) s += U[a + LD * r].x * M[a + rr * j];
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

size_t smem_level_gram() { return 2 * CHUNK_SMEM * sizeof(double); }
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
    double s = 0.0;
    for (int b = wb; b < nblk; b += NT / 32) s += pr.part[(size_t)b * 1024 + e];
    red[wb][lane] = s;
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

// CTAs per problem of a full-array pass: the whole launch targets
// GRID_TARGET CTAs (4 per SM) however many problems it carries, so batched
// launches keep several chunks per CTA (the cp.async double buffer reaches
// steady state) and write few per-CTA partial Grams (8 KiB each).
static constexpr int GRID_TARGET = 4 * 148;
static inline int per_problem(uint64_t nchunks, int nprob) {
  uint64_t want = (uint64_t)((GRID_TARGET + nprob - 1) / nprob);
  if (want > (uint64_t)NBLK_MAX) want = NBLK_MAX;
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

cudaError_t launch_level_solve(const DecProb* tn, int ntens, int nblk, DecParams prm, cudaStream_t st) {
  if (narrow(prm)) k_level_solve<20><<<dim3(1, ntens), NT, smem_level_solve<20>(), st>>>(tn, nblk, prm);
  else k_level_solve<32><<<dim3(1, ntens), NT, smem_level_solve<32>(), st>>>(tn, nblk, prm);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_step_solve(const DecProb* tn, int ntens, int k, int nblk, DecParams prm, cudaStream_t st) {
  if (narrow(prm)) k_step_solve<20><<<dim3(1, ntens), NT, smem_step_solve<20>(), st>>>(tn, k, nblk, prm);
  else k_step_solve<32><<<dim3(1, ntens), NT, smem_step_solve<32>(), st>>>(tn, k, nblk, prm);
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
#undef QTT_SET_SMEM
  return cudaSuccess;
}

// Launch the whole TT-SVD for nprob problems of equal d (device array probs).
cudaError_t launch_ttsvd(const DecProb* probs_dev, int nprob, int d, DecParams prm, cudaStream_t st) {
  if (d <= FIN_D) {
    return launch_finish(probs_dev, nprob, 1, 1, prm, st);
  }
  const int nblk = dec_nblk(d, nprob);
  k_level_gram<<<dim3(nblk, nprob), NT, smem_level_gram(), st>>>(probs_dev, nblk, prm.status);
  count_launches(1);
  launch_level_solve(probs_dev, nprob, nblk, prm, st);
  // K3: W_m from x, Gram for step m+1
  int k = LVL_M;
  {
    int nb = proj_nblk(1 << (d - k), nprob);
    k_project<true><<<dim3(nb, nprob), NT, smem_project(), st>>>(probs_dev, k, nb, 1);
    count_launches(1);
    int src_is_a = 1;  // W_m lives in Wa
    int prev_nb = nb;
    ++k;
    // steps while W_{k-1} has more than FIN_COLS columns
    while ((1 << (d - k + 1)) > FIN_COLS) {
      launch_step_solve(probs_dev, nprob, k, prev_nb, prm, st);
      int nb2 = proj_nblk(1 << (d - k), nprob);
      k_project<false><<<dim3(nb2, nprob), NT, smem_project(), st>>>(probs_dev, k, nb2, src_is_a);
      count_launches(1);
      src_is_a ^= 1;
      prev_nb = nb2;
      ++k;
    }
    launch_finish(probs_dev, nprob, k, src_is_a, prm, st);
  }
  return cudaGetLastError();
}

}  // namespace qtt

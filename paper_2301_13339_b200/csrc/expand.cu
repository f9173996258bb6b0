// expand.cu — QTT-to-full expansion (Alg. 3 "Full", P:408-424;
// Step 4 of Alg. 2) on sm_100a, written straight into the caller's
// layout (1D, or row-major image for the interleaved / concatenated 2D QTT).
//
// y[i] = Re(C_1[i_1] ... C_d[i_d]).  The chain is split at m_e = 8:
//   L = full(cores 1..8)  (256 x r, complex)          k_expand_prep
//   R = full(cores 9..d)  (r x 2^{d-8}), formed per 32768-element super-chunk
//       from a suffix stack of the top cores and a 7-level tree of the mid
//       cores
//   y_tile = [Re L, -Im L] (256 x 2r) . [Re R; Im R] (2r x 128)
// on FP64 tensor cores (DMMA); the accumulator fragments of each 2048-index
// block (256 rows x 8 columns) go through a swizzled shared-memory block and
// leave as 512-byte rows of 16-byte streaming stores (a 64 x 32 rectangle of
// the image in the interleaved layout, 16 KB contiguous otherwise) — the pass
// is bound by HBM writes (tools/probe/store_pattern.cu: direct fragment
// stores 4.4 TB/s, staged 5.9-6.3 TB/s on the interleaved layout).
#include "qtt_kernels.h"

namespace qtt {

static constexpr int NT = 256;
static constexpr int ME = 8;        // bits of L

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
  // cores 2..ME staged in shared memory first (the products below would
  // otherwise wait on a dependent chain of L2 loads per term)
  cplx* cs = reinterpret_cast<cplx*>(smraw + 2 * 256 * RC * sizeof(cplx));
  __shared__ int rk[ME + 1];
  const int tid = threadIdx.x;
  if (tid <= ME) rk[tid] = pr.ranks[tid];
  for (int e = tid; e < (ME - 1) * 2 * RC * RC; e += blockDim.x) {
    const int m = e / (2 * RC * RC), o = e % (2 * RC * RC);
    cs[e] = pr.cores[(size_t)(m + 1) * SLOT + o];   // core m + 2
  }
  int r = pr.ranks[1];
  for (int e = tid; e < 2 * r; e += blockDim.x) {
    int i = e & 1, j = e >> 1;
    A[0][i + 2 * j] = pr.cores[i + 2 * j];     // core 1 is (1, 2, r): (0, i, j) at i + 2 j
  }
  __syncthreads();
  int cur = 0;
  for (int k = 2; k <= ME; ++k) {
    const cplx* c = cs + (size_t)(k - 2) * 2 * RC * RC;
    const int r0 = r, r1 = rk[k];
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
// A super-chunk is 2^(ME+MB) consecutive QTT indices: 256 rows (bits 1..8,
// L) x 128 columns (bits 9..15, the mid tree); the top bits (cores 16..d)
// are fixed per super-chunk and come from an incrementally updated suffix
// stack.  Requires d >= ME + MB = 15.
static constexpr int MB = 7;                 // mid bits
static constexpr int NCOL = 1 << MB;         // 128 R columns per super-chunk
static constexpr int TOP0 = ME + MB + 1;     // first top core (15)
static constexpr int RSLD = NCOL + 4;        // ld of Rs rows (columns + pad)

// R: rank capacity of the tensor (8 for the convolution output, Rhat <= 8;
// 16 otherwise): fragments, tree and stack are sized by it, so the R = 8
// variant keeps 3 CTAs per SM
// Output stage variant (A/B, profiles/r02r_expand_bulk_ab.json: the bulk
// copies lose, C4 1.10 ms against 0.59 ms, so the product build keeps the
// streaming stores; a ring of 3-6 stage buffers leaves one CTA per SM and
// takes 1.75 ms): with
// -DQTT_EXPAND_BULK the interleaved R <= 8 path leaves each 2048-index block
// as 32 rows of 512 bytes written by cp.async.bulk (shared -> global, one
// copy per lane of warp 0) instead of 16-byte streaming stores by every
// thread.  Stage row y sits at 640 y + 32 (y & 1) + 64 ((y >> 4) & 1) bytes:
// linear inside the row (the copy's source), and the fragment stores of a
// warp (lanes over x0, x1, y0, y4, x5) cover 16 distinct 8-byte bank pairs
// per half-warp.
#ifdef QTT_EXPAND_BULK
static constexpr bool EX_BULK = true;
#else
static constexpr bool EX_BULK = false;
#endif
__device__ __forceinline__ int stage_pos_bulk(int q) {
  const int x = (int)compact_even((uint64_t)q), y = (int)compact_even((uint64_t)q >> 1);
  return y * 80 + 4 * (y & 1) + 8 * ((y >> 4) & 1) + x;
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int R>
struct ExSmem {
  double Rs[2 * R * RSLD];    // [Re R; Im R] (KL x 128), row-major, ld RSLD
  cplx stack[MAXD + 2 - TOP0][R];   // stack[k - TOP0] = C_{k+1} ... C_d (size r_k), k >= TOP0 - 1
  cplx top0c[R <= 8 ? 2 * R * R : 1];  // core TOP0 (its bit flips every super-chunk), R <= 8
  cplx tree[2][NCOL * R + (EX_BULK && R <= 8 ? 256 : 0)];   // mid tree (R > 8); the 2 x 2048-double output stage
                              // (bulk-store rows: 32 x 640 bytes)
  // R <= 8: the 7 mid cores as three products computed once per CTA,
  // P_low[b9 b10 b11] = C_9 C_10 C_11, Q_a[b12 b13] = C_12 C_13 and
  // Q_b[b14 b15] = C_14 C_15 (column (b9..b15) of R = P_low Q_a Q_b s)
  cplx qa[R <= 8 ? 4 : 1][R * R];
  cplx qb[R <= 8 ? 4 : 1][R * R];
  cplx plow[R <= 8 ? R * R : 1][8];       // [i + R j][lb]: lanes of consecutive columns read consecutive lb
  cplx ut[R <= 8 ? 2 : 1][16 * R];
  int rk[MAXD + 1];           // ranks
};
static_assert(NCOL * 8 * sizeof(cplx) >= 2048 * sizeof(double), "stage fits a tree buffer");

// Stage position of block-local QTT index q = row + 256 col (bits 0..10).
// Interleaved: x = even bits (6), y = odd bits (5), row-major 32 x 64 with
// the 16-byte pairs swizzled, x' = x ^ (h << 1), h = y0 | y4 << 1 | x5 << 2,
// so the fragment stores (lanes spanning x0, y0, x1, y4, x5) hit 16 distinct
// bank pairs per half-warp; otherwise q ^ (((q >> 9) & 3) << 2).  Both keep
// the pairs (2m, 2m+1) adjacent for the 16-byte reads.
__device__ __forceinline__ int stage_pos(int q, bool il) {
  if (il) {
    const int x = (int)compact_even((uint64_t)q), y = (int)compact_even((uint64_t)q >> 1);
    const int h = (y & 1) | (((y >> 4) & 1) << 1) | (((x >> 5) & 1) << 2);
    return y * 64 + (x ^ (h << 1));
  }
  return q ^ (((q >> 9) & 3) << 2);
}

template <int R>
__global__ void __launch_bounds__(NT, R <= 8 ? 3 : 2) k_expand_main(const ExProb* probs, ExParams P, int per_cta) {
  const ExProb& pr = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  ExSmem<R>& S = *reinterpret_cast<ExSmem<R>*>(smraw);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int d = P.d;
  const uint64_t nsup = 1ull << (d - ME - MB);
  const uint64_t c0 = (uint64_t)blockIdx.x * per_cta;
  uint64_t c1 = c0 + per_cta;
  if (c1 > nsup) c1 = nsup;
  if (c0 >= c1) return;
  const int r8 = pr.ranks[ME];
  const int kl = (2 * r8 + 3) & ~3;
  const int ksteps = kl / 4;
  // A fragments: this warp's 4 m-blocks (rows 32 w .. 32 w + 31), all k-steps
  constexpr int KS = R / 2;            // k-steps of 4 covering 2 R
  double afr[4][KS];
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      int row = 32 * w + 8 * mb + (lane >> 2), col = 4 * ks + (lane & 3);
      afr[mb][ks] = (col < kl) ? pr.lsplit[row + 256 * col] : 0.0;
    }
  if (tid < R) S.stack[d - TOP0 + 1][tid] = cmk(tid == 0 ? 1.0 : 0.0, 0.0);   // empty product
  if constexpr (R <= 8) {
    if (d >= TOP0)
      for (int e = tid; e < 2 * R * R; e += NT) S.top0c[e] = pr.cores[(size_t)(TOP0 - 1) * SLOT + e];
  }
  for (int k = tid; k <= d; k += NT) S.rk[k] = pr.ranks[k];
  if constexpr (R <= 8) {
    // cores 9..15 (<= 7 x 2 R^2 complex) staged in a tree buffer first: the
    // products below then read shared memory instead of chains of L2 loads
    cplx* mc = S.tree[0];
    static_assert(7 * 2 * R * R <= NCOL * R, "mid cores fit a tree buffer");
    for (int e = tid; e < 7 * 2 * R * R; e += NT) {
      const int m = e / (2 * R * R), o = e % (2 * R * R);
      mc[e] = pr.cores[(size_t)(ME + m) * SLOT + o];   // core 9 + m
    }
    __syncthreads();
    auto mcore = [&](int k) -> const cplx* { return mc + (size_t)(k - ME - 1) * 2 * R * R; };
    // Q_a[ha] (r_11 x r_13) = C_12[b12] C_13[b13]; Q_b[hh] (r_13 x r_15) = C_14[b14] C_15[b15]
    for (int e = tid; e < 2 * 4 * R * R; e += NT) {
      const int which = e / (4 * R * R), o = e % (4 * R * R);
      const int h = o / (R * R), i = (o % (R * R)) % R, j = (o % (R * R)) / R;
      const int k0 = which == 0 ? 12 : 14;                    // first core of the pair
      const int ra = pr.ranks[k0 - 1], rm = pr.ranks[k0], rb = pr.ranks[k0 + 1];
      cplx acc = czero();
      if (i < ra && j < rb) {
        const cplx* c0 = mcore(k0);
        const cplx* c1 = mcore(k0 + 1);
        const int b0 = h & 1, b1 = h >> 1;
        for (int a = 0; a < rm; ++a) acc = cfma(c0[i + ra * b0 + 2 * ra * a], c1[a + rm * b1 + 2 * rm * j], acc);
      }
      (which == 0 ? S.qa : S.qb)[h][i + R * j] = acc;
    }
    // P_low[lb] (r_8 x r_11) = C_9[b9] C_10[b10] C_11[b11], lb = b9 + 2 b10 + 4 b11
    const int q8 = pr.ranks[8], q9 = pr.ranks[9], q10 = pr.ranks[10], q11 = pr.ranks[11];
    const cplx* c9 = mcore(9);
    const cplx* c10 = mcore(10);
    const cplx* c11 = mcore(11);
    for (int e = tid; e < 8 * q8 * q11; e += NT) {
      const int i = e % q8, j = (e / q8) % q11, lb = e / (q8 * q11);
      const int b0 = lb & 1, b1 = (lb >> 1) & 1, b2 = lb >> 2;
      cplx acc = czero();
      for (int b = 0; b < q10; ++b) {
        cplx t = czero();
        for (int a = 0; a < q9; ++a) t = cfma(c9[i + q8 * b0 + 2 * q8 * a], c10[a + q9 * b1 + 2 * q9 * b], t);
        acc = cfma(t, c11[b + q10 * b2 + 2 * q10 * j], acc);
      }
      S.plow[i + R * j][lb] = acc;
    }
    // Rs rows 2 r_8 .. kl-1 stay zero
    for (int e = tid; e < (kl - 2 * r8) * NCOL; e += NT) S.Rs[(2 * r8 + e / NCOL) * RSLD + e % NCOL] = 0.0;
  }
  const bool il = P.layout == LAYOUT_INTERLEAVED;
  const bool al16 = ((uintptr_t)pr.y & 15) == 0;   // else two 8-byte stores per pair
  const bool bulk = EX_BULK && R <= 8 && il && al16;
  int spos[4][2];
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int q = 32 * w + 8 * mb + (lane >> 2) + 256 * (2 * (lane & 3) + e);
      spos[mb][e] = bulk ? stage_pos_bulk(q) : stage_pos(q, il);
    }
  const uint64_t W = il ? (1ull << P.bx) : 0;
  uint64_t prev = ~0ull;
  for (uint64_t c = c0; c < c1; ++c) {
    // ---- suffix stack over the top cores TOP0..d for the bits of c
    int hi;
    if (prev == ~0ull) hi = d;
    else hi = TOP0 - 1 + (64 - __clzll((long long)(prev ^ c)));
    if (hi > d) hi = d;
    __syncthreads();
    if (w == 0) {
      for (int k = hi; k >= TOP0; --k) {
        const int r0 = S.rk[k - 1], r1 = S.rk[k];
        const int be = (int)((c >> (k - TOP0)) & 1);
        const cplx* core = (R <= 8 && k == TOP0) ? S.top0c : pr.cores + (size_t)(k - 1) * SLOT;
        if (lane < r0) {
          cplx s = czero();
          for (int j = 0; j < r1; ++j) s = cfma(core[lane + r0 * be + 2 * r0 * j], S.stack[k - TOP0 + 1][j], s);
          S.stack[k - TOP0][lane] = s;
        }
        __syncwarp();
      }
    }
    prev = c;
    if constexpr (R <= 8) {
      // ---- warp 0: v[hh] = Q_b[hh] s (s = C_16 .. C_d, size r_15), then
      //      u[hb] = Q_a[hb & 3] v[hb >> 2] (16 vectors of size r_11,
      //      hb = b12 + 2 b13 + 4 b14 + 8 b15); then all threads:
      //      R[:, col] = P_low[col & 7] u[col >> 3]
      if (w == 0) {
        const cplx* sv = S.stack[0];
        const int r11 = S.rk[ME + 3], r13 = S.rk[ME + 5], r15 = S.rk[ME + 7];
        if (lane < 4 * r13) {
          const int i = lane % r13, hh = lane / r13;
          cplx s0 = czero(), s1 = czero();
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            if (j < r15) s0 = cfma(S.qb[hh][i + R * j], sv[j], s0);
            if (j + 1 < r15) s1 = cfma(S.qb[hh][i + R * (j + 1)], sv[j + 1], s1);
          }
          S.ut[0][hh * R + i] = cadd(s0, s1);
        }
        __syncwarp();
        for (int e = lane; e < 16 * r11; e += 32) {
          const int i = e % r11, hb = e / r11;
          const cplx* vv = S.ut[0] + (hb >> 2) * R;
          const cplx* qa = S.qa[hb & 3];
          cplx s0 = czero(), s1 = czero();
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            if (j < r13) s0 = cfma(qa[i + R * j], vv[j], s0);
            if (j + 1 < r13) s1 = cfma(qa[i + R * (j + 1)], vv[j + 1], s1);
          }
          S.ut[1][hb * R + i] = cadd(s0, s1);
        }
      }
      __syncthreads();
      {
        const cplx* u = S.ut[1];
        const int r11 = S.rk[ME + 3];
        for (int e = tid; e < NCOL * r8; e += NT) {
          const int col = e % NCOL, i = e / NCOL;
          const int lb = col & 7;
          const cplx* uv = u + (col >> 3) * R;
          cplx s0 = czero(), s1 = czero();
#pragma unroll
          for (int j = 0; j < R; j += 2) {
            if (j < r11) s0 = cfma(S.plow[i + R * j][lb], uv[j], s0);
            if (j + 1 < r11) s1 = cfma(S.plow[i + R * (j + 1)][lb], uv[j + 1], s1);
          }
          const cplx v = cadd(s0, s1);
          S.Rs[i * RSLD + col] = v.x;
          S.Rs[(r8 + i) * RSLD + col] = v.y;
        }
      }
      __syncthreads();
    } else {
    __syncthreads();
    // ---- mid tree over cores ME+MB .. ME+1 -> 64 vectors of size r_8
    const cplx* vin = S.stack[0];
    int nv = 1, cur = 0;
#pragma unroll 1
    for (int k = ME + MB; k >= ME + 1; --k) {
      const int r0 = S.rk[k - 1], r1 = S.rk[k];
      const cplx* core = pr.cores + (size_t)(k - 1) * SLOT;
      cplx* vout = S.tree[cur];
      for (int e = tid; e < 2 * nv * r0; e += NT) {
        const int i = e % r0, vv = e / r0;
        const int be = vv & 1, src = vv >> 1;
        cplx s0 = czero(), s1 = czero();
#pragma unroll
        for (int j = 0; j < R; j += 2) {
          if (j < r1) s0 = cfma(core[i + r0 * be + 2 * r0 * j], vin[src * R + j], s0);
          if (j + 1 < r1) s1 = cfma(core[i + r0 * be + 2 * r0 * (j + 1)], vin[src * R + j + 1], s1);
        }
        vout[vv * R + i] = cadd(s0, s1);
      }
      __syncthreads();
      vin = vout;
      cur ^= 1;
      nv *= 2;
    }
    // vector index vv: bits (b_{ME+MB} .. b_{ME+1}), b_{ME+1} the LSB
    for (int e = tid; e < kl * NCOL; e += NT) {
      const int row = e / NCOL, col = e % NCOL;
      double v = 0.0;
      if (row < r8) v = vin[col * R + row].x;
      else if (row < 2 * r8) v = vin[col * R + row - r8].y;
      S.Rs[row * RSLD + col] = v;
    }
    __syncthreads();
    }
    // ---- GEMM (256 x 128) in 16 blocks of 8 columns (2048 QTT indices);
    //      each block is staged in a tree buffer (double-buffered: one barrier
    //      per block) and written as 512-byte rows
    const uint64_t qbase = c << (ME + MB);
#pragma unroll 1
    for (int nb = 0; nb < NCOL / 8; ++nb) {
      double* stg = reinterpret_cast<double*>(S.tree[nb & 1]);
      double acc[4][2];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) acc[mb][0] = acc[mb][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        if (ks < ksteps) {
          const double bb = S.Rs[(4 * ks + (lane & 3)) * RSLD + 8 * nb + (lane >> 2)];
#pragma unroll
          for (int mb = 0; mb < 4; ++mb) dmma884(acc[mb][0], acc[mb][1], afr[mb][ks], bb);
        }
      }
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int e = 0; e < 2; ++e) stg[spos[mb][e]] = acc[mb][e];
      if (bulk) {
        // the stage is read by the async proxy: order the fragment stores
        // before it; warp 0 first makes sure the copies of the block before
        // (the other buffer, rewritten after this barrier) have read it
        fence_async_smem();
        if (w == 0) bulk_wait_read0();
        __syncthreads();
        if (w == 0) {
          double* yb = pr.y + qtt_offset(qbase + ((uint64_t)nb << 11), P.layout, P.bx);
          bulk_s2g(yb + (uint64_t)lane * W, stg + lane * 80 + 4 * (lane & 1) + 8 * ((lane >> 4) & 1), 512u);
          bulk_commit();
        }
        continue;
      }
      __syncthreads();
      double* yb = pr.y + qtt_offset(qbase + ((uint64_t)nb << 11), P.layout, P.bx);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int pi = tid + NT * t;      // 16-byte pair in storage order
        if (il) {
          const int yy = pi >> 5, x = 2 * (pi & 31);
          const int h = (yy & 1) | (((yy >> 4) & 1) << 1) | (((x >> 5) & 1) << 2);
          const double2 v = *reinterpret_cast<const double2*>(stg + yy * 64 + (x ^ (h << 1)));
          double* dst = yb + yy * W + x;
          if (al16) __stcs(reinterpret_cast<double2*>(dst), v);
          else { __stcs(dst, v.x); __stcs(dst + 1, v.y); }
        } else {
          const int q = 2 * pi;
          const double2 v = *reinterpret_cast<const double2*>(stg + (q ^ (((q >> 9) & 3) << 2)));
          if (al16) __stcs(reinterpret_cast<double2*>(yb + q), v);
          else { __stcs(yb + q, v.x); __stcs(yb + q + 1, v.y); }
        }
      }
    }
  }
  // the stage must outlive the copies that read it
  if (bulk && w == 0) bulk_wait_read0();
}

// ------------------------------------------------------- shard tail fold
// One CTA per shard: v = C_{d-l+1}[b_1] ... C_d[b_l] (b = bits of `shard`,
// LSB at position d-l+1), then out = (C_1 .. C_{d-l-1}, C_{d-l} v).
__global__ void k_fold_tail(const FoldProb* probs, int d, int l) {
  const FoldProb& pr = probs[blockIdx.x];
  __shared__ cplx v[2][RC];
  const int tid = threadIdx.x, dl = d - l;
  if (tid < RC) v[0][tid] = cmk(tid == 0 ? 1.0 : 0.0, 0.0);
  __syncthreads();
  int cur = 0;
  for (int k = d; k > dl; --k) {
    const int r0 = pr.ranks[k - 1], r1 = pr.ranks[k];
    const int be = (pr.shard >> (k - dl - 1)) & 1;
    const cplx* c = pr.cores + (size_t)(k - 1) * SLOT;
    if (tid < r0) {
      cplx s = czero();
      for (int j = 0; j < r1; ++j) s = cfma(c[tid + r0 * be + 2 * r0 * j], v[cur][j], s);
      v[cur ^ 1][tid] = s;
    }
    __syncthreads();
    cur ^= 1;
  }
  // core dl folded with v: (r0, 2, r1) -> (r0, 2, 1)
  {
    const int r0 = pr.ranks[dl - 1], r1 = pr.ranks[dl];
    const cplx* c = pr.cores + (size_t)(dl - 1) * SLOT;
    cplx* o = pr.out_cores + (size_t)(dl - 1) * SLOT;
    for (int e = tid; e < 2 * r0; e += blockDim.x) {
      cplx s = czero();
      for (int j = 0; j < r1; ++j) s = cfma(c[e + 2 * r0 * j], v[cur][j], s);
      o[e] = s;
    }
  }
  for (int k = 1; k < dl; ++k) {
    const int n = 2 * pr.ranks[k - 1] * pr.ranks[k];
    const cplx* c = pr.cores + (size_t)(k - 1) * SLOT;
    cplx* o = pr.out_cores + (size_t)(k - 1) * SLOT;
    for (int e = tid; e < n; e += blockDim.x) o[e] = c[e];
  }
  for (int k = tid; k < 64; k += blockDim.x) pr.out_ranks[k] = k < dl ? pr.ranks[k] : (k == dl ? 1 : 0);
}

cudaError_t launch_fold_tail(const FoldProb* probs_dev, int nprob, int d, int l, cudaStream_t st) {
  k_fold_tail<<<nprob, 256, 0, st>>>(probs_dev, d, l);
  count_launches(1);
  return cudaGetLastError();
}

static constexpr size_t PREP_SMEM = 2 * 256 * RC * sizeof(cplx) + (ME - 1) * 2 * RC * RC * sizeof(cplx);

cudaError_t setup_expand_kernels() {
  cudaError_t e = cudaFuncSetAttribute(k_expand_main<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(ExSmem<8>));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_expand_main<RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ExSmem<RC>));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_expand_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PREP_SMEM);
}

cudaError_t launch_expand(const ExProb* probs_dev, int nprob, const ExParams& prm, cudaStream_t st) {
  const int d = prm.d;
  if (d < ME + MB) {
    int nb = (int)(((1ull << d) + 255) / 256);
    k_expand_small<<<dim3(nb, nprob), 256, 0, st>>>(probs_dev, prm);
    count_launches(1);
    return cudaGetLastError();
  }
  k_expand_prep<<<nprob, 256, PREP_SMEM, st>>>(probs_dev, prm);
  const uint64_t nsup = 1ull << (d - ME - MB);
  // aim for a full wave (2 or 3 CTAs per SM) over all problems, contiguous
  // ranges per CTA
  const bool r8 = prm.rcap <= 8;
  const int waves = (r8 ? 3 : 2) * sm_count();
  uint64_t target = (uint64_t)(waves + nprob - 1) / nprob;
  if (target < 1) target = 1;
  int per = (int)((nsup + target - 1) / target);
  int nb = (int)((nsup + per - 1) / per);
  prof_pass(PASS_EXPAND, 0, st);
  if (r8) k_expand_main<8><<<dim3(nb, nprob), NT, sizeof(ExSmem<8>), st>>>(probs_dev, prm, per);
  else k_expand_main<RC><<<dim3(nb, nprob), NT, sizeof(ExSmem<RC>), st>>>(probs_dev, prm, per);
  prof_pass(PASS_EXPAND, 1, st);
  count_launches(2);
  return cudaGetLastError();
}

}  // namespace qtt

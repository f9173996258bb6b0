// hround.cu — core-wise Hadamard product (Alg. 2 Step 3; ranks
// multiply) fused with TT-rounding ROUND_FULL = ROUND_LOCAL(1)
// (readings Q20/Q21) on sm_100a.
//
// Z_k[(a,a'), al, (b,b')] = F_k[a, al, b] G_k[a', al, b'] is never
// materialised.  The right Gram chain GR_{c-1} = sum_al Z_c[al] GR_c
// Z_c[al]^H uses the Kronecker structure (G-side then F-side contractions,
// O(r^5) instead of O(r^6)), and the left-to-right truncation sweep forms
// the pushed core S * Z_{c+1} in two Kronecker steps.  Truncation of cut c
// is the eigendecomposition of K_c = M_c GR_c M_c^H (2 r' x 2 r', r' <= Rhat).
#include "qtt_kernels.h"

namespace qtt {

// optional sweep phase timing (-DQTT_HR_TIMING): cycles of CTA 0 per phase,
// written to the tail of the GR scratch (diagnostic builds only)
#ifdef QTT_HR_TIMING
#define HT_DECL long long ht_t0 = clock64(), ht_acc[6] = {0, 0, 0, 0, 0, 0};
#define HT_MARK(k) { long long _t = clock64(); ht_acc[k] += _t - ht_t0; ht_t0 = _t; }
#define HT_DUMP(ptr) if (threadIdx.x == 0 && blockIdx.x == 0) printf("hround sweep cycles: loadGR %lld T+K %lld eigval %lld rank/vec/core/Sm %lld push %lld loop %lld\n", ht_acc[0], ht_acc[1], ht_acc[2], ht_acc[3], ht_acc[4], ht_acc[5]);
#else
#define HT_DECL
#define HT_MARK(k)
#define HT_DUMP(ptr)
#endif

static constexpr int NT = 512;   // one CTA per SM (190 KB smem): more warps to hide the product latencies
static constexpr int RH = RH_MAX;       // 8
static constexpr int RZ = RH * RH;      // 64
static constexpr int CZ = 2 * RH * RH;  // compact core of F or G

struct HrSmem {
  cplx Y[RZ * RZ];
  cplx Y2[RZ * RZ];
  cplx F[CZ];
  cplx Gc[CZ];
  cplx Eb[RH * 2 * RZ];
  cplx Sm[RH * RZ];
  EigSmem<2 * RH> E;
  int rf[MAXD + 1], rg[MAXD + 1], r[MAXD + 1], rb[MAXD + 1];
  int rk;
  double tau2;
  double mdefer[4];   // deferred T2 record of the last RANK (margins_flush)
};

__device__ void load_core(cplx* dst, const cplx* src, int n) {
  for (int e = threadIdx.x; e < n; e += NT) dst[e] = src[e];
}

__global__ void __launch_bounds__(NT) k_hadamard_round(const HrProb* probs, HrParams P) {
  const HrProb& pr = probs[blockIdx.x];
  extern __shared__ __align__(16) unsigned char smraw[];
  HrSmem& S = *reinterpret_cast<HrSmem*>(smraw);
  constexpr int LD = EigSmem<2 * RH>::LD;
  const int tid = threadIdx.x;
  const int d = P.d;
  for (int q = tid; q <= d; q += NT) { S.rf[q] = pr.f_ranks[q]; S.rg[q] = pr.g_ranks[q]; }
  if (tid == 0) S.mdefer[1] = 0.0;
  __syncthreads();
  // ---------------- right Gram chain (unless launch_hr_gr_chain computed it
  //                  with the mode products spread over the GPU)
  if (!P.gr_ready) {
  {
    // GR_{d-1} = sum_al z z^H, z[(a,a')] = F_d[a,al] G_d[a',al]
    const int af = S.rf[d - 1], ag = S.rg[d - 1], rz = af * ag;
    load_core(S.F, pr.f_cores + (size_t)(d - 1) * SLOT, af * 2);
    load_core(S.Gc, pr.g_cores + (size_t)(d - 1) * SLOT, ag * 2);
    __syncthreads();
    for (int e = tid; e < rz * rz; e += NT) {
      int i = e % rz, j = e / rz;
      int ia = i / ag, ib = i % ag, ja = j / ag, jb = j % ag;
      cplx s = czero();
      for (int al = 0; al < 2; ++al) {
        cplx zi = cmul(S.F[ia + af * al], S.Gc[ib + ag * al]);
        cplx zj = cmul(S.F[ja + af * al], S.Gc[jb + ag * al]);
        s = cfma_bc(zi, zj, s);
      }
      pr.gr[(size_t)(d - 1) * GR_HR + e] = s;
    }
    __syncthreads();
  }
  for (int c = d - 1; c >= 2; --c) {
    // X = GR_c: rows (b, b') = b*gb + b', b < fb = rf[c], b' < gb = rg[c]
    const int fa = S.rf[c - 1], fb = S.rf[c], ga = S.rg[c - 1], gb = S.rg[c];
    load_core(S.F, pr.f_cores + (size_t)(c - 1) * SLOT, fa * 2 * fb);
    load_core(S.Gc, pr.g_cores + (size_t)(c - 1) * SLOT, ga * 2 * gb);
    const cplx* X = pr.gr + (size_t)c * GR_HR;
    const int rzx = fb * gb;          // dim of X
    const int rzo = fa * ga;          // dim of output
    cplx acc[(RZ * RZ) / NT];
#pragma unroll
    for (int i = 0; i < (RZ * RZ) / NT; ++i) acc[i] = czero();
    __syncthreads();
    for (int al = 0; al < 2; ++al) {
      // A1: YA[(b,a'),(c,c')] = sum_b' G[a',al,b'] X[(b,b'),(c,c')]  -> Y2, rows fb*ga, cols rzx
      const int ra = fb * ga;
      for (int e = tid; e < ra * rzx; e += NT) {
        int i = e % ra, j = e / ra;
        int b = i / ga, ap_ = i % ga;
        cplx s = czero();
        for (int bp = 0; bp < gb; ++bp) s = cfma(S.Gc[ap_ + ga * al + 2 * ga * bp], X[(b * gb + bp) + rzx * j], s);
        S.Y2[i + ra * j] = s;
      }
      __syncthreads();
      // A2: Y[(b,a'),(c,e')] = sum_c' YA[(b,a'),(c,c')] conj(G[e',al,c'])  -> Y, ra x ra
      for (int e = tid; e < ra * ra; e += NT) {
        int i = e % ra, j = e / ra;
        int cc = j / ga, ep = j % ga;
        cplx s = czero();
        for (int cp = 0; cp < gb; ++cp)
          s = cfma_bc(S.Y2[i + ra * (cc * gb + cp)], S.Gc[ep + ga * al + 2 * ga * cp], s);
        S.Y[i + ra * j] = s;
      }
      __syncthreads();
      // B1: Y2[(a,a'),(c,e')] = sum_b F[a,al,b] Y[(b,a'),(c,e')]  -> rows rzo, cols ra
      for (int e = tid; e < rzo * ra; e += NT) {
        int i = e % rzo, j = e / rzo;
        int aa = i / ga, ap_ = i % ga;
        cplx s = czero();
        for (int b = 0; b < fb; ++b) s = cfma(S.F[aa + fa * al + 2 * fa * b], S.Y[(b * ga + ap_) + ra * j], s);
        S.Y2[i + rzo * j] = s;
      }
      __syncthreads();
      // B2: out[(a,a'),(e,e')] += sum_c Y2[(a,a'),(c,e')] conj(F[e,al,c])
#pragma unroll
      for (int k = 0; k < (RZ * RZ) / NT; ++k) {
        int e = tid + NT * k;
        if (e < rzo * rzo) {
          int i = e % rzo, j = e / rzo;
          int ee = j / ga, ep = j % ga;
          cplx s = acc[k];
          for (int cc = 0; cc < fb; ++cc)
            s = cfma_bc(S.Y2[i + rzo * (cc * ga + ep)], S.F[ee + fa * al + 2 * fa * cc], s);
          acc[k] = s;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < (RZ * RZ) / NT; ++k) {
      int e = tid + NT * k;
      if (e < rzo * rzo) pr.gr[(size_t)(c - 1) * GR_HR + e] = acc[k];
    }
    __syncthreads();
  }
  }
  // ---------------- LQ rank bounds
  if (tid == 0) {
    S.rb[d] = 1;
    for (int c = d - 1; c >= 1; --c) {
      int v = S.rf[c] * S.rg[c], w = 2 * S.rb[c + 1];
      S.rb[c] = v < w ? v : w;
    }
    S.r[0] = 1;
  }
  // ---------------- E = Z_1 (1 x 2 x rz_1)
  {
    const int fb = S.rf[1], gb = S.rg[1];
    load_core(S.F, pr.f_cores, 2 * fb);
    load_core(S.Gc, pr.g_cores, 2 * gb);
    __syncthreads();
    for (int e = tid; e < 2 * fb * gb; e += NT) {
      int al = e & 1, j = e >> 1;
      int b = j / gb, bp = j % gb;
      S.Eb[e] = cmul(S.F[al + 2 * b], S.Gc[al + 2 * bp]);
    }
    __syncthreads();
  }
  int ap = 1;
  HT_DECL
  for (int c = 1; c <= d - 1; ++c) {
    const int rows = 2 * ap, rz = S.rf[c] * S.rg[c];
    HT_MARK(5)
    for (int e = tid; e < rz * rz; e += NT) S.Y[e] = pr.gr[(size_t)c * GR_HR + e];
    __syncthreads();
    HT_MARK(0)
    // T = E GR (rows x rz, k = rz <= 64) and K = T E^H (rows x rows, k = rz)
    // on DMMA tiles (16 warps: one 8 x 8 tile of T each; the 4 tiles of K
    // with their k-chunks split over the warps and summed in a fixed order)
    cgemm_dmma_sg<NT / 32>(GemmArgs{S.Eb, S.Y, S.Y2, rows, rz, rz, 1, rows, 1, rz, 1, rows, 0, 0});
    __syncthreads();
    {
      // K: tile t = w & 3 (2 x 2 tiles of 8 at rows <= 16), k-split ks = w >> 2
      const int lane = tid & 31, wq = tid >> 5, t = wq & 3, ks = wq >> 2;
      const int ar = lane >> 2, ac = lane & 3, ti = t & 1, tj = t >> 1;
      double r0 = 0.0, r1 = 0.0, i0 = 0.0, i1 = 0.0;
      const int nk = (rz + 3) >> 2;
      for (int kc = ks; kc < nk; kc += 4) {
        const int k = 4 * kc + ac, ri = 8 * ti + ar, cj = 8 * tj + ar;
        const cplx a = (ri < rows && k < rz) ? S.Y2[ri + rows * k] : czero();
        const cplx b = (k < rz && cj < rows) ? cconj(S.Eb[cj + rows * k]) : czero();
        dmma884(r0, r1, a.x, b.x);
        dmma884(r0, r1, -a.y, b.y);
        dmma884(i0, i1, a.x, b.y);
        dmma884(i0, i1, a.y, b.x);
      }
      cplx* part = S.Y;    // 16 x 64 partial tiles (GR is consumed by T)
      part[wq * 64 + ar * 8 + 2 * ac] = cmk(r0, i0);
      part[wq * 64 + ar * 8 + 2 * ac + 1] = cmk(r1, i1);
      __syncthreads();
      if (tid < 256) {
        const int tt = tid >> 6, pos = tid & 63;
        const int i = 8 * (tt & 1) + (pos >> 3), j = 8 * (tt >> 1) + (pos & 7);
        cplx v = part[tt * 64 + pos];
#pragma unroll
        for (int q = 1; q < 4; ++q) v = cadd(v, part[(tt + 4 * q) * 64 + pos]);
        if (i < rows && j < rows) S.E.A[0][i + LD * j] = v;
      }
    }
    __syncthreads();
    if (c == 1) {
      double tr = 0.0;
      if (tid < rows) tr = S.E.A[0][tid + LD * tid].x;
      tr = block_sum<NT>(tr, S.E.red);
      if (tid == 0) S.tau2 = P.eps * P.eps * tr / (double)(d - 1);
      __syncthreads();
    }
    HT_MARK(1)
    eig_values<2 * RH, NT>(S.E, rows);
    HT_MARK(2)
    if (tid < 32) {
      const int mp = rows < S.rb[c] ? rows : S.rb[c];
      const int r = rank_choose_warp(S.E.lam, mp, S.tau2, P.rmax, P.ctol, P.rule, P.delta, P.status, S.mdefer);
      if (tid == 0) S.rk = r;
    }
    __syncthreads();
    auto flush = [&] { if ((tid & 31) == 0) margins_flush(S.mdefer, P.status); };
    const cplx* U = eig_vectors_spec<2 * RH, NT>(S.E, rows, S.rk, nullptr, flush, P.status);
    const int rk = S.rk;
    cplx* oc = pr.out_cores + (size_t)(c - 1) * SLOT;
    for (int e = tid; e < rows * rk; e += NT) {
      int i = e % rows, r = e / rows;
      oc[i + rows * r] = U[i + LD * r];
    }
    // Sm = U_r^H E (rk x rz) on DMMA tiles
    cgemm_dmma_sg<NT / 32>(GemmArgs{U, S.Eb, S.Sm, rk, rz, rows, LD, 1, 1, rows, 1, rk, 1, 0});
    HT_MARK(3)
    // next core's F and G
    const int q = c + 1;
    const int fa = S.rf[q - 1], fb = S.rf[q], ga = S.rg[q - 1], gb = S.rg[q];
    load_core(S.F, pr.f_cores + (size_t)(q - 1) * SLOT, fa * 2 * fb);
    load_core(S.Gc, pr.g_cores + (size_t)(q - 1) * SLOT, ga * 2 * gb);
    if (tid == 0) S.r[c] = rk;
    __syncthreads();
    // H[r, b, al, e'] = sum_b' Sm[r, (b,b')] G[b', al, e']   (stored in Y2)
    const int nh = rk * fa * 2 * gb;
    for (int e = tid; e < nh; e += NT) {
      int r = e % rk, t1 = e / rk;
      int b = t1 % fa, t2 = t1 / fa;
      int al = t2 & 1, ep = t2 >> 1;
      cplx s = czero();
      for (int bp = 0; bp < ga; ++bp) s = cfma(S.Sm[r + rk * (b * ga + bp)], S.Gc[bp + ga * al + 2 * ga * ep], s);
      S.Y2[e] = s;
    }
    __syncthreads();
    // E[r, al, (e,e')] = sum_b H[r,b,al,e'] F[b,al,e]
    for (int e = tid; e < rk * 2 * fb * gb; e += NT) {
      int r = e % rk, al = (e / rk) & 1, j = e / (2 * rk);
      int ee = j / gb, ep = j % gb;
      cplx s = czero();
      for (int b = 0; b < fa; ++b)
        s = cfma(S.Y2[r + rk * (b + fa * (al + 2 * ep))], S.F[b + fa * al + 2 * fa * ee], s);
      S.Eb[e] = s;
    }
    __syncthreads();
    ap = rk;
    HT_MARK(4)
  }
  HT_DUMP(pr.gr + (size_t)MAXD * GR_HR - 8)
  cplx* oc = pr.out_cores + (size_t)(d - 1) * SLOT;
  for (int e = tid; e < 2 * ap; e += NT) oc[e] = S.Eb[e];
  for (int q = tid; q <= d; q += NT) pr.out_ranks[q] = (q == 0 || q == d) ? 1 : S.r[q];
}

cudaError_t setup_hr_kernels() {
  return cudaFuncSetAttribute(k_hadamard_round, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(HrSmem));
}

cudaError_t launch_hadamard_round(const HrProb* probs_dev, int nprob, const HrParams& prm, cudaStream_t st) {
  k_hadamard_round<<<nprob, NT, sizeof(HrSmem), st>>>(probs_dev, prm);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace qtt

// hround_big.cu — Hadamard product + ROUND_FULL (Alg. 2 Step 3, P:395;
// reading Q20) for Rhat up to 16, i.e. Kronecker ranks
// rz = rf rg <= 256 (the paper's cap Rhat_max = 15).
//
// Same mathematics as hround.cu (the rounding is evaluated without the LQ
// sweep: right Gram matrices GR_c of Z = F (.) G built right to left, then
// truncations K_c = E_c GR_c E_c^H left to right), but the 256 x 256 Grams do
// not fit one CTA: every product is its own multi-CTA launch over global
// (L2-resident) buffers, the eigensolve of a cut runs in one CTA.
//   right Gram chain, per core c (d-1 .. 2), per slice al:
//     A1  T1[(b,a'),(c,c')] = sum_b' G[a',al,b'] GR_c[(b,b'),(c,c')]
//     A2  T2[(b,a'),(c,e')] = sum_c' T1[(b,a'),(c,c')] conj(G[e',al,c'])
//     B1  T3[(a,a'),(c,e')] = sum_b F[a,al,b] T2[(b,a'),(c,e')]
//     B2  GR_{c-1}[(a,a'),(e,e')] = sum_al sum_c T3[(a,a'),(c,e')] conj(F[e,al,c])
//   sweep, per cut c (1 .. d-1):
//     T = E GR_c, K = T E^H, eigenpairs, RANK, core c = U_r, Sm = U_r^H E,
//     H = Sm x G_{c+1}, E <- H x F_{c+1}.
#include <cooperative_groups.h>

#include "qtt_kernels.h"

namespace qtt {

static constexpr int NT = 256;
static constexpr int RB = RH_BIG;          // 16
static constexpr int RZB = RB * RB;        // 256
static constexpr int RWB = 2 * RB;         // rows of a cut <= 32

__device__ __forceinline__ const cplx* fcore(const HrBigProb& p, int q) { return p.f_cores + (size_t)(q - 1) * SLOT; }
__device__ __forceinline__ const cplx* gcore(const HrBigProb& p, int q) { return p.g_cores + (size_t)(q - 1) * SLOT; }

// ------------------------------------------------------ right Gram chain
// gs: complex entries per GR slot and per mode-product slice (RZB^2 for the
// multi-CTA rounding, GR_HR when the chain feeds the one-CTA sweep)
__global__ void k_hrb_gr_last(const HrBigProb* probs, int d, int gs) {
  const HrBigProb& p = probs[blockIdx.y];
  const int af = p.f_ranks[d - 1], ag = p.g_ranks[d - 1], rz = af * ag;
  const int e = blockIdx.x * NT + threadIdx.x;
  if (e >= rz * rz) return;
  const int i = e % rz, j = e / rz;
  const int ia = i / ag, ib = i % ag, ja = j / ag, jb = j % ag;
  const cplx* F = fcore(p, d);
  const cplx* G = gcore(p, d);
  cplx s = czero();
  for (int al = 0; al < 2; ++al) {
    const cplx zi = cmul(F[ia + af * al], G[ib + ag * al]);
    const cplx zj = cmul(F[ja + af * al], G[jb + ag * al]);
    s = cfma_bc(zi, zj, s);
  }
  p.gr[(size_t)(d - 1) * gs + e] = s;
}

// stage 0..3 = A1, A2, B1, B2 of core c (1-based), grid (RZB*RZB/NT, 2 slices, nprob)
__global__ void k_hrb_gr_step(const HrBigProb* probs, int c, int stage, int gs) {
  const HrBigProb& p = probs[blockIdx.z];
  const int fa = p.f_ranks[c - 1], fb = p.f_ranks[c], ga = p.g_ranks[c - 1], gb = p.g_ranks[c];
  const int rzx = fb * gb, rzo = fa * ga, ra = fb * ga;
  const int al = blockIdx.y;
  const int e = blockIdx.x * NT + threadIdx.x;
  const cplx* F = fcore(p, c);
  const cplx* G = gcore(p, c);
  cplx* T1 = p.t1 + (size_t)al * gs;
  cplx* T2 = p.t2 + (size_t)al * gs;
  cplx* T3 = p.t3 + (size_t)al * gs;
  if (stage == 0) {
    if (e >= ra * rzx) return;
    const int i = e % ra, j = e / ra;
    const int b = i / ga, ap = i % ga;
    const cplx* X = p.gr + (size_t)c * gs + (size_t)(b * gb) + (size_t)rzx * j;
    cplx s = czero();
    for (int bp = 0; bp < gb; ++bp) s = cfma(G[ap + ga * al + 2 * ga * bp], X[bp], s);
    T1[i + ra * j] = s;
  } else if (stage == 1) {
    if (e >= ra * ra) return;
    const int i = e % ra, j = e / ra;
    const int cc = j / ga, ep = j % ga;
    cplx s = czero();
    for (int cp = 0; cp < gb; ++cp)
      s = cfma_bc(T1[i + ra * (cc * gb + cp)], G[ep + ga * al + 2 * ga * cp], s);
    T2[i + ra * j] = s;
  } else if (stage == 2) {
    if (e >= rzo * ra) return;
    const int i = e % rzo, j = e / rzo;
    const int aa = i / ga, ap = i % ga;
    cplx s = czero();
    for (int b = 0; b < fb; ++b) s = cfma(F[aa + fa * al + 2 * fa * b], T2[(b * ga + ap) + ra * j], s);
    T3[i + rzo * j] = s;
  } else {
    if (al != 0 || e >= rzo * rzo) return;
    const int i = e % rzo, j = e / rzo;
    const int ee = j / ga, ep = j % ga;
    cplx s = czero();
    for (int a2 = 0; a2 < 2; ++a2) {
      const cplx* T3a = p.t3 + (size_t)a2 * gs;
      for (int cc = 0; cc < fb; ++cc)
        s = cfma_bc(T3a[i + rzo * (cc * ga + ep)], F[ee + fa * a2 + 2 * fa * cc], s);
    }
    p.gr[(size_t)(c - 1) * gs + i + rzo * j] = s;
  }
}

// ------------------------------------------------------------- sweep
// state: st[0] = ap (left rank of the current E), st[1] = rk, st[2 + q] = r_q,
// st[40 + q] = LQ rank bound rb_q (q <= d)
__global__ void k_hrb_init(const HrBigProb* probs, int d) {
  const HrBigProb& p = probs[blockIdx.x];
  const int tid = threadIdx.x;
  const int fb = p.f_ranks[1], gb = p.g_ranks[1];
  for (int e = tid; e < 2 * fb * gb; e += NT) {
    const int al = e & 1, j = e >> 1, b = j / gb, bp = j % gb;
    p.e[e] = cmul(p.f_cores[al + 2 * b], p.g_cores[al + 2 * bp]);
  }
  if (tid == 0) {
    p.st[0] = 1;
    p.st[2] = 1;
    p.st[40 + d] = 1;
    for (int c = d - 1; c >= 1; --c) {
      const int v = p.f_ranks[c] * p.g_ranks[c], w = 2 * p.st[40 + c + 1];
      p.st[40 + c] = v < w ? v : w;
    }
  }
}

// T = E GR_c (rows x rz), grid (RWB*RZB/NT, nprob)
__global__ void k_hrb_T(const HrBigProb* probs, int c) {
  const HrBigProb& p = probs[blockIdx.y];
  const int rows = 2 * p.st[0], rz = p.f_ranks[c] * p.g_ranks[c];
  const int e = blockIdx.x * NT + threadIdx.x;
  if (e >= rows * rz) return;
  const int i = e % rows, j = e / rows;
  const cplx* GR = p.gr + (size_t)c * RZB * RZB + (size_t)rz * j;
  cplx s0 = czero(), s1 = czero();
  int l = 0;
  for (; l + 1 < rz; l += 2) {
    s0 = cfma(p.e[i + rows * l], GR[l], s0);
    s1 = cfma(p.e[i + rows * (l + 1)], GR[l + 1], s1);
  }
  if (l < rz) s0 = cfma(p.e[i + rows * l], GR[l], s0);
  p.tb[e] = cadd(s0, s1);
}

struct HrbSolveSmem {
  EigSmem<RWB> E;
  double tau2;
  int rk;
};

// K = T E^H, eigenpairs, RANK, core c, Sm = U_r^H E.  One CTA per problem.
__global__ void __launch_bounds__(NT, 1) k_hrb_solve(const HrBigProb* probs, int c, int d, HrParams P) {
  const HrBigProb& p = probs[blockIdx.x];
  extern __shared__ __align__(16) unsigned char smraw[];
  HrbSolveSmem& S = *reinterpret_cast<HrbSolveSmem*>(smraw);
  constexpr int LD = EigSmem<RWB>::LD;
  const int tid = threadIdx.x;
  const int ap = p.st[0], rows = 2 * ap, rz = p.f_ranks[c] * p.g_ranks[c];
  for (int e = tid; e < rows * rows; e += NT) {
    const int i = e % rows, j = e / rows;
    cplx s0 = czero(), s1 = czero();
    int l = 0;
    for (; l + 1 < rz; l += 2) {
      s0 = cfma_bc(p.tb[i + rows * l], p.e[j + rows * l], s0);
      s1 = cfma_bc(p.tb[i + rows * (l + 1)], p.e[j + rows * (l + 1)], s1);
    }
    if (l < rz) s0 = cfma_bc(p.tb[i + rows * l], p.e[j + rows * l], s0);
    S.E.A[0][i + LD * j] = cadd(s0, s1);
  }
  __syncthreads();
  if (c == 1) {
    double tr = 0.0;
    if (tid < rows) tr = S.E.A[0][tid + LD * tid].x;
    tr = block_sum<NT>(tr, S.E.red);
    if (tid == 0) *p.tau2 = P.eps * P.eps * tr / (double)(d - 1);
    __syncthreads();
  }
  eig_values<RWB, NT>(S.E, rows);
  if (tid == 0) {
    const int rb = p.st[40 + c];
    const int mp = rows < rb ? rows : rb;
    S.rk = rank_choose(S.E.lam, mp, *p.tau2, P.rmax, P.ctol, P.rule, P.delta, P.status);
  }
  __syncthreads();
  const int rk = S.rk;
  const cplx* U = eig_vectors<RWB, NT>(S.E, rows, rk, P.status);
  cplx* oc = p.out_cores + (size_t)(c - 1) * SLOT;
  for (int e = tid; e < rows * rk; e += NT) {
    const int i = e % rows, r = e / rows;
    oc[i + rows * r] = U[i + LD * r];
  }
  for (int e = tid; e < rk * rz; e += NT) {
    const int r = e % rk, l = e / rk;
    cplx s = czero();
    for (int i = 0; i < rows; ++i) s = cfmac(U[i + LD * r], p.e[i + rows * l], s);
    p.sm[e] = s;
  }
  if (tid == 0) {
    p.st[1] = rk;
    p.st[2 + c] = rk;
  }
}

// H[r, b, al, e'] = sum_b' Sm[r, (b,b')] G_{c+1}[b', al, e'], grid (RB*RB*2*RB/NT, nprob)
__global__ void k_hrb_H(const HrBigProb* probs, int c) {
  const HrBigProb& p = probs[blockIdx.y];
  const int rk = p.st[1], q = c + 1;
  const int fa = p.f_ranks[q - 1], ga = p.g_ranks[q - 1], gb = p.g_ranks[q];
  const int e = blockIdx.x * NT + threadIdx.x;
  if (e >= rk * fa * 2 * gb) return;
  const int r = e % rk, t1 = e / rk;
  const int b = t1 % fa, t2 = t1 / fa;
  const int al = t2 & 1, ep = t2 >> 1;
  const cplx* G = gcore(p, q);
  cplx s = czero();
  for (int bp = 0; bp < ga; ++bp) s = cfma(p.sm[r + rk * (b * ga + bp)], G[bp + ga * al + 2 * ga * ep], s);
  p.hb[e] = s;
}

// E[r, al, (e,e')] = sum_b H[r,b,al,e'] F_{c+1}[b,al,e]; then ap <- rk
__global__ void k_hrb_E(const HrBigProb* probs, int c) {
  const HrBigProb& p = probs[blockIdx.y];
  const int rk = p.st[1], q = c + 1;
  const int fa = p.f_ranks[q - 1], fb = p.f_ranks[q], gb = p.g_ranks[q];
  const int e = blockIdx.x * NT + threadIdx.x;
  const cplx* F = fcore(p, q);
  if (e < rk * 2 * fb * gb) {
    const int r = e % rk, al = (e / rk) & 1, j = e / (2 * rk);
    const int ee = j / gb, ep = j % gb;
    cplx s = czero();
    for (int b = 0; b < fa; ++b) s = cfma(p.hb[r + rk * (b + fa * (al + 2 * ep))], F[b + fa * al + 2 * fa * ee], s);
    p.e[e] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.st[0] = rk;
}

__global__ void k_hrb_final(const HrBigProb* probs, int d) {
  const HrBigProb& p = probs[blockIdx.x];
  const int ap = p.st[0];
  cplx* oc = p.out_cores + (size_t)(d - 1) * SLOT;
  for (int e = threadIdx.x; e < 2 * ap; e += NT) oc[e] = p.e[e];
  for (int q = threadIdx.x; q <= d; q += NT) p.out_ranks[q] = (q == 0 || q == d) ? 1 : p.st[2 + q];
}


size_t hr_big_scratch(int d) {
  // gr (d slots) + t1/t2/t3 (2 slices each) + e, tb, sm, hb (complex) ; st, tau2 separate
  return (size_t)d * RZB * RZB + 6 * (size_t)RZB * RZB + 4 * (size_t)RWB * RZB;
}

static int launch_hr_gr_chain_impl(const HrBigProb* probs_dev, int nprob, int d, int gs, cudaStream_t st) {
  const int g2 = (gs + NT - 1) / NT;
  int n = 0;
  k_hrb_gr_last<<<dim3(g2, nprob), NT, 0, st>>>(probs_dev, d, gs);
  ++n;
  for (int c = d - 1; c >= 2; --c) {
    for (int stage = 0; stage < 4; ++stage) {
      k_hrb_gr_step<<<dim3(g2, 2, nprob), NT, 0, st>>>(probs_dev, c, stage, gs);
      ++n;
    }
  }
  return n;
}

// ------------------------------------------- cluster form (ranks <= 8)
// The right-Gram chain of Z = F (.) G for Rhat <= 8 (rz <= 64) in ONE launch:
// a cluster of 8 CTAs per tensor, CTA r owning the column group with F index
// r of every matrix (GR_c columns (r, k'), T1..T3 columns (r, e')), so the
// three mode products A1, A2, B1 are CTA-local; B2 sums over the F index:
// each CTA forms its partial P_r[:, (e, e')] = sum_al T3_al[:, (r, e')]
// conj(F[e, al, r]) for all e, and CTA e adds the partials of every CTA
// (distributed shared memory, ascending r: deterministic) for its column
// group — exactly the layout the next core needs.  Two cluster barriers per
// core instead of four grid-wide launches; every GR slot is also written to
// global memory for the sweep (layout of launch_hr_gr_chain).
static constexpr int CLR = 8;
struct GrClSmem {
  cplx grs[64 * 8];            // own column group of GR_c (rows rzx, ld 64)
  cplx t1[2][64 * 8];          // per slice al: T1 / T3 (rows, ld 64)
  cplx t2[2][64 * 8];          // T2
  cplx part[64 * 64];          // P_r (rows rzo x fa ga columns, ld 64)
  cplx fc[2 * 8 * 8], gc[2 * 8 * 8];
  int rf[MAXD + 1], rg[MAXD + 1];
};
__global__ void __cluster_dims__(CLR, 1, 1) __launch_bounds__(NT) k_hr_gr_cluster(const HrBigProb* probs, int d) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const HrBigProb& p = probs[blockIdx.y];
  extern __shared__ __align__(16) unsigned char smraw[];
  GrClSmem& S = *reinterpret_cast<GrClSmem*>(smraw);
  const int r = (int)cl.block_rank(), tid = threadIdx.x;
  for (int q = tid; q <= d; q += NT) { S.rf[q] = p.f_ranks[q]; S.rg[q] = p.g_ranks[q]; }
  __syncthreads();
  // GR_{d-1}[(a,a'),(b,b')] = sum_al Z[(a,a'),al] conj(Z[(b,b'),al]), Z = F_d[.,al] G_d[.,al]
  {
    const int af = S.rf[d - 1], ag = S.rg[d - 1], rz = af * ag;
    const cplx* F = fcore(p, d);
    const cplx* G = gcore(p, d);
    cplx* slot = p.gr + (size_t)(d - 1) * GR_HR;
    if (r < af)
      for (int e = tid; e < rz * ag; e += NT) {
        const int i = e % rz, jj = e / rz, ia = i / ag, ib = i % ag;
        cplx s = czero();
        for (int al = 0; al < 2; ++al) {
          const cplx zi = cmul(F[ia + af * al], G[ib + ag * al]);
          const cplx zj = cmul(F[r + af * al], G[jj + ag * al]);
          s = cfma_bc(zi, zj, s);
        }
        S.grs[i + 64 * jj] = s;
        slot[i + rz * (r * ag + jj)] = s;
      }
  }
  for (int c = d - 1; c >= 2; --c) {
    const int fa = S.rf[c - 1], fb = S.rf[c], ga = S.rg[c - 1], gb = S.rg[c];
    const int rzx = fb * gb, ra = fb * ga, rzo = fa * ga;
    {
      const cplx* F = fcore(p, c);
      const cplx* G = gcore(p, c);
      for (int e = tid; e < 2 * fa * fb; e += NT) S.fc[e] = F[e];
      for (int e = tid; e < 2 * ga * gb; e += NT) S.gc[e] = G[e];
    }
    __syncthreads();
    const cplx* F = S.fc;
    const cplx* G = S.gc;
    if (r < fb) {
      // A1: T1_al[(b,a'), jj] = sum_b' G[a',al,b'] GR_c[(b,b'), (r, jj)]
      for (int e = tid; e < 2 * ra * gb; e += NT) {
        const int al = e / (ra * gb), o = e % (ra * gb), i = o % ra, jj = o / ra;
        const int b = i / ga, ap = i % ga;
        cplx s = czero();
        for (int bp = 0; bp < gb; ++bp) s = cfma(G[ap + ga * al + 2 * ga * bp], S.grs[(b * gb + bp) + 64 * jj], s);
        S.t1[al][i + 64 * jj] = s;
      }
      __syncthreads();
      // A2: T2_al[(b,a'), ep] = sum_c' T1_al[(b,a'), c'] conj(G[ep,al,c'])
      for (int e = tid; e < 2 * ra * ga; e += NT) {
        const int al = e / (ra * ga), o = e % (ra * ga), i = o % ra, ep = o / ra;
        cplx s = czero();
        for (int cp = 0; cp < gb; ++cp) s = cfma_bc(S.t1[al][i + 64 * cp], G[ep + ga * al + 2 * ga * cp], s);
        S.t2[al][i + 64 * ep] = s;
      }
      __syncthreads();
      // B1: T3_al[(a,a'), ep] = sum_b F[a,al,b] T2_al[(b,a'), ep]   (into t1)
      for (int e = tid; e < 2 * rzo * ga; e += NT) {
        const int al = e / (rzo * ga), o = e % (rzo * ga), i = o % rzo, ep = o / rzo;
        const int aa = i / ga, ap = i % ga;
        cplx s = czero();
        for (int b = 0; b < fb; ++b) s = cfma(F[aa + fa * al + 2 * fa * b], S.t2[al][(b * ga + ap) + 64 * ep], s);
        S.t1[al][i + 64 * ep] = s;
      }
      __syncthreads();
      // B2 partial: P_r[i, (e, ep)] = sum_al T3_al[i, ep] conj(F[e, al, r])
      for (int o = tid; o < rzo * fa * ga; o += NT) {
        const int i = o % rzo, jc = o / rzo, ee = jc / ga, ep = jc % ga;
        cplx s = czero();
        for (int al = 0; al < 2; ++al) s = cfma_bc(S.t1[al][i + 64 * ep], F[ee + fa * al + 2 * fa * r], s);
        S.part[i + 64 * jc] = s;
      }
    }
    cl.sync();
    // B2 sum over the F index k (CTA k's partial), column group r of GR_{c-1}
    if (r < fa) {
      cplx* slot = p.gr + (size_t)(c - 1) * GR_HR;
      for (int o = tid; o < rzo * ga; o += NT) {
        const int i = o % rzo, ep = o / rzo, jc = r * ga + ep;
        cplx s = czero();
        for (int k = 0; k < fb; ++k) {
          const cplx* pk = cl.map_shared_rank(S.part, k);
          s = cadd(s, pk[i + 64 * jc]);
        }
        S.grs[i + 64 * ep] = s;
        slot[i + rzo * jc] = s;
      }
    }
    cl.sync();
  }
}

cudaError_t setup_hr_big_kernels() {
  cudaError_t e = cudaFuncSetAttribute(k_hrb_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HrbSolveSmem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_hr_gr_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(GrClSmem));
}

cudaError_t launch_hr_gr_chain_cluster(const HrBigProb* probs_dev, int nprob, int d, cudaStream_t st) {
  k_hr_gr_cluster<<<dim3(CLR, nprob), NT, sizeof(GrClSmem), st>>>(probs_dev, d);
  count_launches(1);
  return cudaGetLastError();
}

// The right-Gram chain alone for the one-CTA rounding (Kronecker ranks <= 64):
// GR slots of GR_HR entries (the layout k_hadamard_round reads), t1..t3 of
// 2 x GR_HR each.  ~4 (d - 2) launches, every mode product spread over the GPU.
cudaError_t launch_hr_gr_chain(const HrBigProb* probs_dev, int nprob, int d, cudaStream_t st) {
  const int n = launch_hr_gr_chain_impl(probs_dev, nprob, d, GR_HR, st);
  count_launches(n);
  return cudaGetLastError();
}

cudaError_t launch_hadamard_round_big(const HrBigProb* probs_dev, int nprob, const HrParams& prm, cudaStream_t st) {
  const int d = prm.d;
  int n = launch_hr_gr_chain_impl(probs_dev, nprob, d, RZB * RZB, st);
  k_hrb_init<<<nprob, NT, 0, st>>>(probs_dev, d);
  ++n;
  const int gt = (RWB * RZB + NT - 1) / NT, gh = (RB * RB * 2 * RB + NT - 1) / NT;
  for (int c = 1; c <= d - 1; ++c) {
    k_hrb_T<<<dim3(gt, nprob), NT, 0, st>>>(probs_dev, c);
    k_hrb_solve<<<nprob, NT, sizeof(HrbSolveSmem), st>>>(probs_dev, c, d, prm);
    k_hrb_H<<<dim3(gh, nprob), NT, 0, st>>>(probs_dev, c);
    k_hrb_E<<<dim3(gh, nprob), NT, 0, st>>>(probs_dev, c);
    n += 4;
  }
  k_hrb_final<<<nprob, NT, 0, st>>>(probs_dev, d);
  ++n;
  count_launches(n);
  return cudaGetLastError();
}

}  // namespace qtt

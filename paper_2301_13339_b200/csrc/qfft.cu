// qfft.cu — capped QTT-FFT / QTT-iFFT on sm_100a (PAPER.md P:309-321,
// P:370-382; construction of SURVEY.md §8(c) O2, inverse O6, centering O3).
//
// One CTA per transform keeps every core in shared memory and runs the whole
// serial chain on chip.  Stage p (p = d..1; a = axis(p), t = bit(p),
// s = b_a - t + 1):
//   p = d : core_d[:, al, :] <- core_d[:,0,:] + (-1)^al core_d[:,1,:]
//   p < d : cut ranks p..d-1 double: core_p <- [core_p[:,0,:] | (-1)^al
//           core_p[:,1,:]], core_q <- blockdiag(core_q, phi_q core_q),
//           core_d <- vstack(core_d, phi_d core_d), phi_q(1) = exp(-i pi /
//           2^{bit(q)-t}) for axis(q) = a; then ROUND_LOCAL(p).
// ROUND_LOCAL(p) is evaluated without the LQ sweep of the oracle: the right
// Gram matrices GR_c = R_c R_c^H of the doubled cores are built right-to-left
// once per stage, and the truncation of cut c uses the Hermitian
// K_c = M_c GR_c M_c^H, whose eigenvalues are the squared singular values of
// the cut-c unfolding and whose eigenvectors are its left singular vectors
// (the same truncated tensor as LQ + SVD, in exact arithmetic).
// The doubled cores are never stored: the right-Gram chain runs on the
// compact cores in block form, and the sweep forms the pushed doubled core
// on the fly from the compact cores (ranks <= RS_XF) kept in shared memory.
#include "qtt_kernels.h"

namespace qtt {

static constexpr int NT = 256;

// optional phase timing (compile with -DQTT_XF_TIMING): cycles per phase of
// CTA 0 are accumulated into XfProb::gr scratch tail (debug builds only)
#ifdef QTT_XF_TIMING
#define XT_DECL long long xt_t0 = clock64(), xt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define XT_MARK(k) { long long _t = clock64(); xt_acc[k] += _t - xt_t0; xt_t0 = _t; }
#define XT_DUMP(ptr) if (threadIdx.x == 0) { for (int _k = 0; _k < 8; ++_k) ((long long*)(ptr))[_k] = xt_acc[_k]; }
#else
#define XT_DECL
#define XT_MARK(k)
#define XT_DUMP(ptr)
#endif
// Rank capacity RSV of the compact cores: 10 (Rhat <= 8 pipelines; every
// core in shared memory) or 16 (the paper's Rhat = 15; the cores live in the
// workspace, pr.cwork, and stay L2-resident).  Rows of a cut <= 2 RSV.
static_assert(sizeof(EigSmem<16>) <= sizeof(EigSmem<20>), "the width-16 solver overlays S.E");
template <int RSV>
struct XfBufs {
  static constexpr int R2 = 2 * RSV;
  cplx D[R2 * 2 * R2];
  cplx Eb[RSV * 2 * R2];
  cplx G[2][R2 * R2];
  cplx T[2 * R2 * R2];
  cplx Sm[RSV * R2];
  EigSmem<R2> E;
  cplx phtab[32];            // phtab[k] = exp(-i pi / 2^k)
  int r[MAXD + 1];
  int rb[MAXD + 1];
  int rk;
  double tau2;
  double mdefer[4];          // deferred T2 record of the last RANK (margins_flush)
};
template <int RSV, bool SMEM_CORES = (RSV <= 10)>
struct XfSmem : XfBufs<RSV> {
  cplx C[MAXD][2 * RSV * RSV];
};
template <int RSV>
struct XfSmem<RSV, false> : XfBufs<RSV> {};

// twiddle of position q (1-based) in the stage of axis a, bit t, slice be:
// exp(-i pi / 2^k), k = bit(q) - t >= 1, from the per-CTA table S.phtab
// (filled once per launch; a double sincospi per use sat on the chain)
template <class SM>
__device__ __forceinline__ cplx phi_of(const SM& S, const XfParams& P, int q, int a, int t, int be) {
  if (be == 0 || P.axis[q - 1] != a) return cmk(1.0, 0.0);
  return S.phtab[P.bit[q - 1] - t];
}

template <int RSV>
__global__ void __launch_bounds__(NT, 1) k_transform(const XfProb* probs, XfParams P) {
  const XfProb& pr = probs[blockIdx.x];
  extern __shared__ __align__(16) unsigned char smraw[];
  XfSmem<RSV>& S = *reinterpret_cast<XfSmem<RSV>*>(smraw);
  constexpr int RS = RSV, R2 = 2 * RSV, CSZ = 2 * RSV * RSV, GRS = R2 * R2;
  constexpr int LD = EigSmem<R2>::LD;
  auto core = [&](int q) -> cplx* {
    if constexpr (RSV <= 10) return S.C[q];
    else return pr.cwork + (size_t)q * CSZ;
  };
  const int tid = threadIdx.x;
  const int d = P.d;
  // load (conj for the inverse); twiddle table
  for (int q = tid; q <= d; q += NT) S.r[q] = pr.in_ranks[q];
  if (tid < 32) S.phtab[tid] = tid == 0 ? cmk(1.0, 0.0) : cexpipi(-ldexp(1.0, -tid));
  if (tid == 0) S.mdefer[1] = 0.0;
  __syncthreads();
  for (int q = 0; q < d; ++q) {
    const int n = S.r[q] * 2 * S.r[q + 1];
    for (int e = tid; e < n; e += NT) {
      cplx v = pr.in_cores[(size_t)q * SLOT + e];
      core(q)[e] = P.inverse ? cconj(v) : v;
    }
  }
  __syncthreads();
  XT_DECL
  for (int p = d; p >= 1; --p) {
    const int a = P.axis[p - 1], t = P.bit[p - 1];
    if (p == d) {
      const int a0 = S.r[d - 1];
      cplx* c = core(d - 1);
      for (int i = tid; i < a0; i += NT) {
        cplx x0 = c[i], x1 = c[i + a0];
        c[i] = cadd(x0, x1);
        c[i + a0] = csub(x0, x1);
      }
      __syncthreads();
      continue;
    }
    // ---- right Gram chain GR_c, c = d-1 .. p, into global slots.  The
    //      doubled cores blockdiag(C_q, phi_q C_q) (q < d) and vstack(C_d,
    //      phi_d C_d) with |phi| = 1 give GR_c = [[G_c, H_c^H], [H_c, G_c]]:
    //        G_{q-1} = sum_be C_q[be] G_q C_q[be]^H       (plain right Gram)
    //        H_{q-1} = sum_be phi_q(be) C_q[be] H_q C_q[be]^H
    //      from G_{d-1} = sum_be c_d[be] c_d[be]^H, H_{d-1} = sum_be
    //      phi_d(be) c_d[be] c_d[be]^H — two r x r chains on the compact
    //      cores instead of one 2r x 2r chain on materialised doubled cores.
    {
      cplx* SG[2] = {S.G[0], S.G[0] + RS * RS};   // G_c, H_c (ld r_c), generation 0
      cplx* SN[2] = {S.G[1], S.G[1] + RS * RS};   // generation 1
      const int a0 = S.r[d - 1];
      const cplx* c = core(d - 1);
      const cplx ph = phi_of(S, P, d, a, t, 1);
      for (int e = tid; e < 2 * a0 * a0; e += NT) {
        const int w = e / (a0 * a0), ij = e % (a0 * a0), i = ij % a0, j = ij / a0;
        const cplx s0 = cmul(c[i], cconj(c[j]));
        const cplx s1 = cmul(c[i + a0], cconj(c[j + a0]));
        SG[w][i + a0 * j] = w == 0 ? cadd(s0, s1) : cadd(s0, cmul(ph, s1));
      }
      __syncthreads();
      cplx** cur = SG;
      cplx** nxt = SN;
      int rc = a0;   // r_c of the chain's current cut c
      for (int cq = d - 1;; --cq) {
        // write GR_cq = [[G, H^H], [H, G]] (2 rc x 2 rc) to its slot
        {
          const int n2 = 2 * rc;
          cplx* g = pr.gr + (size_t)cq * GRS;
          const bool p16 = n2 == 16;   // steady state: shifts instead of runtime divisions
          for (int e = tid; e < n2 * n2; e += NT) {
            const int i = p16 ? (e & 15) : e % n2, j = p16 ? (e >> 4) : e / n2;
            const int bi = i >= rc, bj = j >= rc, ii = i - bi * rc, jj = j - bj * rc;
            cplx v;
            if (bi == bj) v = cur[0][ii + rc * jj];
            else if (bi) v = cur[1][ii + rc * jj];
            else v = cconj(cur[1][jj + rc * ii]);
            g[e] = v;
          }
        }
        XT_MARK(4)
        if (cq <= p) break;
        // step to cut cq - 1 through core q = cq (compact a1 x 2 x rc)
        const int q = cq;
        const int a1 = S.r[q - 1];
        const cplx* cc = core(q - 1);
        const cplx phq = phi_of(S, P, q, a, t, 1);
        cplx* TG = S.D;                       // [w][be]: a1 x rc, ld a1
        const int tsz = a1 * rc;
        // element (wb, i, j) of the step's two product rounds; ranks <= 8
        // (the steady state) map threads by shifts: the runtime divisions of
        // the general loops cost ~100 cycles each at the head of a round
        auto tg_elem = [&](int wb, int i, int j) {
          const int w = wb >> 1, be = wb & 1;
          const cplx* X = cur[w];
          const cplx* Cr = cc + i + a1 * be;
          TG[wb * tsz + i + a1 * j] =
              dotu<RS>(rc, [&](int l, cplx acc) { return cfma(Cr[2 * a1 * l], X[l + rc * j], acc); });
        };
        auto nx_elem = [&](int w, int i, int j) {
          const cplx* T0 = TG + (2 * w) * tsz + i;
          const cplx* T1 = TG + (2 * w + 1) * tsz + i;
          const cplx* C0 = cc + j;
          const cplx* C1 = cc + j + a1;
          const cplx s0 = dotu<RS>(rc, [&](int l, cplx acc) { return cfma_bc(T0[a1 * l], C0[2 * a1 * l], acc); });
          const cplx s1 = dotu<RS>(rc, [&](int l, cplx acc) { return cfma_bc(T1[a1 * l], C1[2 * a1 * l], acc); });
          nxt[w][i + a1 * j] = w == 0 ? cadd(s0, s1) : cadd(s0, cmul(phq, s1));
        };
        const bool small8 = NT == 256 && a1 <= 8 && rc <= 8;
        if (small8) {
          const int i = tid & 7, j = (tid >> 3) & 7;
          if (i < a1 && j < rc) tg_elem(tid >> 6, i, j);
        } else {
          for (int e = tid; e < 4 * tsz; e += NT) {
            const int wb = e / tsz, ij = e % tsz;
            tg_elem(wb, ij % a1, ij / a1);
          }
        }
        __syncthreads();
        XT_MARK(0)
        if (small8) {
          const int i = tid & 7, j = (tid >> 3) & 7;
          if (tid < 128 && i < a1 && j < a1) nx_elem(tid >> 6, i, j);
        } else {
          for (int e = tid; e < 2 * a1 * a1; e += NT) {
            const int w = e / (a1 * a1), ij = e % (a1 * a1);
            nx_elem(w, ij % a1, ij / a1);
          }
        }
        __syncthreads();
        XT_MARK(0)
        cplx** tmp = cur;
        cur = nxt;
        nxt = tmp;
        rc = a1;
      }
    }
    XT_MARK(0)
    // ---- rank bounds of the LQ sweep (oracle ROUND_LOCAL (i)): rb_c
    if (tid == 0) {
      S.rb[d] = 1;
      for (int c = d - 1; c >= p; --c) {
        int v = 2 * S.r[c], w = 2 * S.rb[c + 1];
        S.rb[c] = v < w ? v : w;
      }
    }
    // ---- E = concat(core_p)
    {
      const int a0 = S.r[p - 1], b0 = S.r[p];
      const cplx* c = core(p - 1);
      for (int e = tid; e < a0 * 2 * 2 * b0; e += NT) {
        int i = e % a0, al = (e / a0) & 1, j = e / (2 * a0);
        cplx v = (j < b0) ? c[i + 2 * a0 * j] : c[i + a0 + 2 * a0 * (j - b0)];
        if (j >= b0 && al) v = cmk(-v.x, -v.y);
        S.Eb[e] = v;
      }
    }
    __syncthreads();
    // ---- truncation sweep, c = p .. d-1.  GR_c comes from the L2-resident
    //      slots through a cp.async double buffer: GR_{c+1} is requested
    //      right after cut c's T = M GR_c and lands during its eigensolve.
    int ap = S.r[p - 1];
    {
      const int cols = 2 * S.r[p];
      for (int e = tid; e < cols * cols; e += NT) cp_async16(&S.G[0][e], &pr.gr[(size_t)p * GRS + e]);
      cp_async_commit();
    }
    for (int c = p; c <= d - 1; ++c) {
      const int rows = 2 * ap, cols = 2 * S.r[c];
      const int gb = (c - p) & 1;
      XT_MARK(5)
      cp_async_wait<0>();
      __syncthreads();
      // T = M G  (rows x cols), M = Eb (ld rows); DMMA tiles
      {
        const cplx* Gm = S.G[gb];
        cgemm_dmma_sg<NT / 32>(GemmArgs{S.Eb, Gm, S.T, rows, cols, cols, 1, rows, 1, cols, 1, rows, 0, 0});
      }
      __syncthreads();
      if (c + 1 <= d - 1) {
        const int cols1 = 2 * S.r[c + 1];
        for (int e = tid; e < cols1 * cols1; e += NT)
          cp_async16(&S.G[gb ^ 1][e], &pr.gr[(size_t)(c + 1) * GRS + e]);
      }
      cp_async_commit();
      // K = T M^H, into the eigensolver of width 16 when rows <= 16 (the
      // steady state at Rhat <= 8; 18% fewer cycles than width R2 at n = 16,
      // tools/dev_trid_timing.py), else width R2; both share S.E's memory
      const bool w16 = (R2 > 16) && rows <= 16;
      EigSmem<16>& E16 = *reinterpret_cast<EigSmem<16>*>(&S.E);
      cplx* Kb = w16 ? E16.A[0] : S.E.A[0];
      const int ldk = w16 ? EigSmem<16>::LD : LD;
      // K = T M^H (rows x rows); DMMA tiles
      cgemm_dmma_sg<NT / 32>(GemmArgs{S.T, S.Eb, Kb, rows, rows, cols, 1, rows, rows, 1, 1, ldk, 0, 1});
      __syncthreads();
      if (c == p) {
        double tr = 0.0;
        if (tid < rows) tr = Kb[tid + ldk * tid].x;
        tr = block_sum<NT>(tr, w16 ? E16.red : S.E.red);
        if (tid == 0) S.tau2 = P.eps * P.eps * tr / (double)(d - 1);
        __syncthreads();
      }
      XT_MARK(1)
      // While warps 0 / 1 tridiagonalise (width 16), warps 2-7 form
      // MD = M x doubled(core c+1) (rows x 4 b1, column oc = be + 2 j' as
      // in the E layout; the last core: rows x 2), so after U only
      // E_next = U^H MD remains (one product instead of U^H M, then x D)
      const int a1n = S.r[c];
      const int b1n = (c + 1 < d) ? S.r[c + 1] : 0;
      const int mdc = (c + 1 < d) ? 4 * b1n : 2;
      cplx* MD = S.D;   // free during the sweep (the right-Gram chain's scratch)
      if (w16) {
        const cplx* cn = core(c);
        const cplx phq = phi_of(S, P, c + 1, a, t, 1);
        auto side = [&] {
          // warps 2, 3, 6, 7 (sub-partitions 2 and 3): the tridiagonalising
          // warps 0 / 1 keep sub-partitions 0 / 1 to themselves
          const int wq = tid >> 5;
          const int sidew = (wq == 2 || wq == 3) ? wq - 2 : ((wq == 6 || wq == 7) ? wq - 4 : -1);
          if (c + 1 < d) {
            cgemm_dmma_wl(
                rows, mdc, 2 * a1n,
                [&](int i, int l) { return (i < rows && l < 2 * a1n) ? S.Eb[i + rows * l] : czero(); },
                [&](int l, int oc) {
                  const int be = oc & 1, jp = oc >> 1, sb = jp >= b1n, j = jp - sb * b1n;
                  const int sl = l >= a1n, ii = l - sl * a1n;
                  if (l >= 2 * a1n || oc >= mdc || sl != sb) return czero();
                  const cplx v = cn[ii + a1n * be + 2 * a1n * j];
                  return (sb && be) ? cmul(phq, v) : v;
                },
                [&](int i, int oc, cplx v) { if (i < rows && oc < mdc) MD[i + rows * oc] = v; }, sidew, 4);
          } else {
            cgemm_dmma_wl(
                rows, 2, 2 * a1n,
                [&](int i, int l) { return (i < rows && l < 2 * a1n) ? S.Eb[i + rows * l] : czero(); },
                [&](int l, int be) {
                  const int sl = l >= a1n, ii = l - sl * a1n;
                  if (l >= 2 * a1n || be >= 2) return czero();
                  const cplx v = cn[ii + a1n * be];
                  return (sl && be) ? cmul(phq, v) : v;
                },
                [&](int i, int be, cplx v) { if (i < rows && be < 2) MD[i + rows * be] = v; }, sidew, 4);
          }
        };
        eig_values<16, NT>(E16, rows, side);
      } else {
        eig_values<R2, NT>(S.E, rows);
      }
      XT_MARK(2)
      // RANK (its T2 record deferred to the last warp during the vectors)
      if (tid < 32) {
        const int mp = rows < S.rb[c] ? rows : S.rb[c];
        const int r = rank_choose_warp(w16 ? E16.lam : S.E.lam, mp, S.tau2, P.rmax, P.ctol, P.rule, P.delta, P.status,
                                       S.mdefer);
        if (tid == 0) S.rk = r;
      }
      __syncthreads();
      XT_MARK(6)
      auto flush = [&] { if ((tid & 31) == 0) margins_flush(S.mdefer, P.status); };
      const cplx* U = w16 ? eig_vectors_spec<16, NT>(E16, rows, S.rk, nullptr, flush, P.status)
                          : eig_vectors_spec<R2, NT>(S.E, rows, S.rk, nullptr, flush, P.status);
      const int rk = S.rk;
      XT_MARK(7)
      // new core c = U_r  (ap x 2 x rk)
      {
        const bool p16 = rows == 16;
        for (int e = tid; e < rows * rk; e += NT) {
          const int i = p16 ? (e & 15) : e % rows, r = p16 ? (e >> 4) : e / rows;
          core(c - 1)[i + rows * r] = U[i + ldk * r];
        }
      }
      if (w16) {
        // next E = U_r^H MD  (rk x mdc: Eb[r + rk oc], the layout r + rk be + 2 rk j')
        cgemm_dmma_sg<NT / 32>(GemmArgs{U, MD, S.Eb, rk, mdc, rows, ldk, 1, 1, rows, 1, rk, 1, 0});
      } else {
      // Sm = U_r^H M  (rk x cols); DMMA tiles
        cgemm_dmma_sg<NT / 32>(GemmArgs{U, S.Eb, S.Sm, rk, cols, rows, ldk, 1, 1, rows, 1, rk, 1, 0});
        __syncthreads();
        // next E = Sm * doubled(core c+1)
        {
          const int q = c + 1;
          const int a1 = S.r[c];
          const cplx* cn = core(q - 1);
          if (q < d) {
            const int b1 = S.r[q];
            for (int e = tid; e < rk * 2 * 2 * b1; e += NT) {
              int r = e % rk, be = (e / rk) & 1, j = e / (2 * rk);
              cplx s;
              if (j < b1) {
                s = dotu<RS>(a1, [&](int i, cplx acc) { return cfma(S.Sm[r + rk * i], cn[i + a1 * be + 2 * a1 * j], acc); });
              } else {
                s = dotu<RS>(a1, [&](int i, cplx acc) {
                  return cfma(S.Sm[r + rk * (a1 + i)], cn[i + a1 * be + 2 * a1 * (j - b1)], acc);
                });
                if (be) s = cmul(phi_of(S, P, q, a, t, 1), s);
              }
              S.Eb[e] = s;
            }
          } else {
            for (int e = tid; e < rk * 2; e += NT) {
              int r = e % rk, be = e / rk;
              const cplx s0 = dotu<RS>(a1, [&](int i, cplx acc) { return cfma(S.Sm[r + rk * i], cn[i + a1 * be], acc); });
              cplx s1 = dotu<RS>(a1, [&](int i, cplx acc) { return cfma(S.Sm[r + rk * (a1 + i)], cn[i + a1 * be], acc); });
              if (be) s1 = cmul(phi_of(S, P, q, a, t, 1), s1);
              S.Eb[e] = cadd(s0, s1);
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0) S.r[c] = rk;   // read next after the barrier at the top of cut c+1
      ap = rk;
      XT_MARK(3)
    }
    for (int e = tid; e < ap * 2; e += NT) core(d - 1)[e] = S.Eb[e];
    __syncthreads();
  }
  XT_MARK(4)
  XT_DUMP(pr.gr + (size_t)MAXD * GRS - 8)
  // ---- reversal (core'_q = core_{d+1-q}, rank indices swapped), center,
  //      conj (inverse), scale core 1
  for (int q = tid; q <= d; q += NT) pr.out_ranks[q] = S.r[d - q];
  for (int q = 1; q <= d; ++q) {
    const cplx* c = core(d - q);
    const int a0 = S.r[d - q], b0 = S.r[d - q + 1];   // source dims (a0, 2, b0)
    cplx ph = cmk(1.0, 0.0);
    if (pr.do_center) {
      const int ax = P.axis[d - q], tt = P.bit[d - q], b = P.bits[ax];
      const int m = b + 1 - tt;
      unsigned long long num = ((unsigned long long)P.shift[ax] << (m - 1)) & ((1ull << b) - 1ull);
      if (num) ph = cexpipi((double)num / (double)(1ull << (b - 1)));
    }
    cplx* o = pr.out_cores + (size_t)(q - 1) * SLOT;
    for (int e = tid; e < a0 * 2 * b0; e += NT) {
      int i = e % b0, be = (e / b0) & 1, j = e / (2 * b0);   // out (b0, 2, a0): (i, be, j)
      cplx v = c[j + a0 * be + 2 * a0 * i];
      if (be) v = cmul(ph, v);
      if (P.inverse) v = cconj(v);
      if (q == 1) v = cscale(v, P.scale);
      o[e] = v;
    }
  }
}

cudaError_t setup_xf_kernels() {
  cudaError_t e = cudaFuncSetAttribute(k_transform<RS_XF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(XfSmem<RS_XF>));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_transform<RS_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(XfSmem<RS_BIG>));
}

size_t xf_gr_slot(int rs) { return (size_t)(2 * rs) * (2 * rs); }

cudaError_t launch_transform(const XfProb* probs_dev, int nprob, const XfParams& prm, cudaStream_t st) {
  if (prm.rs > RS_XF) k_transform<RS_BIG><<<nprob, NT, sizeof(XfSmem<RS_BIG>), st>>>(probs_dev, prm);
  else k_transform<RS_XF><<<nprob, NT, sizeof(XfSmem<RS_XF>), st>>>(probs_dev, prm);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace qtt

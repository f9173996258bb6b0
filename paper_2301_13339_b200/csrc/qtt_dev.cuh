// qtt_dev.cuh — device helpers shared by the libqtt kernels (sm_100a).
//
// Complex arithmetic, QTT-index <-> memory-offset maps (reading
// Q8), the FP64 tensor-core MMA wrapper (mma.sync m8n8k4 f64 -> DMMA; there is
// no tcgen05 kind for f64 on sm_100a), a CTA-cooperative Jacobi
// eigensolver for the small Hermitian Gram matrices of the truncated SVDs
// (Alg. 1 line "Compute truncated SVD") and the rank rule RANK
// (modification (1) P:357, reading Q6').
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qtt {

typedef double2 cplx;

// ----------------------------------------------------------------- complex
__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx czero() { return make_double2(0.0, 0.0); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * b + c
__host__ __device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// conj(a) * b + c
__host__ __device__ __forceinline__ cplx cfmac(cplx a, cplx b, cplx c) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
// a * conj(b) + c
__host__ __device__ __forceinline__ cplx cfma_bc(cplx a, cplx b, cplx c) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.y, b.x, fma(-a.x, b.y, c.y)));
}

// exp(i pi x) for an exact dyadic x (twiddles, reading Q25)
__device__ __forceinline__ cplx cexpipi(double x) {
  double s, c;
  sincospi(x, &s, &c);
  return make_double2(c, s);
}

// ------------------------------------------------------------ layout maps
// QTT index q (LSB first) -> element offset in the caller's array.
//   1D / concat: offset = q (row-major image, x fastest, x bits first).
//   interleaved: bits 0,2,4.. are x bits, 1,3,5.. are y bits (reading Q8).
__host__ __device__ __forceinline__ uint64_t compact_even(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return x;
}

enum { LAYOUT_1D = 0, LAYOUT_INTERLEAVED = 1, LAYOUT_CONCAT = 2 };

__host__ __device__ __forceinline__ uint64_t qtt_offset(uint64_t q, int layout, int bx) {
  if (layout != LAYOUT_INTERLEAVED) return q;
  return compact_even(q) + (compact_even(q >> 1) << bx);
}

// ------------------------------------------------------------------ DMMA
// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor core (SASS DMMA.8x8x4).
// Fragments: a = A[lane>>2][lane&3]; b = B[lane&3][lane>>2];
//            c0,c1 = C[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------------------ status word
enum { ST_OK = 0, ST_NONFINITE = 1, ST_NOCONV = 2, ST_RANKCAP = 4 };
__device__ __forceinline__ void raise_status(int* status, int bit) {
  if (status) atomicOr(status, bit);
}

// -------------------------------------------------------- Jacobi eigensolver
// Hermitian A (n x n, n <= NMAX) in shared memory, column-major with leading
// dimension NMAX+1.  Cyclic two-sided Jacobi with the round-robin parallel
// ordering (n/2 disjoint rotations per round, one fused J^H A J update per
// round).  On return lam[0..n-1] holds the eigenvalues in descending order
// and U (column-major, ld NMAX+1) the matching orthonormal eigenvectors.
// Stops after a sweep in which no pair needed a rotation (see below).
template <int NMAX>
struct EigSmem {
  static constexpr int LD = NMAX + 1;
  cplx A[2][NMAX * LD];
  cplx V[2][NMAX * LD];
  double cs[NMAX + 1];
  cplx co[NMAX + 1];
  int partner[NMAX + 1];
  double nd[NMAX + 1];
  int rot[NMAX + 1];
  double lam[NMAX];
  double red[32];
  int cur;
  int sweeps;
};

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (l < NT / 32) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

// A is read from E.A[0] (caller fills the full Hermitian matrix).  Result:
// E.lam (descending) and a pointer to the sorted eigenvectors (column-major,
// ld NMAX+1) inside E, valid until the next call.  Non-convergence raises
// ST_NOCONV in *status.
template <int NMAX, int NT>
__device__ const cplx* jacobi_eig(EigSmem<NMAX>& E, int n, int* status) {
  constexpr int LD = NMAX + 1;
  const int tid = threadIdx.x;
  const int N = n + (n & 1);
  for (int e = tid; e < n * n; e += NT) {
    int i = e % n, j = e / n;
    E.V[0][i + LD * j] = cmk(i == j ? 1.0 : 0.0, 0.0);
  }
  double nrm2 = 0.0;
  for (int e = tid; e < n * n; e += NT) {
    int i = e % n, j = e / n;
    nrm2 += cabs2(E.A[0][i + LD * j]);
  }
  nrm2 = block_sum<NT>(nrm2, E.red);
  // rotate (p,q) iff |a_pq| > max(1e-18 ||A||_F, 2^-53 sqrt|a_pp a_qq|):
  // high relative accuracy down to the formation noise of A; converged when a
  // whole sweep rotates nothing.
  const double floor_abs = 1e-18 * sqrt(nrm2);
  int cur = 0;
  bool conv = (n <= 1);
  int sweep = 0;
  for (; sweep < 40 && !conv; ++sweep) {
    int any_sweep = 0;
    for (int round = 0; round < N - 1; ++round) {
      const cplx* A = E.A[cur];
      int did = 0;
      if (tid < N / 2) {
        int p, q;
        if (tid == 0) { p = N - 1; q = round; }
        else { p = (round + tid) % (N - 1); q = (round - tid + (N - 1)) % (N - 1); }
        if (p >= n || q >= n) {
          if (p < n) { E.cs[p] = 1.0; E.co[p] = czero(); E.partner[p] = p; E.rot[p] = 0; }
          if (q < n) { E.cs[q] = 1.0; E.co[q] = czero(); E.partner[q] = q; E.rot[q] = 0; }
        } else {
          double a = A[p + LD * p].x, c = A[q + LD * q].x;
          cplx b = A[p + LD * q];
          double ab = sqrt(cabs2(b));
          double thr = fmax(floor_abs, 1.1102230246251565e-16 * sqrt(fabs(a * c)));
          if (!(ab > thr)) {
            E.cs[p] = 1.0; E.co[p] = czero(); E.partner[p] = q; E.rot[p] = 0;
            E.cs[q] = 1.0; E.co[q] = czero(); E.partner[q] = p; E.rot[q] = 0;
          } else {
            double zeta = (c - a) / (2.0 * ab);
            double t = 1.0 / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            if (zeta < 0.0) t = -t;
            double cc = 1.0 / sqrt(1.0 + t * t);
            double ss = t * cc;
            cplx S = cmk(ss * b.x / ab, ss * b.y / ab);
            E.cs[p] = cc; E.co[p] = cmk(-S.x, S.y);  // -conj(S)
            E.cs[q] = cc; E.co[q] = S;
            E.partner[p] = q; E.partner[q] = p;
            E.nd[p] = a - t * ab; E.nd[q] = c + t * ab;
            E.rot[p] = 1; E.rot[q] = 1;
            did = 1;
          }
        }
      }
      if (!__syncthreads_or(did)) continue;
      any_sweep = 1;
      cplx* An = E.A[cur ^ 1];
      const cplx* V = E.V[cur];
      cplx* Vn = E.V[cur ^ 1];
      for (int e = tid; e < 2 * n * n; e += NT) {
        if (e < n * n) {
          int i = e % n, j = e / n;
          int ip = E.partner[i], jp = E.partner[j];
          cplx val;
          if (E.rot[i] && i == j) val = cmk(E.nd[i], 0.0);
          else if (E.rot[i] && jp == i) val = czero();
          else {
            double ci = E.cs[i], cj = E.cs[j];
            cplx oi = E.co[i], oj = E.co[j];
            cplx t0 = cfma(oj, A[i + LD * jp], cscale(A[i + LD * j], cj));
            cplx t1 = cfma(oj, A[ip + LD * jp], cscale(A[ip + LD * j], cj));
            val = cfmac(oi, t1, cscale(t0, ci));
          }
          An[i + LD * j] = val;
        } else {
          int f = e - n * n;
          int i = f % n, j = f / n;
          int jp = E.partner[j];
          Vn[i + LD * j] = cfma(E.co[j], V[i + LD * jp], cscale(V[i + LD * j], E.cs[j]));
        }
      }
      __syncthreads();
      cur ^= 1;
    }
    conv = !any_sweep;
  }
  // stable descending sort; eigenvectors to the free V buffer
  for (int i = tid; i < n; i += NT) {
    double li = E.A[cur][i + LD * i].x;
    int rk = 0;
    for (int j = 0; j < n; ++j) {
      double lj = E.A[cur][j + LD * j].x;
      rk += (lj > li) || (lj == li && j < i);
    }
    E.partner[i] = rk;
  }
  __syncthreads();
  cplx* U = E.V[cur ^ 1];
  for (int i = tid; i < n; i += NT) E.lam[E.partner[i]] = E.A[cur][i + LD * i].x;
  for (int e = tid; e < n * n; e += NT) {
    int i = e % n, j = e / n;
    U[i + LD * E.partner[j]] = E.V[cur][i + LD * j];
  }
  if (tid == 0) E.sweeps = sweep;
  __syncthreads();
  if (!conv && tid == 0) raise_status(status, ST_NOCONV);
  return U;
}

// --------------------------------------------------------------- RANK rule
// lam descending (clamped at 0), m = list length.  See oracle/qtt.py
// rank_rule: r_tau = min{r : sum_{i>r} lam_i <= tau2}; r = min(r_tau, R);
// cluster cl(r): r < m, lam_r > 0, lam_r - lam_{r+1} <= ctol * lam_r.
__device__ __forceinline__ int rank_rule(const double* lam, int m, double tau2, int rmax, double ctol) {
  if (m <= 0) return 1;
  double l0 = fmax(lam[0], 0.0);
  if (!(l0 > 0.0)) return 1;
  // tails from the smallest value up
  double tail = 0.0;
  int r_tau = m;
  // T(r) for r = m..1: find the minimal r with T(r) <= tau2
  // T(m) = 0 <= tau2 always; walk down while T(r-1) <= tau2
  for (int r = m; r >= 1; --r) {
    // here tail = T(r)
    if (tail <= tau2) r_tau = r; else break;
    tail += fmax(lam[r - 1], 0.0);
  }
  int r = r_tau < rmax ? r_tau : rmax;
  auto cl = [&](int q) -> bool {
    if (q >= m) return false;
    double a = fmax(lam[q - 1], 0.0), b = fmax(lam[q], 0.0);
    return a > 0.0 && (a - b) <= ctol * a;
  };
  if (cl(r)) {
    if (r_tau <= rmax) {
      int rp = r + 1;
      while (cl(rp)) ++rp;
      if (rp <= rmax) return rp;
    }
    while (r > 1 && cl(r)) --r;
  }
  return r;
}

}  // namespace qtt

// qtt_kernels.h — device-side problem descriptors and launchers used by the
// C-ABI layer (api.cu).  Internal to libqtt; not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "qtt_dev.cuh"

namespace qtt {

// number of kernels launched by this library (bench evidence: gpu_launches)
void count_launches(int n);
// pass-level profiling (qtt_profile_enable(2)): CUDA events around the
// full-array passes, pass = PASS_*, end = 0 before / 1 after the launch
enum { PASS_LEVEL_GRAM = 0, PASS_PROJECT_X = 1, PASS_PROJECT_W = 2, PASS_EXPAND = 3, PASS_N = 4 };
void prof_pass(int pass, int end, cudaStream_t st);
// SMs of the current device (cached per device; grids are sized from it)
int sm_count();

// A TT core slot holds up to RC x 2 x RC complex entries (RC = 16), stored
// compact column-major: element (a, be, b) of an (r0, 2, r1) core at
// a + r0*be + 2*r0*b (so the r0 x 2r1 and 2r0 x r1 unfoldings of P:234 are
// plain column-major views of the same memory).
static constexpr int RC = 16;
static constexpr int SLOT = 2 * RC * RC;
static constexpr int NBLK_MAX = 296;      // 2 x 148 SMs
static constexpr int MAXD = 30;
static constexpr int RS_XF = 10;          // compact rank capacity of the transform kernels
static constexpr int RS_BIG = 16;         // ... of the large-capacity variant (Rhat up to 16)
static constexpr int RH_MAX = 8;          // Rhat cap of the one-CTA Hadamard rounding (hround.cu)
static constexpr int RH_BIG = 16;         // ... of the multi-CTA variant (hround_big.cu)

// ---------------------------------------------------------------- TT-SVD
struct DecProb {
  const double* x;   // input array (caller layout; a shard's sub-array when sharded)
  int layout, bx, d; // bx: bits of the row stride of x; d: global number of modes
  int dl;            // QTT bits held in x (d - log2 P for a shard, else d)
  double* gsum;      // reduced Gram (1024 doubles) when the Gram is combined across shards
  double* Wa;        // ping-pong unfolding buffers
  double* Wb;
  double* part;      // per-CTA partial Grams [NBLK_MAX][32*32]
  double* proj;      // current projector (<= 32 x 16, ld 32)
  double* tau2;      // per-cut threshold tau^2
  cplx* cores;       // d slots
  int* ranks;        // r_0..r_d
  double* psk;       // per-CTA partial sketches Y = A Omega [NBLK_MAX][32*32] (TT-RSVD)
  unsigned long long seed;   // Omega key of this tensor (TT-RSVD)
};
struct DecParams {
  double eps;
  int rmax;
  double ctol;
  int* status;
  int rule;          // 0: RANK (eps / rmax), 1: SV drop-off (delta), 2: RANK + TT-RSVD
  double delta;
  int kp;            // TT-RSVD sketch width k + p = rmax + p (0: plain SVD steps)
};
cudaError_t setup_ttsvd_kernels();
cudaError_t launch_ttsvd(const DecProb* probs_dev, int nprob, int d, DecParams prm, cudaStream_t st,
                         int reserve = 0);

// Column-sharded TT-SVD: the steps, launched one by one by the
// host driver in api.cu, which inserts the cross-rank collectives.  `sh`
// holds ntens * nlocal shard descriptors (tensor-major), `tn` ntens tensor
// descriptors; shards of a tensor share its cores / ranks / proj / tau2 /
// gsum.  nblk == 0 in a solve step means "read the reduced Gram gsum".
int dec_nblk_loc(int dl, int nprob);                        // CTAs per problem, level-1 Gram pass
int proj_nblk(int ncols, int nprob);                        // CTAs per problem, projection pass
static constexpr int FIN_COLS_HOST = 256;                   // finisher: W columns it holds
cudaError_t launch_level_gram(const DecProb* sh, int nsh, int nblk, int* status, cudaStream_t st);
cudaError_t launch_gram_reduce(const DecProb* sh, int ntens, int nlocal, int nblk, cudaStream_t st);
// nsk: number of per-CTA partial TT-RSVD sketches to sum (0 = none)
cudaError_t launch_level_solve(const DecProb* tn, int ntens, int nblk, DecParams prm, cudaStream_t st, int nsk = 0);
cudaError_t launch_step_solve(const DecProb* tn, int ntens, int k, int nblk, DecParams prm, cudaStream_t st,
                              int nsk = 0);
cudaError_t launch_project(bool from_x, const DecProb* pr, int nprob, int k, int nblk, int src_is_a,
                           cudaStream_t st);
cudaError_t launch_finish(const DecProb* tn, int ntens, int k, int src_is_a, DecParams prm, cudaStream_t st);
// W_{k} of every shard (r_k x nl local columns, in the shard's src buffer)
// -> tn.Wa (r_k x nl*nshards, shard-major columns).  Local shards: read
// directly (gathered = nullptr); after an all-gather: from `gathered`
// (ntens blocks of nshards x RS_GATHER*nl doubles).
static constexpr int RS_GATHER = 10;
static constexpr int SHARD_MIN_DL = 12;   // a shard holds >= 2^12 elements (one Gram chunk)
cudaError_t launch_gather_w(const DecProb* sh, const DecProb* tn, int ntens, int nlocal, int k, long long nl,
                            int src_is_a, const double* gathered, int nshards, cudaStream_t st);

// ------------------------------------------------------------- transforms
struct XfProb {
  const cplx* in_cores;
  const int* in_ranks;
  cplx* out_cores;
  int* out_ranks;
  cplx* gr;          // right-Gram scratch: MAXD slots of (2 rs)^2 (xf_gr_slot)
  int do_center;     // multiply the forward output by the centering phase (O3)
  cplx* cwork;       // rs = RS_BIG only: MAXD compact cores of 2 RS_BIG^2
};
struct XfParams {
  int d;
  int bits[2];
  int axis[MAXD];
  int bit[MAXD];
  double eps;
  int rmax;
  double ctol;
  int inverse;       // conj in / conj out
  double scale;      // multiplies core 1 of the output
  long long shift[2];
  int* status;
  int rule;
  double delta;
  int rs;            // rank capacity variant: RS_XF or RS_BIG
};
static constexpr int GR_XF = 4 * RS_XF * RS_XF;   // complex per GR slot (rs = RS_XF)
size_t xf_gr_slot(int rs);                        // complex per GR slot of a variant
cudaError_t setup_xf_kernels();
cudaError_t launch_transform(const XfProb* probs_dev, int nprob, const XfParams& prm, cudaStream_t st);

// ------------------------------------------------- Hadamard + TT-rounding
struct HrProb {
  const cplx* f_cores;
  const int* f_ranks;
  const cplx* g_cores;
  const int* g_ranks;
  cplx* out_cores;
  int* out_ranks;
  cplx* gr;          // MAXD slots of 64 x 64
};
struct HrParams {
  int d;
  double eps;
  int rmax;
  double ctol;
  int* status;
  int rule;
  double delta;
  int gr_ready;      // 1: pr.gr already holds the right-Gram chain (launch_hr_gr_chain)
};
static constexpr int GR_HR = 64 * 64;
cudaError_t setup_hr_kernels();
cudaError_t launch_hadamard_round(const HrProb* probs_dev, int nprob, const HrParams& prm, cudaStream_t st);

// Rhat up to RH_BIG: Kronecker ranks up to 256, scratch in the workspace
struct HrBigProb {
  const cplx* f_cores;
  const int* f_ranks;
  const cplx* g_cores;
  const int* g_ranks;
  cplx* out_cores;
  int* out_ranks;
  cplx* gr;          // d slots of 256 x 256 (right Grams of Z)
  cplx* t1;          // 2 slices x 256 x 256 each: mode-product intermediates
  cplx* t2;
  cplx* t3;
  cplx* e;           // E of the current cut: rows x rz (rows <= 32, rz <= 256)
  cplx* tb;          // T = E GR
  cplx* sm;          // U_r^H E
  cplx* hb;          // Sm x G
  int* st;           // sweep state (ranks, LQ bounds)
  double* tau2;
};
cudaError_t setup_hr_big_kernels();
size_t hr_big_scratch(int d);   // complex entries of gr + t1..t3 + e, tb, sm, hb
cudaError_t launch_hadamard_round_big(const HrBigProb* probs_dev, int nprob, const HrParams& prm, cudaStream_t st);
// right-Gram chain of Z = F (.) G into GR_HR slots (p.gr) for k_hadamard_round
// (HrParams::gr_ready = 1); uses f/g cores, ranks, gr, t1, t2, t3 of HrBigProb
cudaError_t launch_hr_gr_chain(const HrBigProb* probs_dev, int nprob, int d, cudaStream_t st);
// the same chain for ranks <= 8 (rz <= 64) as one launch of 8-CTA clusters
cudaError_t launch_hr_gr_chain_cluster(const HrBigProb* probs_dev, int nprob, int d, cudaStream_t st);

// -------------------------------------------------------------- expansion
struct ExProb {
  const cplx* cores;
  const int* ranks;
  double* y;         // output (caller layout)
  double* lsplit;    // 256 x 32 scratch (column-major, ld 256)
};
struct ExParams {
  int d;
  int layout;
  int bx;
  int imag;          // 0: y = Re(full), 1: y = Im(full)
  int rcap;          // upper bound of the ranks (selects the kernel variant)
};
cudaError_t setup_expand_kernels();
cudaError_t launch_expand(const ExProb* probs_dev, int nprob, const ExParams& prm, cudaStream_t st);

// Sharded expansion: the shard whose top l QTT bits equal
// `shard` is full(C_1 .. C_{d-l-1}, C_{d-l} v) with v = C_{d-l+1}[b_1] ..
// C_d[b_l]; k_fold_tail writes those d-l cores into out_cores/out_ranks.
struct FoldProb {
  const cplx* cores;
  const int* ranks;
  cplx* out_cores;   // (d - l) slots
  int* out_ranks;    // 64 ints
  int shard;
};
cudaError_t launch_fold_tail(const FoldProb* probs_dev, int nprob, int d, int l, cudaStream_t st);

}  // namespace qtt

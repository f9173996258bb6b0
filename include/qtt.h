/*
 * qtt.h — C ABI of libqtt.so: end-to-end QTT convolution on B200 (sm_100a).
 *
 * Implements the hot path of arXiv 2301.13339, Alg. 2 "QTT convolution"
 * (PAPER.md P:384-399):
 *   Step 1  reshape the full arrays to 2 x ... x 2 tensors
 *   Step 2  max-rank TT-SVD of signal and kernel                  (Alg. 1,
 *           P:275-293, modification (1) P:357-358)
 *   Step 3  QiFFT( QFFT(F) (.) QFFT(G) ) with capped ranks        (P:395,
 *           P:309-321), TT-rounding after the Hadamard product
 *   Step 4  Full                                                   (Alg. 3,
 *           P:408-424)
 * Readings of passages the paper leaves open are listed in DESIGN.md §3
 * (Q1-Q29); the same readings are implemented by the CPU oracle (oracle/).
 *
 * Conventions shared by every call
 *   - Pointers are DEVICE pointers unless the name ends in _host.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream).  Calls do not synchronise the
 *     host unless documented ("syncs").  qtt_conv_full on one image forks
 *     the decomposition of g onto a library-owned non-blocking stream of the
 *     current device and joins it back with events before Step 3, so all
 *     of its work stays ordered after earlier and before later work on
 *     `stream`.  The small per-call descriptor arrays reach the device
 *     through a kernel's parameters (no copy-engine or pageable copy on
 *     `stream`), so qtt_conv_full / qtt_decompose / qtt_convolve /
 *     qtt_to_full without a report can be captured in a CUDA graph on
 *     `stream` (the side-stream fork / join is captured with it; replays
 *     reuse the descriptors and workspace layout of the captured call, so the
 *     shape, policy, pointers and workspace must not change between
 *     replays).  Calls with `rep_host` synchronise and cannot be captured.
 *   - No call allocates device memory: all scratch and all device storage of
 *     TT handles is carved from the caller's workspace `ws` (>= the size
 *     returned by qtt_workspace_bytes, 256-byte aligned).  The workspace must
 *     stay alive and untouched while the handles carved from it are used.
 *   - Arrays are float64.  1D: x[i], i = 0..2^b-1.  2D: row-major image
 *     x[iy * 2^bx + ix] (x fastest).  QTT bit order is LSB first;
 *     the 2D mode order is the `layout` field (reading Q8).  Input arrays
 *     (f, g, x) and every batch entry must start on a 16-byte boundary (the
 *     TT-SVD streams them with 16-byte copies): a misaligned pointer or an
 *     odd batch stride is QTT_EINVAL.  Outputs (y) may have any 8-byte
 *     alignment and stride.
 *   - Truncation (reading Q1-Q6): per-cut threshold
 *     tau^2 = eps^2 ||A||_F^2 / (d-1), rank = min(rank_tau, rmax) moved out
 *     of clusters of relative width cluster_tol (Q6').
 *   - Errors: argument errors are reported synchronously (QTT_EINVAL).
 *     Numeric failures (non-finite input, eigensolver non-convergence) are
 *     latched in a device status word and returned by the next syncing call
 *     (qtt_wait, qtt_ranks, qtt_conv_full with a report) as QTT_ENUMERIC.
 *     CUDA errors -> QTT_ECUDA.  No C++ exception crosses the ABI.  The
 *     message of the last error of the calling thread is qtt_last_error().
 */
#ifndef QTT_H
#define QTT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QTT_OK = 0,
  QTT_EINVAL = 1,    /* bad argument (sizes, caps, layout, workspace)        */
  QTT_ENUMERIC = 2,  /* non-finite data or eigensolver failure (latched)     */
  QTT_ECUDA = 3,     /* CUDA runtime error                                   */
  QTT_ENCCL = 4,     /* collective failure (multi-GPU builds)                */
  QTT_ENOMEM = 5     /* workspace too small                                  */
} qtt_status;

typedef enum {
  QTT_LAYOUT_1D = 0,
  QTT_LAYOUT_INTERLEAVED = 1,  /* QTT position 2t-1 = x-bit t, 2t = y-bit t  */
  QTT_LAYOUT_CONCAT = 2        /* all x-bits, then all y-bits                */
} qtt_layout;

/* Problem shape.  D in {1,2}; bits[0] = bits of x (length 2^bits[0]),
 * bits[1] = bits of y (2D).  d = bits[0] (+ bits[1]) must lie in [2, 30].
 * Interleaved needs bits[0] == bits[1].  batch >= 1 independent signals;
 * f_stride / y_stride: elements between consecutive batch entries
 * (0 => 2^d); g_stride: 0 = one kernel shared by the whole batch. */
typedef struct {
  int D;
  int bits[2];
  int layout;
  int batch;
  long long f_stride, g_stride, y_stride;
} qtt_shape;

/* Truncation policy: eps >= 0, 1 <= rmax <= 16, cluster_tol >= 0.
 * Decomposition caps use rmax (R_max <= 16; <= 10 with a communicator or
 * for the sharded workspace query); transform/rounding caps Rhat
 * (<= 16; the paper's Rhat_max = 15).  Rhat <= 8 runs the
 * one-CTA Hadamard rounding, 9..16 the multi-CTA one (Kronecker ranks of
 * F (.) G up to 160 resp. 256).
 * rule = QTT_RULE_EPS (0): r = RANK(eps, rmax, cluster_tol) — modification
 *   (1), tau^2 = eps^2 ||A||^2 / (d-1);
 * rule = QTT_RULE_DROPOFF (1): SV drop-off, modification (3), P:363-365:
 *   keep sigma_1..sigma_k at the first k with sigma_{k+1}/sigma_k < delta
 *   (0 < delta < 1; no drop: keep sigma_k >= 1e-7 sigma_1), then the
 *   capacity cap rmax (a cap inside a cluster moves down); eps unused.
 *   The paper uses the same delta for the TT-SVD and the QTT-FFT. */
enum { QTT_RULE_EPS = 0, QTT_RULE_DROPOFF = 1, QTT_RULE_RSVD = 2 };
/* rule = QTT_RULE_RSVD (2), decomposition only: RANK as rule 0, but every
 *   TT-SVD step whose unfolding has min(m, n) > rmax + p uses the
 *   randomized SVD of Appendix A (modification (2)):
 *   Y = A Omega with Omega (n x (rmax + p)) ~ N(0,1) from the counter-based
 *   generator of DESIGN.md §3 (key seed + t for tensor t of a call: the f
 *   batch entries 0..B-1, then g), range(Y) -> Rayleigh-Ritz.  Requires
 *   8 <= rmax + p <= 16 and no communicator.  The QTT-FFT / rounding keep
 *   rule 0 or 1 (reading N2). */
typedef struct {
  double eps;
  int rmax;
  double cluster_tol;
  int rule;
  double delta;
  int p;                     /* TT-RSVD oversampling */
  unsigned long long seed;   /* TT-RSVD generator key */
} qtt_trunc;

typedef struct qtt_tt_s* qtt_tt_t;      /* opaque TT tensor (batch of them)  */
typedef struct qtt_comm_s* qtt_comm_t;  /* NULL = single GPU                 */

/* Optional report of qtt_conv_full (host struct, filled when non-NULL;
 * filling it syncs the stream).  ranks_*: r_0..r_d of batch entry 0 of the
 * signal TT-SVD (f), the kernel TT-SVD (g), their QTT-FFTs (fh, gh), the
 * rounded Hadamard product (z) and the output (out, after the QTT-iFFT).
 * min_margin / min_gap: T2 well-posedness evidence over
 * every eps-rule truncation of the call (all batch entries): the smallest
 * |T - tau^2| / tau^2 of a deciding tail sum T (T(r_tau) and T(r_tau - 1)
 * when eps decides, T(R) when the cap does) and the smallest
 * (lambda_r - lambda_{r+1}) / lambda_1 at a chosen rank r < m; a Gram
 * eigenvalue carries ~1e3 m eps_mach lambda_1 of absolute noise, so a margin
 * far above that is a rank decision the SVD oracle takes identically.
 * Both are +inf when nothing was recorded (eps = 0, drop-off rule). */
typedef struct {
  int d;
  int ranks_f[64], ranks_g[64], ranks_fh[64], ranks_gh[64], ranks_z[64],
      ranks_out[64];
  float ms_total;
  int status_bits;   /* device status word: 1 non-finite input, 2 eigensolver
                        failure (both errors), 16 = a tridiagonal eigensolve
                        fell back to Jacobi (information) */
  double min_margin;
  double min_gap;
} qtt_report;

/* Bytes of workspace needed by qtt_conv_full (and enough for any single
 * qtt_decompose / qtt_convolve / qtt_to_full of the same shape and caps).
 * Returns 0 for invalid arguments.  nranks = 1: single GPU (also enough for
 * a 1-rank communicator); nranks = P > 1: per-rank bytes of the P-way
 * column-sharded problem (one shard per rank, see "Multi-GPU" below). */
size_t qtt_workspace_bytes(const qtt_shape* shape, const qtt_trunc* dec,
                           const qtt_trunc* fft, int nranks);
/* Same, for the shards `comm` places in this process (comm may be NULL). */
size_t qtt_comm_workspace_bytes(const qtt_shape* shape, const qtt_trunc* dec,
                                const qtt_trunc* fft, qtt_comm_t comm);

/* Step 1-2: max-rank TT-SVD (Alg. 1 + mod (1)) of the batch of
 * arrays x (shape->batch of them, stride shape->f_stride).  Writes a new
 * handle to *out whose device storage lives in ws.  With comm != NULL, x is
 * this process's shard(s) of the single (batch 1) global array and the
 * handle holds the global cores, identical on every rank. */
qtt_status qtt_decompose(const double* x, const qtt_shape* shape,
                         const qtt_trunc* dec, void* ws, size_t ws_bytes,
                         void* stream, qtt_comm_t comm, qtt_tt_t* out);

/* QTT-FFT (inverse = 0) or QTT-iFFT (inverse = 1) of every tensor of `in`
 * (capped P:370-382).  Forward output is the bit-reversed layout
 * of SURVEY §8(c) O2; if shift != NULL the forward output is multiplied by
 * the centering phase of shift (O3); the inverse output is scaled by
 * scale * 2^{-d}.  Test/diagnostic entry point of the Step-3 machinery. */
qtt_status qtt_transform(qtt_tt_t in, const qtt_trunc* fft, int inverse,
                         const long long shift[2], double scale, void* ws,
                         size_t ws_bytes, void* stream, qtt_tt_t* out);

/* Step 3: QiFFT(round(QFFT(f) (.) center(QFFT(g)))) scaled by
 * `scale` (= dx^D, eq. dconv).  g holds 1 tensor (shared) or as many
 * as f.  y_j = scale sum_i f_i g_{(j - i + shift) mod n} per axis. */
qtt_status qtt_convolve(qtt_tt_t f, qtt_tt_t g, const qtt_trunc* fft,
                        const long long shift[2], double scale, void* ws,
                        size_t ws_bytes, void* stream, qtt_tt_t* out);

/* Step 4 (Alg. 3): y = Re(full(t)) written in the caller layout
 * (batch stride y_stride of t's shape).  If y_imag != NULL the imaginary
 * part is written there too (diagnostics).  With comm != NULL only this
 * process's shard(s) of y are written (no communication). */
qtt_status qtt_to_full(qtt_tt_t t, double* y, double* y_imag, void* ws,
                       size_t ws_bytes, void* stream, qtt_comm_t comm);

/* Alg. 2 end to end: y = QTT convolution of f and g (Steps 1-4).  With
 * comm != NULL, f, g and y are this process's shards (batch 1). */
qtt_status qtt_conv_full(const double* f, const double* g, double* y,
                         const qtt_shape* shape, const qtt_trunc* dec,
                         const qtt_trunc* fft, const long long shift[2],
                         double scale, void* ws, size_t ws_bytes,
                         void* stream, qtt_comm_t comm,
                         qtt_report* rep_host);

/* Syncs; returns the latched numeric status of the handle's stream work. */
qtt_status qtt_wait(qtt_tt_t t);
/* Syncs; copies r_0..r_d of batch entry `index` into ranks_host (cap >= d+1). */
qtt_status qtt_ranks(qtt_tt_t t, int index, int* ranks_host, int cap);
/* Number of modes d of the handle's tensors (host only). */
int qtt_ndims(qtt_tt_t t);
/* Releases the host handle (device storage belongs to the workspace). */
void qtt_destroy(qtt_tt_t t);

/* ------------------------------------------------------------ Multi-GPU
 * Column sharding of the TT-SVD unfoldings (north star
 * "the column dimension of each unfolding is sharded over GPUs, and the tiny
 * Gram matrices are combined with an NCCL allreduce"):
 *   - P = 2^l shards.  Shard s holds the QTT index range
 *     [s 2^{d-l}, (s+1) 2^{d-l}), i.e. the elements whose top l QTT bits
 *     equal s; it is stored as a dense row-major sub-image (1D: a contiguous
 *     range; concat: a block of rows; interleaved: P=2 row halves, P=4
 *     quadrants, ...), see qtt_shard_geometry.  d - l >= 12 is required.
 *   - Alg. 1 steps k <= d - l: every column of the k-th unfolding lies in
 *     one shard, so its Gram is the sum of the shards' Grams (one
 *     ncclAllReduce of f's and g's Grams per step); the projection is local.
 *     When a shard's unfolding gets narrower than 256 columns the small
 *     remainder W is all-gathered and the last steps, the QTT-FFT chain and
 *     the rounding run redundantly (bitwise identical) on every rank.
 *   - Expansion: shard s = full(C_1, ..., C_{d-l} C_{d-l+1}[s_1] ...
 *     C_d[s_l]) — no communication.
 *   Results differ from the single-GPU path only by summation order. */

/* Rank 0 creates the NCCL unique id and broadcasts it (e.g. with
 * torch.distributed); every rank then calls qtt_comm_init with its rank, the
 * CUDA device of the rank current.  NCCL is loaded at run time (the one
 * already in the process, else libnccl.so.2): QTT_ENCCL if unavailable.
 * nranks must be a power of two; rank r holds shard r. */
qtt_status qtt_comm_unique_id(unsigned char id_host[128]);
qtt_status qtt_comm_init(const unsigned char id_host[128], int nranks, int rank,
                         qtt_comm_t* out);
/* TEST-ONLY: a communicator under which THIS process holds all nshards
 * shards on one GPU (shard j at element offset j 2^{d-l} of the f / g / y
 * pointers); the cross-shard Gram sums run as a kernel.  Lets one GPU run
 * the sharded algorithm without ranks that wait on each other. */
qtt_status qtt_comm_init_virtual(int nshards, qtt_comm_t* out);
void qtt_comm_destroy(qtt_comm_t comm);
/* Host only: where shard `shard` of nshards sits in the global array
 * (origin_host = {x0, y0}) and its size in bits (bits_host = {bx, by};
 * 1D: {bits, 0}).  QTT_EINVAL for invalid shapes / shard counts. */
qtt_status qtt_shard_geometry(const qtt_shape* shape, int nshards, int shard,
                              long long origin_host[2], int bits_host[2]);

/* TEST-ONLY: Hermitian eigendecomposition of the n x n (n <= 32) complex
 * matrix A (device, column-major interleaved re/im doubles) by the small
 * eigensolver every truncation of the path uses (mode 0: tridiagonal solver
 * with Jacobi fallback, all n vectors; mode 1: Jacobi only; mode m >= 2: the
 * production solver asked for the m-1 leading vectors only, as the
 * truncations do).  lam (device, n): eigenvalues in
 * descending order; U (device, n x n complex): eigenvectors; sweeps (device,
 * >= 2 ints): Jacobi sweeps, fallbacks taken; reps: repeat count (timing).
 * Stream-ordered. */
int qtt_debug_eigh(const void* A, int n, double* lam, void* U, int* sweeps, int reps, int mode,
                   void* stream);

/* TEST-ONLY: rows j0 .. j0+n-1 of the TT-RSVD test matrix Omega_k (step k,
 * key seed) as a row-major n x kp device array, so tests can compare the
 * generator with the oracle's (oracle/rng.py).  Stream-ordered. */
int qtt_debug_omega(unsigned long long seed, int k, unsigned long long j0, int n, int kp, double* out,
                    void* stream);

/* TEST-ONLY: build a handle from host cores (shape->batch tensors; tensor i,
 * core k occupies the slot of 512 complex starting at ((i*d)+k)*512, compact
 * column-major (r_{k-1}, 2, r_k); ranks_host: 64 ints per tensor).  Syncs.
 * Lets a test run one stage of the GPU path on a known input. */
qtt_status qtt_debug_tt_from_host(const qtt_shape* shape, const void* cores_host,
                                  const int* ranks_host, int rcap, void* ws,
                                  size_t ws_bytes, void* stream, qtt_tt_t* out);

/* Stage profiling of qtt_conv_full: when enabled, CUDA events are recorded
 * on the call's stream at the stage boundaries.  qtt_profile_read syncs on
 * the last call's final event and writes n >= 5 stage times (ms): [0] TT-SVD
 * of f and g, [1] forward QTT-FFTs, [2] Hadamard + rounding, [3] QTT-iFFT,
 * [4] expansion; returns the number written (0 if nothing was recorded). */
void qtt_profile_enable(int on);
int qtt_profile_read(float* ms_host, int n);
/* Total number of kernels this library has launched in the process. */
long long qtt_launch_count(void);

const char* qtt_status_string(qtt_status s);
const char* qtt_last_error(void);   /* thread-local, never NULL */
const char* qtt_build_info(void);   /* arch, compile flags */

#ifdef __cplusplus
}
#endif
#endif /* QTT_H */

// api.cu — the C ABI of libqtt.so (include/qtt.h): argument validation,
// workspace carving and the launch sequence of Alg. 2.
// Every compute step runs in the kernels of ttsvd.cu, qfft.cu, hround.cu and
// expand.cu; this file only marshals pointers.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: the library is dlopen'ed at qtt_comm_init

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qtt.h"
#include "qtt_kernels.h"

using namespace qtt;

namespace {
extern int g_prof;
void prof_pass_impl(int pass, int end, cudaStream_t st);
}
namespace qtt {
static std::atomic<long long> g_launches{0};
void prof_pass(int pass, int end, cudaStream_t st) { prof_pass_impl(pass, end, st); }
void count_launches(int n) { g_launches += n; }
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cache[dev].load();
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v);
  }
  return v;
}
// One non-blocking side stream per device: the f and g decompositions of a
// single-image convolution run as two chains, so the one-CTA solves of one
// overlap the HBM passes of the other.
cudaStream_t side_stream() {
  static std::mutex mu;
  static cudaStream_t cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!cache[dev] && cudaStreamCreateWithFlags(&cache[dev], cudaStreamNonBlocking) != cudaSuccess)
    cache[dev] = nullptr;
  return cache[dev];
}
}  // namespace qtt

#define QTT_XSTR(x) #x
#define QTT_STR(x) QTT_XSTR(x)

// Communicator of the column-sharded path.  NCCL: one shard
// per rank (shard = rank).  Virtual: all nshards shards live in this process
// on one GPU (test / single-GPU emulation of the sharded algorithm; the
// cross-shard sums are done by a kernel instead of a collective).
struct qtt_comm_s {
  int kind;        // 0 = NCCL, 1 = virtual
  int nranks, rank;
  int nshards;     // P (total shards)
  int nlocal;      // shards held by this process
  ncclComm_t nc;
  ncclComm_t nc2;  // second communicator (ncclCommSplit of nc) for the g chain; null: one chain
};

struct qtt_tt_s {
  qtt_shape shape;
  int d;
  int nt;          // tensors in the handle
  int rcap;        // max rank stored
  cplx* cores;     // nt * d * SLOT
  int* ranks;      // nt * 64
  int* status;     // device status word
  cudaStream_t stream;
};

namespace {

thread_local std::string g_err = "";

qtt_status fail(qtt_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

qtt_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return QTT_OK;
  return fail(QTT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ---- optional stage profiling (CUDA events on the caller's stream)
enum { PROF_STAGES = 5, PROF_MARKS = PROF_STAGES + 1 };
int g_prof = 0;
cudaEvent_t g_ev[PROF_MARKS] = {};
int g_ev_ok = 0;
void prof_mark(int i, cudaStream_t st) {
  if (!g_prof) return;
  if (!g_ev_ok) {
    for (int k = 0; k < PROF_MARKS; ++k) cudaEventCreate(&g_ev[k]);
    g_ev_ok = 1;
  }
  cudaEventRecord(g_ev[i], st);
}
cudaEvent_t g_pev[PASS_N][2] = {};
int g_pev_ok = 0;
int g_pev_set[PASS_N] = {};

// level 2: events around the first full-array passes of the call (the
// decomposition then runs as one chain on the caller's stream, so a pass's
// events bracket that pass alone)
void prof_pass_impl(int pass, int end, cudaStream_t st) {
  if (g_prof < 2 || pass < 0 || pass >= PASS_N) return;
  if (!g_pev_ok) {
    for (int k = 0; k < PASS_N; ++k) {
      cudaEventCreate(&g_pev[k][0]);
      cudaEventCreate(&g_pev[k][1]);
    }
    g_pev_ok = 1;
  }
  cudaEventRecord(g_pev[pass][end], st);
  if (end) g_pev_set[pass] = 1;
}

// cudaFuncSetAttribute (dynamic shared memory above 48 KB) is per device
// context: done once per device, retried after a failure
std::mutex g_setup_mu;
bool g_setup_done[64] = {};

cudaError_t setup_all() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_setup_mu);
  if (g_setup_done[dev]) return cudaSuccess;
  if ((e = setup_ttsvd_kernels()) != cudaSuccess) return e;
  if ((e = setup_xf_kernels()) != cudaSuccess) return e;
  if ((e = setup_hr_kernels()) != cudaSuccess) return e;
  if ((e = setup_hr_big_kernels()) != cudaSuccess) return e;
  if ((e = setup_expand_kernels()) != cudaSuccess) return e;
  g_setup_done[dev] = true;
  return cudaSuccess;
}

// events owned by one call, destroyed on every exit path
struct EventGuard {
  cudaEvent_t ev[4] = {};
  int n = 0;
  cudaError_t make(cudaEvent_t* out, unsigned flags) {
    cudaError_t e = cudaEventCreateWithFlags(out, flags);
    if (e == cudaSuccess) ev[n++] = *out;
    return e;
  }
  ~EventGuard() {
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
  }
};

// The TT-SVD chunk loaders read the inputs with 16-byte cp.async copies
// (ttsvd.cu load_chunk_async): every array (and every batch entry) must
// start on a 16-byte boundary.
// Descriptor upload without the copy engine: the (small) host descriptor
// arrays go to device memory through a kernel whose parameter carries the
// bytes.  A cudaMemcpyAsync here would queue behind whatever the copy engine
// is moving for the caller (e.g. the next step's inputs on a copy stream) and
// stall the compute stream; it would also be a pageable copy, which cannot be
// captured in a CUDA graph.
struct DescChunk {
  unsigned int n;
  unsigned char b[2044];
};
__global__ void k_store_desc(unsigned char* dst, const DescChunk c) {
  for (unsigned int i = threadIdx.x; i < c.n; i += blockDim.x) dst[i] = c.b[i];
}
cudaError_t upload_desc(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  const unsigned char* sp = static_cast<const unsigned char*>(src);
  unsigned char* dp = static_cast<unsigned char*>(dst);
  for (size_t off = 0; off < bytes; off += sizeof(DescChunk::b)) {
    DescChunk c;
    c.n = (unsigned int)((bytes - off) < sizeof(c.b) ? (bytes - off) : sizeof(c.b));
    memcpy(c.b, sp + off, c.n);
    k_store_desc<<<1, 128, 0, st>>>(dp + off, c);
    count_launches(1);
  }
  return cudaGetLastError();
}

qtt_status check_input_align(const double* x, long long stride, int n, const char* which) {
  if (((uintptr_t)x & 15) != 0) return fail(QTT_EINVAL, "%s must be 16-byte aligned", which);
  if (n > 1 && (stride & 1)) return fail(QTT_EINVAL, "%s batch stride must be even (16-byte aligned entries)", which);
  return QTT_OK;
}

// bump allocator over the caller's workspace (dry run when base == nullptr)
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base((char*)b) {}
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

int shape_d(const qtt_shape* s) { return s->D == 1 ? s->bits[0] : s->bits[0] + s->bits[1]; }

qtt_status check_shape(const qtt_shape* s) {
  if (!s) return fail(QTT_EINVAL, "shape is NULL");
  if (s->D != 1 && s->D != 2) return fail(QTT_EINVAL, "D must be 1 or 2 (got %d)", s->D);
  if (s->bits[0] < 1 || (s->D == 2 && s->bits[1] < 1)) return fail(QTT_EINVAL, "bits must be >= 1");
  const int d = shape_d(s);
  if (d < 2 || d > MAXD) return fail(QTT_EINVAL, "d = %d outside [2, %d]", d, MAXD);
  if (s->D == 1 && s->layout != QTT_LAYOUT_1D) return fail(QTT_EINVAL, "1D problems need QTT_LAYOUT_1D");
  if (s->D == 2 && s->layout != QTT_LAYOUT_INTERLEAVED && s->layout != QTT_LAYOUT_CONCAT)
    return fail(QTT_EINVAL, "2D problems need the interleaved or concat layout");
  if (s->D == 2 && s->layout == QTT_LAYOUT_INTERLEAVED && s->bits[0] != s->bits[1])
    return fail(QTT_EINVAL, "interleaved layout needs bits[0] == bits[1]");
  if (s->D == 2 && s->bits[0] != s->bits[1])
    return fail(QTT_EINVAL, "the QTT-FFT slot swap needs a square grid (bits[0] == bits[1])");
  if (s->batch < 1) return fail(QTT_EINVAL, "batch must be >= 1");
  if (s->f_stride < 0 || s->g_stride < 0 || s->y_stride < 0) return fail(QTT_EINVAL, "negative stride");
  return QTT_OK;
}

qtt_status check_trunc(const qtt_trunc* t, int rmax_cap, const char* which, bool allow_rsvd = false) {
  if (!t) return fail(QTT_EINVAL, "%s truncation is NULL", which);
  if (!(t->eps >= 0.0)) return fail(QTT_EINVAL, "%s eps must be >= 0", which);
  if (t->rmax < 1 || t->rmax > rmax_cap)
    return fail(QTT_EINVAL, "%s rmax = %d outside [1, %d]", which, t->rmax, rmax_cap);
  if (!(t->cluster_tol >= 0.0)) return fail(QTT_EINVAL, "%s cluster_tol must be >= 0", which);
  if (t->rule != QTT_RULE_EPS && t->rule != QTT_RULE_DROPOFF && !(allow_rsvd && t->rule == QTT_RULE_RSVD))
    return fail(QTT_EINVAL, "%s rule = %d is not allowed here", which, t->rule);
  if (t->rule == QTT_RULE_RSVD && !(t->p >= 0 && t->rmax + t->p >= 8 && t->rmax + t->p <= 16))
    return fail(QTT_EINVAL, "%s TT-RSVD needs p >= 0 and 8 <= rmax + p <= 16", which);
  if (t->rule == QTT_RULE_DROPOFF && !(t->delta > 0.0 && t->delta < 1.0))
    return fail(QTT_EINVAL, "%s drop-off delta must lie in (0, 1)", which);
  return QTT_OK;
}

void axes_of(const qtt_shape* s, int* axis, int* bit) {
  const int d = shape_d(s);
  if (s->D == 1) {
    for (int p = 0; p < d; ++p) { axis[p] = 0; bit[p] = p + 1; }
  } else if (s->layout == QTT_LAYOUT_INTERLEAVED) {
    for (int t = 0; t < s->bits[0]; ++t) {
      axis[2 * t] = 0; bit[2 * t] = t + 1;
      axis[2 * t + 1] = 1; bit[2 * t + 1] = t + 1;
    }
  } else {
    for (int t = 0; t < s->bits[0]; ++t) { axis[t] = 0; bit[t] = t + 1; }
    for (int t = 0; t < s->bits[1]; ++t) { axis[s->bits[0] + t] = 1; bit[s->bits[0] + t] = t + 1; }
  }
}

DecParams dec_params(const qtt_trunc* dec, int* status) {
  DecParams prm{};
  prm.eps = dec->eps;
  prm.rmax = dec->rmax;
  prm.ctol = dec->cluster_tol;
  prm.status = status;
  prm.rule = dec->rule == QTT_RULE_RSVD ? QTT_RULE_EPS : dec->rule;
  prm.delta = dec->delta;
  prm.kp = dec->rule == QTT_RULE_RSVD ? dec->rmax + dec->p : 0;
  return prm;
}

struct TTAlloc {
  cplx* cores;
  int* ranks;
};
TTAlloc take_tt(Carver& cv, int nt, int d) {
  TTAlloc t;
  t.cores = cv.take<cplx>((size_t)nt * d * SLOT);
  t.ranks = cv.take<int>((size_t)nt * 64);
  return t;
}

struct DecScratch {
  double* Wa;
  double* Wb;
  double* part;
  double* proj;
  double* tau2;
  double* psk;
  double* gsum;
};
DecScratch take_dec(Carver& cv, int d, bool rsvd = false) {
  DecScratch s{};
  if (d > 12) {
    s.Wa = cv.take<double>((size_t)RC << (d - 5));
    s.Wb = cv.take<double>((size_t)RC << (d - 6));
    s.part = cv.take<double>((size_t)NBLK_MAX * 1024);
    if (rsvd) s.psk = cv.take<double>((size_t)NBLK_MAX * 1024);
  } else {
    s.Wa = s.Wb = s.part = nullptr;
  }
  s.proj = cv.take<double>(32 * 16);
  s.tau2 = cv.take<double>(1);
  s.gsum = cv.take<double>(1024);
  return s;
}

qtt_tt_t new_handle(const qtt_shape* shape, int nt, int rcap, TTAlloc a, int* status, cudaStream_t st) {
  qtt_tt_t h = new (std::nothrow) qtt_tt_s;
  if (!h) return nullptr;
  h->shape = *shape;
  h->d = shape_d(shape);
  h->nt = nt;
  h->rcap = rcap;
  h->cores = a.cores;
  h->ranks = a.ranks;
  h->status = status;
  h->stream = st;
  return h;
}

// ---------------------------------------------------------------- stages
// TT-SVD of n arrays x_i = base + i*stride into tt (n tensors)
qtt_status run_decompose(const double* base, long long stride, int n, const qtt_shape* s,
                         const qtt_trunc* dec, TTAlloc tt, Carver& cv, int* status, cudaStream_t st) {
  const int d = shape_d(s);
  std::vector<DecProb> h(n);
  const bool rsvd = dec->rule == QTT_RULE_RSVD;
  for (int i = 0; i < n; ++i) {
    DecScratch sc = take_dec(cv, d, rsvd);
    DecProb& p = h[i];
    p.x = base + (size_t)i * (size_t)stride;
    p.layout = s->layout;
    p.bx = s->bits[0];
    p.d = d;
    p.dl = d;
    p.gsum = sc.gsum;
    p.Wa = sc.Wa; p.Wb = sc.Wb; p.part = sc.part; p.proj = sc.proj; p.tau2 = sc.tau2;
    p.cores = tt.cores + (size_t)i * d * SLOT;
    p.ranks = tt.ranks + (size_t)i * 64;
    p.psk = sc.psk;
    p.seed = dec->seed + (unsigned long long)i;
  }
  DecProb* dp = cv.take<DecProb>(n);
  if (!cv.base) return QTT_OK;
  qtt_status r;
  if ((r = cuda_check(upload_desc(dp, h.data(), n * sizeof(DecProb), st),
                      "copy descriptors")))
    return r;
  DecParams prm = dec_params(dec, status);
  return cuda_check(launch_ttsvd(dp, n, d, prm, st), "TT-SVD launch");
}

qtt_status run_transform(const std::vector<XfProb>& hv, const qtt_shape* s, const qtt_trunc* fft, int inverse,
                         const long long* shift, double scale, Carver& cv, int* status, cudaStream_t st,
                         int rs = RS_XF) {
  const int n = (int)hv.size();
  XfProb* dp = cv.take<XfProb>(n);
  if (!cv.base) return QTT_OK;
  XfParams P{};
  P.d = shape_d(s);
  P.bits[0] = s->bits[0];
  P.bits[1] = s->D == 2 ? s->bits[1] : 0;
  axes_of(s, P.axis, P.bit);
  P.eps = fft->eps;
  P.rmax = fft->rmax;
  P.ctol = fft->cluster_tol;
  P.rule = fft->rule;
  P.delta = fft->delta;
  P.rs = rs;
  P.inverse = inverse;
  P.scale = inverse ? scale * ldexp(1.0, -P.d) : 1.0;
  P.shift[0] = shift ? shift[0] : 0;
  P.shift[1] = (shift && s->D == 2) ? shift[1] : 0;
  P.status = status;
  qtt_status r;
  if ((r = cuda_check(upload_desc(dp, hv.data(), n * sizeof(XfProb), st),
                      "copy descriptors")))
    return r;
  return cuda_check(launch_transform(dp, n, P, st), "transform launch");
}

qtt_status run_expand(const cplx* cores, const int* ranks, int nt, int d, double* y, long long ystride,
                      const qtt_shape* s, int imag, Carver& cv, cudaStream_t st, int rcap = RC) {
  std::vector<ExProb> h(nt);
  for (int i = 0; i < nt; ++i) {
    h[i].cores = cores + (size_t)i * d * SLOT;
    h[i].ranks = ranks + (size_t)i * 64;
    h[i].y = y + (size_t)i * (size_t)ystride;
    h[i].lsplit = cv.take<double>(256 * 32);
  }
  ExProb* dp = cv.take<ExProb>(nt);
  if (!cv.base) return QTT_OK;
  ExParams P{d, s->layout, s->bits[0], imag, rcap};
  qtt_status r;
  if ((r = cuda_check(upload_desc(dp, h.data(), nt * sizeof(ExProb), st),
                      "copy descriptors")))
    return r;
  return cuda_check(launch_expand(dp, nt, P, st), "expand launch");
}

// Step 3 on handles' storage: F (nf tensors), G (ng = 1 or nf) -> Y (nf)
qtt_status run_convolve(const cplx* fc, const int* fr, int nf, const cplx* gc, const int* gr, int ng,
                        const qtt_shape* s, const qtt_trunc* fft, const long long* shift, double scale,
                        TTAlloc Y, Carver& cv, int* status, cudaStream_t st, int in_rcap,
                        TTAlloc* stages_out = nullptr) {
  const int d = shape_d(s);
  // Rhat <= RH_MAX: one-CTA rounding; above: the multi-CTA variant (Kronecker ranks <= 256)
  const bool big = fft->rmax > RH_MAX;
  // transform variant: compact cores in shared memory while every rank fits RS_XF
  const int rs = (fft->rmax > RS_XF || in_rcap > RS_XF) ? RS_BIG : RS_XF;
  TTAlloc Fh = take_tt(cv, nf, d);
  TTAlloc Gh = take_tt(cv, ng, d);
  TTAlloc Z = take_tt(cv, nf, d);
  if (stages_out) { stages_out[0] = Fh; stages_out[1] = Gh; stages_out[2] = Z; }
  std::vector<XfProb> fw(nf + ng);
  for (int i = 0; i < nf + ng; ++i) {
    const bool isf = i < nf;
    const int j = isf ? i : i - nf;
    XfProb& p = fw[i];
    p.in_cores = (isf ? fc : gc) + (size_t)j * d * SLOT;
    p.in_ranks = (isf ? fr : gr) + (size_t)j * 64;
    p.out_cores = (isf ? Fh.cores : Gh.cores) + (size_t)j * d * SLOT;
    p.out_ranks = (isf ? Fh.ranks : Gh.ranks) + (size_t)j * 64;
    p.gr = cv.take<cplx>((size_t)MAXD * xf_gr_slot(rs));
    p.cwork = rs == RS_BIG ? cv.take<cplx>((size_t)MAXD * 2 * RS_BIG * RS_BIG) : nullptr;
    p.do_center = (!isf && shift) ? 1 : 0;   // center the kernel's spectrum only (O3)
  }
  // forward transforms of all F's and G's: one launch, one CTA each
  qtt_status r;
  if ((r = run_transform(fw, s, fft, 0, shift, 1.0, cv, status, st, rs))) return r;
  if (cv.base) prof_mark(2, st);
  std::vector<HrProb> hr(big ? 0 : nf);
  std::vector<HrBigProb> hb(big ? nf : 0);
  for (int i = 0; i < nf; ++i) {
    const int j = ng == 1 ? 0 : i;
    if (!big) {
      HrProb& p = hr[i];
      p.f_cores = Fh.cores + (size_t)i * d * SLOT;
      p.f_ranks = Fh.ranks + (size_t)i * 64;
      p.g_cores = Gh.cores + (size_t)j * d * SLOT;
      p.g_ranks = Gh.ranks + (size_t)j * 64;
      p.out_cores = Z.cores + (size_t)i * d * SLOT;
      p.out_ranks = Z.ranks + (size_t)i * 64;
      p.gr = cv.take<cplx>((size_t)MAXD * GR_HR);
      continue;
    }
    HrBigProb& p = hb[i];
    p.f_cores = Fh.cores + (size_t)i * d * SLOT;
    p.f_ranks = Fh.ranks + (size_t)i * 64;
    p.g_cores = Gh.cores + (size_t)j * d * SLOT;
    p.g_ranks = Gh.ranks + (size_t)j * 64;
    p.out_cores = Z.cores + (size_t)i * d * SLOT;
    p.out_ranks = Z.ranks + (size_t)i * 64;
    constexpr size_t Q2 = (size_t)RH_BIG * RH_BIG * RH_BIG * RH_BIG;   // 256 x 256
    constexpr size_t EW = (size_t)2 * RH_BIG * RH_BIG * RH_BIG;        // 32 x 256
    cplx* base = cv.take<cplx>(hr_big_scratch(d));
    p.gr = base;
    p.t1 = base + (size_t)d * Q2;
    p.t2 = p.t1 + 2 * Q2;
    p.t3 = p.t2 + 2 * Q2;
    p.e = p.t3 + 2 * Q2;
    p.tb = p.e + EW;
    p.sm = p.tb + EW;
    p.hb = p.sm + EW;
    p.st = cv.take<int>(128);
    p.tau2 = cv.take<double>(1);
  }
  HrProb* hp = big ? nullptr : cv.take<HrProb>(nf);
  HrBigProb* hbp = cv.take<HrBigProb>(nf);
  // multi-CTA chain for few long tensors (C2-C4: 1.04 -> 0.87 ms at d = 18);
  // a batch already fills the GPU with one CTA per tensor, and short chains
  // are launch-bound (C1 d = 12, C5 64 tensors: the in-CTA chain is faster)
  const bool gr_multi = !big && nf <= 8 && d >= 16;
  if (gr_multi) {
    // the one-CTA rounding's right-Gram chain runs as multi-CTA mode products
    // (launch_hr_gr_chain) into its GR slots
    for (int i = 0; i < nf; ++i) {
      HrBigProb& q = hb.emplace_back();
      q = HrBigProb{};
      q.f_cores = hr[i].f_cores;
      q.f_ranks = hr[i].f_ranks;
      q.g_cores = hr[i].g_cores;
      q.g_ranks = hr[i].g_ranks;
      q.gr = hr[i].gr;
      q.t1 = cv.take<cplx>((size_t)6 * GR_HR);
      q.t2 = q.t1 + 2 * GR_HR;
      q.t3 = q.t2 + 2 * GR_HR;
    }
  }
  std::vector<XfProb> iv(nf);
  for (int i = 0; i < nf; ++i) {
    XfProb& p = iv[i];
    p.in_cores = Z.cores + (size_t)i * d * SLOT;
    p.in_ranks = Z.ranks + (size_t)i * 64;
    p.out_cores = Y.cores + (size_t)i * d * SLOT;
    p.out_ranks = Y.ranks + (size_t)i * 64;
    p.gr = fw[i].gr;   // reuse the forward scratch
    p.cwork = fw[i].cwork;
    p.do_center = 0;
  }
  if (cv.base) {
    HrParams H{d, fft->eps, fft->rmax, fft->cluster_tol, status, fft->rule, fft->delta, gr_multi ? 1 : 0};
    if (big) {
      if ((r = cuda_check(upload_desc(hbp, hb.data(), nf * sizeof(HrBigProb), st),
                          "copy descriptors")))
        return r;
      if ((r = cuda_check(launch_hadamard_round_big(hbp, nf, H, st), "hadamard/round launch"))) return r;
    } else {
      if ((r = cuda_check(upload_desc(hp, hr.data(), nf * sizeof(HrProb), st),
                          "copy descriptors")))
        return r;
      if (gr_multi) {
        if ((r = cuda_check(upload_desc(hbp, hb.data(), nf * sizeof(HrBigProb), st),
                            "copy descriptors")))
          return r;
        if ((r = cuda_check(launch_hr_gr_chain_cluster(hbp, nf, d, st), "right-Gram chain launch"))) return r;
      }
      if ((r = cuda_check(launch_hadamard_round(hp, nf, H, st), "hadamard/round launch"))) return r;
    }
    prof_mark(3, st);
  }
  r = run_transform(iv, s, fft, 1, nullptr, scale, cv, status, st, rs);
  if (cv.base) prof_mark(4, st);
  return r;
}

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;   // optional (NCCL >= 2.18)
};

// The NCCL already loaded in the process (PyTorch's) is preferred; else the
// system one.  No link-time dependency: the library loads without NCCL.
NcclApi& nccl_api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) { a.err = "libnccl.so.2 not found"; return; }
    bool ok = true;
    auto sym = [&](const char* n) { void* p = dlsym(h, n); ok = ok && p; return p; };
    a.getUniqueId = (decltype(a.getUniqueId))sym("ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))sym("ncclCommInitRank");
    a.commDestroy = (decltype(a.commDestroy))sym("ncclCommDestroy");
    a.allReduce = (decltype(a.allReduce))sym("ncclAllReduce");
    a.allGather = (decltype(a.allGather))sym("ncclAllGather");
    a.groupStart = (decltype(a.groupStart))sym("ncclGroupStart");
    a.groupEnd = (decltype(a.groupEnd))sym("ncclGroupEnd");
    a.errStr = (decltype(a.errStr))sym("ncclGetErrorString");
    a.commSplit = (decltype(a.commSplit))dlsym(h, "ncclCommSplit");
    a.ok = ok;
    if (!ok) a.err = "libnccl is missing a required symbol";
  });
  return a;
}

qtt_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return QTT_OK;
  NcclApi& a = nccl_api();
  return fail(QTT_ENCCL, "%s: %s", what, a.errStr ? a.errStr(r) : "NCCL error");
}

// -------------------------------------------------------- shard geometry
// Shard s of P = 2^l holds the QTT index range [s 2^{d-l}, (s+1) 2^{d-l})
// (its top l QTT bits equal s), stored as a dense row-major sub-image.
struct ShardGeom {
  int l, dl;
  int lbits[2];        // bits of the shard along x, y
  long long origin[2]; // position of the shard in the global array
};

int ilog2_exact(long long P) {
  if (P < 1 || (P & (P - 1))) return -1;
  int l = 0;
  while ((1ll << l) < P) ++l;
  return l;
}

qtt_status shard_geom(const qtt_shape* s, int P, int shard, ShardGeom* g) {
  qtt_status r;
  if ((r = check_shape(s))) return r;
  const int l = ilog2_exact(P);
  if (l < 0) return fail(QTT_EINVAL, "number of shards %d is not a power of two", P);
  if (shard < 0 || shard >= P) return fail(QTT_EINVAL, "shard %d outside [0, %d)", shard, P);
  const int d = shape_d(s), dl = d - l;
  if (dl < SHARD_MIN_DL)
    return fail(QTT_EINVAL, "a shard must hold >= 2^%d elements (d - log2 P = %d)", SHARD_MIN_DL, dl);
  g->l = l;
  g->dl = dl;
  if (s->D == 1) {
    g->lbits[0] = dl; g->lbits[1] = 0;
    g->origin[0] = (long long)shard << dl; g->origin[1] = 0;
  } else if (s->layout == QTT_LAYOUT_CONCAT) {
    if (l > s->bits[1]) return fail(QTT_EINVAL, "concat layout: log2 P must be <= bits of y");
    g->lbits[0] = s->bits[0]; g->lbits[1] = s->bits[1] - l;
    g->origin[0] = 0; g->origin[1] = (long long)shard << g->lbits[1];
  } else {
    // QTT position q (1-based): odd -> x-bit (q+1)/2, even -> y-bit q/2
    g->lbits[0] = (dl + 1) / 2; g->lbits[1] = dl / 2;
    g->origin[0] = g->origin[1] = 0;
    for (int j = 0; j < l; ++j) {
      const int q = dl + 1 + j;
      const long long b = (shard >> j) & 1;
      if (q & 1) g->origin[0] |= b << ((q + 1) / 2 - 1);
      else g->origin[1] |= b << (q / 2 - 1);
    }
  }
  return QTT_OK;
}

// ------------------------------------------------- sharded TT-SVD plan
struct ShardDec {
  int ntens = 0, nlocal = 0, P = 1, first = 0, d = 0, dl = 0;
  std::vector<DecProb> sh, tn;
  DecProb* sh_dev = nullptr;
  DecProb* tn_dev = nullptr;
  double* gsum = nullptr;   // ntens x 1024, contiguous (one allreduce per level)
  double* gath = nullptr;   // all-gather landing buffer
};

long long gather_cols_cap(int P) { return P == 1 ? FIN_COLS_HOST : (128ll * P > FIN_COLS_HOST ? 128ll * P : FIN_COLS_HOST); }

// xs[t]: this process's first shard of tensor t (further local shards follow
// at + j 2^{dl}); tts[t]: the tensor's core storage.
void plan_sharded_dec(Carver& cv, const qtt_shape* s, const ShardGeom& g, int P, int nlocal, int first,
                      int ntens, const double* const* xs, const TTAlloc* tts, ShardDec& D) {
  D.ntens = ntens; D.nlocal = nlocal; D.P = P; D.first = first; D.d = shape_d(s); D.dl = g.dl;
  D.sh.assign((size_t)ntens * nlocal, DecProb{});
  D.tn.assign(ntens, DecProb{});
  D.gsum = cv.take<double>((size_t)ntens * 1024);
  const long long gcols = gather_cols_cap(P);
  D.gath = cv.take<double>((size_t)ntens * P * RS_GATHER * gcols);
  for (int t = 0; t < ntens; ++t) {
    DecProb& T = D.tn[t];
    T.x = nullptr;
    T.layout = s->layout;
    T.bx = s->bits[0];
    T.d = D.d;
    T.dl = D.d;
    T.gsum = D.gsum ? D.gsum + (size_t)t * 1024 : nullptr;
    T.Wa = cv.take<double>((size_t)RC * gcols);
    T.Wb = cv.take<double>((size_t)RC * gcols);
    T.part = cv.take<double>((size_t)NBLK_MAX * 1024);
    T.proj = cv.take<double>(32 * 16);
    T.tau2 = cv.take<double>(1);
    T.cores = tts[t].cores;
    T.ranks = tts[t].ranks;
    for (int j = 0; j < nlocal; ++j) {
      DecProb& X = D.sh[(size_t)t * nlocal + j];
      X = T;
      X.x = xs[t] ? xs[t] + ((size_t)j << g.dl) : nullptr;
      X.bx = g.lbits[0];
      X.dl = g.dl;
      X.Wa = cv.take<double>((size_t)RC << (g.dl - 5));
      X.Wb = cv.take<double>((size_t)RC << (g.dl - 6));
      X.part = cv.take<double>((size_t)NBLK_MAX * 1024);
    }
  }
  D.sh_dev = cv.take<DecProb>(D.sh.size());
  D.tn_dev = cv.take<DecProb>(D.tn.size());
}

// Gram of the current level: per-CTA partials -> gsum (sum over the local
// shards) -> sum over ranks (NCCL allreduce, f and g in one call).
qtt_status reduce_grams(ShardDec& D, const qtt_comm_s* comm, ncclComm_t nc, int nblk, cudaStream_t st) {
  qtt_status r;
  if ((r = cuda_check(launch_gram_reduce(D.sh_dev, D.ntens, D.nlocal, nblk, st), "gram reduce"))) return r;
  if (comm->kind == 0)
    return nccl_check(nccl_api().allReduce(D.gsum, D.gsum, (size_t)D.ntens * 1024, ncclDouble, ncclSum, nc, st),
                      "ncclAllReduce(Gram)");
  return QTT_OK;
}

// Alg. 1 over column shards: steps k <= d - l use the summed Grams; W is
// gathered once the local unfolding is too narrow; the remaining steps run
// redundantly on every rank on the (small) gathered W.
qtt_status run_sharded_dec(ShardDec& D, const qtt_comm_s* comm, DecParams prm, cudaStream_t st,
                           ncclComm_t nc_override = nullptr) {
  ncclComm_t nc = nc_override ? nc_override : comm->nc;
  qtt_status r;
  if ((r = cuda_check(upload_desc(D.sh_dev, D.sh.data(), D.sh.size() * sizeof(DecProb), st),
                      "copy descriptors")))
    return r;
  if ((r = cuda_check(upload_desc(D.tn_dev, D.tn.data(), D.tn.size() * sizeof(DecProb), st),
                      "copy descriptors")))
    return r;
  const int d = D.d, dl = D.dl, nsh = (int)D.sh.size();
  int nblk = dec_nblk_loc(dl, nsh);
  if ((r = cuda_check(launch_level_gram(D.sh_dev, nsh, nblk, prm.status, st), "level gram"))) return r;
  if ((r = reduce_grams(D, comm, nc, nblk, st))) return r;
  if ((r = cuda_check(launch_level_solve(D.tn_dev, D.ntens, 0, prm, st), "level solve"))) return r;
  int k = 5;
  nblk = proj_nblk(1 << (dl - k), nsh);
  if ((r = cuda_check(launch_project(true, D.sh_dev, nsh, k, nblk, 1, st), "project"))) return r;
  if ((r = reduce_grams(D, comm, nc, nblk, st))) return r;
  int src_is_a = 1;
  ++k;
  while ((1ll << (dl - k + 1)) >= 256 && (1ll << (d - k + 1)) > FIN_COLS_HOST) {
    if ((r = cuda_check(launch_step_solve(D.tn_dev, D.ntens, k, 0, prm, st), "step solve"))) return r;
    nblk = proj_nblk(1 << (dl - k), nsh);
    if ((r = cuda_check(launch_project(false, D.sh_dev, nsh, k, nblk, src_is_a, st), "project"))) return r;
    if ((r = reduce_grams(D, comm, nc, nblk, st))) return r;
    src_is_a ^= 1;
    ++k;
  }
  // gather W_{k-1}: r_{k-1} x nl per shard -> r_{k-1} x nl P on every rank
  const long long nl = 1ll << (dl - k + 1);
  if (comm->kind == 0) {
    NcclApi& A = nccl_api();
    if ((r = nccl_check(A.groupStart(), "ncclGroupStart"))) return r;
    for (int t = 0; t < D.ntens; ++t) {
      const double* src = src_is_a ? D.sh[t].Wa : D.sh[t].Wb;
      double* dst = D.gath + (size_t)t * D.P * RS_GATHER * nl;
      if ((r = nccl_check(A.allGather(src, dst, (size_t)RS_GATHER * nl, ncclDouble, nc, st), "ncclAllGather(W)"))) {
        A.groupEnd();
        return r;
      }
    }
    if ((r = nccl_check(A.groupEnd(), "ncclGroupEnd"))) return r;
    if ((r = cuda_check(launch_gather_w(D.sh_dev, D.tn_dev, D.ntens, D.nlocal, k - 1, nl, src_is_a, D.gath, D.P, st),
                        "gather")))
      return r;
  } else {
    if ((r = cuda_check(launch_gather_w(D.sh_dev, D.tn_dev, D.ntens, D.nlocal, k - 1, nl, src_is_a, nullptr, D.P, st),
                        "gather")))
      return r;
  }
  // remaining steps on the gathered W (tn.Wa), identical on every rank
  src_is_a = 1;
  int prev_nb = 0;   // the Gram of step k is the reduced one in gsum
  while ((1ll << (d - k + 1)) > FIN_COLS_HOST) {
    if ((r = cuda_check(launch_step_solve(D.tn_dev, D.ntens, k, prev_nb, prm, st), "step solve"))) return r;
    const int nb2 = proj_nblk(1 << (d - k), D.ntens);
    if ((r = cuda_check(launch_project(false, D.tn_dev, D.ntens, k, nb2, src_is_a, st), "project"))) return r;
    src_is_a ^= 1;
    prev_nb = nb2;
    ++k;
  }
  return cuda_check(launch_finish(D.tn_dev, D.ntens, k, src_is_a, prm, st), "finish");
}

// ----------------------------------------------- sharded expansion plan
struct ShardEx {
  std::vector<FoldProb> fp;
  std::vector<ExProb> ex;
  FoldProb* fp_dev = nullptr;
  ExProb* ex_dev = nullptr;
};

void plan_sharded_expand(Carver& cv, const cplx* cores, const int* ranks, const ShardGeom& g, int nlocal, int first,
                         double* y, ShardEx& E) {
  E.fp.assign(nlocal, FoldProb{});
  E.ex.assign(nlocal, ExProb{});
  for (int j = 0; j < nlocal; ++j) {
    FoldProb& f = E.fp[j];
    f.cores = cores;
    f.ranks = ranks;
    f.out_cores = cv.take<cplx>((size_t)g.dl * SLOT);
    f.out_ranks = cv.take<int>(64);
    f.shard = first + j;
    ExProb& e = E.ex[j];
    e.cores = f.out_cores;
    e.ranks = f.out_ranks;
    e.y = y ? y + ((size_t)j << g.dl) : nullptr;
    e.lsplit = cv.take<double>(256 * 32);
  }
  E.fp_dev = cv.take<FoldProb>(nlocal);
  E.ex_dev = cv.take<ExProb>(nlocal);
}

qtt_status run_sharded_expand(ShardEx& E, const qtt_shape* s, const ShardGeom& g, int d, int imag, cudaStream_t st,
                              int rcap = RC) {
  qtt_status r;
  const int n = (int)E.fp.size();
  if ((r = cuda_check(upload_desc(E.fp_dev, E.fp.data(), n * sizeof(FoldProb), st),
                      "copy descriptors")))
    return r;
  if ((r = cuda_check(upload_desc(E.ex_dev, E.ex.data(), n * sizeof(ExProb), st),
                      "copy descriptors")))
    return r;
  if ((r = cuda_check(launch_fold_tail(E.fp_dev, n, d, g.l, st), "fold tail"))) return r;
  ExParams P{g.dl, s->layout, g.lbits[0], imag, rcap};
  return cuda_check(launch_expand(E.ex_dev, n, P, st), "expand launch");
}

qtt_status check_comm(const qtt_comm_s* c, const qtt_shape* s, ShardGeom* g) {
  if (s->batch != 1) return fail(QTT_EINVAL, "sharded problems need batch == 1");
  return shard_geom(s, c->nshards, 0, g);
}

int comm_first(const qtt_comm_s* c) { return c->kind == 0 ? c->rank : 0; }

// Workspace of qtt_conv_full when sharded P ways with nlocal shards here.
size_t ws_sharded(const qtt_shape* shape, const qtt_trunc* fft, int P, int nlocal) {
  ShardGeom g;
  if (shape->batch != 1 || shard_geom(shape, P, 0, &g)) return 0;
  const int d = shape_d(shape);
  Carver cv(nullptr);
  cv.take<int>(64);
  TTAlloc tt[2] = {take_tt(cv, 1, d), take_tt(cv, 1, d)};
  TTAlloc Y = take_tt(cv, 1, d);
  const double* xs[2] = {nullptr, nullptr};
  // the two-chain plan (two single-tensor plans) needs at least as much as
  // the batched one; size for both
  const size_t off0 = cv.off;
  ShardDec D;
  plan_sharded_dec(cv, shape, g, P, nlocal, 0, 2, xs, tt, D);
  const size_t one = cv.off;
  cv.off = off0;
  ShardDec Df, Dg;
  plan_sharded_dec(cv, shape, g, P, nlocal, 0, 1, xs, tt, Df);
  plan_sharded_dec(cv, shape, g, P, nlocal, 0, 1, xs + 1, tt + 1, Dg);
  if (cv.off < one) cv.off = one;
  run_convolve(tt[0].cores, tt[0].ranks, 1, tt[1].cores, tt[1].ranks, 1, shape, fft, nullptr, 1.0, Y, cv, nullptr,
               nullptr, RS_GATHER);
  ShardEx E;
  plan_sharded_expand(cv, Y.cores, Y.ranks, g, nlocal, 0, nullptr, E);
  return cv.off + 4096;
}

qtt_status check_ws(const Carver& cv, void* ws, size_t ws_bytes) {
  if (!ws) return fail(QTT_EINVAL, "workspace is NULL");
  if (((uintptr_t)ws & 255) != 0) return fail(QTT_EINVAL, "workspace must be 256-byte aligned");
  if (cv.off > ws_bytes)
    return fail(QTT_ENOMEM, "workspace too small: need %zu bytes, got %zu", cv.off, ws_bytes);
  return QTT_OK;
}

}  // namespace

// ======================================================================= ABI
extern "C" {

const char* qtt_status_string(qtt_status s) {
  switch (s) {
    case QTT_OK: return "QTT_OK";
    case QTT_EINVAL: return "QTT_EINVAL";
    case QTT_ENUMERIC: return "QTT_ENUMERIC";
    case QTT_ECUDA: return "QTT_ECUDA";
    case QTT_ENCCL: return "QTT_ENCCL";
    case QTT_ENOMEM: return "QTT_ENOMEM";
  }
  return "QTT_UNKNOWN";
}

const char* qtt_last_error(void) { return g_err.c_str(); }

const char* qtt_build_info(void) {
  return "libqtt: sm_100a (compute_100a), FP64 DMMA (mma.sync m8n8k4), cp.async staging, "
         "CTA-resident Jacobi eigensolvers; nvcc " QTT_STR(__CUDACC_VER_MAJOR__) "." QTT_STR(__CUDACC_VER_MINOR__);
}

size_t qtt_workspace_bytes(const qtt_shape* shape, const qtt_trunc* dec, const qtt_trunc* fft, int nranks) {
  if (check_shape(shape) || check_trunc(dec, nranks > 1 ? RS_GATHER : RC, "dec", true) ||
      check_trunc(fft, RH_BIG, "fft") || nranks < 1)
    return 0;
  if (nranks > 1 && dec->rule == QTT_RULE_RSVD) return 0;
  if (nranks > 1) return ws_sharded(shape, fft, nranks, 1);
  const int d = shape_d(shape);
  const int nf = shape->batch, ng = shape->g_stride == 0 ? 1 : shape->batch;
  Carver cv(nullptr);
  cv.take<int>(64);
  TTAlloc F = take_tt(cv, nf, d), G = take_tt(cv, ng, d), Y = take_tt(cv, nf, d);
  // decomposition scratch and descriptors, then Step 3 and Step 4 scratch
  // (dry runs of the same carving sequence qtt_conv_full performs)
  for (int i = 0; i < nf + ng; ++i) take_dec(cv, d, dec->rule == QTT_RULE_RSVD);
  cv.take<DecProb>(nf + ng);
  run_convolve(F.cores, F.ranks, nf, G.cores, G.ranks, ng, shape, fft, nullptr, 1.0, Y, cv, nullptr, nullptr,
               dec->rmax);
  run_expand(Y.cores, Y.ranks, nf, d, nullptr, 0, shape, 0, cv, nullptr);
  const size_t one = ws_sharded(shape, fft, 1, 1);   // a 1-rank communicator takes the sharded path
  return cv.off + 4096 > one ? cv.off + 4096 : one;
}

size_t qtt_comm_workspace_bytes(const qtt_shape* shape, const qtt_trunc* dec, const qtt_trunc* fft,
                                qtt_comm_t comm) {
  if (!comm) return qtt_workspace_bytes(shape, dec, fft, 1);
  if (check_shape(shape) || check_trunc(dec, RS_GATHER, "dec") || check_trunc(fft, RH_BIG, "fft")) return 0;
  return ws_sharded(shape, fft, comm->nshards, comm->nlocal);
}

qtt_status qtt_decompose(const double* x, const qtt_shape* shape, const qtt_trunc* dec, void* ws,
                         size_t ws_bytes, void* stream, qtt_comm_t comm, qtt_tt_t* out) {
  qtt_status r;
  if ((r = check_shape(shape))) return r;
  if (!x || !out) return fail(QTT_EINVAL, "x / out is NULL");
  if ((r = check_trunc(dec, comm ? RS_GATHER : RC, "dec", !comm))) return r;
  const int d = shape_d(shape);
  if ((r = check_input_align(x, shape->f_stride ? shape->f_stride : (1ll << d), comm ? 1 : shape->batch, "x")))
    return r;
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  if (comm) {
    ShardGeom g;
    if ((r = check_comm(comm, shape, &g))) return r;
    cudaStream_t st = (cudaStream_t)stream;
    auto plan = [&](Carver& cv, int*& status, TTAlloc& tt, ShardDec& D) {
      status = cv.take<int>(64);
      tt = take_tt(cv, 1, d);
      plan_sharded_dec(cv, shape, g, comm->nshards, comm->nlocal, comm_first(comm), 1, &x, &tt, D);
    };
    Carver dry(nullptr);
    int* status;
    TTAlloc tt;
    ShardDec D;
    plan(dry, status, tt, D);
    if ((r = check_ws(dry, ws, ws_bytes))) return r;
    Carver cv(ws);
    plan(cv, status, tt, D);
    if ((r = cuda_check(cudaMemsetAsync(status, 0, STATUS_BYTES, st), "status reset"))) return r;
    DecParams prm = dec_params(dec, status);
    if ((r = run_sharded_dec(D, comm, prm, st))) return r;
    *out = new_handle(shape, 1, dec->rmax, tt, status, st);
    return *out ? QTT_OK : fail(QTT_ENOMEM, "host allocation failed");
  }
  const int n = shape->batch;
  const long long stride = shape->f_stride ? shape->f_stride : (1ll << d);
  cudaStream_t st = (cudaStream_t)stream;
  Carver dry(nullptr);
  int* status = dry.take<int>(64);
  TTAlloc tt = take_tt(dry, n, d);
  run_decompose(x, stride, n, shape, dec, tt, dry, nullptr, st);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  status = cv.take<int>(64);
  tt = take_tt(cv, n, d);
  if ((r = cuda_check(cudaMemsetAsync(status, 0, STATUS_BYTES, st), "status reset"))) return r;
  if ((r = run_decompose(x, stride, n, shape, dec, tt, cv, status, st))) return r;
  *out = new_handle(shape, n, dec->rmax, tt, status, st);
  if (!*out) return fail(QTT_ENOMEM, "host allocation failed");
  return QTT_OK;
}

qtt_status qtt_transform(qtt_tt_t in, const qtt_trunc* fft, int inverse, const long long shift[2], double scale,
                         void* ws, size_t ws_bytes, void* stream, qtt_tt_t* out) {
  qtt_status r;
  if (!in || !out) return fail(QTT_EINVAL, "in / out is NULL");
  if ((r = check_trunc(fft, RS_BIG, "fft"))) return r;
  if (in->rcap > RS_BIG) return fail(QTT_EINVAL, "input ranks may exceed %d", RS_BIG);
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = in->d, n = in->nt;
  // the shared-memory variant holds ranks <= RS_XF; above that the cores live in the workspace
  const int rs = (in->rcap > RS_XF || fft->rmax > RS_XF) ? RS_BIG : RS_XF;
  cudaStream_t st = (cudaStream_t)stream;
  auto plan = [&](Carver& cv, TTAlloc& o, std::vector<XfProb>& v) {
    o = take_tt(cv, n, d);
    v.resize(n);
    for (int i = 0; i < n; ++i) {
      v[i].in_cores = in->cores + (size_t)i * d * SLOT;
      v[i].in_ranks = in->ranks + (size_t)i * 64;
      v[i].out_cores = o.cores + (size_t)i * d * SLOT;
      v[i].out_ranks = o.ranks + (size_t)i * 64;
      v[i].gr = cv.take<cplx>((size_t)MAXD * xf_gr_slot(rs));
      v[i].cwork = rs == RS_BIG ? cv.take<cplx>((size_t)MAXD * 2 * RS_BIG * RS_BIG) : nullptr;
      v[i].do_center = (!inverse && shift) ? 1 : 0;
    }
  };
  Carver dry(nullptr);
  TTAlloc o;
  std::vector<XfProb> v;
  plan(dry, o, v);
  run_transform(v, &in->shape, fft, inverse, shift, scale, dry, nullptr, st, rs);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  plan(cv, o, v);
  if ((r = run_transform(v, &in->shape, fft, inverse, shift, scale, cv, in->status, st, rs))) return r;
  *out = new_handle(&in->shape, n, fft->rmax, o, in->status, st);
  return *out ? QTT_OK : fail(QTT_ENOMEM, "host allocation failed");
}

qtt_status qtt_convolve(qtt_tt_t f, qtt_tt_t g, const qtt_trunc* fft, const long long shift[2], double scale,
                        void* ws, size_t ws_bytes, void* stream, qtt_tt_t* out) {
  qtt_status r;
  if (!f || !g || !out) return fail(QTT_EINVAL, "f / g / out is NULL");
  if ((r = check_trunc(fft, RH_BIG, "fft"))) return r;
  if (f->d != g->d) return fail(QTT_EINVAL, "f and g have different d");
  if (g->nt != 1 && g->nt != f->nt) return fail(QTT_EINVAL, "g must hold 1 tensor or as many as f");
  if (f->rcap > RS_BIG || g->rcap > RS_BIG) return fail(QTT_EINVAL, "input ranks may exceed %d", RS_BIG);
  const int in_rcap = f->rcap > g->rcap ? f->rcap : g->rcap;
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = f->d;
  cudaStream_t st = (cudaStream_t)stream;
  Carver dry(nullptr);
  TTAlloc Y = take_tt(dry, f->nt, d);
  run_convolve(f->cores, f->ranks, f->nt, g->cores, g->ranks, g->nt, &f->shape, fft, shift, scale, Y, dry,
               nullptr, st, in_rcap);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  Y = take_tt(cv, f->nt, d);
  if ((r = run_convolve(f->cores, f->ranks, f->nt, g->cores, g->ranks, g->nt, &f->shape, fft, shift, scale, Y,
                        cv, f->status, st, in_rcap)))
    return r;
  *out = new_handle(&f->shape, f->nt, fft->rmax, Y, f->status, st);
  return *out ? QTT_OK : fail(QTT_ENOMEM, "host allocation failed");
}

qtt_status qtt_to_full(qtt_tt_t t, double* y, double* y_imag, void* ws, size_t ws_bytes, void* stream,
                       qtt_comm_t comm) {
  qtt_status r;
  if (!t || !y) return fail(QTT_EINVAL, "t / y is NULL");
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = t->d;
  if (comm) {
    ShardGeom g;
    if ((r = check_comm(comm, &t->shape, &g))) return r;
    if (t->nt != 1) return fail(QTT_EINVAL, "sharded expansion needs a single tensor");
    cudaStream_t st = (cudaStream_t)stream;
    Carver dry(nullptr);
    ShardEx E;
    plan_sharded_expand(dry, t->cores, t->ranks, g, comm->nlocal, comm_first(comm), y, E);
    if ((r = check_ws(dry, ws, ws_bytes))) return r;
    for (int im = 0; im < (y_imag ? 2 : 1); ++im) {
      Carver cv(ws);
      plan_sharded_expand(cv, t->cores, t->ranks, g, comm->nlocal, comm_first(comm), im ? y_imag : y, E);
      if ((r = run_sharded_expand(E, &t->shape, g, d, im, st, t->rcap))) return r;
    }
    return QTT_OK;
  }
  const long long ys = t->shape.y_stride ? t->shape.y_stride : (1ll << d);
  cudaStream_t st = (cudaStream_t)stream;
  Carver dry(nullptr);
  run_expand(t->cores, t->ranks, t->nt, d, y, ys, &t->shape, 0, dry, st);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  if ((r = run_expand(t->cores, t->ranks, t->nt, d, y, ys, &t->shape, 0, cv, st, t->rcap))) return r;
  if (y_imag) {
    Carver cv2(ws);
    if ((r = run_expand(t->cores, t->ranks, t->nt, d, y_imag, ys, &t->shape, 1, cv2, st, t->rcap))) return r;
  }
  return QTT_OK;
}

qtt_status qtt_conv_full(const double* f, const double* g, double* y, const qtt_shape* shape, const qtt_trunc* dec,
                         const qtt_trunc* fft, const long long shift[2], double scale, void* ws, size_t ws_bytes,
                         void* stream, qtt_comm_t comm, qtt_report* rep_host) {
  qtt_status r;
  if ((r = check_shape(shape))) return r;
  if ((r = check_trunc(dec, comm ? RS_GATHER : RC, "dec", !comm))) return r;
  if ((r = check_trunc(fft, RH_BIG, "fft"))) return r;
  if (!f || !g || !y) return fail(QTT_EINVAL, "f / g / y is NULL");
  ShardGeom geo{};
  if (comm && (r = check_comm(comm, shape, &geo))) return r;
  const size_t need = comm ? ws_sharded(shape, fft, comm->nshards, comm->nlocal)
                           : qtt_workspace_bytes(shape, dec, fft, 1);
  if (!ws) return fail(QTT_EINVAL, "workspace is NULL");
  if (((uintptr_t)ws & 255) != 0) return fail(QTT_EINVAL, "workspace must be 256-byte aligned");
  if (ws_bytes < need) return fail(QTT_ENOMEM, "workspace too small: need %zu bytes, got %zu", need, ws_bytes);
  const int d = shape_d(shape);
  const int nf = shape->batch, ng = shape->g_stride == 0 ? 1 : shape->batch;
  const long long fs = shape->f_stride ? shape->f_stride : (1ll << d);
  const long long gs = shape->g_stride;
  const long long ys = shape->y_stride ? shape->y_stride : (1ll << d);
  if (!comm) {
    if ((r = check_input_align(f, fs, nf, "f"))) return r;
    if ((r = check_input_align(g, gs, ng, "g"))) return r;
  } else {
    if ((r = check_input_align(f, 0, 1, "f"))) return r;
    if ((r = check_input_align(g, 0, 1, "g"))) return r;
  }
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  cudaStream_t st = (cudaStream_t)stream;
  EventGuard evg;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (rep_host) {
    if ((r = cuda_check(evg.make(&e0, cudaEventDefault), "event"))) return r;
    if ((r = cuda_check(evg.make(&e1, cudaEventDefault), "event"))) return r;
    cudaEventRecord(e0, st);
  }
  Carver cv(ws);
  int* status = cv.take<int>(64);
  TTAlloc F = take_tt(cv, nf, d), G = take_tt(cv, ng, d), Y = take_tt(cv, nf, d);
  if ((r = cuda_check(cudaMemsetAsync(status, 0, STATUS_BYTES, st), "status reset"))) return r;
  prof_mark(0, st);
  DecParams prm = dec_params(dec, status);
  if (comm) {
    // Step 1-2 column-sharded.  With a second communicator (or a virtual one)
    // f and g run as two chains on two streams, as on one GPU: the one-CTA
    // solves and the allreduces of one hide under the passes of the other;
    // each chain issues its collectives on its own communicator, so the two
    // streams never interleave operations of one NCCL communicator.
    // Otherwise: one batched chain, one allreduce per level for f and g.
    const double* xs[2] = {f, g};
    TTAlloc tts[2] = {F, G};
    cudaStream_t side = (comm->kind == 1 || comm->nc2) && g_prof < 2 ? side_stream() : nullptr;
    if (side) {
      ShardDec Df, Dg;
      plan_sharded_dec(cv, shape, geo, comm->nshards, comm->nlocal, comm_first(comm), 1, xs, tts, Df);
      plan_sharded_dec(cv, shape, geo, comm->nshards, comm->nlocal, comm_first(comm), 1, xs + 1, tts + 1, Dg);
      cudaEvent_t fork = nullptr, join = nullptr;
      if ((r = cuda_check(evg.make(&fork, cudaEventDisableTiming), "event"))) return r;
      if ((r = cuda_check(evg.make(&join, cudaEventDisableTiming), "event"))) return r;
      cudaEventRecord(fork, st);
      cudaStreamWaitEvent(side, fork, 0);
      r = run_sharded_dec(Dg, comm, prm, side, comm->nc2);
      if (!r) r = run_sharded_dec(Df, comm, prm, st);
      // the join is recorded even after a failed launch (see the one-GPU path)
      cudaEventRecord(join, side);
      qtt_status rj = cuda_check(cudaStreamWaitEvent(st, join, 0), "join");
      if (r || (r = rj)) return r;
    } else {
      ShardDec D;
      plan_sharded_dec(cv, shape, geo, comm->nshards, comm->nlocal, comm_first(comm), 2, xs, tts, D);
      if ((r = run_sharded_dec(D, comm, prm, st))) return r;
    }
  } else {
    // Step 1-2: all signals and the kernel(s) in one batched TT-SVD
    const int d_ = d;
    std::vector<DecProb> h(nf + ng);
    for (int i = 0; i < nf + ng; ++i) {
      const bool isf = i < nf;
      const int j = isf ? i : i - nf;
      DecScratch sc = take_dec(cv, d_, dec->rule == QTT_RULE_RSVD);
      DecProb& p = h[i];
      p.x = isf ? f + (size_t)j * (size_t)fs : g + (size_t)j * (size_t)gs;
      p.layout = shape->layout;
      p.bx = shape->bits[0];
      p.d = d_;
      p.dl = d_;
      p.gsum = sc.gsum;
      p.Wa = sc.Wa; p.Wb = sc.Wb; p.part = sc.part; p.proj = sc.proj; p.tau2 = sc.tau2;
      p.cores = (isf ? F.cores : G.cores) + (size_t)j * d_ * SLOT;
      p.ranks = (isf ? F.ranks : G.ranks) + (size_t)j * 64;
      p.psk = sc.psk;
      p.seed = dec->seed + (unsigned long long)i;   // f batch entries, then g
    }
    DecProb* dp = cv.take<DecProb>(nf + ng);
    if ((r = cuda_check(upload_desc(dp, h.data(), h.size() * sizeof(DecProb), st),
                        "copy descriptors")))
      return r;
    const int ntot = nf + ng;
    cudaStream_t side = (ntot >= 2 && g_prof < 2) ? side_stream() : nullptr;
    if (side) {
      // the first half of the tensors (f, or the first batch entries) on the
      // caller's stream, the rest on the side stream (fork / join events):
      // the one-CTA solves of one chain run under the HBM passes of the other
      const int na = (ntot + 1) / 2;
      cudaEvent_t fork = nullptr, join = nullptr;
      if ((r = cuda_check(evg.make(&fork, cudaEventDisableTiming), "event"))) return r;
      if ((r = cuda_check(evg.make(&join, cudaEventDisableTiming), "event"))) return r;
      cudaEventRecord(fork, st);
      cudaStreamWaitEvent(side, fork, 0);
      r = cuda_check(launch_ttsvd(dp + na, ntot - na, d_, prm, side, 4), "TT-SVD launch");
      // the join is recorded even after a failed launch, so `st` never runs
      // ahead of work already queued on the side stream
      if (!r) r = cuda_check(launch_ttsvd(dp, na, d_, prm, st, 4), "TT-SVD launch");
      cudaEventRecord(join, side);
      qtt_status rj = cuda_check(cudaStreamWaitEvent(st, join, 0), "join");
      if (r || (r = rj)) return r;
    } else if ((r = cuda_check(launch_ttsvd(dp, nf + ng, d_, prm, st), "TT-SVD launch"))) {
      return r;
    }
  }
  prof_mark(1, st);
  // Step 3
  TTAlloc mid[3];
  if ((r = run_convolve(F.cores, F.ranks, nf, G.cores, G.ranks, ng, shape, fft, shift, scale, Y, cv, status, st,
                        dec->rmax, mid)))
    return r;
  // Step 4
  if (comm) {
    ShardEx E;
    plan_sharded_expand(cv, Y.cores, Y.ranks, geo, comm->nlocal, comm_first(comm), y, E);
    if ((r = run_sharded_expand(E, shape, geo, d, 0, st, fft->rmax))) return r;
  } else if ((r = run_expand(Y.cores, Y.ranks, nf, d, y, ys, shape, 0, cv, st, fft->rmax))) {
    return r;
  }
  prof_mark(5, st);
  if (cv.off > ws_bytes) return fail(QTT_ENOMEM, "internal: workspace plan overflow");
  if (rep_host) {
    cudaEventRecord(e1, st);
    if ((r = cuda_check(cudaStreamSynchronize(st), "stream sync"))) return r;
    memset(rep_host, 0, sizeof(*rep_host));
    rep_host->d = d;
    cudaEventElapsedTime(&rep_host->ms_total, e0, e1);
    const size_t rb = (d + 1) * sizeof(int);
    cudaMemcpy(rep_host->ranks_f, F.ranks, rb, cudaMemcpyDeviceToHost);
    cudaMemcpy(rep_host->ranks_g, G.ranks, rb, cudaMemcpyDeviceToHost);
    cudaMemcpy(rep_host->ranks_fh, mid[0].ranks, rb, cudaMemcpyDeviceToHost);
    cudaMemcpy(rep_host->ranks_gh, mid[1].ranks, rb, cudaMemcpyDeviceToHost);
    cudaMemcpy(rep_host->ranks_z, mid[2].ranks, rb, cudaMemcpyDeviceToHost);
    cudaMemcpy(rep_host->ranks_out, Y.ranks, rb, cudaMemcpyDeviceToHost);
    int hst[16] = {};
    cudaMemcpy(hst, status, STATUS_BYTES, cudaMemcpyDeviceToHost);
    const int hs = hst[0];
    rep_host->status_bits = hs;
    auto unmin = [](const int* w) {
      unsigned long long b;
      memcpy(&b, w, sizeof b);
      if (!b) return HUGE_VAL;
      b = ~b;
      double v;
      memcpy(&v, &b, sizeof v);
      return v;
    };
    rep_host->min_margin = unmin(hst + 2);
    rep_host->min_gap = unmin(hst + 4);
    if ((r = cuda_check(cudaGetLastError(), "report"))) return r;
    if (hs & ST_ERRORS) return fail(QTT_ENUMERIC, "numeric status 0x%x (1 = non-finite input, 2 = eigensolver)", hs);
  }
  return QTT_OK;
}

qtt_status qtt_wait(qtt_tt_t t) {
  if (!t) return fail(QTT_EINVAL, "handle is NULL");
  qtt_status r;
  if ((r = cuda_check(cudaStreamSynchronize(t->stream), "stream sync"))) return r;
  int hs = 0;
  if ((r = cuda_check(cudaMemcpy(&hs, t->status, sizeof(int), cudaMemcpyDeviceToHost), "status read"))) return r;
  if (hs & ST_ERRORS) return fail(QTT_ENUMERIC, "numeric status 0x%x (1 = non-finite input, 2 = eigensolver)", hs);
  return QTT_OK;
}

qtt_status qtt_ranks(qtt_tt_t t, int index, int* ranks_host, int cap) {
  if (!t || !ranks_host) return fail(QTT_EINVAL, "handle / ranks is NULL");
  if (index < 0 || index >= t->nt) return fail(QTT_EINVAL, "index %d outside [0, %d)", index, t->nt);
  if (cap < t->d + 1) return fail(QTT_EINVAL, "cap must be >= d+1 = %d", t->d + 1);
  qtt_status r;
  if ((r = qtt_wait(t)) && r != QTT_ENUMERIC) return r;
  qtt_status r2 = cuda_check(
      cudaMemcpy(ranks_host, t->ranks + (size_t)index * 64, (t->d + 1) * sizeof(int), cudaMemcpyDeviceToHost),
      "ranks read");
  return r2 ? r2 : r;
}

int qtt_ndims(qtt_tt_t t) { return t ? t->d : 0; }

void qtt_profile_enable(int on) {
  g_prof = on < 0 ? 0 : (on > 2 ? 2 : on);
  for (int k = 0; k < PASS_N; ++k) g_pev_set[k] = 0;
}

int qtt_profile_read(float* ms_host, int n) {
  if (!g_ev_ok || !ms_host || n < PROF_STAGES) return 0;
  if (cudaEventSynchronize(g_ev[PROF_MARKS - 1]) != cudaSuccess) return 0;
  for (int k = 0; k < PROF_STAGES; ++k) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_ev[k], g_ev[k + 1]);
    ms_host[k] = ms;
  }
  if (n < PROF_STAGES + PASS_N || g_prof < 2) return PROF_STAGES;
  for (int k = 0; k < PASS_N; ++k) {
    float ms = -1.f;
    if (g_pev_set[k]) cudaEventElapsedTime(&ms, g_pev[k][0], g_pev[k][1]);
    ms_host[PROF_STAGES + k] = ms;
  }
  return PROF_STAGES + PASS_N;
}

long long qtt_launch_count(void) { return qtt::g_launches.load(); }

qtt_status qtt_debug_tt_from_host(const qtt_shape* shape, const void* cores_host, const int* ranks_host, int rcap,
                                  void* ws, size_t ws_bytes, void* stream, qtt_tt_t* out) {
  qtt_status r;
  if ((r = check_shape(shape))) return r;
  if (!cores_host || !ranks_host || !out) return fail(QTT_EINVAL, "NULL argument");
  if (rcap < 1 || rcap > RC) return fail(QTT_EINVAL, "rcap outside [1, %d]", RC);
  const int d = shape_d(shape), n = shape->batch;
  Carver dry(nullptr);
  dry.take<int>(64);
  take_tt(dry, n, d);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  int* status = cv.take<int>(64);
  TTAlloc tt = take_tt(cv, n, d);
  cudaStream_t st = (cudaStream_t)stream;
  if ((r = cuda_check(cudaMemsetAsync(status, 0, STATUS_BYTES, st), "status reset"))) return r;
  if ((r = cuda_check(cudaMemcpyAsync(tt.cores, cores_host, (size_t)n * d * SLOT * sizeof(cplx),
                                      cudaMemcpyHostToDevice, st), "cores upload")))
    return r;
  if ((r = cuda_check(cudaMemcpyAsync(tt.ranks, ranks_host, (size_t)n * 64 * sizeof(int), cudaMemcpyHostToDevice, st),
                      "ranks upload")))
    return r;
  if ((r = cuda_check(cudaStreamSynchronize(st), "sync"))) return r;
  *out = new_handle(shape, n, rcap, tt, status, st);
  return *out ? QTT_OK : fail(QTT_ENOMEM, "host allocation failed");
}

void qtt_destroy(qtt_tt_t t) { delete t; }

qtt_status qtt_comm_unique_id(unsigned char id_host[128]) {
  if (!id_host) return fail(QTT_EINVAL, "id is NULL");
  NcclApi& A = nccl_api();
  if (!A.ok) return fail(QTT_ENCCL, "NCCL unavailable: %s", A.err.c_str());
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  qtt_status r;
  if ((r = nccl_check(A.getUniqueId(&id), "ncclGetUniqueId"))) return r;
  memcpy(id_host, &id, 128);
  return QTT_OK;
}

qtt_status qtt_comm_init(const unsigned char id_host[128], int nranks, int rank, qtt_comm_t* out) {
  if (!id_host || !out) return fail(QTT_EINVAL, "id / out is NULL");
  if (nranks < 1 || ilog2_exact(nranks) < 0) return fail(QTT_EINVAL, "nranks = %d is not a power of two", nranks);
  if (rank < 0 || rank >= nranks) return fail(QTT_EINVAL, "rank %d outside [0, %d)", rank, nranks);
  NcclApi& A = nccl_api();
  if (!A.ok) return fail(QTT_ENCCL, "NCCL unavailable: %s", A.err.c_str());
  ncclUniqueId id;
  memcpy(&id, id_host, 128);
  ncclComm_t nc;
  qtt_status r;
  if ((r = nccl_check(A.commInitRank(&nc, nranks, id, rank), "ncclCommInitRank"))) return r;
  // a second communicator over the same ranks for the g chain of the
  // sharded TT-SVD (collective; without ncclCommSplit the chains are batched)
  ncclComm_t nc2 = nullptr;
  if (A.commSplit && A.commSplit(nc, 0, rank, &nc2, nullptr) != ncclSuccess) nc2 = nullptr;
  qtt_comm_t c = new (std::nothrow) qtt_comm_s{0, nranks, rank, nranks, 1, nc, nc2};
  if (!c) {
    if (nc2) A.commDestroy(nc2);
    A.commDestroy(nc);
    return fail(QTT_ENOMEM, "host allocation failed");
  }
  *out = c;
  return QTT_OK;
}

qtt_status qtt_comm_init_virtual(int nshards, qtt_comm_t* out) {
  if (!out) return fail(QTT_EINVAL, "out is NULL");
  if (nshards < 1 || ilog2_exact(nshards) < 0)
    return fail(QTT_EINVAL, "nshards = %d is not a power of two", nshards);
  qtt_comm_t c = new (std::nothrow) qtt_comm_s{1, 1, 0, nshards, nshards, nullptr};
  if (!c) return fail(QTT_ENOMEM, "host allocation failed");
  *out = c;
  return QTT_OK;
}

void qtt_comm_destroy(qtt_comm_t c) {
  if (!c) return;
  if (c->kind == 0 && c->nc2) nccl_api().commDestroy(c->nc2);
  if (c->kind == 0 && c->nc) nccl_api().commDestroy(c->nc);
  delete c;
}

qtt_status qtt_shard_geometry(const qtt_shape* shape, int nshards, int shard, long long origin_host[2],
                              int bits_host[2]) {
  if (!origin_host || !bits_host) return fail(QTT_EINVAL, "origin / bits is NULL");
  ShardGeom g;
  qtt_status r;
  if ((r = shard_geom(shape, nshards, shard, &g))) return r;
  origin_host[0] = g.origin[0];
  origin_host[1] = g.origin[1];
  bits_host[0] = g.lbits[0];
  bits_host[1] = g.lbits[1];
  return QTT_OK;
}

}  // extern "C"

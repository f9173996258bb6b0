// api.cu — the C ABI of libqtt.so (include/qtt.h): argument validation,
// workspace carving and the launch sequence of Alg. 2.
// Every compute step runs in the kernels of ttsvd.cu, qfft.cu, hround.cu and
// expand.cu; this file only marshals pointers.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qtt.h"
#include "qtt_kernels.h"

using namespace qtt;

namespace qtt {
static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches += n; }
}  // namespace qtt

#define QTT_XSTR(x) #x
#define QTT_STR(x) QTT_XSTR(x)

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

std::once_flag g_setup_once;
cudaError_t g_setup_err = cudaSuccess;

cudaError_t setup_all() {
  std::call_once(g_setup_once, [] {
    cudaError_t e;
    if ((e = setup_ttsvd_kernels()) != cudaSuccess) { g_setup_err = e; return; }
    if ((e = setup_xf_kernels()) != cudaSuccess) { g_setup_err = e; return; }
    if ((e = setup_hr_kernels()) != cudaSuccess) { g_setup_err = e; return; }
    if ((e = setup_expand_kernels()) != cudaSuccess) { g_setup_err = e; return; }
  });
  return g_setup_err;
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

qtt_status check_trunc(const qtt_trunc* t, int rmax_cap, const char* which) {
  if (!t) return fail(QTT_EINVAL, "%s truncation is NULL", which);
  if (!(t->eps >= 0.0)) return fail(QTT_EINVAL, "%s eps must be >= 0", which);
  if (t->rmax < 1 || t->rmax > rmax_cap)
    return fail(QTT_EINVAL, "%s rmax = %d outside [1, %d]", which, t->rmax, rmax_cap);
  if (!(t->cluster_tol >= 0.0)) return fail(QTT_EINVAL, "%s cluster_tol must be >= 0", which);
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
};
DecScratch take_dec(Carver& cv, int d) {
  DecScratch s{};
  if (d > 12) {
    s.Wa = cv.take<double>((size_t)RC << (d - 5));
    s.Wb = cv.take<double>((size_t)RC << (d - 6));
    s.part = cv.take<double>((size_t)NBLK_MAX * 1024);
  } else {
    s.Wa = s.Wb = s.part = nullptr;
  }
  s.proj = cv.take<double>(32 * 16);
  s.tau2 = cv.take<double>(1);
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
  for (int i = 0; i < n; ++i) {
    DecScratch sc = take_dec(cv, d);
    DecProb& p = h[i];
    p.x = base + (size_t)i * (size_t)stride;
    p.layout = s->layout;
    p.bx = s->bits[0];
    p.d = d;
    p.Wa = sc.Wa; p.Wb = sc.Wb; p.part = sc.part; p.proj = sc.proj; p.tau2 = sc.tau2;
    p.cores = tt.cores + (size_t)i * d * SLOT;
    p.ranks = tt.ranks + (size_t)i * 64;
  }
  DecProb* dp = cv.take<DecProb>(n);
  if (!cv.base) return QTT_OK;
  qtt_status r;
  if ((r = cuda_check(cudaMemcpyAsync(dp, h.data(), n * sizeof(DecProb), cudaMemcpyHostToDevice, st),
                      "copy descriptors")))
    return r;
  DecParams prm{dec->eps, dec->rmax, dec->cluster_tol, status};
  return cuda_check(launch_ttsvd(dp, n, d, prm, st), "TT-SVD launch");
}

qtt_status run_transform(const std::vector<XfProb>& hv, const qtt_shape* s, const qtt_trunc* fft, int inverse,
                         const long long* shift, double scale, Carver& cv, int* status, cudaStream_t st) {
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
  P.inverse = inverse;
  P.scale = inverse ? scale * ldexp(1.0, -P.d) : 1.0;
  P.shift[0] = shift ? shift[0] : 0;
  P.shift[1] = (shift && s->D == 2) ? shift[1] : 0;
  P.status = status;
  qtt_status r;
  if ((r = cuda_check(cudaMemcpyAsync(dp, hv.data(), n * sizeof(XfProb), cudaMemcpyHostToDevice, st),
                      "copy descriptors")))
    return r;
  return cuda_check(launch_transform(dp, n, P, st), "transform launch");
}

qtt_status run_expand(const cplx* cores, const int* ranks, int nt, int d, double* y, long long ystride,
                      const qtt_shape* s, int imag, Carver& cv, cudaStream_t st) {
  std::vector<ExProb> h(nt);
  for (int i = 0; i < nt; ++i) {
    h[i].cores = cores + (size_t)i * d * SLOT;
    h[i].ranks = ranks + (size_t)i * 64;
    h[i].y = y + (size_t)i * (size_t)ystride;
    h[i].lsplit = cv.take<double>(256 * 32);
  }
  ExProb* dp = cv.take<ExProb>(nt);
  if (!cv.base) return QTT_OK;
  ExParams P{d, s->layout, s->bits[0], imag};
  qtt_status r;
  if ((r = cuda_check(cudaMemcpyAsync(dp, h.data(), nt * sizeof(ExProb), cudaMemcpyHostToDevice, st),
                      "copy descriptors")))
    return r;
  return cuda_check(launch_expand(dp, nt, P, st), "expand launch");
}

// Step 3 on handles' storage: F (nf tensors), G (ng = 1 or nf) -> Y (nf)
qtt_status run_convolve(const cplx* fc, const int* fr, int nf, const cplx* gc, const int* gr, int ng,
                        const qtt_shape* s, const qtt_trunc* fft, const long long* shift, double scale,
                        TTAlloc Y, Carver& cv, int* status, cudaStream_t st) {
  const int d = shape_d(s);
  TTAlloc Fh = take_tt(cv, nf, d);
  TTAlloc Gh = take_tt(cv, ng, d);
  TTAlloc Z = take_tt(cv, nf, d);
  std::vector<XfProb> fw(nf + ng);
  for (int i = 0; i < nf + ng; ++i) {
    const bool isf = i < nf;
    const int j = isf ? i : i - nf;
    XfProb& p = fw[i];
    p.in_cores = (isf ? fc : gc) + (size_t)j * d * SLOT;
    p.in_ranks = (isf ? fr : gr) + (size_t)j * 64;
    p.out_cores = (isf ? Fh.cores : Gh.cores) + (size_t)j * d * SLOT;
    p.out_ranks = (isf ? Fh.ranks : Gh.ranks) + (size_t)j * 64;
    p.gr = cv.take<cplx>((size_t)MAXD * GR_XF);
    p.do_center = (!isf && shift) ? 1 : 0;   // center the kernel's spectrum only (O3)
  }
  // forward transforms of all F's and G's: one launch, one CTA each
  qtt_status r;
  if ((r = run_transform(fw, s, fft, 0, shift, 1.0, cv, status, st))) return r;
  if (cv.base) prof_mark(2, st);
  std::vector<HrProb> hr(nf);
  for (int i = 0; i < nf; ++i) {
    HrProb& p = hr[i];
    p.f_cores = Fh.cores + (size_t)i * d * SLOT;
    p.f_ranks = Fh.ranks + (size_t)i * 64;
    const int j = ng == 1 ? 0 : i;
    p.g_cores = Gh.cores + (size_t)j * d * SLOT;
    p.g_ranks = Gh.ranks + (size_t)j * 64;
    p.out_cores = Z.cores + (size_t)i * d * SLOT;
    p.out_ranks = Z.ranks + (size_t)i * 64;
    p.gr = cv.take<cplx>((size_t)MAXD * GR_HR);
  }
  HrProb* hp = cv.take<HrProb>(nf);
  std::vector<XfProb> iv(nf);
  for (int i = 0; i < nf; ++i) {
    XfProb& p = iv[i];
    p.in_cores = Z.cores + (size_t)i * d * SLOT;
    p.in_ranks = Z.ranks + (size_t)i * 64;
    p.out_cores = Y.cores + (size_t)i * d * SLOT;
    p.out_ranks = Y.ranks + (size_t)i * 64;
    p.gr = fw[i].gr;   // reuse the forward scratch
    p.do_center = 0;
  }
  if (cv.base) {
    HrParams H{d, fft->eps, fft->rmax, fft->cluster_tol, status};
    if ((r = cuda_check(cudaMemcpyAsync(hp, hr.data(), nf * sizeof(HrProb), cudaMemcpyHostToDevice, st),
                        "copy descriptors")))
      return r;
    if ((r = cuda_check(launch_hadamard_round(hp, nf, H, st), "hadamard/round launch"))) return r;
    prof_mark(3, st);
  }
  r = run_transform(iv, s, fft, 1, nullptr, scale, cv, status, st);
  if (cv.base) prof_mark(4, st);
  return r;
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
  if (check_shape(shape) || check_trunc(dec, RS_XF, "dec") || check_trunc(fft, RH_MAX, "fft") || nranks != 1)
    return 0;
  const int d = shape_d(shape);
  const int nf = shape->batch, ng = shape->g_stride == 0 ? 1 : shape->batch;
  Carver cv(nullptr);
  cv.take<int>(64);
  TTAlloc F = take_tt(cv, nf, d), G = take_tt(cv, ng, d), Y = take_tt(cv, nf, d);
  // decomposition scratch and descriptors, then Step 3 and Step 4 scratch
  // (dry runs of the same carving sequence qtt_conv_full performs)
  for (int i = 0; i < nf + ng; ++i) take_dec(cv, d);
  cv.take<DecProb>(nf + ng);
  run_convolve(F.cores, F.ranks, nf, G.cores, G.ranks, ng, shape, fft, nullptr, 1.0, Y, cv, nullptr, nullptr);
  run_expand(Y.cores, Y.ranks, nf, d, nullptr, 0, shape, 0, cv, nullptr);
  return cv.off + 4096;
}

qtt_status qtt_decompose(const double* x, const qtt_shape* shape, const qtt_trunc* dec, void* ws,
                         size_t ws_bytes, void* stream, qtt_comm_t comm, qtt_tt_t* out) {
  qtt_status r;
  if ((r = check_shape(shape))) return r;
  if ((r = check_trunc(dec, RC, "dec"))) return r;
  if (!x || !out) return fail(QTT_EINVAL, "x / out is NULL");
  if (comm) return fail(QTT_EINVAL, "multi-GPU communicators are not supported by this build");
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = shape_d(shape);
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
  if ((r = cuda_check(cudaMemsetAsync(status, 0, sizeof(int), st), "status reset"))) return r;
  if ((r = run_decompose(x, stride, n, shape, dec, tt, cv, status, st))) return r;
  *out = new_handle(shape, n, dec->rmax, tt, status, st);
  if (!*out) return fail(QTT_ENOMEM, "host allocation failed");
  return QTT_OK;
}

qtt_status qtt_transform(qtt_tt_t in, const qtt_trunc* fft, int inverse, const long long shift[2], double scale,
                         void* ws, size_t ws_bytes, void* stream, qtt_tt_t* out) {
  qtt_status r;
  if (!in || !out) return fail(QTT_EINVAL, "in / out is NULL");
  if ((r = check_trunc(fft, RS_XF, "fft"))) return r;
  if (in->rcap > RS_XF) return fail(QTT_EINVAL, "input ranks may exceed %d", RS_XF);
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = in->d, n = in->nt;
  cudaStream_t st = (cudaStream_t)stream;
  auto plan = [&](Carver& cv, TTAlloc& o, std::vector<XfProb>& v) {
    o = take_tt(cv, n, d);
    v.resize(n);
    for (int i = 0; i < n; ++i) {
      v[i].in_cores = in->cores + (size_t)i * d * SLOT;
      v[i].in_ranks = in->ranks + (size_t)i * 64;
      v[i].out_cores = o.cores + (size_t)i * d * SLOT;
      v[i].out_ranks = o.ranks + (size_t)i * 64;
      v[i].gr = cv.take<cplx>((size_t)MAXD * GR_XF);
      v[i].do_center = (!inverse && shift) ? 1 : 0;
    }
  };
  Carver dry(nullptr);
  TTAlloc o;
  std::vector<XfProb> v;
  plan(dry, o, v);
  run_transform(v, &in->shape, fft, inverse, shift, scale, dry, nullptr, st);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  plan(cv, o, v);
  if ((r = run_transform(v, &in->shape, fft, inverse, shift, scale, cv, in->status, st))) return r;
  *out = new_handle(&in->shape, n, fft->rmax, o, in->status, st);
  return *out ? QTT_OK : fail(QTT_ENOMEM, "host allocation failed");
}

qtt_status qtt_convolve(qtt_tt_t f, qtt_tt_t g, const qtt_trunc* fft, const long long shift[2], double scale,
                        void* ws, size_t ws_bytes, void* stream, qtt_tt_t* out) {
  qtt_status r;
  if (!f || !g || !out) return fail(QTT_EINVAL, "f / g / out is NULL");
  if ((r = check_trunc(fft, RH_MAX, "fft"))) return r;
  if (f->d != g->d) return fail(QTT_EINVAL, "f and g have different d");
  if (g->nt != 1 && g->nt != f->nt) return fail(QTT_EINVAL, "g must hold 1 tensor or as many as f");
  if (f->rcap > RS_XF || g->rcap > RS_XF) return fail(QTT_EINVAL, "input ranks may exceed %d", RS_XF);
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = f->d;
  cudaStream_t st = (cudaStream_t)stream;
  Carver dry(nullptr);
  TTAlloc Y = take_tt(dry, f->nt, d);
  run_convolve(f->cores, f->ranks, f->nt, g->cores, g->ranks, g->nt, &f->shape, fft, shift, scale, Y, dry,
               nullptr, st);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  Y = take_tt(cv, f->nt, d);
  if ((r = run_convolve(f->cores, f->ranks, f->nt, g->cores, g->ranks, g->nt, &f->shape, fft, shift, scale, Y,
                        cv, f->status, st)))
    return r;
  *out = new_handle(&f->shape, f->nt, fft->rmax, Y, f->status, st);
  return *out ? QTT_OK : fail(QTT_ENOMEM, "host allocation failed");
}

qtt_status qtt_to_full(qtt_tt_t t, double* y, double* y_imag, void* ws, size_t ws_bytes, void* stream,
                       qtt_comm_t comm) {
  qtt_status r;
  if (!t || !y) return fail(QTT_EINVAL, "t / y is NULL");
  if (comm) return fail(QTT_EINVAL, "multi-GPU communicators are not supported by this build");
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = t->d;
  const long long ys = t->shape.y_stride ? t->shape.y_stride : (1ll << d);
  cudaStream_t st = (cudaStream_t)stream;
  Carver dry(nullptr);
  run_expand(t->cores, t->ranks, t->nt, d, y, ys, &t->shape, 0, dry, st);
  if ((r = check_ws(dry, ws, ws_bytes))) return r;
  Carver cv(ws);
  if ((r = run_expand(t->cores, t->ranks, t->nt, d, y, ys, &t->shape, 0, cv, st))) return r;
  if (y_imag) {
    Carver cv2(ws);
    if ((r = run_expand(t->cores, t->ranks, t->nt, d, y_imag, ys, &t->shape, 1, cv2, st))) return r;
  }
  return QTT_OK;
}

qtt_status qtt_conv_full(const double* f, const double* g, double* y, const qtt_shape* shape, const qtt_trunc* dec,
                         const qtt_trunc* fft, const long long shift[2], double scale, void* ws, size_t ws_bytes,
                         void* stream, qtt_comm_t comm, qtt_report* rep_host) {
  qtt_status r;
  if ((r = check_shape(shape))) return r;
  if ((r = check_trunc(dec, RS_XF, "dec"))) return r;
  if ((r = check_trunc(fft, RH_MAX, "fft"))) return r;
  if (!f || !g || !y) return fail(QTT_EINVAL, "f / g / y is NULL");
  if (comm) return fail(QTT_EINVAL, "multi-GPU communicators are not supported by this build");
  const size_t need = qtt_workspace_bytes(shape, dec, fft, 1);
  if (!ws) return fail(QTT_EINVAL, "workspace is NULL");
  if (((uintptr_t)ws & 255) != 0) return fail(QTT_EINVAL, "workspace must be 256-byte aligned");
  if (ws_bytes < need) return fail(QTT_ENOMEM, "workspace too small: need %zu bytes, got %zu", need, ws_bytes);
  cudaError_t ce;
  if ((ce = setup_all())) return cuda_check(ce, "kernel setup");
  const int d = shape_d(shape);
  const int nf = shape->batch, ng = shape->g_stride == 0 ? 1 : shape->batch;
  const long long fs = shape->f_stride ? shape->f_stride : (1ll << d);
  const long long gs = shape->g_stride;
  const long long ys = shape->y_stride ? shape->y_stride : (1ll << d);
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (rep_host) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  Carver cv(ws);
  int* status = cv.take<int>(64);
  TTAlloc F = take_tt(cv, nf, d), G = take_tt(cv, ng, d), Y = take_tt(cv, nf, d);
  if ((r = cuda_check(cudaMemsetAsync(status, 0, sizeof(int), st), "status reset"))) return r;
  prof_mark(0, st);
  // Step 1-2: all signals and the kernel(s) in one batched TT-SVD
  {
    const int d_ = d;
    std::vector<DecProb> h(nf + ng);
    for (int i = 0; i < nf + ng; ++i) {
      const bool isf = i < nf;
      const int j = isf ? i : i - nf;
      DecScratch sc = take_dec(cv, d_);
      DecProb& p = h[i];
      p.x = isf ? f + (size_t)j * (size_t)fs : g + (size_t)j * (size_t)gs;
      p.layout = shape->layout;
      p.bx = shape->bits[0];
      p.d = d_;
      p.Wa = sc.Wa; p.Wb = sc.Wb; p.part = sc.part; p.proj = sc.proj; p.tau2 = sc.tau2;
      p.cores = (isf ? F.cores : G.cores) + (size_t)j * d_ * SLOT;
      p.ranks = (isf ? F.ranks : G.ranks) + (size_t)j * 64;
    }
    DecProb* dp = cv.take<DecProb>(nf + ng);
    if ((r = cuda_check(cudaMemcpyAsync(dp, h.data(), h.size() * sizeof(DecProb), cudaMemcpyHostToDevice, st),
                        "copy descriptors")))
      return r;
    DecParams prm{dec->eps, dec->rmax, dec->cluster_tol, status};
    if ((r = cuda_check(launch_ttsvd(dp, nf + ng, d_, prm, st), "TT-SVD launch"))) return r;
  }
  prof_mark(1, st);
  // Step 3
  if ((r = run_convolve(F.cores, F.ranks, nf, G.cores, G.ranks, ng, shape, fft, shift, scale, Y, cv, status, st)))
    return r;
  // Step 4
  if ((r = run_expand(Y.cores, Y.ranks, nf, d, y, ys, shape, 0, cv, st))) return r;
  prof_mark(5, st);
  if (cv.off > ws_bytes) return fail(QTT_ENOMEM, "internal: workspace plan overflow");
  if (rep_host) {
    cudaEventRecord(e1, st);
    if ((r = cuda_check(cudaStreamSynchronize(st), "stream sync"))) return r;
    memset(rep_host, 0, sizeof(*rep_host));
    rep_host->d = d;
    cudaEventElapsedTime(&rep_host->ms_total, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaMemcpy(rep_host->ranks_f, F.ranks, (d + 1) * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(rep_host->ranks_g, G.ranks, (d + 1) * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(rep_host->ranks_out, Y.ranks, (d + 1) * sizeof(int), cudaMemcpyDeviceToHost);
    int hs = 0;
    cudaMemcpy(&hs, status, sizeof(int), cudaMemcpyDeviceToHost);
    rep_host->status_bits = hs;
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

void qtt_profile_enable(int on) { g_prof = on ? 1 : 0; }

int qtt_profile_read(float* ms_host, int n) {
  if (!g_ev_ok || !ms_host || n < PROF_STAGES) return 0;
  if (cudaEventSynchronize(g_ev[PROF_MARKS - 1]) != cudaSuccess) return 0;
  for (int k = 0; k < PROF_STAGES; ++k) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_ev[k], g_ev[k + 1]);
    ms_host[k] = ms;
  }
  return PROF_STAGES;
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
  if ((r = cuda_check(cudaMemsetAsync(status, 0, sizeof(int), st), "status reset"))) return r;
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

}  // extern "C"

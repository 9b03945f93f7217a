// capi.cu — the extern "C" boundary (include/seqreg_b200.h): argument checks,
// per-context scratch, dispatch to the template instantiations, and the host
// pieces that are O(k) or O(n) (Thomas factorisation of the shared tridiagonal).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/seqreg_b200.h"
#include "launch.cuh"
#include "pyramid.cuh"

using namespace sr;

namespace sr {
namespace lbfgs {
struct Workspace;
int minimize(Workspace*& wsp, cudaStream_t st, int sms, long long n, double* x, const sr_lbfgs_options& o,
             sr_objective_fn objective, void* ouser, sr_trace_fn trace, void* tuser, sr_lbfgs_result* res,
             char* err, size_t errlen);
void destroy(Workspace* w);
}  // namespace lbfgs
}  // namespace sr

struct sr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sms = 148;
  int grid_override = 0;
  int legacy = 0;  // SEQREG_B200_LEGACY=1: non-specialized kernels only
  int tc = 1;      // SEQREG_B200_TC=0: SIMT Gram instead of tcgen05 in pass 1
  int graphs = 1;  // SEQREG_B200_GRAPH=0: sr_evaluate launches its kernels one by one (no graph replay)
  float* vbuf = nullptr;  // split pass 1: V = v - shift, [K][vstride]
  size_t vbuf_bytes = 0;
  float* gbuf = nullptr;  // split pass 1 with the streaming pass 2: grad T, [K][d][vstride]
  size_t gbuf_bytes = 0;
  float* ngfbuf = nullptr;  // split NGF path: u, grad T, n, rho, z in one allocation
  size_t ngfbuf_bytes = 0;
  int p2s = 1;            // SEQREG_B200_P2S=0: re-gathering pass 2 instead of the streaming pass 2
  int sample_reuse = 0;   // sr_set_sample_reuse: sr_grad may reuse the samples of the last sr_corr_partial
  // what vbuf / gbuf hold: the samples of this (y, slab, frames, subset); pass 2 reuses them on a match
  struct VTag {
    int valid = 0, k = 0, ndim = 0, has_g = 0;
    const void* y = nullptr;
    const void* frames = nullptr;
    const void* shifts = nullptr;
    int64_t y_off = 0, y_stride = 0, pix_lo = 0, pix_hi = 0, vstride = 0;
    int feature = 0;
    sr::NgfBufs ngf{};  // the split NGF path's buffers and ranges (feature == SR_NGF)
    int frame_index[SR_MAX_FRAMES];
  } vtag;
  // One captured sr_evaluate (CUDA graph): the problem, weights and buffers it was captured for, its own
  // device copy of the per-call constants (Job), the scratch epoch it is valid in, and what the sample
  // buffers hold after it ran (restored into vtag on every replay).
  struct EvalGraph {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec = nullptr;
    Job* job = nullptr;
    unsigned long long epoch = 0;
    unsigned long long last_use = 0;
    int seen = 0;  // evaluations of this key so far (captured on the second)
    VTag vt;
  };
  std::vector<EvalGraph> egraphs;
  unsigned long long graph_clock = 0;
  cudaStream_t cap_stream = nullptr;  // capture stream of the evaluation graphs
  Job* job_dev = nullptr;
  Job* job_host = nullptr;  // pinned staging
  Job job_last{};           // content of the last upload (skip identical re-uploads)
  bool job_valid = false;
  double* part = nullptr;
  size_t part_cap = 0;  // doubles
  unsigned* ticket = nullptr;  // last-block ticket of k_reduce_finalize
  cudaEvent_t order_ev = nullptr;  // orders calls across a change of stream (sr_set_stream)
  sr::lbfgs::Workspace* lbfgs = nullptr;  // device L-BFGS vectors (lbfgs.cu)
  void* zbuf = nullptr;
  size_t zbuf_bytes = 0;
  double* aux = nullptr;  // small device scratch (temporal factors, S partial reduce)
  size_t aux_cap = 0;
  // curvature regulariser of the current sr_evaluate_reg call (alpha > 0): pass 2 adds alpha h L L (y - x)
  // to the gradient and writes S to curv_s (one double)
  double curv_alpha = 0.0, curv_h = 0.0;
  double* curv_s = nullptr;
  double* curv_part = nullptr;
  size_t curv_part_cap = 0;
  // subsets of more than kBlockMax frames: one sub-problem's raw sums, stats, fields and gradient rows
  double* lraw = nullptr;
  size_t lraw_cap = 0;
  double* lstats = nullptr;
  size_t lstats_cap = 0;
  void* ly = nullptr;
  size_t ly_bytes = 0;
  void* lgrad = nullptr;
  size_t lgrad_bytes = 0;
  int* iaux = nullptr;
  size_t iaux_cap = 0;
};


static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(SR_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));        \
  } while (0)

static int kp_of(int k) {
  if (k <= 8) return 8;
  if (k <= 16) return 16;
  if (k <= 32) return 32;
  if (k <= 64) return 64;
  return 128;
}

static bool is_pow2(double s) {
  int e;
  const double m = std::frexp(s, &e);
  return m == 0.5;
}

static Geo make_geo(const sr_grid& gr) {
  Geo g{};
  g.nd = gr.ndim;
  long long st = 1;
  g.pow2 = 1;
  for (int a = 0; a < 3; ++a) {
    const bool used = a < gr.ndim;
    g.n[a] = used ? gr.dims[a] : 1;
    g.st[a] = st;
    st *= g.n[a];
    g.o[a] = used ? gr.origin[a] : 0.0;
    g.s[a] = used ? gr.spacing[a] : 1.0;
    g.inv[a] = 1.0 / g.s[a];
    g.sti[a] = (int)g.st[a];
    g.of[a] = (float)g.o[a];
    g.sf[a] = (float)g.s[a];
    g.invf[a] = (float)g.inv[a];
    if (used && !is_pow2(g.s[a])) g.pow2 = 0;
  }
  g.N = st;
  return g;
}

static int check_grid(const sr_grid& g) {
  if (g.ndim < 2 || g.ndim > 3) return fail(SR_ERR_ARG, "grid must be 2- or 3-dimensional, got %d axes", g.ndim);
  for (int a = 0; a < g.ndim; ++a) {
    if (g.dims[a] < 2) return fail(SR_ERR_ARG, "all dims must be >= 2");
    if (!(g.spacing[a] > 0)) return fail(SR_ERR_ARG, "all spacings must be > 0");
  }
  return SR_OK;
}

// bumped by every scratch (re)allocation: a captured evaluation graph embeds scratch pointers and is
// dropped once the epoch it was captured in has passed
static unsigned long long g_alloc_epoch = 0;

static int ensure(void** p, size_t* cap, size_t need_bytes) {
  if (*cap >= need_bytes) return SR_OK;
  ++g_alloc_epoch;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  CK(cudaMalloc(p, need_bytes));
  *cap = need_bytes;
  return SR_OK;
}

static int ensure_d(double** p, size_t* cap_doubles, size_t need) {
  void* v = *p;
  size_t bytes = *cap_doubles * 8;
  int rc = ensure(&v, &bytes, need * 8);
  *p = (double*)v;
  *cap_doubles = bytes / 8;
  return rc;
}

static int check_problem(sr_ctx* ctx, const sr_problem* p) {
  if (!ctx || !p) return fail(SR_ERR_ARG, "null context or problem");
  int rc = check_grid(p->grid);
  if (rc) return rc;
  if (p->dtype != SR_F32 && p->dtype != SR_F64) return fail(SR_ERR_ARG, "dtype must be SR_F32 or SR_F64");
  if (p->feature != SR_NCC && p->feature != SR_NGF) return fail(SR_ERR_ARG, "feature must be SR_NCC or SR_NGF");
  if (p->param != SR_AFFINE && p->param != SR_DISPLACEMENT) return fail(SR_ERR_ARG, "param must be SR_AFFINE or SR_DISPLACEMENT");
  if (p->k < 1) return fail(SR_ERR_ARG, "subset must be nonempty");
  if (p->k > SR_MAX_FRAMES) return fail(SR_ERR_UNSUPPORTED, "subset of %d frames exceeds SR_MAX_FRAMES=%d", p->k, SR_MAX_FRAMES);
  if (p->feature == SR_NGF && !(p->ngf_eps > 0)) return fail(SR_ERR_ARG, "ngf_eps must be > 0");
  if (!p->frames_dev) return fail(SR_ERR_ARG, "frames_dev is null");
  if (!p->frame_index) return fail(SR_ERR_ARG, "frame_index is null");
  for (int j = 0; j < p->k; ++j)
    if (p->frame_index[j] < 0 || p->frame_index[j] >= p->nframes)
      return fail(SR_ERR_ARG, "frame_index[%d]=%d outside 0..%d", j, p->frame_index[j], p->nframes - 1);
  const Geo g = make_geo(p->grid);
  if (g.N > 2147483647LL) return fail(SR_ERR_UNSUPPORTED, "frames of more than 2^31-1 cells are not supported");
  if (p->pix_lo < 0 || p->pix_hi > g.N || p->pix_lo > p->pix_hi)
    return fail(SR_ERR_ARG, "pixel range [%lld, %lld) outside [0, %lld)", (long long)p->pix_lo, (long long)p->pix_hi, g.N);
  if (p->param == SR_DISPLACEMENT) {
    if (!p->y_dev) return fail(SR_ERR_ARG, "y_dev is null");
    if (p->y_stride < 1) return fail(SR_ERR_ARG, "y_stride must be >= 1");
  } else {
    if (!p->affine) return fail(SR_ERR_ARG, "affine parameters are null");
    const int na = p->grid.ndim * p->grid.ndim + p->grid.ndim;
    for (int i = 0; i < p->k * na; ++i)
      if (!std::isfinite(p->affine[i])) return fail(SR_ERR_ARG, "affine entries must be finite");
  }
  return SR_OK;
}

static Args make_args(sr_ctx* ctx, const sr_problem* p) {
  Args a{};
  a.g = make_geo(p->grid);
  a.frames = p->frames_dev;
  a.shifts = p->shifts_dev;
  a.y = p->y_dev;
  a.y_off = p->y_off;
  a.y_stride = p->y_stride;
  a.job = ctx->job_dev;
  a.K = p->k;
  a.pix_lo = p->pix_lo;
  a.pix_hi = p->pix_hi;
  a.eps = p->ngf_eps;
  return a;
}

// Stage the per-call constants (frame indices, weights, affine rows) and upload them
// when they differ from the last upload.  Identical constants cost nothing, which keeps
// repeated evaluations (and CUDA-graph capture of them) free of host synchronisation.
static void build_job(sr_ctx* ctx, const sr_problem* p, const double* weights, Job& nj) {
  nj = ctx->job_last;
  for (int j = 0; j < p->k; ++j) {
    nj.frame_index[j] = p->frame_index[j];
    if (weights) nj.weights[j] = weights[j];
  }
  if (p->param == SR_AFFINE) {
    const int d = p->grid.ndim, na = d * d + d;
    for (int j = 0; j < p->k; ++j)
      for (int e = 0; e < na; ++e) nj.affine[j * 12 + e] = p->affine[j * na + e];
  }
}

static int upload_job(sr_ctx* ctx, const sr_problem* p, const double* weights) {
  Job nj;
  build_job(ctx, p, weights, nj);
  if (ctx->job_valid && std::memcmp(&nj, &ctx->job_last, sizeof(Job)) == 0) return SR_OK;
  // the previous upload may still be in flight from the pinned staging buffer
  CK(cudaStreamSynchronize(ctx->stream));
  *ctx->job_host = nj;
  CK(cudaMemcpyAsync(ctx->job_dev, ctx->job_host, sizeof(Job), cudaMemcpyHostToDevice, ctx->stream));
  ctx->job_last = nj;
  ctx->job_valid = true;
  return SR_OK;
}

static Launch launch_of(sr_ctx* ctx) {
  return Launch{ctx->stream, ctx->sms, ctx->grid_override, ctx->legacy, ctx->tc};
}

#define SR_SWITCH(dtype, nd, FN, ...)                                    \
  ((dtype) == SR_F32 ? ((nd) == 2 ? FN##_f32_d2(__VA_ARGS__) : FN##_f32_d3(__VA_ARGS__)) \
                     : ((nd) == 2 ? FN##_f64_d2(__VA_ARGS__) : FN##_f64_d3(__VA_ARGS__)))

template <typename T>
static cudaError_t launch_reduce_finalize(sr_ctx* c, const sr_problem* p, int nblk, int KP, long long count,
                                          double* raw, int do_final, double h, double* stats) {
  const size_t dsm = do_final ? (size_t)p->k * p->k * 8 : 0;
  auto kern = k_reduce_finalize<T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(dsm, 1));
  if (e != cudaSuccess) return e;
  const int stride = KP * KP + 3 * KP;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((stride + 31) / 32);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = dsm;
  cfg.stream = c->stream;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kern, (const double*)c->part, nblk, KP, (int)p->k, count, raw, do_final,
                            (const Job*)c->job_dev, (int)p->feature, (int)p->grid.ndim, h, (const T*)p->shifts_dev,
                            stats, c->ticket);
}

// pass 1 over the slab, then the fixed-order cross-CTA reduction into raw (and, with
// stats != nullptr, the finalize in the same launch)
// KP of the pass-1 partial layout: the tcgen05 kernel always uses 32 (frames padded)
// the split NGF path: fp32 displacement fields, K <= 128, tensor-core Gram (KP = 128 partials)
static bool ngf_split(const sr_ctx* c, const sr_problem* p) {
  return p->dtype == SR_F32 && p->feature == SR_NGF && p->param == SR_DISPLACEMENT && p->k <= 128 && !c->legacy &&
         c->tc;
}

static int pass1_kp(const sr_ctx* c, const sr_problem* p) {
  if (p->dtype == SR_F32 && p->feature == SR_NCC && p->param == SR_DISPLACEMENT && p->k <= 32 && !c->legacy &&
      c->tc)
    return 32;
  if (ngf_split(c, p)) return p->k <= 32 ? 32 : p->k <= 64 ? 64 : 128;  // 32: TMA-fed mma.sync Gram
  return kp_of(p->k);
}

static void set_vtag(sr_ctx* c, const sr_problem* p, long long vstride, int has_g) {
  sr_ctx::VTag& t = c->vtag;
  t.valid = 1;
  t.k = p->k;
  t.ndim = p->grid.ndim;
  t.has_g = has_g;
  t.y = p->y_dev;
  t.frames = p->frames_dev;
  t.shifts = p->shifts_dev;
  t.y_off = p->y_off;
  t.y_stride = p->y_stride;
  t.pix_lo = p->pix_lo;
  t.pix_hi = p->pix_hi;
  t.vstride = vstride;
  t.feature = p->feature;
  for (int k = 0; k < p->k; ++k) t.frame_index[k] = p->frame_index[k];
}

// pass 2 may reuse vbuf / gbuf: same y buffer, slab, frames and subset as the last split pass 1
// (the caller's contract: sr_grad follows the sr_corr_* calls at the same y)
static bool vtag_matches(const sr_ctx* c, const sr_problem* p) {
  const sr_ctx::VTag& t = c->vtag;
  if (!t.valid || !t.has_g || t.feature != p->feature || t.k != p->k || t.ndim != p->grid.ndim || t.y != p->y_dev ||
      t.frames != p->frames_dev || t.shifts != p->shifts_dev || t.y_off != p->y_off || t.y_stride != p->y_stride ||
      t.pix_lo != p->pix_lo || t.pix_hi != p->pix_hi)
    return false;
  for (int k = 0; k < p->k; ++k)
    if (t.frame_index[k] != p->frame_index[k]) return false;
  return true;
}

static int corr_partial_impl(sr_ctx* c, const sr_problem* p, double* raw, double h = 0.0,
                             double* stats = nullptr) {
  const int KP = pass1_kp(c, p);
  const size_t stride = (size_t)KP * KP + 3 * KP;
  const size_t want = stride * (size_t)c->sms * 4;
  int rc = ensure_d(&c->part, &c->part_cap, want);
  if (rc) return rc;
  Args a = make_args(c, p);
  const Launch L = launch_of(c);
  int nblk = 0;
  const long long npix = p->pix_hi - p->pix_lo;
  if ((KP == 32 || KP == 64 || KP == 128) && ngf_split(c, p) && npix > 0) {
    const Geo g = a.g;
    const long long row = g.st[g.nd - 1];
    sr::NgfBufs B{};
    B.vlo = std::max<long long>(0, p->pix_lo - 2 * row);
    B.vhi = std::min<long long>(g.N, p->pix_hi + 2 * row);
    B.zlo = std::max<long long>(0, p->pix_lo - row);
    B.zhi = std::min<long long>(g.N, p->pix_hi + row);
    B.vstride = (B.vhi - B.vlo + 3) & ~3LL;
    B.zstride = (B.zhi - B.zlo + 3) & ~3LL;
    const int d = g.nd;
    const size_t nv = (size_t)p->k * B.vstride, nz = (size_t)p->k * B.zstride;
    const size_t total = nv * (2 + d) + nz * (2 * d + 1);  // u, grad T, u lo | n, z, rho
    void* nb = c->ngfbuf;
    rc = ensure(&nb, &c->ngfbuf_bytes, total * 4);
    if (rc) return rc;
    c->ngfbuf = (float*)nb;
    B.V = c->ngfbuf;
    B.G = B.V + nv;
    B.Nf = B.G + nv * d;
    B.Z = B.Nf + nz * d;
    B.Rho = B.Z + nz * d;
    B.VL = B.Rho + nz;
    c->vtag.valid = 0;
    const cudaError_t e1 = KP == 32 ? (d == 2 ? ngf_pass1_mma_d2(L, a, B, c->part, c->part_cap, &nblk)
                                              : ngf_pass1_mma_d3(L, a, B, c->part, c->part_cap, &nblk))
                                    : (d == 2 ? ngf_pass1_d2(L, a, B, c->part, c->part_cap, &nblk)
                                              : ngf_pass1_d3(L, a, B, c->part, c->part_cap, &nblk));
    if (e1 == cudaSuccess) {
      set_vtag(c, p, B.vstride, 1);
      c->vtag.ngf = B;
    } else if (e1 != cudaErrorNotSupported) {
      CK(e1);
    } else {  // layout the tensor map cannot express: the generic kernels with the same KP layout
      CK(SR_SWITCH(p->dtype, p->grid.ndim, pass1, p->feature, p->param, KP, L, a, c->part, c->part_cap, &nblk));
    }
  } else if (KP == 32 && p->dtype == SR_F32 && p->feature == SR_NCC && p->param == SR_DISPLACEMENT && c->tc &&
             !c->legacy && npix > 0) {
    // split NCC pass 1: k_sample_vp (V = v - shift and grad T) + the TMA-fed mma.sync Gram (engine_mma.cuh);
    // SEQREG_B200_P2S=0 leaves V, grad T unused by pass 2 (which then re-gathers)
    const long long vstride = (npix + 3) & ~3LL;  // V = v - shift, [K][vstride]
    void* vb = c->vbuf;
    rc = ensure(&vb, &c->vbuf_bytes, (size_t)p->k * vstride * 4);
    if (rc) return rc;
    c->vbuf = (float*)vb;
    void* gb = c->gbuf;
    rc = ensure(&gb, &c->gbuf_bytes, (size_t)p->k * p->grid.ndim * vstride * 4);
    if (rc) return rc;
    c->gbuf = (float*)gb;
    float* G = c->gbuf;
    c->vtag.valid = 0;
    CK(p->grid.ndim == 2 ? sample_then_gram_d2(L, a, c->vbuf, G, vstride, c->part, c->part_cap, &nblk)
                         : sample_then_gram_d3(L, a, c->vbuf, G, vstride, c->part, c->part_cap, &nblk));
    set_vtag(c, p, vstride, c->p2s);
  } else {
    c->vtag.valid = 0;
    CK(SR_SWITCH(p->dtype, p->grid.ndim, pass1, p->feature, p->param, KP, L, a, c->part, c->part_cap, &nblk));
  }
  const long long count = (long long)(p->pix_hi - p->pix_lo);
  const int fin = stats != nullptr;
  if (p->dtype == SR_F32)
    CK(launch_reduce_finalize<float>(c, p, nblk, KP, count, raw, fin, h, stats));
  else
    CK(launch_reduce_finalize<double>(c, p, nblk, KP, count, raw, fin, h, stats));
  return SR_OK;
}

template <typename T>
static cudaError_t launch_finalize(sr_ctx* c, const sr_problem* p, const double* raw, double h, int64_t n_total,
                                   double* stats) {
  const size_t dsm = (size_t)p->k * p->k * 8;
  auto kern = k_finalize<T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e != cudaSuccess) return e;
  kern<<<1, 1024, dsm, c->stream>>>(raw, c->job_dev, p->k, p->feature, p->grid.ndim, (double)n_total, h,
                                    (const T*)p->shifts_dev, stats);
  return cudaGetLastError();
}

static int finalize_impl(sr_ctx* c, const sr_problem* p, const double* raw, double h, int64_t n_total,
                         double* stats) {
  if (p->dtype == SR_F32) CK(launch_finalize<float>(c, p, raw, h, n_total, stats));
  else CK(launch_finalize<double>(c, p, raw, h, n_total, stats));
  return SR_OK;
}

extern "C" {

int64_t sr_raw_size(int32_t k) { return (int64_t)k * k + 3 * k + 1; }
int64_t sr_stats_size(int32_t k) { return StatsLayout(k).total; }
int64_t sr_stats_offset(int32_t k, int32_t field) {
  const StatsLayout L(k);
  switch (field) {
    case 0: return L.C;
    case 1: return L.sigma;
    case 2: return L.mean;
    case 3: return L.vmax;
    case 4: return L.degen;
    case 5: return L.weights;
    case 6: return L.M;
    case 7: return L.beta;
    case 8: return L.shift;
    case 9: return L.Mf;
    default: return -1;
  }
}

int sr_abi_version(void) { return SR_ABI_VERSION; }
const char* sr_last_error(void) { return g_err.c_str(); }
const char* sr_status_string(int s) {
  switch (s) {
    case SR_OK: return "ok";
    case SR_ERR_ARG: return "invalid argument";
    case SR_ERR_CUDA: return "cuda error";
    case SR_ERR_SINGULAR: return "singular system";
    case SR_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown";
  }
}

int sr_create(int32_t device, sr_ctx** out) {
  if (!out) return fail(SR_ERR_ARG, "out is null");
  *out = nullptr;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(SR_ERR_ARG, "device %d outside 0..%d", device, ndev - 1);
  CK(cudaSetDevice(device));
  sr_ctx* c = new sr_ctx();
  c->device = device;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  c->sms = prop.multiProcessorCount;
  {
    // A/B switches kept for the test suite (tests/test_variants_gpu.py): every one keeps results within
    // tolerance; the slower kernel variants of round 1 were removed
    const char* lg = getenv("SEQREG_B200_LEGACY");
    c->legacy = (lg && lg[0] == '1') ? 1 : 0;
    const char* tcs = getenv("SEQREG_B200_TC");
    c->tc = (tcs && tcs[0] == '0') ? 0 : 1;
    const char* ps = getenv("SEQREG_B200_P2S");
    c->p2s = (ps && ps[0] == '0') ? 0 : 1;
    const char* gr = getenv("SEQREG_B200_GRAPH");
    c->graphs = (gr && gr[0] == '0') ? 0 : 1;
  }
  CK(cudaMalloc(&c->job_dev, sizeof(Job)));
  CK(cudaMalloc(&c->ticket, sizeof(unsigned)));
  CK(cudaMemset(c->ticket, 0, sizeof(unsigned)));
  CK(cudaMallocHost(&c->job_host, sizeof(Job)));
  std::memset(c->job_host, 0, sizeof(Job));
  *out = c;
  return SR_OK;
}

int sr_destroy(sr_ctx* c) {
  if (!c) return SR_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaFree(c->job_dev);
  cudaFreeHost(c->job_host);
  cudaFree(c->part);
  cudaFree(c->ticket);
  cudaFree(c->curv_part);
  cudaFree(c->lraw);
  cudaFree(c->lstats);
  cudaFree(c->ly);
  cudaFree(c->lgrad);
  if (c->order_ev) cudaEventDestroy(c->order_ev);
  sr::lbfgs::destroy(c->lbfgs);
  cudaFree(c->vbuf);
  cudaFree(c->gbuf);
  cudaFree(c->ngfbuf);
  cudaFree(c->zbuf);
  cudaFree(c->aux);
  cudaFree(c->iaux);
  for (auto& eg : c->egraphs) {
    if (eg.exec) cudaGraphExecDestroy(eg.exec);
    cudaFree(eg.job);
  }
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
  return SR_OK;
}

// A context's scratch (job constants, partials, tickets, split-path buffers) is shared by every call, so
// calls issued from different streams must not overlap: when the stream changes, the new stream waits
// for everything already queued on the previous one (an event, no host synchronisation).
int sr_set_stream(sr_ctx* c, void* stream) {
  if (!c) return fail(SR_ERR_ARG, "null context");
  const cudaStream_t ns = (cudaStream_t)stream;
  if (ns != c->stream) {
    cudaStreamCaptureStatus a = cudaStreamCaptureStatusNone, b = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(c->stream, &a));
    CK(cudaStreamIsCapturing(ns, &b));
    if (a == cudaStreamCaptureStatusNone && b == cudaStreamCaptureStatusNone) {
      if (!c->order_ev) CK(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming));
      CK(cudaEventRecord(c->order_ev, c->stream));
      CK(cudaStreamWaitEvent(ns, c->order_ev, 0));
    }
    c->stream = ns;
  }
  return SR_OK;
}

int sr_set_sample_reuse(sr_ctx* c, int32_t enable) {
  if (!c) return fail(SR_ERR_ARG, "null context");
  c->sample_reuse = enable ? 1 : 0;
  return SR_OK;
}

int sr_set_grid_ctas(sr_ctx* c, int32_t ctas) {
  if (!c) return fail(SR_ERR_ARG, "null context");
  if (ctas < 0) return fail(SR_ERR_ARG, "ctas must be >= 0");
  c->grid_override = ctas;
  return SR_OK;
}


int sr_frame_shifts(sr_ctx* c, int32_t dtype, const void* frames, int32_t nframes, int64_t n,
                    void* shifts) {
  if (!c || !frames || !shifts || nframes < 1 || n < 1) return fail(SR_ERR_ARG, "bad sr_frame_shifts arguments");
  CK(cudaSetDevice(c->device));
  if (dtype == SR_F32)
    k_frame_mean<float><<<nframes, 1024, 0, c->stream>>>((const float*)frames, n, (float*)shifts);
  else
    k_frame_mean<double><<<nframes, 1024, 0, c->stream>>>((const double*)frames, n, (double*)shifts);
  CK(cudaGetLastError());
  return SR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- subsets of more than kBlockMax frames
// (ADVICE: the paper's schedule build_temporal_levels(129, 17) ends with a 129-frame level.)  The subset is
// cut into blocks of kBlockFrames; pass 1 runs once per pair of blocks (<= 128 frames per launch) and its
// raw sums are scattered into the K x K ones; the finalize runs on all K frames; pass 2 runs once per
// (input block, output block) with the gradient coefficients restricted to that block pair (k_sub_stats) and
// the output rows accumulated into the gradient (k_acc_rows).  Each kernel is unchanged, so the results are
// the single-launch arithmetic up to the order of the pass-2 sums over input blocks.
static constexpr int kBlockFrames = 64;

static SubIdx sub_blocks(int K, int bi, int bj) {  // frames of block bi (then block bj when different)
  SubIdx s{};
  auto add = [&](int b, unsigned char part) {
    for (int f = b * kBlockFrames; f < std::min(K, (b + 1) * kBlockFrames); ++f) {
      s.idx[s.n] = f;
      s.part[s.n] = part;
      ++s.n;
    }
  };
  if (bi == bj) {
    add(bi, 2);
  } else {
    add(bi, 0);
    add(bj, 1);
  }
  return s;
}

struct SubProblem {
  sr_problem q;
  std::vector<int32_t> fi;
  std::vector<double> aff;
};

// the sub-problem of frames s.idx (the displacement fields gathered into ctx->ly)
static int make_sub(sr_ctx* c, const sr_problem* p, const SubIdx& s, SubProblem& sp) {
  sp.q = *p;
  sp.q.k = s.n;
  sp.fi.resize(s.n);
  for (int i = 0; i < s.n; ++i) sp.fi[i] = p->frame_index[s.idx[i]];
  sp.q.frame_index = sp.fi.data();
  const int d = p->grid.ndim;
  if (p->param == SR_AFFINE) {
    const int na = d * d + d;
    sp.aff.resize((size_t)s.n * na);
    for (int i = 0; i < s.n; ++i)
      for (int e = 0; e < na; ++e) sp.aff[(size_t)i * na + e] = p->affine[(size_t)s.idx[i] * na + e];
    sp.q.affine = sp.aff.data();
    return SR_OK;
  }
  const size_t esz = p->dtype == SR_F32 ? 4 : 8;
  const long long row = (long long)d * p->y_stride;
  int rc = ensure(&c->ly, &c->ly_bytes, (size_t)kBlockMax * row * esz);
  if (rc) return rc;
  const dim3 grid((unsigned)std::min<long long>((row + 255) / 256, 4096), (unsigned)s.n);
  if (p->dtype == SR_F32)
    k_gather_rows<float><<<grid, 256, 0, c->stream>>>((const float*)p->y_dev, row, s, (float*)c->ly);
  else
    k_gather_rows<double><<<grid, 256, 0, c->stream>>>((const double*)p->y_dev, row, s, (double*)c->ly);
  CK(cudaGetLastError());
  sp.q.y_dev = c->ly;
  return SR_OK;
}

static int corr_partial_large(sr_ctx* c, const sr_problem* p, double* raw) {
  const int K = p->k, nb = (K + kBlockFrames - 1) / kBlockFrames;
  CK(cudaMemsetAsync(raw, 0, sizeof(double) * (size_t)sr_raw_size(K), c->stream));
  int rc = ensure_d(&c->lraw, &c->lraw_cap, (size_t)sr_raw_size(kBlockMax));
  if (rc) return rc;
  for (int bi = 0; bi < nb; ++bi)
    for (int bj = bi + 1; bj < nb; ++bj) {
      const SubIdx s = sub_blocks(K, bi, bj);
      SubProblem sp;
      rc = make_sub(c, p, s, sp);
      if (rc) return rc;
      rc = upload_job(c, &sp.q, nullptr);
      if (rc) return rc;
      rc = corr_partial_impl(c, &sp.q, c->lraw);
      if (rc) return rc;
      k_scatter_raw<<<64, 256, 0, c->stream>>>(c->lraw, s, K, raw);
      CK(cudaGetLastError());
    }
  c->vtag.valid = 0;  // the split paths' samples belong to the last sub-problem
  return SR_OK;
}

extern "C" {  // (defined below, inside the boundary's extern "C" block)
static int grad_impl_core(sr_ctx* c, const sr_problem* p, const double* stats, void* grad, int64_t g_off,
                          int64_t g_stride, bool reuse, bool* curv_done);
}

static int grad_large(sr_ctx* c, const sr_problem* p, const double* stats, void* grad, int64_t g_off,
                      int64_t g_stride) {
  const int K = p->k, nb = (K + kBlockFrames - 1) / kBlockFrames, d = p->grid.ndim;
  const bool aff = p->param == SR_AFFINE;
  const size_t esz = aff ? 8 : (p->dtype == SR_F32 ? 4 : 8);
  const long long row = aff ? d * d + d : (long long)d * g_stride;
  int rc = ensure_d(&c->lstats, &c->lstats_cap, (size_t)StatsLayout(kBlockMax).total);
  if (rc) return rc;
  rc = ensure(&c->lgrad, &c->lgrad_bytes, (size_t)kBlockMax * row * esz);
  if (rc) return rc;
  for (int bj = 0; bj < nb; ++bj)
    for (int bi = 0; bi < nb; ++bi) {
      const SubIdx s = sub_blocks(K, bi, bj);
      SubProblem sp;
      rc = make_sub(c, p, s, sp);
      if (rc) return rc;
      rc = upload_job(c, &sp.q, nullptr);
      if (rc) return rc;
      k_sub_stats<<<64, 256, 0, c->stream>>>(stats, K, s, bi == 0 ? 1 : 0, c->lstats);
      CK(cudaGetLastError());
      bool done = false;
      rc = grad_impl_core(c, &sp.q, c->lstats, c->lgrad, g_off, g_stride, false, &done);
      if (rc) return rc;
      const dim3 grid((unsigned)std::min<long long>((row + 255) / 256, 4096), (unsigned)s.n);
      if (esz == 4)
        k_acc_rows<float><<<grid, 256, 0, c->stream>>>((const float*)c->lgrad, row, s, bi == 0, (float*)grad);
      else
        k_acc_rows<double><<<grid, 256, 0, c->stream>>>((const double*)c->lgrad, row, s, bi == 0, (double*)grad);
      CK(cudaGetLastError());
    }
  return SR_OK;
}

extern "C" {

int sr_corr_partial(sr_ctx* c, const sr_problem* p, double* raw_dev) {
  int rc = check_problem(c, p);
  if (rc) return rc;
  if (!raw_dev) return fail(SR_ERR_ARG, "raw_dev is null");
  CK(cudaSetDevice(c->device));
  if (p->k > kBlockMax) return corr_partial_large(c, p, raw_dev);
  rc = upload_job(c, p, nullptr);
  if (rc) return rc;
  return corr_partial_impl(c, p, raw_dev);
}

int sr_corr_finalize(sr_ctx* c, const sr_problem* p, const double* raw_dev, const double* weights,
                     double cell_volume, int64_t n_total, double* stats_dev) {
  int rc = check_problem(c, p);
  if (rc) return rc;
  if (!raw_dev || !stats_dev || !weights) return fail(SR_ERR_ARG, "null raw/stats/weights");
  if (n_total < 2) return fail(SR_ERR_ARG, "feature needs at least 2 values");
  CK(cudaSetDevice(c->device));
  rc = upload_job(c, p, weights);
  if (rc) return rc;
  return finalize_impl(c, p, raw_dev, cell_volume, n_total, stats_dev);
}

static int curvature_impl(sr_ctx* c, const sr_problem* p, double alpha, double h, void* grad, int64_t g_off,
                          int64_t g_stride, double* s_out);

// bool *curv_done: the pass-2 kernel added the curvature term itself (the split NGF path)
static int grad_impl_core(sr_ctx* c, const sr_problem* p, const double* stats, void* grad, int64_t g_off,
                          int64_t g_stride, bool reuse, bool* curv_done) {
  const int KP = kp_of(p->k);
  const int d = p->grid.ndim, na = d * d + d;
  const Launch L = launch_of(c);
  Args a = make_args(c, p);
  a.stats = stats;
  const size_t esz = p->dtype == SR_F32 ? 4 : 8;
  // affine partial scratch: pass 2 NCC [grid][KP][na]; NGF adjoint [K][blocks][na]
  const long long npix = p->pix_hi - p->pix_lo;
  const size_t aff_need = std::max((size_t)c->sms * 8 * KP * na,
                                   (size_t)p->k * (size_t)((npix + 255) / 256 + 1) * na);
  int rc = ensure_d(&c->aux, &c->aux_cap, aff_need);
  if (rc) return rc;
  int nblk = 0;
  if (p->feature == SR_NCC) {
    a.out = grad;
    a.o_off = g_off;
    a.o_stride = g_stride;
    if (reuse && p->dtype == SR_F32 && p->param == SR_DISPLACEMENT && p->k <= 32 && vtag_matches(c, p)) {
      const long long lim = 1LL << 31;  // k_pass2_mma uses 32-bit element offsets
      if ((long long)p->k * d * c->vtag.vstride < lim && (long long)p->k * d * g_stride < lim)
        CK(d == 2 ? pass2_mma_d2(L, a, c->vbuf, c->gbuf, c->vtag.vstride)
                  : pass2_mma_d3(L, a, c->vbuf, c->gbuf, c->vtag.vstride));
      else
        CK(d == 2 ? pass2_stream_d2(L, a, c->vbuf, c->gbuf, c->vtag.vstride)
                  : pass2_stream_d3(L, a, c->vbuf, c->gbuf, c->vtag.vstride));
      return SR_OK;
    }
    CK(SR_SWITCH(p->dtype, d, pass2, p->feature, p->param, KP, L, a, c->aux, c->aux_cap, &nblk));
    if (p->param == SR_AFFINE) {
      const int warps = p->k * na;
      k_affine_rows<<<(warps * 32 + 255) / 256, 256, 0, c->stream>>>(c->aux, nblk, KP, p->k, na, 0, (double*)grad);
      CK(cudaGetLastError());
    }
    return SR_OK;
  }
  if (reuse && ngf_split(c, p) && vtag_matches(c, p)) {  // split NGF pass 2: no re-sampling
    a.out = grad;
    a.o_off = g_off;
    a.o_stride = g_stride;
    const bool fuse = c->curv_alpha > 0 && p->param == SR_DISPLACEMENT && p->dtype == SR_F32;
    int nb = 0;
    if (fuse) {  // the curvature term inside k_ngf_adj4 (one pass-2 launch, no read-modify-write of grad)
      nb = (int)((npix + 1023) / 1024) * p->k;
      rc = ensure_d(&c->curv_part, &c->curv_part_cap, (size_t)nb);
      if (rc) return rc;
      a.curv_alpha = c->curv_alpha;
      a.curv_h = c->curv_h;
      a.curv_part = c->curv_part;
    }
    CK(d == 2 ? ngf_pass2_d2(L, a, c->vtag.ngf) : ngf_pass2_d3(L, a, c->vtag.ngf));
    if (fuse) {
      k_sum1<<<1, 1024, 0, c->stream>>>(c->curv_part, nb, c->curv_s);
      CK(cudaGetLastError());
      *curv_done = true;
    }
    return SR_OK;
  }
  // NGF: z over the slab extended by one slowest-axis row on each side (the adjoint stencil)
  const Geo g = a.g;
  const long long row = g.st[d - 1];
  const long long zlo = std::max<long long>(0, p->pix_lo - row);
  const long long zhi = std::min<long long>(g.N, p->pix_hi + row);
  const long long zs = zhi - zlo;
  rc = ensure(&c->zbuf, &c->zbuf_bytes, (size_t)p->k * d * zs * esz);
  if (rc) return rc;
  Args z = a;
  z.pix_lo = zlo;
  z.pix_hi = zhi;
  z.out = c->zbuf;
  z.o_off = zlo;
  z.o_stride = zs;
  CK(SR_SWITCH(p->dtype, d, pass2, p->feature, p->param, KP, L, z, c->aux, c->aux_cap, &nblk));
  a.out = grad;
  a.o_off = g_off;
  a.o_stride = g_stride;
  CK(SR_SWITCH(p->dtype, d, adjoint, p->param, L, a, c->zbuf, zlo, zs, c->aux, c->aux_cap, &nblk));
  if (p->param == SR_AFFINE) {
    const int warps = p->k * na;
    k_affine_rows<<<(warps * 32 + 255) / 256, 256, 0, c->stream>>>(c->aux, nblk, KP, p->k, na, 1, (double*)grad);
    CK(cudaGetLastError());
  }
  return SR_OK;
}

static int grad_impl(sr_ctx* c, const sr_problem* p, const double* stats, void* grad, int64_t g_off,
                     int64_t g_stride, bool reuse) {
  bool done = false;
  int rc = grad_impl_core(c, p, stats, grad, g_off, g_stride, reuse, &done);
  if (rc || done || !(c->curv_alpha > 0) || p->param != SR_DISPLACEMENT) return rc;
  // every other pass 2: the curvature kernel after it (adds into grad)
  return curvature_impl(c, p, c->curv_alpha, c->curv_h, grad, g_off, g_stride, c->curv_s);
}

int sr_grad(sr_ctx* c, const sr_problem* p, const double* stats_dev, void* grad_dev, int64_t g_off,
            int64_t g_stride) {
  int rc = check_problem(c, p);
  if (rc) return rc;
  if (!stats_dev || !grad_dev) return fail(SR_ERR_ARG, "null stats/grad");
  if (p->param == SR_DISPLACEMENT && g_stride < 1) return fail(SR_ERR_ARG, "g_stride must be >= 1");
  CK(cudaSetDevice(c->device));
  if (p->k > kBlockMax) return grad_large(c, p, stats_dev, grad_dev, g_off, g_stride);
  rc = upload_job(c, p, nullptr);
  if (rc) return rc;
  return grad_impl(c, p, stats_dev, grad_dev, g_off, g_stride, c->sample_reuse != 0);
}

static int evaluate_impl(sr_ctx* c, const sr_problem* p, double cell_volume, double* raw_dev, double* stats_dev,
                         void* grad_dev) {
  int rc = corr_partial_impl(c, p, raw_dev, cell_volume, stats_dev);
  if (rc) return rc;
  if (!grad_dev) return SR_OK;
  return grad_impl(c, p, stats_dev, grad_dev, p->y_off, p->param == SR_DISPLACEMENT ? p->y_stride : 0, true);
}

// Everything an evaluation's launches depend on: the problem's scalars and device pointers, the subset,
// weights, affine parameters, cell volume and output buffers (the scratch pointers are covered by the
// allocation epoch).
static std::vector<unsigned char> eval_key(const sr_problem* p, const double* weights, double cell_volume,
                                           const double* raw_dev, const double* stats_dev, const void* grad_dev) {
  std::vector<unsigned char> k;
  auto put = [&](const void* v, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(v);
    k.insert(k.end(), b, b + n);
  };
  sr_problem q = *p;
  q.frame_index = nullptr;
  q.affine = nullptr;
  put(&q, sizeof q);
  put(p->frame_index, sizeof(int32_t) * p->k);
  put(weights, sizeof(double) * p->k);
  if (p->param == SR_AFFINE) put(p->affine, sizeof(double) * p->k * (p->grid.ndim * p->grid.ndim + p->grid.ndim));
  put(&cell_volume, sizeof cell_volume);
  put(&raw_dev, sizeof raw_dev);
  put(&stats_dev, sizeof stats_dev);
  put(&grad_dev, sizeof grad_dev);
  return k;
}

static void key_put_curv(std::vector<unsigned char>& k, const sr_ctx* c) {
  const unsigned char* b = reinterpret_cast<const unsigned char*>(&c->curv_alpha);
  k.insert(k.end(), b, b + sizeof(double));
  b = reinterpret_cast<const unsigned char*>(&c->curv_h);
  k.insert(k.end(), b, b + sizeof(double));
  b = reinterpret_cast<const unsigned char*>(&c->curv_s);
  k.insert(k.end(), b, b + sizeof(double*));
}

int sr_evaluate_reg(sr_ctx* c, const sr_problem* p, const double* weights, double cell_volume, double alpha,
                    double* raw_dev, double* stats_dev, void* grad_dev, double* s_out_dev) {
  if (!c) return fail(SR_ERR_ARG, "null context");
  if (alpha > 0) {
    if (!p || p->param != SR_DISPLACEMENT) return fail(SR_ERR_ARG, "the curvature regulariser acts on displacement fields");
    if (!grad_dev || !s_out_dev) return fail(SR_ERR_ARG, "null grad/s_out");
  } else if (alpha < 0 || alpha != alpha) {
    return fail(SR_ERR_ARG, "alpha must be >= 0");
  }
  c->curv_alpha = alpha > 0 ? alpha : 0.0;
  c->curv_h = alpha > 0 ? cell_volume : 0.0;
  c->curv_s = alpha > 0 ? s_out_dev : nullptr;
  const int rc = sr_evaluate(c, p, weights, cell_volume, raw_dev, stats_dev, grad_dev);
  c->curv_alpha = 0.0;
  c->curv_h = 0.0;
  c->curv_s = nullptr;
  return rc;
}

int sr_evaluate(sr_ctx* c, const sr_problem* p, const double* weights, double cell_volume,
                double* raw_dev, double* stats_dev, void* grad_dev) {
  int rc = check_problem(c, p);
  if (rc) return rc;
  if (!raw_dev || !stats_dev || !weights) return fail(SR_ERR_ARG, "null raw/stats/weights");
  const Geo g = make_geo(p->grid);
  if (p->pix_lo != 0 || p->pix_hi != g.N) return fail(SR_ERR_ARG, "sr_evaluate covers the whole grid");
  CK(cudaSetDevice(c->device));
  if (p->k > kBlockMax) {  // frame blocks (no graph replay)
    rc = corr_partial_large(c, p, raw_dev);
    if (rc) return rc;
    rc = upload_job(c, p, weights);
    if (rc) return rc;
    rc = finalize_impl(c, p, raw_dev, cell_volume, g.N, stats_dev);
    if (rc || !grad_dev) return rc;
    rc = grad_large(c, p, stats_dev, grad_dev, p->y_off, p->param == SR_DISPLACEMENT ? p->y_stride : 0);
    if (rc) return rc;
    if (c->curv_alpha > 0 && p->param == SR_DISPLACEMENT)
      return curvature_impl(c, p, c->curv_alpha, c->curv_h, grad_dev, p->y_off, p->y_stride, c->curv_s);
    return SR_OK;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(c->stream, &cs));
  if (!c->graphs || cs != cudaStreamCaptureStatusNone) {  // (the caller may be capturing)
    rc = upload_job(c, p, weights);
    if (rc) return rc;
    return evaluate_impl(c, p, cell_volume, raw_dev, stats_dev, grad_dev);
  }
  // CUDA-graph replay of a repeated evaluation (the objective inside an optimiser loop): one graph
  // launch instead of the per-kernel launches.  A key is captured on its second evaluation (the first
  // runs eagerly and sizes every scratch buffer); the graph reads its own device copy of the Job.
  std::vector<unsigned char> key = eval_key(p, weights, cell_volume, raw_dev, stats_dev, grad_dev);
  key_put_curv(key, c);
  sr_ctx::EvalGraph* eg = nullptr;
  for (auto& e : c->egraphs)
    if (e.key == key) eg = &e;
  if (eg && eg->exec && eg->epoch != g_alloc_epoch) {  // scratch moved since the capture
    cudaGraphExecDestroy(eg->exec);
    eg->exec = nullptr;
    eg->seen = 0;
  }
  if (eg && eg->exec) {
    eg->last_use = ++c->graph_clock;
    c->vtag = eg->vt;
    CK(cudaGraphLaunch(eg->exec, c->stream));
    return SR_OK;
  }
  if (!eg) {
    if (c->egraphs.size() >= 8) {  // replace the least recently used entry
      auto lru = std::min_element(c->egraphs.begin(), c->egraphs.end(),
                                  [](const sr_ctx::EvalGraph& x, const sr_ctx::EvalGraph& y) {
                                    return x.last_use < y.last_use;
                                  });
      if (lru->exec) cudaGraphExecDestroy(lru->exec);
      cudaFree(lru->job);
      c->egraphs.erase(lru);
    }
    c->egraphs.push_back(sr_ctx::EvalGraph{});
    eg = &c->egraphs.back();
    eg->key = key;
  }
  eg->last_use = ++c->graph_clock;
  if (eg->seen++ == 0) {  // first evaluation of this key: eager
    rc = upload_job(c, p, weights);
    if (rc) return rc;
    return evaluate_impl(c, p, cell_volume, raw_dev, stats_dev, grad_dev);
  }
  // second evaluation: capture (scratch is sized by the eager run), then launch
  Job nj;
  build_job(c, p, weights, nj);
  if (!eg->job) CK(cudaMalloc(&eg->job, sizeof(Job)));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(eg->job, &nj, sizeof(Job), cudaMemcpyHostToDevice));
  const unsigned long long epoch = g_alloc_epoch;
  Job* saved = c->job_dev;
  c->job_dev = eg->job;
  // capture on a private stream (the legacy default stream cannot be captured); the graph is then
  // launched into the context's stream
  if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  const cudaStream_t user_stream = c->stream;
  c->stream = c->cap_stream;
  cudaGraph_t graph = nullptr;
  cudaError_t be = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
  rc = be == cudaSuccess ? evaluate_impl(c, p, cell_volume, raw_dev, stats_dev, grad_dev) : SR_OK;
  const cudaError_t ce = be == cudaSuccess ? cudaStreamEndCapture(c->stream, &graph) : be;
  c->stream = user_stream;
  c->job_dev = saved;
  if (rc == SR_OK && ce == cudaSuccess && epoch == g_alloc_epoch) {
    const cudaError_t ie = cudaGraphInstantiate(&eg->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie == cudaSuccess) {
      eg->epoch = epoch;
      eg->vt = c->vtag;
      CK(cudaGraphLaunch(eg->exec, c->stream));
      return SR_OK;
    }
    eg->exec = nullptr;
  } else if (graph) {
    cudaGraphDestroy(graph);
  }
  cudaGetLastError();  // clear a capture error; fall back to the eager path for this call
  c->graphs = 0;       // and for the rest of this context's life
  rc = upload_job(c, p, weights);
  if (rc) return rc;
  return evaluate_impl(c, p, cell_volume, raw_dev, stats_dev, grad_dev);
}

int sr_curvature(sr_ctx* c, const sr_problem* p, double alpha, double h, void* grad, int64_t g_off,
                 int64_t g_stride, double* s_out) {
  int rc = check_problem(c, p);
  if (rc) return rc;
  if (p->param != SR_DISPLACEMENT) return fail(SR_ERR_ARG, "the curvature regulariser acts on displacement fields");
  if (!grad || !s_out) return fail(SR_ERR_ARG, "null grad/s_out");
  CK(cudaSetDevice(c->device));
  return curvature_impl(c, p, alpha, h, grad, g_off, g_stride, s_out);
}

static int curvature_impl(sr_ctx* c, const sr_problem* p, double alpha, double h, void* grad, int64_t g_off,
                          int64_t g_stride, double* s_out) {
  int rc = SR_OK;
  const int d = p->grid.ndim;
  const long long npix = p->pix_hi - p->pix_lo;
  const size_t need = (size_t)((npix + 255) / 256 + 1) * p->k * d;
  rc = ensure_d(&c->aux, &c->aux_cap, need);
  if (rc) return rc;
  Args a = make_args(c, p);
  a.out = grad;
  a.o_off = g_off;
  a.o_stride = g_stride;
  int nb = 0;
  CK(SR_SWITCH(p->dtype, d, curvature, launch_of(c), a, alpha, h, c->aux, c->aux_cap, &nb));
  k_sum1<<<1, 1024, 0, c->stream>>>(c->aux, nb, s_out);
  CK(cudaGetLastError());
  return SR_OK;
}

int sr_sample(sr_ctx* c, const sr_problem* p, void* out_dev) {
  int rc = check_problem(c, p);
  if (rc) return rc;
  if (!out_dev) return fail(SR_ERR_ARG, "null out");
  CK(cudaSetDevice(c->device));
  rc = upload_job(c, p, nullptr);
  if (rc) return rc;
  Args a = make_args(c, p);
  CK(SR_SWITCH(p->dtype, p->grid.ndim, sample, p->param, launch_of(c), a, out_dev));
  return SR_OK;
}

int sr_ls_predict(sr_ctx* c, int32_t dtype, int32_t n, int64_t m, const uint8_t* mask, double beta,
                  const void* eta, const void* ref, void* zeta) {
  if (!c || !mask || !eta || !ref || !zeta) return fail(SR_ERR_ARG, "null argument");
  if (!(beta > 0)) return fail(SR_ERR_ARG, "beta must be > 0");
  if (n < 2) return fail(SR_ERR_ARG, "need at least 2 frames");
  if (m < 1) return fail(SR_ERR_ARG, "m must be >= 1");
  // shared tridiagonal factor, exactly thomas_solve's recurrences (temporal.py:166-191)
  std::vector<double> fac(3 * (size_t)n);
  double* mk = fac.data();
  double* cp = mk + n;
  double* piv = cp + n;
  std::vector<double> diag(n);
  double dmax = 0.0;
  for (int i = 0; i < n; ++i) {
    mk[i] = mask[i] ? 1.0 : 0.0;
    const double lap = (i == 0 || i == n - 1) ? 1.0 : 2.0;
    diag[i] = mk[i] + beta * lap;
    dmax = std::max(dmax, std::fabs(diag[i]));
  }
  const double tol = 1e-14 * dmax, off = -beta;
  double p0 = diag[0];
  if (std::fabs(p0) <= tol) return fail(SR_ERR_SINGULAR, "zero pivot at row 0");
  piv[0] = p0;
  cp[0] = off / p0;
  for (int i = 1; i < n; ++i) {
    const double pv = diag[i] - off * cp[i - 1];
    if (std::fabs(pv) <= tol) return fail(SR_ERR_SINGULAR, "zero pivot at row %d", i);
    piv[i] = pv;
    cp[i] = i < n - 1 ? off / pv : 0.0;
  }
  CK(cudaSetDevice(c->device));
  int rc = ensure_d(&c->aux, &c->aux_cap, fac.size());
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->aux, fac.data(), fac.size() * 8, cudaMemcpyHostToDevice, c->stream));
  const int blocks = (int)((m + 255) / 256);
  if (dtype == SR_F32)
    k_ls_predict<float><<<blocks, 256, 0, c->stream>>>(n, m, c->aux, beta, (const float*)eta, (const float*)ref, (float*)zeta);
  else
    k_ls_predict<double><<<blocks, 256, 0, c->stream>>>(n, m, c->aux, beta, (const double*)eta, (const double*)ref, (double*)zeta);
  CK(cudaGetLastError());
  // the host factor buffer is stack/heap memory: make the copy complete before returning
  CK(cudaStreamSynchronize(c->stream));
  return SR_OK;
}

int sr_interp_linear(sr_ctx* c, int32_t dtype, int32_t n, int64_t m, const int32_t* left,
                     const int32_t* right, const double* theta, const void* src, void* zeta) {
  if (!c || !left || !right || !theta || !src || !zeta) return fail(SR_ERR_ARG, "null argument");
  if (n < 1 || m < 1) return fail(SR_ERR_ARG, "bad sizes");
  CK(cudaSetDevice(c->device));
  // pack [left | right] as ints and theta as doubles into device scratch
  void* ip = c->iaux;
  size_t icap = c->iaux_cap * 4;
  int rc = ensure(&ip, &icap, (size_t)2 * n * 4);
  if (rc) return rc;
  c->iaux = (int*)ip;
  c->iaux_cap = icap / 4;
  rc = ensure_d(&c->aux, &c->aux_cap, n);
  if (rc) return rc;
  std::vector<int> lr(2 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    lr[i] = left[i];
    lr[n + i] = right[i];
  }
  CK(cudaMemcpyAsync(c->iaux, lr.data(), lr.size() * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->aux, theta, (size_t)n * 8, cudaMemcpyHostToDevice, c->stream));
  dim3 grid((unsigned)((m + 255) / 256), n);
  if (dtype == SR_F32)
    k_interp_linear<float><<<grid, 256, 0, c->stream>>>(n, m, c->iaux, c->iaux + n, c->aux, (const float*)src, (float*)zeta);
  else
    k_interp_linear<double><<<grid, 256, 0, c->stream>>>(n, m, c->iaux, c->iaux + n, c->aux, (const double*)src, (double*)zeta);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return SR_OK;
}

int sr_pyramid_step(sr_ctx* c, int32_t dtype, int32_t ndim, const int32_t* dims, int32_t nframes,
                    const void* src_dev, void* dst_dev) {
  if (!c || !dims || !src_dev || !dst_dev) return fail(SR_ERR_ARG, "null argument");
  if (ndim < 1 || ndim > 3 || nframes < 1) return fail(SR_ERR_ARG, "bad ndim/nframes");
  if (dtype != SR_F32 && dtype != SR_F64) return fail(SR_ERR_ARG, "bad dtype");
  PyrDims f{ndim, {1, 1, 1}, 1}, cg{ndim, {1, 1, 1}, 1};
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1) return fail(SR_ERR_ARG, "dims must be >= 1");
    f.n[a] = dims[a];
    cg.n[a] = (dims[a] + 1) / 2;  // ceil(dims / 2) (pyramid.py:48)
    f.N *= dims[a];
    cg.N *= cg.n[a];
  }
  CK(cudaSetDevice(c->device));
  if (cg.n[1] * cg.n[2] > 65535 || nframes > 65535 || f.N > (1LL << 31)) return fail(SR_ERR_ARG, "stack too large");
  const dim3 grid((unsigned)((cg.n[0] + 127) / 128), (unsigned)(cg.n[1] * cg.n[2]), (unsigned)nframes);
  if (dtype == SR_F32) {
    if (ndim == 3) k_pyramid<float, true><<<grid, 128, 0, c->stream>>>((const float*)src_dev, (float*)dst_dev, f, cg);
    else k_pyramid<float, false><<<grid, 128, 0, c->stream>>>((const float*)src_dev, (float*)dst_dev, f, cg);
  } else {
    if (ndim == 3) k_pyramid<double, true><<<grid, 128, 0, c->stream>>>((const double*)src_dev, (double*)dst_dev, f, cg);
    else k_pyramid<double, false><<<grid, 128, 0, c->stream>>>((const double*)src_dev, (double*)dst_dev, f, cg);
  }
  CK(cudaGetLastError());
  return SR_OK;
}

int sr_prolong_field(sr_ctx* c, int32_t dtype, const sr_grid* coarse, const sr_grid* fine, int32_t k,
                     const void* yc_dev, void* yf_dev) {
  if (!c || !coarse || !fine || !yc_dev || !yf_dev) return fail(SR_ERR_ARG, "null argument");
  if (k < 1 || coarse->ndim != fine->ndim || coarse->ndim < 2 || coarse->ndim > 3)
    return fail(SR_ERR_ARG, "bad k / ndim");
  if (dtype != SR_F32 && dtype != SR_F64) return fail(SR_ERR_ARG, "bad dtype");
  for (int a = 0; a < coarse->ndim; ++a)
    if (coarse->dims[a] < 2 || fine->dims[a] < 1 || !(coarse->spacing[a] > 0) || !(fine->spacing[a] > 0))
      return fail(SR_ERR_ARG, "coarse dims must be >= 2 and spacings > 0");
  CK(cudaSetDevice(c->device));
  const Geo gc = make_geo(*coarse), gf = make_geo(*fine);
  if (gf.N > (1LL << 31) || gc.N > (1LL << 31)) return fail(SR_ERR_ARG, "grid too large");
  constexpr int FG = 4;  // frames per thread
  const dim3 grid((unsigned)((gf.N + 255) / 256), (unsigned)((k + FG - 1) / FG));
  if (dtype == SR_F32) {
    if (gf.nd == 2) k_prolong_field<float, 2, FG><<<grid, 256, 0, c->stream>>>((const float*)yc_dev, (float*)yf_dev, gc, gf, k);
    else k_prolong_field<float, 3, FG><<<grid, 256, 0, c->stream>>>((const float*)yc_dev, (float*)yf_dev, gc, gf, k);
  } else {
    if (gf.nd == 2) k_prolong_field<double, 2, FG><<<grid, 256, 0, c->stream>>>((const double*)yc_dev, (double*)yf_dev, gc, gf, k);
    else k_prolong_field<double, 3, FG><<<grid, 256, 0, c->stream>>>((const double*)yc_dev, (double*)yf_dev, gc, gf, k);
  }
  CK(cudaGetLastError());
  return SR_OK;
}

void sr_lbfgs_defaults(sr_lbfgs_options* o) {
  if (!o) return;
  o->memory = 5;
  o->max_iters = 50;
  o->grad_tol = 1e-4;
  o->step_tol = 1e-7;
  o->f_tol = 1e-5;
  o->armijo_c1 = 1e-4;
  o->backtrack_factor = 0.5;
  o->max_backtracks = 20;
}

int sr_lbfgs_minimize(sr_ctx* c, int64_t n, double* x_dev, const sr_lbfgs_options* o, sr_objective_fn objective,
                      void* objective_user, sr_trace_fn trace, void* trace_user, sr_lbfgs_result* result) {
  if (!c || !x_dev || !o || !objective || !result) return fail(SR_ERR_ARG, "null argument");
  if (n < 1) return fail(SR_ERR_ARG, "n must be >= 1");
  // OptimOptions.__post_init__ (optimizer.py:38-46)
  if (o->memory < 1 || o->max_iters < 1 || o->max_backtracks < 1)
    return fail(SR_ERR_ARG, "memory, max_iters, max_backtracks must be >= 1");
  if (!(o->grad_tol > 0) || !(o->step_tol > 0) || !(o->f_tol > 0)) return fail(SR_ERR_ARG, "tolerances must be > 0");
  if (!(o->armijo_c1 > 0 && o->armijo_c1 < 1)) return fail(SR_ERR_ARG, "armijo_c1 must be in (0, 1)");
  if (!(o->backtrack_factor > 0 && o->backtrack_factor < 1))
    return fail(SR_ERR_ARG, "backtrack_factor must be in (0, 1)");
  CK(cudaSetDevice(c->device));
  char err[256] = {0};
  const int rc = sr::lbfgs::minimize(c->lbfgs, c->stream, c->sms, n, x_dev, *o, objective, objective_user, trace,
                                     trace_user, result, err, sizeof err);
  if (rc) return fail(rc, "%s", err);
  return SR_OK;
}

}  // extern "C"

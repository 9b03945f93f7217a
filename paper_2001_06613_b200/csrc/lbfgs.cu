// lbfgs.cu — device-resident L-BFGS with Armijo backtracking, the algorithm of
// /root/reference/pkg/src/seqreg/optimizer.py:59-168 with every vector in HBM (fp64).
//
// Vectors: x (caller's buffer), g, p (= the two-loop's q, negated in place), x_new, g_new and the
// m curvature pairs (s_i, y_i) as a ring.  Scalars that steer the control flow (g.p, the Armijo
// test, s.y / |s| / |y| of the curvature test, |g|_inf) come back to the host; the two-loop's
// alphas and betas stay in device memory (no host round trip inside the recursion).
//
// Rounding: element-wise updates use explicit __dmul_rn / __dadd_rn / __dsub_rn, i.e. the two
// roundings numpy performs for `q -= a * y` (temporary a * y, then the subtraction), never an
// FMA.  Reductions are fixed-order two-stage trees over a fixed grid (bitwise deterministic).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "../../include/seqreg_b200.h"

namespace sr {
namespace lbfgs {

constexpr int RB = 592;  // stage-1 blocks (fixed: the reduction order must not depend on the launch)
constexpr int RT = 256;  // threads per block

enum RMode { R_DOT = 0, R_ABSMAX = 1 };

__device__ __forceinline__ double warp_red(double v, int mode) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = mode == R_ABSMAX ? fmax(v, u) : __dadd_rn(v, u);
  }
  return v;
}

// stage 1: partial[r * RB + block] for each of nr reductions (a_r . b_r or max |a_r|)
struct RedSet {
  const double* a[4];
  const double* b[4];
  int mode[4];
  int nr;
};

__global__ void __launch_bounds__(RT) k_reduce1(const RedSet rs, long long n, double* __restrict__ partial) {
  __shared__ double sm[4][RT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < rs.nr; ++r) {
    const double* a = rs.a[r];
    const double* b = rs.b[r];
    const int mode = rs.mode[r];
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * RT + threadIdx.x; i < n; i += (long long)RB * RT) {
      if (mode == R_ABSMAX) acc = fmax(acc, fabs(a[i]));
      else acc = __dadd_rn(acc, __dmul_rn(a[i], b[i]));
    }
    acc = warp_red(acc, mode);
    if (lane == 0) sm[r][warp] = acc;
  }
  __syncthreads();
  if (warp == 0) {
    for (int r = 0; r < rs.nr; ++r) {
      double v = lane < RT / 32 ? sm[r][lane] : 0.0;
      v = warp_red(v, rs.mode[r]);
      if (lane == 0) partial[r * RB + blockIdx.x] = v;
    }
  }
}

// stage 2: out[r] = coef_r * (reduction of the RB partials), fixed order
struct Red2 {
  double* out[4];
  double coef[4];
  int mode[4];
  int nr;
};

__global__ void __launch_bounds__(1024) k_reduce2(const double* __restrict__ partial, const Red2 rs) {
  __shared__ double sm[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = 0; r < rs.nr; ++r) {
    double v = threadIdx.x < RB ? partial[r * RB + threadIdx.x] : 0.0;
    v = warp_red(v, rs.mode[r]);
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    if (warp == 0) {
      v = sm[lane];
      v = warp_red(v, rs.mode[r]);
      if (lane == 0) *rs.out[r] = rs.mode[r] == R_ABSMAX ? v : __dmul_rn(rs.coef[r], v);
    }
    __syncthreads();
  }
}

// y += c * x with c = sign * (a_dev ? *a_dev : 1) - (b_dev ? *b_dev : 0), or c = a_host
__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, long long n, double a_host,
                       const double* __restrict__ a_dev, const double* __restrict__ b_dev, double sign) {
  double c = a_host;
  if (a_dev) c = sign * *a_dev;
  if (a_dev && b_dev) c = __dsub_rn(*a_dev, *b_dev);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(y[i], __dmul_rn(c, x[i]));
}

// out = s * src   (s host scalar)
__global__ void k_scale(double* __restrict__ out, const double* __restrict__ src, long long n, double s) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __dmul_rn(s, src[i]);
}

// out = a - b
__global__ void k_sub(double* __restrict__ out, const double* __restrict__ a, const double* __restrict__ b,
                      long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __dsub_rn(a[i], b[i]);
}

// out = x + step * p
__global__ void k_step(double* __restrict__ out, const double* __restrict__ x, const double* __restrict__ p,
                       long long n, double step) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(x[i], __dmul_rn(step, p[i]));
}

// any non-finite entry -> flag
__global__ void k_nonfinite(const double* __restrict__ a, long long n, int* __restrict__ flag) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) *flag = 1;
}

struct Workspace {
  long long n = 0;
  long long cap = 0;  // entries every n-vector is allocated for (grow-only: a multilevel run solves problems of
                      // 16 different sizes, and cudaFree / cudaMalloc of its 14 vectors, 1 GB each at C5's finest
                      // level, cost more than the solves)
  int m = 0;
  double *g = nullptr, *p = nullptr, *xn = nullptr, *gn = nullptr, *partial = nullptr, *scal = nullptr;
  std::vector<double*> S, Y;
  int* flag = nullptr;
  double* host = nullptr;  // pinned scalar readback
  void release() {
    for (double* q : {g, p, xn, gn, partial, scal}) cudaFree(q);
    for (double* q : S) cudaFree(q);
    for (double* q : Y) cudaFree(q);
    cudaFree(flag);
    cudaFreeHost(host);
    *this = Workspace();
  }
};

static Workspace* g_ws_dummy = nullptr;  // (keeps the type complete for the destroy hook)

struct Ctx {
  cudaStream_t st;
  int grid;
};

static cudaError_t reduce(const Ctx& c, Workspace& w, long long n, int nr, const double* const* a,
                          const double* const* b, const int* mode, double* const* out, const double* coef) {
  RedSet s{};
  Red2 r{};
  s.nr = r.nr = nr;
  for (int i = 0; i < nr; ++i) {
    s.a[i] = a[i];
    s.b[i] = b ? b[i] : nullptr;
    s.mode[i] = r.mode[i] = mode[i];
    r.out[i] = out[i];
    r.coef[i] = coef ? coef[i] : 1.0;
  }
  k_reduce1<<<RB, RT, 0, c.st>>>(s, n, w.partial);
  k_reduce2<<<1, 1024, 0, c.st>>>(w.partial, r);
  return cudaGetLastError();
}

#define LK(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) {                              \
      snprintf(err, errlen, "%s: %s", #call, cudaGetErrorString(e_)); \
      return SR_ERR_CUDA;                                 \
    }                                                     \
  } while (0)

static int ensure(Workspace& w, long long n, int m, char* err, size_t errlen) {
  if (w.cap >= n && w.m == m && w.g) {
    w.n = n;
    return SR_OK;
  }
  w.release();
  w.n = n;
  w.cap = n;
  w.m = m;
  const size_t b = (size_t)n * sizeof(double);
  LK(cudaMalloc(&w.g, b));
  LK(cudaMalloc(&w.p, b));
  LK(cudaMalloc(&w.xn, b));
  LK(cudaMalloc(&w.gn, b));
  LK(cudaMalloc(&w.partial, 4 * RB * sizeof(double)));
  LK(cudaMalloc(&w.scal, (8 + 2 * (size_t)m) * sizeof(double)));
  LK(cudaMalloc(&w.flag, sizeof(int)));
  LK(cudaMallocHost(&w.host, 8 * sizeof(double)));
  w.S.assign(m, nullptr);
  w.Y.assign(m, nullptr);
  for (int i = 0; i < m; ++i) {
    LK(cudaMalloc(&w.S[i], b));
    LK(cudaMalloc(&w.Y[i], b));
  }
  return SR_OK;
}

int minimize(Workspace*& wsp, cudaStream_t st, int sms, long long n, double* x, const sr_lbfgs_options& o,
             sr_objective_fn objective, void* ouser, sr_trace_fn trace, void* tuser, sr_lbfgs_result* res,
             char* err, size_t errlen) {
  (void)g_ws_dummy;
  if (!wsp) wsp = new Workspace();
  Workspace& w = *wsp;
  int rc = ensure(w, n, o.memory, err, errlen);
  if (rc) return rc;
  const Ctx c{st, sms * 4};
  const int EB = 256;
  const int egrid = (int)std::min<long long>((n + EB - 1) / EB, (long long)sms * 8);
  double* sc = w.scal;  // [0] g.p, [1] s.y, [2] s.s, [3] y.y, [4] |g|_inf, [8 + i] alpha_i, [8 + m + i] beta
  double* hs = w.host;
  int evals = 0;
  auto evaluate = [&](const double* pt, double* gout, double* f) -> int {
    ++evals;
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      snprintf(err, errlen, "stream error before the objective call");
      return SR_ERR_CUDA;
    }
    if (objective(ouser, pt, f, gout) != 0) {
      snprintf(err, errlen, "objective callback failed");
      return SR_ERR_CALLBACK;
    }
    return SR_OK;
  };
  auto read = [&](int k) -> int {  // first k scalars -> host
    if (cudaMemcpyAsync(hs, sc, k * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      snprintf(err, errlen, "scalar readback failed: %s", cudaGetErrorString(cudaGetLastError()));
      return SR_ERR_CUDA;
    }
    return SR_OK;
  };
  auto all_finite = [&](const double* v, bool& ok) -> int {
    LK(cudaMemsetAsync(w.flag, 0, sizeof(int), st));
    k_nonfinite<<<egrid, EB, 0, st>>>(v, n, w.flag);
    int h = 0;
    LK(cudaMemcpyAsync(&h, w.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    LK(cudaStreamSynchronize(st));
    ok = h == 0;
    return SR_OK;
  };

  double f = 0.0;
  rc = evaluate(x, w.g, &f);
  if (rc) return rc;
  bool gfin = true;
  rc = all_finite(w.g, gfin);
  if (rc) return rc;
  if (!std::isfinite(f) || !gfin) {
    snprintf(err, errlen, "objective is not finite at the starting point");
    return SR_ERR_ARG;
  }
  const double f_initial = f;
  {
    const double* a[1] = {w.g};
    const int md[1] = {R_ABSMAX};
    double* out[1] = {sc + 4};
    LK(reduce(c, w, n, 1, a, nullptr, md, out, nullptr));
    rc = read(5);
    if (rc) return rc;
  }
  const double g_inf0 = hs[4];
  const double grad_target = o.grad_tol * g_inf0;
  res->f_initial = f_initial;
  if (g_inf0 <= grad_target) {
    res->f_final = f;
    res->iterations = 0;
    res->objective_evaluations = evals;
    res->converged_reason = SR_LBFGS_GRAD_TOL;
    return SR_OK;
  }

  // curvature pairs: ring of slots, hist[k] = slot of the k-th oldest pair; rho on the host
  std::vector<int> hist;
  std::vector<double> rho_of(o.memory, 0.0), sy_of(o.memory, 0.0), yy_of(o.memory, 0.0);
  int next_slot = 0;
  int reason = SR_LBFGS_MAX_ITERS;
  int iteration = 0;
  for (iteration = 1; iteration <= o.max_iters; ++iteration) {
    // ---- two-loop recursion (optimizer.py:59-73), q in w.p
    LK(cudaMemcpyAsync(w.p, w.g, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    const int L = (int)hist.size();
    for (int k = L - 1; k >= 0; --k) {
      const int sl = hist[k];
      const double* a[1] = {w.S[sl]};
      const double* b[1] = {w.p};
      const int md[1] = {R_DOT};
      double* out[1] = {sc + 8 + k};
      const double cf[1] = {rho_of[sl]};
      LK(reduce(c, w, n, 1, a, b, md, out, cf));                                 // alpha = rho (s . q)
      k_axpy<<<egrid, EB, 0, st>>>(w.p, w.Y[sl], n, 0.0, sc + 8 + k, nullptr, -1.0);  // q -= alpha y
    }
    if (L > 0) {
      const int sl = hist[L - 1];
      const double gamma = sy_of[sl] / yy_of[sl];
      k_scale<<<egrid, EB, 0, st>>>(w.p, w.p, n, gamma);  // q *= gamma
    }
    for (int k = 0; k < L; ++k) {
      const int sl = hist[k];
      const double* a[1] = {w.Y[sl]};
      const double* b[1] = {w.p};
      const int md[1] = {R_DOT};
      double* out[1] = {sc + 8 + o.memory + k};
      const double cf[1] = {rho_of[sl]};
      LK(reduce(c, w, n, 1, a, b, md, out, cf));                                            // beta = rho (y . q)
      k_axpy<<<egrid, EB, 0, st>>>(w.p, w.S[sl], n, 0.0, sc + 8 + k, sc + 8 + o.memory + k, 1.0);  // q += (a - b) s
    }
    k_scale<<<egrid, EB, 0, st>>>(w.p, w.p, n, -1.0);  // p = -q
    LK(cudaGetLastError());
    {
      const double* a[1] = {w.g};
      const double* b[1] = {w.p};
      const int md[1] = {R_DOT};
      double* out[1] = {sc + 0};
      LK(reduce(c, w, n, 1, a, b, md, out, nullptr));
      rc = read(1);
      if (rc) return rc;
    }
    double gp = hs[0];
    if (gp >= 0.0) {  // not a descent direction: steepest descent
      k_scale<<<egrid, EB, 0, st>>>(w.p, w.g, n, -1.0);
      const double* a[1] = {w.g};
      const double* b[1] = {w.p};
      const int md[1] = {R_DOT};
      double* out[1] = {sc + 0};
      LK(reduce(c, w, n, 1, a, b, md, out, nullptr));
      rc = read(1);
      if (rc) return rc;
      gp = hs[0];
    }
    // ---- Armijo backtracking (optimizer.py:123-134)
    double step = 1.0, f_new = 0.0;
    bool accepted = false;
    for (int t = 0; t < o.max_backtracks; ++t) {
      k_step<<<egrid, EB, 0, st>>>(w.xn, x, w.p, n, step);
      LK(cudaGetLastError());
      rc = evaluate(w.xn, w.gn, &f_new);
      if (rc) return rc;
      if (std::isfinite(f_new) && f_new <= f + o.armijo_c1 * step * gp) {
        accepted = true;
        break;
      }
      step *= o.backtrack_factor;
    }
    if (!accepted) {
      reason = SR_LBFGS_LINE_SEARCH_FAILURE;
      iteration -= 1;
      break;
    }
    // ---- curvature pair (optimizer.py:136-151): s, y into the next ring slot
    const int sl = (int)hist.size() < o.memory ? (int)hist.size() : next_slot;
    double* s = w.S[sl];
    double* yv = w.Y[sl];
    k_sub<<<egrid, EB, 0, st>>>(s, w.xn, x, n);
    k_sub<<<egrid, EB, 0, st>>>(yv, w.gn, w.g, n);
    {
      const double* a[4] = {s, s, yv, w.gn};
      const double* b[4] = {yv, s, yv, nullptr};
      const int md[4] = {R_DOT, R_DOT, R_DOT, R_ABSMAX};
      double* out[4] = {sc + 1, sc + 2, sc + 3, sc + 4};
      LK(reduce(c, w, n, 4, a, b, md, out, nullptr));
      rc = read(5);
      if (rc) return rc;
    }
    const double sy = hs[1], ss = hs[2], yy = hs[3], g_inf = hs[4];
    const double snorm = std::sqrt(ss), ynorm = std::sqrt(yy);
    if (sy > 1e-10 * snorm * ynorm) {
      if ((int)hist.size() < o.memory) {
        hist.push_back(sl);
      } else {  // drop the oldest pair: its slot was just overwritten
        hist.erase(hist.begin());
        hist.push_back(sl);
      }
      next_slot = hist.front();
      rho_of[sl] = 1.0 / sy;
      sy_of[sl] = sy;
      yy_of[sl] = yy;
    } else {
      hist.clear();
      next_slot = 0;
    }
    const double decrease = f - f_new;
    // x, f, g <- x_new, f_new, g_new
    LK(cudaMemcpyAsync(x, w.xn, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    std::swap(w.g, w.gn);
    f = f_new;
    if (trace) trace(tuser, iteration, f, g_inf, step, evals);
    if (g_inf <= grad_target) {
      reason = SR_LBFGS_GRAD_TOL;
      break;
    }
    if (snorm <= o.step_tol) {
      reason = SR_LBFGS_STEP_TOL;
      break;
    }
    if (decrease <= o.f_tol * (1.0 + std::fabs(f))) {
      reason = SR_LBFGS_F_TOL;
      break;
    }
  }
  if (iteration > o.max_iters) iteration = o.max_iters;
  LK(cudaStreamSynchronize(st));
  res->f_final = f;
  res->iterations = iteration;
  res->objective_evaluations = evals;
  res->converged_reason = reason;
  return SR_OK;
}

void destroy(Workspace* w) {
  if (!w) return;
  w->release();
  delete w;
}

}  // namespace lbfgs
}  // namespace sr

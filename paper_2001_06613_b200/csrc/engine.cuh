// engine.cuh — the fused D(y) / grad D(y) kernels (sm_100a, SIMT path).
//
// Pass 1  (k_pass1)      : warp every subset frame, form the feature, and accumulate the
//                          raw Gram G = sum_rows v v^T plus per-frame sum / max / min.
//                          Replaces correlation_state (similarity.py:128-164) with
//                          sample (grid.py:236-243) and feature (similarity.py:73-87) fused.
// Reduce  (k_reduce_finalize, k_sum1): fixed-order cross-CTA sums (deterministic, no float atomics,
//                          SPEC.md:318 determinism).
// Finalize(k_finalize)   : centre/normalise -> C, degenerate flags, D (similarity.py:167-177)
//                          and the gradient coefficients M', beta'.
// Pass 2  (k_pass2)      : re-warp with the interpolant gradient, q = M'^T v + beta' per
//                          pixel (a K x K contraction per pixel tile), chain rule to
//                          dD/dy or to the affine parameters (similarity.py:203-217).
//                          For NGF it stops at z = dD/d(grad u) and k_ngf_adjoint applies
//                          the adjoint of the discrete gradient and the chain rule.
// k_curvature, k_ls_predict, k_interp_linear, k_frame_mean: regulariser, temporal
//                          prolongation (temporal.py:109-239) and frame shifts.
//
// Raw-sum layout (fp64): [G (k*k) | s (k) | vmax (k) | -vmin (k) | count]; the two
// extremum blocks all-reduce with MAX, everything else with SUM.
#pragma once
#include "common.cuh"

namespace sr {

enum { NCC = 0, NGF = 1 };
enum { AFFINE = 0, DISP = 1 };

struct Args {
  Geo g;
  const void* frames;
  const void* shifts;   // per frame (indexed by frame index), may be null
  const void* y;        // displacement [K][D][y_stride]
  long long y_off, y_stride;
  const Job* job;
  int K;
  long long pix_lo, pix_hi;
  double eps;           // NGF epsilon
  double* part;         // per-CTA partial sums
  const double* stats;  // finalize output (pass 2)
  void* out;            // pass 2 output: grad (disp) / z buffer (NGF)
  long long o_off, o_stride;
  double* part_aff;     // pass 2 affine partials
  int ymap_ok;          // a y tensor map was encoded for the warp-specialized kernels
  double curv_alpha;    // > 0: pass 2 adds the curvature gradient alpha h L L (y - x) (sr_evaluate_reg)
  double curv_h;
  double* curv_part;    // per-CTA partial sums of S (reduced by k_sum1)
};

// --------------------------------------------------------- stats buffer layout
struct StatsLayout {
  long long C, sigma, mean, vmax, degen, weights, M, beta, shift, Mf, total;
  __host__ __device__ StatsLayout(int K) {
    C = 8;
    sigma = C + (long long)K * K;
    mean = sigma + K;
    vmax = mean + K;
    degen = vmax + K;
    weights = degen + K;
    M = weights + K;
    beta = M + (long long)K * K;
    shift = beta + K;
    Mf = shift + K;
    total = Mf + ((long long)K * K + 1) / 2;
  }
};

__host__ __device__ constexpr int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

// Pixel-tile / ownership configuration of the Gram phase of pass 1.
template <typename T, int KP, int FEAT = NGF>
struct G1 {
  static constexpr int RB = KP == 8 ? 2 : KP == 16 ? 4 : 8;
  static constexpr int CB = KP == 8 ? 1 : KP == 16 ? 2 : (KP == 128 && sizeof(T) == 4) ? 8 : 4;
  static constexpr int RG = KP / RB, CG = KP / CB, OWN = RG * CG;
  // fp32 NCC with KP <= 32: 512 threads (16 warps) so each thread samples only a few
  // frames per tile and can keep the next tile's y in flight during the Gram phase
  static constexpr int NT = (FEAT == NCC && sizeof(T) == 4 && KP <= 32) ? 512 : (OWN > 256 ? OWN : 256);
  static constexpr int NW = NT / 32, NG = NT / OWN, OPT = RB * CB;
  static constexpr int ROWS = (32768 / (KP * (int)sizeof(T))) < 32 ? 32
                              : (32768 / (KP * (int)sizeof(T))) > 512 ? 512
                              : 32768 / (KP * (int)sizeof(T));
};

template <typename T, int D, int FEAT, int KP>
struct Tile1 {
  static constexpr int FD = FEAT == NGF ? D : 1;
  static constexpr int TP0 = pow2_floor(G1<T, KP>::ROWS / FD);
  static constexpr int TP = TP0 < 8 ? 8 : TP0;  // power of two
  static constexpr int R = TP * FD;
  static constexpr int RS = ((R + 31) / 32) * 32 + 4;
  static constexpr int QT = TP / 4;                            // pixel quads per tile
  static constexpr int FPT = KP * QT / G1<T, KP, FEAT>::NT;    // NCC: frames per thread
  static constexpr int KSTEP = G1<T, KP, FEAT>::NT / QT;
};

// Pixel-tile configuration of pass 2: a thread owns JB frames x one quad of pixels.
template <typename T, int KP>
struct G2 {
  static constexpr int JB = (sizeof(T) == 8 && KP == 128) ? 2 : 4;
  static constexpr int TP = 4 * 256 * JB / KP;
  static constexpr int QN = TP / 4, JG = KP / JB, NT = QN * JG;
  static constexpr int TS = TP + 4;
  static constexpr bool MSMEM = KP <= 64;  // stage M' in shared memory
};

template <typename T, int D, int FEAT, int PARAM, int KP>
constexpr size_t pass1_smem() {
  using C = G1<T, KP, FEAT>;
  using Tl = Tile1<T, D, FEAT, KP>;
  return (size_t)KP * Tl::RS * sizeof(T) + (size_t)C::OPT * C::NT * 8 + (size_t)3 * Tl::TP * 4 +
         (size_t)KP * 8 + 2 * (size_t)KP * sizeof(T) + 32;
}
template <typename T, int D, int FEAT, int KP>
constexpr size_t pass2_smem() {
  using C = G2<T, KP>;
  return (size_t)KP * C::TS * sizeof(T) * (1 + D) + (size_t)3 * C::TP * 4 +
         (C::MSMEM ? (size_t)KP * KP * sizeof(T) : 0) + 32;
}

// ----------------------------------------------------------- sample positions
// World point at which subset frame j is sampled for pixel `pix` (coords c).
template <typename T, typename P, int D, int PARAM>
__device__ __forceinline__ void warp_point(const Args& a, int j, long long pix, const int (&c)[3],
                                           P (&p)[D]) {
  if (PARAM == AFFINE) {
    // apply_affine (transform.py:95): pts @ A.T + b
    const double* A = a.job->affine + j * 12;
    double x[D];
#pragma unroll
    for (int b = 0; b < D; ++b) x[b] = center(a.g, b, c[b]);
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double acc = x[0] * A[r * D + 0];
#pragma unroll
      for (int b = 1; b < D; ++b) acc = fma(x[b], A[r * D + b], acc);
      p[r] = (P)__dadd_rn(acc, A[D * D + r]);
    }
  } else {
    const T* y = reinterpret_cast<const T*>(a.y);
    const long long off = pix - a.y_off;
#pragma unroll
    for (int r = 0; r < D; ++r) p[r] = (P)ldg(y + (long long)(j * D + r) * a.y_stride + off);
  }
}

template <typename T, typename P, int D, int PARAM, bool GRAD, bool POW2>
__device__ __forceinline__ T sample_at(const Args& a, const T* img, int j, long long pix,
                                       const int (&c)[3], T (&gr)[D]) {
  P p[D];
  warp_point<T, P, D, PARAM>(a, j, pix, c, p);
  return interp<T, P, D, GRAD, POW2>(img, a.g, p, gr);
}

// Four consecutive pixels p0..p0+3 (nvalid of them inside the slab) of subset frame j.
// Displacement: the y quads are one 16-byte load per component when aligned.
template <typename T, typename P, int D, int PARAM, bool GRAD, bool POW2>
__device__ __forceinline__ void sample_quad(const Args& a, const T* img, int j, long long p0, int nvalid,
                                            bool vec, const int* crd4, T (&v)[4], T (&gr)[4][D]) {
  P p[4][D];
  if (PARAM == DISP) {
    const T* y = reinterpret_cast<const T*>(a.y) + (p0 - a.y_off);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const T* yc = y + (long long)(j * D + c) * a.y_stride;
      if (vec) {
        T q[4];
        ldg4(yc, q);
#pragma unroll
        for (int e = 0; e < 4; ++e) p[e][c] = (P)q[e];
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) p[e][c] = e < nvalid ? (P)ldg(yc + e) : (P)0;
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c[3] = {crd4[3 * e], crd4[3 * e + 1], crd4[3 * e + 2]};
      warp_point<T, P, D, PARAM>(a, j, p0 + e, c, p[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) v[e] = interp<T, P, D, GRAD, POW2>(img, a.g, p[e], gr[e]);
}

// Interpolate four prepared points (the quad's y already in registers).
template <typename T, typename P, int D, bool GRAD, bool POW2>
__device__ __forceinline__ void sample_pts4(const T* img, const Geo& g, const T (&yq)[D][4], T (&v)[4],
                                            T (&gr)[4][D]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    P p[D];
#pragma unroll
    for (int c = 0; c < D; ++c) p[c] = (P)yq[c][e];
    v[e] = interp<T, P, D, GRAD, POW2>(img, g, p, gr[e]);
  }
}

// Load the quad's y (all components) of subset frame j: 16-byte loads when aligned.
template <typename T, int D>
__device__ __forceinline__ void load_yq(const Args& a, int j, long long p0, int nvalid, bool vec,
                                        T (&yq)[D][4]) {
  const T* y = reinterpret_cast<const T*>(a.y) + (p0 - a.y_off);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const T* yc = y + (long long)(j * D + c) * a.y_stride;
    if (vec) {
      ldg4(yc, yq[c]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) yq[c][e] = e < nvalid ? ldg(yc + e) : (T)0;
    }
  }
}

// NGF feature at one pixel: u = T_j(y_j) on the cell centres, p = grad_h u (central
// differences, one-sided at the domain edge), rho = sqrt(|p|^2 + eps^2), n = p / rho.
template <typename T, typename P, int D, int PARAM, bool POW2>
__device__ __forceinline__ void ngf_at(const Args& a, const T* img, int j, long long pix,
                                       const int (&c)[3], T (&n)[D], T& rho) {
  T dummy[D];
  const T u0 = sample_at<T, P, D, PARAM, false, POW2>(a, img, j, pix, c, dummy);
  T up[D], um[D];
#pragma unroll
  for (int ax = 0; ax < D; ++ax) {
    const bool hp = c[ax] < a.g.n[ax] - 1, hm = c[ax] > 0;
    int cp[3] = {c[0], c[1], c[2]}, cm[3] = {c[0], c[1], c[2]};
    cp[ax] += hp ? 1 : 0;
    cm[ax] -= hm ? 1 : 0;
    up[ax] = sample_at<T, P, D, PARAM, false, POW2>(a, img, j, pix + (hp ? a.g.st[ax] : 0), cp, dummy);
    um[ax] = sample_at<T, P, D, PARAM, false, POW2>(a, img, j, pix - (hm ? a.g.st[ax] : 0), cm, dummy);
  }
  T pn = (T)0;
#pragma unroll
  for (int ax = 0; ax < D; ++ax) {
    const bool hp = c[ax] < a.g.n[ax] - 1, hm = c[ax] > 0;
    const T inv = (T)a.g.inv[ax];
    const T gax = (hp && hm) ? (up[ax] - um[ax]) * (inv * (T)0.5) : (up[ax] - um[ax]) * inv;
    n[ax] = gax;
    pn += gax * gax;
  }
  (void)u0;
  const T e = (T)a.eps;
  rho = sqrt(pn + e * e);
  const T ir = (T)1 / rho;
#pragma unroll
  for (int ax = 0; ax < D; ++ax) n[ax] *= ir;
}

__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<long long*>(addr), __double_as_longlong(v));
}

// ===================================================================== pass 1
template <typename T, int D, int FEAT, int PARAM, int KP, bool POW2>
__device__ __forceinline__ void pass1_body(const Args& a) {
  using C = G1<T, KP, FEAT>;
  using Tl = Tile1<T, D, FEAT, KP>;
  using P = typename std::conditional<PARAM == AFFINE, double, T>::type;
  constexpr int TP = Tl::TP, R = Tl::R, RS = Tl::RS, NT = C::NT;
  constexpr int RB = C::RB, CB = C::CB, RG = C::RG, CG = C::CG, OWN = C::OWN, NG = C::NG;
  constexpr int QT = Tl::QT, FPT = Tl::FPT, KSTEP = Tl::KSTEP;
  constexpr bool NEED_CRD = (FEAT == NGF) || (PARAM == AFFINE);
  static_assert(FEAT == NGF || (NT % QT == 0 && FPT >= 1 && FPT * KSTEP == KP), "NCC tile mapping");

  extern __shared__ __align__(16) unsigned char smem[];
  T* V = reinterpret_cast<T*>(smem);
  double* slot = reinterpret_cast<double*>(smem + (size_t)KP * RS * sizeof(T));
  int* crd = reinterpret_cast<int*>(slot + (size_t)C::OPT * NT);
  double* ssum = reinterpret_cast<double*>(crd + 3 * TP);  // NGF: unused
  T* smax = reinterpret_cast<T*>(ssum + KP);                // NGF: max |n| per frame
  T* sminn = smax + KP;

  const int tid = threadIdx.x;
  const int K = a.K;
  for (int e = tid; e < C::OPT * NT; e += NT) slot[e] = 0.0;
  for (int k = tid; k < KP; k += NT) {
    ssum[k] = 0.0;
    smax[k] = (T)0;
    sminn[k] = (T)0;
  }
  for (int e = tid; e < (KP - K) * RS; e += NT) V[(size_t)K * RS + e] = (T)0;
  __syncthreads();

  const int o = tid % OWN, grp = tid / OWN;
  const int rg = o / CG, cg = o % CG;
  T acc[RB][CB];
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int j = 0; j < CB; ++j) acc[i][j] = (T)0;

  // NCC per-thread running sum / max / min of its fixed frame set (k = kb + KSTEP*i)
  const int q = tid % QT, kb = tid / QT;
  T fsum[FEAT == NCC ? FPT : 1];
  T fmx[FEAT == NCC ? FPT : 1], fmn[FEAT == NCC ? FPT : 1];
#pragma unroll
  for (int i = 0; i < (FEAT == NCC ? FPT : 1); ++i) {
    fsum[i] = (T)0;
    fmx[i] = -INFINITY;
    fmn[i] = INFINITY;
  }

  const T* frames = reinterpret_cast<const T*>(a.frames);
  const T* shifts = reinterpret_cast<const T*>(a.shifts);
  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (npix + TP - 1) / TP;
  const bool yvec = PARAM == DISP && (a.y_stride % 4 == 0) &&
                    ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
  T ypf[(FEAT == NCC && PARAM == DISP) ? FPT : 1][D][4];
  bool first = true;

  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long t0 = a.pix_lo + tile * TP;
    if (NEED_CRD) {
      for (int pp = tid; pp < TP; pp += NT) {
        int c[3];
        coords<D>(a.g, t0 + pp, c);
        crd[3 * pp] = c[0];
        crd[3 * pp + 1] = c[1];
        crd[3 * pp + 2] = c[2];
      }
      __syncthreads();
    }
    if (FEAT == NCC) {
      // ---- sampling: thread -> one pixel quad of FPT frames; the quad's y was prefetched
      // during the previous tile's Gram phase (displacement), so only the gathers wait
      const long long p0 = t0 + 4 * q;
      const long long nv = a.pix_hi - p0;
      const int nvalid = nv >= 4 ? 4 : (nv > 0 ? (int)nv : 0);
      if (PARAM == DISP && first) {
        const bool vec = yvec && nvalid == 4 && (((p0 - a.y_off) & 3) == 0);
#pragma unroll
        for (int i = 0; i < FPT; ++i) {
          const int k = kb + KSTEP * i;
          if (k < K) load_yq<T, D>(a, k, p0, nvalid, vec, ypf[PARAM == DISP ? i : 0]);
        }
      }
      first = false;
#pragma unroll
      for (int i = 0; i < FPT; ++i) {
        const int k = kb + KSTEP * i;
        if (k < K) {
          const int fi = a.job->frame_index[k];
          const T* img = frames + (long long)fi * a.g.N;
          const T sh = shifts ? shifts[fi] : (T)0;
          T v[4], gr[4][D];
          if (PARAM == DISP) sample_pts4<T, P, D, false, POW2>(img, a.g, ypf[PARAM == DISP ? i : 0], v, gr);
          else sample_quad<T, P, D, PARAM, false, POW2>(a, img, k, p0, nvalid, false, crd + 12 * q, v, gr);
          T out[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool ok = e < nvalid;
            out[e] = ok ? v[e] - sh : (T)0;
            fsum[i] += out[e];
            fmx[i] = ok ? max(fmx[i], v[e]) : fmx[i];
            fmn[i] = ok ? min(fmn[i], v[e]) : fmn[i];
          }
          sts4(V + (size_t)k * RS + 4 * q, out);
        }
      }
      if (PARAM == DISP) {
        // prefetch the next tile's y: in flight while this tile's Gram runs
        const long long nt = tile + gridDim.x;
        if (nt < ntiles) {
          const long long p1 = a.pix_lo + nt * TP + 4 * q;
          const long long nv1 = a.pix_hi - p1;
          const int nval1 = nv1 >= 4 ? 4 : (nv1 > 0 ? (int)nv1 : 0);
          const bool vec1 = yvec && nval1 == 4 && (((p1 - a.y_off) & 3) == 0);
#pragma unroll
          for (int i = 0; i < FPT; ++i) {
            const int k = kb + KSTEP * i;
            if (k < K) load_yq<T, D>(a, k, p1, nval1, vec1, ypf[PARAM == DISP ? i : 0]);
          }
        }
      }
    } else {
      // ---- NGF sampling: (frame, pixel) items, 2d+1 samples per item in flight
      T lmax = (T)0;
      int kcur = -1;
      for (int it = tid; it < K * TP; it += NT) {
        const int k = it / TP, pp = it % TP;
        if (k != kcur) {
          if (kcur >= 0 && lmax > (T)0) atomic_max_nonneg(&smax[kcur], lmax);
          kcur = k;
          lmax = (T)0;
        }
        const long long pix = t0 + pp;
        T n[D];
        if (pix < a.pix_hi) {
          const int fi = a.job->frame_index[k];
          const T* img = frames + (long long)fi * a.g.N;
          const int c[3] = {crd[3 * pp], crd[3 * pp + 1], crd[3 * pp + 2]};
          T rho;
          ngf_at<T, P, D, PARAM, POW2>(a, img, k, pix, c, n, rho);
        } else {
#pragma unroll
          for (int cc = 0; cc < D; ++cc) n[cc] = (T)0;
        }
#pragma unroll
        for (int cc = 0; cc < D; ++cc) {
          V[(size_t)k * RS + cc * TP + pp] = n[cc];
          lmax = max(lmax, abs(n[cc]));
        }
      }
      if (kcur >= 0 && lmax > (T)0) atomic_max_nonneg(&smax[kcur], lmax);
    }
    __syncthreads();
    // ---- Gram: each owner accumulates an RB x CB block over its row quads
#pragma unroll 1
    for (int qq = grp; qq < R / 4; qq += NG) {
      T rv[RB][4], cv[CB][4];
#pragma unroll
      for (int i = 0; i < RB; ++i) lds4(V + (size_t)(rg + RG * i) * RS + 4 * qq, rv[i]);
#pragma unroll
      for (int j = 0; j < CB; ++j) lds4(V + (size_t)(cg + CG * j) * RS + 4 * qq, cv[j]);
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int j = 0; j < CB; ++j) acc[i][j] = fma(rv[i][e], cv[j][e], acc[i][j]);
    }
    // ---- flush the tile's short run into the thread's fp64 slots
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        slot[(size_t)(i * CB + j) * NT + tid] += (double)acc[i][j];
        acc[i][j] = (T)0;
      }
    __syncthreads();
  }

  // ---- cross-group Gram reduction in a fixed order, one CTA partial
  constexpr int STRIDE = KP * KP + 3 * KP;
  double* out = a.part + (size_t)blockIdx.x * STRIDE;
  for (int e2 = tid; e2 < KP * KP; e2 += NT) {
    const int i = e2 / KP, j = e2 % KP;
    const int ai = i / RG, rgi = i % RG, bj = j / CG, cgj = j % CG;
    const int oo = rgi * CG + cgj, e = ai * CB + bj;
    double s = 0.0;
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) s += slot[(size_t)e * NT + gg * OWN + oo];
    out[e2] = s;
  }
  __syncthreads();
  if (FEAT == NCC) {
    // per-frame sums / extrema over the QT threads sharing a frame set (fixed order)
    double* rs = reinterpret_cast<double*>(smem);
    T* rmx = reinterpret_cast<T*>(rs + (size_t)KP * QT);
    T* rmn = rmx + (size_t)KP * QT;
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      const int k = kb + KSTEP * i;
      rs[(size_t)k * QT + q] = (double)fsum[i];
      rmx[(size_t)k * QT + q] = fmx[i];
      rmn[(size_t)k * QT + q] = fmn[i];
    }
    __syncthreads();
    for (int k = tid; k < KP; k += NT) {
      double s = 0.0;
      T mx = -INFINITY, mn = INFINITY;
      for (int qq = 0; qq < QT; ++qq) {
        s += rs[(size_t)k * QT + qq];
        mx = max(mx, rmx[(size_t)k * QT + qq]);
        mn = min(mn, rmn[(size_t)k * QT + qq]);
      }
      out[KP * KP + k] = s;
      out[KP * KP + KP + k] = (double)mx;
      out[KP * KP + 2 * KP + k] = -(double)mn;
    }
  } else {
    for (int k = tid; k < KP; k += NT) {
      out[KP * KP + k] = 0.0;
      out[KP * KP + KP + k] = (double)smax[k];
      out[KP * KP + 2 * KP + k] = (double)smax[k];
    }
  }
}

template <typename T, int D, int FEAT, int PARAM, int KP>
__global__ void __launch_bounds__(G1<T, KP, FEAT>::NT) k_pass1(const Args a) {
  if (a.g.pow2) pass1_body<T, D, FEAT, PARAM, KP, true>(a);
  else pass1_body<T, D, FEAT, PARAM, KP, false>(a);
}

// Fixed-order sum of n partials into one scalar (S(y): one partial per CTA of the curvature kernels, 65,536 at
// C5's finest level, where the generic partial reduction's single active lane per warp took 2 ms): thread t sums partials
// t, t + 1024, ... in batches of 8 independent loads, then a fixed tree over the 1024 thread sums.
static __global__ void __launch_bounds__(1024) k_sum1(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double buf[1024];
  const int t = threadIdx.x;
  double acc = 0.0;
  for (int b0 = t; b0 < n; b0 += 8 * 1024) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int b = b0 + 1024 * u;
      v[u] = b < n ? __ldcg(part + b) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  buf[t] = acc;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (t < o) buf[t] += buf[t + o];
    __syncthreads();
  }
  if (t == 0) *out = buf[0];
}

// ==================================================================== finalize
// Block-level finalize (any blockDim that is a power of two, <= 1024).  raw = [G | s | vmax |
// -vmin | count] (all-reduced when sharded), read with ld.global.cg (it may have just been
// written by other CTAs of the same grid).  Cmat: dynamic shared memory of K*K doubles.
template <typename T>
__device__ void finalize_block(const double* __restrict__ raw, const Job* job, int K, int feat, int D,
                               double n_total, double h, const T* shifts, double* __restrict__ stats,
                               double* Cmat) {
  __shared__ double sig[kMaxFrames], isg[kMaxFrames], mu[kMaxFrames], w[kMaxFrames], cj[kMaxFrames],
      sv[kMaxFrames];
  __shared__ int deg[kMaxFrames];
  __shared__ double red[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const StatsLayout L(K);
  const double N = n_total;
  // one round trip for every input: the raw Gram into shared memory (C is formed in place), the
  // per-frame sums / extrema, weights, frame indices and shifts into registers of threads < K
  for (int e = tid; e < K * K; e += nt) Cmat[e] = __ldcg(raw + e);
  double si = 0.0, vmx = 0.0, vmnn = 0.0, wt = 0.0, sh = 0.0;
  if (tid < K) {
    si = __ldcg(raw + K * K + tid);
    vmx = __ldcg(raw + K * K + K + tid);
    vmnn = __ldcg(raw + K * K + 2 * K + tid);
    wt = job->weights[tid];
    sh = (feat == NCC && shifts) ? (double)shifts[job->frame_index[tid]] : 0.0;
  }
  __syncthreads();
  if (tid < K) {
    const double gii = Cmat[tid * K + tid];
    const double amax = fmax(vmx, vmnn);  // max |v|
    double sg, m = 0.0, thr;
    int dg;
    if (feat == NCC) {
      m = si / N;
      const double var = gii - si * m;
      sg = sqrt(fmax(var, 0.0));
      thr = 1e-12 * sqrt(N) * (1.0 + amax);  // similarity.py:84-86
      // an exactly constant frame has centred norm 0 in the reference; the raw-moment
      // form cannot see that through cancellation, the extrema can
      const bool constant = vmx == -vmnn;
      dg = !(sg >= thr) || constant;
      if (constant) sg = 0.0;
    } else {
      sg = sqrt(fmax(gii, 0.0));
      thr = 1e-12 * sqrt(N * D) * (1.0 + amax);
      dg = !(sg >= thr);
    }
    sig[tid] = sg;
    isg[tid] = dg ? 0.0 : 1.0 / sg;
    mu[tid] = m;
    sv[tid] = si;
    deg[tid] = dg;
    w[tid] = wt;
    stats[L.sigma + tid] = sg;
    stats[L.mean + tid] = feat == NCC ? sh + m : 0.0;
    stats[L.vmax + tid] = amax;
    stats[L.degen + tid] = dg;
    stats[L.weights + tid] = wt;
    stats[L.shift + tid] = sh;
  }
  __syncthreads();
  // C (upper triangle computed once, mirrored -> exactly symmetric, similarity.py:155)
  // (in place: the thread of (i, j), i <= j, reads G_ij and writes C_ij and C_ji; G_ji (i < j) is never read)
  for (int e = tid; e < K * K; e += nt) {
    const int i = e / K, j = e % K;
    if (i > j) continue;
    double c = 0.0;
    if (!deg[i] && !deg[j]) {
      const double gij = Cmat[i * K + j];
      const double num = feat == NCC ? gij - sv[i] * mu[j] : gij;
      c = num * (isg[i] * isg[j]);
    }
    Cmat[i * K + j] = c;
    Cmat[j * K + i] = c;
  }
  __syncthreads();
  // warp per column j, lanes over i, fixed-order shuffle reductions:
  //   c_j = sum_i w_i C_ij^2  (= f_j . g_j, similarity.py:210)
  //   dcol_j = sum_{i != j} w_i w_j C_ij^2  (D = h [(sum w)^2 - sum w^2 - sum_j dcol_j], similarity.py:167-177)
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int j = warp; j < K; j += nw) {
    double cp = 0.0, dp = 0.0;
    for (int i = lane; i < K; i += 32) {
      const double c = Cmat[i * K + j];
      const double wc2 = w[i] * c * c;
      cp += wc2;
      if (i != j) dp += wc2 * w[j];
    }
    cp = warp_sum(cp);
    dp = warp_sum(dp);
    if (lane == 0) {
      cj[j] = cp;
      red[j] = dp;
    }
  }
  __syncthreads();
  for (int e = tid; e < K * K; e += nt) stats[L.C + e] = Cmat[e];  // coalesced
  __syncthreads();
  // M'_ij = -4 h w_j (w_i C_ij / sig_i - delta_ij c_j / sig_j) / sig_j ;  beta'_j = -sum_i M'_ij mu_i
  // (M' overwrites C in shared memory: each element is read and written by the same thread)
  for (int j = warp; j < K; j += nw) {
    double bp = 0.0;
    for (int i = lane; i < K; i += 32) {
      double m = 0.0;
      if (!deg[i] && !deg[j]) {
        double t = w[i] * Cmat[i * K + j] * isg[i];
        if (i == j) t -= cj[j] * isg[j];
        m = -4.0 * h * w[j] * t * isg[j];
      }
      Cmat[i * K + j] = m;
      bp += m * mu[i];
    }
    bp = warp_sum(bp);
    if (lane == 0) stats[L.beta + j] = feat == NCC ? -bp : 0.0;
  }
  __syncthreads();
  float* Mf = reinterpret_cast<float*>(stats + L.Mf);
  for (int e = tid; e < K * K; e += nt) {  // coalesced
    const double m = Cmat[e];
    stats[L.M + e] = m;
    Mf[e] = (float)m;
  }
  if (warp == 0) {
    double dsum = 0.0, sw = 0.0, sw2 = 0.0;
    for (int i = lane; i < K; i += 32) {
      dsum += red[i];
      sw += w[i];
      sw2 += w[i] * w[i];
    }
    dsum = warp_sum(dsum);
    sw = warp_sum(sw);
    sw2 = warp_sum(sw2);
    if (lane == 0) {
      stats[0] = fmax(0.0, h * ((sw * sw - sw2) - dsum));
      stats[1] = K;
      stats[2] = N;
      stats[3] = h;
    }
  }
}

// Finalize for K <= 32 with 1024 threads: warp i owns row i, lane j column j, so that every per-frame
// quantity a thread needs is either its own lane's (frame j) or a shuffle from lane i (frame i):
// one global round trip, two CTA barriers.  C_ij is formed from the upper element G[min][max] with
// the factors in (min, max) order, so C is exactly symmetric; c_j and dcol_j are row sums of warp j
// (C symmetric), in the generic finalize's lane order and xor tree (bitwise the same numbers).
template <typename T>
__device__ void finalize_k32(const double* __restrict__ raw, const Job* job, int K, int feat, int D,
                             double n_total, double h, const T* shifts, double* __restrict__ stats) {
  __shared__ double colp[32][33];  // M'_ij mu_i, for the column sums of beta'
  __shared__ double dcol[32];
  const int tid = threadIdx.x, lane = tid & 31, i = tid >> 5;
  const StatsLayout L(K);
  const double N = n_total;
  const int j = lane;
  const bool act = i < K && j < K;
  const int lo = min(i, j), hi = max(i, j);
  // ---- inputs (one round trip): the Gram element, frame j's sums / extrema / weight / shift
  double gij = 0.0, gjj = 0.0, sj = 0.0, vmx = 0.0, vmnn = 0.0, wj = 0.0, shj = 0.0;
  if (act) gij = __ldcg(raw + lo * K + hi);
  if (j < K) {
    gjj = __ldcg(raw + j * K + j);
    sj = __ldcg(raw + K * K + j);
    vmx = __ldcg(raw + K * K + K + j);
    vmnn = __ldcg(raw + K * K + 2 * K + j);
    wj = job->weights[j];
    shj = (feat == NCC && shifts) ? (double)shifts[job->frame_index[j]] : 0.0;
  }
  // ---- per-frame statistics of frame j (every warp, redundantly)
  const double amax = fmax(vmx, vmnn);
  double sg = 0.0, mj = 0.0;
  int dg = 1;
  if (j < K) {
    if (feat == NCC) {
      mj = sj / N;
      const double var = gjj - sj * mj;
      sg = sqrt(fmax(var, 0.0));
      const double thr = 1e-12 * sqrt(N) * (1.0 + amax);  // similarity.py:84-86
      const bool constant = vmx == -vmnn;  // exactly constant frame (see finalize_block)
      dg = !(sg >= thr) || constant;
      if (constant) sg = 0.0;
    } else {
      sg = sqrt(fmax(gjj, 0.0));
      const double thr = 1e-12 * sqrt(N * D) * (1.0 + amax);
      dg = !(sg >= thr);
    }
  }
  const double isgj = dg ? 0.0 : 1.0 / sg;
  // frame i's (= row) quantities from lane i
  const double isgi = __shfl_sync(0xffffffffu, isgj, i & 31);
  const double si = __shfl_sync(0xffffffffu, sj, i & 31), mi = __shfl_sync(0xffffffffu, mj, i & 31);
  const double wi = __shfl_sync(0xffffffffu, wj, i & 31);
  const int dgi = __shfl_sync(0xffffffffu, dg, i & 31);
  if (i == 0 && j < K) {
    stats[L.sigma + j] = sg;
    stats[L.mean + j] = feat == NCC ? shj + mj : 0.0;
    stats[L.vmax + j] = amax;
    stats[L.degen + j] = dg;
    stats[L.weights + j] = wj;
    stats[L.shift + j] = shj;
  }
  // ---- C_ij (exactly symmetric: the (lo, hi) formula)
  double c = 0.0;
  if (act && !dg && !dgi) {
    const double s_lo = lo == i ? si : sj, m_hi = hi == j ? mj : mi;
    const double i_lo = lo == i ? isgi : isgj, i_hi = hi == j ? isgj : isgi;
    const double num = feat == NCC ? gij - s_lo * m_hi : gij;
    c = num * (i_lo * i_hi);
  }
  if (act) stats[L.C + i * K + j] = c;
  // ---- c_i = sum_j w_j C_ij^2 and dcol_i = sum_{j != i} w_j w_i C_ij^2 (row sums of warp i)
  const double wc2 = act ? wj * c * c : 0.0;
  const double cp = warp_sum(wc2);
  const double dp = warp_sum(act && j != i ? wc2 * wi : 0.0);
  if (lane == 0 && i < 32) dcol[i] = i < K ? dp : 0.0;
  // ---- M'_ij = -4 h w_j (w_i C_ij / sig_i - delta_ij c_j / sig_j) / sig_j
  double m = 0.0;
  if (act && !dg && !dgi) {
    double t = wi * c * isgi;
    if (i == j) t -= cp * isgj;
    m = -4.0 * h * wj * t * isgj;
  }
  if (act) {
    stats[L.M + i * K + j] = m;
    reinterpret_cast<float*>(stats + L.Mf)[i * K + j] = (float)m;
  }
  colp[i & 31][j] = m * mi;
  __syncthreads();
  // ---- beta'_j = -sum_i M'_ij mu_i (warp j sums column j over lanes i); D
  if (i < K) {
    const double bp = warp_sum(lane < K ? colp[lane][i] : 0.0);
    if (lane == 0) stats[L.beta + i] = feat == NCC ? -bp : 0.0;
  }
  if (i == 0) {
    const double dsum = warp_sum(dcol[lane]);
    const double sw = warp_sum(j < K ? wj : 0.0), sw2 = warp_sum(j < K ? wj * wj : 0.0);
    if (lane == 0) {
      stats[0] = fmax(0.0, h * ((sw * sw - sw2) - dsum));
      stats[1] = K;
      stats[2] = N;
      stats[3] = h;
    }
  }
}

// Cross-CTA reduction of the pass-1 partials (fixed order: warp w of a block sums CTAs
// w, w+32, ..., then warp 0 combines the 32 warp sums in order) packed straight into the
// caller's raw layout; the last block to finish (atomic ticket) writes the count and, when
// asked, runs the finalize on the complete raw sums.  One launch instead of three.
template <typename T>
__global__ void __launch_bounds__(1024) k_reduce_finalize(const double* __restrict__ part, int nblk, int KP,
                                                          int K, long long count, double* raw, int do_final,
                                                          const Job* job, int feat, int D, double h,
                                                          const T* shifts, double* stats,
                                                          unsigned* ticket) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ double buf[32][33];
  __shared__ int is_last;
  pdl_wait();     // the pass-1 partials
  pdl_trigger();  // pass 2 may be scheduled now (it waits for this grid's completion itself)
  const int stride = KP * KP + 3 * KP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const bool is_max = e >= KP * KP + KP && e < stride;
  double acc = is_max ? -INFINITY : 0.0;
  if (e < stride) {
    // all of this lane's partials in flight at once (up to 16 per warp, i.e. 512 CTAs), then the
    // fixed-order sum; beyond that, batches of 16
    for (int b0 = warp; b0 < nblk; b0 += 32 * 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int b = b0 + 32 * u;
        v[u] = b < nblk ? __ldcg(part + (size_t)b * stride + e) : (is_max ? -INFINITY : 0.0);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = is_max ? fmax(acc, v[u]) : acc + v[u];
    }
  }
  buf[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && e < stride) {
    double s = buf[0][lane];
    for (int w2 = 1; w2 < 32; ++w2) s = is_max ? fmax(s, buf[w2][lane]) : s + buf[w2][lane];
    int r = -1;
    if (e < KP * KP) {
      const int i = e / KP, j = e % KP;
      if (i < K && j < K) r = i * K + j;
    } else {
      const int blk = (e - KP * KP) / KP, k = (e - KP * KP) % KP;
      if (k < K) r = K * K + blk * K + k;
    }
    if (r >= 0) raw[r] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    raw[K * K + 3 * K] = (double)count;
    *ticket = 0u;
  }
  if (!do_final) return;
  if (K <= 32 && blockDim.x == 1024) finalize_k32<T>(raw, job, K, feat, D, (double)count, h, shifts, stats);
  else finalize_block<T>(raw, job, K, feat, D, (double)count, h, shifts, stats, reinterpret_cast<double*>(dsm));
}

// Finalize only (sharded path: raw sums all-reduced by the caller).
template <typename T>
__global__ void __launch_bounds__(1024) k_finalize(const double* __restrict__ raw, const Job* job, int K,
                                                   int feat, int D, double n_total, double h,
                                                   const T* shifts, double* __restrict__ stats) {
  extern __shared__ __align__(16) unsigned char dsm[];
  if (K <= 32 && blockDim.x == 1024) finalize_k32<T>(raw, job, K, feat, D, n_total, h, shifts, stats);
  else finalize_block<T>(raw, job, K, feat, D, n_total, h, shifts, stats, reinterpret_cast<double*>(dsm));
}

// ===================================================================== pass 2
template <typename T>
__device__ __forceinline__ const T* coef_ptr(const double* stats, const StatsLayout& L);
template <>
__device__ __forceinline__ const float* coef_ptr<float>(const double* stats, const StatsLayout& L) {
  return reinterpret_cast<const float*>(stats + L.Mf);
}
template <>
__device__ __forceinline__ const double* coef_ptr<double>(const double* stats,
                                                          const StatsLayout& L) {
  return stats + L.M;
}

template <typename T, int D, int FEAT, int PARAM, int KP, bool POW2>
__device__ __forceinline__ void pass2_body(const Args& a) {
  using C = G2<T, KP>;
  using P = typename std::conditional<PARAM == AFFINE, double, T>::type;
  constexpr int TP = C::TP, TS = C::TS, NT = C::NT, JB = C::JB, QN = C::QN;
  constexpr int FD = FEAT == NGF ? D : 1;
  constexpr int NA = D * (D + 1);  // affine parameters per frame
  constexpr int KSTEP2 = NT / QN;  // NCC sampling: frames k = tid/QN + KSTEP2*i
  static_assert(NT % QN == 0 && KSTEP2 * JB == KP, "pass-2 mapping");

  extern __shared__ __align__(16) unsigned char smem[];
  T* V = reinterpret_cast<T*>(smem);      // NCC: shifted values; NGF: rho
  T* GT = V + (size_t)KP * TS;            // NCC: grad T at the warped point; NGF: n
  int* crd = reinterpret_cast<int*>(GT + (size_t)KP * D * TS);
  T* Ms = reinterpret_cast<T*>(crd + 3 * TP);  // staged M' (KP <= 64)

  const int tid = threadIdx.x;
  const int K = a.K;
  const int qd = tid % QN, jg = tid / QN;
  const StatsLayout L(K);
  const T* Mg = coef_ptr<T>(a.stats, L);
  const T* frames = reinterpret_cast<const T*>(a.frames);
  const T* shifts = reinterpret_cast<const T*>(a.shifts);
  if (C::MSMEM) {
    for (int e = tid; e < KP * KP; e += NT) {
      const int i = e / KP, j = e % KP;
      Ms[e] = (i < K && j < K) ? Mg[i * K + j] : (T)0;
    }
  }
  // frames k >= K: zero rows (rho = 1 for NGF), never rewritten
  for (int e = tid; e < (KP - K) * TS; e += NT) {
    V[(size_t)K * TS + e] = FEAT == NGF ? (T)1 : (T)0;
#pragma unroll
    for (int cc = 0; cc < D; ++cc) GT[((size_t)K * D + cc) * TS + (e / TS) * D * TS + e % TS] = (T)0;
  }

  T bet[JB];
#pragma unroll
  for (int b = 0; b < JB; ++b) {
    const int j = jg * JB + b;
    bet[b] = (FEAT == NCC && j < K) ? (T)a.stats[L.beta + j] : (T)0;
  }
  double aff[PARAM == AFFINE ? JB : 1][PARAM == AFFINE ? NA : 1];
  if (PARAM == AFFINE) {
#pragma unroll
    for (int b = 0; b < JB; ++b)
#pragma unroll
      for (int e = 0; e < NA; ++e) aff[b][e] = 0.0;
  }

  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (npix + TP - 1) / TP;
  const bool yvec = PARAM == DISP && (a.y_stride % 4 == 0) &&
                    ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
  const bool ovec = PARAM == DISP && FEAT == NCC && (a.o_stride % 4 == 0) &&
                    ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0);
  const int kb = tid / QN;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long t0 = a.pix_lo + tile * TP;
    for (int pp = tid; pp < TP; pp += NT) {
      int c[3];
      coords<D>(a.g, t0 + pp, c);
      crd[3 * pp] = c[0];
      crd[3 * pp + 1] = c[1];
      crd[3 * pp + 2] = c[2];
    }
    __syncthreads();
    // ---- sampling with gradient
    if (FEAT == NCC) {
      const long long p0 = t0 + 4 * qd;
      const long long nv = a.pix_hi - p0;
      const int nvalid = nv >= 4 ? 4 : (nv > 0 ? (int)nv : 0);
      const bool vec = yvec && nvalid == 4 && (((p0 - a.y_off) & 3) == 0);
#pragma unroll
      for (int i = 0; i < JB; ++i) {
        const int k = kb + KSTEP2 * i;
        if (k < K) {
          const int fi = a.job->frame_index[k];
          const T* img = frames + (long long)fi * a.g.N;
          const T sh = shifts ? shifts[fi] : (T)0;
          T v[4], gr[4][D];
          sample_quad<T, P, D, PARAM, true, POW2>(a, img, k, p0, nvalid, vec, crd + 12 * qd, v, gr);
          T o4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) o4[e] = e < nvalid ? v[e] - sh : (T)0;
          sts4(V + (size_t)k * TS + 4 * qd, o4);
#pragma unroll
          for (int cc = 0; cc < D; ++cc) {
#pragma unroll
            for (int e = 0; e < 4; ++e) o4[e] = e < nvalid ? gr[e][cc] : (T)0;
            sts4(GT + ((size_t)k * D + cc) * TS + 4 * qd, o4);
          }
        }
      }
    } else {
      for (int it = tid; it < K * TP; it += NT) {
        const int k = it / TP, pp = it % TP;
        const long long pix = t0 + pp;
        T n[D], rho;
        if (pix < a.pix_hi) {
          const int fi = a.job->frame_index[k];
          const T* img = frames + (long long)fi * a.g.N;
          const int c[3] = {crd[3 * pp], crd[3 * pp + 1], crd[3 * pp + 2]};
          ngf_at<T, P, D, PARAM, POW2>(a, img, k, pix, c, n, rho);
        } else {
          rho = (T)1;
#pragma unroll
          for (int cc = 0; cc < D; ++cc) n[cc] = (T)0;
        }
        V[(size_t)k * TS + pp] = rho;
#pragma unroll
        for (int cc = 0; cc < D; ++cc) GT[((size_t)k * D + cc) * TS + pp] = n[cc];
      }
    }
    __syncthreads();
    // ---- coefficient contraction: acc[b][c][e] = sum_i M'_{i, j_b} X_i(c, 4qd+e)
    T acc[JB][FD][4];
#pragma unroll
    for (int b = 0; b < JB; ++b)
#pragma unroll
      for (int cc = 0; cc < FD; ++cc)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[b][cc][e] = (T)0;
    const int jb0 = jg * JB;
#pragma unroll 4
    for (int i = 0; i < K; ++i) {
      T m[JB];
      if (C::MSMEM) {
        if (JB == 4) {
          T m4[4];
          lds4(Ms + (size_t)i * KP + jb0, m4);
#pragma unroll
          for (int b = 0; b < JB; ++b) m[b] = m4[b];
        } else {
#pragma unroll
          for (int b = 0; b < JB; ++b) m[b] = Ms[(size_t)i * KP + jb0 + b];
        }
      } else {
#pragma unroll
        for (int b = 0; b < JB; ++b) m[b] = (jb0 + b < K) ? ldg(Mg + (size_t)i * K + jb0 + b) : (T)0;
      }
#pragma unroll
      for (int cc = 0; cc < FD; ++cc) {
        T x4[4];
        if (FEAT == NCC) lds4(V + (size_t)i * TS + 4 * qd, x4);
        else lds4(GT + ((size_t)i * D + cc) * TS + 4 * qd, x4);
#pragma unroll
        for (int b = 0; b < JB; ++b)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[b][cc][e] = fma(m[b], x4[e], acc[b][cc][e]);
      }
    }
    // ---- epilogue
    const long long p0 = t0 + 4 * qd;
    const long long nv = a.pix_hi - p0;
    const int nvalid = nv >= 4 ? 4 : (nv > 0 ? (int)nv : 0);
#pragma unroll
    for (int b = 0; b < JB; ++b) {
      const int j = jb0 + b;
      if (j >= K || nvalid == 0) continue;
      if (FEAT == NCC) {
        T qv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) qv[e] = acc[b][0][e] + bet[b];
        if (PARAM == DISP) {
          T* out = reinterpret_cast<T*>(a.out);
          const bool vec = ovec && nvalid == 4 && (((p0 - a.o_off) & 3) == 0);
#pragma unroll
          for (int cc = 0; cc < D; ++cc) {
            T g4[4];
            lds4(GT + ((size_t)j * D + cc) * TS + 4 * qd, g4);
#pragma unroll
            for (int e = 0; e < 4; ++e) g4[e] *= qv[e];
            T* dst = out + (long long)(j * D + cc) * a.o_stride + (p0 - a.o_off);
            if (vec) {
              stg4(dst, g4);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (e < nvalid) dst[e] = g4[e];
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (e >= nvalid) continue;
            const int pp = 4 * qd + e;
            double x[D];
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = center(a.g, d, crd[3 * pp + d]);
#pragma unroll
            for (int cc = 0; cc < D; ++cc) {
              const double gd = (double)(qv[e] * GT[((size_t)j * D + cc) * TS + pp]);
#pragma unroll
              for (int d = 0; d < D; ++d) aff[PARAM == AFFINE ? b : 0][cc * D + d] += gd * x[d];
              aff[PARAM == AFFINE ? b : 0][D * D + cc] += gd;
            }
          }
        }
      } else {
        // z = (r - n (n . r)) / rho : dD/d(grad u) through n = p / sqrt(|p|^2 + eps^2)
        T* out = reinterpret_cast<T*>(a.out);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (e >= nvalid) continue;
          const int pp = 4 * qd + e;
          T dot = (T)0;
#pragma unroll
          for (int cc = 0; cc < D; ++cc) dot += GT[((size_t)j * D + cc) * TS + pp] * acc[b][cc][e];
          const T ir = (T)1 / V[(size_t)j * TS + pp];
#pragma unroll
          for (int cc = 0; cc < D; ++cc) {
            const T z = (acc[b][cc][e] - GT[((size_t)j * D + cc) * TS + pp] * dot) * ir;
            out[(long long)(j * D + cc) * a.o_stride + (p0 + e - a.o_off)] = z;
          }
        }
      }
    }
    __syncthreads();
  }

  if (PARAM == AFFINE && FEAT == NCC) {
    // reduce the per-thread affine sums over the QN threads sharing jg (fixed order)
    double* red = reinterpret_cast<double*>(smem);
#pragma unroll 1
    for (int b = 0; b < JB; ++b) {
      for (int e = 0; e < NA; ++e) red[(size_t)e * NT + tid] = aff[PARAM == AFFINE ? b : 0][e];
      __syncthreads();
      for (int t = tid; t < C::JG * NA; t += NT) {
        const int g = t / NA, e = t % NA;
        double s = 0.0;
        for (int qq = 0; qq < QN; ++qq) s += red[(size_t)e * NT + g * QN + qq];
        const int j = g * JB + b;
        a.part_aff[((size_t)blockIdx.x * KP + j) * NA + e] = s;
      }
      __syncthreads();
    }
  }
}

template <typename T, int D, int FEAT, int PARAM, int KP>
__global__ void __launch_bounds__(G2<T, KP>::NT) k_pass2(const Args a) {
  if (a.g.pow2) pass2_body<T, D, FEAT, PARAM, KP, true>(a);
  else pass2_body<T, D, FEAT, PARAM, KP, false>(a);
}

// NGF second half of pass 2: dD/du_j = sum_a Dx_a^T z_{j,a}, then dD/dy_j = dD/du_j grad T_j(y_j).
// Adjoint of the central/one-sided difference.
template <typename T, int D>
__device__ __forceinline__ T dgrad_adjoint(const T* __restrict__ z, long long idx, long long st,
                                           int i, int n, T inv) {
  // contributions of rows k = i-1, i+1 (interior: central difference) and k = 0, n-1 (edges)
  T out = (T)0;
  const T h2 = inv * (T)0.5;
  if (i - 1 >= 1 && i - 1 <= n - 2) out += ldg(z + idx - st) * h2;
  if (i + 1 >= 1 && i + 1 <= n - 2) out -= ldg(z + idx + st) * h2;
  if (i == 0) out -= ldg(z + idx) * inv;
  if (i == 1) out += ldg(z + idx - st) * inv;
  if (i == n - 1) out += ldg(z + idx) * inv;
  if (i == n - 2) out -= ldg(z + idx + st) * inv;
  return out;
}

template <typename T, int D, int PARAM, bool POW2>
__device__ __forceinline__ void ngf_adjoint_body(const Args& a, const T* __restrict__ zb,
                                                 long long z_off, long long z_stride) {
  using P = typename std::conditional<PARAM == AFFINE, double, T>::type;
  constexpr int NA = D * (D + 1);
  const int j = blockIdx.y;
  const long long pix = a.pix_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double aff[NA];
#pragma unroll
  for (int e = 0; e < NA; ++e) aff[e] = 0.0;
  if (pix < a.pix_hi) {
    int c[3];
    coords<D>(a.g, pix, c);
    T du = (T)0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const T* z = zb + (long long)(j * D + ax) * z_stride;
      du += dgrad_adjoint<T, D>(z, pix - z_off, a.g.st[ax], c[ax], a.g.n[ax], (T)a.g.inv[ax]);
    }
    const int fi = a.job->frame_index[j];
    const T* img = reinterpret_cast<const T*>(a.frames) + (long long)fi * a.g.N;
    T gr[D];
    sample_at<T, P, D, PARAM, true, POW2>(a, img, j, pix, c, gr);
    if (PARAM == DISP) {
      T* out = reinterpret_cast<T*>(a.out);
#pragma unroll
      for (int cc = 0; cc < D; ++cc)
        out[(long long)(j * D + cc) * a.o_stride + (pix - a.o_off)] = du * gr[cc];
    } else {
      double x[D];
#pragma unroll
      for (int d = 0; d < D; ++d) x[d] = center(a.g, d, c[d]);
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        const double gd = (double)(du * gr[cc]);
#pragma unroll
        for (int d = 0; d < D; ++d) aff[cc * D + d] += gd * x[d];
        aff[D * D + cc] += gd;
      }
    }
  }
  if (PARAM == AFFINE) {
    __shared__ double red[8][NA];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < NA; ++e) {
      const double v = warp_sum(aff[e]);
      if (lane == 0) red[warp][e] = v;
    }
    __syncthreads();
    if (threadIdx.x < NA) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
      a.part_aff[((size_t)j * gridDim.x + blockIdx.x) * NA + threadIdx.x] = s;
    }
  }
}

template <typename T, int D, int PARAM>
__global__ void __launch_bounds__(256) k_ngf_adjoint(const Args a, const T* __restrict__ zb,
                                                     long long z_off, long long z_stride) {
  if (a.g.pow2) ngf_adjoint_body<T, D, PARAM, true>(a, zb, z_off, z_stride);
  else ngf_adjoint_body<T, D, PARAM, false>(a, zb, z_off, z_stride);
}

// Gather affine partials [nblk][KP][NA] (pass 2 NCC) or [K][nblk][NA] (NGF) into rows
// [K][NA] with NA = d*d + d in vec(A) ++ b order.  One warp per output element.
static __global__ void k_affine_rows(const double* __restrict__ part, int nblk, int KP, int K, int NA,
                              int layout, double* __restrict__ rows) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= K * NA) return;
  const int j = gw / NA, e = gw % NA;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32)
    s += layout == 0 ? part[((size_t)b * KP + j) * NA + e] : part[((size_t)j * nblk + b) * NA + e];
  s = warp_sum(s);
  if (lane == 0) rows[(size_t)j * NA + e] = s;
}

// ================================================================== regulariser
// Neumann Laplacian of u = y - x at integer coordinates c (one component).
template <typename T, int D>
__device__ __forceinline__ double lap_u(const Args& a, const T* __restrict__ yc, int comp,
                                        long long pix, const int (&c)[3]) {
  const double u0 = (double)ldg(yc + pix - a.y_off) - center(a.g, comp, c[comp]);
  double out = 0.0;
#pragma unroll
  for (int ax = 0; ax < D; ++ax) {
    double up = u0, um = u0;
    if (c[ax] < a.g.n[ax] - 1) {
      const int ci = ax == comp ? c[comp] + 1 : c[comp];
      up = (double)ldg(yc + pix + a.g.st[ax] - a.y_off) - center(a.g, comp, ci);
    }
    if (c[ax] > 0) {
      const int ci = ax == comp ? c[comp] - 1 : c[comp];
      um = (double)ldg(yc + pix - a.g.st[ax] - a.y_off) - center(a.g, comp, ci);
    }
    out += (up - 2.0 * u0 + um) * a.g.inv[ax] * a.g.inv[ax];
  }
  return out;
}

// ---- subsets of more than kBlockMax frames (capi.cu, large-K path): the problem runs as sub-problems of
// at most kBlockMax frames (pairs of frame blocks); these kernels move rows between the full problem and a
// sub-problem.  SubIdx: sub-problem position i <-> subset position idx[i]; part[i] = 0 input block only,
// 1 output block only, 2 both.
struct SubIdx {
  int n;
  int idx[kBlockMax];
  unsigned char part[kBlockMax];
};

// scatter a sub-problem's raw sums [G n^2 | s n | vmax n | -vmin n | count] into the full raw sums
static __global__ void __launch_bounds__(256) k_scatter_raw(const double* __restrict__ sub, const SubIdx s, int K,
                                                     double* __restrict__ raw) {
  const int n = s.n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n + 3 * n + 1; e += gridDim.x * blockDim.x) {
    if (e < n * n) {
      raw[(long long)s.idx[e / n] * K + s.idx[e % n]] = sub[e];
    } else if (e < n * n + 3 * n) {
      const int f = (e - n * n) / n, i = (e - n * n) % n;
      raw[(long long)K * K + (long long)f * K + s.idx[i]] = sub[e];
    } else {
      raw[(long long)K * K + 3LL * K] = sub[e];
    }
  }
}

// the gradient coefficients of a sub-problem: M'_sub[i][j] = M'[idx_i][idx_j] for an input frame i and an
// output frame j (else 0), beta'_sub[j] = beta'[idx_j] for an output frame when add_beta (the first input
// block of this output block), in the sub-problem's stats layout (fp64 M, fp32 copy Mf, beta)
static __global__ void __launch_bounds__(256) k_sub_stats(const double* __restrict__ stats, int K, const SubIdx s,
                                                   int add_beta, double* __restrict__ sub) {
  const StatsLayout L(K), Ls(s.n);
  const int n = s.n;
  float* mf = reinterpret_cast<float*>(sub + Ls.Mf);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n + n; e += gridDim.x * blockDim.x) {
    if (e < n * n) {
      const int i = e / n, j = e % n;
      const double v = (s.part[i] != 1 && s.part[j] != 0) ? stats[L.M + (long long)s.idx[i] * K + s.idx[j]] : 0.0;
      sub[Ls.M + e] = v;
      mf[e] = (float)v;
    } else {
      const int j = e - n * n;
      sub[Ls.beta + j] = (add_beta && s.part[j] != 0) ? stats[L.beta + s.idx[j]] : 0.0;
    }
  }
}

// rows of the sub-problem's output frames into the full gradient (first: copy, else add); rows of row_len
// elements ([d][g_stride] for displacement fields, the d*d + d affine parameters)
template <typename T>
__global__ void __launch_bounds__(256) k_acc_rows(const T* __restrict__ tmp, long long row_len, const SubIdx s,
                                                  int first, T* __restrict__ grad) {
  const int j = blockIdx.y;
  if (s.part[j] == 0) return;
  const T* src = tmp + (long long)j * row_len;
  T* dst = grad + (long long)s.idx[j] * row_len;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < row_len; e += (long long)gridDim.x * blockDim.x)
    dst[e] = first ? src[e] : dst[e] + src[e];
}

// gather rows: out[i] = src[idx_i] (the sub-problem's displacement fields)
template <typename T>
__global__ void __launch_bounds__(256) k_gather_rows(const T* __restrict__ src, long long row_len, const SubIdx s,
                                                     T* __restrict__ out) {
  const int i = blockIdx.y;
  const T* a = src + (long long)s.idx[i] * row_len;
  T* b = out + (long long)i * row_len;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < row_len; e += (long long)gridDim.x * blockDim.x)
    b[e] = a[e];
}

// T_j(y_j(x)) for every subset frame j and pixel of [pix_lo, pix_hi): out[j][pix - pix_lo] (sr_sample; the
// warped values behind CorrelationState.features, similarity.py:143-150)
template <typename T, int D, int PARAM>
__global__ void __launch_bounds__(256) k_sample_values(const Args a, T* __restrict__ out) {
  const int j = blockIdx.y;
  const long long pix = a.pix_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= a.pix_hi) return;
  int c[3];
  coords<D>(a.g, pix, c);
  const T* img = reinterpret_cast<const T*>(a.frames) + (long long)a.job->frame_index[j] * a.g.N;
  using P = typename std::conditional<PARAM == AFFINE, double, T>::type;
  P p[D];
  warp_point<T, P, D, PARAM>(a, j, pix, c, p);
  T gr[D];
  const T v = a.g.pow2 ? interp<T, P, D, false, true>(img, a.g, p, gr) : interp<T, P, D, false, false>(img, a.g, p, gr);
  out[(long long)j * (a.pix_hi - a.pix_lo) + (pix - a.pix_lo)] = v;
}

// alpha h (L L u)(pix) for u = y - x of one component (the arithmetic of k_curvature); adds this
// pixel's 1/2 alpha h (L u)^2 to *sval
template <typename T, int D>
__device__ __forceinline__ double curv_grad_at(const Args& a, const T* __restrict__ yc, int comp, long long pix,
                                               const int (&c)[3], double alpha, double h, double& sval) {
  const double l0 = lap_u<T, D>(a, yc, comp, pix, c);
  sval += 0.5 * alpha * h * l0 * l0;
  double ll = 0.0;
#pragma unroll
  for (int ax = 0; ax < D; ++ax) {
    double lp = l0, lm = l0;
    if (c[ax] < a.g.n[ax] - 1) {
      int cc[3] = {c[0], c[1], c[2]};
      cc[ax] += 1;
      lp = lap_u<T, D>(a, yc, comp, pix + a.g.st[ax], cc);
    }
    if (c[ax] > 0) {
      int cc[3] = {c[0], c[1], c[2]};
      cc[ax] -= 1;
      lm = lap_u<T, D>(a, yc, comp, pix - a.g.st[ax], cc);
    }
    ll += (lp - 2.0 * l0 + lm) * a.g.inv[ax] * a.g.inv[ax];
  }
  return alpha * h * ll;
}

template <typename T, int D>
__global__ void __launch_bounds__(256) k_curvature(const Args a, double alpha, double h,
                                                   double* __restrict__ part) {
  const int jc = blockIdx.y;  // j * D + comp
  const int comp = jc % D;
  const long long pix = a.pix_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const T* yc = reinterpret_cast<const T*>(a.y) + (long long)jc * a.y_stride;
  double sval = 0.0;
  if (pix < a.pix_hi) {
    int c[3];
    coords<D>(a.g, pix, c);
    const double l0 = lap_u<T, D>(a, yc, comp, pix, c);
    sval = 0.5 * alpha * h * l0 * l0;
    double ll = 0.0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      double lp = l0, lm = l0;
      if (c[ax] < a.g.n[ax] - 1) {
        int cc[3] = {c[0], c[1], c[2]};
        cc[ax] += 1;
        lp = lap_u<T, D>(a, yc, comp, pix + a.g.st[ax], cc);
      }
      if (c[ax] > 0) {
        int cc[3] = {c[0], c[1], c[2]};
        cc[ax] -= 1;
        lm = lap_u<T, D>(a, yc, comp, pix - a.g.st[ax], cc);
      }
      ll += (lp - 2.0 * l0 + lm) * a.g.inv[ax] * a.g.inv[ax];
    }
    T* out = reinterpret_cast<T*>(a.out) + (long long)jc * a.o_stride;
    out[pix - a.o_off] += (T)(alpha * h * ll);
  }
  __shared__ double red[8];
  const double v = warp_sum(sval);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

// ============================================================ temporal kernels
// Forward elimination / back substitution with the shared factor (cp, piv) of
// (Mask + beta*Lap); one thread per component m (thomas_solve, temporal.py:166-191).
template <typename T>
__global__ void __launch_bounds__(256) k_ls_predict(int n, long long M, const double* __restrict__ fac,
                                                    double beta, const T* __restrict__ eta,
                                                    const T* __restrict__ ref, T* __restrict__ zeta) {
  // fac layout: mask[n] | cp[n] | piv[n]
  const long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const double* mask = fac;
  const double* cp = fac + n;
  const double* piv = fac + 2 * n;
  const double off = -beta;
  double dprev = 0.0;
  for (int i = 0; i < n; ++i) {
    // Laplacian of ref at i (temporal.py:228-233)
    const double rc = (double)ref[(long long)i * M + m];
    const double rm = i > 0 ? (double)ref[(long long)(i - 1) * M + m] : 0.0;
    const double rp = i + 1 < n ? (double)ref[(long long)(i + 1) * M + m] : 0.0;
    const double lap = i == 0 ? rc - rp : (i == n - 1 ? rc - rm : 2.0 * rc - rm - rp);
    const double e = mask[i] != 0.0 ? (double)eta[(long long)i * M + m] : 0.0;
    const double rhs = mask[i] * e + beta * lap;
    const double d = i == 0 ? rhs / piv[0] : (rhs - off * dprev) / piv[i];
    zeta[(long long)i * M + m] = (T)d;  // dp, overwritten by the back substitution
    dprev = d;
  }
  double x = dprev;
  zeta[(long long)(n - 1) * M + m] = (T)x;
  for (int i = n - 2; i >= 0; --i) {
    // keep dp in double: recompute from storage only when T == double is exact
    x = (double)zeta[(long long)i * M + m] - cp[i] * x;
    zeta[(long long)i * M + m] = (T)x;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_interp_linear(int n, long long M, const int* __restrict__ left,
                                                       const int* __restrict__ right,
                                                       const double* __restrict__ theta,
                                                       const T* __restrict__ src, T* __restrict__ dst) {
  const long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (m >= M) return;
  const int l = left[t], r = right[t];
  if (r < 0) {
    dst[(long long)t * M + m] = src[(long long)l * M + m];
  } else {
    const double th = theta[t];
    dst[(long long)t * M + m] =
        (T)((1.0 - th) * (double)src[(long long)l * M + m] + th * (double)src[(long long)r * M + m]);
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) k_frame_mean(const T* __restrict__ frames, long long N,
                                                     T* __restrict__ out) {
  // one block per frame (fixed summation order: deterministic); 4 independent fp64 chains per
  // thread over 16-byte loads when the frame is 16-byte aligned
  __shared__ double red[32];
  const T* f = frames + (long long)blockIdx.x * N;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  long long head = 0;
  if (sizeof(T) == 4 && (reinterpret_cast<uintptr_t>(f) & 15) == 0) {
    const long long n4 = N / 4;
    const float4* f4 = reinterpret_cast<const float4*>(f);
    for (long long i = threadIdx.x; i < n4; i += blockDim.x) {
      const float4 v = __ldg(f4 + i);
      s[0] += (double)v.x;
      s[1] += (double)v.y;
      s[2] += (double)v.z;
      s[3] += (double)v.w;
    }
    head = n4 * 4;
  }
  for (long long i = head + threadIdx.x; i < N; i += blockDim.x) s[i & 3] += (double)f[i];
  double t0 = (s[0] + s[1]) + (s[2] + s[3]);
  t0 = warp_sum(t0);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t0;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[blockIdx.x] = (T)(v / (double)N);
  }
}

}  // namespace sr

#include "engine_ws.cuh"
#include "engine_tc.cuh"
#include "engine_ngf.cuh"

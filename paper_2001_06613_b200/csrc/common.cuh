// common.cuh — geometry, multilinear sampling and small device helpers shared by
// every kernel of the engine.  Sampling semantics follow the reference exactly
// (/root/reference/pkg/src/seqreg/grid.py:199-233):
//   t = (p - origin) / spacing - 0.5                  (cell-centre coordinate)
//   inside = all(0 <= t <= dims - 1)                   (inclusive hull test)
//   i0 = min(floor(t), dims - 2), frac = t - i0        (right-sided at nodes)
//   value = sum over 2^d corners (product((0,1), repeat=d) order) of w * T
//   grad  = d value / d t  / spacing, zero outside the hull.
// The expression order of t is kept (no FMA contraction, true division unless
// the spacing is a power of two, where multiplying by 1/s is bit-identical), so
// identity warps land exactly on nodes as in the reference.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

namespace sr {

constexpr int kMaxFrames = 256;  // subset size limit (SR_MAX_FRAMES); the kernels see at most 128 (kBlockMax)
constexpr int kBlockMax = 128;   // frames per kernel launch: larger subsets run as frame blocks (capi.cu)

// Grid geometry passed by value to every kernel.
struct Geo {
  int nd;
  int n[3];
  long long N;
  long long st[3];    // flat strides (first axis fastest)
  int sti[3];         // the same strides as int (a frame has < 2^31 cells)
  double o[3], s[3];  // origin, spacing
  double inv[3];      // 1/spacing (exact when pow2)
  float of[3], sf[3], invf[3];  // float copies for the fp32 kernels
  int pow2;           // every spacing is a power of two
};

template <typename P> __device__ __forceinline__ P geo_o(const Geo& g, int a);
template <> __device__ __forceinline__ float geo_o<float>(const Geo& g, int a) { return g.of[a]; }
template <> __device__ __forceinline__ double geo_o<double>(const Geo& g, int a) { return g.o[a]; }
template <typename P> __device__ __forceinline__ P geo_s(const Geo& g, int a);
template <> __device__ __forceinline__ float geo_s<float>(const Geo& g, int a) { return g.sf[a]; }
template <> __device__ __forceinline__ double geo_s<double>(const Geo& g, int a) { return g.s[a]; }
template <typename P> __device__ __forceinline__ P geo_inv(const Geo& g, int a);
template <> __device__ __forceinline__ float geo_inv<float>(const Geo& g, int a) { return g.invf[a]; }
template <> __device__ __forceinline__ double geo_inv<double>(const Geo& g, int a) { return g.inv[a]; }

// Per-call constants living in device memory (uploaded by the host per call).
struct Job {
  int frame_index[kMaxFrames];
  double weights[kMaxFrames];
  double affine[kMaxFrames * 12];
};

// ---------------------------------------------------------------- rounding ops
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// ---- L2 eviction-priority hints for streams that are touched once (warp y, gradient out), so
// they do not push the frames and the pass-1 samples (re-read later in the evaluation) out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float ldg_hint(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;\n" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
// the same load as a non-volatile asm: the compiler may schedule it across other memory operations
// (use only for data no kernel in flight writes)
__device__ __forceinline__ float ldg_hint_nv(const float* p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;\n" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ldg4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;\n" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg4_hint(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;\n" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}

// Programmatic dependent launch (PDL): a dependent kernel launched with programmatic stream
// serialization may start while its predecessor drains; it must wait before touching the
// predecessor's results (a no-op when launched normally).  The predecessor lets it launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Cell-centre world coordinate o + (i + 0.5) * s, rounded like numpy
// (grid.py:172-177: origin + (arange + 0.5) * spacing).
__device__ __forceinline__ double center(const Geo& g, int a, int i) {
  return __dadd_rn(g.o[a], __dmul_rn((double)i + 0.5, g.s[a]));
}

// Multilinear interpolation of `img` at world point p (precision P), values
// and gradient in precision T.  grid.py:199-233, in the reference's own
// clip-then-select form (tc = clip(t), i0 = min(floor(tc), n-2), value zeroed
// outside) so the code is branch-free and the corner loads of several samples can
// be in flight together.
__device__ __forceinline__ float clampP(float t, float hi) { return fminf(fmaxf(t, 0.f), hi); }
__device__ __forceinline__ double clampP(double t, double hi) { return fmin(fmax(t, 0.0), hi); }

__device__ __forceinline__ float floor_to(float t) { return floorf(t); }
__device__ __forceinline__ double floor_to(double t) { return floor(t); }

// POW2: every spacing is a power of two, so (p - o) / s == (p - o) * (1/s) exactly and
// the -0.5 can be fused (the product is exact, one rounding either way).
template <typename T, typename P, int D, bool GRAD, bool POW2>
__device__ __forceinline__ T interp(const T* __restrict__ img, const Geo& g, const P (&p)[D],
                                    T (&gr)[D]) {
  bool inside = true;
  T f[D];
  int base = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const P q = sub_rn(p[a], geo_o<P>(g, a));
    const P t = POW2 ? fma(q, geo_inv<P>(g, a), (P)-0.5) : sub_rn(div_rn(q, geo_s<P>(g, a)), (P)0.5);
    const P hi = (P)(g.n[a] - 1);
    const P tc = clampP(t, hi);  // NaN -> 0 (fmax returns the non-NaN operand)
    inside = inside && (tc == t);
    const P fl = fmin(floor_to(tc), hi - (P)1);  // min(floor(tc), n-2), exact in P
    f[a] = (T)(tc - fl);
    base += (int)fl * g.sti[a];
  }
  const T* q0 = img + base;
  T val;
  T gv[D];
  if (D == 2) {
    const int s1 = g.sti[1];
    const T v00 = ldg(q0), v10 = ldg(q0 + 1), v01 = ldg(q0 + s1), v11 = ldg(q0 + s1 + 1);
    const T d0 = v10 - v00, d1 = v11 - v01;
    const T a0 = fma(f[0], d0, v00), a1 = fma(f[0], d1, v01);
    const T e = a1 - a0;
    val = fma(f[1], e, a0);
    if (GRAD) {
      gv[0] = fma(f[1], d1 - d0, d0);
      gv[1] = e;
    }
  } else {
    const int s1 = g.sti[1], s2 = g.sti[D == 3 ? 2 : 1];
    T a[2][2], d[2][2];
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
      for (int c1 = 0; c1 < 2; ++c1) {
        const T* r = q0 + c1 * s1 + c2 * s2;
        const T v0 = ldg(r), v1 = ldg(r + 1);
        d[c1][c2] = v1 - v0;
        a[c1][c2] = fma(f[0], d[c1][c2], v0);
      }
    const T e0 = a[1][0] - a[0][0], e1 = a[1][1] - a[0][1];
    const T b0 = fma(f[1], e0, a[0][0]), b1 = fma(f[1], e1, a[0][1]);
    const T eb = b1 - b0;
    val = fma(f[D - 1], eb, b0);
    if (GRAD) {
      const T dz0 = fma(f[1], d[1][0] - d[0][0], d[0][0]);
      const T dz1 = fma(f[1], d[1][1] - d[0][1], d[0][1]);
      gv[0] = fma(f[2 % D], dz1 - dz0, dz0);
      gv[1] = fma(f[2 % D], e1 - e0, e0);
      gv[D - 1] = eb;
    }
  }
  if (GRAD) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const T gg = POW2 ? gv[a] * (T)geo_inv<P>(g, a) : gv[a] / (T)geo_s<P>(g, a);
      gr[a] = inside ? gg : (T)0;
    }
  }
  return inside ? val : (T)0;
}


// The value of the multilinear interpolant of an fp32 image in fp64 arithmetic (the corners are exact
// fp32 numbers, the fractions exact in P): error ~1e-16 |u| instead of ~6e-8 |u|.  The NGF feature
// takes central differences of u over one cell (h = 1/1024 at C3), which amplify an fp32 rounding of u
// by 1/(2h) relative to grad u; with |grad u| ~ eps that exceeds the 1e-4 fp32 budget, so the NGF path
// samples u through this and keeps it as an unevaluated fp32 pair hi + lo (hi = fl32(u), lo = fl32(u - hi)).
// Same corner selection, hull test and zeroing as interp (grid.py:199-233).
template <int D, bool POW2>
__device__ __forceinline__ double interp_v64(const float* __restrict__ img, const Geo& g, const float (&p)[D],
                                             float (&gr)[D]) {
  bool inside = true;
  float f[D];
  int base = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const float q = sub_rn(p[a], g.of[a]);
    const float t = POW2 ? fmaf(q, g.invf[a], -0.5f) : sub_rn(div_rn(q, g.sf[a]), 0.5f);
    const float hi = (float)(g.n[a] - 1);
    const float tc = clampP(t, hi);
    inside = inside && (tc == t);
    const float fl = fminf(floorf(tc), hi - 1.f);
    f[a] = tc - fl;
    base += (int)fl * g.sti[a];
  }
  const float* q0 = img + base;
  double val;
  float gv[D];
  if (D == 2) {
    const int s1 = g.sti[1];
    const float v00 = __ldg(q0), v10 = __ldg(q0 + 1), v01 = __ldg(q0 + s1), v11 = __ldg(q0 + s1 + 1);
    const float d0 = v10 - v00, d1 = v11 - v01;
    const float a0f = fmaf(f[0], d0, v00), a1f = fmaf(f[0], d1, v01);
    gv[0] = fmaf(f[1], d1 - d0, d0);
    gv[1] = a1f - a0f;
    const double a0 = fma((double)f[0], (double)v10 - (double)v00, (double)v00);
    const double a1 = fma((double)f[0], (double)v11 - (double)v01, (double)v01);
    val = fma((double)f[1], a1 - a0, a0);
  } else {
    const int s1 = g.sti[1], s2 = g.sti[D == 3 ? 2 : 1];
    float a[2][2], d[2][2];
    double ad[2][2];
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
      for (int c1 = 0; c1 < 2; ++c1) {
        const float* r = q0 + c1 * s1 + c2 * s2;
        const float v0 = __ldg(r), v1 = __ldg(r + 1);
        d[c1][c2] = v1 - v0;
        a[c1][c2] = fmaf(f[0], d[c1][c2], v0);
        ad[c1][c2] = fma((double)f[0], (double)v1 - (double)v0, (double)v0);
      }
    const float e0 = a[1][0] - a[0][0], e1 = a[1][1] - a[0][1];
    const float b0 = fmaf(f[1], e0, a[0][0]), b1 = fmaf(f[1], e1, a[0][1]);
    const float dz0 = fmaf(f[1], d[1][0] - d[0][0], d[0][0]);
    const float dz1 = fmaf(f[1], d[1][1] - d[0][1], d[0][1]);
    gv[0] = fmaf(f[2 % D], dz1 - dz0, dz0);
    gv[1] = fmaf(f[2 % D], e1 - e0, e0);
    gv[D - 1] = b1 - b0;
    const double b0d = fma((double)f[1], ad[1][0] - ad[0][0], ad[0][0]);
    const double b1d = fma((double)f[1], ad[1][1] - ad[0][1], ad[0][1]);
    val = fma((double)f[D - 1], b1d - b0d, b0d);
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const float gg = POW2 ? gv[a] * g.invf[a] : gv[a] / g.sf[a];
    gr[a] = inside ? gg : 0.f;
  }
  return inside ? val : 0.0;
}

// ---- split multilinear sampling (2-D), used to batch the corner gathers of many samples:
// prep: index + fractions + inside flag; fetch: the 4 corner loads; finish: the lerps.
template <typename P, bool POW2>
__device__ __forceinline__ void interp2_prep(const Geo& g, P px, P py, int& base, float& f0, float& f1,
                                             bool& inside) {
  const P q0 = sub_rn(px, geo_o<P>(g, 0)), q1 = sub_rn(py, geo_o<P>(g, 1));
  const P t0 = POW2 ? fma(q0, geo_inv<P>(g, 0), (P)-0.5) : sub_rn(div_rn(q0, geo_s<P>(g, 0)), (P)0.5);
  const P t1 = POW2 ? fma(q1, geo_inv<P>(g, 1), (P)-0.5) : sub_rn(div_rn(q1, geo_s<P>(g, 1)), (P)0.5);
  const P h0 = (P)(g.n[0] - 1), h1 = (P)(g.n[1] - 1);
  const P c0 = clampP(t0, h0), c1 = clampP(t1, h1);
  inside = (c0 == t0) && (c1 == t1);
  const P l0 = fmin(floor_to(c0), h0 - (P)1), l1 = fmin(floor_to(c1), h1 - (P)1);
  f0 = (float)(c0 - l0);
  f1 = (float)(c1 - l1);
  base = (int)l0 + (int)l1 * g.sti[1];
}


// Flat pixel index -> integer coordinates.
template <int D>
__device__ __forceinline__ void coords(const Geo& g, long long pix, int (&c)[3]) {
  c[0] = (int)(pix % g.n[0]);
  if (D >= 2) {
    long long r = pix / g.n[0];
    c[1] = (int)(r % g.n[1]);
    if (D == 3) c[2] = (int)(r / g.n[1]);
    else c[2] = 0;
  } else {
    c[1] = 0;
    c[2] = 0;
  }
}

// ------------------------------------------------------------ warp reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// 4 consecutive T from global memory (16B-aligned): LDG.128 (float) or 2x LDG.128 (double).
__device__ __forceinline__ void ldg4(const float* p, float (&r)[4]) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
}
__device__ __forceinline__ void ldg4(const double* p, double (&r)[4]) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p + 2));
  r[0] = a.x; r[1] = a.y; r[2] = b.x; r[3] = b.y;
}
__device__ __forceinline__ void sts4(float* p, const float (&r)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
}
__device__ __forceinline__ void sts4(double* p, const double (&r)[4]) {
  *reinterpret_cast<double2*>(p) = make_double2(r[0], r[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(r[2], r[3]);
}
__device__ __forceinline__ void stg4(float* p, const float (&r)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
}
__device__ __forceinline__ void stg4(double* p, const double (&r)[4]) {
  *reinterpret_cast<double2*>(p) = make_double2(r[0], r[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(r[2], r[3]);
}

// 4 consecutive T from shared memory (16B-aligned): one LDS.128 (float) or two (double).
__device__ __forceinline__ void lds4(const float* p, float (&r)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
}
__device__ __forceinline__ void lds4(const double* p, double (&r)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  r[0] = a.x; r[1] = a.y; r[2] = b.x; r[3] = b.y;
}

}  // namespace sr

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

constexpr int kMaxFrames = 128;

// Grid geometry passed by value to every kernel.
struct Geo {
  int nd;
  int n[3];
  long long N;
  long long st[3];    // flat strides (first axis fastest)
  double o[3], s[3];  // origin, spacing
  double inv[3];      // 1/spacing (exact when pow2)
  int pow2;           // every spacing is a power of two
};

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

template <typename T, typename P, int D, bool GRAD>
__device__ __forceinline__ T interp(const T* __restrict__ img, const Geo& g, const P (&p)[D],
                                    T (&gr)[D]) {
  bool inside = true;
  T f[D], h[D];
  long long base = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    P q = sub_rn(p[a], (P)g.o[a]);
    q = g.pow2 ? mul_rn(q, (P)g.inv[a]) : div_rn(q, (P)g.s[a]);
    const P t = sub_rn(q, (P)0.5);
    const P hi = (P)(g.n[a] - 1);
    inside = inside && (t >= (P)0) && (t <= hi);
    const P tc = clampP(t, hi);  // NaN -> 0 (fmax returns the non-NaN operand)
    int i = (int)tc;
    i = min(i, g.n[a] - 2);
    f[a] = (T)(tc - (P)i);
    h[a] = (T)1 - f[a];
    base += (long long)i * g.st[a];
  }
  T val = (T)0;
  T gacc[D];
#pragma unroll
  for (int a = 0; a < D; ++a) gacc[a] = (T)0;
  // corners in itertools.product((0,1), repeat=D) order: axis 0 is the slowest bit
#pragma unroll
  for (int c = 0; c < (1 << D); ++c) {
    long long off = 0;
    T w = (T)1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int ca = (c >> (D - 1 - a)) & 1;
      off += ca ? g.st[a] : 0;
      w *= ca ? f[a] : h[a];
    }
    const T v = ldg(img + base + off);
    val += w * v;
    if (GRAD) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        T dw = (T)1;
#pragma unroll
        for (int b = 0; b < D; ++b) {
          if (b == a) continue;
          const int cb = (c >> (D - 1 - b)) & 1;
          dw *= cb ? f[b] : h[b];
        }
        const int ca = (c >> (D - 1 - a)) & 1;
        gacc[a] += ca ? dw * v : -dw * v;
      }
    }
  }
  if (GRAD) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const T gv = g.pow2 ? gacc[a] * (T)g.inv[a] : gacc[a] / (T)g.s[a];
      gr[a] = inside ? gv : (T)0;
    }
  }
  return inside ? val : (T)0;
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

// pyramid.cuh — spatial hierarchy kernels.
//
// Pyramid step (/root/reference/pkg/src/seqreg/pyramid.py:22-54, build_pyramid 68-91):
//   smooth   separable [1, 2, 1] / 4 along axis 0, then 1 (then 2), scipy.ndimage.convolve1d with
//            mode="reflect" (x[-1] = x[0], x[n] = x[n-1]).  scipy's symmetric-kernel loop computes
//            0.5 x[i] + 0.25 (x[i-1] + x[i+1]) (checked bit for bit); the products are exact, so
//            the only roundings are the pair sum and the final add, reproduced here in fp64.
//   restrict block means of 2^d cells, axis 0 first (np.add.reduceat then / size): per axis
//            (a + b) / 2, or a / 1 for the trailing cell of an odd axis.
// fp64 stacks are bit-identical to the reference; fp32 stacks are computed in fp64 from the fp32
// values and rounded to fp32 once per level.
//
// Field prolongation (absent in the reference): u = y - x on the coarse grid is
// interpolated multilinearly at the fine cell centres with coordinates clamped to the coarse hull
// (edge replication); y_fine = x_fine + u.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace sr {

struct PyrDims {
  int nd;
  int n[3];
  long long N;
};

// One pyramid step, fused: thread = one coarse cell of one frame.  The smoothed values of the
// (up to) 2^d fine cells of the block are formed from their 4^d neighbourhood in registers in the
// reference's order (S0 along axis 0, then S1 along axis 1, then S2 along axis 2, each
// 0.5 x + 0.25 (x- + x+) with clamped neighbours = reflect for a 3-tap kernel), then the block
// mean axis 0 first.  Axes of length 1 (1-D / 2-D stacks) reproduce the reference exactly:
// smoothing a length-1 axis is the identity in floating point and its block has one cell.
__device__ __forceinline__ double smooth3(double xm, double x, double xp) {
  return __dadd_rn(__dmul_rn(0.5, x), __dmul_rn(0.25, __dadd_rn(xm, xp)));
}
__device__ __forceinline__ double bmean(double a, double b, int cnt) {
  return cnt == 2 ? __ddiv_rn(__dadd_rn(a, b), 2.0) : __ddiv_rn(a, 1.0);
}

template <typename T, bool D3>
__global__ void __launch_bounds__(256) k_pyramid(const T* __restrict__ src, T* __restrict__ dst, PyrDims f,
                                                 PyrDims c) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;  // coarse axis-0 index
  const int JK = blockIdx.y;                              // coarse (axis-1, axis-2) row
  if (I >= c.n[0]) return;
  const int J = JK % c.n[1], K2 = JK / c.n[1];
  const long long fr = blockIdx.z;
  const T* s = src + fr * f.N;
  const int n0 = f.n[0], n1 = f.n[1], n2 = f.n[2];
  const int cnt0 = 2 * I + 1 < n0 ? 2 : 1, cnt1 = 2 * J + 1 < n1 ? 2 : 1, cnt2 = 2 * K2 + 1 < n2 ? 2 : 1;
  auto cl = [](int v, int n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); };
  int xs[4], ys[4], zs[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    xs[q] = cl(2 * I - 1 + q, n0);
    ys[q] = cl(2 * J - 1 + q, n1);
    zs[q] = cl(2 * K2 - 1 + q, n2);
  }
  // S0 at x in {2I, 2I+1} for y rows q = 0..3 (and z planes)
  constexpr int NZ = D3 ? 4 : 1;
  double s1v[NZ][2][2];  // [z plane][y in {2J, 2J+1}][x in {2I, 2I+1}] after S0 and S1
#pragma unroll
  for (int zq = 0; zq < NZ; ++zq) {
    const long long zoff = D3 ? (long long)zs[zq] * n0 * n1 : 0;
    double s0v[4][2];
#pragma unroll
    for (int yq = 0; yq < 4; ++yq) {
      const T* row = s + zoff + (long long)ys[yq] * n0;
      const double a = (double)row[xs[0]], b = (double)row[xs[1]], cc = (double)row[xs[2]], d = (double)row[xs[3]];
      s0v[yq][0] = smooth3(a, b, cc);
      s0v[yq][1] = smooth3(b, cc, d);
    }
#pragma unroll
    for (int yy = 0; yy < 2; ++yy)
#pragma unroll
      for (int xx = 0; xx < 2; ++xx) s1v[zq][yy][xx] = smooth3(s0v[yy][xx], s0v[yy + 1][xx], s0v[yy + 2][xx]);
  }
  double m2[2];
#pragma unroll
  for (int zz = 0; zz < (D3 ? 2 : 1); ++zz) {
    double sv[2][2];
#pragma unroll
    for (int yy = 0; yy < 2; ++yy)
#pragma unroll
      for (int xx = 0; xx < 2; ++xx)
        sv[yy][xx] = D3 ? smooth3(s1v[zz][yy][xx], s1v[zz + 1][yy][xx], s1v[zz + 2][yy][xx]) : s1v[0][yy][xx];
    const double r0 = bmean(sv[0][0], sv[0][1], cnt0), r1 = bmean(sv[1][0], sv[1][1], cnt0);
    m2[zz] = bmean(r0, r1, cnt1);
  }
  const double v = D3 ? bmean(m2[0], m2[1], cnt2) : m2[0];
  dst[fr * c.N + ((long long)K2 * c.n[1] + J) * c.n[0] + I] = (T)v;
}

// y_fine[j][c][p] = x_fine_c(p) + interp(u_c)(x_fine(p)),  u_c = y_coarse[j][c] - x_coarse_c.
// Thread = one fine cell x FG frames (blockIdx.y = frame group); the interpolation geometry is formed
// once and reused for the group.
template <typename T, int D, int FG>
__global__ void __launch_bounds__(256) k_prolong_field(const T* __restrict__ yc, T* __restrict__ yf, Geo gc, Geo gf,
                                                       int k) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= gf.N) return;
  int cf[3] = {p % gf.n[0], 0, 0};
  if (D > 1) cf[1] = (p / gf.n[0]) % gf.n[1];
  if (D > 2) cf[2] = p / (gf.n[0] * gf.n[1]);
  double xf[D], fr[D];
  int i0[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    xf[a] = center(gf, a, cf[a]);
    const double t = (xf[a] - gc.o[a]) / gc.s[a] - 0.5;
    const double hi = (double)(gc.n[a] - 1);
    const double tc = fmin(fmax(t, 0.0), hi);
    const double fl = fmin(floor(tc), hi - 1.0);
    i0[a] = (int)fl;
    fr[a] = tc - fl;
  }
  constexpr int NC = 1 << D;
  double w[NC], xcc[D][2];
  int idx[NC];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    xcc[a][0] = center(gc, a, i0[a]);
    xcc[a][1] = center(gc, a, i0[a] + 1);
  }
#pragma unroll
  for (int corner = 0; corner < NC; ++corner) {
    double ww = 1.0;
    int id = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int b = (corner >> a) & 1;
      ww *= b ? fr[a] : 1.0 - fr[a];
      id += (i0[a] + b) * gc.sti[a];
    }
    w[corner] = ww;
    idx[corner] = id;
  }
#pragma unroll
  for (int jj = 0; jj < FG; ++jj) {
    const int j = blockIdx.y * FG + jj;
    if (j >= k) break;
#pragma unroll
    for (int comp = 0; comp < D; ++comp) {
      const T* u = yc + ((long long)j * D + comp) * gc.N;
      double acc = 0.0;
#pragma unroll
      for (int corner = 0; corner < NC; ++corner)
        acc += w[corner] * ((double)u[idx[corner]] - xcc[comp][(corner >> comp) & 1]);
      yf[((long long)j * D + comp) * gf.N + p] = (T)(xf[comp] + acc);
    }
  }
}

}  // namespace sr

// engine_ngf.cuh — split NGF path (fp32, displacement fields, K <= 128): no neighbour re-sampling,
// tensor-core Gram, streaming pass 2.  DESIGN.md §4.
//
//   k_ngf_sfeat2f (2-D)                    sampling fused with the feature: u = T_k(y_k) (fp64 value),
//                                          n = grad_h u / rho, 1/rho, grad T_k; one warp per (frame, row
//                                          segment, 62-column chunk); k_ngf_sfeat2 = its generic fallback
//   k_sample_vp<LO> (engine_tc.cuh)        3-D: u (fp64 arithmetic, kept as an fp32 pair) and grad T_k over
//   + k_ngf_feat4                          the slab +- 2 rows, then n, 1/rho (the stencil of ngf_at)
//   k_gram_h<64|128>                       raw Gram  sum_(p, c) n_i n_j  over the slab on tcgen05 (kind::f16,
//                                          hi / lo split), K > 32; k_gram_tma<NGF> (mma.sync) for K <= 32
//   k_ngf_z_tc (engine_ngf_tc.cuh)         r = M'^T n (per pixel and component) on tcgen05,
//                                          z = (r - n (n.r)) / rho
//   k_ngf_adj4                             dD/dy = (D_h^T z) grad T
#pragma once
#include <cuda_fp16.h>

namespace sr {

__device__ __forceinline__ void coords_flat(const Geo& g, int p, int (&c)[3]) {
  c[0] = p % g.n[0];
  c[1] = g.nd > 1 ? (p / g.n[0]) % g.n[1] : 0;
  c[2] = g.nd > 2 ? p / (g.n[0] * g.n[1]) : 0;
}

// n and 1/rho at pixels [zlo, zhi) of every subset frame (the stencil and float arithmetic of ngf_at,
// engine.cuh: central differences inside, one-sided at the domain edge, world units), 4 consecutive pixels
// per thread: one coordinate
// decomposition per thread (then incremented), 32-bit offsets inside a frame's plane, 128-bit stores of
// n and rho when the z plane allows them.  (k_ngf_feat: ~200 instructions per pixel, issue-bound.)
// u = V + VL (an unevaluated fp32 pair, k_sample_vp<LO>): a difference of u is formed as
// (V_+ - V_-) + (VL_+ - VL_-), accurate to fp32 relative to the difference itself.
template <int D>
__global__ void __launch_bounds__(256) k_ngf_feat4(const Args a, const float* __restrict__ V,
                                                   const float* __restrict__ VL, long long vlo,
                                                   long long vstride, float* __restrict__ Nf, float* __restrict__ IRho,
                                                   long long zlo, long long zhi, long long zstride) {
  const int k = blockIdx.y;
  const int nz = (int)(zhi - zlo);
  const int q0 = (blockIdx.x * 256 + threadIdx.x) * 4;  // z-relative first pixel
  if (q0 >= nz) return;
  const float* u = V + (long long)k * vstride + (zlo - vlo);  // u[q]: pixel zlo + q
  const float* ul = VL + (long long)k * vstride + (zlo - vlo);
  float* nb = Nf + (long long)k * D * zstride;
  float* rb = IRho + (long long)k * zstride;
  const int p0 = (int)zlo + q0;
  int c[3];
  coords_flat(a.g, p0, c);
  const float e = (float)a.eps;
  float nv[D][4], rv[4];
  // vector path: the 4 pixels share their row (n0 % 4 == 0, aligned ranges); the u rows come as 128-bit loads.
  // Domain edges are handled without a second path (a 128-pixel 3-D row puts a boundary thread in every
  // warp): the neighbour index is clamped (u(-1) := u(0): the one-sided difference) and the factor is 1/s
  // instead of 1/(2 s) there; the same expressions as the per-pixel path below, so the same bits.
  bool inner = q0 + 4 <= nz && (a.g.n[0] & 3) == 0 && ((zlo | vlo) & 3) == 0 && (vstride & 3) == 0 &&
               ((reinterpret_cast<uintptr_t>(V) | reinterpret_cast<uintptr_t>(VL)) & 15) == 0;
#pragma unroll
  for (int ax = 1; ax < D; ++ax) inner = inner && (a.g.sti[ax] & 3) == 0;
  if (inner) {
    float g4[D][4];
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      float um[4], up[4], dl[4], f[4];
      const float inv = a.g.invf[ax];
      if (ax == 0) {
        const bool hm = c[0] > 0, hp = c[0] + 3 < a.g.n[0] - 1;  // the row continues to the left / right
        const float4 u0 = __ldg(reinterpret_cast<const float4*>(u + q0));
        um[0] = hm ? __ldg(u + q0 - 1) : u0.x, um[1] = u0.x, um[2] = u0.y, um[3] = u0.z;
        up[0] = u0.y, up[1] = u0.z, up[2] = u0.w, up[3] = hp ? __ldg(u + q0 + 4) : u0.w;
        const float4 l0 = __ldg(reinterpret_cast<const float4*>(ul + q0));
        dl[0] = l0.y - (hm ? __ldg(ul + q0 - 1) : l0.x), dl[1] = l0.z - l0.x, dl[2] = l0.w - l0.y;
        dl[3] = (hp ? __ldg(ul + q0 + 4) : l0.w) - l0.z;
        f[0] = hm ? inv * 0.5f : inv, f[1] = f[2] = inv * 0.5f, f[3] = hp ? inv * 0.5f : inv;
      } else {
        const bool hm = c[ax] > 0, hp = c[ax] < a.g.n[ax] - 1;
        const int st = a.g.sti[ax], sm = hm ? st : 0, sp = hp ? st : 0;
        const float4 m4 = __ldg(reinterpret_cast<const float4*>(u + q0 - sm));
        const float4 p4 = __ldg(reinterpret_cast<const float4*>(u + q0 + sp));
        um[0] = m4.x, um[1] = m4.y, um[2] = m4.z, um[3] = m4.w;
        up[0] = p4.x, up[1] = p4.y, up[2] = p4.z, up[3] = p4.w;
        const float4 lm = __ldg(reinterpret_cast<const float4*>(ul + q0 - sm));
        const float4 lp = __ldg(reinterpret_cast<const float4*>(ul + q0 + sp));
        dl[0] = lp.x - lm.x, dl[1] = lp.y - lm.y, dl[2] = lp.z - lm.z, dl[3] = lp.w - lm.w;
        f[0] = f[1] = f[2] = f[3] = (hm && hp) ? inv * 0.5f : inv;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) g4[ax][t] = ((up[t] - um[t]) + dl[t]) * f[t];
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      float pn = 0.f;
#pragma unroll
      for (int ax = 0; ax < D; ++ax) pn += g4[ax][t] * g4[ax][t];
      const float rho = sqrtf(pn + e * e);
      const float ir = 1.f / rho;
#pragma unroll
      for (int ax = 0; ax < D; ++ax) nv[ax][t] = g4[ax][t] * ir;
      rv[t] = ir;
    }
  } else
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int q = q0 + t;
    float g[D], pn = 0.f;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const bool hp = c[ax] < a.g.n[ax] - 1, hm = c[ax] > 0;
      const int st = a.g.sti[ax];
      const int qp = hp ? q + st : q, qm = hm ? q - st : q;
      const float du = (__ldg(u + qp) - __ldg(u + qm)) + (__ldg(ul + qp) - __ldg(ul + qm));
      const float inv = a.g.invf[ax];
      g[ax] = (hp && hm) ? du * (inv * 0.5f) : du * inv;
      pn += g[ax] * g[ax];
    }
    const float rho = sqrtf(pn + e * e);
    const float ir = __frcp_rn(rho);  // = 1.f / rho (correctly rounded)
#pragma unroll
    for (int ax = 0; ax < D; ++ax) nv[ax][t] = g[ax] * ir;
    rv[t] = ir;
    if (++c[0] == a.g.n[0]) {  // next pixel
      c[0] = 0;
      if (D > 1 && ++c[1] == a.g.n[1]) {
        c[1] = 0;
        ++c[2];
      }
    }
  }
  if (q0 + 4 <= nz && (zstride & 3) == 0) {
#pragma unroll
    for (int ax = 0; ax < D; ++ax)
      *reinterpret_cast<float4*>(nb + ax * zstride + q0) = make_float4(nv[ax][0], nv[ax][1], nv[ax][2], nv[ax][3]);
    *reinterpret_cast<float4*>(rb + q0) = make_float4(rv[0], rv[1], rv[2], rv[3]);
  } else {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (q0 + t < nz) {
#pragma unroll
        for (int ax = 0; ax < D; ++ax) nb[ax * zstride + q0 + t] = nv[ax][t];
        rb[q0 + t] = rv[t];
      }
  }
}

// dD/dy = (D_h^T z) grad T, 4 consecutive pixels per thread (same arithmetic as dgrad_adjoint), 128-bit
// grad T loads and dD/dy stores when aligned.
// CURV (sr_evaluate_reg): the curvature gradient alpha h L L (y - x) of the same pixels is added to the
// output in the same launch (same arithmetic and the same float addition as k_curvature after this kernel),
// and the CTA's share of S goes to a.curv_part[blockIdx.y * gridDim.x + blockIdx.x].
// alpha h (L L u) of 4 consecutive pixels of one row (2-D, u = y - x of one component) and their share of S,
// the arithmetic of curv_grad_at / lap_u (Neumann Laplacian: a missing neighbour is the value itself, i.e. every
// index clamped into the grid, first for the position of a Laplacian, then for its neighbours) with the u patch
// loaded once: rows j - 2 .. j + 2, 28 values and 14 Laplacians for the 4 pixels instead of 100 and 20 (the
// per-pixel form costs ~1000 fp64 instructions per voxel-frame and made sr_evaluate_reg 5x a plain evaluation).
template <typename T>
__device__ __forceinline__ void curv4_d2(const Args& a, const T* __restrict__ yc, int comp, long long p0, int c0,
                                         int c1, int nvalid, double alpha, double h, float (&cv)[4], double& sval) {
  const int n0 = a.g.n[0], n1 = a.g.n[1];
  const long long st1 = a.g.st[1];
  const double i0 = a.g.inv[0], i1 = a.g.inv[1];
  const T* yb = yc + (p0 - a.y_off);
  auto U = [&](int i, int j) -> double {  // u at the clamped (i, j)
    const int ic = min(max(i, 0), n0 - 1), jc = min(max(j, 0), n1 - 1);
    const double ctr = comp == 0 ? center(a.g, 0, ic) : center(a.g, 1, jc);
    return (double)ldg(yb + (ic - c0) + (long long)(jc - c1) * st1) - ctr;
  };
  double r0[4], r1[6], r2[8], r3[6], r4[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) r0[e] = U(c0 + e, c1 - 2), r4[e] = U(c0 + e, c1 + 2);
#pragma unroll
  for (int e = 0; e < 6; ++e) r1[e] = U(c0 - 1 + e, c1 - 1), r3[e] = U(c0 - 1 + e, c1 + 1);
#pragma unroll
  for (int e = 0; e < 8; ++e) r2[e] = U(c0 - 2 + e, c1);
  double lc[6], lu[4], ld[4];
#pragma unroll
  for (int e = 0; e < 6; ++e) {  // Laplacian at (c0 - 1 + e, c1)
    double o = 0.0;
    o += (r2[e + 2] - 2.0 * r2[e + 1] + r2[e]) * i0 * i0;
    o += (r3[e] - 2.0 * r2[e + 1] + r1[e]) * i1 * i1;
    lc[e] = o;
  }
  if (c0 == 0) lc[0] = lc[1];            // position -1 := position 0
  if (c0 + 4 >= n0) lc[5] = lc[4];       // position n0 := position n0 - 1
#pragma unroll
  for (int t = 0; t < 4; ++t) {  // Laplacians at (c0 + t, c1 - 1) and (c0 + t, c1 + 1)
    double o = 0.0;
    o += (r1[t + 2] - 2.0 * r1[t + 1] + r1[t]) * i0 * i0;
    o += (r2[t + 2] - 2.0 * r1[t + 1] + r0[t]) * i1 * i1;
    lu[t] = c1 > 0 ? o : lc[t + 1];
    double q = 0.0;
    q += (r3[t + 2] - 2.0 * r3[t + 1] + r3[t]) * i0 * i0;
    q += (r4[t] - 2.0 * r3[t + 1] + r2[t + 2]) * i1 * i1;
    ld[t] = c1 < n1 - 1 ? q : lc[t + 1];
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const double l0 = lc[t + 1];
    double ll = 0.0;
    ll += (lc[t + 2] - 2.0 * l0 + lc[t]) * i0 * i0;
    ll += (ld[t] - 2.0 * l0 + lu[t]) * i1 * i1;
    cv[t] = (float)(alpha * h * ll);
    if (t < nvalid) sval += 0.5 * alpha * h * l0 * l0;
  }
}

// (D_h^T z) terms of one axis at index i of n: rows i - 1, i + 1 (interior) and the one-sided edge rows
// (dgrad_adjoint); zm, z0, zp = z at i - 1, i, i + 1 (any finite value where the row does not exist)
__device__ __forceinline__ float adj_terms(int i, int n, float zm, float z0, float zp, float h2, float inv) {
  float o = 0.f;
  if (i - 1 >= 1 && i - 1 <= n - 2) o += zm * h2;
  if (i + 1 >= 1 && i + 1 <= n - 2) o -= zp * h2;
  if (i == 0) o -= z0 * inv;
  if (i == 1) o += zm * inv;
  if (i == n - 1) o += z0 * inv;
  if (i == n - 2) o -= zp * inv;
  return o;
}

template <int D, bool CURV = false>
__global__ void __launch_bounds__(256) k_ngf_adj4(const Args a, const float* __restrict__ Z, long long zlo,
                                                  long long zstride, const float* __restrict__ Gv, long long vlo,
                                                  long long vstride) {
  const int k = blockIdx.y;
  const int npix = (int)(a.pix_hi - a.pix_lo);
  const int q0 = (blockIdx.x * 256 + threadIdx.x) * 4;  // slab-relative first pixel
  if (!CURV && q0 >= npix) return;
  double sval = 0.0;
  if (q0 < npix) {
  const int p0 = (int)a.pix_lo + q0;
  int c[3];
  coords_flat(a.g, p0, c);
  float du[4];
  // vector path: the 4 pixels share their row; the z rows come as 128-bit loads with clamped row / column
  // offsets at the domain edges (no second path: a 128-pixel 3-D row puts a boundary thread in every warp),
  // and adj_terms applies the per-pixel edge rules: the per-pixel path's expressions, so the same bits
  bool inner3 = D == 3 && q0 + 4 <= npix && (a.g.n[0] & 3) == 0 && (c[0] & 3) == 0 && ((p0 - zlo) & 3) == 0 &&
               (zstride & 3) == 0 && (reinterpret_cast<uintptr_t>(Z) & 15) == 0;
#pragma unroll
  for (int ax = 1; ax < D; ++ax) inner3 = inner3 && (a.g.sti[ax] & 3) == 0;
  if (inner3) {
#pragma unroll
    for (int t = 0; t < 4; ++t) du[t] = 0.f;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const float* z = Z + ((long long)k * D + ax) * zstride + (p0 - zlo);
      const float inv = a.g.invf[ax], h2 = inv * 0.5f;
      const int n = a.g.n[ax];
      float zm[4], zp[4], z0[4];
      if (ax == 0) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(z));
        z0[0] = v.x, z0[1] = v.y, z0[2] = v.z, z0[3] = v.w;
        zm[0] = c[0] > 0 ? __ldg(z - 1) : v.x, zm[1] = v.x, zm[2] = v.y, zm[3] = v.z;
        zp[0] = v.y, zp[1] = v.z, zp[2] = v.w, zp[3] = c[0] + 4 < n ? __ldg(z + 4) : v.w;
#pragma unroll
        for (int t = 0; t < 4; ++t) du[t] += adj_terms(c[0] + t, n, zm[t], z0[t], zp[t], h2, inv);
      } else {
        const int i = c[ax], st = a.g.sti[ax];
        const float4 m4 = __ldg(reinterpret_cast<const float4*>(z - (i > 0 ? st : 0)));
        const float4 p4 = __ldg(reinterpret_cast<const float4*>(z + (i < n - 1 ? st : 0)));
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i == 0 || i == n - 1) v = __ldg(reinterpret_cast<const float4*>(z));
        zm[0] = m4.x, zm[1] = m4.y, zm[2] = m4.z, zm[3] = m4.w;
        zp[0] = p4.x, zp[1] = p4.y, zp[2] = p4.z, zp[3] = p4.w;
        z0[0] = v.x, z0[1] = v.y, z0[2] = v.z, z0[3] = v.w;
#pragma unroll
        for (int t = 0; t < 4; ++t) du[t] += adj_terms(i, n, zm[t], z0[t], zp[t], h2, inv);
      }
    }
  } else {
  // interior fast path: the 4 pixels share their row and every axis index stays in 2 .. n - 3, so
  // (D_h^T z)(p) = sum_ax (z[p - st] - z[p + st]) h / 2; the z rows come as 128-bit loads
  // (2-D only, as in k_ngf_feat4)
  bool inner = D == 2 && q0 + 4 <= npix && c[0] >= 2 && c[0] + 3 <= a.g.n[0] - 3 && ((p0 - zlo) & 3) == 0 &&
               (zstride & 3) == 0 && (reinterpret_cast<uintptr_t>(Z) & 15) == 0;
#pragma unroll
  for (int ax = 1; ax < D; ++ax) inner = inner && c[ax] >= 2 && c[ax] <= a.g.n[ax] - 3 && (a.g.sti[ax] & 3) == 0;
  if (inner) {
#pragma unroll
    for (int t = 0; t < 4; ++t) du[t] = 0.f;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const float* z = Z + ((long long)k * D + ax) * zstride + (p0 - zlo);
      const float h2 = a.g.invf[ax] * 0.5f;
      float zm[4], zp[4];
      if (ax == 0) {
        const float4 z0 = __ldg(reinterpret_cast<const float4*>(z));
        zm[0] = __ldg(z - 1), zm[1] = z0.x, zm[2] = z0.y, zm[3] = z0.z;
        zp[0] = z0.y, zp[1] = z0.z, zp[2] = z0.w, zp[3] = __ldg(z + 4);
      } else {
        const int st = a.g.sti[ax];
        const float4 m4 = __ldg(reinterpret_cast<const float4*>(z - st)), p4 = __ldg(reinterpret_cast<const float4*>(z + st));
        zm[0] = m4.x, zm[1] = m4.y, zm[2] = m4.z, zm[3] = m4.w;
        zp[0] = p4.x, zp[1] = p4.y, zp[2] = p4.z, zp[3] = p4.w;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float o = 0.f;  // the general path's expression order
        o += zm[t] * h2;
        o -= zp[t] * h2;
        du[t] += o;
      }
    }
  } else
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    float acc = 0.f;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const float* z = Z + ((long long)k * D + ax) * zstride + (p0 - zlo);
      const int st = a.g.sti[ax], i = c[ax], n = a.g.n[ax];
      const float inv = a.g.invf[ax];
      const float h2 = inv * 0.5f;
      float o = 0.f;  // dgrad_adjoint: rows i - 1, i + 1 (interior) and the one-sided edge rows
      if (i - 1 >= 1 && i - 1 <= n - 2) o += __ldg(z + t - st) * h2;
      if (i + 1 >= 1 && i + 1 <= n - 2) o -= __ldg(z + t + st) * h2;
      if (i == 0) o -= __ldg(z + t) * inv;
      if (i == 1) o += __ldg(z + t - st) * inv;
      if (i == n - 1) o += __ldg(z + t) * inv;
      if (i == n - 2) o -= __ldg(z + t + st) * inv;
      acc += o;
    }
    du[t] = acc;
    if (++c[0] == a.g.n[0]) {
      c[0] = 0;
      if (D > 1 && ++c[1] == a.g.n[1]) {
        c[1] = 0;
        ++c[2];
      }
    }
  }
  }  // !inner3
  float* out = reinterpret_cast<float*>(a.out);
  const long long go = (long long)(p0 - vlo), oo = (long long)p0 - a.o_off;
  const bool vec = q0 + 4 <= npix && ((go | vstride) & 3) == 0 && ((oo | a.o_stride) & 3) == 0 &&
                   ((reinterpret_cast<uintptr_t>(Gv) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
#pragma unroll
  for (int cc = 0; cc < D; ++cc) {
    const float* gs = Gv + ((long long)k * D + cc) * vstride + go;
    float* dst = out + ((long long)k * D + cc) * a.o_stride + oo;
    float cv[4] = {0.f, 0.f, 0.f, 0.f};
    if (CURV) {
      const float* yc = reinterpret_cast<const float*>(a.y) + (long long)(k * D + cc) * a.y_stride;
      int cq[3];
      coords_flat(a.g, p0, cq);
      if (D == 2 && (a.g.n[0] & 3) == 0 && (cq[0] & 3) == 0 && q0 + 4 <= npix) {
        curv4_d2<float>(a, yc, cc, p0, cq[0], cq[1], 4, a.curv_alpha, a.curv_h, cv, sval);
      } else
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (q0 + t < npix) cv[t] = (float)curv_grad_at<float, D>(a, yc, cc, p0 + t, cq, a.curv_alpha, a.curv_h, sval);
        if (++cq[0] == a.g.n[0]) {
          cq[0] = 0;
          if (D > 1 && ++cq[1] == a.g.n[1]) {
            cq[1] = 0;
            ++cq[2];
          }
        }
      }
    }
    if (vec) {
      const float4 gv = __ldg(reinterpret_cast<const float4*>(gs));
      float4 o = make_float4(du[0] * gv.x, du[1] * gv.y, du[2] * gv.z, du[3] * gv.w);
      if (CURV) o.x += cv[0], o.y += cv[1], o.z += cv[2], o.w += cv[3];
      *reinterpret_cast<float4*>(dst) = o;
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (q0 + t < npix) {
          float o = du[t] * __ldg(gs + t);
          if (CURV) o += cv[t];
          dst[t] = o;
        }
    }
  }
  }  // q0 < npix
  if (CURV) {
    __shared__ double red[8];
    const double v = warp_sum(sval);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
      a.curv_part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
  }
}

// ------------------------------------------------------------------------------------------
// k_gram_h (K in 33..128): raw NGF Gram G_ij = sum over the slab's pixels and components of n_i n_j on
// tcgen05 kind::f16 operands with TMEM accumulators.  (Its round-2 predecessor k_gram_tcx — kind::tf32 hi / lo
// split of 32-pixel tiles, fp64 accumulators in shared memory — was bound by shared-memory traffic and the
// per-tile hand-offs, not by DRAM: 0.84 GB in 0.35 ms at C3; per 32-pixel tile the tensor core read 44 KB of
// fp32 operands, the splitters moved 43 KB and the fp64 flush 29 KB.)  Here a tile is 64 pixels of one component ([KPN frames x 64] fp32 TMA box, 256-byte rows); the
// splitters write n = hi + lo as two f16 halves (hi = f16(n), lo = f16(n - hi): the pair carries n to 2^-22
// relative or 3e-8 absolute, the f16 subnormal spacing, as in k_ngf_z_tc) into one [H (KPN rows); L (KPN rows)]
// SWIZZLE_128B K-major buffer (64 f16 = one 128-byte row); one M128 N(2 KPN) K16 MMA per 16 pixels gives
// [H H^T | H L^T] in fp32 TMEM; the flush adds 0.5 HH + HL in fp64 every R tiles, G = A + A^T at the end.  Half the operand bytes and a quarter of
// the MMA instructions per pixel, half the hand-offs.  max |n| per frame as before (degenerate rule).
__host__ __device__ constexpr uint32_t umma_idesc_h16(int M, int N) {  // kind::f16, f16 A/B, fp32 D, K-major
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
static __device__ __forceinline__ void umma_h16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
struct TGH {
  // 16 splitter warps, 1 MMA issuer warp, 4 flusher warps (one per TMEM lane quarter), 1 TMA producer warp
  static constexpr int NSP = 512, NT = NSP + 32 + 128 + 32;
  static constexpr int NB = 3, NA = 2, RPX = 2048, TS = 256, MAXST = 8;  // RPX pixels per TMEM slot and flush
};
// A tile is natom K-atoms of 64 pixels (tp = 64 natom pixels of one component): 1 atom for more than 64
// frames, 2 for 33..64, 4 for up to 32, so that a tile is 16-32 KB whatever the subset size (the per-tile
// hand-offs, not the bytes, bound the kernel).  Operand buffer: [atom][H (rows); L (rows)][128 B].
struct GhLayout {
  int rows, natom, tp, sbytes, obytes, nst;
};
inline GhLayout tgh_layout(int K, size_t smem_cap) {
  GhLayout L{};
  L.rows = (K + 15) / 16 * 16;
  L.natom = L.rows <= 32 ? 4 : L.rows <= 64 ? 2 : 1;
  L.tp = 64 * L.natom;
  L.sbytes = L.rows * L.tp * 4;
  L.obytes = L.natom * 2 * L.rows * 128;
  const size_t fixed = 1024 + (size_t)TGH::NB * L.obytes + 512;
  const int nst = smem_cap > fixed ? (int)((smem_cap - fixed) / L.sbytes) : 0;
  L.nst = nst > TGH::MAXST ? TGH::MAXST : nst;
  return L;
}
inline size_t tgh_smem(const GhLayout& L) {
  return 1024 + (size_t)L.nst * L.sbytes + (size_t)TGH::NB * L.obytes + 512;
}

// The fp64 accumulators live in the CTA's own partial block in global memory (L2-resident: 131 KB per CTA),
// transposed (entry (row m, column c) at c * KP + m, so the lane-per-row flush is coalesced); each entry is
// only ever touched by one thread.  The shared memory they took in k_gram_tcx buys TMA stages instead (6 of
// 28 KB at K = 100: with 2, the bytes in flight per SM bounded the kernel at 2.9 TB/s).
template <int KP>  // KP = 64 or 128: the partial block layout [KP x KP | s | vmax | -vmin] of the K bucket
__global__ void __launch_bounds__(TGH::NT, 1) k_gram_h(const Args a, const __grid_constant__ CUtensorMap xmap,
                                                       int ntx, int ncomp, const GhLayout lay) {
  using C = TGH;
  constexpr int NB = C::NB, NA = C::NA;
  constexpr int NATOM = KP > 64 ? 1 : KP > 32 ? 2 : 4, TP = 64 * NATOM, R = C::RPX / TP;  // = lay.natom, lay.tp
  const int NST = lay.nst;
  const uint32_t ATOMB = (uint32_t)(2 * lay.rows * 128);  // bytes of one K-atom of the [H; L] operand
  extern __shared__ __align__(1024) unsigned char smem_gh[];
  unsigned char* base = smem_gh + ((1024 - (smem_u32(smem_gh) & 1023)) & 1023);
  unsigned char* Vb = base;                                                      // [NB][2 rows][128 B] SW128
  float* stage = reinterpret_cast<float*>(base + (size_t)NB * lay.obytes);       // [NST][rows][TP] fp32
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)NB * lay.obytes + (size_t)NST * lay.sbytes);
  uint64_t* st_full = bars;
  uint64_t* st_free = st_full + C::MAXST;
  uint64_t* vb_full = st_free + C::MAXST;
  uint64_t* vb_free = vb_full + NB;
  uint64_t* acc_full = vb_free + NB;
  uint64_t* acc_free = acc_full + NA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + NA);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.K, KPN = lay.rows;
  const long long ntiles = (long long)ntx * ncomp;
  const long long nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  // tile n of this CTA = global tile blockIdx.x + n gridDim.x = (column tile tx, component ty), advanced
  // incrementally (no 64-bit division on the single-thread paths)
  int ptx = (int)(blockIdx.x % (unsigned)ntx), pty = (int)(blockIdx.x / (unsigned)ntx);
  const int dtx = (int)(gridDim.x % (unsigned)ntx), dty = (int)(gridDim.x / (unsigned)ntx);
  auto load_next = [&](int st) {
    mbar_arrive_expect_tx(&st_full[st], (uint32_t)lay.sbytes);
    tma_load_3d(stage + (size_t)st * KPN * TP, &xmap, ptx * TP, pty, 0, &st_full[st]);
    ptx += dtx;
    pty += dty;
    if (ptx >= ntx) ptx -= ntx, ++pty;
  };
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_free[s], C::NSP / 32);  // one arrival per splitter warp
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&vb_full[b], C::NSP / 32);
      mbar_init(&vb_free[b], 1);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_free[s], 128);
    }
    fence_mbar_init();
    tma_prefetch_desc(&xmap);
  }
  double* out = a.part + (size_t)blockIdx.x * (KP * KP + 3 * KP);
  for (int e = tid; e < KP * KP; e += C::NT) __stcg(out + e, 0.0);
  if (warp == C::NSP / 32) tmem_alloc(tmem_slot, C::TS * NA);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (tid < C::NSP) {
    // ======================= splitters: a warp takes two stage rows (2 x 256 B) per step, lane = (row of the
    // pair, 16-byte chunk of 4 columns): conflict-free 128-bit reads; 4 steps cover rows 2 (warp + 16 it) + hl.
    // The 4 f16 hi (and lo) of a lane are half a 16-byte operand chunk: 64-bit stores, a half-warp fills one
    // swizzled 128-byte operand row.
    const int hl = lane >> 4, cl = lane & 15;
    const int r0 = 2 * warp + hl;
    // 4 steps per tile: step e = (row block e & (nrb - 1): rows r0 + 32 rbk, atom e >> log2(nrb)), nrb = 4 / NATOM
    constexpr int nrb = 4 / NATOM, lrb = nrb == 4 ? 2 : nrb == 2 ? 1 : 0;
    const uint32_t ooff = (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + ((((cl >> 1) ^ r0) & 7) << 4) + (cl & 1) * 8);
    const uint32_t lrow = (uint32_t)KPN * 128;  // L rows: KPN % 8 == 0
    float fm[4] = {0.f, 0.f, 0.f, 0.f};
    int st = 0;
    uint32_t stph = 0;
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n % NB);
      mbar_wait(&st_full[st], stph);
      const unsigned char* src = reinterpret_cast<const unsigned char*>(stage) + (size_t)st * lay.sbytes;
      uint2 hw[4], lw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int rbk = e & (nrb - 1), at = e >> lrb, row = r0 + 32 * rbk;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < KPN) q = *reinterpret_cast<const float4*>(src + (size_t)(row * TP + at * 64 + 4 * cl) * 4);
        fm[e] = fmaxf(fm[e], fmaxf(fmaxf(fabsf(q.x), fabsf(q.y)), fmaxf(fabsf(q.z), fabsf(q.w))));
        const __half2 h0 = __floats2half2_rn(q.x, q.y), h1 = __floats2half2_rn(q.z, q.w);
        const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
        const __half2 l0 = __floats2half2_rn(q.x - f0.x, q.y - f0.y), l1 = __floats2half2_rn(q.z - f1.x, q.w - f1.y);
        hw[e] = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
        lw[e] = make_uint2(*reinterpret_cast<const uint32_t*>(&l0), *reinterpret_cast<const uint32_t*>(&l1));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&st_free[st]);  // the stage is in registers: the producer may refill it
      if (n >= NB) mbar_wait(&vb_free[b], (uint32_t)((n / NB - 1) & 1));
      unsigned char* ob = Vb + (size_t)b * lay.obytes;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int rbk = e & (nrb - 1), at = e >> lrb;
        if (r0 + 32 * rbk < KPN) {
          unsigned char* dst = ob + (uint32_t)at * ATOMB + ooff + (uint32_t)rbk * 4096;
          *reinterpret_cast<uint2*>(dst) = hw[e];
          *reinterpret_cast<uint2*>(dst + lrow) = lw[e];
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&vb_full[b]);
      if (++st == NST) st = 0, stph ^= 1;
    }
    // max |n| per row: the steps of a row block (one per atom) share the row
    if (nrb == 2) fm[0] = fmaxf(fm[0], fm[2]), fm[1] = fmaxf(fm[1], fm[3]);
    if (nrb == 1) fm[0] = fmaxf(fmaxf(fm[0], fm[1]), fmaxf(fm[2], fm[3]));
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      float v = fm[it];
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      const int r = r0 + 32 * it;
      if (cl == 0 && r < KP && it < nrb) {
        out[KP * KP + r] = 0.0;  // s: unused by NGF
        out[KP * KP + KP + r] = r < K ? (double)v : 0.0;
        out[KP * KP + 2 * KP + r] = r < K ? (double)v : 0.0;
      }
    }
  } else if (warp == C::NSP / 32) {
    // ======================= issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_h16(128, 2 * KPN);
      for (long long n = 0; n < nloc; ++n) {
        const long long grp = n / R;
        const bool first = n % R == 0, last = n % R == R - 1 || n == nloc - 1;
        const int b = (int)(n % NB), s = (int)(grp % NA);
        mbar_wait(&vb_full[b], (uint32_t)((n / NB) & 1));
        if (first && grp >= NA) mbar_wait(&acc_free[s], (uint32_t)((grp / NA - 1) & 1));
        tc_fence_after();
        const uint32_t o0 = smem_u32(Vb + (size_t)b * lay.obytes);
        const uint32_t acc = tmem + (uint32_t)(s * C::TS);
        for (int at = 0; at < NATOM; ++at)
#pragma unroll
          for (int k16 = 0; k16 < 4; ++k16) {
            const uint64_t dh = umma_sdesc_sw128(o0 + (uint32_t)at * ATOMB + (uint32_t)(k16 * 32));
            umma_h16(acc, dh, dh, idesc, (at > 0 || k16 > 0 || !first) ? 1u : 0u);  // A = H (128 rows), B = [H; L]
          }
        umma_commit(&vb_free[b]);
        if (last) umma_commit(&acc_full[s]);
      }
    }
    __syncwarp();
  } else if (warp == C::NT / 32 - 1) {
    // ======================= TMA producer: stage of tile n is refilled (tile n + NST) once the splitters have
    // it in registers (st_free)
    if (lane == 0) {
      for (long long n = 0; n < nloc && n < NST; ++n) load_next((int)n);
      int st = 0;
      uint32_t ph = 0;
      for (long long n = 0; n + NST < nloc; ++n) {
        mbar_wait(&st_free[st], ph);
        load_next(st);
        if (++st == NST) st = 0, ph ^= 1;
      }
    }
    __syncwarp();
  } else {
    // ======================= flushers: TMEM lane quarter q = warp % 4, row m = 32 q + lane; entry (m, c) of
    // A = 0.5 HH + HL accumulates at out[c * KP + m]
    const int q = warp & 3, m = 32 * q + lane;
    const bool mok = m < KPN;  // TMEM lanes past KPN carry garbage rows (not accumulated)
    double* acol = out + (mok ? m : 0);
    const long long ngrp = (nloc + R - 1) / R;
    for (long long n = 0; n < ngrp; ++n) {
      const int s = (int)(n % NA);
      mbar_wait(&acc_full[s], (uint32_t)((n / NA) & 1));
      tc_fence_after();
      const uint32_t ts = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(s * C::TS);
#pragma unroll 1
      for (int c0 = 0; c0 < KPN; c0 += 16) {
        float hh[16], hl[16];
        double old[16];
        if (mok) {
#pragma unroll
          for (int cc = 0; cc < 16; ++cc) old[cc] = __ldcg(acol + (size_t)(c0 + cc) * KP);
        }
        tmem_ld16(ts + (uint32_t)c0, hh);
        tmem_ld16(ts + (uint32_t)(KPN + c0), hl);
        if (mok) {
#pragma unroll
          for (int cc = 0; cc < 16; ++cc)
            __stcg(acol + (size_t)(c0 + cc) * KP, old[cc] + (0.5 * (double)hh[cc] + (double)hl[cc]));
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_free[s]);
    }
  }
  tc_fence_before();
  __syncthreads();
  {
    // G = A + A^T in place (out holds A^T; the pair (i, j), (j, i) belongs to one thread), every thread of
    // the CTA, 4 pairs per batch so that the L2 round trips overlap
    for (int e0 = tid; e0 < KP * KP; e0 += 4 * C::NT) {
      double x[4], y[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * C::NT, i = e / KP, j = e % KP;
        ok[u] = e < KP * KP && j >= i;
        x[u] = y[u] = 0.0;
        if (ok[u]) {
          x[u] = __ldcg(out + (size_t)j * KP + i);
          y[u] = __ldcg(out + (size_t)i * KP + j);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * C::NT, i = e / KP, j = e % KP;
        if (ok[u]) {
          const double g = (i < KPN && j < KPN) ? x[u] + y[u] : 0.0;
          __stcg(out + (size_t)i * KP + j, g);
          __stcg(out + (size_t)j * KP + i, g);
        }
      }
    }
  }
  if (warp == C::NSP / 32) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TS * NA);
  }
}

// ------------------------------------------------------------------------------------------
// 2-D sampling fused with the NGF feature (replaces k_sample_vp<LO> + k_ngf_feat4 and the u round trip):
// CTA = (row segment, subset frame k), thread = 4 consecutive columns of every row (a whole image row per
// CTA, so the x stencil needs no halo: neighbours come from the thread itself, its warp (shuffles) and the
// next/previous warp (shared memory)).  Rows are walked in order with u of rows r - 1, r, r + 1 in
// registers (fp64 values of the bilinear interpolant, grid.py:199-233) while the corner gathers of row
// r + 2 and the y loads of row r + 3 are in flight, so a row's memory latency overlaps two rows of work.
// At row r the thread writes n = grad_h u / rho and 1/rho (z rows [rz0, rz1)); grad T is written when
// its row is sampled (slab rows [rs0, rs1)).  Same stencil as ngf_at (central differences inside,
// one-sided at the domain edge, world units); the differences of u are taken in fp64 and rounded once.
struct Corners2 {
  float v00, v10, v01, v11, f0, f1;
  bool inside;
};
template <bool POW2>
__device__ __forceinline__ Corners2 fetch2(const float* __restrict__ img, const Geo& g, float px, float py) {
  Corners2 c;
  int base;
  interp2_prep<float, POW2>(g, px, py, base, c.f0, c.f1, c.inside);
  const float* q = img + base;
  const int s1 = g.sti[1];
  c.v00 = __ldg(q);
  c.v10 = __ldg(q + 1);
  c.v01 = __ldg(q + s1);
  c.v11 = __ldg(q + s1 + 1);
  return c;
}
// fp64 value and fp32 gradient (the arithmetic of interp_v64<2>)
__device__ __forceinline__ double finish2(const Corners2& c, const Geo& g, bool pow2, float (&gr)[2]) {
  const float d0 = c.v10 - c.v00, d1 = c.v11 - c.v01;
  const float a0f = fmaf(c.f0, d0, c.v00), a1f = fmaf(c.f0, d1, c.v01);
  const float gv0 = fmaf(c.f1, d1 - d0, d0), gv1 = a1f - a0f;
  gr[0] = c.inside ? (pow2 ? gv0 * g.invf[0] : gv0 / g.sf[0]) : 0.f;
  gr[1] = c.inside ? (pow2 ? gv1 * g.invf[1] : gv1 / g.sf[1]) : 0.f;
  const double a0 = fma((double)c.f0, (double)c.v10 - (double)c.v00, (double)c.v00);
  const double a1 = fma((double)c.f0, (double)c.v11 - (double)c.v01, (double)c.v01);
  return c.inside ? fma((double)c.f1, a1 - a0, a0) : 0.0;
}

// PX consecutive columns per thread (2: 512 threads for a 1024-pixel row, 32 warps per SM at <= 64
// registers; 4 held 128 registers and 16 warps)
template <int PX>
struct VecF;
template <>
struct VecF<2> {
  using T = float2;
  static __device__ __forceinline__ void ld(const float* p, float (&v)[2]) {
    const float2 a = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = a.x, v[1] = a.y;
  }
  static __device__ __forceinline__ void st(float* p, const float (&v)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
};
template <>
struct VecF<4> {
  static __device__ __forceinline__ void ld(const float* p, float (&v)[4]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
  }
  static __device__ __forceinline__ void st(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

template <bool POW2, int PX>
__global__ void __launch_bounds__(1024 / (4 / PX) <= 512 ? 512 : 256, 2) k_ngf_sfeat2(
    const Args a, int seg, int rz0, int rz1, int rs0, int rs1, float* __restrict__ Nf, float* __restrict__ IRho,
    long long zlo, long long zstride, float* __restrict__ Gv, long long vlo, long long vstride) {
  __shared__ double edge[2][2][32];  // [row parity][left / right edge][warp]
  const int k = blockIdx.y;
  const int n0 = a.g.n[0], n1 = a.g.n[1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int x0 = PX * tid;
  const bool colok = x0 < n0;
  const int ra = rz0 + blockIdx.x * seg, rb = min(ra + seg, rz1);
  if (ra >= rb) return;
  const int fi = a.job->frame_index[k];
  const float* img = reinterpret_cast<const float*>(a.frames) + (long long)fi * a.g.N;
  const float* y0p = reinterpret_cast<const float*>(a.y) + (long long)(2 * k) * a.y_stride - a.y_off;
  const float* y1p = y0p + a.y_stride;
  const bool vec = (n0 % PX) == 0 && ((a.y_stride | a.y_off) % PX) == 0 &&
                   (reinterpret_cast<uintptr_t>(a.y) & (4 * PX - 1)) == 0 && x0 + PX <= n0;
  const bool vz = vec && (zlo % PX) == 0 && (zstride % PX) == 0, vg = vec && (vlo % PX) == 0 && (vstride % PX) == 0;
  const double h0 = 0.5 * a.g.inv[0], f0 = a.g.inv[0], h1 = 0.5 * a.g.inv[1], f1 = a.g.inv[1];
  const float e = (float)a.eps, e2 = e * e;
  float* gk0 = Gv + (long long)(2 * k) * vstride - vlo;
  float* gk1 = gk0 + vstride;
  auto load_y = [&](int r, float (&py)[PX][2]) {
    const long long pr = (long long)r * n0 + x0;
    if (colok && vec) {
      float a0[PX], a1[PX];
      VecF<PX>::ld(y0p + pr, a0);
      VecF<PX>::ld(y1p + pr, a1);
#pragma unroll
      for (int t = 0; t < PX; ++t) py[t][0] = a0[t], py[t][1] = a1[t];
    } else {
#pragma unroll
      for (int t = 0; t < PX; ++t) {
        const bool ok = colok && x0 + t < n0;
        py[t][0] = ok ? __ldg(y0p + pr + t) : 0.f;
        py[t][1] = ok ? __ldg(y1p + pr + t) : 0.f;
      }
    }
  };
  auto fetch_row = [&](const float (&py)[PX][2], Corners2 (&cr)[PX]) {
#pragma unroll
    for (int t = 0; t < PX; ++t) cr[t] = fetch2<POW2>(img, a.g, py[t][0], py[t][1]);
  };
  // u of row r from its corners; grad T written when r is a slab row of this segment
  auto finish_row = [&](int r, const Corners2 (&cr)[PX], double (&u)[PX]) {
    float gt0[PX], gt1[PX];
#pragma unroll
    for (int t = 0; t < PX; ++t) {
      float gt[2];
      u[t] = finish2(cr[t], a.g, POW2, gt);
      gt0[t] = gt[0], gt1[t] = gt[1];
    }
    if (colok && r >= ra && r < rb && r >= rs0 && r < rs1) {
      const long long q = (long long)r * n0 + x0;
      if (vg) {
        VecF<PX>::st(gk0 + q, gt0);
        VecF<PX>::st(gk1 + q, gt1);
      } else {
#pragma unroll
        for (int t = 0; t < PX; ++t)
          if (x0 + t < n0) {
            gk0[q + t] = gt0[t];
            gk1[q + t] = gt1[t];
          }
      }
    }
  };
  // prologue: u of rows ra - 1, ra, ra + 1 in registers; corners of ra + 2 landing, y of ra + 3 in flight.
  // In iteration r the corners of row r + 3 and the y of row r + 4 are issued, row r + 2's corners (issued
  // one iteration earlier) are finished at its end: every load has a whole row of work to land.
  double um[PX], uc[PX], up[PX];
#pragma unroll
  for (int t = 0; t < PX; ++t) um[t] = up[t] = 0.0;
  float yv[PX][2];
  Corners2 cr[PX], cn[PX];
  if (ra > 0) {
    load_y(ra - 1, yv);
    fetch_row(yv, cr);
    finish_row(ra - 1, cr, um);
  }
  load_y(ra, yv);
  fetch_row(yv, cr);
  finish_row(ra, cr, uc);
  if (ra + 1 < n1) {
    load_y(ra + 1, yv);
    fetch_row(yv, cr);
    finish_row(ra + 1, cr, up);
  }
  const int rlast = min(rb, n1 - 1);  // last row ever sampled by this segment
  if (ra + 2 <= rlast) {
    load_y(ra + 2, yv);
    fetch_row(yv, cr);
  }
  if (ra + 3 <= rlast) load_y(ra + 3, yv);
  for (int r = ra; r < rb; ++r) {
    const int par = r & 1;
    const bool more = r + 2 <= rlast;
    if (r + 3 <= rlast) fetch_row(yv, cn);        // corners of row r + 3 (finished next iteration)
    if (r + 4 <= rlast) load_y(r + 4, yv);        // y of row r + 4
    if (lane == 0) edge[par][1][warp] = uc[0];
    if (lane == 31) edge[par][0][warp] = uc[PX - 1];
    __syncthreads();
    double left = __shfl_up_sync(0xffffffffu, uc[PX - 1], 1), right = __shfl_down_sync(0xffffffffu, uc[0], 1);
    if (lane == 0) left = warp > 0 ? edge[par][0][warp - 1] : uc[0];
    if (lane == 31) right = warp + 1 < nw ? edge[par][1][warp + 1] : uc[PX - 1];
    const bool c1 = r > 0 && r + 1 < n1;
    float nv0[PX], nv1[PX], irv[PX];
#pragma unroll
    for (int t = 0; t < PX; ++t) {
      const int x = x0 + t;
      const double ul = t == 0 ? left : uc[t - 1], ur = t == PX - 1 ? right : uc[t + 1];
      const bool hm = x > 0, hp = x < n0 - 1;
      const double dxl = hm ? ul : uc[t], dxr = hp ? ur : uc[t];
      const double dyl = r > 0 ? um[t] : uc[t], dyr = r + 1 < n1 ? up[t] : uc[t];
      const float g0 = (float)((dxr - dxl) * ((hm && hp) ? h0 : f0));
      const float g1 = (float)((dyr - dyl) * (c1 ? h1 : f1));
      const float rho = sqrtf(g0 * g0 + g1 * g1 + e2);
      const float ir = 1.f / rho;
      nv0[t] = g0 * ir;
      nv1[t] = g1 * ir;
      irv[t] = ir;
    }
    if (colok) {
      const long long q = (long long)r * n0 + x0;
      float* n0p = Nf + (long long)(2 * k) * zstride + (q - zlo);
      float* n1p = n0p + zstride;
      float* irp = IRho + (long long)k * zstride + (q - zlo);
      if (vz) {
        VecF<PX>::st(n0p, nv0);
        VecF<PX>::st(n1p, nv1);
        VecF<PX>::st(irp, irv);
      } else {
#pragma unroll
        for (int t = 0; t < PX; ++t)
          if (x0 + t < n0) {
            n0p[t] = nv0[t];
            n1p[t] = nv1[t];
            irp[t] = irv[t];
          }
      }
    }
    double un[PX];
    if (more) finish_row(r + 2, cr, un);
#pragma unroll
    for (int t = 0; t < PX; ++t) {
      um[t] = uc[t];
      uc[t] = up[t];
      up[t] = more ? un[t] : up[t];
      cr[t] = cn[t];
    }
  }
}
// ---- k_ngf_sfeat2f: the same rows -> (n, 1/rho, grad T) walk as k_ngf_sfeat2 for the aligned common case
// (power-of-two spacings, even n0 and strides / offsets: ngf_sfeat_d2 checks), written for instruction
// count and latency hiding (k_ngf_sfeat2 issued ~227 instructions per voxel-frame and was issue-bound; a
// first rewrite with the same CTA-per-row shape issued 90 and was bound by the per-row barrier and the
// gather latency behind it).  Work unit = one WARP: (frame, segment of rows, chunk of 62 columns).  The
// warp samples 64 columns (its chunk + one halo column each side, clamped into the image, which is
// exactly u(-1) := u(0), u(n0) := u(n0 - 1)), lane i the columns s + 2 i and s + 2 i + 1, so the x stencil
// needs only warp shuffles: no shared memory, no barrier, warps drift freely.  Lane i < 31 stores the
// aligned pair (its second column, lane i + 1's first column).  The u rows rotate through a 3x unrolled
// loop instead of register moves; row ends are handled by a per-row factor; the power-of-two stencil
// factors are applied after the rounding to fp32 (identical bits); 1/rho = rsqrt.approx(|p|^2 + eps^2)
// (2^-22 relative) instead of the IEEE sqrt + division.  Per row: stencil of row r, finish row r + 2
// from the corners fetched one row earlier, fetch the corners of row r + 3, load the y of row r + 4.
static __device__ __forceinline__ float rsqrt_fast(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
struct CornersF {
  float v00, v10, v01, v11, f0, f1;
  bool inside;
};
// iv0, iv1: 1 / spacing when POW2 (exact; t = (p - o) (1/s) - 0.5 in one FMA), else the spacing itself
// (t = (p - o) / s - 0.5 with the true division of grid.py:199-233, as interp2_prep)
template <int PF, bool POW2>
__device__ __forceinline__ CornersF fetch2f(const float* __restrict__ img, float of0, float of1, float iv0, float iv1,
                                            float hi0, float hi1, int m0, int m1, int s1, float px, float py) {
  CornersF c;
  const float q0 = __fsub_rn(px, of0), q1 = __fsub_rn(py, of1);
  const float t0 = POW2 ? fmaf(q0, iv0, -0.5f) : __fsub_rn(__fdiv_rn(q0, iv0), 0.5f);
  const float t1 = POW2 ? fmaf(q1, iv1, -0.5f) : __fsub_rn(__fdiv_rn(q1, iv1), 0.5f);
  const float c0 = fminf(fmaxf(t0, 0.f), hi0), c1 = fminf(fmaxf(t1, 0.f), hi1);
  c.inside = (c0 == t0) && (c1 == t1);
  const int i0 = min(__float2int_rz(c0), m0), i1 = min(__float2int_rz(c1), m1);  // c >= 0: trunc = floor
  c.f0 = c0 - (float)i0;
  c.f1 = c1 - (float)i1;
  const float* q = img + (i0 + i1 * s1);
  c.v00 = __ldg(q);
  c.v10 = __ldg(q + 1);
  c.v01 = __ldg(q + s1);
  c.v11 = __ldg(q + s1 + 1);
  if (PF > 0)  // the image rows the next rows of a smooth field will gather from: into L2 ahead of time
    asm volatile("prefetch.global.L2 [%0];" ::"l"(q + min(PF, m1 + 1 - i1) * s1));
  return c;
}
template <bool POW2>
__device__ __forceinline__ double finish2f(const CornersF& c, float iv0, float iv1, float& g0, float& g1) {
  const float d0 = c.v10 - c.v00, d1 = c.v11 - c.v01;
  const float a0f = fmaf(c.f0, d0, c.v00), a1f = fmaf(c.f0, d1, c.v01);
  const float gv0 = fmaf(c.f1, d1 - d0, d0), gv1 = a1f - a0f;
  g0 = c.inside ? (POW2 ? gv0 * iv0 : __fdiv_rn(gv0, iv0)) : 0.f;
  g1 = c.inside ? (POW2 ? gv1 * iv1 : __fdiv_rn(gv1, iv1)) : 0.f;
  const double a0 = fma((double)c.f0, (double)c.v10 - (double)c.v00, (double)c.v00);
  const double a1 = fma((double)c.f0, (double)c.v11 - (double)c.v01, (double)c.v01);
  return c.inside ? fma((double)c.f1, a1 - a0, a0) : 0.0;
}

template <int MINB, bool POW2>
__global__ void __launch_bounds__(32, MINB) k_ngf_sfeat2f(
    const Args a, int seg, int rz0, int rz1, int rs0, int rs1, float* __restrict__ Nf,
    float* __restrict__ IRho, long long zlo, long long zstride, float* __restrict__ Gv, long long vlo,
    long long vstride) {
  constexpr int CW = 62;  // output columns per warp
  // one warp per CTA (32 CTAs per SM): everything but the column is CTA-uniform (uniform registers)
  const int k = blockIdx.z;
  const int n0 = a.g.n[0], n1 = a.g.n[1];
  const int lane = threadIdx.x;
  const int ch = blockIdx.x;
  const int ra = rz0 + blockIdx.y * seg, rb = min(ra + seg, rz1);
  if (ra >= rb) return;
  const int xa = ch * CW - 1 + 2 * lane;                    // first sampled column (may be -1 or >= n0)
  const int xs0 = min(max(xa, 0), n0 - 1), xs1 = min(xa + 1, n0 - 1);  // clamped sampling columns
  const int xe = xa + 1;                                    // first column of the stored pair (even)
  const bool st_ok = lane < 31 && xe < n0;
  // Per-frame bases kept in registers (opaque to the compiler, which otherwise rebuilds every address from
  // the kernel parameters with 64-bit arithmetic): one IMAD.WIDE per access with a 32-bit index.  The
  // second components sit one (32-bit, checked by the launcher) stride further.
  const float* img = reinterpret_cast<const float*>(a.frames) + (long long)a.job->frame_index[k] * a.g.N;
  const float* y0b = reinterpret_cast<const float*>(a.y) + ((long long)(2 * k) * a.y_stride - a.y_off + xs0);
  float* g0b = Gv + ((long long)(2 * k) * vstride - vlo + xe);
  float* n0b = Nf + ((long long)(2 * k) * zstride - zlo + xe);
  float* irb_ = IRho + ((long long)k * zstride - zlo + xe);
  asm volatile("" : "+l"(img), "+l"(y0b), "+l"(g0b), "+l"(n0b), "+l"(irb_));
  const unsigned ys = (unsigned)a.y_stride, vs = (unsigned)vstride, zs = (unsigned)zstride;
  const unsigned dx1 = (unsigned)(xs1 - xs0);  // 0 on a clamped column, else 1
  const float of0 = a.g.of[0], of1 = a.g.of[1];
  const float iv0 = POW2 ? a.g.invf[0] : a.g.sf[0], iv1 = POW2 ? a.g.invf[1] : a.g.sf[1];  // see fetch2f
  const float hi0 = (float)(n0 - 1), hi1 = (float)(n1 - 1);
  const int m0 = n0 - 2, m1 = n1 - 2, s1 = a.g.sti[1];
  const float e = (float)a.eps, e2 = e * e;
  // stencil factors: central 1/(2 s) inside, one-sided 1/s on the first / last column and row.  POW2: applied
  // in fp32 after the rounding of the fp64 difference (a power of two commutes with the rounding); else in
  // fp64 before it, as k_ngf_sfeat2 / ngf_at do.
  const bool ina = xa > 0 && xa < n0 - 1, inb = xa + 1 > 0 && xa + 1 < n0 - 1;
  const float fxa = ina ? 0.5f * a.g.invf[0] : a.g.invf[0], fxb = inb ? 0.5f * a.g.invf[0] : a.g.invf[0];
  const double dxa = ina ? 0.5 * a.g.inv[0] : a.g.inv[0], dxb = inb ? 0.5 * a.g.inv[0] : a.g.inv[0];
  const int glo = max(ra, rs0), ghi = min(rb, rs1);  // rows whose grad T this segment writes
  const int rlast = min(rb, n1 - 1);                 // last row this segment samples

  float ya0, ya1, yb0, yb1;  // y of one row at the two sampled columns: (y0, y1)
  CornersF ca, cb;
  auto load_y = [&](unsigned q) {  // q = r * n0
    ya0 = __ldg(y0b + q);
    ya1 = __ldg(y0b + (q + ys));
    yb0 = __ldg(y0b + (q + dx1));
    yb1 = __ldg(y0b + (q + dx1 + ys));
  };
  // y streams from DRAM (the T gathers mostly hit L1 / L2): rows PD ahead are pulled into L2 so that the
  // register prefetch (one row of slack) only has to cover the L2 latency
  constexpr int PD = 10, PT = 0;
  auto prefetch_y = [&](unsigned q) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(y0b + q));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(y0b + (q + ys)));
  };
  auto fetch = [&]() {
    ca = fetch2f<PT, POW2>(img, of0, of1, iv0, iv1, hi0, hi1, m0, m1, s1, ya0, ya1);
    cb = fetch2f<0, POW2>(img, of0, of1, iv0, iv1, hi0, hi1, m0, m1, s1, yb0, yb1);
  };
  auto finish = [&](int r, unsigned q, double (&u)[2]) {
    float g0a, g1a, g0c, g1c;
    u[0] = finish2f<POW2>(ca, iv0, iv1, g0a, g1a);
    u[1] = finish2f<POW2>(cb, iv0, iv1, g0c, g1c);
    if (r >= glo && r < ghi) {  // warp-uniform
      const float g0n = __shfl_down_sync(0xffffffffu, g0a, 1), g1n = __shfl_down_sync(0xffffffffu, g1a, 1);
      if (st_ok) {
        *reinterpret_cast<float2*>(g0b + q) = make_float2(g0c, g0n);
        *reinterpret_cast<float2*>(g0b + (q + vs)) = make_float2(g1c, g1n);
      }
    }
  };
  // one row; TAIL = the rows r + 2 .. r + 4 may lie past the last sampled row.  q = r * n0.
  auto step = [&](auto tailc, int r, unsigned q, double (&um)[2], const double (&uc)[2], const double (&up)[2]) {
    constexpr bool TAIL = decltype(tailc)::value;
    const double left = __shfl_up_sync(0xffffffffu, uc[1], 1), right = __shfl_down_sync(0xffffffffu, uc[0], 1);
    const bool iny = r > 0 && r + 1 < n1;
    double uq0 = up[0], uq1 = up[1];
    if (TAIL && r + 1 >= n1) uq0 = uc[0], uq1 = uc[1];  // u(n1) := u(n1 - 1)
    float gxa, gxb, gya, gyb;
    if (POW2) {
      const float fy = iny ? 0.5f * a.g.invf[1] : a.g.invf[1];
      gxa = (float)(uc[1] - left) * fxa, gxb = (float)(right - uc[0]) * fxb;
      gya = (float)(uq0 - um[0]) * fy, gyb = (float)(uq1 - um[1]) * fy;
    } else {
      const double dy = iny ? 0.5 * a.g.inv[1] : a.g.inv[1];
      gxa = (float)((uc[1] - left) * dxa), gxb = (float)((right - uc[0]) * dxb);
      gya = (float)((uq0 - um[0]) * dy), gyb = (float)((uq1 - um[1]) * dy);
    }
    const float ira = rsqrt_fast(fmaf(gxa, gxa, fmaf(gya, gya, e2)));
    const float irb = rsqrt_fast(fmaf(gxb, gxb, fmaf(gyb, gyb, e2)));
    const float nxa = gxa * ira, nya = gya * ira;
    const float nxn = __shfl_down_sync(0xffffffffu, nxa, 1), nyn = __shfl_down_sync(0xffffffffu, nya, 1);
    const float irn = __shfl_down_sync(0xffffffffu, ira, 1);
    if (st_ok) {
      *reinterpret_cast<float2*>(n0b + q) = make_float2(gxb * irb, nxn);
      *reinterpret_cast<float2*>(n0b + (q + zs)) = make_float2(gyb * irb, nyn);
      *reinterpret_cast<float2*>(irb_ + q) = make_float2(irb, irn);
    }
    if (!TAIL || r + 2 <= rlast) finish(r + 2, q + 2 * n0, um);  // um is dead: it becomes the next "up"
    if (!TAIL || r + 3 <= rlast) fetch();
    if (!TAIL || r + 4 <= rlast) load_y(q + 4 * n0);
    if (!TAIL) prefetch_y(q + (unsigned)(min(r + PD, rlast) - r) * n0);
  };

  double u0[2], u1[2], u2[2];
  unsigned q = (unsigned)(ra * n0);
#pragma unroll
  for (int i = -1; i < PD; ++i)
    if (ra + i >= 0 && ra + i <= rlast) prefetch_y(q + (unsigned)(i * n0));
  load_y(q);
  fetch();
  finish(ra, q, u1);
  if (ra > 0) {
    load_y(q - n0);
    fetch();
    finish(ra - 1, q - n0, u0);
  } else {
    u0[0] = u1[0], u0[1] = u1[1];  // u(row -1) := u(row 0)
  }
  u2[0] = u2[1] = 0.0;
  if (ra + 1 < n1) {
    load_y(q + n0);
    fetch();
    finish(ra + 1, q + n0, u2);
  }
  if (ra + 2 <= rlast) {
    load_y(q + 2 * n0);
    fetch();
  }
  if (ra + 3 <= rlast) load_y(q + 3 * n0);
  int r = ra;
  for (; r + 6 <= rlast; r += 3, q += 3 * n0) {  // rows r .. r + 2 with every look-ahead row present
    step(std::false_type{}, r, q, u0, u1, u2);
    step(std::false_type{}, r + 1, q + n0, u1, u2, u0);
    step(std::false_type{}, r + 2, q + 2 * n0, u2, u0, u1);
  }
  while (r < rb) {
    step(std::true_type{}, r, q, u0, u1, u2);
    if (++r >= rb) break;
    q += n0;
    step(std::true_type{}, r, q, u1, u2, u0);
    if (++r >= rb) break;
    q += n0;
    step(std::true_type{}, r, q, u2, u0, u1);
    ++r;
    q += n0;
  }
}
}  // namespace sr

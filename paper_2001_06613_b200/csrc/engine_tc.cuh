// engine_tc.cuh — the sampling kernel of the split paths and the streaming pass 2:
//
//   k_sample_vp     every subset frame sampled at its y over 1024-pixel blocks (grid.py:199-253): writes
//                   V = v - shift (NCC) or u (NGF, as an fp32 pair: fp64 arithmetic, k_sample_vp<LO>) and
//                   grad T for pass 2; the y of the next block is loaded before this block's gathers.
//   k_pass2_stream  q_j = beta'_j + sum_i M'_ij V_i, dD/dy_j = q_j grad T_j from V, grad T (the fallback of
//                   k_pass2_mma when 32-bit offsets would overflow).
//
// (The first iteration's tcgen05 pass-1 / Gram / pass-2 kernels for NCC K <= 32 — fused sampling + Gram,
// k_gram_tc, k_pass2_tc — were measured slower than the mma.sync kernels of engine_mma.cuh and removed;
// DESIGN.md §4 keeps their numbers.)
#pragma once
#include "tma.cuh"

namespace sr {


// k_sample_v with GV, software-pipelined over NI consecutive 1024-pixel blocks of one frame per CTA:
// the y of block i + 1 is loaded before the gathers of block i, so only the gathers' latency is
// exposed per block (k_sample_v exposes the y latency and then the gather latency).
// LO (NGF): u in fp64 arithmetic (interp_v64), written as V = fl32(u) and VL = fl32(u - V).
template <int D, bool POW2, int NI, int SPT = 4, bool LO = false>
__global__ void __launch_bounds__(256, 6) k_sample_vp(const Args a, float* __restrict__ V, float* __restrict__ G,
                                                      long long vstride, float* __restrict__ VL = nullptr) {
  constexpr int BP = 256 * SPT;
  const int npix = (int)(a.pix_hi - a.pix_lo);
  const int k = (int)blockIdx.y;
  const int tid = (int)threadIdx.x;
  const int fi = a.job->frame_index[k];
  const float* img = reinterpret_cast<const float*>(a.frames) + (long long)fi * a.g.N;
  const float* yk = reinterpret_cast<const float*>(a.y) + (long long)(k * D) * a.y_stride + (a.pix_lo - a.y_off);
  float* vk = V + (long long)k * vstride;
  float* gk = G + (long long)(k * D) * vstride;
  const uint64_t pol_first = l2_policy_evict_first();
  const float* shifts = reinterpret_cast<const float*>(a.shifts);
  const float sh = shifts ? shifts[fi] : 0.f;
  const int bfirst = (int)blockIdx.x * NI;
  auto load_y = [&](int blk, float (&p)[SPT][D]) {
    const int b0 = blk * BP, nb = npix - b0;
#pragma unroll
    for (int e = 0; e < SPT; ++e) {
      const int pe = b0 + min(tid + 256 * e, nb - 1);
#pragma unroll
      for (int c = 0; c < D; ++c) p[e][c] = ldg_hint_nv(yk + (long long)c * a.y_stride + pe, pol_first);
    }
  };
  float pc[SPT][D];
  load_y(bfirst, pc);
#pragma unroll
  for (int it = 0; it < NI; ++it) {
    const int blk = bfirst + it;
    const int b0 = blk * BP;
    if (b0 >= npix) break;
    float pn[SPT][D];
    if (it + 1 < NI && b0 + BP < npix) load_y(blk + 1, pn);
    float v[SPT], vl[SPT], gd[SPT][D];
#pragma unroll
    for (int e = 0; e < SPT; ++e) {
      if (LO) {
        const double u = interp_v64<D, POW2>(img, a.g, pc[e], gd[e]);
        v[e] = (float)u;
        vl[e] = (float)(u - (double)v[e]);
      } else {
        v[e] = interp<float, float, D, true, POW2>(img, a.g, pc[e], gd[e]);
      }
    }
    const int nb = npix - b0;
#pragma unroll
    for (int e = 0; e < SPT; ++e) {
      const int pe = tid + 256 * e;
      if (pe < nb) {
        if (LO) VL[(long long)k * vstride + b0 + pe] = vl[e];
        vk[b0 + pe] = v[e] - sh;
#pragma unroll
        for (int c = 0; c < D; ++c) gk[(long long)c * vstride + b0 + pe] = gd[e][c];
      }
    }
    if (it + 1 < NI) {
#pragma unroll
      for (int e = 0; e < SPT; ++e)
#pragma unroll
        for (int c = 0; c < D; ++c) pc[e][c] = pn[e][c];
    }
  }
}

// Streaming pass 2 (fp32 NCC displacement, K <= 32) after a k_sample_v<GV = true> pass 1 on the same
// y: block = 64 pixels x 4 frame groups; thread (pixel, group g) forms q_j = beta'_j + sum_i M'_ij V_i(p)
// for the 8 frames j = 8 g .. 8 g + 7 (V read by the 4 group threads: L1 hits; M' broadcast from
// shared memory) and writes dD/dy_j,c(p) = q_j G_j,c(p).  No gathers and no y: V, G in, dD/dy out.
template <int D>
__global__ void __launch_bounds__(256) k_pass2_stream(const Args a, const float* __restrict__ V,
                                                      const float* __restrict__ G, long long vstride) {
  constexpr int KP = 32, PB = 64, JG = 8;
  __shared__ __align__(16) float Ms[KP * KP];  // Ms[i][j], zero past K
  __shared__ float bs[KP];
  const int tid = threadIdx.x;
  const int K = a.K;
  const StatsLayout L(K);
  const float* Mg = coef_ptr<float>(a.stats, L);
  for (int e = tid; e < KP * KP; e += 256) {
    const int i = e / KP, j = e % KP;
    Ms[e] = (i < K && j < K) ? Mg[i * K + j] : 0.f;
  }
  if (tid < KP) bs[tid] = tid < K ? (float)a.stats[L.beta + tid] : 0.f;
  __syncthreads();
  const int g = tid / PB, px = tid % PB;  // warps 0-1: group 0, ... (lanes on consecutive pixels)
  const int j0 = g * JG;
  if (j0 >= K) return;
  const long long npix = a.pix_hi - a.pix_lo;
  const long long pl = (long long)blockIdx.x * PB + px;
  if (pl >= npix) return;
  const float* __restrict__ vp = V + pl;
  const uint64_t pol = l2_policy_evict_first();  // last use of V / grad T; dD/dy is streamed out
  float v[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i) v[i] = i < K ? __ldg(vp + (long long)i * vstride) : 0.f;
  float q[JG];
#pragma unroll
  for (int jj = 0; jj < JG; ++jj) q[jj] = bs[j0 + jj];
#pragma unroll
  for (int i = 0; i < KP; ++i) {
    const float4 m0 = *reinterpret_cast<const float4*>(Ms + i * KP + j0);
    const float4 m1 = *reinterpret_cast<const float4*>(Ms + i * KP + j0 + 4);
    q[0] = fmaf(m0.x, v[i], q[0]);
    q[1] = fmaf(m0.y, v[i], q[1]);
    q[2] = fmaf(m0.z, v[i], q[2]);
    q[3] = fmaf(m0.w, v[i], q[3]);
    q[4] = fmaf(m1.x, v[i], q[4]);
    q[5] = fmaf(m1.y, v[i], q[5]);
    q[6] = fmaf(m1.z, v[i], q[6]);
    q[7] = fmaf(m1.w, v[i], q[7]);
  }
  float* __restrict__ ob = reinterpret_cast<float*>(a.out) + (a.pix_lo - a.o_off) + pl;
  const float* __restrict__ gp = G + pl;
  float gv[JG][D];
#pragma unroll
  for (int jj = 0; jj < JG; ++jj)
#pragma unroll
    for (int c = 0; c < D; ++c)
      gv[jj][c] = j0 + jj < K ? ldg_hint(gp + (long long)((j0 + jj) * D + c) * vstride, pol) : 0.f;
#pragma unroll
  for (int jj = 0; jj < JG; ++jj)
    if (j0 + jj < K)
#pragma unroll
      for (int c = 0; c < D; ++c) stg_hint(ob + (long long)((j0 + jj) * D + c) * a.o_stride, q[jj] * gv[jj][c], pol);
}

}  // namespace sr

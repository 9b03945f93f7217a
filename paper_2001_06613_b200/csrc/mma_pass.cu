// Launchers for engine_mma.cuh (fp32 NCC displacement fields, K <= 32, 2-D and 3-D).
#include <cstdio>
#include <cstdlib>
#include <utility>
#include "engine_mma.cuh"
#include "engine_ngf_tc.cuh"
#include "launch.cuh"

namespace sr {

// Sampling kernel of the split paths (V = v - shift and grad T): k_sample_vp over 2 blocks of 1024
// pixels per CTA, the y of the next block loaded before this block's corner gathers (33.0 vs 37.5 us at C2
// for the unpipelined sampler); with VL (NGF) u is kept as an fp32 pair (fp64 arithmetic).
template <int D>
static cudaError_t launch_sample_vg(const Launch& L, const Args& a, float* V, float* G, long long vstride,
                                    float* VL = nullptr) {
  const long long npix = a.pix_hi - a.pix_lo;
  const long long nblk = (npix + 1023) / 1024;
  const dim3 sgrid((unsigned)((nblk + 1) / 2), (unsigned)a.K);
  if (VL) {
    if (a.g.pow2) k_sample_vp<D, true, 2, 4, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride, VL);
    else k_sample_vp<D, false, 2, 4, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride, VL);
  } else {
    if (a.g.pow2) k_sample_vp<D, true, 2><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_vp<D, false, 2><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
  }
  return cudaGetLastError();
}
cudaError_t sample_vg_d2(const Launch& L, const Args& a, float* V, float* G, long long vstride, float* VL) {
  return launch_sample_vg<2>(L, a, V, G, vstride, VL);
}
cudaError_t sample_vg_d3(const Launch& L, const Args& a, float* V, float* G, long long vstride, float* VL) {
  return launch_sample_vg<3>(L, a, V, G, vstride, VL);
}

// 3-D view [rows][ncomp][npix] (row stride ncomp * stride, component stride `stride` floats) for the
// TMA-fed Gram: boxes of [32 rows x 1 component x 32 pixels], SWIZZLE_128B, zero fill past the edges
static bool encode_gram_map(EncodeTiledFn fn, CUtensorMap* m, const float* base, long long npix, int ncomp,
                            int rows, long long stride) {
  memset(m, 0, sizeof *m);
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (stride * 4) % 16) return false;
  cuuint64_t gdim[3] = {(cuuint64_t)npix, (cuuint64_t)ncomp, (cuuint64_t)rows};
  cuuint64_t gstr[2] = {(cuuint64_t)stride * 4, (cuuint64_t)ncomp * stride * 4};
  cuuint32_t box[3] = {(cuuint32_t)GTM::BOXP, 1, (cuuint32_t)GTM::KP};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), gdim, gstr, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// grad T [K][D][stride] as a 3-D map for k_pass2_tma: boxes of [32 frames x D components x 32 pixels]
template <int D>
static bool encode_p2g_map(EncodeTiledFn fn, CUtensorMap* m, const float* base, long long npix, int rows,
                           long long stride) {
  memset(m, 0, sizeof *m);
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (stride * 4) % 16) return false;
  cuuint64_t gdim[3] = {(cuuint64_t)npix, (cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t gstr[2] = {(cuuint64_t)stride * 4, (cuuint64_t)D * stride * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)D, 32};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), gdim, gstr, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// split NGF pass 1 for K <= 32: sampling, features, then k_gram_h (tcgen05 kind::f16, 256-pixel tiles) with
// KP = 32 partials (it replaced the TMA-fed mma.sync Gram k_gram_tma<NGF>: C4 0.23 -> 0.17 ms)
template <int D>
static cudaError_t run_ngf_pass1_mma(const Launch& L, const Args& a, const NgfBufs& B, double* part,
                                     size_t part_cap, int* nblk) {
  if (a.K > 32) return cudaErrorNotSupported;
  GramH gh;
  cudaError_t e = gram_h_prepare<D>(a, B, &gh);
  if (e != cudaSuccess) return e;
  Args av = a;  // u and grad T over [vlo, vhi) (no shift: n only sees differences of u)
  av.pix_lo = B.vlo;
  av.pix_hi = B.vhi;
  av.shifts = nullptr;
  e = D == 2 ? ngf_sfeat_d2(L, a, B) : cudaErrorNotSupported;
  if (e == cudaErrorNotSupported) {
    e = launch_sample_vg<D>(L, av, B.V, B.G, B.vstride, B.VL);
    if (e != cudaSuccess) return e;
    const dim3 fgrid((unsigned)((B.zhi - B.zlo + 1023) / 1024), (unsigned)a.K);
    k_ngf_feat4<D><<<fgrid, 256, 0, L.stream>>>(a, B.V, B.VL, B.vlo, B.vstride, B.Nf, B.Rho, B.zlo, B.zhi,
                                                B.zstride);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  return gram_h_launch<D, 32>(L, a, gh, part, part_cap, nblk);
}
cudaError_t ngf_pass1_mma_d2(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t cap, int* nblk) {
  return run_ngf_pass1_mma<2>(L, a, B, part, cap, nblk);
}
cudaError_t ngf_pass1_mma_d3(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t cap, int* nblk) {
  return run_ngf_pass1_mma<3>(L, a, B, part, cap, nblk);
}

// split pass 1: k_sample_v (V = v - shift, grad T) then k_gram_mma (Gram + per-frame stats of V)
template <int D>
static cudaError_t run_sample_then_gram(const Launch& L, const Args& a, float* V, float* G, long long vstride,
                                        double* part, size_t part_cap, int* nblk) {
  const long long npix = a.pix_hi - a.pix_lo;
  if (npix <= 0 || a.K > GMM::KP) return cudaErrorInvalidValue;
  cudaError_t e = launch_sample_vg<D>(L, a, V, G, vstride);
  if (e != cudaSuccess) return e;
  const long long ntiles = (npix + GMM::TP - 1) / GMM::TP;
  const size_t stride = (size_t)GMM::KP * GMM::KP + 3 * GMM::KP;
  EncodeTiledFn fn = encode_tiled_fn();
  if (fn) {  // TMA-fed Gram (k_gram_tma); the register-fed k_gram_mma when the map cannot be encoded
    CUtensorMap vmap;
    if (encode_gram_map(fn, &vmap, V, npix, 1, a.K, vstride)) {
      const size_t smem = gtm_smem();
      auto gk = k_gram_tma<false>;
      e = cudaFuncSetAttribute(gk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      int grid = occupancy_grid(L, gk, GTM::NT, smem, ntiles);
      if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
      Args b = a;
      b.part = part;
      gk<<<grid, GTM::NT, smem, L.stream>>>(b, vmap, (int)ntiles);
      *nblk = grid;
      return cudaGetLastError();
    }
  }
  const size_t smem = 4 * (size_t)GMM::KP * GMM::LD * sizeof(float);
  e = cudaFuncSetAttribute(k_gram_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int grid = occupancy_grid(L, k_gram_mma, GMM::NT, smem, ntiles);
  if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
  Args b = a;
  b.part = part;
  k_gram_mma<<<grid, GMM::NT, smem, L.stream>>>(b, V, vstride);
  *nblk = grid;
  return cudaGetLastError();
}

template <int D>
static cudaError_t run_pass2_mma(const Launch& L, const Args& a, const float* V, const float* G, long long vstride) {
  const long long npix = a.pix_hi - a.pix_lo;
  if (npix <= 0) return cudaSuccess;
  // TMA-fed pass 2 (k_pass2_tma; 24.8 vs 26.1 us at C2); SEQREG_B200_P2TMA=0 (and 3-D): k_pass2_mma
  static const bool p2tma = !(getenv("SEQREG_B200_P2TMA") && getenv("SEQREG_B200_P2TMA")[0] == '0');
  EncodeTiledFn fn = encode_tiled_fn();
  if (p2tma && fn && D == 2) {  // (3-D: 152 registers, one 8-warp CTA per SM — not measured faster)
    CUtensorMap vmap, gmap;
    if (encode_gram_map(fn, &vmap, V, npix, 1, a.K, vstride) && encode_p2g_map<D>(fn, &gmap, G, npix, a.K, vstride)) {
      using C = P2T<D>;
      const size_t smem = C::smem();
      cudaError_t e = cudaFuncSetAttribute(k_pass2_tma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      const int grid = occupancy_grid(L, k_pass2_tma<D>, C::NT, smem, (npix + C::TP - 1) / C::TP);
      k_pass2_tma<D><<<grid, C::NT, smem, L.stream>>>(a, vmap, gmap);
      return cudaGetLastError();
    }
  }
  const long long nblk = (npix + P2M::PW - 1) / P2M::PW;
  const long long want = (nblk + P2M::NT / 32 - 1) / (P2M::NT / 32);
  const int grid = occupancy_grid(L, k_pass2_mma<D, 2>, P2M::NT, 0, want);
  k_pass2_mma<D, 2><<<grid, P2M::NT, 0, L.stream>>>(a, V, G, vstride);
  return cudaGetLastError();
}

// Split NGF pass 2 contraction: k_ngf_z_tc (tcgen05 kind::f16, engine_ngf_tc.cuh), K <= 128
template <int D>
static cudaError_t run_ngf_z_mma(const Launch& L, const Args& a, const NgfBufs& B) {
  const int K = a.K;
  const long long nzp = B.zhi - B.zlo;
  if (nzp <= 0) return cudaSuccess;
  if (K > 128 || (long long)K * D * B.zstride >= (1LL << 31)) return cudaErrorNotSupported;
  if (K <= 32) {  // legacy-pipe mma.sync f16 contraction (k_ngf_z_f16): C4 0.44 vs 0.82 ms for k_ngf_z_tc
    using C = NZ<D>;
    const int JT = (K + 15) / 16, KS = (K + 15) / 16;
    const long long items = (nzp + C::PW - 1) / C::PW * ((JT + C::MW - 1) / C::MW);
    const size_t smem = (size_t)2 * JT * KS * 32 * 16;
    cudaError_t e = cudaFuncSetAttribute(k_ngf_z_f16<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = occupancy_grid(L, k_ngf_z_f16<D>, C::NT, smem, (items + C::NT / 32 - 1) / (C::NT / 32));
    k_ngf_z_f16<D><<<grid, C::NT, smem, L.stream>>>(a, B.Nf, B.Rho, B.zlo, B.zhi, B.zstride, B.Z);
    return cudaGetLastError();
  }
  const size_t smem = ztc_smem<D>(K);
  cudaError_t e = cudaFuncSetAttribute(k_ngf_z_tc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int tp = ztc_mt((K + 15) / 16 * 16) * ZTC<D>::PXT;  // pixels per tile
  const long long ntiles = (nzp + tp - 1) / tp;
  int grid = L.grid_override > 0 ? L.grid_override : L.sms;
  if (grid > ntiles) grid = (int)ntiles;
  k_ngf_z_tc<D><<<grid, ZTC<D>::NT, smem, L.stream>>>(a, B.Nf, B.Rho, B.zlo, B.zhi, B.zstride, B.Z);
  return cudaGetLastError();
}
cudaError_t ngf_z_mma_d2(const Launch& L, const Args& a, const NgfBufs& B) { return run_ngf_z_mma<2>(L, a, B); }
cudaError_t ngf_z_mma_d3(const Launch& L, const Args& a, const NgfBufs& B) { return run_ngf_z_mma<3>(L, a, B); }

cudaError_t sample_then_gram_d2(const Launch& L, const Args& a, float* V, float* G, long long vstride, double* part,
                                size_t cap, int* nblk) {
  return run_sample_then_gram<2>(L, a, V, G, vstride, part, cap, nblk);
}
cudaError_t sample_then_gram_d3(const Launch& L, const Args& a, float* V, float* G, long long vstride, double* part,
                                size_t cap, int* nblk) {
  return run_sample_then_gram<3>(L, a, V, G, vstride, part, cap, nblk);
}
cudaError_t pass2_mma_d2(const Launch& L, const Args& a, const float* V, const float* G, long long vstride) {
  return run_pass2_mma<2>(L, a, V, G, vstride);
}
cudaError_t pass2_mma_d3(const Launch& L, const Args& a, const float* V, const float* G, long long vstride) {
  return run_pass2_mma<3>(L, a, V, G, vstride);
}

}  // namespace sr

// Launchers for engine_mma.cuh (fp32 NCC displacement fields, K <= 32, 2-D and 3-D).
#include <cstdio>
#include <cstdlib>
#include <utility>
#include "engine_mma.cuh"
#include "engine_ngf_tc.cuh"
#include "launch.cuh"

namespace sr {

// launch with programmatic stream serialization (PDL) when SEQREG_B200_PDL=1 (measured slower at C2:
// 95.3 vs 91.1 us per step — early-resident dependent CTAs take slots from the draining predecessor)
template <typename... KArgs, typename... Args2>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args2&&... args) {
  static const bool on = getenv("SEQREG_B200_PDL") && getenv("SEQREG_B200_PDL")[0] == '1';
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args2>(args)...);
}

template <int D>
static cudaError_t run_sample_gram(const Launch& L, const Args& a, float* V, float* G, long long vstride,
                                   double* part, size_t part_cap, int* nblk) {
  const long long npix = a.pix_hi - a.pix_lo;
  if (npix <= 0 || a.K > SG::KP) return cudaErrorInvalidValue;
  const long long ntiles = (npix + SG::TP - 1) / SG::TP;
  // SEQREG_B200_SGB: minimum resident CTAs per SM the kernel is compiled for (register budget)
  static const int minb = getenv("SEQREG_B200_SGB") ? atoi(getenv("SEQREG_B200_SGB")) : 4;
  auto kern = a.g.pow2 ? (minb == 3 ? k_sample_gram<D, true, 3> : minb == 2 ? k_sample_gram<D, true, 2> : k_sample_gram<D, true, 4>)
                       : (minb == 3 ? k_sample_gram<D, false, 3> : minb == 2 ? k_sample_gram<D, false, 2> : k_sample_gram<D, false, 4>);
  int grid = occupancy_grid(L, kern, SG::NT, 0, ntiles);
  const size_t stride = (size_t)SG::KP * SG::KP + 3 * SG::KP;
  if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
  Args b = a;
  b.part = part;
  kern<<<grid, SG::NT, 0, L.stream>>>(b, V, G, vstride);
  *nblk = grid;
  return cudaGetLastError();
}

// SEQREG_B200_GSUP: tiles per k_gram_tma ring stage (1: 2 CTAs x 8 warps per SM; 2: 1 CTA x 16 warps)
static int gram_sup() {
  static const int s = getenv("SEQREG_B200_GSUP") ? atoi(getenv("SEQREG_B200_GSUP")) : 1;
  return s == 2 ? 2 : 1;
}

// Sampling kernel of the split paths (V = v - shift and grad T).  Default: k_sample_vp over 2 blocks
// per CTA (33.0 vs 37.5 us at C2).  SEQREG_B200_SPT: 4 / 2 / 8 = k_sample_v with that many samples in
// flight per thread, 44 = k_sample_vp over 4 blocks.
template <int D>
static cudaError_t launch_sample_vg(const Launch& L, const Args& a, float* V, float* G, long long vstride,
                                    float* VL = nullptr) {
  const long long npix = a.pix_hi - a.pix_lo;
  if (VL) {  // NGF: u as an fp32 pair (k_sample_vp<LO>)
    const long long nblk = (npix + 1023) / 1024;
    const dim3 sgrid((unsigned)((nblk + 1) / 2), (unsigned)a.K);
    if (a.g.pow2) k_sample_vp<D, true, 2, 4, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride, VL);
    else k_sample_vp<D, false, 2, 4, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride, VL);
    return cudaGetLastError();
  }
  // SEQREG_B200_SPT: samples in flight per thread of k_sample_v (2, 4 or 8)
  static const int spt = getenv("SEQREG_B200_SPT") ? atoi(getenv("SEQREG_B200_SPT")) : 42;
  if (spt == 8) {
    const dim3 sgrid((unsigned)((npix + 256 * 8 - 1) / (256 * 8)), (unsigned)a.K);
    if (a.g.pow2) k_sample_v<D, true, 8, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_v<D, false, 8, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
  } else if (spt == 2) {
    const dim3 sgrid((unsigned)((npix + 256 * 2 - 1) / (256 * 2)), (unsigned)a.K);
    if (a.g.pow2) k_sample_v<D, true, 2, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_v<D, false, 2, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
  } else if (spt == 42) {  // software-pipelined over 2 blocks per CTA (k_sample_vp)
    const long long nblk = (npix + 1023) / 1024;
    const dim3 sgrid((unsigned)((nblk + 1) / 2), (unsigned)a.K);
    if (a.g.pow2) k_sample_vp<D, true, 2><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_vp<D, false, 2><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
  } else if (spt == 43) {  // ... over 3 blocks per CTA
    const long long nblk = (npix + 1023) / 1024;
    const dim3 sgrid((unsigned)((nblk + 2) / 3), (unsigned)a.K);
    if (a.g.pow2) k_sample_vp<D, true, 3><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_vp<D, false, 3><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
  } else if (spt == 24) {  // 4 blocks of 512 pixels per CTA, 2 samples per thread per block
    const long long nblk = (npix + 511) / 512;
    const dim3 sgrid((unsigned)((nblk + 3) / 4), (unsigned)a.K);
    if (a.g.pow2) k_sample_vp<D, true, 4, 2><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_vp<D, false, 4, 2><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
  } else if (spt == 44) {  // ... over 4 blocks per CTA
    const long long nblk = (npix + 1023) / 1024;
    const dim3 sgrid((unsigned)((nblk + 3) / 4), (unsigned)a.K);
    if (a.g.pow2) k_sample_vp<D, true, 4><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_vp<D, false, 4><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
  } else {
    constexpr int SPT = 4;
    const dim3 sgrid((unsigned)((npix + 256 * SPT - 1) / (256 * SPT)), (unsigned)a.K);
    if (a.g.pow2) k_sample_v<D, true, SPT, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
    else k_sample_v<D, false, SPT, true><<<sgrid, 256, 0, L.stream>>>(a, V, G, vstride);
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

// split NGF pass 1 for K <= 32: sampling, features, then the TMA-fed mma.sync Gram of n (KP = 32 partials)
template <int D>
static cudaError_t run_ngf_pass1_mma(const Launch& L, const Args& a, const NgfBufs& B, double* part,
                                     size_t part_cap, int* nblk) {
  const long long npix = a.pix_hi - a.pix_lo;
  if (npix <= 0 || a.K > GTM::KP) return cudaErrorNotSupported;
  if (((a.pix_lo - B.zlo) * 4) % 16) return cudaErrorNotSupported;
  EncodeTiledFn fn = encode_tiled_fn();
  CUtensorMap xmap;
  if (!fn || !encode_gram_map(fn, &xmap, B.Nf + (a.pix_lo - B.zlo), npix, D, a.K, B.zstride))
    return cudaErrorNotSupported;
  Args av = a;  // u and grad T over [vlo, vhi) (no shift: n only sees differences of u)
  av.pix_lo = B.vlo;
  av.pix_hi = B.vhi;
  av.shifts = nullptr;
  cudaError_t e = D == 2 ? ngf_sfeat_d2(L, a, B) : cudaErrorNotSupported;
  if (e == cudaErrorNotSupported) {
    e = launch_sample_vg<D>(L, av, B.V, B.G, B.vstride, B.VL);
    if (e != cudaSuccess) return e;
    const dim3 fgrid((unsigned)((B.zhi - B.zlo + 1023) / 1024), (unsigned)a.K);
    k_ngf_feat4<D><<<fgrid, 256, 0, L.stream>>>(a, B.V, B.VL, B.vlo, B.vstride, B.Nf, B.Rho, B.zlo, B.zhi,
                                                B.zstride);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  const int sup = gram_sup();
  const size_t smem = gtm_smem(sup);
  auto gk = sup == 2 ? k_gram_tma<true, 2> : k_gram_tma<true, 1>;
  e = cudaFuncSetAttribute(gk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int ntx = (int)((npix + GTM::TP - 1) / GTM::TP);
  int grid = occupancy_grid(L, gk, GTM::NT * sup, smem, ((long long)ntx * D + sup - 1) / sup);
  const size_t stride = (size_t)GTM::KP * GTM::KP + 3 * GTM::KP;
  if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
  Args b = a;
  b.part = part;
  gk<<<grid, GTM::NT * sup, smem, L.stream>>>(b, xmap, ntx);
  *nblk = grid;
  return cudaGetLastError();
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
  if (fn && !getenv("SEQREG_B200_GRAMREG")) {  // TMA-fed Gram (k_gram_tma)
    CUtensorMap vmap;
    if (encode_gram_map(fn, &vmap, V, npix, 1, a.K, vstride)) {
      const int sup = gram_sup();
      const size_t smem = gtm_smem(sup);
      auto gk = sup == 2 ? k_gram_tma<false, 2> : k_gram_tma<false, 1>;
      e = cudaFuncSetAttribute(gk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      int grid = occupancy_grid(L, gk, GTM::NT * sup, smem, (ntiles + sup - 1) / sup);
      if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
      Args b = a;
      b.part = part;
      e = launch_pdl(gk, dim3(grid), dim3(GTM::NT * sup), smem, L.stream, b, vmap, (int)ntiles);
      *nblk = grid;
      return e;
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
  // TMA-fed pass 2 (k_pass2_tma; 24.8 vs 26.1 us at C2); SEQREG_B200_P2TMA=0: k_pass2_mma
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
  if (getenv("SEQREG_B200_P2BULK") && (vstride & 3) == 0 && (reinterpret_cast<uintptr_t>(V) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(G) & 15) == 0) {
    using C = P2B<D>;
    const size_t smem = C::smem();
    cudaError_t e = cudaFuncSetAttribute(k_pass2_bulk<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long nblk = (npix + C::PW - 1) / C::PW;
    const long long want = (nblk + C::WPC - 1) / C::WPC;
    const int grid = occupancy_grid(L, k_pass2_bulk<D>, C::NT, smem, want);
    k_pass2_bulk<D><<<grid, C::NT, smem, L.stream>>>(a, V, G, vstride);
    return cudaGetLastError();
  }
  const long long nblk = (npix + P2M::PW - 1) / P2M::PW;
  const long long want = (nblk + P2M::NT / 32 - 1) / (P2M::NT / 32);
  // SEQREG_B200_P2B: minimum resident CTAs per SM the pass-2 kernel is compiled for (register budget)
  static const int minb = getenv("SEQREG_B200_P2B") ? atoi(getenv("SEQREG_B200_P2B")) : 2;
  auto kern = minb == 3 ? k_pass2_mma<D, 3> : k_pass2_mma<D, 2>;
  const int grid = occupancy_grid(L, kern, P2M::NT, 0, want);
  return launch_pdl(kern, dim3(grid), dim3(P2M::NT), 0, L.stream, a, V, G, vstride);
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

cudaError_t sample_gram_d2(const Launch& L, const Args& a, float* V, float* G, long long vstride, double* part,
                           size_t cap, int* nblk) {
  return run_sample_gram<2>(L, a, V, G, vstride, part, cap, nblk);
}
cudaError_t sample_gram_d3(const Launch& L, const Args& a, float* V, float* G, long long vstride, double* part,
                           size_t cap, int* nblk) {
  return run_sample_gram<3>(L, a, V, G, vstride, part, cap, nblk);
}
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

// launch.cuh — host-side launchers for one (T, D, FEAT, PARAM, KP) combination.
// Included by the per-(dtype, ndim) instantiation units inst_*.cu.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include "engine.cuh"

namespace sr {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D view of the displacement planes: rows = k*D + c (K*D of them), columns = pixels of the
// y buffer; boxes of `box_cols` pixels x all rows.
template <typename T>
static bool encode_y_map(CUtensorMap* m, const Args& a, int rows, int box_cols) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(a.y) & 15) || ((a.y_stride * (long long)sizeof(T)) % 16) || rows > 256)
    return false;
  cuuint64_t gdim[2] = {(cuuint64_t)a.y_stride, (cuuint64_t)rows};
  cuuint64_t gstr[1] = {(cuuint64_t)a.y_stride * sizeof(T)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
            const_cast<void*>(a.y), gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Launch {
  cudaStream_t stream;
  int sms;
  int grid_override;  // 0 = auto
  int legacy;         // 1 = force the non-specialized kernels (A/B checks)
  int tc;             // 0 = no tensor-core split pass 1 (SIMT Gram k_pass1_ws for fp32 NCC, K <= 32)
};

template <typename K>
static int occupancy_grid(const Launch& L, K kernel, int nt, size_t smem, long long ntiles) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, smem);
  if (per_sm < 1) per_sm = 1;
  long long g = (long long)per_sm * L.sms;
  if (L.grid_override > 0) g = L.grid_override;
  if (g > ntiles) g = ntiles;
  if (g < 1) g = 1;
  return (int)g;
}

template <typename T, int D, int FEAT, int PARAM, int KP>
struct Runner {
  // pass 1; per-CTA partials [grid][KP*KP + 3KP] in `part`, CTA count in *nblk
  static cudaError_t pass1(const Launch& L, const Args& a, double* part, size_t part_cap,
                           int* nblk) {
    if constexpr (FEAT == NCC && PARAM == DISP && KP <= 32) {
      if (!L.legacy) return pass1_ws(L, a, part, part_cap, nblk);
    }
    using C = G1<T, KP, FEAT>;
    using Tl = Tile1<T, D, FEAT, KP>;
    const size_t smem = pass1_smem<T, D, FEAT, PARAM, KP>();
    auto kern = k_pass1<T, D, FEAT, PARAM, KP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long npix = a.pix_hi - a.pix_lo;
    const long long ntiles = (npix + Tl::TP - 1) / Tl::TP;
    int grid = occupancy_grid(L, kern, C::NT, smem, ntiles > 0 ? ntiles : 1);
    const size_t stride = (size_t)KP * KP + 3 * KP;
    if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
    Args b = a;
    b.part = part;
    kern<<<grid, C::NT, smem, L.stream>>>(b);
    *nblk = grid;
    return cudaGetLastError();
  }

  // warp-specialized pass 1 (NCC displacement, KP <= 32), engine_ws.cuh
  static cudaError_t pass1_ws(const Launch& L, const Args& a, double* part, size_t part_cap, int* nblk) {
    using C = WS1<T, KP>;
    const size_t smem = ws1_smem<T, D, KP>();
    auto kern = k_pass1_ws<T, D, KP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long npix = a.pix_hi - a.pix_lo;
    const long long ntiles = (npix + C::TP - 1) / C::TP;
    int grid = occupancy_grid(L, kern, C::NT, smem, ntiles > 0 ? ntiles : 1);
    const size_t stride = (size_t)KP * KP + 3 * KP;
    if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
    Args b = a;
    b.part = part;
    CUtensorMap ymap;
    memset(&ymap, 0, sizeof ymap);
    b.ymap_ok = encode_y_map<T>(&ymap, a, a.K * D, C::TP) ? 1 : 0;
    kern<<<grid, C::NT, smem, L.stream>>>(b, ymap);
    *nblk = grid;
    return cudaGetLastError();
  }

  static cudaError_t pass2(const Launch& L, const Args& a, double* part_aff, size_t aff_cap,
                           int* nblk_out) {
    using C = G2<T, KP>;
    constexpr int NA = D * (D + 1);
    size_t smem = pass2_smem<T, D, FEAT, KP>();
    const size_t need_red = (size_t)NA * C::NT * 8;
    if (smem < need_red) smem = need_red;
    auto kern = k_pass2<T, D, FEAT, PARAM, KP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long npix = a.pix_hi - a.pix_lo;
    const long long ntiles = (npix + C::TP - 1) / C::TP;
    int grid = occupancy_grid(L, kern, C::NT, smem, ntiles > 0 ? ntiles : 1);
    if (PARAM == AFFINE && FEAT == NCC) {
      const size_t stride = (size_t)KP * NA;
      if ((size_t)grid * stride > aff_cap) grid = (int)(aff_cap / stride);
    }
    Args b = a;
    b.part_aff = part_aff;
    kern<<<grid, C::NT, smem, L.stream>>>(b);
    *nblk_out = grid;
    return cudaGetLastError();
  }
};

template <typename T, int D, int PARAM>
cudaError_t run_ngf_adjoint(const Launch& L, const Args& a, const T* zb, long long z_off,
                            long long z_stride, double* part_aff, size_t aff_cap, int* nblk_out) {
  const long long npix = a.pix_hi - a.pix_lo;
  const int gx = (int)((npix + 255) / 256);
  constexpr int NA = D * (D + 1);
  if (PARAM == AFFINE && (size_t)gx * a.K * NA > aff_cap) return cudaErrorInvalidValue;
  dim3 grid(gx > 0 ? gx : 1, a.K);
  Args b = a;
  b.part_aff = part_aff;
  k_ngf_adjoint<T, D, PARAM><<<grid, 256, 0, L.stream>>>(b, zb, z_off, z_stride);
  *nblk_out = grid.x;
  return cudaGetLastError();
}

template <typename T, int D>
cudaError_t run_curvature(const Launch& L, const Args& a, double alpha, double h, double* part,
                          size_t cap, int* nblk_out) {
  const long long npix = a.pix_hi - a.pix_lo;
  const int gx = (int)((npix + 255) / 256);
  dim3 grid(gx > 0 ? gx : 1, a.K * D);
  if ((size_t)grid.x * grid.y > cap) return cudaErrorInvalidValue;
  k_curvature<T, D><<<grid, 256, 0, L.stream>>>(a, alpha, h, part);
  *nblk_out = grid.x * grid.y;
  return cudaGetLastError();
}

// Split NGF path (engine_ngf.cuh).  Ranges: V / grad T over [vlo, vhi) = slab +- 2 rows, n / rho / z over
// [zlo, zhi) = slab +- 1 row, the Gram over the slab.  cudaErrorNotSupported: layouts the TMA map cannot
// express (the caller falls back to the generic kernels).
// the split paths' sampling kernel launcher (mma_pass.cu)
cudaError_t sample_vg_d2(const Launch& L, const Args& a, float* V, float* G, long long vstride, float* VL = nullptr);
cudaError_t sample_vg_d3(const Launch& L, const Args& a, float* V, float* G, long long vstride, float* VL = nullptr);

struct NgfBufs {
  float *V, *G, *Nf, *Rho, *Z;  // Rho holds 1/rho (k_ngf_feat4)
  float* VL;  // low fp32 parts of u (V + VL = u to ~1e-16 relative; interp_v64)
  long long vlo, vhi, vstride, zlo, zhi, zstride;
};

// 2-D fused sampling + NGF feature over the NgfBufs ranges (k_ngf_sfeat2f, else the generic k_ngf_sfeat2);
// NotSupported when the ranges are not whole rows (or, generic kernel only, a row does not fit one CTA)
inline cudaError_t ngf_sfeat_d2(const Launch& L, const Args& a, const NgfBufs& B) {
  const int n0 = a.g.n[0];
  if (a.g.nd != 2 || (B.zlo % n0) || (B.zhi % n0) || (a.pix_lo % n0) || (a.pix_hi % n0)) return cudaErrorNotSupported;
  const int rz0 = (int)(B.zlo / n0), rz1 = (int)(B.zhi / n0);
  const int rs0 = (int)(a.pix_lo / n0), rs1 = (int)(a.pix_hi / n0);
  const auto al8 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7) == 0; };
  const double e2 = a.eps * a.eps;
  const long long smax = 1LL << 30;  // 32-bit index arithmetic inside a frame's rows
  // k_ngf_sfeat2f: one warp per (chunk of 62 columns, segment of rows, frame), any row length; segments as long
  // as >= 4 waves of 32 warps per SM allow (every segment re-samples 2 halo rows and pays an unpipelined prologue)
  const int nchunk = (n0 + 61) / 62;
  int segf = 32;
  if (const char* sv = getenv("SEQREG_B200_SFSEG")) segf = atoi(sv) > 0 ? atoi(sv) : segf;
  while (segf > 8 && (long long)((rz1 - rz0 + segf - 1) / segf) * nchunk * a.K < 4LL * 32 * L.sms) segf /= 2;
  const long long nseg = (rz1 - rz0 + segf - 1) / segf;
  if (n0 >= 2 && n0 % 2 == 0 && a.g.n[1] >= 2 && e2 > 1e-30 && e2 < 1e30 && al8(B.Nf) && al8(B.Rho) && al8(B.G) &&
      ((B.zlo | B.zstride | B.vlo | B.vstride) & 1) == 0 && a.y_stride < smax && B.zstride < smax &&
      B.vstride < smax && a.g.N < smax && nseg <= 65535 && a.K <= 65535 &&
      !(getenv("SEQREG_B200_SFEAT") && getenv("SEQREG_B200_SFEAT")[0] == '0')) {
    const dim3 wgrid((unsigned)nchunk, (unsigned)nseg, (unsigned)a.K);
    if (a.g.pow2)
      k_ngf_sfeat2f<32, true><<<wgrid, 32, 0, L.stream>>>(a, segf, rz0, rz1, rs0, rs1, B.Nf, B.Rho, B.zlo, B.zstride,
                                                          B.G, B.vlo, B.vstride);
    else
      k_ngf_sfeat2f<32, false><<<wgrid, 32, 0, L.stream>>>(a, segf, rz0, rz1, rs0, rs1, B.Nf, B.Rho, B.zlo, B.zstride,
                                                           B.G, B.vlo, B.vstride);
    return cudaGetLastError();
  }
  // generic k_ngf_sfeat2: a whole row per CTA of 2 columns per thread (n0 <= 1024)
  if (n0 > 1024) return cudaErrorNotSupported;
  int seg = 32;
  while (seg > 8 && (long long)((rz1 - rz0 + seg - 1) / seg) * a.K < 8LL * L.sms) seg /= 2;
  const dim3 grid((unsigned)((rz1 - rz0 + seg - 1) / seg), (unsigned)a.K);
  constexpr int PX = 2;
  const int nt = ((n0 + PX - 1) / PX + 31) / 32 * 32;
  if (a.g.pow2)
    k_ngf_sfeat2<true, PX><<<grid, nt, 0, L.stream>>>(a, seg, rz0, rz1, rs0, rs1, B.Nf, B.Rho, B.zlo, B.zstride,
                                                      B.G, B.vlo, B.vstride);
  else
    k_ngf_sfeat2<false, PX><<<grid, nt, 0, L.stream>>>(a, seg, rz0, rz1, rs0, rs1, B.Nf, B.Rho, B.zlo, B.zstride,
                                                       B.G, B.vlo, B.vstride);
  return cudaGetLastError();
}

// k_gram_h over the slab of Nf [K][D][zstride]: [KPN frames x tp pixels] fp32 boxes of one component, zero fill
// past K and past the slab.  gram_h_prepare before the sampling kernels (NotSupported -> generic path).
struct GramH {
  GhLayout gl;
  size_t smem;
  CUtensorMap map;
};
template <int D>
inline cudaError_t gram_h_prepare(const Args& a, const NgfBufs& B, GramH* g) {
  const long long npix = a.pix_hi - a.pix_lo;
  if (npix <= 0) return cudaErrorNotSupported;
  if (((a.pix_lo - B.zlo) * 4) % 16 || (B.zstride * 4) % 16 || (reinterpret_cast<uintptr_t>(B.Nf) & 15))
    return cudaErrorNotSupported;
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return cudaErrorNotSupported;
  int smem_cap = 0;
  cudaDeviceGetAttribute(&smem_cap, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  g->gl = tgh_layout(a.K, (size_t)smem_cap);
  g->smem = tgh_smem(g->gl);
  memset(&g->map, 0, sizeof g->map);
  cuuint64_t gdim[3] = {(cuuint64_t)npix, (cuuint64_t)D, (cuuint64_t)a.K};
  cuuint64_t gstr[2] = {(cuuint64_t)B.zstride * 4, (cuuint64_t)D * B.zstride * 4};
  cuuint32_t hbox[3] = {(cuuint32_t)g->gl.tp, 1, (cuuint32_t)g->gl.rows};
  cuuint32_t es[3] = {1, 1, 1};
  if (g->gl.nst < 2 || g->smem > (size_t)smem_cap || 2 * g->gl.rows > 256 ||
      fn(&g->map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, B.Nf + (a.pix_lo - B.zlo), gdim, gstr, hbox, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  return cudaSuccess;
}
template <int D, int KP>
inline cudaError_t gram_h_launch(const Launch& L, const Args& a, const GramH& g, double* part, size_t part_cap,
                                 int* nblk) {
  const long long npix = a.pix_hi - a.pix_lo;
  cudaError_t e = cudaFuncSetAttribute(k_gram_h<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
  if (e != cudaSuccess) return e;
  const int ntx = (int)((npix + g.gl.tp - 1) / g.gl.tp);
  const long long ntiles = (long long)ntx * D;
  int grid = L.grid_override > 0 ? L.grid_override : L.sms;
  if (grid > ntiles) grid = (int)ntiles;
  const size_t stride = (size_t)KP * KP + 3 * KP;
  if ((size_t)grid * stride > part_cap) grid = (int)(part_cap / stride);
  Args b = a;
  b.part = part;
  k_gram_h<KP><<<grid, TGH::NT, g.smem, L.stream>>>(b, g.map, ntx, D, g.gl);
  *nblk = grid;
  return cudaGetLastError();
}

template <int D, int KP>
cudaError_t run_ngf_pass1_kp(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t part_cap,
                             int* nblk) {
  if (a.K > KP) return cudaErrorNotSupported;
  GramH gh;
  cudaError_t e = gram_h_prepare<D>(a, B, &gh);
  if (e != cudaSuccess) return e;
  e = D == 2 ? ngf_sfeat_d2(L, a, B) : cudaErrorNotSupported;
  if (e == cudaErrorNotSupported) {
    // u (an fp32 pair) and grad T over [vlo, vhi) (no shift: n only sees differences of u), then n, 1/rho
    Args av = a;
    av.pix_lo = B.vlo;
    av.pix_hi = B.vhi;
    av.shifts = nullptr;
    e = D == 2 ? sample_vg_d2(L, av, B.V, B.G, B.vstride, B.VL) : sample_vg_d3(L, av, B.V, B.G, B.vstride, B.VL);
    if (e != cudaSuccess) return e;
    const dim3 fgrid((unsigned)((B.zhi - B.zlo + 1023) / 1024), (unsigned)a.K);
    k_ngf_feat4<D><<<fgrid, 256, 0, L.stream>>>(a, B.V, B.VL, B.vlo, B.vstride, B.Nf, B.Rho, B.zlo, B.zhi,
                                                B.zstride);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  return gram_h_launch<D, KP>(L, a, gh, part, part_cap, nblk);
}

template <int D>
cudaError_t run_ngf_pass1(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t part_cap, int* nblk) {
  return a.K <= 64 ? run_ngf_pass1_kp<D, 64>(L, a, B, part, part_cap, nblk)
                   : run_ngf_pass1_kp<D, 128>(L, a, B, part, part_cap, nblk);
}

cudaError_t ngf_z_mma_d2(const Launch& L, const Args& a, const NgfBufs& B);
cudaError_t ngf_pass1_mma_d2(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t cap, int* nblk);
cudaError_t ngf_pass1_mma_d3(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t cap, int* nblk);
cudaError_t ngf_z_mma_d3(const Launch& L, const Args& a, const NgfBufs& B);

template <int D>
cudaError_t run_ngf_pass2(const Launch& L, const Args& a, const NgfBufs& B) {
  const cudaError_t ez = D == 2 ? ngf_z_mma_d2(L, a, B) : ngf_z_mma_d3(L, a, B);
  if (ez != cudaSuccess) return ez;
  const dim3 g2((unsigned)((a.pix_hi - a.pix_lo + 1023) / 1024), (unsigned)a.K);
  if (a.curv_alpha > 0)
    k_ngf_adj4<D, true><<<g2, 256, 0, L.stream>>>(a, B.Z, B.zlo, B.zstride, B.G, B.vlo, B.vstride);
  else
    k_ngf_adj4<D><<<g2, 256, 0, L.stream>>>(a, B.Z, B.zlo, B.zstride, B.G, B.vlo, B.vstride);
  return cudaGetLastError();
}
cudaError_t ngf_pass1_d2(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t cap, int* nblk);
cudaError_t ngf_pass1_d3(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t cap, int* nblk);
cudaError_t ngf_pass2_d2(const Launch& L, const Args& a, const NgfBufs& B);
cudaError_t ngf_pass2_d3(const Launch& L, const Args& a, const NgfBufs& B);

template <int D>
cudaError_t run_pass2_stream(const Launch& L, const Args& a, const float* V, const float* G, long long vstride) {
  const long long npix = a.pix_hi - a.pix_lo;
  if (npix <= 0) return cudaSuccess;
  k_pass2_stream<D><<<(unsigned)((npix + 63) / 64), 256, 0, L.stream>>>(a, V, G, vstride);
  return cudaGetLastError();
}
cudaError_t pass2_stream_d2(const Launch& L, const Args& a, const float* V, const float* G, long long vstride);
// engine_mma.cuh (mma_pass.cu): sampling + TMA-fed mma.sync Gram pass 1, mma.sync streaming pass 2
cudaError_t sample_then_gram_d2(const Launch& L, const Args& a, float* V, float* G, long long vstride, double* part,
                                size_t cap, int* nblk);
cudaError_t sample_then_gram_d3(const Launch& L, const Args& a, float* V, float* G, long long vstride, double* part,
                                size_t cap, int* nblk);
cudaError_t pass2_mma_d2(const Launch& L, const Args& a, const float* V, const float* G, long long vstride);
cudaError_t pass2_mma_d3(const Launch& L, const Args& a, const float* V, const float* G, long long vstride);
cudaError_t pass2_stream_d3(const Launch& L, const Args& a, const float* V, const float* G, long long vstride);

// Dispatch over (FEAT, PARAM, KP) for fixed (T, D).
template <typename T, int D>
struct Dispatch {
  template <int FEAT, int PARAM>
  static cudaError_t p1k(int KP, const Launch& L, const Args& a, double* part, size_t cap, int* red) {
    switch (KP) {
      case 8: return Runner<T, D, FEAT, PARAM, 8>::pass1(L, a, part, cap, red);
      case 16: return Runner<T, D, FEAT, PARAM, 16>::pass1(L, a, part, cap, red);
      case 32: return Runner<T, D, FEAT, PARAM, 32>::pass1(L, a, part, cap, red);
      case 64: return Runner<T, D, FEAT, PARAM, 64>::pass1(L, a, part, cap, red);
      default: return Runner<T, D, FEAT, PARAM, 128>::pass1(L, a, part, cap, red);
    }
  }
  template <int FEAT, int PARAM>
  static cudaError_t p2k(int KP, const Launch& L, const Args& a, double* pa, size_t cap, int* nb) {
    switch (KP) {
      case 8: return Runner<T, D, FEAT, PARAM, 8>::pass2(L, a, pa, cap, nb);
      case 16: return Runner<T, D, FEAT, PARAM, 16>::pass2(L, a, pa, cap, nb);
      case 32: return Runner<T, D, FEAT, PARAM, 32>::pass2(L, a, pa, cap, nb);
      case 64: return Runner<T, D, FEAT, PARAM, 64>::pass2(L, a, pa, cap, nb);
      default: return Runner<T, D, FEAT, PARAM, 128>::pass2(L, a, pa, cap, nb);
    }
  }
  static cudaError_t pass1(int feat, int param, int KP, const Launch& L, const Args& a,
                           double* part, size_t cap, int* red) {
    if (feat == NCC) return param == AFFINE ? p1k<NCC, AFFINE>(KP, L, a, part, cap, red)
                                            : p1k<NCC, DISP>(KP, L, a, part, cap, red);
    return param == AFFINE ? p1k<NGF, AFFINE>(KP, L, a, part, cap, red)
                           : p1k<NGF, DISP>(KP, L, a, part, cap, red);
  }
  static cudaError_t pass2(int feat, int param, int KP, const Launch& L, const Args& a,
                           double* pa, size_t cap, int* nb) {
    if (feat == NCC) return param == AFFINE ? p2k<NCC, AFFINE>(KP, L, a, pa, cap, nb)
                                            : p2k<NCC, DISP>(KP, L, a, pa, cap, nb);
    return param == AFFINE ? p2k<NGF, AFFINE>(KP, L, a, pa, cap, nb)
                           : p2k<NGF, DISP>(KP, L, a, pa, cap, nb);
  }
  static cudaError_t adjoint(int param, const Launch& L, const Args& a, const void* zb, long long zo,
                             long long zs, double* pa, size_t cap, int* nb) {
    const T* z = reinterpret_cast<const T*>(zb);
    return param == AFFINE ? run_ngf_adjoint<T, D, AFFINE>(L, a, z, zo, zs, pa, cap, nb)
                           : run_ngf_adjoint<T, D, DISP>(L, a, z, zo, zs, pa, cap, nb);
  }
  static cudaError_t curvature(const Launch& L, const Args& a, double alpha, double h, double* part,
                               size_t cap, int* nb) {
    return run_curvature<T, D>(L, a, alpha, h, part, cap, nb);
  }
  static cudaError_t sample(int param, const Launch& L, const Args& a, void* out) {
    const long long npix = a.pix_hi - a.pix_lo;
    if (npix <= 0) return cudaSuccess;
    const dim3 grid((unsigned)((npix + 255) / 256), (unsigned)a.K);
    if (param == AFFINE) k_sample_values<T, D, AFFINE><<<grid, 256, 0, L.stream>>>(a, reinterpret_cast<T*>(out));
    else k_sample_values<T, D, DISP><<<grid, 256, 0, L.stream>>>(a, reinterpret_cast<T*>(out));
    return cudaGetLastError();
  }
};

// Entry points implemented in inst_<dtype>_d<D>.cu
#define SR_DECLARE_INST(TT, DD)                                                               \
  cudaError_t pass1_##TT##_d##DD(int feat, int param, int KP, const Launch& L, const Args& a, \
                                 double* part, size_t cap, int* red);                        \
  cudaError_t pass2_##TT##_d##DD(int feat, int param, int KP, const Launch& L, const Args& a, \
                                 double* pa, size_t cap, int* nb);                           \
  cudaError_t adjoint_##TT##_d##DD(int param, const Launch& L, const Args& a, const void* zb, \
                                   long long zo, long long zs, double* pa, size_t cap, int* nb); \
  cudaError_t curvature_##TT##_d##DD(const Launch& L, const Args& a, double alpha, double h,  \
                                     double* part, size_t cap, int* nb);                     \
  cudaError_t sample_##TT##_d##DD(int param, const Launch& L, const Args& a, void* out);

#define SR_DEFINE_INST(TT, T, DD)                                                             \
  cudaError_t pass1_##TT##_d##DD(int feat, int param, int KP, const Launch& L, const Args& a, \
                                 double* part, size_t cap, int* red) {                       \
    return Dispatch<T, DD>::pass1(feat, param, KP, L, a, part, cap, red);                     \
  }                                                                                           \
  cudaError_t pass2_##TT##_d##DD(int feat, int param, int KP, const Launch& L, const Args& a, \
                                 double* pa, size_t cap, int* nb) {                          \
    return Dispatch<T, DD>::pass2(feat, param, KP, L, a, pa, cap, nb);                        \
  }                                                                                           \
  cudaError_t adjoint_##TT##_d##DD(int param, const Launch& L, const Args& a, const void* zb, \
                                   long long zo, long long zs, double* pa, size_t cap, int* nb) { \
    return Dispatch<T, DD>::adjoint(param, L, a, zb, zo, zs, pa, cap, nb);                    \
  }                                                                                           \
  cudaError_t curvature_##TT##_d##DD(const Launch& L, const Args& a, double alpha, double h,  \
                                     double* part, size_t cap, int* nb) {                     \
    return Dispatch<T, DD>::curvature(L, a, alpha, h, part, cap, nb);                         \
  }                                                                                           \
  cudaError_t sample_##TT##_d##DD(int param, const Launch& L, const Args& a, void* out) {     \
    return Dispatch<T, DD>::sample(param, L, a, out);                                         \
  }

SR_DECLARE_INST(f32, 2)
SR_DECLARE_INST(f32, 3)
SR_DECLARE_INST(f64, 2)
SR_DECLARE_INST(f64, 3)

}  // namespace sr

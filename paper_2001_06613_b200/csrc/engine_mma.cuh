// engine_mma.cuh — the fp32 NCC displacement-field path (K <= 32) with both K x K contractions on
// the warp-level tensor path (mma.sync tf32, 3xTF32), plus the K <= 32 NGF z contraction (f16):
//
//   k_gram_tma / k_gram_mma (pass 1b): the raw Gram G = sum_p V V^T of the sampled values V = v - shift
//                  (written by k_sample_vp, engine_tc.cuh) and the per-frame sum / max / min;
//                  TMA-fed (default) or register-fed.
//   k_pass2_tma / k_pass2_mma (pass 2): q = M'^T V + beta' for the pixels of a warp on the tensor
//                  cores (M' fragments in shared memory), dD/dy_j = q_j grad T_j (similarity.py:
//                  203-217 restated in DESIGN.md §3.3).  A pure stream: V, grad T in, dD/dy out.
//   k_ngf_z_f16    (split NGF pass 2, K <= 32): r = M'^T n, z = (r - n (n.r)) / rho.
//
// 3xTF32: x = hi + lo with hi = tf32(x), lo = x - hi; a.b ~ hi_a hi_b + lo_a hi_b + hi_a lo_b (the
// lo*lo term, 2^-22 relative, is dropped) — fp32-class products, fp32 accumulation inside a tile.
// The legacy tensor path runs ~270 TFLOP/s tf32 on B200 (scripts/probe_mma_sync.cu); each pass
// needs ~1.6 GFLOP at C2, on a pipe the sampling and streaming instructions do not use.
#pragma once
#include <cuda_fp16.h>

#include "engine.cuh"
#include "tma.cuh"

namespace sr {

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// m16n8k4 tf32: A = {(g, t), (g + 8, t)}, B = (k = t, n = g) — operands that ldmatrix.x4 delivers in
// place (no register moves to form operand pairs)
__device__ __forceinline__ void mma_tf32_k4(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(b0));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

// Split pass 1, Gram kernel (after k_sample_vp wrote V = v - shift as [K][vstride], mostly still in L2).
// Persistent CTAs over 128-pixel tiles.  Load: warp w reads rows 4w .. 4w+3 of the tile, lane l
// columns 4l .. 4l+3 (one 512-byte row per 128-bit load instruction); the next tile's rows are loaded
// before the current tile's MMAs.  Split: hi/lo tf32 halves stored row-major (row stride LD = 132
// words, conflict-free for the 128-bit stores and for ldmatrix), per-frame sum / max / min in
// registers.  MMA: warp = one m16 x n8 block of the 32 x 32 Gram; per 8-pixel k-step one ldmatrix.x4
// each for A hi, A lo and [B hi | B lo] (tf32 fragments read as b16 pairs), three HMMAs (3xTF32) on
// two alternating accumulator sets; fp32 per tile, fp64 across tiles.  Double-buffered hi/lo tiles:
// one CTA barrier per tile.
struct GMM {
  static constexpr int KP = 32, TP = 128, NT = 256, LD = TP + 4;
};
constexpr int GMM_LD = GMM::LD;

// One warp's share of a tile's Gram: the six m16 x n8 blocks on or above the diagonal of the 32 x 32
// Gram (block rows 0..15 x n-tiles 0..3, rows 16..31 x n-tiles 2..3; the two blocks strictly below
// are their mirror images), over 16 pixels (2 k-steps of 8).  Per k-step, ldmatrix.x4 of hi and lo
// rows 0..15 and 16..31 delivers {V[g][t], V[g+8][t], V[g][t+4], V[g+8][t+4]} of each 16-row block:
// the A operand of block row m, and (a0, a2) / (a1, a3) = the B operand of n-tile 2 m / 2 m + 1.
// (m16n8k4, whose operands the quad holds in place, measured slower — half the work per HMMA.)
__device__ __forceinline__ void gram_eighth(float (&acc)[6][4], uint32_t addr, uint32_t baddr) {
  constexpr uint32_t LDB = GMM_LD * 4, LOB = 2 * 32 * GMM_LD * 4;  // row bytes; hi -> lo offset
#pragma unroll
  for (int kq = 0; kq < 2; ++kq) {
    // A-order quads {V[g][t], V[g+8][t], V[g][t+4], V[g+8][t+4]} and B-order quads
    // {V[g][t], V[g][t+4], V[g+8][t], V[g+8][t+4]} (B of n-tile 2m = regs 0, 1; 2m + 1 = regs 2, 3):
    // two more ldmatrix per k-step instead of the register moves that would pair (a0, a2) / (a1, a3)
    uint32_t FH[2][4], FL[2][4], BH[2][4], BL[2][4];
#pragma unroll
    for (int m2 = 0; m2 < 2; ++m2) {
      ldsm_x4(FH[m2], addr + m2 * 16 * LDB + 32 * kq);
      ldsm_x4(FL[m2], addr + m2 * 16 * LDB + LOB + 32 * kq);
      ldsm_x4(BH[m2], baddr + m2 * 16 * LDB + 32 * kq);
      ldsm_x4(BL[m2], baddr + m2 * 16 * LDB + LOB + 32 * kq);
    }
    // block b: (m, n) = (0, 0..3), (1, 2), (1, 3)
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      const int m = b < 4 ? 0 : 1, n = b < 4 ? b : b - 2;
      mma_tf32(acc[b], FH[m], BH[n >> 1][2 * (n & 1)], BH[n >> 1][2 * (n & 1) + 1]);
    }
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      const int m = b < 4 ? 0 : 1, n = b < 4 ? b : b - 2;
      mma_tf32(acc[b], FL[m], BH[n >> 1][2 * (n & 1)], BH[n >> 1][2 * (n & 1) + 1]);
    }
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      const int m = b < 4 ? 0 : 1, n = b < 4 ? b : b - 2;
      mma_tf32(acc[b], FH[m], BL[n >> 1][2 * (n & 1)], BL[n >> 1][2 * (n & 1) + 1]);
    }
  }
}

__global__ void __launch_bounds__(GMM::NT, 2) k_gram_mma(const Args a, const float* __restrict__ V, long long vstride) {
  constexpr int KP = GMM::KP, TP = GMM::TP, LD = GMM::LD;
  extern __shared__ __align__(16) float gmm_smem[];
  float* Hs = gmm_smem;                // [2][KP * LD]
  float* Ls = gmm_smem + 2 * KP * LD;  // [2][KP * LD]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int K = a.K;
  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (npix + TP - 1) / TP;
  const int r0 = 4 * warp;  // this warp's load rows
  const bool vec = (vstride & 3) == 0 && (reinterpret_cast<uintptr_t>(V) & 15) == 0;
  float fsum[4], fmx[4], fmn[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    fsum[q] = 0.f;
    fmx[q] = -INFINITY;
    fmn[q] = INFINITY;
  }
  double gacc[6][4] = {};
  float acc[6][4] = {};
  int nt = 0;  // MMA role: the upper Gram blocks over pixel eighth `warp` (k-steps 2 warp, 2 warp + 1) of each tile
  // ldmatrix row addresses (bytes, buffer 0, rows 0.., k-step 0): lane L feeds row L & 7 of matrix L >> 3
  const int lr = lane & 7, lj = lane >> 3;
  const uint32_t sbase = smem_u32(gmm_smem);
  const uint32_t aoff = (uint32_t)(((lr + 8 * (lj & 1)) * LD + 4 * (lj >> 1)) * 4);  // A-order
  const uint32_t boff = (uint32_t)(((lr + 8 * (lj >> 1)) * LD + 4 * (lj & 1)) * 4);  // B-order
  // rows r0 .. r0+3, columns 4 lane .. 4 lane + 3 of tile `tile` (zero past K and past the slab)
  auto load = [&](long long tile, float4 (&x)[4]) {
    const long long c0 = tile * TP + 4 * lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + q;
      x[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < K) {
        const float* src = V + (long long)r * vstride + c0;
        if (vec && c0 + 3 < npix) {
          x[q] = __ldcg(reinterpret_cast<const float4*>(src));
        } else {
          if (c0 < npix) x[q].x = src[0];
          if (c0 + 1 < npix) x[q].y = src[1];
          if (c0 + 2 < npix) x[q].z = src[2];
          if (c0 + 3 < npix) x[q].w = src[3];
        }
      }
    }
  };
  float4 x[4];
  if ((long long)blockIdx.x < ntiles) load(blockIdx.x, x);
  int buf = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    const long long c0 = tile * TP + 4 * lane;
    float* H = Hs + buf * KP * LD;
    float* Lo = Ls + buf * KP * LD;
    // ---- split + stats
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + q;
      const float4 v = x[q];
      if (r < K) {
        fsum[q] += (v.x + v.y) + (v.z + v.w);
        if (c0 + 3 < npix) {
          fmx[q] = fmaxf(fmx[q], fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
          fmn[q] = fminf(fmn[q], fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
        } else {  // columns past the slab are zero-filled: exclude them from the extrema
          const float e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c0 + u < npix) {
              fmx[q] = fmaxf(fmx[q], e4[u]);
              fmn[q] = fminf(fmn[q], e4[u]);
            }
        }
      }
      const float4 hv = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
      *reinterpret_cast<float4*>(H + r * LD + 4 * lane) = hv;
      *reinterpret_cast<float4*>(Lo + r * LD + 4 * lane) = make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
    }
    __syncthreads();
    // ---- prefetch the next tile's rows, then the MMAs of this tile (gram_eighth)
    if (tile + gridDim.x < ntiles) load(tile + gridDim.x, x);
    const uint32_t bb = sbase + (uint32_t)(buf * KP * LD * 4);
    gram_eighth(acc, bb + aoff + (uint32_t)(64 * warp), bb + boff + (uint32_t)(64 * warp));
    ++nt;
    if ((nt & 7) == 0 || tile + gridDim.x >= ntiles) {  // fp32 over <= 8 tiles (128 pixels), fp64 across
#pragma unroll
      for (int b = 0; b < 6; ++b)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          gacc[b][r] += (double)acc[b][r];
          acc[b][r] = 0.f;
        }
    }
    // the next iteration writes the other buffer; the barrier after its split orders this buffer's reuse
  }
  // ---- CTA reduction over the eight pixel eighths (fixed order) through shared memory
  __syncthreads();
  double* red = reinterpret_cast<double*>(gmm_smem);  // [warp 8][block 6][r 4][lane 32]
#pragma unroll
  for (int b = 0; b < 6; ++b)
#pragma unroll
    for (int r = 0; r < 4; ++r) red[((warp * 6 + b) * 4 + r) * 32 + lane] = gacc[b][r];
  __syncthreads();
  double* out = a.part + (size_t)blockIdx.x * (KP * KP + 3 * KP);
  for (int e = tid; e < 6 * 4 * 32; e += GMM::NT) {
    double v = red[e];
#pragma unroll
    for (int w2 = 1; w2 < 8; ++w2) v += red[w2 * 6 * 4 * 32 + e];
    const int b = e >> 7, r = (e >> 5) & 3, ln = e & 31;
    const int m = b < 4 ? 0 : 1, n = b < 4 ? b : b - 2;
    const int i = 16 * m + (ln >> 2) + 8 * (r >> 1), j = 8 * n + 2 * (ln & 3) + (r & 1);
    out[i * KP + j] = v;
    if (j >= 16 && i < 16) out[j * KP + i] = v;  // mirror of the strictly-upper blocks (0, 2), (0, 3)
  }
  const float* shifts = reinterpret_cast<const float*>(a.shifts);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = r0 + q;
    double s = (double)fsum[q];
    float mx = fmx[q], mn = fmn[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
      const double sh = (k < K && shifts) ? (double)shifts[a.job->frame_index[k]] : 0.0;
      out[KP * KP + k] = k < K ? s : 0.0;
      out[KP * KP + KP + k] = (double)mx + sh;
      out[KP * KP + 2 * KP + k] = -((double)mn + sh);
    }
  }
}

__device__ __forceinline__ void stsm_x4(uint32_t addr, float c0, float c1, float c2, float c3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "r"(__float_as_uint(c0)),
               "r"(__float_as_uint(c1)), "r"(__float_as_uint(c2)), "r"(__float_as_uint(c3))
               : "memory");
}

// Split pass 1, Gram kernel, TMA-fed (default): persistent CTAs over 128-pixel tiles; one thread
// streams [32 frames x 32 pixels] boxes of V (SWIZZLE_128B, zero fill past K and past the slab) into an
// NST-stage ring (full: TMA transaction barrier, empty: one arrival per warp), so NST tiles are in
// flight per CTA and no thread holds in-flight data.  Warp w owns pixels 16 w .. 16 w + 15 of every
// tile (2 k-steps): ldmatrix.x4 of the raw fp32 rows in A order {V[g][t], V[g+8][t], V[g][t+4],
// V[g+8][t+4]} and in B order {V[g][t], V[g][t+4], V[g+8][t], V[g+8][t+4]}, hi/lo split in registers,
// the six upper m16n8 blocks with 3 HMMAs each (fp32 per <= 8 tiles, fp64 across), per-frame sum /
// max / min from the A-order fragments (every element lies in exactly one of them).
struct GTM {
  static constexpr int KP = 32, TP = 128, NT = 256, NST = 3, BOXP = 32;
  static constexpr int SBYTES = KP * TP * 4;          // one stage: 4 boxes of [32 rows x 128 B]
  static constexpr int ABYTES = 8 * 6 * 4 * 32 * 8;  // fp64 Gram accumulators [warp][block][r][lane]
};
constexpr size_t gtm_smem(int sup = 1) {
  return 1024 + (size_t)GTM::NST * GTM::SBYTES * sup + 256 + (size_t)GTM::ABYTES * sup;
}

// hi = v with the 13 low mantissa bits cleared (exact in tf32; one LOP3 instead of the ~4-instruction
// cvt.rna), lo = v - hi exactly (|lo| < 2^-10 |v|, truncated to tf32 by the MMA: 2^-20 relative).
__device__ __forceinline__ void split_q(const uint32_t (&q)[4], uint32_t (&h)[4], uint32_t (&l)[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    h[u] = q[u] & 0xffffe000u;
    l[u] = __float_as_uint(__uint_as_float(q[u]) - __uint_as_float(h[u]));
  }
}

// NGF: the same Gram over the feature array n [K][ncomp][zstride] (rows = frames, columns = (component,
// pixel) tiles of a 3-D map); the statistics slots then carry max |n| (the NGF degeneracy threshold).
// SUP: tiles per ring stage (CTA of 8 SUP warps, warp w on tile w >> 3 of the stage); the launcher uses
// SUP = 1 (two 8-warp CTAs per SM; one 16-warp CTA measured 15.3 vs 13.7 us at C2).
template <bool NGF, int SUP = 1>
__global__ void __launch_bounds__(GTM::NT * SUP, SUP == 1 ? 2 : 1) k_gram_tma(const Args a,
                                                                             const __grid_constant__ CUtensorMap vmap,
                                                                             int ntx) {
  constexpr int KP = GTM::KP, TP = GTM::TP, NST = GTM::NST, NTT = GTM::NT * SUP, NW = NTT / 32;
  constexpr int SB = GTM::SBYTES * SUP;  // one stage
  extern __shared__ __align__(1024) unsigned char gtm_sh[];
  unsigned char* base = gtm_sh + ((1024 - (smem_u32(gtm_sh) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)NST * SB);
  uint64_t* empty = full + NST;
  // fp64 accumulators in shared memory (not registers): [warp NW][block 6][r 4][lane 32]
  double* gsm = reinterpret_cast<double*>(base + (size_t)NST * SB + 256);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int K = a.K;
  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (long long)ntx * (NGF ? a.g.nd : 1);  // tile t: component t / ntx, x-tile t % ntx
  const long long nsup = (ntiles + SUP - 1) / SUP;                // stage-sized groups of SUP tiles
  const long long nloc = nsup > blockIdx.x ? (nsup - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int sub = warp >> 3, wl = warp & 7;  // this warp's tile in the stage and pixel slice of it
  if (tid == 0) {
    for (int s2 = 0; s2 < NST; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], NW);
    }
    fence_mbar_init();
    tma_prefetch_desc(&vmap);
  }
  pdl_wait();  // V of the sampling kernel
  pdl_trigger();
  __syncthreads();
  auto issue = [&](long long n, int s2) {  // tiles past the end load as zeros (out-of-range coordinates)
    unsigned char* st = base + (size_t)s2 * SB;
    mbar_arrive_expect_tx(&full[s2], (uint32_t)SB);
#pragma unroll
    for (int u = 0; u < SUP; ++u) {
      const long long tt = (blockIdx.x + n * gridDim.x) * SUP + u;
      const int x0 = (int)(tt % ntx) * TP, c = (int)(tt / ntx);
#pragma unroll
      for (int b = 0; b < TP / GTM::BOXP; ++b)
        tma_load_3d(st + u * GTM::SBYTES + b * 4096, &vmap, x0 + GTM::BOXP * b, c, 0, &full[s2]);
    }
  };
  if (tid == 0)
    for (long long n = 0; n < nloc && n < NST; ++n) issue(n, (int)n);
  // this warp's ldmatrix row addresses inside a stage: tile sub, box wl >> 1, pixel columns 16 (wl & 1) + 8 kq
  const int lr = lane & 7, lj = lane >> 3;
  uint32_t aadr[2][2], badr[2][2];  // [m][kq], swizzled (16-byte chunk ^ (row & 7))
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int kq = 0; kq < 2; ++kq) {
      const int c = 16 * (wl & 1) + 8 * kq;
      const int ra = 16 * m + lr + 8 * (lj & 1), ca = c + 4 * (lj >> 1);
      const int rb = 16 * m + lr + 8 * (lj >> 1), cb = c + 4 * (lj & 1);
      aadr[m][kq] = (uint32_t)(sub * GTM::SBYTES + (wl >> 1) * 4096 + ra * 128 + (((ca >> 2) ^ (ra & 7)) << 4));
      badr[m][kq] = (uint32_t)(sub * GTM::SBYTES + (wl >> 1) * 4096 + rb * 128 + (((cb >> 2) ^ (rb & 7)) << 4));
    }
  const uint32_t sb = smem_u32(base);
  float acc[6][4] = {};
  double* ga = gsm + warp * 6 * 4 * 32 + lane;  // this lane's accumulators, stride 32
#pragma unroll
  for (int e = 0; e < 24; ++e) ga[e * 32] = 0.0;
  float fs[2][2] = {}, fmx[2][2], fmn[2][2];  // [m][h]: rows 16 m + g + 8 h
  double ds[2][2] = {};
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      fmx[m][h] = -INFINITY;
      fmn[m][h] = INFINITY;
    }
  for (long long n = 0; n < nloc; ++n) {
    const int s2 = (int)(n % NST);
    const uint32_t st = sb + (uint32_t)(s2 * SB);
    const long long tt = (blockIdx.x + n * gridDim.x) * SUP + sub;
    // this warp's first pixel (npix for a tile past the end: every pixel masked)
    const long long p0 = tt < ntiles ? (tt % ntx) * TP + 16 * wl : npix;
    mbar_wait(&full[s2], (uint32_t)((n / NST) & 1));
    uint32_t QA[2][2][4], QB[2][2][4];
#pragma unroll
    for (int kq = 0; kq < 2; ++kq)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        ldsm_x4(QA[kq][m], st + aadr[m][kq]);
        ldsm_x4(QB[kq][m], st + badr[m][kq]);
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s2]);
    if (tid == 0 && n + NST < nloc) {  // refill this stage once every warp has read it
      mbar_wait(&empty[s2], (uint32_t)((n / NST) & 1));
      issue(n + NST, s2);
    }
#pragma unroll
    for (int kq = 0; kq < 2; ++kq) {
      // per-frame statistics from the A-order fragments: rows 16 m + g (+ 8), pixels p0 + 8 kq + t (+ 4)
      const long long pc = p0 + 8 * kq + t;
      if (p0 + 16 <= npix) {  // warp-uniform: every pixel of this warp's slice is inside the slab
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float v0 = __uint_as_float(QA[kq][m][h]), v1 = __uint_as_float(QA[kq][m][2 + h]);
            fs[m][h] += v0 + v1;
            fmx[m][h] = fmaxf(fmx[m][h], fmaxf(v0, v1));
            fmn[m][h] = fminf(fmn[m][h], fminf(v0, v1));
          }
      } else {
        const bool ok0 = pc < npix, ok1 = pc + 4 < npix;
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float v0 = __uint_as_float(QA[kq][m][h]), v1 = __uint_as_float(QA[kq][m][2 + h]);
            fs[m][h] += v0 + v1;  // zero past the slab
            if (ok0) {
              fmx[m][h] = fmaxf(fmx[m][h], v0);
              fmn[m][h] = fminf(fmn[m][h], v0);
            }
            if (ok1) {
              fmx[m][h] = fmaxf(fmx[m][h], v1);
              fmn[m][h] = fminf(fmn[m][h], v1);
            }
          }
      }
      uint32_t AH[2][4], AL[2][4], BH[2][4], BL[2][4];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        split_q(QA[kq][m], AH[m], AL[m]);
        split_q(QB[kq][m], BH[m], BL[m]);
      }
      // block b: (m, n) = (0, 0..3), (1, 2), (1, 3); B of n-tile nn = BX[nn >> 1][2 (nn & 1) + 0, 1]
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        const int m = b < 4 ? 0 : 1, nn = b < 4 ? b : b - 2;
        mma_tf32(acc[b], AH[m], BH[nn >> 1][2 * (nn & 1)], BH[nn >> 1][2 * (nn & 1) + 1]);
      }
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        const int m = b < 4 ? 0 : 1, nn = b < 4 ? b : b - 2;
        mma_tf32(acc[b], AL[m], BH[nn >> 1][2 * (nn & 1)], BH[nn >> 1][2 * (nn & 1) + 1]);
      }
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        const int m = b < 4 ? 0 : 1, nn = b < 4 ? b : b - 2;
        mma_tf32(acc[b], AH[m], BL[nn >> 1][2 * (nn & 1)], BL[nn >> 1][2 * (nn & 1) + 1]);
      }
    }
    if ((n & 7) == 7 || n == nloc - 1) {  // fp32 over <= 8 tiles (128 pixels per warp), fp64 across
#pragma unroll
      for (int b = 0; b < 6; ++b)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          ga[(b * 4 + r) * 32] += (double)acc[b][r];
          acc[b][r] = 0.f;
        }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          ds[m][h] += (double)fs[m][h];
          fs[m][h] = 0.f;
        }
    }
  }
  // ---- CTA reduction (fixed order) through shared memory (the stages are no longer in use)
  __syncthreads();
  const double* red = gsm;  // [warp 8][block 6][r 4][lane 32]
  // per-frame stats: reduce over the 4 lanes t of a row (xor tree), then over warps in smem
  double* rs = reinterpret_cast<double*>(base);  // [warp 8][row 32] x {sum, max, -min} (ring area)
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double sv = ds[m][h];
      float mx = fmx[m][h], mn = fmn[m][h];
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        sv += __shfl_xor_sync(0xffffffffu, sv, o);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      if (t == 0) {
        const int row = 16 * m + g + 8 * h;
        rs[(warp * 32 + row) * 3 + 0] = sv;
        rs[(warp * 32 + row) * 3 + 1] = (double)mx;
        rs[(warp * 32 + row) * 3 + 2] = (double)mn;
      }
    }
  __syncthreads();
  double* out = a.part + (size_t)blockIdx.x * (KP * KP + 3 * KP);
  for (int e = tid; e < 6 * 4 * 32; e += NTT) {
    double v = red[e];
#pragma unroll
    for (int w2 = 1; w2 < NW; ++w2) v += red[w2 * 6 * 4 * 32 + e];
    const int b = e >> 7, r = (e >> 5) & 3, ln = e & 31;
    const int m = b < 4 ? 0 : 1, nn = b < 4 ? b : b - 2;
    const int i = 16 * m + (ln >> 2) + 8 * (r >> 1), j = 8 * nn + 2 * (ln & 3) + (r & 1);
    out[i * KP + j] = v;
    if (j >= 16 && i < 16) out[j * KP + i] = v;  // mirror of the strictly-upper blocks (0, 2), (0, 3)
  }
  if (tid < KP) {
    const int k = tid;
    double sv = 0.0, mx = -INFINITY, mn = INFINITY;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) {
      sv += rs[(w2 * 32 + k) * 3 + 0];
      mx = fmax(mx, rs[(w2 * 32 + k) * 3 + 1]);
      mn = fmin(mn, rs[(w2 * 32 + k) * 3 + 2]);
    }
    if (NGF) {  // k_gram_h's layout: s unused, both extremum slots = max |n| (0 when no pixel)
      const double am = k < K && mx >= mn ? fmax(mx, -mn) : 0.0;
      out[KP * KP + k] = 0.0;
      out[KP * KP + KP + k] = am;
      out[KP * KP + 2 * KP + k] = am;
      return;
    }
    const float* shifts = reinterpret_cast<const float*>(a.shifts);
    const double sh = (k < K && shifts) ? (double)shifts[a.job->frame_index[k]] : 0.0;
    out[KP * KP + k] = k < K ? sv : 0.0;
    out[KP * KP + KP + k] = mx + sh;
    out[KP * KP + 2 * KP + k] = -(mn + sh);
  }
}

// Pass 2 (streaming, after a split pass 1 on the same y; default).  Warp = 8 consecutive pixels per
// step, all 32 output frames, Q^T = M'^T V + beta' on the tensor cores: A = M'^T (m = frame j, k =
// frame i; hi/lo fragments from shared memory), B = V (k = frame i, n = pixel; fragments straight
// from global, every V element loaded once), C initialised with beta'.  A lane's outputs are two
// adjacent pixels of frames j = 16 m + g (+ 8): grad T is read and dD/dy written as float2 (full
// 32-byte sectors).  All of a step's loads are issued before its MMAs.
// Measured alternatives (C2, 34 us for this kernel): 32-pixel warp blocks staged through shared memory
// with coalesced 128-bit loads and a stmatrix epilogue (48.6 us: two exposed latencies per block at 24
// warps/SM), and the same math fed by per-warp two-stage 1-D bulk-copy pipelines (k_pass2_bulk, 41.8 us).
struct P2M {
  static constexpr int KP = 32, NT = 256, PW = 16;
};

template <int D, int MINB>
__global__ void __launch_bounds__(P2M::NT, MINB) k_pass2_mma(const Args a, const float* __restrict__ V,
                                                          const float* __restrict__ G, long long vstride) {
  // A fragments: [mtile 2][kstep 4][lane 32] x {hi a0..a3} and {lo a0..a3}
  __shared__ __align__(16) float4 Ah[2 * 4 * 32], Al[2 * 4 * 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int K = a.K;
  const StatsLayout L(K);
  const double* Md = a.stats + L.M;
  pdl_wait();  // M', beta' of the finalize
  for (int e = tid; e < 2 * 4 * 32; e += P2M::NT) {
    const int m = e >> 7, ks = (e >> 5) & 3, ln = e & 31;
    const int gg = ln >> 2, tt = ln & 3;
    float hv[4], lv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {  // a0 (g, t), a1 (g + 8, t), a2 (g, t + 4), a3 (g + 8, t + 4); A[j][i] = M'[i][j]
      const int j = 16 * m + gg + 8 * (r & 1), i = 8 * ks + tt + 4 * (r >> 1);
      const double mv = (i < K && j < K) ? Md[i * K + j] : 0.0;
      hv[r] = to_tf32((float)mv);
      lv[r] = (float)(mv - (double)hv[r]);
    }
    Ah[e] = make_float4(hv[0], hv[1], hv[2], hv[3]);
    Al[e] = make_float4(lv[0], lv[1], lv[2], lv[3]);
  }
  __syncthreads();
  float bet[2][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = 16 * m + g + 8 * h;
      bet[m][h] = j < K ? (float)a.stats[L.beta + j] : 0.f;
    }
  // 32-bit element offsets: the launcher guarantees K D vstride and K D o_stride < 2^31
  const int npix = (int)(a.pix_hi - a.pix_lo);
  const int nblk = (npix + P2M::PW - 1) / P2M::PW;
  const int vs = (int)vstride, os = (int)a.o_stride;
  const uint64_t pol = l2_policy_evict_first();
  float* __restrict__ ob = reinterpret_cast<float*>(a.out) + (a.pix_lo - a.o_off);
  // 128-bit accesses need 16-byte aligned rows (else the scalar paths)
  const bool vin = (vs & 3) == 0 && (reinterpret_cast<uintptr_t>(G) & 15) == 0;
  const bool vout = (os & 3) == 0 && (reinterpret_cast<uintptr_t>(ob) & 15) == 0;
  for (int blk = blockIdx.x * (P2M::NT / 32) + warp; blk < nblk; blk += gridDim.x * (P2M::NT / 32)) {
    const int p0 = blk * P2M::PW;
    const bool fullb = p0 + P2M::PW <= npix;
    // B column g of n-tile nt carries pixel 4 (g >> 1) + 2 nt + (g & 1), so that the C fragments of a
    // lane (columns 2t, 2t + 1 of both n-tiles) are the 4 consecutive pixels p0 + 4t .. p0 + 4t + 3
    float bv[4][2][2];  // [ks][nt][u]: V[8 ks + t + 4 u][p0 + pixel(g, nt)]
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int pg = p0 + 4 * (g >> 1) + 2 * nt + (g & 1);
      const bool okg = pg < npix;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i = 8 * ks + t + 4 * u;
          bv[ks][nt][u] = (i < K && okg) ? ldg_hint_nv(V + (i * vs + pg), pol) : 0.f;
        }
    }
    // grad T of this lane's outputs: frames 16 m + g + 8 h, pixels p0 + 4t .. + 3 (one 128-bit load)
    const int pq = p0 + 4 * t;
    auto load_g = [&](int m, int h, int c) {
      const int j = min(16 * m + g + 8 * h, K - 1);
      const float* src = G + ((j * D + c) * vs + pq);
      float4 r;
      if (fullb && vin) {
        r = __ldcs(reinterpret_cast<const float4*>(src));
      } else {
        r.x = pq < npix ? src[0] : 0.f;
        r.y = pq + 1 < npix ? src[1] : 0.f;
        r.z = pq + 2 < npix ? src[2] : 0.f;
        r.w = pq + 3 < npix ? src[3] : 0.f;
      }
      return r;
    };
    // MINB <= 2: all of the step's grad T loads are issued before the MMAs (128 registers, 16 warps/SM);
    // MINB >= 3: loaded in the epilogue (fewer registers, more warps to hide the latency)
    float4 gv[2][2][D];
    if constexpr (MINB <= 2) {
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < D; ++c) gv[m][h][c] = load_g(m, h, c);
    }
    float acc[2][2][4];  // [m][nt]: four independent accumulator chains (beta' + HH + LH + HL)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        acc[m][nt][0] = acc[m][nt][1] = bet[m][0];
        acc[m][nt][2] = acc[m][nt][3] = bet[m][1];
      }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t bh[2][2], bl[2][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {  // hi by truncation (exact in tf32), lo = v - hi exactly (see split_q)
          bh[nt][u] = __float_as_uint(bv[ks][nt][u]) & 0xffffe000u;
          bl[nt][u] = __float_as_uint(bv[ks][nt][u] - __uint_as_float(bh[nt][u]));
        }
      uint32_t AH[2][4], AL[2][4];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const float4 ah = Ah[(m * 4 + ks) * 32 + lane], al = Al[(m * 4 + ks) * 32 + lane];
        AH[m][0] = __float_as_uint(ah.x), AH[m][1] = __float_as_uint(ah.y);
        AH[m][2] = __float_as_uint(ah.z), AH[m][3] = __float_as_uint(ah.w);
        AL[m][0] = __float_as_uint(al.x), AL[m][1] = __float_as_uint(al.y);
        AL[m][2] = __float_as_uint(al.z), AL[m][3] = __float_as_uint(al.w);
      }
      // one product at a time over the four (m, n-tile) accumulators: consecutive HMMAs are independent
#pragma unroll
      for (int mn = 0; mn < 4; ++mn) mma_tf32(acc[mn >> 1][mn & 1], AH[mn >> 1], bh[mn & 1][0], bh[mn & 1][1]);
#pragma unroll
      for (int mn = 0; mn < 4; ++mn) mma_tf32(acc[mn >> 1][mn & 1], AL[mn >> 1], bh[mn & 1][0], bh[mn & 1][1]);
#pragma unroll
      for (int mn = 0; mn < 4; ++mn) mma_tf32(acc[mn >> 1][mn & 1], AH[mn >> 1], bl[mn & 1][0], bl[mn & 1][1]);
    }
    // epilogue: acc[m][nt][2h + u] = q_j(p0 + 4t + 2 nt + u), j = 16 m + g + 8 h; one 128-bit store per (j, c)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 16 * m + g + 8 * h;
        if (j < K) {
          const float q0 = acc[m][0][2 * h], q1 = acc[m][0][2 * h + 1];
          const float q2 = acc[m][1][2 * h], q3 = acc[m][1][2 * h + 1];
#pragma unroll
          for (int c = 0; c < D; ++c) {
            float* dst = ob + ((j * D + c) * os + pq);
            const float4 gg = MINB <= 2 ? gv[m][h][c] : load_g(m, h, c);
            const float4 r = make_float4(q0 * gg.x, q1 * gg.y, q2 * gg.z, q3 * gg.w);
            if (fullb && vout) {
              __stcs(reinterpret_cast<float4*>(dst), r);
            } else {
              if (pq < npix) __stcs(dst, r.x);
              if (pq + 1 < npix) __stcs(dst + 1, r.y);
              if (pq + 2 < npix) __stcs(dst + 2, r.z);
              if (pq + 3 < npix) __stcs(dst + 3, r.w);
            }
          }
        }
      }
  }
}


// Pass 2, TMA-fed (fp32 NCC displacement, K <= 32): the math and lane layout of k_pass2_mma, but the
// tile's V rows ([32 frames x 128 pixels]) and grad T rows ([32 D rows x 128 pixels]) arrive by 3-D TMA
// (SWIZZLE_128B boxes of 32 pixels, zero fill past K and past the slab) into a 2-stage ring, so the next
// tile is in flight while this one is contracted and no register holds in-flight data.
template <int D>
struct P2T {
  static constexpr int NT = 256, TP = 128, NST = 2;
  static constexpr int VB = 32 * 32 * 4, GB = 32 * D * 32 * 4;     // one V box, one grad T box
  static constexpr int SBYTES = 4 * VB + 4 * GB;                    // one stage
  static constexpr size_t smem() { return 1024 + (size_t)NST * SBYTES + 256 + 2 * 2 * 4 * 32 * 16; }
};

template <int D>
__global__ void __launch_bounds__(P2T<D>::NT, D == 2 ? 2 : 1) k_pass2_tma(const Args a, const __grid_constant__ CUtensorMap vmap,
                                                            const __grid_constant__ CUtensorMap gmap) {
  using C = P2T<D>;
  constexpr int NST = C::NST, TP = C::TP;
  extern __shared__ __align__(1024) unsigned char p2t_sh[];
  unsigned char* base = p2t_sh + ((1024 - (smem_u32(p2t_sh) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)NST * C::SBYTES);
  uint64_t* empty = full + NST;
  float4* Ah = reinterpret_cast<float4*>(base + (size_t)NST * C::SBYTES + 256);  // [m 2][ks 4][lane 32]
  float4* Al = Ah + 2 * 4 * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int K = a.K;
  const StatsLayout L(K);
  const double* Md = a.stats + L.M;
  const int npix = (int)(a.pix_hi - a.pix_lo);
  const int ntiles = (npix + TP - 1) / TP;
  const int nloc = ntiles > (int)blockIdx.x ? (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  if (tid == 0) {
    for (int s2 = 0; s2 < NST; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], C::NT / 32);
    }
    fence_mbar_init();
    tma_prefetch_desc(&vmap);
    tma_prefetch_desc(&gmap);
  }
  auto issue = [&](int n, int s2) {
    const int x0 = ((int)blockIdx.x + n * (int)gridDim.x) * TP;
    unsigned char* st = base + (size_t)s2 * C::SBYTES;
    mbar_arrive_expect_tx(&full[s2], (uint32_t)C::SBYTES);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      tma_load_3d(st + b * C::VB, &vmap, x0 + 32 * b, 0, 0, &full[s2]);
      tma_load_3d(st + 4 * C::VB + b * C::GB, &gmap, x0 + 32 * b, 0, 0, &full[s2]);
    }
  };
  for (int e = tid; e < 2 * 4 * 32; e += C::NT) {
    const int m = e >> 7, ks = (e >> 5) & 3, ln = e & 31;
    const int gg = ln >> 2, tt = ln & 3;
    float hv[4], lv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {  // A[j][i] = M'[i][j]
      const int j = 16 * m + gg + 8 * (r & 1), i = 8 * ks + tt + 4 * (r >> 1);
      const double mv = (i < K && j < K) ? Md[i * K + j] : 0.0;
      hv[r] = to_tf32((float)mv);
      lv[r] = (float)(mv - (double)hv[r]);
    }
    Ah[e] = make_float4(hv[0], hv[1], hv[2], hv[3]);
    Al[e] = make_float4(lv[0], lv[1], lv[2], lv[3]);
  }
  __syncthreads();
  if (tid == 0)
    for (int n = 0; n < nloc && n < NST; ++n) issue(n, n);
  float bet[2][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = 16 * m + g + 8 * h;
      bet[m][h] = j < K ? (float)a.stats[L.beta + j] : 0.f;
    }
  const int os = (int)a.o_stride;
  float* __restrict__ ob = reinterpret_cast<float*>(a.out) + (a.pix_lo - a.o_off);
  const bool vout = (os & 3) == 0 && (reinterpret_cast<uintptr_t>(ob) & 15) == 0;
  const int bx = warp >> 1, half = warp & 1;  // this warp's box and 16-pixel half of it
  const int pq_in = 16 * half + 4 * t;        // this lane's first output pixel inside the box
  for (int n = 0; n < nloc; ++n) {
    const int s2 = n % NST;
    const unsigned char* st = base + (size_t)s2 * C::SBYTES;
    const unsigned char* vbx = st + bx * C::VB;
    const unsigned char* gbx = st + 4 * C::VB + bx * C::GB;
    const int p0 = ((int)blockIdx.x + n * (int)gridDim.x) * TP + 16 * warp;  // this warp's first pixel
    mbar_wait(&full[s2], (uint32_t)((n / NST) & 1));
    // B fragments: V[8 ks + t + 4u][pixel(g, nt)], pixel(g, nt) = 4 (g >> 1) + 2 nt + (g & 1)
    float bv[4][2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int px = 16 * half + 4 * (g >> 1) + 2 * nt + (g & 1);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int r = 8 * ks + t + 4 * u;
          bv[ks][nt][u] = *reinterpret_cast<const float*>(vbx + r * 128 + ((((px >> 2) ^ (r & 7))) << 4) + (px & 3) * 4);
        }
    }
    // grad T rows (16 m + g + 8 h) D + c, pixels pq_in .. + 3 of the box
    float4 gv[2][2][D];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const int r = (16 * m + g + 8 * h) * D + c;
          gv[m][h][c] = *reinterpret_cast<const float4*>(gbx + r * 128 + ((((pq_in >> 2) ^ (r & 7))) << 4));
        }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s2]);
    if (tid == 0 && n + NST < nloc) {  // refill once every warp has read the stage
      mbar_wait(&empty[s2], (uint32_t)((n / NST) & 1));
      issue(n + NST, s2);
    }
    float acc[2][2][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        acc[m][nt][0] = acc[m][nt][1] = bet[m][0];
        acc[m][nt][2] = acc[m][nt][3] = bet[m][1];
      }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t bh[2][2], bl[2][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          bh[nt][u] = __float_as_uint(bv[ks][nt][u]) & 0xffffe000u;
          bl[nt][u] = __float_as_uint(bv[ks][nt][u] - __uint_as_float(bh[nt][u]));
        }
      uint32_t AH[2][4], AL[2][4];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const float4 ah = Ah[(m * 4 + ks) * 32 + lane], al = Al[(m * 4 + ks) * 32 + lane];
        AH[m][0] = __float_as_uint(ah.x), AH[m][1] = __float_as_uint(ah.y);
        AH[m][2] = __float_as_uint(ah.z), AH[m][3] = __float_as_uint(ah.w);
        AL[m][0] = __float_as_uint(al.x), AL[m][1] = __float_as_uint(al.y);
        AL[m][2] = __float_as_uint(al.z), AL[m][3] = __float_as_uint(al.w);
      }
#pragma unroll
      for (int mn = 0; mn < 4; ++mn) mma_tf32(acc[mn >> 1][mn & 1], AH[mn >> 1], bh[mn & 1][0], bh[mn & 1][1]);
#pragma unroll
      for (int mn = 0; mn < 4; ++mn) mma_tf32(acc[mn >> 1][mn & 1], AL[mn >> 1], bh[mn & 1][0], bh[mn & 1][1]);
#pragma unroll
      for (int mn = 0; mn < 4; ++mn) mma_tf32(acc[mn >> 1][mn & 1], AH[mn >> 1], bl[mn & 1][0], bl[mn & 1][1]);
    }
    const int pq = p0 + 4 * t;
    const bool fullb = p0 + 16 <= npix;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 16 * m + g + 8 * h;
        if (j < K) {
          const float q0 = acc[m][0][2 * h], q1 = acc[m][0][2 * h + 1];
          const float q2 = acc[m][1][2 * h], q3 = acc[m][1][2 * h + 1];
#pragma unroll
          for (int c = 0; c < D; ++c) {
            float* dst = ob + ((j * D + c) * os + pq);
            const float4 gg = gv[m][h][c];
            const float4 r = make_float4(q0 * gg.x, q1 * gg.y, q2 * gg.z, q3 * gg.w);
            if (fullb && vout) {
              __stcs(reinterpret_cast<float4*>(dst), r);
            } else {
              if (pq < npix) __stcs(dst, r.x);
              if (pq + 1 < npix) __stcs(dst + 1, r.y);
              if (pq + 2 < npix) __stcs(dst + 2, r.z);
              if (pq + 3 < npix) __stcs(dst + 3, r.w);
            }
          }
        }
      }
  }
}

// Split NGF pass 2, z = dD/d(grad u) on the tensor cores (fp32 displacement fields, K <= 128):
//   R^T = M'^T N: A = M'^T (m = frame j, k = frame i; hi/lo fragments for every (m-tile, k-step) staged
//   once per persistent CTA in shared memory), B = N (k = frame i, n = (component, pixel); fragments
//   straight from global, each n element loaded once per warp item), 3xTF32, fp32 accumulation.
//   B column g of the n-tile pair q of component c carries pixel 4 (g >> 1) + 2 q + (g & 1), so a lane
//   owns 4 consecutive pixels of rows j = 16 m + g (+ 8) for every component: the epilogue
//   z_(j,c) = (r_(j,c) - n_(j,c) sum_c' n_(j,c') r_(j,c')) / rho_j (the k_ngf_z arithmetic) reads n and
//   rho and writes z with 128-bit accesses.
// Work item = (16-pixel block of [zlo, zhi), group of MW m-tiles); warps stride over items.
template <int D>
struct NZ {
  static constexpr int NT = 512, PW = 16, MW = D == 2 ? 4 : 2, NTL = 2 * D;  // n-tiles per item
};

__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// (x0, x1) -> packed f16 hi and lo halves: hi = f16(x), lo = f16(x - hi) (x ~ hi + lo to 2^-22 relative)
__device__ __forceinline__ void split_h2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// The K x K contraction of split NGF pass 2 for K <= 32 (k_ngf_z_tc above 32): the legacy tensor path runs m16n8k16 f16 at twice the
// tf32 rate (scripts/probe_mma_sync.cu), so each product takes 3 f16 HMMAs per 16 frames instead of per 8.
// 2-way split: x = hi + lo, hi = f16(x), lo = f16(x - hi): 22 significant bits, products exact in the
// fp32 accumulator, a.b ~ hi hi + lo hi + hi lo.  n is in [-1, 1] (normalised gradients); M' is scaled by
// 2^s (max |M'| 2^s in [2^13, 2^14), exact) so that it sits in the f16 normal range, and r = acc 2^-s.
template <int D>
__global__ void __launch_bounds__(NZ<D>::NT, 1) k_ngf_z_f16(const Args a, const float* __restrict__ Nf,
                                                           const float* __restrict__ Rho, long long zlo,
                                                           long long zhi, long long zstride, float* __restrict__ Z) {
  using C = NZ<D>;
  constexpr int MW = C::MW, NTL = C::NTL, PW = C::PW;
  extern __shared__ __align__(16) uint4 nzh_sh[];
  __shared__ float red_max[32];
  const int K = a.K;
  const int KS = (K + 15) / 16, JT = (K + 15) / 16;  // k-steps of 16 frames, m-tiles
  uint4* Ah = nzh_sh;                 // [JT][KS][32] packed hi {a0..a3}
  uint4* Al = nzh_sh + JT * KS * 32;  // lo
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const StatsLayout L(K);
  const double* Md = a.stats + L.M;
  // scale: 2^s with max |M'| 2^s in [2^13, 2^14)
  float mx = 0.f;
  for (int e = tid; e < K * K; e += C::NT) mx = fmaxf(mx, fabsf((float)Md[e]));
  mx = warp_max(mx);
  if (lane == 0) red_max[warp] = mx;
  __syncthreads();
  if (warp == 0) {
    float v = lane < C::NT / 32 ? red_max[lane] : 0.f;
    v = warp_max(v);
    if (lane == 0) red_max[0] = v;
  }
  __syncthreads();
  const float mmax = red_max[0];
  const int sexp = mmax > 0.f ? 13 - ilogbf(mmax) : 0;
  const float scale = ldexpf(1.f, sexp), unscale = ldexpf(1.f, -sexp);
  for (int e = tid; e < JT * KS * 32; e += C::NT) {
    const int m = e / (KS * 32), ks = (e / 32) % KS, ln = e & 31;
    const int gg = ln >> 2, tt = ln & 3;
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {  // a_r = (row g + 8 (r & 1), frames 16 ks + 2t + 8 (r >> 1) + {0, 1}); A[j][i] = M'[i][j]
      const int j = 16 * m + gg + 8 * (r & 1), i = 16 * ks + 2 * tt + 8 * (r >> 1);
      const float m0 = (i < K && j < K) ? (float)Md[i * K + j] * scale : 0.f;
      const float m1 = (i + 1 < K && j < K) ? (float)Md[(i + 1) * K + j] * scale : 0.f;
      split_h2(m0, m1, hv[r], lv[r]);
    }
    Ah[e] = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    Al[e] = make_uint4(lv[0], lv[1], lv[2], lv[3]);
  }
  __syncthreads();
  const int nzp = (int)(zhi - zlo);
  const int zs = (int)zstride;
  const int nblk = (nzp + PW - 1) / PW;
  const int ngrp = (JT + MW - 1) / MW;
  const bool vec = (zs & 3) == 0 && ((reinterpret_cast<uintptr_t>(Nf) | reinterpret_cast<uintptr_t>(Rho) |
                                     reinterpret_cast<uintptr_t>(Z)) & 15) == 0;
  for (int item = blockIdx.x * (C::NT / 32) + warp; item < nblk * ngrp; item += gridDim.x * (C::NT / 32)) {
    const int blk = item / ngrp, m0 = (item % ngrp) * MW;
    const int mc = min(MW, JT - m0);
    const int p0 = blk * PW;
    const bool fullb = p0 + PW <= nzp && vec;
    float acc[MW][NTL][4];
#pragma unroll
    for (int m = 0; m < MW; ++m)
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[m][nt][r] = 0.f;
    int pq[2];
    bool okq[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      pq[q] = p0 + 4 * (g >> 1) + 2 * q + (g & 1);
      okq[q] = pq[q] < nzp;
    }
    // n values of k-step ks: b_u = (frames 16 ks + 2t + 8u + {0, 1}, column g); the next k-step's are
    // loaded before this one's MMAs (one step of software pipelining: no exposed load latency per k-step)
    auto load_n = [&](int ks, float (&nv)[NTL][2][2]) {
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i = 16 * ks + 2 * t + 8 * u, c = nt >> 1, q = nt & 1;
          nv[nt][u][0] = (i < K && okq[q]) ? __ldg(Nf + ((i * D + c) * zs + pq[q])) : 0.f;
          nv[nt][u][1] = (i + 1 < K && okq[q]) ? __ldg(Nf + (((i + 1) * D + c) * zs + pq[q])) : 0.f;
        }
    };
    float nvc[NTL][2][2];
    load_n(0, nvc);
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t bh[NTL][2], bl[NTL][2];
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) split_h2(nvc[nt][u][0], nvc[nt][u][1], bh[nt][u], bl[nt][u]);
      if (ks + 1 < KS) load_n(ks + 1, nvc);
#pragma unroll
      for (int m = 0; m < MW; ++m) {
        if (m < mc) {
          const uint4 ah = Ah[((m0 + m) * KS + ks) * 32 + lane], al = Al[((m0 + m) * KS + ks) * 32 + lane];
          const uint32_t AH[4] = {ah.x, ah.y, ah.z, ah.w}, AL[4] = {al.x, al.y, al.z, al.w};
          // one product at a time over the n-tiles: consecutive HMMAs hit independent accumulators
#pragma unroll
          for (int nt = 0; nt < NTL; ++nt) mma_f16(acc[m][nt], AH, bh[nt][0], bh[nt][1]);
#pragma unroll
          for (int nt = 0; nt < NTL; ++nt) mma_f16(acc[m][nt], AL, bh[nt][0], bh[nt][1]);
#pragma unroll
          for (int nt = 0; nt < NTL; ++nt) mma_f16(acc[m][nt], AH, bl[nt][0], bl[nt][1]);
        }
      }
    }
    const int pz = p0 + 4 * t;
#pragma unroll
    for (int m = 0; m < MW; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 16 * (m0 + m) + g + 8 * h;
        if (m < mc && j < K) {
          float r[D][4], n[D][4], rho[4];
#pragma unroll
          for (int c = 0; c < D; ++c) {
            r[c][0] = acc[m][2 * c][2 * h] * unscale;
            r[c][1] = acc[m][2 * c][2 * h + 1] * unscale;
            r[c][2] = acc[m][2 * c + 1][2 * h] * unscale;
            r[c][3] = acc[m][2 * c + 1][2 * h + 1] * unscale;
          }
          if (fullb) {
#pragma unroll
            for (int c = 0; c < D; ++c) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(Nf + ((j * D + c) * zs + pz)));
              n[c][0] = v.x, n[c][1] = v.y, n[c][2] = v.z, n[c][3] = v.w;
            }
            const float4 v = __ldg(reinterpret_cast<const float4*>(Rho + (j * zs + pz)));
            rho[0] = v.x, rho[1] = v.y, rho[2] = v.z, rho[3] = v.w;
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const bool ok = pz + u < nzp;
#pragma unroll
              for (int c = 0; c < D; ++c) n[c][u] = ok ? Nf[(j * D + c) * zs + pz + u] : 0.f;
              rho[u] = ok ? Rho[j * zs + pz + u] : 1.f;
            }
          }
          float zz[D][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float dot = 0.f;
#pragma unroll
            for (int c = 0; c < D; ++c) dot += n[c][u] * r[c][u];
            const float ir = rho[u];  // IRho holds fl(1 / rho) (k_ngf_feat4)
#pragma unroll
            for (int c = 0; c < D; ++c) zz[c][u] = (r[c][u] - n[c][u] * dot) * ir;
          }
#pragma unroll
          for (int c = 0; c < D; ++c) {
            float* dst = Z + ((j * D + c) * zs + pz);
            if (fullb) {
              *reinterpret_cast<float4*>(dst) = make_float4(zz[c][0], zz[c][1], zz[c][2], zz[c][3]);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (pz + u < nzp) dst[u] = zz[c][u];
            }
          }
        }
      }
  }
}


}  // namespace sr

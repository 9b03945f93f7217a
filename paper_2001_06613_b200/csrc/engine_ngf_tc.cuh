// engine_ngf_tc.cuh — NGF pass-2 contraction on the 5th-generation tensor cores (tcgen05 kind::f16,
// accumulators in TMEM).  Replaces the per-pixel K x K product of dissimilarity_gradient
// (/root/reference/pkg/src/seqreg/similarity.py:207-211, restated for NGF in DESIGN.md §3.4):
//
//   r_(j,c)(p) = sum_i M'_ij n_(i,c)(p),   z_(j,c)(p) = (r_(j,c) - n_(j,c) (n_j . r_j)) / rho_j(p)
//
// One persistent CTA per SM walks tiles of MT x PXT pixels (MT = 2 operands when K <= 64).  An operand is
// M = 128 rows: row pc = 32 q + l holds pixel PXW q + l / D, component l % D (PXW = 32 / D pixels per TMEM
// lane quarter, so a pixel's components sit in one warp's lanes); columns = frames i.  B = M'^T (rows j,
// columns i), staged once per CTA.  Both operands are f16 with a 2-way split (x = hi + lo, hi = f16(x),
// lo = f16(x - hi); n in [-1, 1], M' scaled by 2^s into the f16 range), and D = A_h B_h + A_l B_h + A_h B_l
// accumulates in fp32 in TMEM (3 MMAs per K16 step; the dropped lo.lo term is 2^-22 relative).
// 16 worker warps (4 per lane quarter) are producer and epilogue at once: in iteration n a worker writes
// tile n + 1's A operand from registers (split, SWIZZLE_128B K-major, 16-byte conflict-free stores), issues
// tile n + 2's n loads, and forms z of tile n from TMEM (r), the A operand (n = hi + lo) and 1/rho (loaded
// at the top of the iteration), so every global load has an iteration to land.  One thread issues the MMAs.
// Two A stages / TMEM slots: full (workers -> MMA), acc (MMA commit -> workers), free (workers -> workers).
// Measured at C3 (K = 100): 0.48-0.53 ms vs 1.09 ms for the mma.sync kernel it replaces; for K <= 32 the
// mma.sync kernel k_ngf_z_f16 (engine_mma.cuh) stays faster (C4: 0.44 vs 0.82 ms) and is used there.
#pragma once
#include <cuda_fp16.h>
#include "engine.cuh"
#include "tma.cuh"

namespace sr {

// Instruction descriptor: kind::f16 with f16 A/B, fp32 accumulate, both operands K-major.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 8 floats -> 8 f16 hi and 8 f16 lo (16 bytes each)
__device__ __forceinline__ void split8_h(const float (&x)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const __half2 hh = __floats2half2_rn(x[2 * u], x[2 * u + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(x[2 * u] - hf.x, x[2 * u + 1] - hf.y);
    h[u] = *reinterpret_cast<const uint32_t*>(&hh);
    l[u] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// byte offset of the 16-byte chunk `ch` (8 f16 = K elements 8 ch .. 8 ch + 7 of the atom) of row r in a
// K-major SWIZZLE_128B block (8-row atoms of 1024 B)
__device__ __forceinline__ uint32_t sw128_chunk(int r, int ch) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((ch ^ r) & 7) << 4));
}

// 32 lanes x 8 columns from TMEM
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = __uint_as_float(r[c]);
}

// 32 lanes x 8 columns of 32-bit to TMEM (warp w writes lanes [32 (w % 4), 32 (w % 4) + 32))
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// 32 lanes x 8 columns from TMEM without waiting (tmem_wait_ld8 completes it)
__device__ __forceinline__ void tmem_ld8_async(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// wait for the thread's outstanding tcgen05.ld; the registers pass through the asm so no use of them
// can be scheduled before the wait
__device__ __forceinline__ void tmem_wait_ld8(uint32_t (&a)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld8x2(uint32_t (&a)[8], uint32_t (&b)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7])
               :
               : "memory");
}

template <int D>
struct ZTC {
  static constexpr int PXW = 32 / D;   // pixels per lane quarter
  static constexpr int PXT = 4 * PXW;  // pixels per M = 128 operand (2-D 64, 3-D 40)
  // 16 worker warps (4 per TMEM lane quarter) + 1 MMA warp: 17 warps, at most 5 on one SM sub-partition
  // (16K registers each) -> 96 registers per thread.  A worker owns frame groups wq, wq + 4, ... of its
  // quarter both as producer (units of 8 frames) and as epilogue (8-column chunks of r).  A tile holds
  // MT = 2 operands of 128 rows when K <= 64 (one SWIZZLE_128B K-atom each), else 1, so a tile has
  // 8 K-frame groups of work per quarter or more and the per-tile hand-offs stay amortised.
  static constexpr int NWK = 16, WPQ = 4, MAXU = 4;
  static constexpr int NT = (NWK + 1) * 32;
  static constexpr int NST = 2;             // A stages = TMEM accumulator slots
  static constexpr int ATOM_A = 128 * 128;  // one K-atom (64 f16) of the 128-row A operand
};

// shared-memory bytes for K frames
__host__ __device__ inline int ztc_mt(int KN) { return KN <= 64 ? 2 : 1; }
template <int D>
inline size_t ztc_smem(int K) {
  const int KN = (K + 15) / 16 * 16, KS = (K + 15) / 16, NATOM = (KS + 3) / 4;
  return 1024 + (size_t)2 * NATOM * KN * 128 + (size_t)ZTC<D>::NST * ztc_mt(KN) * 2 * NATOM * ZTC<D>::ATOM_A + 256;
}

template <int D>
__global__ void __maxnreg__(96) k_ngf_z_tc(const Args a, const float* __restrict__ Nf,
                                                           const float* __restrict__ IRho, long long zlo,
                                                           long long zhi, long long zstride, float* __restrict__ Z) {
  using C = ZTC<D>;
  constexpr int PXW = C::PXW, PXT = C::PXT, NST = C::NST;
  extern __shared__ __align__(1024) unsigned char smem_zt[];
  unsigned char* base = smem_zt + ((1024 - (smem_u32(smem_zt) & 1023)) & 1023);
  const int K = a.K;
  const int KN = (K + 15) / 16 * 16, KS = (K + 15) / 16, NATOM = (KS + 3) / 4;
  const int MT = ztc_mt(KN), TP = MT * PXT;  // operands and pixels per tile
  const int ATOM_B = KN * 128;
  const size_t AOP = (size_t)NATOM * C::ATOM_A;  // one 128-row operand (hi or lo)
  unsigned char* Bh = base;
  unsigned char* Bl = Bh + (size_t)NATOM * ATOM_B;
  unsigned char* Ab = Bl + (size_t)NATOM * ATOM_B;  // [NST][MT][hi, lo][NATOM][128 rows x 128 B]
  const size_t ASTAGE = (size_t)MT * 2 * AOP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Ab + NST * ASTAGE);
  uint64_t* a_full = bars;
  uint64_t* a_free = a_full + NST;
  uint64_t* acc_full = a_free + NST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + NST);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [NT / 32]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const StatsLayout L(K);
  const double* Md = a.stats + L.M;

  // ---- M' scale: 2^s with max |M'| 2^s in [2^13, 2^14) (exact), as k_ngf_z_f16
  float mx = 0.f;
  for (int e = tid; e < K * K; e += C::NT) mx = fmaxf(mx, fabsf((float)Md[e]));
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&a_full[s], C::NWK);   // workers: A tile written
      mbar_init(&a_free[s], C::NWK);   // workers: done with the A tile and the TMEM slot (z formed)
      mbar_init(&acc_full[s], 1);      // MMA commit
    }
    fence_mbar_init();
  }
  if (warp == C::NWK) tmem_alloc(tmem_slot, 256);  // slot s: R in columns 128 s + [0, 128)
  __syncthreads();
  float mmax = 0.f;
  for (int w = 0; w < C::NT / 32; ++w) mmax = fmaxf(mmax, red[w]);
  const int sexp = mmax > 0.f ? 13 - ilogbf(mmax) : 0;
  const float scale = ldexpf(1.f, sexp), unscale = ldexpf(1.f, -sexp);
  // ---- B = M'^T (row j, column i = M'_ij 2^s), zero past K: chunks of 8 columns
  for (int e = tid; e < KN * NATOM * 8; e += C::NT) {
    const int j = e / (NATOM * 8), ck = e % (NATOM * 8);  // column chunk: i = 8 ck .. 8 ck + 7
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = 8 * ck + u;
      x[u] = (i < K && j < K) ? (float)Md[(long long)i * K + j] * scale : 0.f;
    }
    uint4 hi, lo;
    split8_h(x, hi, lo);
    const uint32_t off = (uint32_t)(ck >> 3) * ATOM_B + sw128_chunk(j, ck & 7);
    *reinterpret_cast<uint4*>(Bh + off) = hi;
    *reinterpret_cast<uint4*>(Bl + off) = lo;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int nzp = (int)(zhi - zlo);
  const int zs = (int)zstride;
  const long long ntiles = (nzp + TP - 1) / TP;
  const long long nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp < C::NWK) {
    // ======================= workers: lane quarter qb = warp % 4 (TMEM lanes 32 qb ..), index wq = warp / 4.
    // Iteration n: write tile n + 1's A stage and 1/rho (loaded during iteration n - 1), issue tile n + 2's
    // loads, then form z of tile n (its MMA ran meanwhile) from TMEM and the A stage.
    const int nfg = 2 * KS;  // frame groups of 8 per operand
    const int nun = MT * nfg;  // units (operand mt = u / nfg, frame group fg = u % nfg) per quarter
    const unsigned sn = (unsigned)(D * zs), zsu = (unsigned)zs;
    const int qb = warp & 3, wq = warp >> 2;
    const int l = lane, pxl = l / D, c = l % D, g0 = D * pxl;
    const bool lane_ok = l < PXW * D;
    const int row = 32 * qb + l;
    // 1/rho of a unit: lane (pixel, component c) loads frames 8 fg + c, 8 fg + c + D, ... (the pixel's D
    // lanes split the 8 loads); the other values come from the pixel's lanes by shuffles
    constexpr int IRL = (8 + D - 1) / D;
    float x[C::MAXU][8], irh[C::MAXU][IRL];
    auto load_tile = [&](long long n) {
      const long long t = blockIdx.x + n * gridDim.x;
#pragma unroll
      for (int m = 0; m < C::MAXU; ++m) {
        const int u = wq + C::WPQ * m, mt = u >= nfg ? 1 : 0, fg = u - mt * nfg;  // MT <= 2: no division
        const int p = (int)(t * TP) + mt * PXT + PXW * qb + pxl;
        const bool ok = lane_ok && p < nzp;
        // running pointer over the unit's 8 frames (one 64-bit add per load)
        const float* np = Nf + ((unsigned)c * zsu + (ok ? (unsigned)p : 0u)) + (size_t)(8 * fg) * sn;
        if (u < nun) {
          if (8 * fg + 8 <= K) {
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              x[m][v] = ok ? __ldg(np) : 0.f;
              np += sn;
            }
          } else {
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              x[m][v] = (ok && 8 * fg + v < K) ? __ldg(np) : 0.f;
              np += sn;
            }
          }
        }
      }
    };
    // 1/rho of the epilogue chunks of tile n (chunk = unit fg): lane (pixel, component c) loads frames
    // 8 fg + c, 8 fg + c + D, ... (the pixel's D lanes split the 8 loads); the others come by shuffles
    auto load_ir = [&](long long n) {
      const long long t = blockIdx.x + n * gridDim.x;
#pragma unroll
      for (int m = 0; m < C::MAXU; ++m) {
        const int u = wq + C::WPQ * m, mt = u >= nfg ? 1 : 0, fg = u - mt * nfg;  // MT <= 2: no division
        const int p = (int)(t * TP) + mt * PXT + PXW * qb + pxl;
        const bool ok = lane_ok && p < nzp;
        const float* rb = IRho + (ok ? (unsigned)p : 0u);
        const unsigned o = (unsigned)(8 * fg);
#pragma unroll
        for (int v = 0; v < IRL; ++v) {
          const int f = c + D * v;
          irh[m][v] = (u < nun && ok && f < 8 && 8 * fg + f < K) ? __ldg(rb + (o + f) * zsu) : 0.f;
        }
      }
    };
    auto write_tile = [&](long long n) {  // A stage of tile n from x
      const int s = (int)(n % NST);
      if (n >= NST) mbar_wait_sleep(&a_free[s], (uint32_t)((n / NST - 1) & 1));
#pragma unroll
      for (int m = 0; m < C::MAXU; ++m) {
        const int u = wq + C::WPQ * m, mt = u >= nfg ? 1 : 0, fg = u - mt * nfg;  // MT <= 2: no division
        if (u < nun) {
          unsigned char* Ah = Ab + s * ASTAGE + (size_t)(2 * mt) * AOP;
          unsigned char* Al = Ah + AOP;
          uint4 hi, lo;
          split8_h(x[m], hi, lo);
          const uint32_t off = (uint32_t)(fg >> 3) * C::ATOM_A + sw128_chunk(row, fg & 7);
          *reinterpret_cast<uint4*>(Ah + off) = hi;
          *reinterpret_cast<uint4*>(Al + off) = lo;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[s]);
    };
    if (nloc > 0) {
      load_tile(0);
      write_tile(0);
    }
    if (nloc > 1) load_tile(1);
    for (long long n = 0; n < nloc; ++n) {
      load_ir(n);
      if (n + 1 < nloc) write_tile(n + 1);
      if (n + 2 < nloc) load_tile(n + 2);
      // ---- epilogue of tile n: r and 2^-s/rho from TMEM, n = hi + lo from the A stage (the pair carries
      // n to 2^-22 relative), z = (r - n dot) / rho with dot = sum_c n_c r_c, in the raw scaled r
      const int s = (int)(n % NST);
      const long long t = blockIdx.x + n * gridDim.x;
      mbar_wait_sleep(&acc_full[s], (uint32_t)((n / NST) & 1));
      tc_fence_after();
#pragma unroll
      for (int m = 0; m < C::MAXU; ++m) {
        const int u = wq + C::WPQ * m, mt = u >= nfg ? 1 : 0, ch = u - mt * nfg;
        if (u >= nun) break;
        const int p = (int)(t * TP) + mt * PXT + PXW * qb + pxl;
        const bool ok = lane_ok && p < nzp;
        float* zb = Z + ((unsigned)c * zsu + (ok ? (unsigned)p : 0u));
        const unsigned char* Ah = Ab + s * ASTAGE + (size_t)(2 * mt) * AOP;
        const unsigned char* Al = Ah + AOP;
        const uint32_t tl = tmem + ((uint32_t)(qb * 32) << 16) + (uint32_t)(s * 128 + mt * KN);
        uint32_t rr[8];
        tmem_ld8_async(tl + (uint32_t)(8 * ch), rr);
        const uint32_t off = (uint32_t)(ch >> 3) * C::ATOM_A + sw128_chunk(row, ch & 7);
        const uint4 hv = *reinterpret_cast<const uint4*>(Ah + off);
        const uint4 lv = *reinterpret_cast<const uint4*>(Al + off);
        const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
        float nv[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 a2 = __half22float2(*reinterpret_cast<const __half2*>(&hw[u]));
          const float2 b2 = __half22float2(*reinterpret_cast<const __half2*>(&lw[u]));
          nv[2 * u] = a2.x + b2.x;
          nv[2 * u + 1] = a2.y + b2.y;
        }
        float ir[8];
#pragma unroll
        for (int f = 0; f < 8; ++f) {  // frame f was loaded by lane g0 + f % D as its value f / D
          float vsel = irh[m][0];
#pragma unroll
          for (int v = 1; v < IRL; ++v)
            if (v == f / D) vsel = irh[m][v];
          ir[f] = __shfl_sync(0xffffffffu, vsel, min(g0 + f % D, 31)) * unscale;  // exact (power of 2)
        }
        tmem_wait_ld8(rr);
        float zz[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const float r = __uint_as_float(rr[jj]);
          const float pr = nv[jj] * r;
          float dot;
          if (D == 2) {
            dot = pr + __shfl_xor_sync(0xffffffffu, pr, 1);  // a + b == b + a: both lanes hold the same dot
          } else {
            const float s0 = __shfl_sync(0xffffffffu, pr, g0), s1 = __shfl_sync(0xffffffffu, pr, g0 + 1);
            const float s2 = __shfl_sync(0xffffffffu, pr, g0 + 2 < 32 ? g0 + 2 : 31);
            dot = s0 + s1 + s2;
          }
          zz[jj] = (r - nv[jj] * dot) * ir[jj];
        }
        if (ok) {
          float* zp = zb + (size_t)(ch * 8) * sn;  // running pointer over the chunk's 8 frames
          if (ch * 8 + 8 <= K) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              *zp = zz[jj];
              zp += sn;
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              if (ch * 8 + jj < K) *zp = zz[jj];
              zp += sn;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_free[s]);
    }
  } else {
    // ======================= MMA issuer (slot s is free once its A stage is: the workers release both)
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_f16(128, KN);
      for (long long n = 0; n < nloc; ++n) {
        const int s = (int)(n % NST);
        mbar_wait_sleep(&a_full[s], (uint32_t)((n / NST) & 1));
        tc_fence_after();
        const uint32_t bh0 = smem_u32(Bh), bl0 = smem_u32(Bl);
        for (int mt = 0; mt < MT; ++mt)
        for (int ks = 0; ks < KS; ++ks) {
          const uint32_t ah0 = smem_u32(Ab + s * ASTAGE + (size_t)(2 * mt) * AOP), al0 = ah0 + (uint32_t)AOP;
          const uint32_t acc = tmem + (uint32_t)(s * 128 + mt * KN);
          const uint32_t ko = (uint32_t)((ks & 3) * 32);
          const uint64_t dah = umma_sdesc_sw128(ah0 + (ks >> 2) * C::ATOM_A + ko);
          const uint64_t dal = umma_sdesc_sw128(al0 + (ks >> 2) * C::ATOM_A + ko);
          const uint64_t dbh = umma_sdesc_sw128(bh0 + (ks >> 2) * ATOM_B + ko);
          const uint64_t dbl = umma_sdesc_sw128(bl0 + (ks >> 2) * ATOM_B + ko);
          umma_f16(acc, dah, dbh, idesc, ks > 0 ? 1u : 0u);
          umma_f16(acc, dal, dbh, idesc, 1u);
          umma_f16(acc, dah, dbl, idesc, 1u);
        }
        umma_commit(&acc_full[s]);
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::NWK) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace sr

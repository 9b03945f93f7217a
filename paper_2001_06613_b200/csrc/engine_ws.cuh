// engine_ws.cuh — warp-specialized pass 1 for the NCC displacement-field path (the metric
// path, BASELINE configs[1]).  One CTA per SM, 12 warps:
//
//   producer warps (8):  TMA bulk copies stage the next tiles' y in shared memory (issued two
//                        tiles ahead, completion on an mbarrier); the producers interpolate all
//                        subset frames at their pixel quad (the frame gathers hit L2), keep the
//                        per-frame sum / max / min, and write the shifted values to V[b].
//   consumer warps (4):  accumulate the K x K raw Gram of V[b] (fp32 within a tile, fp64
//                        across tiles, fixed order).
//
// V and the y stage are double buffered; producers and consumers hand V over through named
// barriers FULL[b] / EMPTY[b], so the gather latency of tile n overlaps the Gram of tile n-1.
// Output: the same per-CTA partial layout as k_pass1 ([KP*KP | s | vmax | -vmin]).
#pragma once
#include "tma.cuh"

namespace sr {

template <typename T, int KP>
struct WS1 {
  // 16 producer warps: the gathers are latency-bound, so thread-level parallelism wins
  static constexpr int NP = sizeof(T) == 4 ? 512 : 256, NC = 128, NT = NP + NC;
  static constexpr int TP = sizeof(T) == 4 ? 128 : 64;  // pixels per tile
  static constexpr int QT = TP / 4;                      // pixel quads per tile
  static constexpr int KSTEP = NP / QT;                  // producer frame stride
  static constexpr int FPT = (KP + KSTEP - 1) / KSTEP;   // frames per producer thread
  static constexpr int RS = TP + 4;                      // V row stride (bank spread)
  static constexpr int RB = KP == 32 ? 4 : KP == 16 ? 2 : 1;
  static constexpr int CB = KP == 32 ? 2 : 1;
  static constexpr int RG = KP / RB, CG = KP / CB, OWN = RG * CG;
  static constexpr int NG = NC / OWN;
  static_assert(KP <= 32 && NC % OWN == 0, "ws pass 1 covers KP <= 32");
  static constexpr int BAR_FULL = 1, BAR_EMPTY = 3, BAR_PROD = 5;
  static constexpr int NS = 3;  // y stages in flight (TMA)
};

template <typename T, int D, int KP>
constexpr size_t ws1_smem() {
  using C = WS1<T, KP>;
  return (size_t)C::NS * KP * D * C::TP * sizeof(T) + 2 * (size_t)KP * C::RS * sizeof(T) + 64;
}

template <typename T, int D, int KP, bool POW2>
__device__ __forceinline__ void pass1_ws_body(const Args& a, const CUtensorMap* ymap) {
  using C = WS1<T, KP>;
  using P = T;
  constexpr int TP = C::TP, QT = C::QT, RS = C::RS, NT = C::NT, NP = C::NP;
  constexpr int RB = C::RB, CB = C::CB, RG = C::RG, CG = C::CG, OWN = C::OWN, NG = C::NG;
  constexpr int FPT = C::FPT, KSTEP = C::KSTEP;

  extern __shared__ __align__(128) unsigned char smem_ws[];
  constexpr int NS = C::NS;
  T* ybuf = reinterpret_cast<T*>(smem_ws);                           // [NS][K*D rows][TP]
  T* Vb = ybuf + (size_t)NS * KP * D * TP;                           // [2][KP][RS]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Vb + 2 * (size_t)KP * RS);

  const int tid = threadIdx.x;
  const int K = a.K;
  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (npix + TP - 1) / TP;
  const long long nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  // y of a tile = one 2-D TMA box [K*D rows x TP pixels] of the tensor map (columns past
  // the plane are zero-filled); without a map (unaligned y) the producers load y themselves
  const bool usemap = a.ymap_ok != 0 && !(a.dbg & 8);
  const bool yal = (a.y_stride % (16 / sizeof(T)) == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
  auto issue = [&](long long n) {  // one thread: stage y of local tile n into stage n % NS
    if (n >= nloc || !usemap) return;
    const long long tile = blockIdx.x + n * gridDim.x;
    const long long t0 = a.pix_lo + tile * TP;
    const int s = (int)(n % NS);
    mbar_arrive_expect_tx(&mbar[s], (uint32_t)(K * D * TP * sizeof(T)));
    tma_load_2d(ybuf + (size_t)s * KP * D * TP, ymap, (int)(t0 - a.y_off), 0, &mbar[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
    if (usemap) tma_prefetch_desc(ymap);
  }
  // warm L2 with this CTA's share of the subset frames: the gathers of later tiles then hit L2
  if (tid == 32 && !(a.dbg & 16))
    prefetch_frames_l2<T>(reinterpret_cast<const T*>(a.frames), a.job->frame_index, K, a.g.N, blockIdx.x,
                          gridDim.x);
  // rows of padded frames (k >= K) stay zero in both V buffers
  for (int e = tid; e < 2 * KP * RS; e += NT)
    if ((e / RS) % KP >= K) Vb[e] = (T)0;
  __syncthreads();

  double* out = a.part + (size_t)blockIdx.x * (KP * KP + 3 * KP);

  if (tid < NP) {
    // =============================== producers
    if (tid == 0)
      for (int s = 0; s < NS; ++s) issue(s);
    const int q = tid % QT, kb = tid / QT;
    const T* frames = reinterpret_cast<const T*>(a.frames);
    const T* shifts = reinterpret_cast<const T*>(a.shifts);
    T fsum[FPT], fmx[FPT], fmn[FPT];
    const T* img[FPT];
    T sh[FPT];
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      fsum[i] = (T)0;
      fmx[i] = -INFINITY;
      fmn[i] = INFINITY;
      const int k = kb + KSTEP * i;
      const int fi = k < K ? a.job->frame_index[k] : 0;
      img[i] = frames + (long long)fi * a.g.N;
      sh[i] = (k < K && shifts) ? shifts[fi] : (T)0;
    }
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1);
      const int st = (int)(n % NS);
      const long long tile = blockIdx.x + n * gridDim.x;
      const long long t0 = a.pix_lo + tile * TP;
      const bool viatma = usemap;
      if (viatma) mbar_wait(&mbar[st], (uint32_t)((n / NS) & 1));
      named_sync(C::BAR_EMPTY + b, NT);
      const long long p0 = t0 + 4 * q;
      const long long nv = a.pix_hi - p0;
      const int nvalid = nv >= 4 ? 4 : (nv > 0 ? (int)nv : 0);
      const bool vec = yal && nvalid == 4 && (((p0 - a.y_off) * (long long)sizeof(T)) % 16 == 0);
      const T* ys = ybuf + (size_t)st * KP * D * TP;
      T* V = Vb + (size_t)b * KP * RS;
      if (a.dbg & 4) {
        // profiling: producers only wait for the stage and hand V over
      } else if (sizeof(T) == 4 && viatma && a.use_tex) {
        // texture-gather path: one tld4 per (2-D) sample, D*4 y values from shared memory
        const long long rem = a.pix_hi - t0;
        float vv[FPT][4];
#pragma unroll
        for (int i = 0; i < FPT; ++i) {
          const int k = min(kb + KSTEP * i, K - 1);
          const unsigned long long tx = a.job->tex[k];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float p[D], gdummy[D];
#pragma unroll
            for (int c = 0; c < D; ++c) p[c] = (float)ys[((size_t)k * D + c) * TP + q + QT * e];
            vv[i][e] = interp_tex<D, false, POW2>(tx, a.g, p, gdummy);
          }
        }
#pragma unroll
        for (int i = 0; i < FPT; ++i) {
          const int k = kb + KSTEP * i;
          if (k < K) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float v = vv[i][e];
              const bool ok = q + QT * e < rem;
              const T o = ok ? (T)v - sh[i] : (T)0;
              fsum[i] += o;
              fmx[i] = ok ? max(fmx[i], (T)v) : fmx[i];
              fmn[i] = ok ? min(fmn[i], (T)v) : fmn[i];
              V[(size_t)k * RS + q + QT * e] = o;
            }
          }
        }
      } else if (D == 2 && sizeof(T) == 4 && viatma) {
        const long long rem = a.pix_hi - t0;  // valid pixels of this tile (< TP only for the tail)
        // batched: all positions, then every corner gather of all FPT frames, then the lerps.
        // Lane -> pixel mapping is lane + QT*e (consecutive lanes, consecutive pixels), so one
        // gather instruction of a warp touches ~5 sectors instead of ~20 for pixel quads.
        int bidx[FPT][4];
        float fx[FPT][4], fy[FPT][4];
        bool ins[FPT][4];
#pragma unroll
        for (int i = 0; i < FPT; ++i) {
          const int k = min(kb + KSTEP * i, K - 1);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float px = ys[((size_t)k * D + 0) * TP + q + QT * e];
            const float py = ys[((size_t)k * D + 1) * TP + q + QT * e];
            interp2_prep<float, POW2>(a.g, px, py, bidx[i][e], fx[i][e], fy[i][e], ins[i][e]);
          }
        }
        const int s1 = a.g.sti[1];
        float c00[FPT][4], c10[FPT][4], c01[FPT][4], c11[FPT][4];
#pragma unroll
        for (int i = 0; i < FPT; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float* r = reinterpret_cast<const float*>(img[i]) + ((a.dbg & 2) ? 0 : bidx[i][e]);
            c00[i][e] = __ldg(r);
            c10[i][e] = __ldg(r + 1);
            c01[i][e] = __ldg(r + s1);
            c11[i][e] = __ldg(r + s1 + 1);
          }
#pragma unroll
        for (int i = 0; i < FPT; ++i) {
          const int k = kb + KSTEP * i;
          if (k < K) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a0 = fmaf(fx[i][e], c10[i][e] - c00[i][e], c00[i][e]);
              const float a1 = fmaf(fx[i][e], c11[i][e] - c01[i][e], c01[i][e]);
              const float v = ins[i][e] ? fmaf(fy[i][e], a1 - a0, a0) : 0.f;
              const bool ok = q + QT * e < rem;
              const T o = ok ? (T)v - sh[i] : (T)0;
              fsum[i] += o;
              fmx[i] = ok ? max(fmx[i], (T)v) : fmx[i];
              fmn[i] = ok ? min(fmn[i], (T)v) : fmn[i];
              V[(size_t)k * RS + q + QT * e] = o;
            }
          }
        }
      } else {
#pragma unroll
      for (int i = 0; i < FPT; ++i) {
        const int k = kb + KSTEP * i;
        if (k < K) {
          T yq[D][4];
          if (viatma) {
#pragma unroll
            for (int c = 0; c < D; ++c) lds4(ys + ((size_t)k * D + c) * TP + 4 * q, yq[c]);
          } else {
            load_yq<T, D>(a, k, p0, nvalid, vec, yq);
          }
          T v[4], gr[4][D];
          sample_pts4<T, P, D, false, POW2>(img[i], a.g, yq, v, gr);
          T o4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool ok = e < nvalid;
            o4[e] = ok ? v[e] - sh[i] : (T)0;
            fsum[i] += o4[e];
            fmx[i] = ok ? max(fmx[i], v[e]) : fmx[i];
            fmn[i] = ok ? min(fmn[i], v[e]) : fmn[i];
          }
          sts4(V + (size_t)k * RS + 4 * q, o4);
        }
      }
      }
      named_sync(C::BAR_PROD, NP);  // every producer is done with y stage st
      named_arrive(C::BAR_FULL + b, NT);  // hand V[b] over before issuing the next copy
      if (tid == 0) issue(n + NS);
    }
    // per-frame sum / extrema over the QT lanes sharing a frame (fixed xor tree)
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      double s = (double)fsum[i];
      T mx = fmx[i], mn = fmn[i];
#pragma unroll
      for (int o = QT / 2; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      const int k = kb + KSTEP * i;
      if (q == 0 && k < KP) {
        out[KP * KP + k] = k < K ? s : 0.0;
        out[KP * KP + KP + k] = (double)mx;
        out[KP * KP + 2 * KP + k] = -(double)mn;
      }
    }
  } else {
    // =============================== consumers
    const int ct = tid - NP;
    const int o = ct % OWN, grp = ct / OWN;
    const int rg = o / CG, cg = o % CG;
    double acc64[RB][CB];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int j = 0; j < CB; ++j) acc64[i][j] = 0.0;
    if (nloc > 0) named_arrive(C::BAR_EMPTY + 0, NT);
    if (nloc > 1) named_arrive(C::BAR_EMPTY + 1, NT);
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1);
      named_sync(C::BAR_FULL + b, NT);
      const T* V = Vb + (size_t)b * KP * RS;
      T acc[RB][CB];
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < CB; ++j) acc[i][j] = (T)0;
#pragma unroll 4
      for (int qq = grp; qq < ((a.dbg & 1) ? 0 : QT); qq += NG) {
        T rv[RB][4], cv[CB][4];
#pragma unroll
        for (int i = 0; i < RB; ++i) lds4(V + (size_t)(rg + RG * i) * RS + 4 * qq, rv[i]);
#pragma unroll
        for (int j = 0; j < CB; ++j) lds4(V + (size_t)(cg + CG * j) * RS + 4 * qq, cv[j]);
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int i = 0; i < RB; ++i)
#pragma unroll
            for (int j = 0; j < CB; ++j) acc[i][j] = fma(rv[i][e], cv[j][e], acc[i][j]);
      }
      if (n + 2 < nloc) named_arrive(C::BAR_EMPTY + b, NT);
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < CB; ++j) acc64[i][j] += (double)acc[i][j];
    }
    if (NG == 1) {
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < CB; ++j) out[(rg + RG * i) * KP + cg + CG * j] = acc64[i][j];
    } else {
      // combine the groups in a fixed order through shared memory (ybuf is free now)
      double* red = reinterpret_cast<double*>(smem_ws);
      named_sync(C::BAR_PROD + 1, C::NC);
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < CB; ++j) red[(size_t)grp * KP * KP + (rg + RG * i) * KP + cg + CG * j] = acc64[i][j];
      named_sync(C::BAR_PROD + 1, C::NC);
      for (int e = ct; e < KP * KP; e += C::NC) {
        double s = 0.0;
        for (int g2 = 0; g2 < NG; ++g2) s += red[(size_t)g2 * KP * KP + e];
        out[e] = s;
      }
    }
  }
}

template <typename T, int D, int KP>
__global__ void __launch_bounds__(WS1<T, KP>::NT, 1) k_pass1_ws(const Args a, const __grid_constant__ CUtensorMap ymap) {
  if (a.g.pow2) pass1_ws_body<T, D, KP, true>(a, &ymap);
  else pass1_ws_body<T, D, KP, false>(a, &ymap);
}


// =====================================================================================
// Warp-specialized pass 2 (NCC displacement, KP <= 32): producers stage y by TMA and
// interpolate value + gradient of every subset frame at consecutive pixels (V, GT in
// shared memory, double buffered); consumers contract q = M'^T v + beta' per pixel and
// write dD/dy_j = q_j grad T_j with 16-byte coalesced stores.
template <typename T, int KP>
struct WS2 {
  static constexpr int NP = sizeof(T) == 4 ? 512 : 256, NC = 128, NT = NP + NC;
  static constexpr int TP = sizeof(T) == 4 ? 64 : 32;   // pixels per tile
  static constexpr int PXL = TP / 32;                    // pixels per producer lane
  static constexpr int PW = NP / 32;                     // producer warps
  static constexpr int FPT = (KP + PW - 1) / PW;         // frames per producer thread
  static constexpr int RS = TP + 4;
  static constexpr int QN = TP / 4;                      // consumer pixel quads
  static constexpr int JG = NC / QN;                     // consumer frame groups
  static constexpr int JB = KP / JG >= 1 ? KP / JG : 1;  // frames per consumer thread
  static constexpr int NS = 3;
  static constexpr int BAR_FULL = 1, BAR_EMPTY = 3, BAR_PROD = 5;
};

template <typename T, int D, int KP>
constexpr size_t ws2_smem() {
  using C = WS2<T, KP>;
  return (size_t)C::NS * KP * D * C::TP * sizeof(T) + 2 * (size_t)KP * (1 + D) * C::RS * sizeof(T) +
         (size_t)KP * KP * sizeof(T) + 64;
}

template <typename T, int D, int KP, bool POW2>
__device__ __forceinline__ void pass2_ws_body(const Args& a, const CUtensorMap* ymap) {
  using C = WS2<T, KP>;
  using P = T;
  constexpr int TP = C::TP, RS = C::RS, NT = C::NT, NP = C::NP, NS = C::NS;
  constexpr int PXL = C::PXL, PW = C::PW, FPT = C::FPT, QN = C::QN, JB = C::JB;

  extern __shared__ __align__(128) unsigned char smem_ws2[];
  T* ybuf = reinterpret_cast<T*>(smem_ws2);            // [NS][K*D][TP]
  T* Vb = ybuf + (size_t)NS * KP * D * TP;              // [2][KP][RS]
  T* Gb = Vb + 2 * (size_t)KP * RS;                     // [2][KP*D][RS]
  T* Ms = Gb + 2 * (size_t)KP * D * RS;                 // [KP][KP]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Ms + (size_t)KP * KP);

  const int tid = threadIdx.x;
  const int K = a.K;
  const StatsLayout L(K);
  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (npix + TP - 1) / TP;
  const long long nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const bool usemap = a.ymap_ok != 0;
  auto issue = [&](long long n) {
    if (n >= nloc || !usemap) return;
    const long long t0 = a.pix_lo + (blockIdx.x + n * gridDim.x) * TP;
    const int s = (int)(n % NS);
    mbar_arrive_expect_tx(&mbar[s], (uint32_t)(K * D * TP * sizeof(T)));
    tma_load_2d(ybuf + (size_t)s * KP * D * TP, ymap, (int)(t0 - a.y_off), 0, &mbar[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
    if (usemap) tma_prefetch_desc(ymap);
  }
  {
    const T* Mg = coef_ptr<T>(a.stats, L);
    for (int e = tid; e < KP * KP; e += NT) {
      const int i = e / KP, j = e % KP;
      Ms[e] = (i < K && j < K) ? Mg[i * K + j] : (T)0;
    }
    // frames k >= K: zero rows in both buffers, never rewritten
    for (int e = tid; e < 2 * KP * RS; e += NT)
      if ((e / RS) % KP >= K) Vb[e] = (T)0;
    for (int e = tid; e < 2 * KP * D * RS; e += NT)
      if (((e / RS) % (KP * D)) / D >= K) Gb[e] = (T)0;
  }
  __syncthreads();

  if (tid < NP) {
    // =============================== producers
    if (tid == 0)
      for (int s = 0; s < NS; ++s) issue(s);
    const int lane = tid & 31, warp = tid >> 5;
    const T* frames = reinterpret_cast<const T*>(a.frames);
    const T* shifts = reinterpret_cast<const T*>(a.shifts);
    const T* img[FPT];
    T sh[FPT];
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      const int k = warp + PW * i;
      const int fi = k < K ? a.job->frame_index[k] : 0;
      img[i] = frames + (long long)fi * a.g.N;
      sh[i] = (k < K && shifts) ? shifts[fi] : (T)0;
    }
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1);
      const int st = (int)(n % NS);
      const long long t0 = a.pix_lo + (blockIdx.x + n * gridDim.x) * TP;
      const long long rem = a.pix_hi - t0;
      if (usemap) mbar_wait(&mbar[st], (uint32_t)((n / NS) & 1));
      named_sync(C::BAR_EMPTY + b, NT);
      const T* ys = ybuf + (size_t)st * KP * D * TP;
      T* V = Vb + (size_t)b * KP * RS;
      T* G = Gb + (size_t)b * KP * D * RS;
      T pv[FPT][PXL][D];
#pragma unroll
      for (int i = 0; i < FPT; ++i) {
        const int k = min(warp + PW * i, K - 1);
#pragma unroll
        for (int e = 0; e < PXL; ++e) {
          const int pp = lane + 32 * e;
#pragma unroll
          for (int c = 0; c < D; ++c) {
            if (usemap) {
              pv[i][e][c] = ys[((size_t)k * D + c) * TP + pp];
            } else {
              const long long pix = pp < rem ? t0 + pp : t0;
              pv[i][e][c] = ldg(reinterpret_cast<const T*>(a.y) + (long long)(k * D + c) * a.y_stride + (pix - a.y_off));
            }
          }
        }
      }
      T v[FPT][PXL], gr[FPT][PXL][D];
#pragma unroll
      for (int i = 0; i < FPT; ++i)
#pragma unroll
        for (int e = 0; e < PXL; ++e) {
          if (a.dbg & 2) {
            v[i][e] = pv[i][e][0];
#pragma unroll
            for (int c = 0; c < D; ++c) gr[i][e][c] = pv[i][e][c];
          } else if constexpr (sizeof(T) == 4) {
            if (a.use_tex)
              v[i][e] = interp_tex<D, true, POW2>(a.job->tex[min(warp + PW * i, K - 1)], a.g, pv[i][e], gr[i][e]);
            else
              v[i][e] = interp<T, P, D, true, POW2>(img[i], a.g, pv[i][e], gr[i][e]);
          } else {
            v[i][e] = interp<T, P, D, true, POW2>(img[i], a.g, pv[i][e], gr[i][e]);
          }
        }
#pragma unroll
      for (int i = 0; i < FPT; ++i) {
        const int k = warp + PW * i;
        if (k < K) {
#pragma unroll
          for (int e = 0; e < PXL; ++e) {
            const int pp = lane + 32 * e;
            const bool ok = pp < rem;
            V[(size_t)k * RS + pp] = ok ? v[i][e] - sh[i] : (T)0;
#pragma unroll
            for (int c = 0; c < D; ++c) G[((size_t)k * D + c) * RS + pp] = ok ? gr[i][e][c] : (T)0;
          }
        }
      }
      named_sync(C::BAR_PROD, NP);
      named_arrive(C::BAR_FULL + b, NT);
      if (tid == 0) issue(n + NS);
    }
  } else {
    // =============================== consumers
    const int ct = tid - NP;
    const int pq = ct % QN, jg = ct / QN;
    const int jb0 = jg * JB;
    const bool active = jb0 < KP;
    T bet[JB];
#pragma unroll
    for (int bb = 0; bb < JB; ++bb) {
      const int j = jb0 + bb;
      bet[bb] = (j < K) ? (T)a.stats[L.beta + j] : (T)0;
    }
    T* out = reinterpret_cast<T*>(a.out);
    const bool ovec = ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0) && (a.o_stride % (16 / sizeof(T)) == 0);
    if (nloc > 0) named_arrive(C::BAR_EMPTY + 0, NT);
    if (nloc > 1) named_arrive(C::BAR_EMPTY + 1, NT);
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1);
      const long long t0 = a.pix_lo + (blockIdx.x + n * gridDim.x) * TP;
      named_sync(C::BAR_FULL + b, NT);
      const T* V = Vb + (size_t)b * KP * RS;
      const T* G = Gb + (size_t)b * KP * D * RS;
      if (active) {
        T acc[JB][4];
#pragma unroll
        for (int bb = 0; bb < JB; ++bb)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[bb][e] = (T)0;
#pragma unroll 4
        for (int i = 0; i < ((a.dbg & 1) ? 0 : K); ++i) {
          T x4[4];
          lds4(V + (size_t)i * RS + 4 * pq, x4);
          T m[JB];
          if (JB == 4) {
            T m4[4];
            lds4(Ms + (size_t)i * KP + jb0, m4);
#pragma unroll
            for (int bb = 0; bb < JB; ++bb) m[bb] = m4[bb];
          } else {
#pragma unroll
            for (int bb = 0; bb < JB; ++bb) m[bb] = Ms[(size_t)i * KP + jb0 + bb];
          }
#pragma unroll
          for (int bb = 0; bb < JB; ++bb)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[bb][e] = fma(m[bb], x4[e], acc[bb][e]);
        }
        const long long p0 = t0 + 4 * pq;
        const long long nv = a.pix_hi - p0;
        const int nvalid = nv >= 4 ? 4 : (nv > 0 ? (int)nv : 0);
        const bool vec = ovec && nvalid == 4 && (((p0 - a.o_off) * (long long)sizeof(T)) % 16 == 0);
#pragma unroll
        for (int bb = 0; bb < JB; ++bb) {
          const int j = jb0 + bb;
          if (j >= K || nvalid == 0) continue;
#pragma unroll
          for (int c = 0; c < D; ++c) {
            T g4[4];
            lds4(G + ((size_t)j * D + c) * RS + 4 * pq, g4);
#pragma unroll
            for (int e = 0; e < 4; ++e) g4[e] *= acc[bb][e] + bet[bb];
            T* dst = out + (long long)(j * D + c) * a.o_stride + (p0 - a.o_off);
            if (vec) {
              stg4(dst, g4);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (e < nvalid) dst[e] = g4[e];
            }
          }
        }
      }
      if (n + 2 < nloc) named_arrive(C::BAR_EMPTY + b, NT);
    }
  }
}

template <typename T, int D, int KP>
__global__ void __launch_bounds__(WS2<T, KP>::NT, 1) k_pass2_ws(const Args a, const __grid_constant__ CUtensorMap ymap) {
  if (a.g.pow2) pass2_ws_body<T, D, KP, true>(a, &ymap);
  else pass2_ws_body<T, D, KP, false>(a, &ymap);
}

}  // namespace sr

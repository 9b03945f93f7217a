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
  const bool usemap = a.ymap_ok != 0;
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
  if (tid == 32)
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
      if (D == 2 && sizeof(T) == 4 && viatma) {
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
            const float* r = reinterpret_cast<const float*>(img[i]) + bidx[i][e];
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
      for (int qq = grp; qq < QT; qq += NG) {
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


}  // namespace sr

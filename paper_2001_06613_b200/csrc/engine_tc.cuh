// engine_tc.cuh — pass 1 with the K x K raw Gram on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM), fp32 NCC displacement path, K <= 32.
//
// 3xTF32 in one MMA per 8 pixels: the producers split every shifted value into
// hi = tf32(v) and lo = v - hi and write both as rows of one K-major SWIZZLE_128B operand tile
// (rows 0..31 hi, 32..63 lo; K = pixels).  A = that 64-row tile, B = its first 32 rows, so
// D[0:32] = HH and D[32:64] = LH, and G = HH + LH + LH^T (the lo*lo term, 2^-22 relative, is
// dropped).  One consumer thread issues the MMAs of a tile into one of two TMEM accumulators
// (ping-pong); the consumer warps flush the other one into fp64 registers (tcgen05.ld), so the
// Gram keeps fp32 tensor-core sums per tile and fp64 sums across tiles, in a fixed order.
// The frame sampling side is the same as the warp-specialized kernel (TMA-staged y, 16
// producer warps, lane-consecutive pixels).
#pragma once
#include "tma.cuh"

namespace sr {

template <int D>
struct TC1 {
  static constexpr int NP = 512, NC = 128, NT = NP + NC;
  static constexpr int KP = 32;
  static constexpr int TP = 128;            // pixels per tile = 4 swizzle atoms of 32
  static constexpr int QT = 32;             // producer lanes along pixels
  static constexpr int KSTEP = NP / QT;     // 16 frame rows per producer pass
  static constexpr int FPT = KP / KSTEP;    // 2 frames per producer thread
  static constexpr int NS = D == 2 ? 3 : 2; // y stages in flight
  static constexpr int VBYTES = 64 * TP * 4;  // hi + lo rows, 32 KB per V stage
  static constexpr int YBYTES = KP * D * TP * 4;
  static constexpr int BAR_FULL = 1, BAR_EMPTY = 3, BAR_PROD = 5, BAR_CONS = 6;
  static constexpr uint32_t IDESC = umma_idesc_tf32(64, 32);
};

template <int D>
constexpr size_t tc1_smem() {
  using C = TC1<D>;
  return 1024 + (size_t)C::NS * C::YBYTES + 2 * (size_t)C::VBYTES + 128 + 64 * 33 * 8;
}

template <int D, bool POW2>
__device__ __forceinline__ void pass1_tc_body(const Args& a, const CUtensorMap* ymap) {
  using C = TC1<D>;
  constexpr int TP = C::TP, NT = C::NT, NP = C::NP, NC = C::NC, NS = C::NS, KP = C::KP;
  constexpr int FPT = C::FPT, KSTEP = C::KSTEP;

  extern __shared__ __align__(1024) unsigned char smem_tc[];
  // SWIZZLE_128B operand atoms need 1024-byte alignment
  unsigned char* base = smem_tc + ((1024 - (smem_u32(smem_tc) & 1023)) & 1023);
  float* ybuf = reinterpret_cast<float*>(base);                                  // [NS][K*D][TP]
  unsigned char* Vb = base + (size_t)NS * C::YBYTES;                             // [2][VBYTES]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Vb + 2 * (size_t)C::VBYTES);      // [NS] y + [2] mma
  uint64_t* mbar_mma = mbar + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar_mma + 2);
  double* accs = reinterpret_cast<double*>(mbar + 16);  // [64][33] fp64 Gram rows (consumers)

  const int tid = threadIdx.x;
  const int K = a.K;
  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (npix + TP - 1) / TP;
  const long long nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const bool usemap = a.ymap_ok != 0;
  auto issue = [&](long long n) {
    if (n >= nloc || !usemap) return;
    const long long t0 = a.pix_lo + (blockIdx.x + n * gridDim.x) * TP;
    const int s = (int)(n % NS);
    mbar_arrive_expect_tx(&mbar[s], (uint32_t)(K * D * TP * 4));
    tma_load_2d(ybuf + (size_t)s * KP * D * TP, ymap, (int)(t0 - a.y_off), 0, &mbar[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&mbar[s], 1);
    mbar_init(&mbar_mma[0], 1);
    mbar_init(&mbar_mma[1], 1);
    fence_mbar_init();
    if (usemap) tma_prefetch_desc(ymap);
  }
  // padded frames (k >= K): hi and lo rows stay zero in both V stages
  for (int e = tid; e < 2 * C::VBYTES / 4; e += NT) reinterpret_cast<float*>(Vb)[e] = 0.f;
  if (tid >= NP && tid < NP + 32) tmem_alloc(tmem_slot, 64);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  double* out = a.part + (size_t)blockIdx.x * (KP * KP + 3 * KP);

  if (tid < NP) {
    // =============================== producers (16 warps): sampling
    if (tid == 0)
      for (int s = 0; s < NS; ++s) issue(s);
    const int q = tid & 31, kb = tid >> 5;
    const float* frames = reinterpret_cast<const float*>(a.frames);
    const float* shifts = reinterpret_cast<const float*>(a.shifts);
    float fsum[FPT], fmx[FPT], fmn[FPT], sh[FPT];
    const float* img[FPT];
    uint32_t soff_hi[FPT], soff_lo[FPT];  // swizzled operand offsets of (row k, pixel q) in atom 0
    int yoff[FPT][D];                     // y stage offsets of (k, c, pixel q)
    bool kvalid[FPT];
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      fsum[i] = 0.f;
      fmx[i] = -INFINITY;
      fmn[i] = INFINITY;
      const int k = kb + KSTEP * i;
      kvalid[i] = k < K;
      const int fi = k < K ? a.job->frame_index[k] : 0;
      img[i] = frames + (long long)fi * a.g.N;
      sh[i] = (k < K && shifts) ? shifts[fi] : 0.f;
      soff_hi[i] = sw128_off(k, q);
      soff_lo[i] = sw128_off(32 + k, q);
      const int kc = min(k, K - 1);
#pragma unroll
      for (int c = 0; c < D; ++c) yoff[i][c] = (kc * D + c) * TP + q;
    }
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1);
      const int st = (int)(n % NS);
      const long long t0 = a.pix_lo + (blockIdx.x + n * gridDim.x) * TP;
      const long long rem = a.pix_hi - t0;
      if (usemap) mbar_wait(&mbar[st], (uint32_t)((n / NS) & 1));
      named_sync(C::BAR_EMPTY + b, NT);
      const float* ys = ybuf + (size_t)st * KP * D * TP;
      unsigned char* V = Vb + (size_t)b * C::VBYTES;
      // positions of all FPT x 4 samples (from the TMA stage), every corner gather, then the
      // lerps and the hi/lo stores; all shared-memory offsets are loop invariants
      float pv[FPT][4][D];
      if (usemap) {
#pragma unroll
        for (int i = 0; i < FPT; ++i)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const float* yrow = ys + yoff[i][c];
#pragma unroll
            for (int e = 0; e < 4; ++e) pv[i][e][c] = yrow[32 * e];
          }
      } else {
#pragma unroll
        for (int i = 0; i < FPT; ++i) {
          const int k = min(kb + KSTEP * i, K - 1);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int pp = q + 32 * e;
            const long long pix = pp < rem ? t0 + pp : t0;
#pragma unroll
            for (int c = 0; c < D; ++c)
              pv[i][e][c] = __ldg(reinterpret_cast<const float*>(a.y) + (long long)(k * D + c) * a.y_stride +
                                  (pix - a.y_off));
          }
        }
      }
      float vv[FPT][4];
#pragma unroll
      for (int i = 0; i < FPT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float gdummy[D];
          vv[i][e] = interp<float, float, D, false, POW2>(img[i], a.g, pv[i][e], gdummy);
        }
      const bool full = rem >= TP;
#pragma unroll
      for (int i = 0; i < FPT; ++i) {
        if (kvalid[i]) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float v = vv[i][e];
            const bool ok = full || q + 32 * e < rem;
            const float o = ok ? v - sh[i] : 0.f;
            fsum[i] += o;
            fmx[i] = ok ? fmaxf(fmx[i], v) : fmx[i];
            fmn[i] = ok ? fminf(fmn[i], v) : fmn[i];
            const float hi = to_tf32(o);
            *reinterpret_cast<float*>(V + soff_hi[i] + 8192 * e) = hi;
            *reinterpret_cast<float*>(V + soff_lo[i] + 8192 * e) = o - hi;
          }
        }
      }
      fence_proxy_async_smem();     // make the operand tile visible to the tensor core
      named_sync(C::BAR_PROD, NP);  // every producer is done with y stage st
      named_arrive(C::BAR_FULL + b, NT);
      if (tid == 0) issue(n + NS);
    }
    // per-frame sum / extrema over the 32 lanes sharing a frame (fixed xor tree)
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      double s = (double)fsum[i];
      float mx = fmx[i], mn = fmn[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      const int k = kb + KSTEP * i;
      if (q == 0) {
        out[KP * KP + k] = k < K ? s : 0.0;
        out[KP * KP + KP + k] = (double)mx;
        out[KP * KP + 2 * KP + k] = -(double)mn;
      }
    }
  } else {
    // =============================== consumers (4 warps): tensor-core Gram
    const int ct = tid - NP, cw = ct >> 5, cl = ct & 31;
    const int mrow = 16 * cw + cl;  // D row held by this lane (valid for cl < 16)
    if (cl < 16)
      for (int c = 0; c < 32; ++c) accs[mrow * 33 + c] = 0.0;
    auto flush = [&](long long m) {
      const int bm = (int)(m & 1);
      mbar_wait(&mbar_mma[bm], (uint32_t)((m >> 1) & 1));
      tc_fence_after();
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(cw * 32) << 16) + (uint32_t)(bm * 32), v);
      if (cl < 16) {
#pragma unroll
        for (int c = 0; c < 32; ++c) accs[mrow * 33 + c] += (double)v[c];
      }
      tc_fence_before();
      if (m + 2 < nloc) named_arrive(C::BAR_EMPTY + bm, NT);  // the MMAs reading V[bm] are done
    };
    if (nloc > 0) named_arrive(C::BAR_EMPTY + 0, NT);
    if (nloc > 1) named_arrive(C::BAR_EMPTY + 1, NT);
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1);
      named_sync(C::BAR_FULL + b, NT);
      named_sync(C::BAR_CONS, NC);  // every consumer warp has finished reading TMEM buffer b
      if (ct == 0) {
        tc_fence_after();
        const uint32_t vaddr = smem_u32(Vb + (size_t)b * C::VBYTES);
#pragma unroll
        for (int s = 0; s < TP / 8; ++s) {
          const uint64_t d = umma_sdesc_sw128(vaddr + (uint32_t)((s >> 2) * 8192 + (s & 3) * 32));
          umma_tf32(tmem + (uint32_t)(b * 32), d, d, C::IDESC, s > 0 ? 1u : 0u);
        }
        umma_commit(&mbar_mma[b]);
      }
      __syncwarp();
      if (n > 0) flush(n - 1);
    }
    if (nloc > 0) flush(nloc - 1);
    // D rows: m = 16 cw + cl (cl < 16); rows 0..31 = HH, rows 32..63 = LH; G = HH + LH + LH^T
    const double* red = accs;
    named_sync(C::BAR_CONS, NC);
    for (int e = ct; e < KP * KP; e += NC) {
      const int i = e / KP, j = e % KP;
      out[e] = red[i * 33 + j] + red[(32 + i) * 33 + j] + red[(32 + j) * 33 + i];
    }
    tc_fence_before();
    named_sync(C::BAR_CONS, NC);
    if (cw == 0) {
      tc_fence_after();
      tmem_dealloc(tmem, 64);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(TC1<D>::NT, 1) k_pass1_tc(const Args a, const __grid_constant__ CUtensorMap ymap) {
  if (a.g.pow2) pass1_tc_body<D, true>(a, &ymap);
  else pass1_tc_body<D, false>(a, &ymap);
}

}  // namespace sr

namespace sr {

// =====================================================================================
// Split pass 1 (fp32 NCC displacement, K <= 32), kernel A: high-occupancy sampling.
// Thread = 4 pixels (lane-consecutive, stride 256) of one subset frame; writes the shifted
// value v - shift to V[k][p - pix_lo] (row stride vstride).  Read y (d floats) + gather T,
// write V: the sampling runs at full occupancy with no Gram registers or barriers.
// GV: also write grad T_k(y_k(p)) (interpolant gradient / spacing, zero outside the hull; the
// values pass 2 would re-gather) as G[(k D + c) vstride + p], so pass 2 becomes a pure stream.
template <int D, bool POW2, int SPT, bool GV>
__global__ void __launch_bounds__(256, SPT <= 4 ? 8 : 4) k_sample_v(const Args a, float* __restrict__ V, float* __restrict__ G,
                                                     long long vstride) {
  // grid (pixel blocks, K): block-uniform 64-bit bases, 32-bit per-thread offsets
  constexpr int BP = 256 * SPT;  // pixels per block
  if (GV) pdl_trigger();  // the Gram kernel may be scheduled as this grid's last wave starts
  const int npix = (int)(a.pix_hi - a.pix_lo);
  const int k = (int)blockIdx.y;
  const int b0 = (int)blockIdx.x * BP;
  const int tid = (int)threadIdx.x;
  const int fi = a.job->frame_index[k];
  const float* img = reinterpret_cast<const float*>(a.frames) + (long long)fi * a.g.N;
  const float* yb = reinterpret_cast<const float*>(a.y) + (long long)(k * D) * a.y_stride + (a.pix_lo - a.y_off) + b0;
  float* vb = V + (long long)k * vstride + b0;
  const int nb = npix - b0;  // pixels left from this block's start
  const bool full = nb >= BP;
  // GV: y is read once (evict first); V and grad T are re-read by the Gram and the streaming pass 2
  // (evict last), so they should survive in L2 until then
  const uint64_t pol_first = GV ? l2_policy_evict_first() : 0;
  float p[SPT][D];
#pragma unroll
  for (int e = 0; e < SPT; ++e) {
    const int pe = full ? tid + 256 * e : min(tid + 256 * e, nb - 1);
#pragma unroll
    for (int c = 0; c < D; ++c)
      p[e][c] = GV ? ldg_hint(yb + (long long)c * a.y_stride + pe, pol_first) : __ldg(yb + (long long)c * a.y_stride + pe);
  }
  float v[SPT], gd[SPT][D];
#pragma unroll
  for (int e = 0; e < SPT; ++e) v[e] = interp<float, float, D, GV, POW2>(img, a.g, p[e], gd[e]);
  const float* shifts = reinterpret_cast<const float*>(a.shifts);
  const float sh = shifts ? shifts[fi] : 0.f;
  float* gb = GV ? G + (long long)(k * D) * vstride + b0 : nullptr;
#pragma unroll
  for (int e = 0; e < SPT; ++e) {
    const int pe = tid + 256 * e;
    if (full || pe < nb) {
      if (GV) {
        // plain stores (default L2 policy): measured faster than evict_last-hinted volatile-asm stores
        // (34.4 vs 38.4 us at C2 — the hinted stores serialised against the gathers' scheduling)
        if (a.dbg & 16384) {  // profiling comparison: evict_last-hinted stores
          stg_hint(vb + pe, v[e] - sh, pol_first ^ pol_first ^ l2_policy_evict_last());
#pragma unroll
          for (int c = 0; c < D; ++c) stg_hint(gb + (long long)c * vstride + pe, gd[e][c], l2_policy_evict_last());
        } else {
          vb[pe] = v[e] - sh;
#pragma unroll
          for (int c = 0; c < D; ++c) gb[(long long)c * vstride + pe] = gd[e][c];
        }
      } else {
        vb[pe] = v[e] - sh;
      }
    }
  }
}

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

// Split pass 1, kernel B: the K x K raw Gram of V on the tensor cores.  mbarrier pipeline,
// no CTA-wide barrier inside the loop:
//   issuer lane (warp 16): TMA box [32 frames x 128 pixels] of V -> stage (zero-filled past K
//     and past the slab); per tile 16 MMAs (M64 N32 K8, A = [V_hi; V_lo], B = V_hi) into TMEM
//     accumulator ring slot n % NA; tcgen05.commit frees the operand buffer and fills the slot;
//   16 splitter warps: stage -> hi/lo SW128 operand buffer n % NB, per-frame sum / max / min;
//   4 flusher warps: TMEM slot -> fp64 accumulators in smem (G = HH + LH + LH^T at the end).
// The flush lags the MMAs by up to NA tiles, so it never stalls the splitters.
struct TCG {
  static constexpr int NSP = 512, NT = NSP + 32 + 128;  // splitters, issuer warp, flushers
  static constexpr int KP = 32, TP = 128, NST = 6, NB = 3, NA = 4, NACC = 1;  // NACC chains per tile
  static constexpr int R = 2;  // tiles accumulated in one TMEM slot (fp32) between fp64 flushes
  static constexpr int VBYTES = 64 * TP * 4, SBYTES = KP * TP * 4;
  static constexpr uint32_t IDESC = umma_idesc_tf32(64, 32);
};

constexpr size_t tcg_smem() {
  return 1024 + (size_t)TCG::NST * TCG::SBYTES + (size_t)TCG::NB * TCG::VBYTES + 256 + 64 * 33 * 8;
}

static __global__ void __launch_bounds__(TCG::NT, 1) k_gram_tc(const Args a, const __grid_constant__ CUtensorMap vmap) {
  using C = TCG;
  constexpr int TP = C::TP, KP = C::KP, NST = C::NST, NB = C::NB, NA = C::NA;
  extern __shared__ __align__(1024) unsigned char smem_tcg[];
  unsigned char* base = smem_tcg + ((1024 - (smem_u32(smem_tcg) & 1023)) & 1023);
  float* stage = reinterpret_cast<float*>(base);                             // [NST][32][TP]
  unsigned char* Vb = base + (size_t)NST * C::SBYTES;                        // [NB][VBYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(Vb + (size_t)NB * C::VBYTES);
  uint64_t* st_full = bars;              // [NST] TMA transaction barriers
  uint64_t* vb_full = st_full + NST;     // [NB]  512 splitter arrivals
  uint64_t* vb_free = vb_full + NB;      // [NB]  tcgen05.commit
  uint64_t* acc_full = vb_free + NB;     // [NA]  tcgen05.commit
  uint64_t* acc_free = acc_full + NA;    // [NA]  128 flusher arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + NA);
  double* accs = reinterpret_cast<double*>(bars + 32);                       // [64][33]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.K;
  const long long npix = a.pix_hi - a.pix_lo;
  const long long ntiles = (npix + TP - 1) / TP;
  const long long nloc = (a.dbg & 256) ? 0 : ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&st_full[s], 1);
    for (int b = 0; b < NB; ++b) {
      mbar_init(&vb_full[b], C::NSP);
      mbar_init(&vb_free[b], 1);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_free[s], 128);
    }
    fence_mbar_init();
    tma_prefetch_desc(&vmap);
  }
  if (K < KP) {  // operand rows K..31 (hi) and 32+K..63 (lo) stay zero; rows < K are rewritten every tile
    const int zr = KP - K;
    for (int e = tid; e < NB * 2 * zr * 128; e += C::NT) {
      const int b = e / (2 * zr * 128), rr = (e / 128) % (2 * zr), w = e % 128;
      const int row = rr < zr ? K + rr : 32 + K + (rr - zr);
      // word w % 32 of the 128-byte row in column atom w / 32 (a whole row: the swizzle is irrelevant)
      *reinterpret_cast<float*>(Vb + (size_t)b * C::VBYTES + (w >> 5) * 8192 + (row >> 3) * 1024 + (row & 7) * 128 +
                                (w & 31) * 4) = 0.f;
    }
  }
  for (int e = tid; e < 64 * 33; e += C::NT) accs[e] = 0.0;
  if (warp == C::NSP / 32) tmem_alloc(tmem_slot, 32 * NA * C::NACC);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  double* out = a.part + (size_t)blockIdx.x * (KP * KP + 3 * KP);
  auto tile_col = [&](long long n) { return (blockIdx.x + n * gridDim.x) * TP; };
  auto load_tile = [&](long long n, int st) {  // box [32 frames x 128 pixels], zero-filled past K / the slab
    mbar_arrive_expect_tx(&st_full[st], (uint32_t)C::SBYTES);
    tma_load_2d(stage + (size_t)st * KP * TP, &vmap, (int)tile_col(n), 0, &st_full[st]);
  };

  if (tid < C::NSP) {
    // =============================== splitters: frame row r = tid / 16, two float4 groups each
    const int r = tid >> 4, part = tid & 15;
    // group g (of 32 per 128-pixel row) = 2 part + h; atom g / 8 (8 KB column block), chunk g % 8
    uint32_t off_hi[2], off_lo[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = 2 * part + h;
      off_hi[h] = (uint32_t)((g >> 3) * 8192 + (r >> 3) * 1024 + (r & 7) * 128 + ((((g & 7) ^ (r & 7))) << 4));
      off_lo[h] = (uint32_t)((g >> 3) * 8192 + ((32 + r) >> 3) * 1024 + ((32 + r) & 7) * 128 +
                             ((((g & 7) ^ ((32 + r) & 7))) << 4));
    }
    float fsum = 0.f, fmx = -INFINITY, fmn = INFINITY;
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n % NB), st = (int)(n % NST);
      const long long rem = npix - tile_col(n);
      mbar_wait(&st_full[st], (uint32_t)((n / NST) & 1));
      float4 q4[2];
      const float* src = stage + (size_t)st * KP * TP + (size_t)r * TP + part * 8;
      q4[0] = *reinterpret_cast<const float4*>(src);
      q4[1] = *reinterpret_cast<const float4*>(src + 4);
      if (n >= NB) mbar_wait(&vb_free[b], (uint32_t)((n / NB - 1) & 1));
      unsigned char* vb = Vb + (size_t)b * C::VBYTES;
      if (r < K && !(a.dbg & 128)) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float qv[4] = {q4[h].x, q4[h].y, q4[h].z, q4[h].w};
          float hi[4], lo[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float o = qv[u];
            const bool ok = part * 8 + 4 * h + u < rem;
            fsum += o;  // zero-filled past the slab
            fmx = ok ? fmaxf(fmx, o) : fmx;
            fmn = ok ? fminf(fmn, o) : fmn;
            hi[u] = to_tf32(o);
            lo[u] = o - hi[u];
          }
          *reinterpret_cast<float4*>(vb + off_hi[h]) = make_float4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<float4*>(vb + off_lo[h]) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&vb_full[b]);  // also releases stage st (read above)
    }
    // per-frame sums over the 16 threads of a row (fixed xor tree); extrema of v - shift
    double s = (double)fsum;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
      fmn = fminf(fmn, __shfl_xor_sync(0xffffffffu, fmn, o));
    }
    if (part == 0) {
      const float* shifts = reinterpret_cast<const float*>(a.shifts);
      const double sh = (r < K && shifts) ? (double)shifts[a.job->frame_index[r]] : 0.0;
      out[KP * KP + r] = r < K ? s : 0.0;
      out[KP * KP + KP + r] = (double)fmx + sh;      // max v  (= max(v - shift) + shift)
      out[KP * KP + 2 * KP + r] = -((double)fmn + sh);
    }
  } else if (warp == C::NSP / 32) {
    // =============================== issuer: TMA loads and MMAs
    if (lane == 0) {
      for (long long n = 0; n < nloc && n < NST; ++n) load_tile(n, (int)n);
      for (long long n = 0; n < nloc; ++n) {
        const long long grp = n / C::R;  // accumulation group: R consecutive tiles share a TMEM slot
        const bool first = n % C::R == 0, last = n % C::R == C::R - 1 || n == nloc - 1;
        const int b = (int)(n % NB), s = (int)(grp % NA), st = (int)(n % NST);
        mbar_wait(&vb_full[b], (uint32_t)((n / NB) & 1));
        if (n + NST < nloc) load_tile(n + NST, st);  // every splitter has read stage st: refill it
        if (first && grp >= NA) mbar_wait(&acc_free[s], (uint32_t)((grp / NA - 1) & 1));
        tc_fence_after();
        const uint32_t vaddr = smem_u32(Vb + (size_t)b * C::VBYTES);
#pragma unroll
        for (int k8 = 0; k8 < TP / 8; ++k8) {
          const uint64_t d = umma_sdesc_sw128(vaddr + (uint32_t)((k8 >> 2) * 8192 + (k8 & 3) * 32));
          umma_tf32(tmem + (uint32_t)((s * C::NACC + k8 % C::NACC) * 32), d, d, C::IDESC,
                    (k8 >= C::NACC || !first) ? 1u : 0u);
        }
        umma_commit(&vb_free[b]);
        if (last) umma_commit(&acc_full[s]);
      }
    }
    __syncwarp();
  } else {
    // =============================== flushers: TMEM lane quarter q = warp % 4 holds rows 16q..16q+15
    const int q = warp & 3, mrow = 16 * q + lane;
    double* acc = accs + mrow * 33;
    const long long ngrp = (nloc + C::R - 1) / C::R;
    for (long long n = 0; n < ngrp; ++n) {
      const int s = (int)(n % NA);
      mbar_wait(&acc_full[s], (uint32_t)((n / NA) & 1));
      tc_fence_after();
      float v[32], w[32];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(s * C::NACC * 32);
      tmem_ld32(ta, v);
#pragma unroll
      for (int c2 = 1; c2 < C::NACC; ++c2) {
        tmem_ld32(ta + 32 * c2, w);
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] += w[c];
      }
      tc_fence_before();
      mbar_arrive(&acc_free[s]);
      if (lane < 16)
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] += (double)v[c];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid >= C::NSP + 32) {
    for (int e = tid - (C::NSP + 32); e < KP * KP; e += 128) {
      const int i = e / KP, j = e % KP;
      out[e] = accs[i * 33 + j] + accs[(32 + i) * 33 + j] + accs[(32 + j) * 33 + i];
    }
  } else if (warp == C::NSP / 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 32 * NA * C::NACC);
  }
}

}  // namespace sr

namespace sr {

// =====================================================================================
// Pass 2 on the tensor cores (fp32 NCC displacement, 2-D, K <= 32).
// Producers (16 warps) stage y by TMA, interpolate value and gradient of every subset frame at
// consecutive pixels, and write V_hi / V_lo as K-major SWIZZLE_128B operand tiles with the pixel
// as the row (one 128-byte atom row = the 32 frames of a pixel) plus grad T into a row-major
// [frame][comp][pixel] tile.  One consumer thread issues, per 8 frames, two MMAs
// (A = V_hi then V_lo, B = [M'_hi | M'_lo], N = 64) so that TMEM holds, per pixel lane,
// V.M'_hi (cols 0..31) + V.M'_lo (cols 32..63); q_j = col j + col 32+j + beta'_j.  The consumer
// warps read their 32 pixel lanes and write dD/dy_j = q_j grad T_j with coalesced stores.
struct TC2 {
  static constexpr int NP = 512, NC = 256, NT = NP + NC;
  static constexpr int KP = 32, TP = 128, D = 2, NS = 2;
  static constexpr int ABYTES = TP * 128;              // one operand tile (hi or lo): 128 rows x 128 B
  static constexpr int GBYTES = KP * D * TP * 4;       // grad T tile
  static constexpr int YBYTES = KP * D * TP * 4;
  static constexpr int BBYTES = 64 * 128;              // [M'_hi | M'_lo]^T, 64 rows x 128 B
  static constexpr int BAR_FULL = 1, BAR_EMPTY = 3, BAR_PROD = 5, BAR_CONS = 6;
  static constexpr uint32_t IDESC = umma_idesc_tf32(128, 64);
};

constexpr size_t tc2_smem() {
  return 1024 + (size_t)TC2::NS * TC2::YBYTES + 2 * (2 * (size_t)TC2::ABYTES + TC2::GBYTES) + TC2::BBYTES + 256;
}

template <bool POW2>
__device__ __forceinline__ void pass2_tc_body(const Args& a, const CUtensorMap* ymap) {
  using C = TC2;
  constexpr int TP = C::TP, NT = C::NT, NP = C::NP, NC = C::NC, NS = C::NS, KP = C::KP, D = C::D;
  extern __shared__ __align__(1024) unsigned char smem_tc2[];
  unsigned char* base = smem_tc2 + ((1024 - (smem_u32(smem_tc2) & 1023)) & 1023);
  float* ybuf = reinterpret_cast<float*>(base);                                     // [NS][K*D][TP]
  unsigned char* Ab = base + (size_t)NS * C::YBYTES;                                // [2][hi|lo]
  float* Gb = reinterpret_cast<float*>(Ab + 2 * 2 * (size_t)C::ABYTES);            // [2][KP*D][TP]
  unsigned char* Bm = reinterpret_cast<unsigned char*>(Gb) + 2 * (size_t)C::GBYTES; // [64 rows x 128 B]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Bm + C::BBYTES);                    // [NS] y + [2] mma
  uint64_t* mbar_mma = mbar + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar_mma + 2);
  float* beta_s = reinterpret_cast<float*>(mbar + 8);  // [32] beta'

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
    mbar_arrive_expect_tx(&mbar[s], (uint32_t)(K * D * TP * 4));
    tma_load_2d(ybuf + (size_t)s * KP * D * TP, ymap, (int)(t0 - a.y_off), 0, &mbar[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&mbar[s], 1);
    mbar_init(&mbar_mma[0], 1);
    mbar_init(&mbar_mma[1], 1);
    fence_mbar_init();
    if (usemap) tma_prefetch_desc(ymap);
  }
  if (tid < KP) beta_s[tid] = tid < K ? (float)a.stats[L.beta + tid] : 0.f;
  // operand tiles: frames k >= K stay zero (both buffers); B = [M'_hi | M'_lo]^T rows n, K = i
  for (int e = tid; e < 2 * 2 * C::ABYTES / 4; e += NT) reinterpret_cast<float*>(Ab)[e] = 0.f;
  {
    const float* Mf = reinterpret_cast<const float*>(a.stats + L.Mf);
    for (int e = tid; e < 64 * KP; e += NT) {
      const int n = e / KP, i = e % KP, j = n & 31;
      const float m = (i < K && j < K) ? Mf[i * K + j] : 0.f;
      const float hi = to_tf32(m);
      *reinterpret_cast<float*>(Bm + sw128_off(n, i)) = n < 32 ? hi : m - hi;
    }
  }
  if (tid >= NP && tid < NP + 32) tmem_alloc(tmem_slot, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (tid < NP) {
    // =============================== producers
    if (tid == 0)
      for (int s = 0; s < NS; ++s) issue(s);
    const int q = tid & 31, kb = tid >> 5;
    const float* frames = reinterpret_cast<const float*>(a.frames);
    const float* shifts = reinterpret_cast<const float*>(a.shifts);
    constexpr int FPT = 2;
    const float* img[FPT];
    float sh[FPT];
    bool kvalid[FPT];
    uint32_t aoff[FPT];  // swizzled offset of (row = pixel q, K = frame k)
    int yoff[FPT][D], goff[FPT][D];
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      const int k = kb + 16 * i;
      kvalid[i] = k < K;
      const int kc = min(k, K - 1);
      const int fi = a.job->frame_index[kc];
      img[i] = frames + (long long)fi * a.g.N;
      sh[i] = shifts ? shifts[fi] : 0.f;
      aoff[i] = sw128_off(q, k);
#pragma unroll
      for (int c = 0; c < D; ++c) {
        yoff[i][c] = (kc * D + c) * TP + q;
        goff[i][c] = (k * D + c) * TP + q;
      }
    }
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1), st = (int)(n % NS);
      const long long t0 = a.pix_lo + (blockIdx.x + n * gridDim.x) * TP;
      const long long rem = a.pix_hi - t0;
      if (usemap) mbar_wait(&mbar[st], (uint32_t)((n / NS) & 1));
      named_sync(C::BAR_EMPTY + b, NT);
      const float* ys = ybuf + (size_t)st * KP * D * TP;
      unsigned char* Ahi = Ab + (size_t)b * 2 * C::ABYTES;
      unsigned char* Alo = Ahi + C::ABYTES;
      float* G = Gb + (size_t)b * KP * D * TP;
      float pv[FPT][4][D];
#pragma unroll
      for (int i = 0; i < FPT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
#pragma unroll
          for (int c = 0; c < D; ++c) {
            if (usemap) {
              pv[i][e][c] = ys[yoff[i][c] + 32 * e];
            } else {
              const int k = min(kb + 16 * i, K - 1);
              const long long pp = q + 32 * e;
              const long long pix = pp < rem ? t0 + pp : t0;
              pv[i][e][c] = __ldg(reinterpret_cast<const float*>(a.y) + (long long)(k * D + c) * a.y_stride +
                                  (pix - a.y_off));
            }
          }
        }
      float vv[FPT][4], gg[FPT][4][D];
#pragma unroll
      for (int i = 0; i < FPT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) vv[i][e] = interp<float, float, D, true, POW2>(img[i], a.g, pv[i][e], gg[i][e]);
      const bool full = rem >= TP;
#pragma unroll
      for (int i = 0; i < FPT; ++i) {
        if (kvalid[i]) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool ok = full || q + 32 * e < rem;
            const float o = ok ? vv[i][e] - sh[i] : 0.f;
            const float hi = to_tf32(o);
            *reinterpret_cast<float*>(Ahi + aoff[i] + 4096 * e) = hi;  // +32 rows per e
            *reinterpret_cast<float*>(Alo + aoff[i] + 4096 * e) = o - hi;
#pragma unroll
            for (int c = 0; c < D; ++c) G[goff[i][c] + 32 * e] = gg[i][e][c];
          }
        }
      }
      fence_proxy_async_smem();
      named_sync(C::BAR_PROD, NP);
      named_arrive(C::BAR_FULL + b, NT);
      if (tid == 0) issue(n + NS);
    }
  } else {
    // =============================== consumers: MMA issue + epilogue
    const int ct = tid - NP, cw = ct >> 5, cl = ct & 31;
    float* out = reinterpret_cast<float*>(a.out);
    const uint32_t bdesc_base = smem_u32(Bm);
    // consumer warp cw: TMEM lane quarter (cw & 3) = pixels 32 (cw & 3) + cl, frame half (cw >> 2)
    const int quarter = cw & 3, half = cw >> 2;
    auto epilogue = [&](long long m) {
      const int bm = (int)(m & 1);
      const long long t0 = a.pix_lo + (blockIdx.x + m * gridDim.x) * TP;
      const long long pix = t0 + 32 * quarter + cl;
      mbar_wait(&mbar_mma[bm], (uint32_t)((m >> 1) & 1));
      tc_fence_after();
      float v0[16], v1[16];
      const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(bm * 64 + 16 * half);
      tmem_ld16(ta, v0);
      tmem_ld16(ta + 32, v1);
      tc_fence_before();
      const float* G = Gb + (size_t)bm * KP * D * TP + 32 * quarter + cl;
      if (pix < a.pix_hi) {
        float* o = out + (pix - a.o_off);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = 16 * half + jj;
          if (j < K) {
            const float qj = v0[jj] + v1[jj] + beta_s[j];
#pragma unroll
            for (int c = 0; c < D; ++c) o[(long long)(j * D + c) * a.o_stride] = qj * G[(j * D + c) * TP];
          }
        }
      }
      if (m + 2 < nloc) named_arrive(C::BAR_EMPTY + bm, NT);
    };
    if (nloc > 0) named_arrive(C::BAR_EMPTY + 0, NT);
    if (nloc > 1) named_arrive(C::BAR_EMPTY + 1, NT);
    for (long long n = 0; n < nloc; ++n) {
      const int b = (int)(n & 1);
      named_sync(C::BAR_FULL + b, NT);
      named_sync(C::BAR_CONS, NC);  // TMEM buffer b has been read by every consumer warp
      if (ct == 0) {
        tc_fence_after();
        const uint32_t ahi = smem_u32(Ab + (size_t)b * 2 * C::ABYTES), alo = ahi + C::ABYTES;
#pragma unroll
        for (int s = 0; s < KP / 8; ++s) {
          const uint64_t bd = umma_sdesc_sw128(bdesc_base + (uint32_t)(s * 32));
          umma_tf32(tmem + (uint32_t)(b * 64), umma_sdesc_sw128(ahi + (uint32_t)(s * 32)), bd, C::IDESC,
                    s > 0 ? 1u : 0u);
          umma_tf32(tmem + (uint32_t)(b * 64), umma_sdesc_sw128(alo + (uint32_t)(s * 32)), bd, C::IDESC, 1u);
        }
        umma_commit(&mbar_mma[b]);
      }
      __syncwarp();
      if (n > 0) epilogue(n - 1);
    }
    if (nloc > 0) epilogue(nloc - 1);
    tc_fence_before();
    named_sync(C::BAR_CONS, NC);
    if (cw == 0) {
      tc_fence_after();
      tmem_dealloc(tmem, 128);
    }
  }
}

static __global__ void __launch_bounds__(TC2::NT, 1) k_pass2_tc(const Args a, const __grid_constant__ CUtensorMap ymap) {
  if (a.g.pow2) pass2_tc_body<true>(a, &ymap);
  else pass2_tc_body<false>(a, &ymap);
}

}  // namespace sr

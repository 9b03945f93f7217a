// Probe: tcgen05.mma.kind::f16 with the A operand in TMEM (the ".ts" form: A [lane m][column c] holds the
// f16 pair (k = 2c, 2c + 1) of row m, K16 step ks at columns 8 ks..8 ks + 7) and B in shared memory
// (SWIZZLE_128B K-major, as k_ngf_z_tc).  B = identity, so D[m][j] = A[m][j] reveals how the MMA reads A:
//   test 0: A value = k      -> D[m][j] == j
//   test 1: A value = m      -> D[m][j] == m
//   test 2: random A, random B, 3 MMAs per K16 step with hi/lo splits vs a host fp64 product
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/probe_umma_ts scripts/probe_umma_ts.cu && scripts/probe_umma_ts
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2001_06613_b200/csrc/tma.cuh"
using namespace sr;

constexpr int KN = 112, KS = KN / 16, NATOM = (KS + 3) / 4;

__device__ __forceinline__ uint32_t sw128_chunk(int r, int ch) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((ch ^ r) & 7) << 4));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]));
}
__device__ __forceinline__ void umma_f16_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24); }

// A[m][k] fp32 (128 x KN), B[j][k] fp32 (KN x KN); split = 1: 2-way f16 split of both, 3 MMAs per step
__global__ void probe(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  unsigned char* Bh = base;
  unsigned char* Bl = base + NATOM * KN * 128;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < KN * NATOM * 8; e += blockDim.x) {
    const int j = e / (NATOM * 8), ck = e % (NATOM * 8);
    uint32_t h[4], l[4];
    for (int u = 0; u < 4; ++u) {
      const int k0 = 8 * ck + 2 * u;
      const float x0 = k0 < KN ? B[j * KN + k0] : 0.f, x1 = k0 + 1 < KN ? B[j * KN + k0 + 1] : 0.f;
      const __half2 hh = __floats2half2_rn(x0, x1);
      const float2 hf = __half22float2(hh);
      h[u] = pack2(x0, x1);
      l[u] = split ? pack2(x0 - hf.x, x1 - hf.y) : 0u;
    }
    const uint32_t off = (uint32_t)(ck >> 3) * (KN * 128) + sw128_chunk(j, ck & 7);
    *reinterpret_cast<uint4*>(Bh + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(Bl + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // A hi at columns 128 + [0, KN/2), A lo at 192 + [0, KN/2); D at columns [0, KN)
  const uint32_t cah = 128, cal = 192;
  if (warp < 4) {
    const int m = 32 * warp + lane;
    for (int c0 = 0; c0 < KN / 2; c0 += 4) {
      uint32_t h[4], l[4];
      for (int u = 0; u < 4; ++u) {
        const int k = 2 * (c0 + u);
        const float x0 = A[m * KN + k], x1 = A[m * KN + k + 1];
        const __half2 hh = __floats2half2_rn(x0, x1);
        const float2 hf = __half22float2(hh);
        h[u] = pack2(x0, x1);
        l[u] = split ? pack2(x0 - hf.x, x1 - hf.y) : 0u;
      }
      const uint32_t lrow = (uint32_t)(32 * warp) << 16;
      tmem_st4(tmem + lrow + cah + c0, h);
      tmem_st4(tmem + lrow + cal + c0, l);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_f16(128, KN);
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t ko = (uint32_t)((ks & 3) * 32);
      const uint64_t dbh = umma_sdesc_sw128(smem_u32(Bh) + (ks >> 2) * (KN * 128) + ko);
      const uint64_t dbl = umma_sdesc_sw128(smem_u32(Bl) + (ks >> 2) * (KN * 128) + ko);
      umma_f16_ts(tmem, tmem + cah + 8 * ks, dbh, idesc, ks > 0);
      if (split) {
        umma_f16_ts(tmem, tmem + cal + 8 * ks, dbh, idesc, 1);
        umma_f16_ts(tmem, tmem + cah + 8 * ks, dbl, idesc, 1);
      }
    }
    umma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    const int m = 32 * warp + lane;
    for (int c0 = 0; c0 < KN; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      for (int c = 0; c < 16; ++c) D[m * KN + c0 + c] = v[c];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  std::vector<float> A(128 * KN), B(KN * KN), D(128 * KN);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  const size_t smem = 1024 + 2 * NATOM * KN * 128;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bad_total = 0;
  for (int test = 0; test < 3; ++test) {
    srand(1);
    for (int m = 0; m < 128; ++m)
      for (int k = 0; k < KN; ++k)
        A[m * KN + k] = test == 0 ? (float)k : test == 1 ? (float)m : (float)rand() / RAND_MAX * 2.f - 1.f;
    for (int j = 0; j < KN; ++j)
      for (int k = 0; k < KN; ++k)
        B[j * KN + k] = test < 2 ? (j == k ? 1.f : 0.f) : ((float)rand() / RAND_MAX * 2.f - 1.f) * 1000.f;
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 160, smem>>>(dA, dB, dD, test == 2);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("test %d: CUDA error %s\n", test, cudaGetErrorString(err));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxrel = 0.0;
    for (int m = 0; m < 128; ++m)
      for (int j = 0; j < KN; ++j) {
        double ref = 0.0, mag = 0.0;
        for (int k = 0; k < KN; ++k) {
          ref += (double)A[m * KN + k] * B[j * KN + k];
          mag += fabs((double)A[m * KN + k] * B[j * KN + k]);
        }
        const double err = fabs(D[m * KN + j] - ref) / (mag > 0 ? mag : 1.0);
        maxrel = err > maxrel ? err : maxrel;
        if (err > (test == 2 ? 1e-5 : 0.0)) {
          if (bad < 5) printf("  test %d m %d j %d: D %g ref %g\n", test, m, j, D[m * KN + j], ref);
          ++bad;
        }
      }
    printf("test %d: %d mismatches, max err / sum|terms| %.3g\n", test, bad, maxrel);
    bad_total += bad;
  }
  printf(bad_total ? "PROBE FAILED\n" : "PROBE OK\n");
  return bad_total != 0;
}

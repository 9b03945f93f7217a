// Probe: one tcgen05.mma.kind::tf32 (cta_group::1) with SWIZZLE_128B K-major operands in shared
// memory; dumps the TMEM accumulator so the D-row -> TMEM-lane mapping and the descriptor
// encodings can be checked against a host reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_umma scripts/probe_umma.cu && ./probe_umma
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// element (row r, k) of a K-major SW128 operand: rows of 128 B, 8-row atoms of 1024 B
__device__ __forceinline__ int sw128_off(int r, int k) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ (r & 7)) & 7) << 4) + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;                       // LBO (ignored for swizzled K-major): 16 B
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                         // version = 1 (Blackwell)
  d |= (uint64_t)2 << 61;                         // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                 // D format F32
  d |= 2u << 7;                 // A format TF32
  d |= 2u << 10;                // B format TF32
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

template <int M, int N>
__global__ void probe(float* out, const float* A, const float* B) {
  __shared__ __align__(1024) unsigned char sa[128 * 128];
  __shared__ __align__(1024) unsigned char sb[128 * 128];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * 8; e += blockDim.x) {
    const int r = e / 8, k = e % 8;
    *reinterpret_cast<float*>(sa + sw128_off(r, k)) = A[r * 8 + k];
  }
  for (int e = tid; e < N * 8; e += blockDim.x) {
    const int r = e / 8, k = e % 8;
    *reinterpret_cast<float*>(sb + sw128_off(r, k)) = B[r * 8 + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t ad = sdesc(su32(sa), 1024), bd = sdesc(su32(sb), 1024);
    const uint32_t id = idesc_tf32(M, N);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(id), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
  }
  // wait for the MMA
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // each warp reads its 32-lane subpartition, 32 columns
  uint32_t r[32];
  const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  for (int c = 0; c < 32; ++c) out[(warp * 32 + lane) * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(128));
}

template <int M, int N>
static void run() {
  float hA[128 * 8], hB[128 * 8];
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < 8; ++k) hA[m * 8 + k] = (float)((m % 13) + 1) * (k == 0 ? 1.f : 0.f) + (k == 1 ? 0.001f * m : 0.f);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < 8; ++k) hB[n * 8 + k] = (k == 0 ? 1.f : 0.f) + (k == 1 ? (float)n : 0.f);
  // D[m][n] = (m%13+1) + 0.001*m*n   (tf32-exact enough to identify (m, n))
  float *dA, *dB, *dO;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dO, 128 * 32 * 4);
  cudaMemset(dO, 0, 128 * 32 * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  probe<M, N><<<1, 128>>>(dO, dA, dB);
  cudaError_t e = cudaDeviceSynchronize();
  float hO[128 * 32];
  cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
  printf("M=%d N=%d: %s\n", M, N, cudaGetErrorString(e));
  int ok = 0, bad = 0;
  for (int lane = 0; lane < 128; ++lane)
    for (int c = 0; c < N; ++c) {
      const float v = hO[lane * 32 + c];
      if (lane < M) {
        const float want = (float)((lane % 13) + 1) + 0.001f * lane * c;
        if (fabsf(v - want) < 2e-3f * (1 + fabsf(want))) ++ok; else ++bad;
      }
    }
  printf("  identity mapping (row m -> lane m, col n -> column n): %d ok, %d bad\n", ok, bad);
  for (int lane : {0, 1, 15, 16, 31, 32, 33, 47, 48, 63, 64, 100}) {
    printf("  lane %3d:", lane);
    for (int c = 0; c < 4; ++c) printf(" %9.4f", hO[lane * 32 + c]);
    printf(" ... col31 %9.4f\n", hO[lane * 32 + 31]);
  }
}

int main() {
  run<128, 32>();
  run<64, 32>();
  return 0;
}

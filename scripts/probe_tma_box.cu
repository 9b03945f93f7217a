// Probe: one 3-D TMA box [1 x 8 x 48] of a frame stack into dynamic shared memory, completion on
// an mbarrier, compared with the source; exercises box origins near the frame edges.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tma_box scripts/probe_tma_box.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int WB, int HB>
__global__ void probe(const __grid_constant__ CUtensorMap fmap, const float* frames, int n0, int n1, int x0, int y0,
                      int f, int* bad, unsigned dst_off) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  float* dst = reinterpret_cast<float*>(base + dst_off);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(WB * HB * 4) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(&fmap)), "r"(x0), "r"(y0), "r"(f), "r"(su32(&bar))
        : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  for (int e = threadIdx.x; e < WB * HB; e += blockDim.x) {
    const int r = e / WB, c = e % WB;
    const int gx = x0 + c, gy = y0 + r;
    const float want = (gx < n0 && gy < n1) ? frames[((long long)f * n1 + gy) * n0 + gx] : 0.f;
    if (dst[e] != want) atomicAdd(bad, 1);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int n0 = 64, n1 = 48, nf = 32;
  float* h = new float[(size_t)n0 * n1 * nf];
  for (size_t i = 0; i < (size_t)n0 * n1 * nf; ++i) h[i] = (float)i;
  float* d;
  cudaMalloc(&d, sizeof(float) * n0 * n1 * nf);
  cudaMemcpy(d, h, sizeof(float) * n0 * n1 * nf, cudaMemcpyHostToDevice);
  int* bad;
  cudaMallocManaged(&bad, 4);
  EncodeFn fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  CUtensorMap m;
  memset(&m, 0, sizeof m);
  cuuint64_t gdim[3] = {(cuuint64_t)n0, (cuuint64_t)n1, (cuuint64_t)nf};
  cuuint64_t gstr[2] = {(cuuint64_t)n0 * 4, (cuuint64_t)n0 * n1 * 4};
  cuuint32_t box[3] = {48, 8, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  cudaFuncSetAttribute(probe<48, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  // one case per process: ./probe_tma_box dst_off x0 y0 f
  int c_off = argc > 1 ? atoi(argv[1]) : 0, cx = argc > 2 ? atoi(argv[2]) : 0, cy = argc > 3 ? atoi(argv[3]) : 0,
      cf = argc > 4 ? atoi(argv[4]) : 0;
  *bad = 0;
  probe<48, 8><<<1, 128, 200 * 1024>>>(m, d, n0, n1, cx, cy, cf, bad, (unsigned)c_off);
  cudaError_t e = cudaDeviceSynchronize();
  printf("x0=%d y0=%d f=%d dst_off=%d: %s, bad=%d\n", cx, cy, cf, c_off, cudaGetErrorString(e), e == cudaSuccess ? *bad : -1);
  return 0;
}

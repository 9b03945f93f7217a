// probe_mma_sync.cu — throughput of the legacy warp-level tensor path (mma.sync.m16n8k8 tf32,
// HMMA in SASS) on B200, to size the split pass-1 Gram / pass-2 contraction.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/probe_mma_sync scripts/probe_mma_sync.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_mma(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  float c[CH][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ch = 0; ch < CH; ++ch)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[ch][0]), "+f"(c[ch][1]), "+f"(c[ch][2]), "+f"(c[ch][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
  for (int ch = 0; ch < CH; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_mma16(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
  for (int i = 0; i < 2; ++i) b[i] = 0x38003800u + i;
  float c[CH][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ch = 0; ch < CH; ++ch)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[ch][0]), "+f"(c[ch][1]), "+f"(c[ch][2]), "+f"(c[ch][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
  for (int ch = 0; ch < CH; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 32 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    k_mma<4><<<148, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    k_mma<4><<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * warps * iters * 4 * (2.0 * 16 * 8 * 8);
    printf("mma.sync m16n8k8 tf32: %2d warps/SM, 4 chains: %.1f us, %.1f TFLOP/s, %.2f mma/clk/SM @1.965GHz\n",
           warps, ms * 1e3, flops / (ms * 1e-3) / 1e12, 148.0 * warps * iters * 4 / (ms * 1e-3) / 1.965e9 / 148);
  }
  for (int warps : {8, 16, 32}) {
    k_mma16<4><<<148, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    k_mma16<4><<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * warps * iters * 4 * (2.0 * 16 * 8 * 16);
    printf("mma.sync m16n8k16 f16: %2d warps/SM: %.1f TFLOP/s, %.2f mma/clk/SM @1.965GHz\n", warps,
           flops / (ms * 1e-3) / 1e12, 148.0 * warps * iters * 4 / (ms * 1e-3) / 1.965e9 / 148);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

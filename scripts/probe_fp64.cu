// Latency probe: dependent chains of fp64 / fp32 ops and double shuffles, in cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, float* outf, long long* cyc, double a, double b) {
  double x = a + threadIdx.x;
  float y = (float)a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, b, a);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) y = fmaf(y, (float)b, (float)a);
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = x * b;
  long long t4 = clock64();
  out[threadIdx.x] = x;
  outf[threadIdx.x] = y;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; float* of; long long* c;
  cudaMalloc(&o, 8 * 1024); cudaMalloc(&of, 4 * 1024); cudaMallocManaged(&c, 64);
  for (int threads : {32, 1024}) {
    chain<<<1, threads>>>(o, of, c, 1.0, 0.999);
    cudaDeviceSynchronize();
    printf("threads %4d: DFMA %.1f  FFMA %.1f  SHFL.f64+DADD %.1f  DMUL %.1f cycles/op\n", threads, c[0] / 1000.0,
           c[1] / 1000.0, c[2] / 1000.0, c[3] / 1000.0);
  }
  return 0;
}

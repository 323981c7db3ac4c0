// Microbenchmark: FFMA vs FFMA2 (packed fp32x2) issue/throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 0.001f + i;
  const float m = 0.9999f, c = 0.0001f;
  for (int it = 0; it < iters; it++)
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], m, c);
  float s = 0;
  for (int i = 0; i < 8; i++) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, int iters) {
  float2 a[8];
  for (int i = 0; i < 8; i++) a[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
  const float2 m = make_float2(0.9999f, 0.9998f), c = make_float2(0.0001f, 0.0002f);
  for (int it = 0; it < iters; it++)
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = __ffma2_rn(a[i], m, c);
  float s = 0;
  for (int i = 0; i < 8; i++) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; rep++) {
    float t1, t2;
    cudaEventRecord(e0);
    k1<<<148 * 8, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t1, e0, e1);
    cudaEventRecord(e0);
    k2<<<148 * 8, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t2, e0, e1);
    const double n1 = 148.0 * 8 * 256 * iters * 8, n2 = 2 * n1;
    printf("FFMA : %.3f ms  %.2f Tflop-lane-ops/s (fma count %.3g)\n", t1, n1 / t1 / 1e9, n1);
    printf("FFMA2: %.3f ms  %.2f T fp32 ops/s (2 per instr)\n", t2, n2 / t2 / 1e9);
  }
  return 0;
}

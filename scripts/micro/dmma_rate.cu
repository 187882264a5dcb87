// Microbenchmark: DMMA.8x8x4 vs DFMA issue rate on this GPU (one launch each).
#include <cstdio>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma884(d[c][0], d[c][1], a, b);
  }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[16] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 16; ++c) d[c] = fma(a, b, d[c]);
  }
  double s = 0;
  for (int c = 0; c < 16; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_dmma<<<148 * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * 4 * 8 * iters * 8 * 512.0;   // CTAs*warps*iters*8 dmma*512 flop
    printf("DMMA: %.3f ms, %.1f TFLOP/s\n", ms, flops / ms / 1e9);
    cudaEventRecord(e0); k_dfma<<<148 * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 148.0 * 4 * 256 * iters * 16 * 2.0;
    printf("DFMA: %.3f ms, %.1f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  return 0;
}

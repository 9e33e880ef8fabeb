// DMMA.8x8x4 throughput vs resident warps per SM (16 independent accumulators per warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[16][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[r][0]), "+d"(c[r][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int r = 0; r < 16; ++r) s += c[r][0] + c[r][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void kdep(double* out, int iters) {  // one dependent chain per warp
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[2] = {};
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
  if (c[0] == 1.2345) out[0] = c[0];
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  for (int wps : {1, 2, 4, 8, 16, 32}) {
    int blocks = 148, threads = 32 * wps;
    k<<<blocks, threads>>>(d, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); k<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dm = 16.0 * iters * blocks * wps;  // DMMAs
    printf("warps/SM %2d: %.2f TF/s, %.1f cycles per DMMA per SM (at 1.965 GHz)\n", wps,
           dm * 512 / ms / 1e9, ms * 1e-3 * 1.965e9 / (dm / 148));
  }
  kdep<<<148, 32>>>(d, 10); cudaDeviceSynchronize();
  cudaEventRecord(e0); kdep<<<148, 32>>>(d, iters * 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("dependent DMMA latency: %.1f cycles\n", ms * 1e-3 * 1.965e9 / (iters * 4));
  return 0;
}

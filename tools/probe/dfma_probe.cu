// FP64 CUDA-core probe: DFMA/DADD dependent latency and per-SM throughput, and
// shared-memory LDS.128 + barrier round trip (cycles, one CTA on one SM).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void k_dfma(double* out, long long* cyc, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_bar(long long* cyc, int iters) {
  __shared__ double2 buf[2048];
  double2 v = make_double2(threadIdx.x, 0);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    buf[(threadIdx.x * 7 + i) & 2047] = v;
    __syncthreads();
    v = buf[(threadIdx.x * 5 + i * 3) & 2047];
    v.x += 1.0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0 + (long long)v.x * 0;
  if (v.y == 12345.0) buf[0] = v;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1 << 16);
  long long h;
  const int iters = 4096;
  for (int threads : {32, 128, 256, 512, 1024}) {
    k_dfma<1><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9);
    k_dfma<1><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double lat = (double)h / iters;
    k_dfma<8><<<1, threads>>>(out, cyc, iters, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double per = (double)h / (iters * 8.0);
    printf("threads %4d: 1-chain cycles/iter %.2f; 8-chain cycles/DFMA-instr-per-thread %.3f -> %.1f DFMA/clk/SM\n",
           threads, lat, per, threads / per);
  }
  for (int threads : {128, 256, 512}) {
    k_bar<<<1, threads>>>(cyc, 1000);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d: STS + bar + LDS + bar round trip %.1f cycles\n", threads, (double)h / 1000);
  }
  return 0;
}

// Probe: (1) verify mma.sync m8n8k4 f64 fragment layout, (2) DMMA vs DFMA peak.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void layout_test(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];       // A 8x4 row-major
  double b = B[t * 8 + g];       // B 4x8 row-major (k, n)
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[g * 8 + 2 * t] = c0; C[g * 8 + 2 * t + 1] = c1;
}
__global__ void dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[r][0]), "+d"(c[r][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int r = 0; r < 8; ++r) s += c[r][0] + c[r][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void dfma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[16] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) c[r] = fma(a, b, c[r]);
  }
  double s = 0; for (int r = 0; r < 16; ++r) s += c[r];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = (i * 7) % 11 - 5; }
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[i*4+k]*hB[k*8+j]; ref[i*8+j] = s; }
  double *dA, *dB, *dC; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  layout_test<<<1, 32>>>(dA, dB, dC); cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < 64; ++i) bad += hC[i] != ref[i];
  printf("layout mismatches: %d\n", bad);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int iters = 20000, blocks = 148 * 8, threads = 256;
  for (int w = 0; w < 2; ++w) dmma_peak<<<blocks, threads>>>(dC, 100);
  cudaEventRecord(e0); dmma_peak<<<blocks, threads>>>(dC, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * 8 * iters * (double)blocks * threads / 32;
  printf("DMMA m8n8k4: %.2f TFLOP/s\n", fl / ms / 1e9);
  for (int w = 0; w < 2; ++w) dfma_peak<<<blocks, threads>>>(dC, 100);
  cudaEventRecord(e0); dfma_peak<<<blocks, threads>>>(dC, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 16 * iters * (double)blocks * threads;
  printf("DFMA: %.2f TFLOP/s\n", fl / ms / 1e9);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Pointer-chase latency: one warp-lane chasing through a buffer of the given size.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const unsigned* __restrict__ next, int iters, unsigned* out, long long* cyc) {
  unsigned p = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = t1 - t0;
}
int main() {
  for (size_t mb : {1, 8, 32, 64, 100, 256, 1024}) {
    size_t n = mb * 1024 * 1024 / 4;
    std::vector<unsigned> h(n);
    // random cyclic permutation with stride >= 128 B
    size_t lines = n / 32;
    std::vector<unsigned> perm(lines);
    for (size_t i = 0; i < lines; ++i) perm[i] = i;
    srand(1);
    for (size_t i = lines - 1; i > 0; --i) { size_t j = rand() % (i + 1); std::swap(perm[i], perm[j]); }
    for (size_t i = 0; i < lines; ++i) h[perm[i] * 32] = perm[(i + 1) % lines] * 32;
    unsigned *d, *o; long long* c;
    cudaMalloc(&d, n * 4); cudaMalloc(&o, 4); cudaMalloc(&c, 8);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    int iters = 20000;
    chase<<<1, 1>>>(d, iters, o, c);  // warm
    chase<<<1, 1>>>(d, iters, o, c);
    long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("%5zu MB: %.0f cycles/load (%.0f ns at 1.965 GHz)\n", mb, (double)cyc / iters, (double)cyc / iters / 1.965);
    cudaFree(d); cudaFree(o); cudaFree(c);
  }
  return 0;
}

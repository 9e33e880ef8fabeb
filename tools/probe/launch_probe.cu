// Floor of a chain of dependent kernel launches in a CUDA graph, with and
// without programmatic dependent launch (PDL): per-launch time of N trivial
// kernels (grid G x 256, griddepcontrol.wait at entry, one store per thread).
// nvcc -gencode arch=compute_100a,code=sm_100a -o launch_probe launch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_touch(double* p, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1.0;
}

int main() {
  const int N = 120;
  double* p;
  cudaMalloc(&p, 1 << 24);
  cudaMemset(p, 0, 1 << 24);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int grids[] = {33, 148, 384, 576, 1184};
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int g : grids) {
      cudaGraph_t graph;
      cudaGraphExec_t exec;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < N; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_touch, p, g * 256);
      }
      cudaStreamEndCapture(s, &graph);
      cudaGraphInstantiate(&exec, graph, 0);
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(exec, s);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(exec, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("pdl=%d grid=%5d: %.2f us per launch\n", pdl, g, ms * 1e3 / (10 * N));
      cudaGraphExecDestroy(exec);
      cudaGraphDestroy(graph);
    }
  return 0;
}

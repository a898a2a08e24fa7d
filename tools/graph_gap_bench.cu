// Microbenchmark: per-kernel cost of a CUDA graph of N dependent launches
// (148 x k blocks each, trivial work), with and without programmatic
// dependent launch (PDL: the next kernel's blocks launch while the previous
// drains, and wait in-kernel with griddepcontrol.wait). Answers how much of a
// slice's ~200 kernel boundaries is launch/drain overhead.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o graph_gap_bench tools/graph_gap_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void work(float* buf, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = buf[i] * 1.0001f + 1.f;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
  const int kernels = 200;
  float* buf;
  cudaMalloc(&buf, 64 << 20);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int blocks : {1, 148, 592, 4096})
    for (int pdl : {0, 1}) {
      cudaGraph_t g;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < kernels; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, work, buf, blocks * 256, pdl);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphExec_t ex;
      if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
        std::printf("instantiate failed\n");
        return 1;
      }
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(ex, st);
      cudaEventRecord(a, st);
      const int reps = 20;
      for (int r = 0; r < reps; ++r) cudaGraphLaunch(ex, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      std::printf("blocks %5d pdl %d: %.2f us per kernel (%s)\n", blocks, pdl, 1e3 * ms / reps / kernels,
                  cudaGetErrorString(cudaGetLastError()));
      cudaGraphExecDestroy(ex);
      cudaGraphDestroy(g);
    }
  return 0;
}

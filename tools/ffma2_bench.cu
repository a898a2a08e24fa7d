// FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) issue throughput: does the packed
// form double CUDA-core FP32 rate? Same flop count both ways.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ffma2_bench.cu -o /tmp/ffma2 && /tmp/ffma2
#include <cstdint>
#include <cstdio>

constexpr int kIters = 4096;

__global__ void scalar_k(float* out, float s) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 1e-7f);
  float t = 0;
  for (int i = 0; i < 16; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void packed_k(float* out, float s) {
  uint64_t a[8];
  for (int i = 0; i < 8; ++i) {
    float2 v = make_float2(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
    a[i] = *reinterpret_cast<uint64_t*>(&v);
  }
  float2 sv = make_float2(s, s), cv = make_float2(1e-7f, 1e-7f);
  const uint64_t S = *reinterpret_cast<uint64_t*>(&sv), Cc = *reinterpret_cast<uint64_t*>(&cv);
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(S), "l"(Cc));
  float t = 0;
  for (int i = 0; i < 8; ++i) {
    float2 v = *reinterpret_cast<float2*>(&a[i]);
    t += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double flops = 2.0 * 16 * kIters * double(blocks) * threads;
  for (int rep = 0; rep < 3; ++rep) {
    float ms[2];
    for (int v = 0; v < 2; ++v) {
      cudaEventRecord(e0);
      if (v == 0) scalar_k<<<blocks, threads>>>(out, 0.999f);
      else packed_k<<<blocks, threads>>>(out, 0.999f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms[v], e0, e1);
    }
    std::printf("FFMA  %.3f ms  %.1f TFLOP/s   FFMA2 %.3f ms  %.1f TFLOP/s\n", ms[0], flops / ms[0] / 1e9,
                ms[1], flops / ms[1] / 1e9);
  }
  return 0;
}

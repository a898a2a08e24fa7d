// Microbenchmark: TMEM -> register bandwidth (tcgen05.ld) per SM, for the
// 32x32b shape at .x16 / .x32 / .x64 and 4 / 8 / 16 warps, each warp reading
// its lane quarter's columns repeatedly (the epilogue's access pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld_bench tools/tmem_ld_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int X>
__device__ __forceinline__ uint32_t ld(uint32_t taddr);

template <>
__device__ __forceinline__ uint32_t ld<16>(uint32_t t) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= r[i];
  return s;
}

template <>
__device__ __forceinline__ uint32_t ld<32>(uint32_t t) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
  for (int i = 0; i < 32; ++i) s ^= r[i];
  return s;
}

template <int X>
__global__ void bench(int reps, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
  const int nw = blockDim.x / 32;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    // warps of one lane quarter take different column ranges
    const uint32_t col = static_cast<uint32_t>(((i * (nw / 4) + warp / 4) * X) % 512);
    acc ^= ld<X>(tmem + lane_base + col);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) *out = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int X>
void run(int warps) {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4 * 1024);
  const int reps = 2048;
  bench<X><<<1, 32 * warps>>>(reps, d, sink);
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    std::printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  const double bytes = double(reps) * warps * 32 * X * 4;
  std::printf("32x32b.x%-3d %2d warps: %8.1f B/cycle (TMEM -> registers, one SM)\n", X, warps, bytes / h);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<16>(w);
    run<32>(w);
  }
  return 0;
}

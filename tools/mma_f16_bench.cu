// Microbenchmark: cycles per tcgen05.mma for the operand layouts the complex
// GEMM can use — kind::f16 / kind::tf32, K-major SWIZZLE_64B (64-byte rows) vs
// SWIZZLE_128B (128-byte rows), cta_group::1 (M = 128) and cta_group::2
// (M = 256 over a CTA pair) — chained into one accumulator as in the kernel's
// main loop. Operands are zeros (timing does not depend on values).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_f16_bench tools/mma_f16_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major swizzled descriptor: rows of `row_bytes` (64 or 128), 8-row atoms
__device__ __forceinline__ uint64_t desc(uint32_t saddr, int row_bytes) {
  const uint64_t sbo = row_bytes * 8 / 16;
  const uint64_t layout = row_bytes == 128 ? 2 : 4;
  return (uint64_t{(saddr >> 4) & 0x3FFFu}) | (uint64_t{1} << 16) | (sbo << 32) | (uint64_t{1} << 46) |
         (layout << 61);
}

template <bool F16, bool PAIR>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (PAIR) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else if constexpr (F16) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}

template <bool F16, bool PAIR>
__global__ void bench(int n, int row_bytes, int count, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  uint32_t rank = 0;
  if constexpr (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                   "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                   "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const int m = PAIR ? 256 : 128;
  const uint32_t idesc = (1u << 4) | (F16 ? 0u : (2u << 7) | (2u << 10)) |
                         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
  const uint32_t a = smem_u32(base), b = smem_u32(base + 128 * 128);
  const int ksteps = row_bytes / 32;  // 32-byte k-steps per row
  for (int rep = 0; rep < 2; ++rep) {
    const unsigned long long t0 = clock64();
    if (threadIdx.x < 32 && rank == 0) {
      const uint64_t ad = desc(a, row_bytes), bd = desc(b, row_bytes);
      for (int i = 0; i < count; ++i) {
        const int k = i % ksteps;
        mma<F16, PAIR>(tmem, ad + 2 * k, bd + 2 * k, idesc, i > 0 ? 1u : 0u);
      }
      if constexpr (PAIR)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                smem_u32(&bar)),
            "h"(static_cast<uint16_t>(3))
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar))
            : "memory");
    }
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)), "r"(rep & 1)
          : "memory");
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[rep] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  } else {
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

template <bool F16, bool PAIR>
void run(const char* name, int n, int row_bytes, unsigned long long* d) {
  const int smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(bench<F16, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int count = 512;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(PAIR ? 2 : 1);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, bench<F16, PAIR>, n, row_bytes, count, d);
  unsigned long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    std::printf("%s error %s\n", name, cudaGetErrorString(e));
    return;
  }
  const double m = PAIR ? 256 : 128, kk = F16 ? 16 : 8;
  const double cyc = double(h[1]) / count;
  // FMAs per SM per cycle (a pair MMA's work is split over 2 SMs)
  std::printf("%-28s N=%3d rows %3dB: %7.1f cycles/MMA  %6.0f FMA/clk/SM\n", name, n, row_bytes, cyc,
              m * n * kk / cyc / (PAIR ? 2 : 1));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  for (int n : {128, 256})
    for (int rb : {64, 128}) {
      run<false, false>("tf32 cta_group::1 M=128", n, rb, d);
      run<true, false>("f16  cta_group::1 M=128", n, rb, d);
      run<true, true>("f16  cta_group::2 M=256", n, rb, d);
    }
  return 0;
}

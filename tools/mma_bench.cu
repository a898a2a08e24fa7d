// Microbenchmark: tcgen05.mma.kind::tf32 (cta_group::1, M=128) issue-to-
// completion time for chains of MMAs into 1, 2 or 4 TMEM accumulators, per N.
// Answers whether small-N tiles are bound by the dependent-accumulate latency
// (same accumulator) rather than the per-dispatch throughput floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t{(saddr >> 4) & 0x3FFFu}) | (uint64_t{1} << 16) | (uint64_t{64} << 32) |
         (uint64_t{1} << 46) | (uint64_t{2} << 61);
}

__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

// four MMAs (k offsets 0, 32, 64, 96 bytes: descriptor +2 per 32 B) under one
// elect, descriptors advanced inside the asm block
__device__ __forceinline__ void mma4_elect(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a1, b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a2, b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a3, b3, %3, 1;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc));
}
__device__ __forceinline__ void mma4_single(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], a1, b1, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], a2, b2, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], a3, b3, %3, 1;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc));
}

__global__ void bench(int n, int n_acc, int count, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x)
    reinterpret_cast<float*>(base)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (mode > 0 && threadIdx.x < 32) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                           ((128 >> 4) << 24);
    const uint32_t a = smem_u32(base), b = smem_u32(base + 128 * 128);
    uint32_t cols = 32;
    while (cols < static_cast<uint32_t>(n)) cols <<= 1;
    for (int rep = 0; rep < 2; ++rep) {
      const unsigned long long t0 = clock64();
      if (mode == 1) {
        for (int i = 0; i < count; ++i) {
          const uint32_t d = tmem + (i % n_acc) * cols;
          mma_elect(d, sw128_desc(a + (i % 4) * 32), sw128_desc(b + (i % 4) * 32), idesc,
                    i >= n_acc ? 1u : 0u);
        }
      } else if (mode == 3) {
        const uint64_t ad = sw128_desc(a), bd = sw128_desc(b);
        for (int i = 0; i < count; i += 4) mma4_elect(tmem + (i / 4 % n_acc) * cols, ad, bd, idesc);
      } else if (mode == 4) {
        const uint64_t ad = sw128_desc(a), bd = sw128_desc(b);
        if (threadIdx.x == 0)
          for (int i = 0; i < count; i += 4) mma4_single(tmem + (i / 4 % n_acc) * cols, ad, bd, idesc);
        __syncwarp();
      } else {
        const uint64_t ad = sw128_desc(a), bd = sw128_desc(b);
        for (int i = 0; i < count; i += 4) {
          mma_elect(tmem, ad, bd, idesc, 1u);
          mma_elect(tmem, ad + 2, bd + 2, idesc, 1u);
          mma_elect(tmem, ad + 4, bd + 4, idesc, 1u);
          mma_elect(tmem, ad + 6, bd + 6, idesc, 1u);
        }
      }
      const unsigned long long t1 = clock64();
      if (threadIdx.x == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
      uint32_t ok = 0;
      while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(&bar)), "r"(rep & 1)
            : "memory");
      }
      const unsigned long long t2 = clock64();
      if (threadIdx.x == 0) {
        out[2 * rep] = t1 - t0;
        out[2 * rep + 1] = t2 - t0;
      }
    }
  } else if (mode == 0 && threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                           ((128 >> 4) << 24);
    const uint32_t a = smem_u32(base), b = smem_u32(base + 128 * 128);
    uint32_t cols = 32;
    while (cols < static_cast<uint32_t>(n)) cols <<= 1;
    for (int rep = 0; rep < 2; ++rep) {
      const unsigned long long t0 = clock64();
      for (int i = 0; i < count; ++i) {
        const uint32_t d = tmem + (i % n_acc) * cols;
        const uint64_t ad = sw128_desc(a + (i % 4) * 32), bd = sw128_desc(b + (i % 4) * 32);
        const uint32_t acc = i >= n_acc ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      const unsigned long long t1 = clock64();
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
      uint32_t ok = 0;
      while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(&bar)), "r"(rep & 1)
            : "memory");
      }
      const unsigned long long t2 = clock64();
      out[2 * rep] = t1 - t0;
      out[2 * rep + 1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int count = 240;
  std::printf("%d tf32 MMAs 128xNx8, cycles per MMA (issue loop / until commit)\n", count);
  for (int mode : {0, 2, 3, 4})
  for (int n : {16, 32, 64, 128, 256}) {
    for (int acc : {1, 2, 4, 8}) {
      if (acc * (n < 32 ? 32 : n) > 512) continue;
      if (mode == 2 && acc > 1) continue;
      if (mode >= 3 && acc > 2) continue;
      bench<<<1, 128, smem>>>(n, acc, count, mode, d);
      unsigned long long h[4];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        std::printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      std::printf("mode %d N=%3d acc=%d  issue %6.1f  complete %6.1f  \n", mode, n, acc,
                  double(h[2]) / count, double(h[3]) / count);
    }
  }
  return 0;
}

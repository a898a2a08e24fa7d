// Microbenchmark + sign check for the exact-integer tensor-core scheme:
// cycles per tcgen05.mma for kind::i8 (s8 x s8 -> s32) against kind::f16,
// cta_group::1 (M = 128) and cta_group::2 (M = 256 over a CTA pair), N = 128 /
// 256, issued either as one chain into a single accumulator or in the 3-digit
// pattern of the split-integer GEMM (per 32-byte k-step: acc0 <- d0 g0;
// acc1 <- d0 g1, d1 g0; acc2 <- d0 g2, d1 g1, d2 g0). A one-MMA check with
// row/column-constant operands (a[r][k] = (r % 7) - 3, b[n][k] = (n % 5) - 2,
// K = 32: D = 32 a b) validates the s8 idesc and the TMEM row/column mapping.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_i8_bench tools/mma_i8_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major SWIZZLE_64B descriptor: 64-byte rows, 8-row atoms 512 B apart
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t{(saddr >> 4) & 0x3FFFu}) | (uint64_t{1} << 16) | (uint64_t{32} << 32) | (uint64_t{1} << 46) |
         (uint64_t{4} << 61);
}

template <int KIND, bool PAIR>  // KIND 0: f16, 1: i8
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (PAIR && KIND == 1)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if constexpr (PAIR)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if constexpr (KIND == 1)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <bool PAIR>
__device__ __forceinline__ void commit(uint64_t* bar) {
  if constexpr (PAIR)
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}

// mode 0: chain into one accumulator; mode 1: 3-digit pattern (6 MMAs per
// k-step over 3 accumulators N columns apart)
template <int KIND, bool PAIR>
__global__ void bench(int n, int mode, int count, unsigned long long* out, int* check) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  uint32_t rank = 0;
  if constexpr (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  // A: 128 rows x 64 B at base; B: up to 256 rows x 64 B at base + 8 KB.
  // Values constant along a row (k), so the swizzle does not matter.
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64;
    base[i] = static_cast<uint8_t>(static_cast<int8_t>(KIND == 1 ? (r % 7) - 3 : 0));
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
    const int r = i / 64 + (PAIR ? static_cast<int>(rank) * (n / 2) : 0);
    base[8192 + i] = static_cast<uint8_t>(static_cast<int8_t>(KIND == 1 ? (r % 5) - 2 : 0));
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                   "r"(512));
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
  // c_format: F32 (1) for f16, S32 (2) for i8; a/b format: F16 (0) / S8 (1)
  const uint32_t fmt = KIND == 1 ? (2u << 4) | (1u << 7) | (1u << 10) : (1u << 4);
  const uint32_t idesc = fmt | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
  const uint32_t a = smem_u32(base), b = smem_u32(base + 8192);
  const uint64_t ad = desc(a), bd = desc(b);
  // correctness: one MMA (k-step 0) into column 0
  if (threadIdx.x < 32 && rank == 0) {
    mma<KIND, PAIR>(tmem, ad, bd, idesc, 0u);
    commit<PAIR>(&bar);
  }
  wait_bar(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (KIND == 1 && threadIdx.x < 128) {
    // warp w reads TMEM lanes 32w..32w+31, first 32 columns
    uint32_t v[32];
    const uint32_t ta = tmem + (static_cast<uint32_t>((threadIdx.x / 32) * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int r = threadIdx.x + static_cast<int>(rank) * 128;  // global row (A rows repeat per CTA)
    int bad = 0;
    for (int c = 0; c < 32; ++c) {
      const int want = 32 * ((threadIdx.x % 7) - 3) * ((c % 5) - 2);
      if (static_cast<int>(v[c]) != want) ++bad;
    }
    (void)r;
    if (bad) atomicAdd(check + rank, bad);
  }
  for (int rep = 0; rep < 2; ++rep) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned long long t0 = clock64();
    if (threadIdx.x < 32 && rank == 0) {
      for (int i = 0; i < count; ++i) {
        const int k = i & 1;  // two 32-byte k-steps per 64-byte row
        if (mode == 0) {
          mma<KIND, PAIR>(tmem, ad + 2 * k, bd + 2 * k, idesc, i > 0 ? 1u : 0u);
        } else {
          const uint32_t acc = i > 0 ? 1u : 0u;
          mma<KIND, PAIR>(tmem, ad + 2 * k, bd + 2 * k, idesc, acc);
          mma<KIND, PAIR>(tmem + n, ad + 2 * k, bd + 2 * k, idesc, acc);
          mma<KIND, PAIR>(tmem + n, ad + 2 * k, bd + 2 * k, idesc, 1u);
          mma<KIND, PAIR>(tmem + 2 * n, ad + 2 * k, bd + 2 * k, idesc, acc);
          mma<KIND, PAIR>(tmem + 2 * n, ad + 2 * k, bd + 2 * k, idesc, 1u);
          mma<KIND, PAIR>(tmem + 2 * n, ad + 2 * k, bd + 2 * k, idesc, 1u);
        }
      }
      commit<PAIR>(&bar);
    }
    wait_bar(&bar, (rep + 1) & 1);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[rep] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  } else {
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int KIND, bool PAIR>
void run(const char* name, int n, int mode, unsigned long long* d, int* chk) {
  const int smem = 1024 + 8192 + 256 * 64;
  cudaFuncSetAttribute(bench<KIND, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int count = mode == 0 ? 768 : 128;
  cudaMemset(chk, 0, 8);
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
  cudaLaunchKernelEx(&cfg, bench<KIND, PAIR>, n, mode, count, d, chk);
  unsigned long long h[2];
  int bad[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(bad, chk, sizeof(bad), cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    std::printf("%s error %s\n", name, cudaGetErrorString(e));
    return;
  }
  const int mmas = mode == 0 ? count : 6 * count;
  const double mm = PAIR ? 256 : 128, kk = KIND == 1 ? 32 : 16;
  const double cyc = double(h[1]) / mmas;
  std::printf("%-26s N=%3d %-7s %7.1f cycles/MMA %6.0f MAC/clk/SM%s\n", name, n, mode ? "3-digit" : "chain", cyc,
              mm * n * kk / cyc / (PAIR ? 2 : 1), KIND == 1 ? (bad[0] || bad[1] ? "  CHECK FAILED" : "  check ok") : "");
}

int main() {
  unsigned long long* d;
  int* chk;
  cudaMalloc(&d, 64);
  cudaMalloc(&chk, 8);
  for (int n : {128, 160, 256})
    for (int mode : {0, 1}) {
      if (mode == 1 && n > 160) continue;
      run<0, false>("f16 cta_group::1 M=128", n, mode, d, chk);
      run<1, false>("i8  cta_group::1 M=128", n, mode, d, chk);
      run<0, true>("f16 cta_group::2 M=256", n, mode, d, chk);
      run<1, true>("i8  cta_group::2 M=256", n, mode, d, chk);
    }
  return 0;
}

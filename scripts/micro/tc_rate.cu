// Throughput probe: tcgen05.mma kind::tf32, M = 128, cta_group::1, issued
// back to back by one elected thread per CTA (one CTA per SM), A from TMEM
// (TS) or shared memory (SS), B from shared memory, N in {64, 128, 256},
// K = 8 per instruction.  Operand values are garbage (the rate does not
// depend on them).  Prints dense TF32 TFLOP/s and MACs/clk/SM at the clock
// the run saw.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_rate scripts/micro/tc_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    if (pred) {
      const uint64_t bd = sdesc(smem_u32(smem)), ad = sdesc(smem_u32(smem + 32768));
      constexpr uint32_t ID = idesc_tf32(128, N);
      const uint32_t acol = tmem + 256;   // A planes (TS) after the accumulator
      unsigned long long t0 = clock64();
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t acc = (i | j) ? 1u : 0u;
          if constexpr (TS) {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(tmem), "r"(acol + 8 * (j & 3)), "l"(bd + 16 * (j & 1)), "r"(ID), "r"(acc));
          } else {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(ad + 16 * (j & 1)), "l"(bd + 16 * (j & 1)), "r"(ID), "r"(acc));
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W_%=;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
      unsigned long long t1 = clock64();
      if (blockIdx.x == 0) *cycles = t1 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, bool TS>
void run(int sms) {
  auto k = rate<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  unsigned long long *cyc;
  cudaMalloc(&cyc, 8);
  k<<<sms, 128, 100 * 1024>>>(10, cyc);
  cudaDeviceSynchronize();
  const int iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, 128, 100 * 1024>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double macs = 128.0 * N * 8 * 8 * iters;   // per SM
  printf("{\"N\": %d, \"A\": \"%s\", \"tflops\": %.1f, \"mac_per_clk_sm\": %.0f, \"clk_ghz\": %.3f, \"err\": \"%s\"}\n",
         N, TS ? "tmem" : "smem", 2 * macs * sms / ms / 1e9, macs / c, c / (ms * 1e6),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms = 148;
  run<64, true>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  run<64, false>(sms);
  run<128, false>(sms);
  run<256, false>(sms);
  return 0;
}

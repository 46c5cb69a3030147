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

template <int N, bool TS, int CE = 0, int WF = 0>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  __shared__ __align__(8) uint64_t bar3;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar2)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar3)), "r"(1));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar3)) : "memory");
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
      uint32_t pend = 1;
      unsigned long long t0 = clock64();
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (CE > 0 && ((i * 8 + j) % CE) == 0) {  // a commit every CE MMAs (to a barrier nobody waits on)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
            if (WF & 1)   // + a wait on an already-completed barrier
              asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W_%=;\n\t}" ::"r"(smem_u32(&bar3)) : "memory");
            if (WF & 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (WF & 4) {   // non-blocking test_wait whose result is consumed one group later
              if (!pend) {
                asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W_%=;\n\t}" ::"r"(smem_u32(&bar3)) : "memory");
              }
              asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pend) : "r"(smem_u32(&bar3)) : "memory");
            }
          }
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

template <int N, bool TS, int CE = 0, int WF = 0>
void run(int sms) {
  auto k = rate<N, TS, CE, WF>;
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
  printf("{\"N\": %d, \"commit_every\": %d, \"wait_fence\": %d, \"A\": \"%s\", \"tflops\": %.1f, \"mac_per_clk_sm\": %.0f, \"clk_ghz\": %.3f, \"err\": \"%s\"}\n",
         N, CE, WF, TS ? "tmem" : "smem", 2 * macs * sms / ms / 1e9, macs / c, c / (ms * 1e6),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// the kernel's issuer shape: the whole warp loops, per group of G MMAs one
// elected lane issues them + a commit, then __syncwarp, then (W) a wait on
// an already-completed barrier by the whole warp
template <int N, int G, bool W>
__global__ void __launch_bounds__(128, 1) rate_warp(int iters, unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bar2, bar3;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar2)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar3)), "r"(1));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar3)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint64_t bd = sdesc(smem_u32(smem));
    constexpr uint32_t ID = idesc_tf32(128, N);
    const uint32_t acol = tmem + 256;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (W) {
        asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W_%=;\n\t}" ::"r"(smem_u32(&bar3)) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      uint32_t pred;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      if (pred) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const uint32_t acc = (i | j) ? 1u : 0u;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(tmem + 64 * (j / 3)), "r"(acol + 8 * (j & 3)), "l"(bd + 16 * (j & 1)), "r"(ID), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) {
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

template <int N, int G, bool W>
void run_warp(int sms) {
  auto k = rate_warp<N, G, W>;
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
  const double macs = 128.0 * N * 8 * G * iters;
  printf("{\"warp_loop\": true, \"N\": %d, \"group\": %d, \"wait\": %d, \"mac_per_clk_sm\": %.0f, \"clk_ghz\": %.3f, \"err\": \"%s\"}\n",
         N, G, (int)W, macs / c, c / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// the Gauss kernel's exact MMA pattern (no waits): 4 stages cycling A by 48
// TMEM columns and B by 12 KB of smem; per stage 3 accumulators x (hi.hi,
// hi.lo, lo.hi) with N = 64, then a commit to the stage's barrier
template <int MODE>
__global__ void __launch_bounds__(128, 1) rate_g3(int iters, unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bars[4];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint64_t desc0 = sdesc(smem_u32(smem));
    constexpr uint32_t ID = idesc_tf32(128, 64);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t s = i & 3;
      uint32_t pred;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      if (pred) {
        const uint64_t bh = desc0 + (uint64_t)(s * (12288 >> 4)), bl = bh + (6144 >> 4);
        const uint32_t a = tmem + 320 + s * 48;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const uint32_t d = tmem + 64 * j;
          const uint64_t b0 = bh + j * (2048 >> 4), b1 = bl + j * (2048 >> 4);
          const uint32_t acc = i ? 1u : 0u;
          const uint32_t a0 = MODE == 1 ? a : a + 16 * j;   // MODE 1: one A plane only
#define MMA(D, A, B, ACC) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(D), "r"(A), "l"(B), "r"(ID), "r"(ACC))
          MMA(d, a0, b0, acc);
          MMA(d, a0, b1, 1u);
          MMA(d, a0 + 8, b0, 1u);
#undef MMA
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) {
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

template <int MODE>
void run_g3(int sms) {
  auto k = rate_g3<MODE>;
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
  const double macs = 128.0 * 64 * 8 * 9 * iters;
  printf("{\"g3_pattern_mode\": %d, \"mac_per_clk_sm\": %.0f, \"clk_ghz\": %.3f, \"err\": \"%s\"}\n", MODE,
         macs / c, c / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// the stage handshake alone: warp 0 issues the Gauss pattern per stage after
// waiting full[s]; warp 1 ("converter") waits bars[s] (the MMA commit of the
// stage) and arrives on full[s + ST] -- a ring of ST stages
template <int ST, bool PAIRS, int NC = 1, int NIDLE = 0, int MW = 0>
__global__ void __launch_bounds__(512, 1) rate_ring(int iters, unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bars[8], full[8];
  const int nw = (int)(blockDim.x >> 5);
  const int warp = (int)((threadIdx.x >> 5) + nw - MW) % nw, lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    for (int i = 0; i < 8; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(NC));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
#define WAITB(B, P) asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(smem_u32(B)), "r"(P) : "memory")
  if (warp > NC && warp <= NC + NIDLE) {   // idle pollers (the promotion warps' pattern)
    WAITB(&bar, 0u);
  } else if (warp >= 1 && warp <= NC) {   // converter: stage q is free once MMA(q - ST) completed
    for (int q = 0; q < iters; ++q) {
      const int s = q % ST;
      if (q >= ST) WAITB(&bars[s], (uint32_t)(((q / ST) + 1) & 1));
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
  } else if (warp == 0) {
    const uint64_t desc0 = sdesc(smem_u32(smem));
    constexpr uint32_t ID = idesc_tf32(128, 64);
    unsigned long long t0 = clock64();
    for (int q = 0; q < iters; ++q) {
      const uint32_t s = q % ST;
      if (!PAIRS) {
        WAITB(&full[s], (uint32_t)((q / ST) & 1));
      } else if ((q & 1) == 0) {
        const int qw = q + 1 < iters ? q + 1 : q;
        WAITB(&full[qw % ST], (uint32_t)((qw / ST) & 1));
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t pred;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      if (pred) {
        const uint64_t bh = desc0 + (uint64_t)((s & 3) * (12288 >> 4)), bl = bh + (6144 >> 4);
        const uint32_t a = tmem + 320 + (s & 3) * 48;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const uint32_t d = tmem + 64 * j;
          const uint64_t b0 = bh + j * (2048 >> 4), b1 = bl + j * (2048 >> 4);
          const uint32_t acc = q ? 1u : 0u;
#define MMA(D, A, B, ACC) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(D), "r"(A), "l"(B), "r"(ID), "r"(ACC))
          MMA(d, a + 16 * j, b0, acc);
          MMA(d, a + 16 * j, b1, 1u);
          MMA(d, a + 16 * j + 8, b0, 1u);
#undef MMA
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[s])) : "memory");
      }
      __syncwarp();
    }
    if (lane == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      WAITB(&bar, 0u);
      unsigned long long t1 = clock64();
      if (blockIdx.x == 0) *cycles = t1 - t0;
    }
  }
#undef WAITB
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int ST, bool PAIRS, int NC = 1, int NIDLE = 0, int MW = 0>
void run_ring(int sms) {
  auto k = rate_ring<ST, PAIRS, NC, NIDLE, MW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  unsigned long long *cyc;
  cudaMalloc(&cyc, 8);
  k<<<sms, 32 * (1 + NC + NIDLE), 100 * 1024>>>(16, cyc);
  cudaDeviceSynchronize();
  const int iters = 40000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, 32 * (1 + NC + NIDLE), 100 * 1024>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double macs = 128.0 * 64 * 8 * 9 * iters;
  printf("{\"mma_warp\": %d, \"conv_warps\": %d, \"idle_pollers\": %d, \"ring_stages\": %d, \"pairs\": %d, \"mac_per_clk_sm\": %.0f, \"clk_per_stage\": %.0f, \"err\": \"%s\"}\n", MW, NC, NIDLE, ST, (int)PAIRS,
         macs / c, (double)c / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms = 148;
  run_ring<4, false, 8, 4, 0>(sms);
  run_ring<4, false, 8, 4, 1>(sms);
  run_ring<4, false, 8, 4, 13>(sms);
  return 0;
}

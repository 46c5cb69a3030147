// Inline-PTX building blocks of the tcgen05 complex GEMM kernels (sm_100a):
// mbarriers, UMMA shared-memory descriptors, tensor-memory loads/stores,
// tcgen05.mma issue/commit, the TF32 hi/lo split and the staged epilogue
// store.  Shared by qf_gemm_tc.cu (3xTF32 real-block form) and
// qf_gemm_tcw.cu (the 128 x 128 Gauss-form long-K kernel).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "qf_common.cuh"

namespace qf {
namespace tc {

constexpr int BM = 128;     // rows per tile (= TMEM lanes)
constexpr int KB = 8;       // complex k per stage (= one tf32 MMA K step)
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// hi = tf32(x), lo = tf32(x - hi); returned as raw fp32 bit patterns
__device__ __forceinline__ void split3(float x, uint32_t &hi, uint32_t &lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// the same wait for long, expected waits (a warp idle for a whole chunk of
// k-blocks): each try_wait may suspend the thread up to `ns` before it
// re-polls, so idle warps stop burning issue slots (and power)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
      "@!P bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(ns)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major, SWIZZLE_NONE UMMA shared-memory descriptor.  Core matrix = 8
// rows x 16 B; the two 16-byte K halves of one tf32 K=8 step are LBO=128 B
// apart, consecutive 8-row groups SBO=256 B apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// byte offset of (row r, k) inside a [rows x 8 tf32] K-major core-matrix tile
__device__ __forceinline__ uint32_t core_off(int r, int kchunk) {
  return (uint32_t)((r >> 3) * 256 + kchunk * 128 + (r & 7) * 16);
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)            // D format f32
         | (2u << 7)          // A format tf32
         | (2u << 10)         // B format tf32
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred;
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}


constexpr int V2_THREADS = 256;
constexpr int V2_BN = 64;

__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c,
                                         uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

__device__ __forceinline__ void split_fast(float x, uint32_t &hi, uint32_t &lo) {
  // (measured and rejected: hi = the raw bits -- the tensor core reads the top
  // 19 -- and lo = x - trunc(x) saves one of the three ALU ops per split:
  // +1% on the wide kernel, +2% on K = 16 shapes, error 3.7e-6 -> 4.3e-6)
  const uint32_t h = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;  // round-half-away to tf32
  hi = h;
  lo = __float_as_uint(x - __uint_as_float(h));  // exact; the tensor core keeps its top 19 bits
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b)
               : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}

template <int CPW>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&v)[CPW]) {
  if constexpr (CPW == 32) tmem_ld32(taddr, v);
  else if constexpr (CPW == 16) tmem_ld16(taddr, v);
  else if constexpr (CPW == 8) tmem_ld8(taddr, v);
  else __trap();  // narrower column groups only exist in instantiations that never run them
}

// One warp's 32-row x CH-column output chunk (lane = row, values vr/vi as
// fp32 bit patterns) -> C through the warp's staging tile: alpha applied in
// registers, then each store instruction covers whole row segments; beta and
// ragged edges are handled per 16-byte pair.  `c` = C at (row m0, column c0).
template <int CPW>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t (&v)[CPW]) {
  if constexpr (CPW == 32) tmem_st32(taddr, v);
  else if constexpr (CPW == 16) tmem_st16(taddr, v);
  else if constexpr (CPW == 8) tmem_st8(taddr, v);
  else __trap();
}

template <int CH, int PITCH>
__device__ __forceinline__ void stage_store_chunk(uint8_t *stg, const uint32_t (&vr)[CH],
                                                  const uint32_t (&vi)[CH], float2 *c, int64_t ldc,
                                                  int64_t rows, int64_t cols, float ar, float ai,
                                                  float br, float bi, bool use_beta, bool vec,
                                                  int lane) {
  const bool plain = ar == 1.f && ai == 0.f;
#pragma unroll
  for (int j = 0; j < CH / 2; ++j) {
    const float x0 = __uint_as_float(vr[2 * j]), y0 = __uint_as_float(vi[2 * j]);
    const float x1 = __uint_as_float(vr[2 * j + 1]), y1 = __uint_as_float(vi[2 * j + 1]);
    *reinterpret_cast<float4 *>(stg + lane * PITCH + j * 16) =
        plain ? make_float4(x0, y0, x1, y1)
              : make_float4(ar * x0 - ai * y0, ar * y0 + ai * x0, ar * x1 - ai * y1, ar * y1 + ai * x1);
  }
  __syncwarp();
  constexpr int LPR = CH / 2, RPI = 32 / LPR;  // lanes per row (16 B each), rows per store
  const int rs = lane / LPR, cc = lane % LPR;
  if (!use_beta && vec && rows >= 32 && cols >= CH) {  // whole chunk: plain 16-byte stores
#pragma unroll
    for (int i = 0; i < 32 / RPI; ++i) {
      const int r = RPI * i + rs;
      // streaming (evict-first) stores: big results do not push the operands
      // that later tiles re-read (A tiles across N tiles) out of L2
      __stcs(reinterpret_cast<float4 *>(c + r * ldc + 2 * cc),
             *reinterpret_cast<const float4 *>(stg + r * PITCH + cc * 16));
    }
    __syncwarp();
    return;
  }
#pragma unroll
  for (int i = 0; i < 32 / RPI; ++i) {
    const int r = RPI * i + rs;
    const int64_t col = 2 * cc;
    if (r < rows && col < cols) {
      float4 v = *reinterpret_cast<const float4 *>(stg + r * PITCH + cc * 16);
      float2 *p = c + r * ldc + col;
      if (vec && col + 1 < cols) {
        if (use_beta) {
          const float4 o = *reinterpret_cast<const float4 *>(p);
          v.x += br * o.x - bi * o.y;
          v.y += br * o.y + bi * o.x;
          v.z += br * o.z - bi * o.w;
          v.w += br * o.w + bi * o.z;
        }
        *reinterpret_cast<float4 *>(p) = v;
      } else {
        float2 v0 = make_float2(v.x, v.y), v1 = make_float2(v.z, v.w);
        if (use_beta) {
          const float2 o0 = p[0];
          v0.x += br * o0.x - bi * o0.y;
          v0.y += br * o0.y + bi * o0.x;
        }
        p[0] = v0;
        if (col + 1 < cols) {
          if (use_beta) {
            const float2 o1 = p[1];
            v1.x += br * o1.x - bi * o1.y;
            v1.y += br * o1.y + bi * o1.x;
          }
          p[1] = v1;
        }
      }
    }
  }
  __syncwarp();
}

// host side (qf_gemm_tc.cu): TMA tensor maps over float data (dims innermost
// first, byte strides) and the operand test for them
bool make_tmap(CUtensorMap *m, const void *ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
               uint64_t s2, uint32_t b0, uint32_t b1, bool swz64);
bool make_tmap5(CUtensorMap *m, const void *ptr, const uint64_t (&dims)[5],
                const uint64_t (&strides)[4], const uint32_t (&box)[5], bool swz64 = true);
bool tma_ok(const GemmArgs &g);

}  // namespace tc

// qf_gemm_tcw.cu: the wide (128 x 128) Gauss-form long-K kernel
bool tc3w_ok(const GemmArgs &g);
// qf_gemm_tcs.cu: streaming kernel for huge M with K = 16, N = 16 / 32
bool tc3s_ok(const GemmArgs &g);
int gemm_tc3s(const GemmArgs &g, cudaStream_t s);
bool tc3w_pair_ok(const GemmArgs &g);
int gemm_tc3w(const GemmArgs &g, cudaStream_t s, int ck, int pair);

}  // namespace qf

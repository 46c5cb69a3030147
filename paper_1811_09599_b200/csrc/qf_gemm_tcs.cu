// K2d -- streaming complex GEMM for a huge M with tiny K and N (K = 16,
// N = 16 or 32): the bond-16 region builds of config 5 (m x 16 x 16 with
// m = 2^24 .. 2^26), replacing the OpenBLAS cgemm behind `@` at
// rq/tensor_core.py:417 for those shapes.
//
// The generic short-K kernel (qf_gemm_tc.cu) ran them at 0.52 of HBM,
// issue-bound on per-tile bookkeeping (profiles/r2e_k16_full.txt: 57% of its
// warp instructions are ISETP/BRA/IMAD/IADD3/LOP3/SEL/LEA; a tile is only two
// k-blocks).  Here a tile is ONE pipeline step: the 128 x 16 block of A is one
// contiguous 16 KB TMA box (128-byte swizzle), a converter thread owns a row
// (8 LDS.128, 32 hi/lo splits, 8 tcgen05.st), the MMA lane issues the 12 real-
// block 3xTF32 MMAs of the tile against B' planes that were converted once per
// CTA, and the epilogue warps hand the 128 x N result to a TMA bulk store.
// HBM bound: 8 (K + N) bytes per row.
//
// Math: [Dre | Dim] += Ar.[Br | Bi] + Ai.[-Bi | Br] with a = hi + lo (TF32),
// a.b ~ ah.bh + ah.bl + al.bh (as qf_gemm_tc.cu).
#include <algorithm>

#include "qf_tc_ptx.cuh"

namespace qf {
namespace tcs {

using namespace tc;

constexpr int KS = 16;            // complex K (two tf32 k-blocks)
constexpr int RAW = 6;            // raw A tiles in flight (16 KB each)
constexpr int STAGES = 4;         // converted A tiles in TMEM (64 columns each)
constexpr int THREADS_S = 12 * 32;  // warps 0-3 convert, 4 TMA, 5 MMA, 6-7 idle, 8-11 epilogue

template <int BN>
struct Ls {
  static constexpr int NP = 2 * BN;                  // real N of one MMA: [Dre | Dim]
  static constexpr int B_BLOCK = BN * 32;            // BN n x 8 tf32, K-major core matrices
  static constexpr int B_PLANE = 3 * B_BLOCK;        // [-Bi | Br | Bi]
  static constexpr int B_KB = 2 * B_PLANE;           // hi plane, lo plane of one k-block
  static constexpr int RAW_SLOT = BM * KS * 8;       // 16 KB
  static constexpr int OUT_BOX = BM * 128;           // one 128-byte-wide store box
  static constexpr int OUT_SLOT = BM * BN * 8;       // BN / 16 boxes
  static constexpr int RAW_OFF = 0;
  static constexpr int OUT_OFF = RAW_OFF + RAW * RAW_SLOT;
  static constexpr int B_OFF = OUT_OFF + 2 * OUT_SLOT;
  static constexpr int BAR_OFF = B_OFF + 2 * B_KB;
  static constexpr int SMEM = BAR_OFF + 1024;
  static constexpr int A_COL0 = 2 * NP;              // after two accumulator buffers
  static constexpr int A_STAGE_COLS = 64;            // 2 k-blocks x (rh, rl, ih, il) x 8
  static_assert(A_COL0 + STAGES * A_STAGE_COLS <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(B_OFF % 1024 == 0 && OUT_SLOT % 1024 == 0, "TMA boxes are 1 KB aligned");
};

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int BN>
__global__ void __launch_bounds__(THREADS_S, 1)
    cgemm_tc3s_kernel(const __grid_constant__ GemmArgs g, uint32_t tiles,
                      const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmC) {
  using L = Ls<BN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *rawfull = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);  // [RAW]
  uint64_t *rawfree = rawfull + RAW;                                    // [RAW]
  uint64_t *afull = rawfree + RAW;                                      // [STAGES]
  uint64_t *afree = afull + STAGES;                                     // [STAGES]
  uint64_t *accfull = afree + STAGES;                                   // [2]
  uint64_t *accfree = accfull + 2;                                      // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accfree + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int i = 0; i < RAW; ++i) {
      mbar_init(&rawfull[i], 1);
      mbar_init(&rawfree[i], 4);
    }
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&afull[i], 4);
      mbar_init(&afree[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accfull[i], 1);
      mbar_init(&accfree[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B' planes, once per CTA: element (k, n) of B -> blocks [-Bi | Br | Bi] of
  // k-block k / 8, hi and lo planes (K-major core matrices: 8 n x 16 B)
  {
    const float2 *Bg = reinterpret_cast<const float2 *>(g.B);
    for (int e = tid; e < KS * BN; e += THREADS_S) {
      const int k = e % KS, n = e / KS;
      const float2 v = g.opB == QF_OP_N ? Bg[(int64_t)k * g.ldb + n] : Bg[(int64_t)n * g.ldb + k];
      uint32_t hr, lr, hi, li;
      split_fast(v.x, hr, lr);
      split_fast(v.y, hi, li);
      uint8_t *kb = smem + L::B_OFF + (k >> 3) * L::B_KB;
      const uint32_t off = core_off(n, (k & 7) >> 2) + (uint32_t)((k & 3) * 4);
      *reinterpret_cast<uint32_t *>(kb + 0 * L::B_BLOCK + off) = hi ^ 0x80000000u;
      *reinterpret_cast<uint32_t *>(kb + 1 * L::B_BLOCK + off) = hr;
      *reinterpret_cast<uint32_t *>(kb + 2 * L::B_BLOCK + off) = hi;
      *reinterpret_cast<uint32_t *>(kb + L::B_PLANE + 0 * L::B_BLOCK + off) = li ^ 0x80000000u;
      *reinterpret_cast<uint32_t *>(kb + L::B_PLANE + 1 * L::B_BLOCK + off) = lr;
      *reinterpret_cast<uint32_t *>(kb + L::B_PLANE + 2 * L::B_BLOCK + off) = li;
    }
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t0 = blockIdx.x, tstep = gridDim.x;

  if (warp == 4) {
    // ===== TMA producer: one 128 x 16 box of A per tile
    if (elect_one()) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      uint32_t f = 0;
      for (uint32_t t = t0; t < tiles; t += tstep, ++f) {
        const uint32_t slot = f % RAW;
        if (f >= RAW) mbar_wait(&rawfree[slot], ((f / RAW) + 1) & 1u);
        const uint32_t bar = smem_u32(&rawfull[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)L::RAW_SLOT)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem + L::RAW_OFF + slot * L::RAW_SLOT)),
            "l"(&tmA), "r"(0), "r"((int32_t)(t * BM)), "r"(bar)
            : "memory");
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ===== MMA issuer: 12 MMAs per tile (2 k-blocks x 6), accumulators double buffered
    const uint64_t dB = smem_desc(smem_u32(smem + L::B_OFF));
    constexpr uint32_t KB16 = (uint32_t)L::B_KB >> 4, BP16 = (uint32_t)L::B_PLANE >> 4,
                       BB16 = (uint32_t)L::B_BLOCK >> 4;
    constexpr uint32_t IDESC = idesc_tf32(BM, L::NP);
    uint32_t q = 0;
    for (uint32_t t = t0; t < tiles; t += tstep, ++q) {
      const uint32_t s = q % STAGES, buf = q & 1u;
      mbar_wait(&afull[s], (q / STAGES) & 1u);
      if (q >= 2) mbar_wait(&accfree[buf], ((q >> 1) + 1) & 1u);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d = tmem + buf * (uint32_t)L::NP;
#pragma unroll
        for (uint32_t kb = 0; kb < 2; ++kb) {
          const uint64_t bh = dB + (uint64_t)(kb * KB16), bl = bh + BP16;
          const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * (uint32_t)L::A_STAGE_COLS + kb * 32u;
          // [Dre|Dim] += Ar.[Br|Bi] + Ai.[-Bi|Br]: windows at B' blocks 1 and 0
          mma_ts(d, a + 0, bh + BB16, IDESC, kb);
          mma_ts(d, a + 0, bl + BB16, IDESC, 1u);
          mma_ts(d, a + 8, bh + BB16, IDESC, 1u);
          mma_ts(d, a + 16, bh, IDESC, 1u);
          mma_ts(d, a + 16, bl, IDESC, 1u);
          mma_ts(d, a + 24, bh, IDESC, 1u);
        }
        mma_commit(&afree[s]);
        mma_commit(&accfull[buf]);
      }
      __syncwarp();
    }
  } else if (warp >= 8) {
    // ===== epilogue warps (TMEM lane quadrant = warp - 8): accumulator ->
    // registers -> swizzled staging rows -> one TMA store per 16 columns
    const int lg = warp - 8, row = lg * 32 + lane;
    const float ar = (float)g.ar, ai = (float)g.ai;
    const bool plain = ar == 1.f && ai == 0.f;
    uint32_t q = 0;
    for (uint32_t t = t0; t < tiles; t += tstep, ++q) {
      const uint32_t buf = q & 1u;
      mbar_wait(&accfull[buf], (q >> 1) & 1u);
      tc_fence_after();
      // the staging slot of tile q - 2 must have been read by its store
      if (q >= 2 && tid == 8 * 32) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      named_bar(1, 128);
      uint8_t *out = smem + L::OUT_OFF + buf * L::OUT_SLOT;
      const uint32_t base = tmem + ((uint32_t)(lg * 32) << 16) + buf * (uint32_t)L::NP;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t vr[16], vi[16];
        tmem_ld16(base + c0, vr);
        tmem_ld16(base + BN + c0, vi);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c0 + 16 >= BN) {   // the accumulator is in registers: hand it back
          tc_fence_before();
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accfree[buf]))
                         : "memory");
        }
        uint8_t *rowp = out + (c0 / 16) * L::OUT_BOX + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {   // 16-byte chunk j of the row at chunk j ^ (row & 7)
          const float x0 = __uint_as_float(vr[2 * j]), y0 = __uint_as_float(vi[2 * j]);
          const float x1 = __uint_as_float(vr[2 * j + 1]), y1 = __uint_as_float(vi[2 * j + 1]);
          *reinterpret_cast<float4 *>(rowp + ((j ^ (row & 7)) << 4)) =
              plain ? make_float4(x0, y0, x1, y1)
                    : make_float4(ar * x0 - ai * y0, ar * y0 + ai * x0, ar * x1 - ai * y1,
                                  ar * y1 + ai * x1);
        }
      }
      fence_async_smem();
      named_bar(1, 128);
      if (tid == 8 * 32) {
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 16)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::
                           "l"(&tmC), "r"(2 * c0), "r"((int32_t)(t * BM)),
                       "r"(smem_u32(out + (c0 / 16) * L::OUT_BOX))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (tid == 8 * 32) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp < 4) {
    // ===== converter warps: thread = A row = TMEM lane; raw row (128 B, 128-byte
    // swizzle: chunk c at c ^ (row & 7)) -> hi/lo planes of both k-blocks
    const int row = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    uint32_t q = 0;
    for (uint32_t t = t0; t < tiles; t += tstep, ++q) {
      const uint32_t slot = q % RAW, s = q % STAGES;
      mbar_wait(&rawfull[slot], (q / RAW) & 1u);
      const uint8_t *rp = smem + L::RAW_OFF + slot * L::RAW_SLOT + row * 128;
      float4 av[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) av[c] = *reinterpret_cast<const float4 *>(rp + ((c ^ (row & 7)) << 4));
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rawfree[slot]))
                     : "memory");
      if (q >= STAGES) mbar_wait(&afree[s], ((q / STAGES) + 1) & 1u);
      const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * L::A_STAGE_COLS);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        uint32_t rh[8], rl[8], ih[8], il[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = av[4 * kb + c];
          split_fast(v.x, rh[2 * c], rl[2 * c]);
          split_fast(v.y, ih[2 * c], il[2 * c]);
          split_fast(v.z, rh[2 * c + 1], rl[2 * c + 1]);
          split_fast(v.w, ih[2 * c + 1], il[2 * c + 1]);
        }
        tmem_st8(acol + kb * 32 + 0, rh);
        tmem_st8(acol + kb * 32 + 8, rl);
        tmem_st8(acol + kb * 32 + 16, ih);
        tmem_st8(acol + kb * 32 + 24, il);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&afull[s])) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// 2-D float tensor map: rows of `inner` floats, 128-byte-swizzled {32, 128} boxes
static bool make_tmap2(CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t rows,
                       uint64_t row_bytes) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const cuuint64_t dims[2] = {inner, rows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {32, 128};
  const cuuint32_t es[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box,
                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static int launch_stream(const GemmArgs &g, cudaStream_t s) {
  using L = Ls<BN>;
  auto kern = cgemm_tc3s_kernel<BN>;
  CUtensorMap tmA{}, tmC{};
  if (!make_tmap2(&tmA, g.A, 2 * KS, g.M, KS * 8) || !make_tmap2(&tmC, g.C, 2 * BN, g.M, BN * 8)) {
    set_error("tc3s: cuTensorMapEncodeTiled failed (M=%lld N=%lld)", (long long)g.M, (long long)g.N);
    return QF_ERR_CUDA;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3s: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  const int64_t tiles = (g.M + BM - 1) / BM;
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)sm_count());
  kern<<<(unsigned)grid, THREADS_S, L::SMEM, s>>>(g, (uint32_t)tiles, tmA, tmC);
  return check_launch("cgemm_tc3s");
}

}  // namespace tcs

// One entry, A row-major and dense ([M][16]), C dense ([M][N]), no beta, no
// offset tables / views, enough rows to fill the machine.
bool tc3s_ok(const GemmArgs &g) {
  if (g.batch != 1 || g.K != tcs::KS || (g.N != 16 && g.N != 32)) return false;
  if (g.opA != QF_OP_N || g.lda != g.K || g.ldc != g.N) return false;
  if (g.a_roff || g.a_boff || g.b_boff || g.v_kin || g.c_trans || g.c_nblk || g.a_rin) return false;
  if (g.br != 0.0 || g.bi != 0.0) return false;
  if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.C) & 15)) return false;
  return g.M >= 128 * 148 && g.M < ((int64_t)1 << 31) - 128;
}

int gemm_tc3s(const GemmArgs &g, cudaStream_t s) {
  return g.N == 16 ? tcs::launch_stream<16>(g, s) : tcs::launch_stream<32>(g, s);
}

}  // namespace qf

// K2 -- complex64 GEMM on the 5th-generation tensor cores (tcgen05,
// kind::tf32) with a 3xTF32 split, for sm_100a.
//
// Replaces the OpenBLAS cgemm behind `@` at rq/tensor_core.py:417 for the
// shapes that fill tensor-core tiles.
//
// Math.  Per complex index k the real-block form
//     [Dre | Dim] += Ar[:,k] x [ Br | Bi ]  +  Ai[:,k] x [ -Bi | Br ]
// turns one complex MAC into two real MMAs with N' = 2*BN.  Each operand
// x is split x = hi + lo with hi = tf32(x), lo = tf32(x - hi), and
// a*b ~ ah*bh + ah*bl + al*bh (3 MMAs) keeps ~fp32 accuracy -- six
// tcgen05.mma per 8 complex k.  Algorithmic flops = 8*M*N*K as in the
// reference's cost model; the tensor pipe issues 3x the flops of a 1xTF32
// complex GEMM, so the roofline is TF32_peak / 3.
//
// Data flow per CTA (128 threads = 4 warps, one 128 x BN complex C tile):
//   global (any N/T layout, complex64) --ld.global--> registers (2-deep
//   prefetch) --split hi/lo--> B' planes in shared memory, in the UMMA
//   K-major SWIZZLE_NONE core-matrix layout, stored once as three row
//   blocks [-Bi | Br | Bi] so [Br|Bi] and [-Bi|Br] are both contiguous
//   descriptor windows; A planes (Ar/Ai x hi/lo) either in shared memory
//   (SS variant) or written straight into tensor memory with tcgen05.st
//   (TS variant: thread t owns row t == TMEM lane t, A never touches smem,
//   which halves the smem traffic of the MMAs).  One elected thread issues
//   the six MMAs per stage and tcgen05.commit's an mbarrier that frees the
//   stage; a ring of S stages keeps the tensor pipe busy while the next
//   stages are converted.  Accumulators [Dre | Dim] live in TMEM
//   (2*BN fp32 columns); the epilogue reads them with tcgen05.ld, applies
//   alpha/beta and writes interleaved complex64.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>
#include <utility>

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

// ---------------------------------------------------------------------------

template <int BN, int STAGES, bool A_TMEM>
struct Layout {
  static constexpr int NP = 2 * BN;                       // real MMA N
  static constexpr int B_BLOCK = BN * 32;                 // bytes of one BN-row block (8 tf32)
  static constexpr int B_PLANE = 3 * B_BLOCK;             // [-Bi | Br | Bi]
  static constexpr int B_STAGE = 2 * B_PLANE;             // hi, lo
  static constexpr int A_PLANE = BM * 32;                 // 128 rows x 8 tf32
  static constexpr int A_STAGE = A_TMEM ? 0 : 4 * A_PLANE;  // re_hi, re_lo, im_hi, im_lo
  static constexpr int STAGE = B_STAGE + A_STAGE;
  static constexpr int SMEM = STAGES * STAGE + 1024;     // + barriers / tmem slot
  static constexpr int ACC_COLS = NP;
  static constexpr int A_COLS = A_TMEM ? STAGES * 32 : 0;
  static constexpr int TMEM_COLS = (ACC_COLS + A_COLS) <= 128   ? 128
                                   : (ACC_COLS + A_COLS) <= 256 ? 256
                                                                : 512;
};

template <int BN, int STAGES, bool A_TMEM>
__global__ void __launch_bounds__(THREADS, 1)
    cgemm_tc3_kernel(const __grid_constant__ GemmArgs g, int64_t tiles_n, int64_t tiles) {
  using L = Layout<BN, STAGES, A_TMEM>;
  static_assert(BN == 128 || BN == 64, "BN");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * L::STAGE);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + STAGES + 1);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t d_tmem = tmem;                      // accumulators: cols [0, 2*BN)
  const uint32_t a_tmem = tmem + L::ACC_COLS;        // TS: A planes after the accumulators
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  constexpr uint32_t IDESC = idesc_tf32(BM, L::NP);

  const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
  const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
  float2 *Cb = reinterpret_cast<float2 *>(g.C);
  const int64_t nk = (g.K + KB - 1) / KB;
  // B elements per thread per stage: KB * BN / THREADS
  constexpr int BE = KB * BN / THREADS;  // 8 (BN=128) or 4 (BN=64)
  uint32_t phase_bits = 0;              // per-stage parity of the next wait

  for (int64_t work = blockIdx.x; work < tiles * g.batch; work += gridDim.x) {
    const int64_t bidx = work / tiles;
    const int64_t tile = work - bidx * tiles;
    const int64_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    const float2 *A = Ab + a_batch_off(g, bidx);
    const float2 *B = Bb + b_batch_off(g, bidx);
    float2 *C = Cb + bidx * g.sC;

    // thread -> operand element mapping
    const int64_t am = m0 + tid;                      // A row owned by this thread
    // B: thread owns column n = n0 + (tid % BN), k in [kq*BE, kq*BE+BE)
    const int bn_local = tid % BN;
    const int kq = tid / BN;
    const int64_t bn = n0 + bn_local;

    float2 ra[2][KB], rb[2][BE];
    auto load = [&](auto bufc, int64_t kb) {
      constexpr int buf = decltype(bufc)::value;
      const int64_t k0 = kb * KB;
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int64_t gk = k0 + k;
        float2 v = make_float2(0.f, 0.f);
        if (am < g.M && gk < g.K)
          v = (g.opA == QF_OP_N) ? __ldg(A + am * g.lda + gk) : __ldg(A + gk * g.lda + am);
        ra[buf][k] = v;
      }
#pragma unroll
      for (int e = 0; e < BE; ++e) {
        const int64_t gk = k0 + kq * BE + e;
        float2 v = make_float2(0.f, 0.f);
        if (bn < g.N && gk < g.K)
          v = (g.opB == QF_OP_N) ? __ldg(B + gk * g.ldb + bn) : __ldg(B + bn * g.ldb + gk);
        rb[buf][e] = v;
      }
    };

    auto convert = [&](auto bufc, int s) {
      constexpr int buf = decltype(bufc)::value;
      uint8_t *stage = smem + s * L::STAGE;
      // ---- B planes: rows [-Bi | Br | Bi], hi then lo
      {
        uint32_t hr[BE], lr[BE], hi_[BE], li[BE];
#pragma unroll
        for (int e = 0; e < BE; ++e) {
          split3(rb[buf][e].x, hr[e], lr[e]);
          split3(rb[buf][e].y, hi_[e], li[e]);
        }
        // BE consecutive k: BE==8 -> two 16 B chunks, BE==4 -> one chunk (chunk kq)
#pragma unroll
        for (int c = 0; c < BE / 4; ++c) {
          const int chunk = (BE == 8) ? c : kq;
          const uint32_t off = core_off(bn_local, chunk);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint8_t *plane = stage + h * L::B_PLANE;
            const uint32_t *re = h ? lr : hr;
            const uint32_t *im = h ? li : hi_;
            uint4 vneg = make_uint4(im[4 * c] ^ 0x80000000u, im[4 * c + 1] ^ 0x80000000u,
                                    im[4 * c + 2] ^ 0x80000000u, im[4 * c + 3] ^ 0x80000000u);
            uint4 vre = make_uint4(re[4 * c], re[4 * c + 1], re[4 * c + 2], re[4 * c + 3]);
            uint4 vim = make_uint4(im[4 * c], im[4 * c + 1], im[4 * c + 2], im[4 * c + 3]);
            *reinterpret_cast<uint4 *>(plane + 0 * L::B_BLOCK + off) = vneg;
            *reinterpret_cast<uint4 *>(plane + 1 * L::B_BLOCK + off) = vre;
            *reinterpret_cast<uint4 *>(plane + 2 * L::B_BLOCK + off) = vim;
          }
        }
      }
      // ---- A planes for row `tid`: re_hi, re_lo, im_hi, im_lo
      uint32_t p[4][KB];
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        split3(ra[buf][k].x, p[0][k], p[1][k]);
        split3(ra[buf][k].y, p[2][k], p[3][k]);
      }
      if constexpr (A_TMEM) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          tmem_st8(a_tmem + lane_base + (uint32_t)(s * 32 + q * 8), p[q]);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else {
        uint8_t *ab = stage + L::B_STAGE;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            *reinterpret_cast<uint4 *>(ab + q * L::A_PLANE + core_off(tid, c)) =
                make_uint4(p[q][4 * c], p[q][4 * c + 1], p[q][4 * c + 2], p[q][4 * c + 3]);
      }
    };

    auto issue = [&](int s, int64_t kb) {
      uint8_t *stage = smem + s * L::STAGE;
      const uint32_t bhi = smem_u32(stage), blo = smem_u32(stage + L::B_PLANE);
      // [Br | Bi] window starts at block 1; [-Bi | Br] at block 0
      const uint64_t b1h = smem_desc(bhi + L::B_BLOCK), b1l = smem_desc(blo + L::B_BLOCK);
      const uint64_t b2h = smem_desc(bhi), b2l = smem_desc(blo);
      const uint32_t acc0 = kb > 0 ? 1u : 0u;
      if constexpr (A_TMEM) {
        const uint32_t a = a_tmem + (uint32_t)(s * 32);
        mma_ts(d_tmem, a + 0, b1h, IDESC, acc0);   // re_hi x [Br|Bi]_hi
        mma_ts(d_tmem, a + 0, b1l, IDESC, 1u);     // re_hi x [Br|Bi]_lo
        mma_ts(d_tmem, a + 8, b1h, IDESC, 1u);     // re_lo x [Br|Bi]_hi
        mma_ts(d_tmem, a + 16, b2h, IDESC, 1u);    // im_hi x [-Bi|Br]_hi
        mma_ts(d_tmem, a + 16, b2l, IDESC, 1u);    // im_hi x [-Bi|Br]_lo
        mma_ts(d_tmem, a + 24, b2h, IDESC, 1u);    // im_lo x [-Bi|Br]_hi
      } else {
        const uint32_t ab = smem_u32(stage + L::B_STAGE);
        const uint64_t arh = smem_desc(ab), arl = smem_desc(ab + L::A_PLANE);
        const uint64_t aih = smem_desc(ab + 2 * L::A_PLANE), ail = smem_desc(ab + 3 * L::A_PLANE);
        mma_ss(d_tmem, arh, b1h, IDESC, acc0);
        mma_ss(d_tmem, arh, b1l, IDESC, 1u);
        mma_ss(d_tmem, arl, b1h, IDESC, 1u);
        mma_ss(d_tmem, aih, b2h, IDESC, 1u);
        mma_ss(d_tmem, aih, b2l, IDESC, 1u);
        mma_ss(d_tmem, ail, b2h, IDESC, 1u);
      }
      mma_commit(&bars[s]);
    };

    using B0 = std::integral_constant<int, 0>;
    using B1 = std::integral_constant<int, 1>;
    auto step = [&](auto bufc, int64_t kb) {
      const int s = (int)(kb % STAGES);
      if (kb >= STAGES) {
        mbar_wait(&bars[s], (phase_bits >> s) & 1u);
        phase_bits ^= 1u << s;
      }
      convert(bufc, s);
      if (kb + 2 < nk) load(bufc, kb + 2);
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        issue(s, kb);
      }
    };
    if (nk > 0) load(B0{}, 0);
    if (nk > 1) load(B1{}, 1);
    for (int64_t kb = 0; kb < nk; kb += 2) {
      step(B0{}, kb);
      if (kb + 1 < nk) step(B1{}, kb + 1);
    }
    // drain: wait for every stage's outstanding commit (the last STAGES k-blocks)
    for (int64_t kb = (nk > STAGES ? nk - STAGES : 0); kb < nk; ++kb) {
      const int s = (int)(kb % STAGES);
      mbar_wait(&bars[s], (phase_bits >> s) & 1u);
      phase_bits ^= 1u << s;
    }
    tc_fence_after();

    // ---- epilogue: TMEM -> registers -> C (row tid of the tile)
    const int64_t row = m0 + tid;
    const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
    const bool use_beta = (br != 0.f || bi != 0.f);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t vr[32], vi[32];
      tmem_ld32(d_tmem + lane_base + (uint32_t)c0, vr);
      tmem_ld32(d_tmem + lane_base + (uint32_t)(BN + c0), vi);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < g.M && nk > 0) {
        float2 *crow = C + row * g.ldc + n0 + c0;
        const int64_t ncols = min((int64_t)32, g.N - (n0 + c0));
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < ncols) {
            const float x = __uint_as_float(vr[j]), y = __uint_as_float(vi[j]);
            float2 o = make_float2(ar * x - ai * y, ar * y + ai * x);
            if (use_beta) {
              const float2 c = crow[j];
              o.x += br * c.x - bi * c.y;
              o.y += br * c.y + bi * c.x;
            }
            crow[j] = o;
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();  // all TMEM reads done before the next tile's MMAs overwrite
    tc_fence_after();
  }

  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
}

template <int BN, int STAGES, bool A_TMEM>
int launch(const GemmArgs &g, cudaStream_t s) {
  using L = Layout<BN, STAGES, A_TMEM>;
  auto kern = cgemm_tc3_kernel<BN, STAGES, A_TMEM>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  const int64_t tiles_n = (g.N + BN - 1) / BN, tiles_m = (g.M + BM - 1) / BM;
  const int64_t tiles = tiles_n * tiles_m;
  const int64_t work = tiles * g.batch;
  const int64_t grid = std::min<int64_t>(work, (int64_t)sm_count());
  kern<<<(unsigned)grid, THREADS, L::SMEM, s>>>(g, tiles_n, tiles);
  return check_launch("cgemm_tc3");
}


// ---------------------------------------------------------------------------
// v2: promoted accumulation.  The tensor pipe's fp32 accumulation truncates,
// so error grows ~linearly with K (measured: 1.4e-8 * K relative).  As in
// DeepGEMM's FP8 "promotion", each chunk of CK k-blocks accumulates fresh in
// one of two TMEM partial buffers; after the chunk's MMAs retire the CUDA
// cores add that partial into fp32 registers (round-to-nearest) while the
// tensor pipe fills the other buffer.  256 threads: warp w owns TMEM lanes
// 32*(w%4).. and half (w/4) of every row's columns.

constexpr int V2_THREADS = 256;
constexpr int V2_BN = 64;

__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c,
                                         uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

template <int STAGES, int CK>
struct LayoutV2 {
  static constexpr int BN = V2_BN;
  static constexpr int NP = 2 * BN;            // 128 real columns per partial
  static constexpr int B_BLOCK = BN * 32;
  static constexpr int B_PLANE = 3 * B_BLOCK;
  static constexpr int STAGE = 2 * B_PLANE;    // B planes only (A lives in TMEM)
  static constexpr int SMEM = STAGES * STAGE + 1024;
  static constexpr int P_COLS = NP;            // one partial buffer
  static constexpr int A_COL0 = 2 * P_COLS;    // A ring after the two partials
  static constexpr int TMEM_COLS = 512;
  static_assert(2 * P_COLS + STAGES * 32 <= 512, "TMEM budget");
};

template <int STAGES, int CK>
__global__ void __launch_bounds__(V2_THREADS, 1)
    cgemm_tc3p_kernel(const __grid_constant__ GemmArgs g, int64_t tiles_n, int64_t tiles) {
  using L = LayoutV2<STAGES, CK>;
  constexpr int BN = L::BN;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * L::STAGE);  // [STAGES]
  uint64_t *pbar = bars + STAGES;                                           // [2] chunk done
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(pbar + 2);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3;       // TMEM lane group
  const int half = warp >> 2;    // which half of the columns / k
  const int row_l = lg * 32 + lane;

  if (tid == 0) {
    for (int s = 0; s < STAGES + 2; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
  constexpr uint32_t IDESC = idesc_tf32(BM, L::NP);

  const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
  const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
  float2 *Cb = reinterpret_cast<float2 *>(g.C);
  const int64_t nk = (g.K + KB - 1) / KB;
  const int64_t nchunks = (nk + CK - 1) / CK;
  constexpr int BE = KB * BN / V2_THREADS;  // 2 B elements (consecutive k) per thread
  uint32_t phase_bits = 0;                  // bits [0,STAGES): stage barriers; +STAGES: partials

  for (int64_t work = blockIdx.x; work < tiles * g.batch; work += gridDim.x) {
    const int64_t bidx = work / tiles;
    const int64_t tile = work - bidx * tiles;
    const int64_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    const float2 *A = Ab + a_batch_off(g, bidx);
    const float2 *B = Bb + b_batch_off(g, bidx);
    float2 *C = Cb + bidx * g.sC;
    const int64_t am = m0 + row_l;           // A row (this thread: k in [4*half, 4*half+4))
    const int bn_local = tid % BN;
    const int kq = tid / BN;                 // 0..3 -> k = 2*kq, 2*kq+1
    const int64_t bn = n0 + bn_local;

    float racc[32], iacc[32];                // promoted sums: columns n0 + 32*half + j
#pragma unroll
    for (int j = 0; j < 32; ++j) racc[j] = iacc[j] = 0.f;

    float2 ra[2][4], rb[2][BE];
    auto load = [&](auto bufc, int64_t kb) {
      constexpr int buf = decltype(bufc)::value;
      const int64_t k0 = kb * KB;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t gk = k0 + 4 * half + k;
        float2 v = make_float2(0.f, 0.f);
        if (am < g.M && gk < g.K)
          v = (g.opA == QF_OP_N) ? __ldg(A + am * g.lda + gk) : __ldg(A + gk * g.lda + am);
        ra[buf][k] = v;
      }
#pragma unroll
      for (int e = 0; e < BE; ++e) {
        const int64_t gk = k0 + kq * BE + e;
        float2 v = make_float2(0.f, 0.f);
        if (bn < g.N && gk < g.K)
          v = (g.opB == QF_OP_N) ? __ldg(B + gk * g.ldb + bn) : __ldg(B + bn * g.ldb + gk);
        rb[buf][e] = v;
      }
    };
    auto convert = [&](auto bufc, int s) {
      constexpr int buf = decltype(bufc)::value;
      uint8_t *stage = smem + s * L::STAGE;
      uint32_t hr[BE], lr[BE], hi_[BE], li[BE];
#pragma unroll
      for (int e = 0; e < BE; ++e) {
        split3(rb[buf][e].x, hr[e], lr[e]);
        split3(rb[buf][e].y, hi_[e], li[e]);
      }
      const int kfirst = kq * BE;  // 0,2,4,6
      const uint32_t off = core_off(bn_local, kfirst >> 2) + (uint32_t)((kfirst & 3) * 4);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint8_t *plane = stage + h * L::B_PLANE;
        const uint32_t *re = h ? lr : hr;
        const uint32_t *im = h ? li : hi_;
        *reinterpret_cast<uint2 *>(plane + 0 * L::B_BLOCK + off) =
            make_uint2(im[0] ^ 0x80000000u, im[1] ^ 0x80000000u);
        *reinterpret_cast<uint2 *>(plane + 1 * L::B_BLOCK + off) = make_uint2(re[0], re[1]);
        *reinterpret_cast<uint2 *>(plane + 2 * L::B_BLOCK + off) = make_uint2(im[0], im[1]);
      }
      uint32_t p[4][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        split3(ra[buf][k].x, p[0][k], p[1][k]);
        split3(ra[buf][k].y, p[2][k], p[3][k]);
      }
      const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * 32 + 4 * half);
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_st4(acol + q * 8, p[q][0], p[q][1], p[q][2], p[q][3]);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    };
    auto promote = [&](int pb) {
      // wait for the chunk that used partial buffer pb, then add it into registers
      mbar_wait(&pbar[pb], (phase_bits >> (STAGES + pb)) & 1u);
      phase_bits ^= 1u << (STAGES + pb);
      tc_fence_after();
      uint32_t v[32];
      const uint32_t base = tmem + lane_base + (uint32_t)(pb * L::P_COLS + 32 * half);
      tmem_ld32(base, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) racc[j] += __uint_as_float(v[j]);
      tmem_ld32(base + BN, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) iacc[j] += __uint_as_float(v[j]);
    };
    auto issue = [&](int s, int64_t kb) {
      const int64_t chunk = kb / CK;
      const int pos = (int)(kb - chunk * CK);
      const uint32_t d = tmem + (uint32_t)((chunk & 1) * L::P_COLS);
      uint8_t *stage = smem + s * L::STAGE;
      const uint32_t bhi = smem_u32(stage), blo = smem_u32(stage + L::B_PLANE);
      const uint64_t b1h = smem_desc(bhi + L::B_BLOCK), b1l = smem_desc(blo + L::B_BLOCK);
      const uint64_t b2h = smem_desc(bhi), b2l = smem_desc(blo);
      const uint32_t a = tmem + (uint32_t)(L::A_COL0 + s * 32);
      const uint32_t acc0 = pos > 0 ? 1u : 0u;
      mma_ts(d, a + 0, b1h, IDESC, acc0);
      mma_ts(d, a + 0, b1l, IDESC, 1u);
      mma_ts(d, a + 8, b1h, IDESC, 1u);
      mma_ts(d, a + 16, b2h, IDESC, 1u);
      mma_ts(d, a + 16, b2l, IDESC, 1u);
      mma_ts(d, a + 24, b2h, IDESC, 1u);
      mma_commit(&bars[s]);
      if (pos == CK - 1 || kb == nk - 1) mma_commit(&pbar[chunk & 1]);
    };

    using B0 = std::integral_constant<int, 0>;
    using B1 = std::integral_constant<int, 1>;
    auto step = [&](auto bufc, int64_t kb) {
      const int s = (int)(kb % STAGES);
      if (kb >= STAGES) {
        mbar_wait(&bars[s], (phase_bits >> s) & 1u);
        phase_bits ^= 1u << s;
      }
      convert(bufc, s);
      if (kb + 2 < nk) load(bufc, kb + 2);
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        issue(s, kb);
      }
      // one chunk behind: promote the previous chunk's partial
      const int64_t chunk = kb / CK;
      if (kb == chunk * CK && chunk >= 1) promote((int)((chunk - 1) & 1));
    };
    if (nk > 0) load(B0{}, 0);
    if (nk > 1) load(B1{}, 1);
    for (int64_t kb = 0; kb < nk; kb += 2) {
      step(B0{}, kb);
      if (kb + 1 < nk) step(B1{}, kb + 1);
    }
    if (nchunks > 0) promote((int)((nchunks - 1) & 1));
    // drain the stage barriers of the last STAGES k-blocks (keeps parity in sync)
    for (int64_t kb = (nk > STAGES ? nk - STAGES : 0); kb < nk; ++kb) {
      const int s = (int)(kb % STAGES);
      mbar_wait(&bars[s], (phase_bits >> s) & 1u);
      phase_bits ^= 1u << s;
    }

    // ---- epilogue from registers: row row_l, columns n0 + 32*half + j
    const int64_t row = m0 + row_l;
    if (row < g.M) {
      const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
      const bool use_beta = (br != 0.f || bi != 0.f);
      const int64_t c0 = n0 + 32 * half;
      float2 *crow = C + row * g.ldc + c0;
      const int64_t ncols = min((int64_t)32, g.N - c0);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < ncols) {
          float2 o = make_float2(ar * racc[j] - ai * iacc[j], ar * iacc[j] + ai * racc[j]);
          if (use_beta) {
            const float2 c = crow[j];
            o.x += br * c.x - bi * c.y;
            o.y += br * c.y + bi * c.x;
          }
          crow[j] = o;
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
}

template <int STAGES, int CK>
int launch_v2(const GemmArgs &g, cudaStream_t s) {
  using L = LayoutV2<STAGES, CK>;
  auto kern = cgemm_tc3p_kernel<STAGES, CK>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3p: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  const int64_t tiles_n = (g.N + L::BN - 1) / L::BN, tiles_m = (g.M + BM - 1) / BM;
  const int64_t tiles = tiles_n * tiles_m;
  const int64_t grid = std::min<int64_t>(tiles * g.batch, (int64_t)sm_count());
  kern<<<(unsigned)grid, V2_THREADS, L::SMEM, s>>>(g, tiles_n, tiles);
  return check_launch("cgemm_tc3p");
}

// ---------------------------------------------------------------------------
// v3 ("stream"): v2's math (A in TMEM, promoted accumulation, BN = 64) fed by
// an asynchronous operand stream.  Every thread owns fixed operand elements
// of every k-block (A: 4 consecutive k of one row; B: 2 consecutive k of one
// column) and fetches them with cp.async into its private slots of a
// RAW-deep shared-memory ring, so it converts exactly the bytes it fetched
// after cp.async.wait_group -- no block barrier between fetch and convert.
// The fetch cursor walks source pointers incrementally and runs RAW-1
// k-blocks ahead across tile boundaries (the next tile's operands stream in
// while the current tile's epilogue runs).  Rings are powers of two and all
// per-k-block index math is 32-bit.  tf32 hi/lo splitting is two integer
// ops + one FADD (inputs are finite).

__device__ __forceinline__ void split_fast(float x, uint32_t &hi, uint32_t &lo) {
  const uint32_t h = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;  // round-half-away to tf32
  hi = h;
  lo = __float_as_uint(x - __uint_as_float(h));  // exact; the tensor core keeps its top 19 bits
}

template <int STAGES, int CK, int RAW>
struct LayoutV3 {
  static_assert((STAGES & (STAGES - 1)) == 0 && (CK & (CK - 1)) == 0 && (RAW & (RAW - 1)) == 0,
                "rings must be powers of two");
  static constexpr int BN = V2_BN;
  static constexpr int NP = 2 * BN;
  static constexpr int B_BLOCK = BN * 32;
  static constexpr int B_PLANE = 3 * B_BLOCK;
  static constexpr int STAGE = 2 * B_PLANE;                 // B planes per stage
  static constexpr int RAWA_SLOT = V2_THREADS * 32;         // 4 complex of A per thread
  static constexpr int RAWB_SLOT = V2_THREADS * 16;         // 2 complex of B per thread
  static constexpr int RAWA_OFF = STAGES * STAGE;
  static constexpr int RAWB_OFF = RAWA_OFF + RAW * RAWA_SLOT;
  static constexpr int BAR_OFF = RAWB_OFF + RAW * RAWB_SLOT;
  static constexpr int COFF_OFF = BAR_OFF + 1024;           // gathered-A K offsets (int32)
  static constexpr int COFF_MAX = 4096;
  static constexpr int SMEM = COFF_OFF + 4 * COFF_MAX;
  static constexpr int P_COLS = NP;
  static constexpr int A_COL0 = 2 * P_COLS;
  static constexpr int TMEM_COLS = 512;
  static constexpr int LOG_STAGES = STAGES == 1 ? 0 : STAGES == 2 ? 1 : STAGES == 4 ? 2 : 3;
  static constexpr int LOG_CK = CK == 1 ? 0 : CK == 2 ? 1 : CK == 4 ? 2 : CK == 8 ? 3 : 4;
  static_assert(2 * P_COLS + STAGES * 32 <= 512, "TMEM budget");
};

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

template <int STAGES, int CK, int RAW>
__global__ void __launch_bounds__(V2_THREADS, 1)
    cgemm_tc3s_kernel(const __grid_constant__ GemmArgs g, int64_t tiles_n, int64_t tiles) {
  using L = LayoutV3<STAGES, CK, RAW>;
  constexpr int BN = L::BN;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);  // [STAGES]
  uint64_t *pbar = bars + STAGES;                                    // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(pbar + 2);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3, half = warp >> 2;
  const int row_l = lg * 32 + lane;              // A row / TMEM lane of this thread
  // B mapping: two threads share one 16-byte core-matrix row segment, so a
  // 16-lane phase writes 8 rows x 16 B = 128 contiguous bytes (no conflicts)
  const int b_kp = tid & 1;                      // which k pair inside a 4-k chunk
  const int b_n = (tid >> 1) & (BN - 1);         // B column (row of B')
  const int b_chunk = tid >> 7;                  // k 0-3 or 4-7
  const int b_k = b_chunk * 4 + b_kp * 2;        // first of the thread's two k

  if (tid == 0) {
    for (int i = 0; i < STAGES + 2; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
  constexpr uint32_t IDESC = idesc_tf32(BM, L::NP);
  // A slot = two 16-byte lanes per thread, each lane contiguous across threads,
  // so the 128-bit accesses of a quarter warp hit 8 distinct bank groups
  const uint32_t rawa0 = smem_u32(smem + L::RAWA_OFF) + (uint32_t)tid * 16;
  const uint32_t rawb0 = smem_u32(smem + L::RAWB_OFF) + (uint32_t)tid * 16;
  const uint32_t boff = core_off(b_n, b_chunk) + (uint32_t)(b_kp * 8);

  const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
  const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
  float2 *Cb = reinterpret_cast<float2 *>(g.C);
  const uint32_t nk = (uint32_t)((g.K + KB - 1) / KB);
  const bool k_tail = (g.K % KB) != 0;
  const int64_t total_work = tiles * g.batch;
  const bool a_vec = (g.opA == QF_OP_N) && (g.lda % 2 == 0) && (g.sA % 2 == 0);
  const bool b_vec = (g.opB == QF_OP_T) && (g.ldb % 2 == 0) && (g.sB % 2 == 0);
  const int64_t a_kstride = (g.opA == QF_OP_N) ? 1 : g.lda;   // elements between consecutive k
  const int64_t b_kstride = (g.opB == QF_OP_N) ? g.ldb : 1;

  // ---- fetch cursor: incremental source pointers, set up once per tile
  int64_t f_work = blockIdx.x;
  uint32_t f_kb = 0;
  const float2 *fa = Ab, *fb = Bb;
  bool fa_ok = false, fb_ok = false;
  auto fetch_setup = [&]() {
    if (f_work >= total_work) return;
    const int64_t bidx = f_work / tiles;
    const int64_t tile = f_work - bidx * tiles;
    const int64_t am = (tile / tiles_n) * BM + row_l;
    const int64_t bn = (tile % tiles_n) * BN + b_n;
    fa_ok = am < g.M;
    fb_ok = bn < g.N;
    const float2 *A = Ab + a_batch_off(g, bidx);
    const float2 *B = Bb + b_batch_off(g, bidx);
    fa = (g.opA == QF_OP_N) ? A + am * g.lda + 4 * half : A + (int64_t)(4 * half) * g.lda + am;
    fb = (g.opB == QF_OP_N) ? B + (int64_t)b_k * g.ldb + bn : B + bn * g.ldb + b_k;
    if (!fa_ok) fa = Ab;
    if (!fb_ok) fb = Bb;
  };
  auto fetch = [&](uint32_t slot) {
    if (f_work < total_work) {
      const uint32_t da = rawa0 + slot * L::RAWA_SLOT, db = rawb0 + slot * L::RAWB_SLOT;
      if (!(k_tail && f_kb == nk - 1)) {
        if (a_vec) {
          cp_async16(da, fa, fa_ok);
          cp_async16(da + V2_THREADS * 16, fa + 2, fa_ok);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            cp_async8(da + (k >> 1) * V2_THREADS * 16 + (k & 1) * 8, fa + k * a_kstride, fa_ok);
        }
        if (b_vec) {
          cp_async16(db, fb, fb_ok);
        } else {
          cp_async8(db, fb, fb_ok);
          cp_async8(db + 8, fb + b_kstride, fb_ok);
        }
      } else {  // ragged last k-block: per-element predicates
        const int64_t k0 = (int64_t)f_kb * KB;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool ok = fa_ok && k0 + 4 * half + k < g.K;
          cp_async8(da + (k >> 1) * V2_THREADS * 16 + (k & 1) * 8, ok ? fa + k * a_kstride : Ab, ok);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = fb_ok && k0 + b_k + e < g.K;
          cp_async8(db + 8 * e, ok ? fb + e * b_kstride : Bb, ok);
        }
      }
      if (fa_ok) fa += KB * a_kstride;
      if (fb_ok) fb += KB * b_kstride;
      if (++f_kb == nk) {
        f_kb = 0;
        f_work += gridDim.x;
        fetch_setup();
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // uniform group count
  };

  uint32_t q = 0;            // k-blocks consumed by this CTA (drives every ring)
  uint32_t pwaits[2] = {0, 0};
  fetch_setup();
  for (int i = 0; i < RAW - 1; ++i) fetch((uint32_t)i);

  for (int64_t work = blockIdx.x; work < total_work; work += gridDim.x) {
    const int64_t bidx = work / tiles;
    const int64_t tile = work - bidx * tiles;
    const int64_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    float2 *C = Cb + bidx * g.sC;
    float racc[32], iacc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) racc[j] = iacc[j] = 0.f;

    auto promote = [&](int pb) {
      mbar_wait(&pbar[pb], pwaits[pb] & 1u);
      ++pwaits[pb];
      tc_fence_after();
      uint32_t v[32];
      const uint32_t base = tmem + lane_base + (uint32_t)(pb * L::P_COLS + 32 * half);
      tmem_ld32(base, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) racc[j] += __uint_as_float(v[j]);
      tmem_ld32(base + BN, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) iacc[j] += __uint_as_float(v[j]);
    };

    for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
      fetch((q + RAW - 1) & (RAW - 1));
      asm volatile("cp.async.wait_group %0;" ::"n"(RAW - 1) : "memory");
      const uint32_t s = q & (STAGES - 1);
      if (q >= STAGES) mbar_wait(&bars[s], ((q >> L::LOG_STAGES) + 1) & 1u);
      const uint32_t slot = q & (RAW - 1);
      // ---- convert this thread's own bytes
      const float4 a01 = *reinterpret_cast<const float4 *>(smem + L::RAWA_OFF +
                                                            slot * L::RAWA_SLOT + tid * 16);
      const float4 a23 = *reinterpret_cast<const float4 *>(
          smem + L::RAWA_OFF + slot * L::RAWA_SLOT + V2_THREADS * 16 + tid * 16);
      const float4 bb = *reinterpret_cast<const float4 *>(smem + L::RAWB_OFF +
                                                           slot * L::RAWB_SLOT + tid * 16);
      {
        uint32_t hr0, lr0, hi0, li0, hr1, lr1, hi1, li1;
        split_fast(bb.x, hr0, lr0);
        split_fast(bb.y, hi0, li0);
        split_fast(bb.z, hr1, lr1);
        split_fast(bb.w, hi1, li1);
        uint8_t *stage = smem + s * L::STAGE;
        uint8_t *ph = stage, *pl = stage + L::B_PLANE;
        *reinterpret_cast<uint2 *>(ph + 0 * L::B_BLOCK + boff) =
            make_uint2(hi0 ^ 0x80000000u, hi1 ^ 0x80000000u);
        *reinterpret_cast<uint2 *>(ph + 1 * L::B_BLOCK + boff) = make_uint2(hr0, hr1);
        *reinterpret_cast<uint2 *>(ph + 2 * L::B_BLOCK + boff) = make_uint2(hi0, hi1);
        *reinterpret_cast<uint2 *>(pl + 0 * L::B_BLOCK + boff) =
            make_uint2(li0 ^ 0x80000000u, li1 ^ 0x80000000u);
        *reinterpret_cast<uint2 *>(pl + 1 * L::B_BLOCK + boff) = make_uint2(lr0, lr1);
        *reinterpret_cast<uint2 *>(pl + 2 * L::B_BLOCK + boff) = make_uint2(li0, li1);
      }
      {
        uint32_t rh[4], rl[4], ih[4], il[4];
        split_fast(a01.x, rh[0], rl[0]);
        split_fast(a01.y, ih[0], il[0]);
        split_fast(a01.z, rh[1], rl[1]);
        split_fast(a01.w, ih[1], il[1]);
        split_fast(a23.x, rh[2], rl[2]);
        split_fast(a23.y, ih[2], il[2]);
        split_fast(a23.z, rh[3], rl[3]);
        split_fast(a23.w, ih[3], il[3]);
        const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * 32 + 4 * half);
        tmem_st4(acol + 0, rh[0], rh[1], rh[2], rh[3]);
        tmem_st4(acol + 8, rl[0], rl[1], rl[2], rl[3]);
        tmem_st4(acol + 16, ih[0], ih[1], ih[2], ih[3]);
        tmem_st4(acol + 24, il[0], il[1], il[2], il[3]);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
      const uint32_t pos = kb & (CK - 1);
      const uint32_t chunk = kb >> L::LOG_CK;
      if (tid == 0) {
        tc_fence_after();
        const uint32_t d = tmem + (chunk & 1u) * (uint32_t)L::P_COLS;
        uint8_t *stage = smem + s * L::STAGE;
        const uint32_t bhi = smem_u32(stage), blo = smem_u32(stage + L::B_PLANE);
        const uint64_t b1h = smem_desc(bhi + L::B_BLOCK), b1l = smem_desc(blo + L::B_BLOCK);
        const uint64_t b2h = smem_desc(bhi), b2l = smem_desc(blo);
        const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * 32u;
        const uint32_t acc0 = pos > 0 ? 1u : 0u;
        mma_ts(d, a + 0, b1h, IDESC, acc0);
        mma_ts(d, a + 0, b1l, IDESC, 1u);
        mma_ts(d, a + 8, b1h, IDESC, 1u);
        mma_ts(d, a + 16, b2h, IDESC, 1u);
        mma_ts(d, a + 16, b2l, IDESC, 1u);
        mma_ts(d, a + 24, b2h, IDESC, 1u);
        mma_commit(&bars[s]);
        if (pos == CK - 1 || kb == nk - 1) mma_commit(&pbar[chunk & 1u]);
      }
      if (pos == 0 && kb > 0) promote((int)((chunk - 1) & 1u));
    }
    if (nk > 0) promote((int)(((nk - 1) >> L::LOG_CK) & 1u));

    const int64_t row = m0 + row_l;
    if (row < g.M) {
      const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
      const bool use_beta = (br != 0.f || bi != 0.f);
      const int64_t c0 = n0 + 32 * half;
      float2 *crow = C + row * g.ldc + c0;
      const int64_t ncols = min((int64_t)32, g.N - c0);
      if (!use_beta && ncols == 32 && ar == 1.f && ai == 0.f && (((uintptr_t)crow) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          *reinterpret_cast<float4 *>(crow + j) =
              make_float4(racc[j], iacc[j], racc[j + 1], iacc[j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < ncols) {
            float2 o = make_float2(ar * racc[j] - ai * iacc[j], ar * iacc[j] + ai * racc[j]);
            if (use_beta) {
              const float2 c = crow[j];
              o.x += br * c.x - bi * c.y;
              o.y += br * c.y + bi * c.x;
            }
            crow[j] = o;
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
}

// warp-specialised twin: 8 converter warps + 1 MMA-issue warp, per-stage
// `full` mbarriers instead of a block barrier per k-block
template <int STAGES, int CK, int RAW, bool SHORTK, int KS>
__global__ void __launch_bounds__(V2_THREADS + 32, 1)
    cgemm_tc3w_kernel(const __grid_constant__ GemmArgs g, int64_t tiles_n, int64_t tiles) {
  using L = LayoutV3<STAGES, CK, RAW>;
  constexpr int BN = L::BN;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);  // [STAGES] stage free
  uint64_t *pbar = bars + STAGES;                                    // [2] chunk done
  uint64_t *full = pbar + 2;                                         // [STAGES] stage converted
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(full + STAGES);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3, half = warp >> 2;
  const int row_l = lg * 32 + lane;              // A row / TMEM lane of this thread
  // B mapping: two threads share one 16-byte core-matrix row segment, so a
  // 16-lane phase writes 8 rows x 16 B = 128 contiguous bytes (no conflicts)
  const int b_kp = tid & 1;                      // which k pair inside a 4-k chunk
  const int b_n = (tid >> 1) & (BN - 1);         // B column (row of B')
  const int b_chunk = tid >> 7;                  // k 0-3 or 4-7
  const int b_k = b_chunk * 4 + b_kp * 2;        // first of the thread's two k

  if (tid == 0) {
    for (int i = 0; i < STAGES + 2; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < STAGES / KS; ++i) mbar_init(&full[i], V2_THREADS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const bool gat = g.a_roff != nullptr;
  int32_t *s_coff = reinterpret_cast<int32_t *>(smem + L::COFF_OFF);
  if (gat)
    for (int i = tid; i < (int)g.K; i += blockDim.x) s_coff[i] = g.a_coff[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
  constexpr uint32_t IDESC = idesc_tf32(BM, L::NP);
  // A slot = two 16-byte lanes per thread, each lane contiguous across threads,
  // so the 128-bit accesses of a quarter warp hit 8 distinct bank groups
  const uint32_t rawa0 = smem_u32(smem + L::RAWA_OFF) + (uint32_t)tid * 16;
  const uint32_t rawb0 = smem_u32(smem + L::RAWB_OFF) + (uint32_t)tid * 16;
  const uint32_t boff = core_off(b_n, b_chunk) + (uint32_t)(b_kp * 8);

  const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
  const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
  float2 *Cb = reinterpret_cast<float2 *>(g.C);
  const uint32_t nk = (uint32_t)((g.K + KB - 1) / KB);
  const bool k_tail = (g.K % KB) != 0;
  const int64_t total_work = tiles * g.batch;
  const bool a_vec = (g.opA == QF_OP_N) && (g.lda % 2 == 0) && (g.sA % 2 == 0);
  const bool b_vec = (g.opB == QF_OP_T) && (g.ldb % 2 == 0) && (g.sB % 2 == 0);
  const int64_t a_kstride = (g.opA == QF_OP_N) ? 1 : g.lda;   // elements between consecutive k
  const int64_t b_kstride = (g.opB == QF_OP_N) ? g.ldb : 1;

  // A fetch modes.  The converter thread of TMEM lane r needs row r's k
  // values, but one-row-per-lane global loads touch 32 sectors per warp
  // instruction; instead each warp fetches its own 32 rows x 4 k with lanes
  // spread along k (whole 32-byte sectors per row) and the rows land in the
  // owning lanes' raw slots -- the hand-off stays inside the warp.
  //   1: gathered  -- lane (r4 = lane/4, kq = lane%4): rows 8i + r4, k kq (8 B)
  //   2: row-major -- lane (r2 = lane/2, kp = lane%2): rows 16i + r2, k 2kp..2kp+1 (16 B)
  //   0: column-major (lane = row is already coalesced) or odd lda
  const int a_mode = gat ? 1 : (a_vec ? 2 : 0);
  const uint32_t rawa_m =
      smem_u32(smem + L::RAWA_OFF) +
      (a_mode == 1 ? (uint32_t)(((lane & 3) >> 1) * V2_THREADS * 16 + (warp * 32 + (lane >> 2)) * 16 +
                                (lane & 1) * 8)
                   : (uint32_t)((lane & 1) * V2_THREADS * 16 + (warp * 32 + (lane >> 1)) * 16));

  // ---- fetch cursor: incremental source pointers, set up once per tile
  int64_t f_work = blockIdx.x;
  uint32_t f_kb = 0;
  const float2 *fa = Ab, *fb = Bb;
  bool fa_ok = false, fb_ok = false;
  uint32_t amask = 0, amask_next = 0;       // valid rows of this / the next tile
  int32_t ro[4] = {0, 0, 0, 0}, ro_next[4] = {0, 0, 0, 0};
  // gathered row offsets are loaded one tile ahead so the load latency hides
  // behind a whole tile of k-blocks
  auto load_ro = [&](int64_t work, int32_t (&dst)[4], uint32_t &mask) {
    mask = 0;
    if (work >= total_work) return;
    const int64_t tile = work % tiles;
    const int64_t r0 = (tile / tiles_n) * BM + lg * 32 + (lane >> 2);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = r0 + 8 * i < g.M;
      dst[i] = ok ? __ldg(g.a_roff + r0 + 8 * i) : 0;
      mask |= ok ? (1u << i) : 0u;
    }
  };
  if (SHORTK && a_mode == 1) load_ro(f_work, ro_next, amask_next);
  auto fetch_setup = [&]() {
    if (f_work >= total_work) return;
    const int64_t bidx = f_work / tiles;
    const int64_t tile = f_work - bidx * tiles;
    const int64_t mt0 = (tile / tiles_n) * BM;
    const int64_t am = mt0 + row_l;
    const int64_t bn = (tile % tiles_n) * BN + b_n;
    fa_ok = am < g.M;
    fb_ok = bn < g.N;
    const float2 *A = Ab + a_batch_off(g, bidx);
    const float2 *B = Bb + b_batch_off(g, bidx);
    if (a_mode == 1) {
      fa = A;
      if constexpr (SHORTK) {  // short tiles: hide the table load behind the current tile
#pragma unroll
        for (int i = 0; i < 4; ++i) ro[i] = ro_next[i];
        amask = amask_next;
        load_ro(f_work + gridDim.x, ro_next, amask_next);
      } else {
        load_ro(f_work, ro, amask);
      }
    } else if (a_mode == 2) {
      const int64_t r0 = mt0 + lg * 32 + (lane >> 1);
      amask = (r0 < g.M ? 1u : 0u) | (r0 + 16 < g.M ? 2u : 0u);
      fa = A + r0 * g.lda + 4 * half + 2 * (lane & 1);  // row r0 + 16 is fa + 16 lda
    } else {
      fa = (g.opA == QF_OP_N) ? A + am * g.lda + 4 * half : A + (int64_t)(4 * half) * g.lda + am;
      if (!fa_ok) fa = Ab;
    }
    fb = (g.opB == QF_OP_N) ? B + (int64_t)b_k * g.ldb + bn : B + bn * g.ldb + b_k;
    if (!fb_ok) fb = Bb;
  };
  auto fetch = [&](uint32_t slot) {
    if (f_work < total_work) {
      const uint32_t da = rawa0 + slot * L::RAWA_SLOT, db = rawb0 + slot * L::RAWB_SLOT;
      const uint32_t dm = rawa_m + slot * L::RAWA_SLOT;
      if (a_mode == 1) {  // row offsets in registers + per-k offset from the staged table
        const int64_t kk = (int64_t)f_kb * KB + 4 * half + (lane & 3);
        const bool kok = kk < g.K;
        const int32_t c = kok ? s_coff[kk] : 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool ok = kok && ((amask >> i) & 1u);
          cp_async8(dm + i * 128, ok ? fa + ro[i] + c : Ab, ok);
        }
      }
      if (!(k_tail && f_kb == nk - 1)) {
        if (a_mode == 1) {
        } else if (a_mode == 2) {
          cp_async16(dm, (amask & 1u) ? fa : Ab, amask & 1u);
          cp_async16(dm + 256, (amask & 2u) ? fa + 16 * g.lda : Ab, (amask >> 1) & 1u);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            cp_async8(da + (k >> 1) * V2_THREADS * 16 + (k & 1) * 8, fa + k * a_kstride, fa_ok);
        }
        if (b_vec) {
          cp_async16(db, fb, fb_ok);
        } else {
          cp_async8(db, fb, fb_ok);
          cp_async8(db + 8, fb + b_kstride, fb_ok);
        }
      } else {  // ragged last k-block: per-element predicates
        const int64_t k0 = (int64_t)f_kb * KB;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (a_mode != 0) break;
          const bool ok = fa_ok && k0 + 4 * half + k < g.K;
          cp_async8(da + (k >> 1) * V2_THREADS * 16 + (k & 1) * 8, ok ? fa + k * a_kstride : Ab, ok);
        }
        if (a_mode == 2) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = e >> 1, j = e & 1;
            const bool ok = ((amask >> i) & 1u) && k0 + 4 * half + 2 * (lane & 1) + j < g.K;
            cp_async8(dm + i * 256 + j * 8, ok ? fa + i * 16 * g.lda + j : Ab, ok);
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = fb_ok && k0 + b_k + e < g.K;
          cp_async8(db + 8 * e, ok ? fb + e * b_kstride : Bb, ok);
        }
      }
      if (a_mode == 2) {
        fa += KB;
      } else if (a_mode == 0 && fa_ok) {
        fa += KB * a_kstride;
      }
      if (fb_ok) fb += KB * b_kstride;
      if (++f_kb == nk) {
        f_kb = 0;
        f_work += gridDim.x;
        fetch_setup();
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // uniform group count
  };

  if (warp == V2_THREADS / 32) {
    // ===== MMA issuer: the whole warp walks the k-block sequence (operands stay
    // warp-uniform, i.e. in uniform registers); one elected lane issues
    {
      uint32_t qm = 0, tcount = 0, gq = 0;
      constexpr uint32_t NG = STAGES / KS;     // converted groups in flight
      for (int64_t work = blockIdx.x; work < total_work; work += gridDim.x, ++tcount) {
        for (uint32_t kb = 0; kb < nk; ++kb, ++qm) {
          const uint32_t s = qm & (STAGES - 1);
          if (kb % KS == 0) {  // one handoff per group of KS k-blocks (aligned to tiles)
            mbar_wait(&full[gq % NG], (gq / NG) & 1u);
            tc_fence_after();
            ++gq;
          }
          // SHORTK: one accumulation per tile, buffers alternate per tile;
          // otherwise chunks of CK k-blocks alternate (promotion)
          const uint32_t pos = SHORTK ? kb : (kb & (CK - 1));
          const uint32_t chunk = SHORTK ? tcount : (kb >> L::LOG_CK);
          const uint32_t d = tmem + (chunk & 1u) * (uint32_t)L::P_COLS;
          uint8_t *stage = smem + s * L::STAGE;
          const uint32_t bhi = smem_u32(stage), blo = smem_u32(stage + L::B_PLANE);
          const uint64_t b1h = smem_desc(bhi + L::B_BLOCK), b1l = smem_desc(blo + L::B_BLOCK);
          const uint64_t b2h = smem_desc(bhi), b2l = smem_desc(blo);
          const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * 32u;
          const uint32_t acc0 = pos > 0 ? 1u : 0u;
          if (elect_one()) {
            mma_ts(d, a + 0, b1h, IDESC, acc0);
            mma_ts(d, a + 0, b1l, IDESC, 1u);
            mma_ts(d, a + 8, b1h, IDESC, 1u);
            mma_ts(d, a + 16, b2h, IDESC, 1u);
            mma_ts(d, a + 16, b2l, IDESC, 1u);
            mma_ts(d, a + 24, b2h, IDESC, 1u);
            mma_commit(&bars[s]);
            if (SHORTK ? kb == nk - 1 : (pos == CK - 1 || kb == nk - 1))
              mma_commit(&pbar[chunk & 1u]);
          }
          __syncwarp();
        }
      }
    }
    __syncwarp();
  } else {
  uint32_t q = 0;            // k-blocks consumed by this CTA (drives every ring)
  uint32_t gc = 0;           // groups handed to the MMA warp
  uint32_t pwaits[2] = {0, 0};
  fetch_setup();
  for (int i = 0; i < RAW - 1; ++i) fetch((uint32_t)i);
  // SHORTK: the accumulators of tile t stay in TMEM buffer (t & 1); tile t's
  // epilogue runs after tile t+1's first k-block is converted, so the tensor
  // pipe never drains at a tile boundary and no accumulator lives in registers
  bool have_prev = false;
  int prev_pb = 0;
  int64_t prev_m0 = 0, prev_n0 = 0;
  float2 *prev_C = nullptr;
  uint32_t tcount = 0;
  auto tmem_epilogue = [&](int pb, int64_t em0, int64_t en0, float2 *eC) {
    mbar_wait(&pbar[pb], pwaits[pb] & 1u);
    ++pwaits[pb];
    tc_fence_after();
    uint32_t vr[32], vi[32];
    const uint32_t base = tmem + lane_base + (uint32_t)(pb * L::P_COLS + 32 * half);
    tmem_ld32(base, vr);
    tmem_ld32(base + BN, vi);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int64_t row = em0 + row_l;
    if (row < g.M) {
      const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
      const bool use_beta = (br != 0.f || bi != 0.f);
      const int64_t c0 = en0 + 32 * half;
      float2 *crow = eC + row * g.ldc + c0;
      const int64_t ncols = min((int64_t)32, g.N - c0);
      if (!use_beta && ncols == 32 && ar == 1.f && ai == 0.f && (((uintptr_t)crow) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          *reinterpret_cast<float4 *>(crow + j) =
              make_float4(__uint_as_float(vr[j]), __uint_as_float(vi[j]),
                          __uint_as_float(vr[j + 1]), __uint_as_float(vi[j + 1]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < ncols) {
            const float x = __uint_as_float(vr[j]), y = __uint_as_float(vi[j]);
            float2 o = make_float2(ar * x - ai * y, ar * y + ai * x);
            if (use_beta) {
              const float2 c = crow[j];
              o.x += br * c.x - bi * c.y;
              o.y += br * c.y + bi * c.x;
            }
            crow[j] = o;
          }
        }
      }
    }
    tc_fence_before();
  };

  for (int64_t work = blockIdx.x; work < total_work; work += gridDim.x) {
    const int64_t bidx = work / tiles;
    const int64_t tile = work - bidx * tiles;
    const int64_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    float2 *C = Cb + bidx * g.sC;
    float racc[32], iacc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) racc[j] = iacc[j] = 0.f;

    auto promote = [&](int pb) {
      mbar_wait(&pbar[pb], pwaits[pb] & 1u);
      ++pwaits[pb];
      tc_fence_after();
      uint32_t v[32];
      const uint32_t base = tmem + lane_base + (uint32_t)(pb * L::P_COLS + 32 * half);
      tmem_ld32(base, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) racc[j] += __uint_as_float(v[j]);
      tmem_ld32(base + BN, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) iacc[j] += __uint_as_float(v[j]);
    };

    for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
      fetch((q + RAW - 1) & (RAW - 1));
      asm volatile("cp.async.wait_group %0;" ::"n"(RAW - 1) : "memory");
      if (a_mode != 0) __syncwarp();  // raw A rows were fetched by other lanes of this warp
      const uint32_t s = q & (STAGES - 1);
      if (q >= STAGES) mbar_wait(&bars[s], ((q >> L::LOG_STAGES) + 1) & 1u);
      const uint32_t slot = q & (RAW - 1);
      // ---- convert this thread's own bytes
      const float4 a01 = *reinterpret_cast<const float4 *>(smem + L::RAWA_OFF +
                                                            slot * L::RAWA_SLOT + tid * 16);
      const float4 a23 = *reinterpret_cast<const float4 *>(
          smem + L::RAWA_OFF + slot * L::RAWA_SLOT + V2_THREADS * 16 + tid * 16);
      const float4 bb = *reinterpret_cast<const float4 *>(smem + L::RAWB_OFF +
                                                           slot * L::RAWB_SLOT + tid * 16);
      {
        uint32_t hr0, lr0, hi0, li0, hr1, lr1, hi1, li1;
        split_fast(bb.x, hr0, lr0);
        split_fast(bb.y, hi0, li0);
        split_fast(bb.z, hr1, lr1);
        split_fast(bb.w, hi1, li1);
        uint8_t *stage = smem + s * L::STAGE;
        uint8_t *ph = stage, *pl = stage + L::B_PLANE;
        *reinterpret_cast<uint2 *>(ph + 0 * L::B_BLOCK + boff) =
            make_uint2(hi0 ^ 0x80000000u, hi1 ^ 0x80000000u);
        *reinterpret_cast<uint2 *>(ph + 1 * L::B_BLOCK + boff) = make_uint2(hr0, hr1);
        *reinterpret_cast<uint2 *>(ph + 2 * L::B_BLOCK + boff) = make_uint2(hi0, hi1);
        *reinterpret_cast<uint2 *>(pl + 0 * L::B_BLOCK + boff) =
            make_uint2(li0 ^ 0x80000000u, li1 ^ 0x80000000u);
        *reinterpret_cast<uint2 *>(pl + 1 * L::B_BLOCK + boff) = make_uint2(lr0, lr1);
        *reinterpret_cast<uint2 *>(pl + 2 * L::B_BLOCK + boff) = make_uint2(li0, li1);
      }
      {
        uint32_t rh[4], rl[4], ih[4], il[4];
        split_fast(a01.x, rh[0], rl[0]);
        split_fast(a01.y, ih[0], il[0]);
        split_fast(a01.z, rh[1], rl[1]);
        split_fast(a01.w, ih[1], il[1]);
        split_fast(a23.x, rh[2], rl[2]);
        split_fast(a23.y, ih[2], il[2]);
        split_fast(a23.z, rh[3], rl[3]);
        split_fast(a23.w, ih[3], il[3]);
        const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * 32 + 4 * half);
        tmem_st4(acol + 0, rh[0], rh[1], rh[2], rh[3]);
        tmem_st4(acol + 8, rl[0], rl[1], rl[2], rl[3]);
        tmem_st4(acol + 16, ih[0], ih[1], ih[2], ih[3]);
        tmem_st4(acol + 24, il[0], il[1], il[2], il[3]);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (kb % KS == KS - 1 || kb == nk - 1) {  // group (or tile) converted
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                           smem_u32(&full[gc % (STAGES / KS)]))
                       : "memory");
        ++gc;
      }
      const uint32_t pos = kb & (CK - 1);
      const uint32_t chunk = kb >> L::LOG_CK;
      if constexpr (SHORTK) {
        if (kb == 0 && have_prev) {
          tmem_epilogue(prev_pb, prev_m0, prev_n0, prev_C);
          have_prev = false;
        }
      } else {
        if (pos == 0 && kb > 0) promote((int)((chunk - 1) & 1u));
      }
    }
    if constexpr (SHORTK) {
      have_prev = nk > 0;
      prev_pb = (int)(tcount & 1u);
      prev_m0 = m0;
      prev_n0 = n0;
      prev_C = C;
      ++tcount;
      continue;
    }
    if (nk > 0) promote((int)(((nk - 1) >> L::LOG_CK) & 1u));

    const int64_t row = m0 + row_l;
    if (row < g.M) {
      const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
      const bool use_beta = (br != 0.f || bi != 0.f);
      const int64_t c0 = n0 + 32 * half;
      float2 *crow = C + row * g.ldc + c0;
      const int64_t ncols = min((int64_t)32, g.N - c0);
      if (!use_beta && ncols == 32 && ar == 1.f && ai == 0.f && (((uintptr_t)crow) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          *reinterpret_cast<float4 *>(crow + j) =
              make_float4(racc[j], iacc[j], racc[j + 1], iacc[j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < ncols) {
            float2 o = make_float2(ar * racc[j] - ai * iacc[j], ar * iacc[j] + ai * racc[j]);
            if (use_beta) {
              const float2 c = crow[j];
              o.x += br * c.x - bi * c.y;
              o.y += br * c.y + bi * c.x;
            }
            crow[j] = o;
          }
        }
      }
    }
  }
  if constexpr (SHORTK) {
    if (have_prev) tmem_epilogue(prev_pb, prev_m0, prev_n0, prev_C);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  }  // converter warps
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
}

template <int STAGES, int CK, int RAW, bool SHORTK, int KS = 1>
int launch_ws(const GemmArgs &g, cudaStream_t s) {
  using L = LayoutV3<STAGES, CK, RAW>;
  auto kern = cgemm_tc3w_kernel<STAGES, CK, RAW, SHORTK, KS>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3w: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  const int64_t tiles_n = (g.N + L::BN - 1) / L::BN, tiles_m = (g.M + BM - 1) / BM;
  const int64_t tiles = tiles_n * tiles_m;
  const int64_t grid = std::min<int64_t>(tiles * g.batch, (int64_t)sm_count());
  kern<<<(unsigned)grid, V2_THREADS + 32, L::SMEM, s>>>(g, tiles_n, tiles);
  return check_launch("cgemm_tc3w");
}

// ---------------------------------------------------------------------------
// Short-K twin of tc3w (K <= 256: one TMEM accumulation per tile, no
// promotion).  Differences that matter for the batched small-tile GEMMs of
// the amplitude batch (e.g. 1024 x (4096 x 64 x 64)):
//   * each CTA walks a contiguous run of tiles, M tile fastest, so
//     consecutive tiles share one B panel; when the k-block count divides
//     the stage ring, stage s holds the same B k-block for every tile of the
//     run and the B' planes are fetched and split once per run -- a tile
//     then only streams A (fetch + split + tcgen05.st);
//   * tile t's epilogue runs after tile t+1's LAST k-block is converted, so
//     the converters can run a whole tile ahead of the tensor pipe, and it
//     goes through a per-warp staging tile so every store instruction
//     writes whole row segments;
//   * NW converter warps (8 or 16): NW/4 warps share each 32-lane TMEM
//     quadrant and split the k-block's 8 k (and the epilogue's 64 columns)
//     between them -- 16 warps hide twice the latency of 8;
//   * 32-bit tile arithmetic, gathered row offsets prefetched a tile ahead.

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

// shared memory of the short-K kernel: B' stages, raw A/B rings, a per-warp
// epilogue staging tile (32 rows x CPW complex, rows padded by 16 B so both
// the row-per-lane writes and the row-contiguous reads are conflict-free)
template <int STAGES, int RAW, int NW, int NE, int BN_ = V2_BN, int CK_ = 0, int NPW_ = 0,
          bool TMA_ = false>
struct LayoutK {
  static_assert(NPW_ == 0 || (NPW_ == (TMA_ ? 1 : 4) && NE == 4 && (BN_ == 64 || (TMA_ && BN_ == 32))),
                "producer warps (4 cp.async or 1 TMA) need epilogue/promotion warps and 64-column "
                "tiles (32 with TMA)");

  static constexpr int NPW = NPW_;                   // producer (fetch) warps
  static constexpr int RPITCH = 80;                  // producer mode: raw row = 8 complex + 16 B
  static_assert((STAGES & (STAGES - 1)) == 0 && (RAW & (RAW - 1)) == 0, "rings must be powers of two");
  static_assert(NW == 8 || NW == 16, "8 or 16 converter warps");
  static_assert((CK_ == 0 && (NE == 0 || NE == 4)) || (CK_ > 0 && NE == 4 && BN_ == 64),
                "short K: epilogue on the converters or 4 epilogue warps; long K: 4 promotion warps");
  static_assert((CK_ & (CK_ - 1)) == 0, "promotion chunk must be a power of two");
  static_assert(BN_ == 64 || (NE >= 4 && (BN_ == 8 || BN_ == 16 || BN_ == 32)),
                "narrow N tiles need the epilogue warps");
  static constexpr int NT = NW * 32;                 // converter threads
  static constexpr int NWG = NW / 4;                 // warps per TMEM lane quadrant
  static constexpr int KPW = KB / NWG;               // k of a k-block per warp
  static constexpr int BN = BN_;                     // complex output columns per tile
  static constexpr int CPW = BN / NWG;               // epilogue columns per warp
  static constexpr int NP = 2 * BN;
  static constexpr int B_BLOCK = BN * 32;
  static constexpr int B_PLANE = 3 * B_BLOCK;
  static constexpr int STAGE = 2 * B_PLANE;
  // TMA: dense boxes (A: 128 rows x 64 B, 64-byte swizzle, or 8 k x 1 KB; B: 64 n x
  // 64 B swizzled or 8 k x 512 B), 1 KB aligned
  static constexpr int RAWA_SLOT = TMA_ ? BM * 64 : NPW_ ? BM * RPITCH : NT * KPW * 8;
  static constexpr int RAWB_SLOT = TMA_ ? BN * 64 : NPW_ ? BN * RPITCH : BN * KB * 8;
  static constexpr int RAWA_OFF = STAGES * STAGE;
  static constexpr int RAWB_OFF = RAWA_OFF + RAW * RAWA_SLOT;
  static constexpr int EPI_CH = NE ? (BN < 16 ? BN : 16) : CPW;  // columns per staging pass
  static constexpr int EPI_PITCH = EPI_CH * 8 + 16;
  static constexpr int EPI_OFF = RAWB_OFF + RAW * RAWB_SLOT;
  static constexpr int BAR_OFF = EPI_OFF + (NE ? NE : NW) * 32 * EPI_PITCH;
  static constexpr int COFF_OFF = BAR_OFF + 1024;
  static constexpr int COFF_MAX = CK_ ? 4096 : 256;  // gathered-A k offsets
  static constexpr int SMEM = COFF_OFF + 4 * COFF_MAX;
  static constexpr int P_COLS = NP;
  static constexpr int MASTER_COL = 2 * P_COLS;              // long K: fp32 master accumulator
  static constexpr int A_COL0 = (CK_ ? 3 : 2) * P_COLS;
  static constexpr int TMEM_COLS = 512;
  static_assert(A_COL0 + STAGES * 32 <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

template <int STAGES, int RAW, int NW, int NE, int BN_, int CK_, int NPW, bool TMA>
__global__ void __launch_bounds__((NW + NE + NPW) * 32 + 32, 1)
    cgemm_tc3k_kernel(const __grid_constant__ GemmArgs g, uint32_t tiles_m, uint32_t tiles_n,
                      uint32_t total, uint32_t chunk, const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB) {
  using L = LayoutK<STAGES, RAW, NW, NE, BN_, CK_, NPW, TMA>;
  // NPW > 0: 4 producer warps own the global fetch (cp.async into padded raw
  // rows, completion signalled on per-slot mbarriers); the converter warps
  // only read, split and store into TMEM / the B' planes.
  // CK_ > 0: long-K mode.  Every CK_ k-blocks the tensor pipe's partial sum
  // (double-buffered in TMEM) is added by 4 promotion warps into an fp32
  // master accumulator that also lives in TMEM (CUDA-core adds: round to
  // nearest, flat error in K), so the converter warps never stall on
  // promotion; tiles are strided over the grid (neighbouring CTAs share A
  // rows / B panels in L2).
  constexpr bool PROMO = CK_ > 0;
  constexpr int BN = L::BN, NT = L::NT, KPW = L::KPW, CPW = L::CPW;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);  // [STAGES] stage free
  uint64_t *pbar = bars + STAGES;                                    // [2] tile accumulated
  uint64_t *full = pbar + 2;                                         // [STAGES] stage converted
  uint64_t *accfree = full + STAGES;                                 // [2] accumulator drained
  uint64_t *rawfull = accfree + 2;                                   // [RAW] producer fill landed
  uint64_t *rawfree = rawfull + RAW;                                 // [RAW] converters read it
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rawfree + RAW);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3, wg = warp >> 2;
  const int row_l = lg * 32 + lane;

  if (tid == 0) {
    for (int i = 0; i < STAGES + 2; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], NW);
    for (int i = 0; i < 2; ++i) mbar_init(&accfree[i], NE ? NE : 1);
    for (int i = 0; i < RAW; ++i) {
      mbar_init(&rawfull[i], (NPW && !TMA) ? NPW * 32 : 1);
      mbar_init(&rawfree[i], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const bool gat = g.a_roff != nullptr;
  int32_t *s_coff = reinterpret_cast<int32_t *>(smem + L::COFF_OFF);
  if (gat)
    for (int i = tid; i < (int)g.K; i += blockDim.x) s_coff[i] = g.a_coff[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
  constexpr uint32_t IDESC = idesc_tf32(BM, L::NP);

  const uint32_t w0 = PROMO ? blockIdx.x : blockIdx.x * chunk;
  const uint32_t w1 = PROMO ? total : min(total, w0 + chunk);
  const uint32_t wstep = PROMO ? gridDim.x : 1u;
  const uint32_t K = (uint32_t)g.K;
  const uint32_t nk = (K + KB - 1) / KB;
  // B of a tile sits in the stages iff the tile rd earlier in this run had
  // the same (batch, N tile) key, i.e. >= rd tiles of the key precede it here
  const uint32_t rd = (!PROMO && STAGES % nk == 0) ? STAGES / nk : 0u;

  // tile cursors advance incrementally (M tile fastest, then N tile, batch);
  // `run` = tiles of the current (batch, N tile) key before this one here
  struct Cur {
    uint32_t w, mt, nt, bidx, run;
  };
  auto cur_init = [&](Cur &c, uint32_t w) {
    c.w = w;
    if constexpr (PROMO) {
      // strided long-K tiles in groups of GM M tiles: the ~148 tiles in
      // flight cover a GM x (148/GM) block, so A and B panels are each
      // reused ~GM times out of L2 instead of re-streamed from HBM
      constexpr uint32_t GM = 16;
      const uint32_t tiles = tiles_m * tiles_n;
      c.bidx = w / tiles;
      const uint32_t t = w - c.bidx * tiles;
      const uint32_t group = t / (GM * tiles_n), first_m = group * GM;
      const uint32_t gsize = min(tiles_m - first_m, GM);
      const uint32_t r = t - group * GM * tiles_n;
      c.mt = first_m + r % gsize;
      c.nt = r / gsize;
      c.run = 0;
      return;
    }
    const uint32_t key = w / tiles_m;
    c.mt = w - key * tiles_m;
    c.bidx = key / tiles_n;
    c.nt = key - c.bidx * tiles_n;
    c.run = 0;
  };
  auto cur_next = [&](Cur &c) {
    if constexpr (PROMO) {
      cur_init(c, c.w + wstep);
      return;
    }
    ++c.w;
    ++c.run;
    if (++c.mt == tiles_m) {
      c.mt = 0;
      c.run = 0;
      if (++c.nt == tiles_n) {
        c.nt = 0;
        ++c.bidx;
      }
    }
  };


  if (warp == NW + NE + NPW) {
    // ===== MMA issuer (whole warp walks the sequence, one elected lane issues)
    uint32_t q = 0, t = 0, chunkc = 0;
    for (uint32_t w = w0; w < w1; w += wstep, ++t) {
      for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
        const uint32_t s = q & (STAGES - 1);
        mbar_wait(&full[s], (q / STAGES) & 1u);
        tc_fence_after();
        uint32_t pbuf = t & 1u;
        uint32_t pos = kb;
        if constexpr (PROMO) {
          pos = kb & (CK_ - 1);
          pbuf = chunkc & 1u;
          if (pos == 0 && chunkc >= 2) {  // promotion warps drained this partial
            mbar_wait(&accfree[pbuf], ((chunkc >> 1) + 1) & 1u);
            tc_fence_after();
          }
        }
        const uint32_t d = tmem + pbuf * (uint32_t)L::P_COLS;
        uint8_t *stage = smem + s * L::STAGE;
        const uint32_t bhi = smem_u32(stage), blo = smem_u32(stage + L::B_PLANE);
        const uint64_t b1h = smem_desc(bhi + L::B_BLOCK), b1l = smem_desc(blo + L::B_BLOCK);
        const uint64_t b2h = smem_desc(bhi), b2l = smem_desc(blo);
        const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * 32u;
        const uint32_t acc0 = pos > 0 ? 1u : 0u;
        const bool chunk_end = PROMO ? (pos == CK_ - 1 || kb == nk - 1) : (kb == nk - 1);
        if (!PROMO && NE > 0 && kb == 0 && t >= 2) {  // epilogue warps drained this buffer (tile t-2)
          mbar_wait(&accfree[t & 1u], ((t >> 1) + 1) & 1u);
          tc_fence_after();
        }
        if (elect_one()) {
          mma_ts(d, a + 0, b1h, IDESC, acc0);
          mma_ts(d, a + 0, b1l, IDESC, 1u);
          mma_ts(d, a + 8, b1h, IDESC, 1u);
          mma_ts(d, a + 16, b2h, IDESC, 1u);
          mma_ts(d, a + 16, b2l, IDESC, 1u);
          mma_ts(d, a + 24, b2h, IDESC, 1u);
          mma_commit(&bars[s]);
          if (chunk_end) mma_commit(&pbar[pbuf]);
        }
        if (PROMO && chunk_end) ++chunkc;
        __syncwarp();
      }
    }
  } else if (TMA && warp >= NW + NE) {
    // ===== TMA producer (one elected lane): per k-block one box of A and,
    // unless resident, one box of B into the raw ring; the mbarrier's
    // transaction count completes when both have landed
    if (elect_one()) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      const uint32_t rawa = smem_u32(smem + L::RAWA_OFF), rawb = smem_u32(smem + L::RAWB_OFF);
      Cur pc;
      cur_init(pc, w0);
      uint32_t f = 0;
      for (; pc.w < w1; cur_next(pc)) {
        const bool breuse = rd != 0u && pc.run >= rd;
        const int32_t m0 = (int32_t)(pc.mt * BM), n0 = (int32_t)(pc.nt * BN), b = (int32_t)pc.bidx;
        const int32_t bslice =
            g.b_boff ? (int32_t)(__ldg(g.b_boff + pc.bidx) / (g.K * g.N)) : b;
        const int32_t aslice = g.a_boff ? (int32_t)(__ldg(g.a_boff + pc.bidx) / g.sA) : b;
        // A view: row coordinates of this tile, k-block -> (ki, ko) counters
        int32_t v_ra = 0, v_rb = 0, v_ki = 0, v_ko = 0;
        const int32_t v_kbi = g.v_kin ? (int32_t)(g.v_kin / KB) : 1;
        if (g.v_kin) {
          v_rb = (int32_t)(m0 / (int32_t)g.v_ra);
          v_ra = g.v_ra >= BM ? m0 - v_rb * (int32_t)g.v_ra : 0;
          if (g.v_t) v_ra *= 2;  // float coordinate of the contiguous row run
        }
        for (uint32_t kb = 0; kb < nk; ++kb, ++f) {
          const uint32_t slot = f & (RAW - 1);
          if (f >= RAW) mbar_wait(&rawfree[slot], ((f / RAW) + 1) & 1u);
          const uint32_t bar = smem_u32(&rawfull[slot]);
          const uint32_t bytes = L::RAWA_SLOT + (breuse ? 0u : (uint32_t)L::RAWB_SLOT);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                       : "memory");
          const int32_t k0 = (int32_t)(kb * KB);
          if (g.v_t) {
            // transposed view: {2 ra, rb, ki, ko, b}; the box is [8 k][128 rows]
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(rawa + slot * L::RAWA_SLOT),
                "l"(&tmA), "r"(v_ra), "r"(v_rb), "r"(v_ki * KB), "r"(v_ko), "r"(b), "r"(bar)
                : "memory");
            if (++v_ki == v_kbi) {
              v_ki = 0;
              ++v_ko;
            }
          } else if (g.v_kin) {
            // A view: {2 ki, ra, ko, rb, b}; the box spans 128 rows of (ra, rb)
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(rawa + slot * L::RAWA_SLOT),
                "l"(&tmA), "r"(v_ki * 2 * KB), "r"(v_ra), "r"(v_ko), "r"(v_rb), "r"(aslice), "r"(bar)
                : "memory");
            if (++v_ki == v_kbi) {
              v_ki = 0;
              ++v_ko;
            }
          } else {
            // A: opA N -> coords {2k, m, b}; opA T -> {2m, k, b}
            const int32_t a0 = g.opA == QF_OP_N ? 2 * k0 : 2 * m0, a1 = g.opA == QF_OP_N ? m0 : k0;
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(rawa + slot * L::RAWA_SLOT),
                "l"(&tmA), "r"(a0), "r"(a1), "r"(aslice), "r"(bar)
                : "memory");
          }
          if (!breuse) {
            // B: opB N -> {2n, k, slice}; opB T -> {2k, n, slice}
            const int32_t c0 = g.opB == QF_OP_N ? 2 * n0 : 2 * k0, c1 = g.opB == QF_OP_N ? k0 : n0;
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(rawb + slot * L::RAWB_SLOT),
                "l"(&tmB), "r"(c0), "r"(c1), "r"(bslice), "r"(bar)
                : "memory");
          }
        }
      }
    }
    __syncwarp();
  } else if (!TMA && NPW > 0 && warp >= NW + NE) {
    // ===== producer warps: fetch A (and B unless it is resident) for every
    // k-block into the raw ring, rows padded to 80 B; the layout's
    // contiguous axis is spread across lanes so requests are whole sectors
    const int pt = tid - (NW + NE) * 32;  // 0..127
    const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
    const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
    const bool rows_unit = gat && g.M > 1 && __ldg(g.a_roff + 1) - __ldg(g.a_roff) == 1;
    const bool a_vec = !gat && g.opA == QF_OP_N && g.lda % 2 == 0 && g.sA % 2 == 0;
    const bool b_vec = g.opB == QF_OP_T && g.ldb % 2 == 0 && g.sB % 2 == 0;
    // 0 gathered, lane = row; 1 gathered, lanes along k; 2 column-major, lane = row;
    // 3 row-major, 16-byte k pairs; 4 row-major, lanes along k
    const int pmode = gat ? (rows_unit ? 0 : 1) : (g.opA == QF_OP_T ? 2 : (a_vec ? 3 : 4));
    const uint32_t rawa = smem_u32(smem + L::RAWA_OFF), rawb = smem_u32(smem + L::RAWB_OFF);
    const bool k_tail = (K % KB) != 0;
    Cur pc;
    cur_init(pc, w0);
    uint32_t f = 0;
    for (; pc.w < w1; cur_next(pc)) {
      const bool breuse = rd != 0u && pc.run >= rd;
      const float2 *A = Ab + a_batch_off(g, pc.bidx);
      const float2 *B = Bb + b_batch_off(g, pc.bidx);
      const int64_t m0 = (int64_t)pc.mt * BM, n0 = (int64_t)pc.nt * BN;
      // per-tile row bases
      int32_t ro[8];
      uint32_t rmask = 0;
      if (pmode == 0 || pmode == 2) {
        const int64_t r = m0 + pt;
        rmask = r < g.M ? 1u : 0u;
        ro[0] = pmode == 0 ? __ldg(g.a_roff + min(r, g.M - 1)) : 0;
      } else if (pmode == 1 || pmode == 4) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t r = m0 + (pt >> 3) + 16 * i;
          rmask |= r < g.M ? (1u << i) : 0u;
          ro[i] = pmode == 1 ? __ldg(g.a_roff + min(r, g.M - 1)) : 0;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) rmask |= (m0 + (pt >> 2) + 32 * i < g.M) ? (1u << i) : 0u;
      }
      for (uint32_t kb = 0; kb < nk; ++kb, ++f) {
        const uint32_t slot = f & (RAW - 1);
        if (f >= RAW) mbar_wait(&rawfree[slot], ((f / RAW) + 1) & 1u);
        const uint32_t dA = rawa + slot * L::RAWA_SLOT, dB = rawb + slot * L::RAWB_SLOT;
        const uint32_t k0 = kb * KB;
        const bool tail = k_tail && kb == nk - 1;
        if (pmode == 0) {
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            const bool ok = (rmask & 1u) && (!tail || k0 + k < K);
            cp_async8(dA + pt * L::RPITCH + k * 8, ok ? A + ro[0] + s_coff[k0 + k] : Ab, ok);
          }
        } else if (pmode == 2) {
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            const bool ok = (rmask & 1u) && (!tail || k0 + k < K);
            cp_async8(dA + pt * L::RPITCH + k * 8, ok ? A + (int64_t)(k0 + k) * g.lda + m0 + pt : Ab, ok);
          }
        } else if (pmode == 1 || pmode == 4) {
          const int k = pt & 7;
          const bool kok = !tail || k0 + k < K;
          const int32_t c = pmode == 1 ? s_coff[kok ? k0 + k : 0u] : 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = (pt >> 3) + 16 * i;
            const bool ok = kok && ((rmask >> i) & 1u);
            const float2 *src = pmode == 1 ? A + (ro[i] + c) : A + (m0 + r) * g.lda + k0 + k;
            cp_async8(dA + r * L::RPITCH + k * 8, ok ? src : Ab, ok);
          }
        } else {  // pmode 3: row-major, 16-byte k pairs
          const int kp = pt & 3;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = (pt >> 2) + 32 * i;
            const bool rok = (rmask >> i) & 1u;
            const float2 *src = A + (m0 + r) * g.lda + k0 + 2 * kp;
            if (!tail) {
              cp_async16(dA + r * L::RPITCH + kp * 16, rok ? src : Ab, rok);
            } else {
              const bool ok0 = rok && k0 + 2 * kp < K, ok1 = rok && k0 + 2 * kp + 1 < K;
              cp_async8(dA + r * L::RPITCH + kp * 16, ok0 ? src : Ab, ok0);
              cp_async8(dA + r * L::RPITCH + kp * 16 + 8, ok1 ? src + 1 : Ab, ok1);
            }
          }
        }
        if (!breuse) {
          if (g.opB == QF_OP_N) {  // rows of B are k: lanes along n
            const int n = pt & 63;
            const bool nok = n0 + n < g.N;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t k = (pt >> 6) + 2 * i;
              const bool ok = nok && (!tail || k0 + k < K);
              cp_async8(dB + n * L::RPITCH + k * 8, ok ? B + (int64_t)(k0 + k) * g.ldb + n0 + n : Bb, ok);
            }
          } else if (b_vec && !tail) {  // rows of B are n, k contiguous: 16-byte k pairs
            const int kp = pt & 3;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int n = (pt >> 2) + 32 * i;
              const bool ok = n0 + n < g.N;
              cp_async16(dB + n * L::RPITCH + kp * 16, ok ? B + (n0 + n) * g.ldb + k0 + 2 * kp : Bb, ok);
            }
          } else {
            const int k = pt & 7;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int n = (pt >> 3) + 16 * i;
              const bool ok = n0 + n < g.N && (!tail || k0 + k < K);
              cp_async8(dB + n * L::RPITCH + k * 8, ok ? B + (n0 + n) * g.ldb + k0 + k : Bb, ok);
            }
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         smem_u32(&rawfull[slot]))
                     : "memory");
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (PROMO && warp >= NW) {
    // ===== promotion warps (one per TMEM lane quadrant, 32 rows x 64 columns):
    // master (+)= partial in 16-column pieces, then the tile's epilogue
    float2 *Cb = reinterpret_cast<float2 *>(g.C);
    const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
    const bool use_beta = (br != 0.f || bi != 0.f);
    uint8_t *stg = smem + L::EPI_OFF + (warp - NW) * 32 * L::EPI_PITCH;
    const uint32_t nchunks = (nk + CK_ - 1) / CK_;
    const uint32_t mbase = tmem + lane_base + (uint32_t)L::MASTER_COL;
    uint32_t chunkc = 0;
    Cur ec;
    cur_init(ec, w0);
    for (; ec.w < w1; cur_next(ec)) {
      for (uint32_t c = 0; c < nchunks; ++c, ++chunkc) {
        const uint32_t pbuf = chunkc & 1u;
        mbar_wait(&pbar[pbuf], (chunkc >> 1) & 1u);
        tc_fence_after();
        const uint32_t pbase = tmem + lane_base + pbuf * (uint32_t)L::P_COLS;
#pragma unroll 1
        for (int piece = 0; piece < 2 * BN / 32; ++piece) {  // 32 columns per round trip
          uint32_t pv[32], mv[32];
          tmem_ld32(pbase + piece * 32, pv);
          if (c > 0) tmem_ld32(mbase + piece * 32, mv);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c > 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              pv[j] = __float_as_uint(__uint_as_float(pv[j]) + __uint_as_float(mv[j]));
          }
          tmem_st32(mbase + piece * 32, pv);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accfree[pbuf]))
                       : "memory");
      }
      // ---- epilogue from the master accumulator, 16 columns per pass
      const int64_t m0 = (int64_t)ec.mt * BM + lg * 32;
      float2 *cw = Cb + (int64_t)ec.bidx * g.sC + m0 * g.ldc + (int64_t)ec.nt * BN;
      const int64_t ntile = min((int64_t)BN, g.N - (int64_t)ec.nt * BN);
      const bool vec = g.ldc % 2 == 0 && (((uintptr_t)cw) & 15) == 0;
#pragma unroll 1
      for (int ch = 0; ch < BN / 16; ++ch) {
        uint32_t vr[16], vi[16];
        tmem_ld16(mbase + ch * 16, vr);
        tmem_ld16(mbase + BN + ch * 16, vi);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        stage_store_chunk<16, L::EPI_PITCH>(stg, vr, vi, cw + ch * 16, g.ldc, g.M - m0,
                                            ntile - ch * 16, ar, ai, br, bi, use_beta, vec, lane);
      }
      tc_fence_before();  // master reads done before the next tile's first promotion
    }
  } else if (NE > 0 && warp >= NW) {
    // ===== epilogue warps: drain tile t's accumulators while the converters
    // and the tensor pipe work on tile t+1; columns in passes of 16 through
    // the warp's staging tile so every store writes whole 128-byte segments
    float2 *Cb = reinterpret_cast<float2 *>(g.C);
    const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
    const bool use_beta = (br != 0.f || bi != 0.f);
    uint8_t *stg = smem + L::EPI_OFF + (warp - NW) * 32 * L::EPI_PITCH;
    Cur ec;
    cur_init(ec, w0);
    for (uint32_t t = 0; ec.w < w1; cur_next(ec), ++t) {
      const uint32_t pb = t & 1u;
      mbar_wait(&pbar[pb], (t >> 1) & 1u);
      tc_fence_after();
      const int64_t m0 = (int64_t)ec.mt * BM + lg * 32;
      float2 *cw = Cb + (int64_t)ec.bidx * g.sC + m0 * g.ldc + (int64_t)ec.nt * BN;
      const int64_t ntile = min((int64_t)BN, g.N - (int64_t)ec.nt * BN);
      const bool vec = g.ldc % 2 == 0 && (((uintptr_t)cw) & 15) == 0;
      constexpr int CH = L::EPI_CH;
#pragma unroll 1
      for (int ch = 0; ch < BN / CH; ++ch) {
        uint32_t vr[CH], vi[CH];
        const uint32_t base = tmem + lane_base + pb * (uint32_t)L::P_COLS + (uint32_t)(ch * CH);
        tmem_ld_cols<CH>(base, vr);
        tmem_ld_cols<CH>(base + BN, vi);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (ch == BN / CH - 1) {  // the whole tile is in registers/staging: free the buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accfree[pb]))
                         : "memory");
        }
        if (g.c_nblk && !use_beta && g.c_nblk % 2 == 0 && g.ldc % 2 == 0 && g.c_bstride % 2 == 0) {
          // column blocks, 16-byte stores: a column pair never straddles a block
          const int64_t m = m0 + lane;
          float2 *cb = Cb + (int64_t)ec.bidx * g.sC + m * g.ldc;
#pragma unroll
          for (int c = 0; c < CH; c += 2) {
            const int64_t n = (int64_t)ec.nt * BN + ch * CH + c;
            if (ch * CH + c < ntile && m < g.M) {
              const int64_t q = n / g.c_nblk;
              const float xr = __uint_as_float(vr[c]), xi = __uint_as_float(vi[c]);
              const float yr = __uint_as_float(vr[c + 1]), yi = __uint_as_float(vi[c + 1]);
              *reinterpret_cast<float4 *>(cb + q * g.c_bstride + (n - q * g.c_nblk)) =
                  make_float4(ar * xr - ai * xi, ar * xi + ai * xr, ar * yr - ai * yi, ar * yi + ai * yr);
            }
          }
        } else if (g.c_nblk) {
          // column blocks: this lane's row, c_nblk consecutive columns per block
          const int64_t m = m0 + lane;
          float2 *cb = Cb + (int64_t)ec.bidx * g.sC + m * g.ldc;
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int64_t n = (int64_t)ec.nt * BN + ch * CH + c;
            if (ch * CH + c < ntile && m < g.M) {
              const int64_t q = n / g.c_nblk;
              const float xr = __uint_as_float(vr[c]), xi = __uint_as_float(vi[c]);
              float2 o = make_float2(ar * xr - ai * xi, ar * xi + ai * xr);
              float2 *cp = cb + q * g.c_bstride + (n - q * g.c_nblk);
              if (use_beta) {
                const float2 cv = *cp;
                o.x += br * cv.x - bi * cv.y;
                o.y += br * cv.y + bi * cv.x;
              }
              *cp = o;
            }
          }
        } else if (g.c_trans) {
          // transposed C: column n of these 32 rows is one 256-byte run
          const int64_t m = m0 + lane;
          float2 *ct = Cb + (int64_t)ec.bidx * g.sC + m;
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int64_t n = (int64_t)ec.nt * BN + ch * CH + c;
            if (ch * CH + c < ntile && m < g.M) {
              const float xr = __uint_as_float(vr[c]), xi = __uint_as_float(vi[c]);
              float2 o = make_float2(ar * xr - ai * xi, ar * xi + ai * xr);
              if (use_beta) {
                const float2 cv = ct[n * g.ldc];
                o.x += br * cv.x - bi * cv.y;
                o.y += br * cv.y + bi * cv.x;
              }
              ct[n * g.ldc] = o;
            }
          }
        } else {
          stage_store_chunk<CH, L::EPI_PITCH>(stg, vr, vi, cw + ch * CH, g.ldc, g.M - m0,
                                              ntile - ch * CH, ar, ai, br, bi, use_beta, vec, lane);
        }
      }
    }
  } else if constexpr (NPW > 0) {
    // ===== converter warps fed by the producers: raw rows -> registers
    // (slot released at once), split, B' planes + tcgen05.st of A
    int b_n, b_k;
    uint32_t boff;
    constexpr int BE = (BN * KB) / NT;  // B elements per thread per k-block (BN = 64)
    if constexpr (BE == 2) {
      // half-warps split by k pair: each half reads one contiguous 128-byte
      // run of a k row of the raw B box (conflict-free), the B' stores of the
      // two halves interleave 8-byte words of the same core-matrix rows
      const int b_kp = (tid >> 4) & 1, b_chunk = tid >> 7;
      b_n = (tid & 15) | (((tid >> 5) & 3) << 4);
      b_k = b_chunk * 4 + b_kp * 2;
      boff = core_off(b_n, b_chunk) + (uint32_t)(b_kp * 8);
    } else {
      b_k = tid & 7;
      b_n = tid >> 3;
      boff = core_off(b_n, b_k >> 2) + (uint32_t)((b_k & 3) * 4);
    }
    const uint32_t kw0 = (uint32_t)(wg * KPW);
    constexpr int CPR = KPW / 2;
    Cur cc;
    cur_init(cc, w0);
    uint32_t q = 0;
    for (; cc.w < w1; cur_next(cc)) {
      const bool breuse = rd != 0u && cc.run >= rd;
      for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
        const uint32_t slot = q & (RAW - 1), s = q & (STAGES - 1);
        mbar_wait(&rawfull[slot], (q / RAW) & 1u);
        const uint8_t *rA = smem + L::RAWA_OFF + slot * L::RAWA_SLOT;
        const uint8_t *rB = smem + L::RAWB_OFF + slot * L::RAWB_SLOT;
        float4 av[CPR];
        float4 bb4 = make_float4(0.f, 0.f, 0.f, 0.f);
        float2 bb2 = make_float2(0.f, 0.f);
        if constexpr (TMA) {
          // 64-byte swizzle: the 16-byte chunk c of row r sits at chunk c ^ ((r >> 1) & 3)
          if (g.opA == QF_OP_N) {
#pragma unroll
            for (int p = 0; p < CPR; ++p) {
              const int c = (int)(kw0 >> 1) + p;
              av[p] = *reinterpret_cast<const float4 *>(rA + row_l * 64 + ((c ^ ((row_l >> 1) & 3)) << 4));
            }
          } else {  // [8 k][128 rows] dense
#pragma unroll
            for (int p = 0; p < CPR; ++p) {
              const float2 x0 = *reinterpret_cast<const float2 *>(rA + (kw0 + 2 * p) * 1024 + row_l * 8);
              const float2 x1 = *reinterpret_cast<const float2 *>(rA + (kw0 + 2 * p + 1) * 1024 + row_l * 8);
              av[p] = make_float4(x0.x, x0.y, x1.x, x1.y);
            }
          }
          if (!breuse) {
            if (g.opB == QF_OP_N) {  // [8 k][64 n] dense
              const float2 y0 = *reinterpret_cast<const float2 *>(rB + b_k * (BN * 8) + b_n * 8);
              if constexpr (BE == 2) {
                const float2 y1 = *reinterpret_cast<const float2 *>(rB + (b_k + 1) * (BN * 8) + b_n * 8);
                bb4 = make_float4(y0.x, y0.y, y1.x, y1.y);
              } else {
                bb2 = y0;
              }
            } else {  // [64 n][64 B] swizzled
              const int c = b_k >> 1;
              const uint8_t *rowp = rB + b_n * 64 + ((c ^ ((b_n >> 1) & 3)) << 4);
              if constexpr (BE == 2) bb4 = *reinterpret_cast<const float4 *>(rowp);
              else bb2 = *reinterpret_cast<const float2 *>(rowp + (b_k & 1) * 8);
            }
          }
        } else {
          const uint8_t *ra = rA + row_l * L::RPITCH + kw0 * 8;
#pragma unroll
          for (int p = 0; p < CPR; ++p) av[p] = *reinterpret_cast<const float4 *>(ra + 16 * p);
          if (!breuse) {
            const uint8_t *rb = rB + b_n * L::RPITCH + b_k * 8;
            if constexpr (BE == 2) bb4 = *reinterpret_cast<const float4 *>(rb);
            else bb2 = *reinterpret_cast<const float2 *>(rb);
          }
        }
        __syncwarp();
        if (lane == 0)  // release semantics order the reads above before the refill
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rawfree[slot]))
                       : "memory");
        if (q >= STAGES) mbar_wait(&bars[s], ((q / STAGES) + 1) & 1u);
        if (!breuse) {
          uint8_t *stage = smem + s * L::STAGE;
          uint8_t *ph = stage, *pl = stage + L::B_PLANE;
          if constexpr (BE == 2) {
            uint32_t hr0, lr0, hi0, li0, hr1, lr1, hi1, li1;
            split_fast(bb4.x, hr0, lr0);
            split_fast(bb4.y, hi0, li0);
            split_fast(bb4.z, hr1, lr1);
            split_fast(bb4.w, hi1, li1);
            *reinterpret_cast<uint2 *>(ph + 0 * L::B_BLOCK + boff) =
                make_uint2(hi0 ^ 0x80000000u, hi1 ^ 0x80000000u);
            *reinterpret_cast<uint2 *>(ph + 1 * L::B_BLOCK + boff) = make_uint2(hr0, hr1);
            *reinterpret_cast<uint2 *>(ph + 2 * L::B_BLOCK + boff) = make_uint2(hi0, hi1);
            *reinterpret_cast<uint2 *>(pl + 0 * L::B_BLOCK + boff) =
                make_uint2(li0 ^ 0x80000000u, li1 ^ 0x80000000u);
            *reinterpret_cast<uint2 *>(pl + 1 * L::B_BLOCK + boff) = make_uint2(lr0, lr1);
            *reinterpret_cast<uint2 *>(pl + 2 * L::B_BLOCK + boff) = make_uint2(li0, li1);
          } else {
            uint32_t hr, lr, hi, li;
            split_fast(bb2.x, hr, lr);
            split_fast(bb2.y, hi, li);
            *reinterpret_cast<uint32_t *>(ph + 0 * L::B_BLOCK + boff) = hi ^ 0x80000000u;
            *reinterpret_cast<uint32_t *>(ph + 1 * L::B_BLOCK + boff) = hr;
            *reinterpret_cast<uint32_t *>(ph + 2 * L::B_BLOCK + boff) = hi;
            *reinterpret_cast<uint32_t *>(pl + 0 * L::B_BLOCK + boff) = li ^ 0x80000000u;
            *reinterpret_cast<uint32_t *>(pl + 1 * L::B_BLOCK + boff) = lr;
            *reinterpret_cast<uint32_t *>(pl + 2 * L::B_BLOCK + boff) = li;
          }
          fence_async_smem();
        }
        {
          uint32_t rh[KPW], rl[KPW], ih[KPW], il[KPW];
#pragma unroll
          for (int p = 0; p < CPR; ++p) {
            split_fast(av[p].x, rh[2 * p], rl[2 * p]);
            split_fast(av[p].y, ih[2 * p], il[2 * p]);
            split_fast(av[p].z, rh[2 * p + 1], rl[2 * p + 1]);
            split_fast(av[p].w, ih[2 * p + 1], il[2 * p + 1]);
          }
          const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * 32) + kw0;
          if constexpr (KPW == 4) {
            tmem_st4(acol + 0, rh[0], rh[1], rh[2], rh[3]);
            tmem_st4(acol + 8, rl[0], rl[1], rl[2], rl[3]);
            tmem_st4(acol + 16, ih[0], ih[1], ih[2], ih[3]);
            tmem_st4(acol + 24, il[0], il[1], il[2], il[3]);
          } else {
            tmem_st2(acol + 0, rh[0], rh[1]);
            tmem_st2(acol + 8, rl[0], rl[1]);
            tmem_st2(acol + 16, ih[0], ih[1]);
            tmem_st2(acol + 24, il[0], il[1]);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      }
    }
  } else {
    const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
    const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
    float2 *Cb = reinterpret_cast<float2 *>(g.C);
    const bool k_tail = (K % KB) != 0;
    const bool a_vec = (g.opA == QF_OP_N) && (g.lda % 2 == 0) && (g.sA % 2 == 0);
    const bool b_vec = (g.opB == QF_OP_T) && (g.ldb % 2 == 0) && (g.sB % 2 == 0);
    const int64_t a_kstride = (g.opA == QF_OP_N) ? 1 : g.lda;
    const int64_t b_kstride = (g.opB == QF_OP_N) ? g.ldb : 1;
    const uint32_t kw0 = (uint32_t)(wg * KPW);  // this warp's first k inside a k-block

    // ---- A fetch.  The converter lane of TMEM row r needs row r's KPW k values.
    //   1 gathered, k contiguous : lanes along k (kq = lane % KPW), rows
    //                              lane/KPW + (32/KPW) i, 8 B each
    //   3 gathered, rows contiguous (the innermost memory axis is a row
    //                              label): lane = row, KPW 8-byte loads
    //   2 row-major: lanes along k pairs (kp = lane % CPR), rows lane/CPR + (32/CPR) i, 16 B
    //   0 otherwise: lane = row, KPW 8-byte loads
    // Raw slot: thread t's k pair p at p * NT * 16 + t * 16.
    constexpr int CPR = KPW / 2;
    const bool rows_unit = gat && g.M > 1 && __ldg(g.a_roff + 1) - __ldg(g.a_roff) == 1;
    const int a_mode = gat ? (rows_unit ? 3 : 1) : (a_vec ? 2 : 0);
    const uint32_t rawa_base = smem_u32(smem + L::RAWA_OFF);
    const uint32_t rawa_m =
        rawa_base + (a_mode == 1 ? (uint32_t)(((lane % KPW) >> 1) * NT * 16 +
                                              (warp * 32 + lane / KPW) * 16 + (lane & 1) * 8)
                                 : (uint32_t)((lane % CPR) * NT * 16 + (warp * 32 + lane / CPR) * 16));
    const uint32_t rawa0 = rawa_base + (uint32_t)tid * 16;
    // ---- B fetch: NW = 8 -> 2 consecutive k of one column per thread (16 B);
    // NW = 16 -> one element per thread, k fastest
    constexpr int BEL = BN * KB;                   // B elements per k-block
    constexpr int BE = BEL >= NT ? BEL / NT : 1;   // per participating thread
    const bool b_thr = tid < BEL;
    int b_n, b_k;
    uint32_t boff;
    if constexpr (BE == 2) {
      const int b_kp = tid & 1, b_chunk = tid >> 7;
      b_n = (tid >> 1) & (BN - 1);
      b_k = b_chunk * 4 + b_kp * 2;
      boff = core_off(b_n, b_chunk) + (uint32_t)(b_kp * 8);
    } else {
      b_k = tid & 7;
      b_n = tid >> 3;
      boff = core_off(b_n, b_k >> 2) + (uint32_t)((b_k & 3) * 4);
    }
    const uint32_t rawb0 = smem_u32(smem + L::RAWB_OFF) + (uint32_t)tid * (8 * BE);

    Cur fc;
    cur_init(fc, w0);
    uint32_t f_kb = 0;
    const float2 *fa = Ab, *fb = Bb;
    bool fa_ok = false, fb_ok = false, f_breuse = false;
    uint32_t amask = 0, amask_next = 0;
    int32_t ro[KPW], ro_next[KPW];
#pragma unroll
    for (int i = 0; i < KPW; ++i) ro[i] = ro_next[i] = 0;
    // gathered row offsets of M tile mt (clamped loads: the value lands in its
    // register without a predicated copy, so the prefetch really overlaps)
    auto load_ro = [&](uint32_t mt, int32_t(&dst)[KPW], uint32_t &mask) {
      mask = 0;
      const int64_t mlast = g.M - 1;
      if (a_mode == 3) {
        const int64_t r = (int64_t)mt * BM + row_l;
        dst[0] = __ldg(g.a_roff + min(r, mlast));
        mask = r <= mlast ? 1u : 0u;
        return;
      }
      const int64_t r0 = (int64_t)mt * BM + lg * 32 + lane / KPW;
#pragma unroll
      for (int i = 0; i < KPW; ++i) {
        const int64_t r = r0 + (32 / KPW) * i;
        dst[i] = __ldg(g.a_roff + min(r, mlast));
        mask |= r <= mlast ? (1u << i) : 0u;
      }
    };
    auto fetch_setup = [&]() {
      if (fc.w >= w1) return;
      const float2 *A = Ab + a_batch_off(g, fc.bidx);
      const float2 *B = Bb + b_batch_off(g, fc.bidx);
      const int64_t m0 = (int64_t)fc.mt * BM;
      if (a_mode == 1 || a_mode == 3) {
#pragma unroll
        for (int i = 0; i < KPW; ++i) ro[i] = ro_next[i];
        amask = amask_next;
        fa = a_mode == 3 ? A + ro[0] : A;
        if (fc.w + 1 < w1) load_ro(fc.mt + 1 == tiles_m ? 0u : fc.mt + 1, ro_next, amask_next);
      } else if (a_mode == 2) {
        const int64_t r0 = m0 + lg * 32 + lane / CPR;
        amask = 0;
#pragma unroll
        for (int i = 0; i < CPR; ++i) amask |= (r0 + (32 / CPR) * i < g.M) ? (1u << i) : 0u;
        fa = A + r0 * g.lda + kw0 + 2 * (lane % CPR);
      } else {
        const int64_t am = m0 + row_l;
        fa_ok = am < g.M;
        fa = (g.opA == QF_OP_N) ? A + am * g.lda + kw0 : A + (int64_t)kw0 * g.lda + am;
        if (!fa_ok) fa = Ab;
      }
      f_breuse = rd != 0u && fc.run >= rd;
      const int64_t bn = (int64_t)fc.nt * BN + b_n;
      fb_ok = bn < g.N;
      fb = (g.opB == QF_OP_N) ? B + (int64_t)b_k * g.ldb + bn : B + bn * g.ldb + b_k;
      if (!fb_ok) fb = Bb;
    };
    auto fetch = [&](uint32_t slot) {
      if (fc.w < w1) {
        const bool tail = k_tail && f_kb == nk - 1;
        const uint32_t dm = rawa_m + slot * L::RAWA_SLOT;
        const uint32_t kk0 = f_kb * KB + kw0;
        if (a_mode == 3) {  // lane = row: KPW offsets of this warp's k from the table
          const uint32_t da = rawa0 + slot * L::RAWA_SLOT;
          int32_t c[KPW];
          if constexpr (KPW == 4) {
            const int4 v = *reinterpret_cast<const int4 *>(s_coff + kk0);
            c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
          } else {
            const int2 v = *reinterpret_cast<const int2 *>(s_coff + kk0);
            c[0] = v.x; c[1] = v.y;
          }
          if (tail) {
#pragma unroll
            for (int k = 0; k < KPW; ++k) c[k] = kk0 + k < K ? c[k] : 0;
          }
#pragma unroll
          for (int k = 0; k < KPW; ++k)
            cp_async8(da + (k >> 1) * NT * 16 + (k & 1) * 8, fa + c[k],
                      (amask & 1u) && (!tail || kk0 + k < K));
        } else if (a_mode == 1) {  // lanes along k, KPW rows each
          const uint32_t kk = kk0 + (lane % KPW);
          const bool kok = !tail || kk < K;
          const int32_t c = s_coff[kok ? kk : 0u];
#pragma unroll
          for (int i = 0; i < KPW; ++i)
            cp_async8(dm + i * (32 / KPW) * 16, fa + (ro[i] + c), kok && ((amask >> i) & 1u));
        } else if (a_mode == 2) {
          if (!tail) {
#pragma unroll
            for (int i = 0; i < CPR; ++i) {
              const bool ok = (amask >> i) & 1u;
              cp_async16(dm + i * (32 / CPR) * 16, ok ? fa + i * (32 / CPR) * g.lda : Ab, ok);
            }
          } else {
            const uint32_t k0 = kk0 + 2 * (lane % CPR);
#pragma unroll
            for (int e = 0; e < 2 * CPR; ++e) {
              const int i = e >> 1, j = e & 1;
              const bool ok = ((amask >> i) & 1u) && k0 + j < K;
              cp_async8(dm + i * (32 / CPR) * 16 + j * 8, ok ? fa + i * (32 / CPR) * g.lda + j : Ab, ok);
            }
          }
          fa += KB;
        } else {
          const uint32_t da = rawa0 + slot * L::RAWA_SLOT;
#pragma unroll
          for (int k = 0; k < KPW; ++k) {
            const bool ok = fa_ok && (!tail || kk0 + k < K);
            cp_async8(da + (k >> 1) * NT * 16 + (k & 1) * 8, ok ? fa + k * a_kstride : Ab, ok);
          }
          if (fa_ok) fa += KB * a_kstride;
        }
        if (!f_breuse && b_thr) {
          const uint32_t db = rawb0 + slot * L::RAWB_SLOT;
          const uint32_t k0 = f_kb * KB + b_k;
          if constexpr (BE == 2) {
            if (!tail) {
              if (b_vec) {
                cp_async16(db, fb, fb_ok);
              } else {
                cp_async8(db, fb, fb_ok);
                cp_async8(db + 8, fb + b_kstride, fb_ok);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const bool ok = fb_ok && k0 + e < K;
                cp_async8(db + 8 * e, ok ? fb + e * b_kstride : Bb, ok);
              }
            }
          } else {
            const bool ok = fb_ok && (!tail || k0 < K);
            cp_async8(db, ok ? fb : Bb, ok);
          }
          if (fb_ok) fb += KB * b_kstride;
        }
        if (++f_kb == nk) {
          f_kb = 0;
          cur_next(fc);
          fetch_setup();
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");  // uniform group count
    };

    auto epilogue = [&](uint32_t mt, uint32_t nt, uint32_t bidx, uint32_t t) {
      const uint32_t pb = t & 1u;
      mbar_wait(&pbar[pb], (t >> 1) & 1u);
      tc_fence_after();
      uint32_t vr[CPW], vi[CPW];
      const uint32_t base = tmem + lane_base + pb * (uint32_t)L::P_COLS + (uint32_t)(wg * CPW);
      tmem_ld_cols<CPW>(base, vr);
      tmem_ld_cols<CPW>(base + BN, vi);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      const int64_t m0 = (int64_t)mt * BM + lg * 32;  // this warp's 32 rows
      const int64_t c0 = (int64_t)nt * BN + wg * CPW;
      const int64_t ncols = min((int64_t)CPW, g.N - c0);
      const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
      const bool use_beta = (br != 0.f || bi != 0.f);
      float2 *cw = Cb + (int64_t)bidx * g.sC + m0 * g.ldc + c0;
      // staged, coalesced stores for every case (alpha/beta/ragged edges
      // included): no lane-divergent path next to the .sync.aligned
      // tcgen05 instructions of the following k-block
      uint8_t *stg = smem + L::EPI_OFF + warp * 32 * L::EPI_PITCH;
      const bool vec = g.ldc % 2 == 0 && (((uintptr_t)cw) & 15) == 0;
      if constexpr (CPW >= 8)
        stage_store_chunk<CPW, L::EPI_PITCH>(stg, vr, vi, cw, g.ldc, g.M - m0, ncols, ar, ai, br,
                                             bi, use_beta, vec, lane);
    };

    if ((a_mode == 1 || a_mode == 3) && w0 < w1) load_ro(fc.mt, ro_next, amask_next);
    fetch_setup();
    for (int i = 0; i < RAW - 1; ++i) fetch((uint32_t)i);
    Cur cc;
    cur_init(cc, w0);
    uint32_t pmt = 0, pnt = 0, pbidx = 0;  // the previous tile (its epilogue is pending)
    uint32_t q = 0, t = 0;
    for (; cc.w < w1; cur_next(cc), ++t) {
      const bool breuse = rd != 0u && cc.run >= rd;
      for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
        fetch((q + RAW - 1) & (RAW - 1));
        asm volatile("cp.async.wait_group %0;" ::"n"(RAW - 1) : "memory");
        if (a_mode == 1 || a_mode == 2) __syncwarp();  // rows fetched by other lanes of this warp
        const uint32_t s = q & (STAGES - 1);
        if (q >= STAGES) mbar_wait(&bars[s], ((q / STAGES) + 1) & 1u);
        const uint32_t slot = q & (RAW - 1);
        float4 av[CPR];
#pragma unroll
        for (int p = 0; p < CPR; ++p)
          av[p] = *reinterpret_cast<const float4 *>(smem + L::RAWA_OFF + slot * L::RAWA_SLOT +
                                                     p * NT * 16 + tid * 16);
        if (!breuse && b_thr) {
          uint8_t *stage = smem + s * L::STAGE;
          uint8_t *ph = stage, *pl = stage + L::B_PLANE;
          if constexpr (BE == 2) {
            const float4 bb = *reinterpret_cast<const float4 *>(smem + L::RAWB_OFF +
                                                                 slot * L::RAWB_SLOT + tid * 16);
            uint32_t hr0, lr0, hi0, li0, hr1, lr1, hi1, li1;
            split_fast(bb.x, hr0, lr0);
            split_fast(bb.y, hi0, li0);
            split_fast(bb.z, hr1, lr1);
            split_fast(bb.w, hi1, li1);
            *reinterpret_cast<uint2 *>(ph + 0 * L::B_BLOCK + boff) =
                make_uint2(hi0 ^ 0x80000000u, hi1 ^ 0x80000000u);
            *reinterpret_cast<uint2 *>(ph + 1 * L::B_BLOCK + boff) = make_uint2(hr0, hr1);
            *reinterpret_cast<uint2 *>(ph + 2 * L::B_BLOCK + boff) = make_uint2(hi0, hi1);
            *reinterpret_cast<uint2 *>(pl + 0 * L::B_BLOCK + boff) =
                make_uint2(li0 ^ 0x80000000u, li1 ^ 0x80000000u);
            *reinterpret_cast<uint2 *>(pl + 1 * L::B_BLOCK + boff) = make_uint2(lr0, lr1);
            *reinterpret_cast<uint2 *>(pl + 2 * L::B_BLOCK + boff) = make_uint2(li0, li1);
          } else {
            const float2 bb = *reinterpret_cast<const float2 *>(smem + L::RAWB_OFF +
                                                                 slot * L::RAWB_SLOT + tid * 8);
            uint32_t hr, lr, hi, li;
            split_fast(bb.x, hr, lr);
            split_fast(bb.y, hi, li);
            *reinterpret_cast<uint32_t *>(ph + 0 * L::B_BLOCK + boff) = hi ^ 0x80000000u;
            *reinterpret_cast<uint32_t *>(ph + 1 * L::B_BLOCK + boff) = hr;
            *reinterpret_cast<uint32_t *>(ph + 2 * L::B_BLOCK + boff) = hi;
            *reinterpret_cast<uint32_t *>(pl + 0 * L::B_BLOCK + boff) = li ^ 0x80000000u;
            *reinterpret_cast<uint32_t *>(pl + 1 * L::B_BLOCK + boff) = lr;
            *reinterpret_cast<uint32_t *>(pl + 2 * L::B_BLOCK + boff) = li;
          }
          fence_async_smem();
        }
        {
          uint32_t rh[KPW], rl[KPW], ih[KPW], il[KPW];
#pragma unroll
          for (int p = 0; p < CPR; ++p) {
            split_fast(av[p].x, rh[2 * p], rl[2 * p]);
            split_fast(av[p].y, ih[2 * p], il[2 * p]);
            split_fast(av[p].z, rh[2 * p + 1], rl[2 * p + 1]);
            split_fast(av[p].w, ih[2 * p + 1], il[2 * p + 1]);
          }
          const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * 32) + kw0;
          if constexpr (KPW == 4) {
            tmem_st4(acol + 0, rh[0], rh[1], rh[2], rh[3]);
            tmem_st4(acol + 8, rl[0], rl[1], rl[2], rl[3]);
            tmem_st4(acol + 16, ih[0], ih[1], ih[2], ih[3]);
            tmem_st4(acol + 24, il[0], il[1], il[2], il[3]);
          } else {
            tmem_st2(acol + 0, rh[0], rh[1]);
            tmem_st2(acol + 8, rl[0], rl[1]);
            tmem_st2(acol + 16, ih[0], ih[1]);
            tmem_st2(acol + 24, il[0], il[1]);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        if (NE == 0 && kb == nk - 1 && t > 0) epilogue(pmt, pnt, pbidx, t - 1);
      }
      pmt = cc.mt;
      pnt = cc.nt;
      pbidx = cc.bidx;
    }
    if (NE == 0 && t > 0) epilogue(pmt, pnt, pbidx, t - 1);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
}

// 3-D float tensor map (dims innermost first, strides in bytes) for TMA boxes
static bool make_tmap(CUtensorMap *m, const void *ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t s1, uint64_t s2, uint32_t b0, uint32_t b1, bool swz64) {
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {s1, s2};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  // driver entry point fetched through the runtime, so the library has no
  // link-time libcuda dependency (it must load on GPU-less build hosts)
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(ptr), dims, strides, box,
                es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                swz64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 5-D float tensor map of an A view (dims innermost first, byte strides)
static bool make_tmap5(CUtensorMap *m, const void *ptr, const uint64_t (&dims)[5],
                       const uint64_t (&strides)[4], const uint32_t (&box)[5], bool swz64 = true) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  cuuint64_t d[5];
  cuuint64_t st[4];
  cuuint32_t bx[5];
  for (int i = 0; i < 5; ++i) d[i] = dims[i], bx[i] = box[i];
  for (int i = 0; i < 4; ++i) st[i] = strides[i];
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void *>(ptr), d, st, bx, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE,
                swz64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA needs 16-byte global strides and A/B entries addressable by coordinates
// (no offset tables; B entry offsets only as whole [K][N] slices)
bool tma_ok(const GemmArgs &g) {
  const bool a_ok = !g.a_roff && (!g.a_boff || g.a_nslice > 0) && g.sA > 0 && g.sA % 2 == 0 &&
                    g.lda % 2 == 0;
  const bool b_ok = g.b_boff ? (g.b_nslice > 0 && (g.K * g.N) % 2 == 0)
                             : (g.sB > 0 && g.sB % 2 == 0);
  const bool v_ok = !g.v_kin ||
                    (g.v_t ? (g.v_kin % KB == 0 && g.v_ski % 2 == 0 && g.v_skout % 2 == 0 &&
                              g.v_srb % 2 == 0 && g.v_ra % 2 == 0 &&
                              (g.v_ra >= BM ? g.v_ra % BM == 0 : BM % g.v_ra == 0) &&
                              g.opA == QF_OP_T)
                           : (g.v_kin % KB == 0 && g.v_sra % 2 == 0 && g.v_skout % 2 == 0 &&
                              g.v_srb % 2 == 0 &&
                              (g.v_ra >= BM ? g.v_ra % BM == 0 : BM % g.v_ra == 0) &&
                              g.opA == QF_OP_N));
  return a_ok && b_ok && v_ok && g.ldb % 2 == 0 &&
         (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(g.B) & 15) == 0 &&
         g.batch < ((int64_t)1 << 31);
}

template <int STAGES, int RAW, int NW, int NE, int BN = V2_BN, int CK = 0, int NPW = 0, bool TMA = false>
int launch_short(const GemmArgs &g, cudaStream_t s) {
  using L = LayoutK<STAGES, RAW, NW, NE, BN, CK, NPW, TMA>;
  auto kern = cgemm_tc3k_kernel<STAGES, RAW, NW, NE, BN, CK, NPW, TMA>;
  CUtensorMap tmA{}, tmB{};
  if constexpr (TMA) {
    const uint64_t nb = (uint64_t)std::max<int64_t>(g.batch, 1);
    const uint64_t na = g.a_boff ? (uint64_t)g.a_nslice : nb;   // A entries addressable
    bool okA;
    if (g.v_t) {
      // transposed view: dims {2 ra, rb, ki, ko, b} (strides need not be
      // monotonic), box {2 min(ra, 128), 128 / min(ra, 128), 8, 1, 1} lands as
      // the dense [8 k][128 rows] tile of the plain opA = T path
      const uint32_t bra = (uint32_t)std::min<int64_t>(g.v_ra, BM);
      const uint64_t dims[5] = {(uint64_t)(2 * g.v_ra), (uint64_t)g.v_rb, (uint64_t)g.v_kin,
                                (uint64_t)g.v_kout, na};
      const uint64_t strides[4] = {(uint64_t)g.v_srb * 8, (uint64_t)g.v_ski * 8,
                                   (uint64_t)g.v_skout * 8, (uint64_t)std::max<int64_t>(g.sA, 1) * 8};
      const uint32_t box[5] = {2 * bra, (uint32_t)(BM / bra), (uint32_t)KB, 1, 1};
      okA = make_tmap5(&tmA, g.A, dims, strides, box, false);
    } else if (g.v_kin) {
      const uint32_t bra = (uint32_t)std::min<int64_t>(g.v_ra, BM);
      const uint64_t dims[5] = {(uint64_t)(2 * g.v_kin), (uint64_t)g.v_ra, (uint64_t)g.v_kout,
                                (uint64_t)g.v_rb, na};
      const uint64_t strides[4] = {(uint64_t)g.v_sra * 8, (uint64_t)g.v_skout * 8,
                                   (uint64_t)g.v_srb * 8, (uint64_t)std::max<int64_t>(g.sA, 1) * 8};
      const uint32_t box[5] = {16, bra, 1, (uint32_t)(BM / bra), 1};
      okA = make_tmap5(&tmA, g.A, dims, strides, box);
    } else {
      okA = g.opA == QF_OP_N
                ? make_tmap(&tmA, g.A, 2 * g.K, g.M, na, g.lda * 8, std::max<int64_t>(g.sA, 1) * 8, 16, 128, true)
                : make_tmap(&tmA, g.A, 2 * g.M, g.K, na, g.lda * 8, std::max<int64_t>(g.sA, 1) * 8, 256, 8, false);
    }
    // B entries: strided batch, or b_nslice whole [K][N] slices picked per entry
    const uint64_t nbs = g.b_boff ? (uint64_t)g.b_nslice : nb;
    const int64_t sbs = g.b_boff ? g.K * g.N : std::max<int64_t>(g.sB, 1);
    const bool okB = g.opB == QF_OP_N
                         ? make_tmap(&tmB, g.B, 2 * g.N, g.K, nbs, g.ldb * 8, sbs * 8, 2 * BN, 8, false)
                         : make_tmap(&tmB, g.B, 2 * g.K, g.N, nbs, g.ldb * 8, sbs * 8, 16, BN, true);
    if (!okA || !okB) {
      set_error("tc3k: cuTensorMapEncodeTiled failed (M=%lld N=%lld K=%lld)", (long long)g.M,
                (long long)g.N, (long long)g.K);
      return QF_ERR_CUDA;
    }
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3k: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  if ((CK == 0 && g.K > 256) || (g.a_roff && g.K > L::COFF_MAX)) {
    set_error("tc3k: K = %lld exceeds the %s limit", (long long)g.K,
              CK == 0 ? "short-K (unpromoted) 256" : "gathered-A 4096");
    return QF_ERR_INVALID;
  }
  const int64_t tiles_n = (g.N + L::BN - 1) / L::BN, tiles_m = (g.M + BM - 1) / BM;
  const int64_t total = tiles_n * tiles_m * g.batch;
  if (total >= (int64_t)1 << 31) {
    set_error("tc3k: %lld tiles exceed the 32-bit tile index", (long long)total);
    return QF_ERR_INVALID;
  }
  const int64_t grid0 = std::min<int64_t>(total, (int64_t)sm_count());
  const int64_t chunk = (total + grid0 - 1) / grid0;
  const int64_t grid = CK > 0 ? grid0 : (total + chunk - 1) / chunk;  // long K: strided tiles
  kern<<<(unsigned)grid, (NW + NE + NPW) * 32 + 32, L::SMEM, s>>>(
      g, (uint32_t)tiles_m, (uint32_t)tiles_n, (uint32_t)total, (uint32_t)chunk, tmA, tmB);
  return check_launch("cgemm_tc3k");
}

template <int STAGES, int CK, int RAW>
int launch_v3(const GemmArgs &g, cudaStream_t s) {
  using L = LayoutV3<STAGES, CK, RAW>;
  auto kern = cgemm_tc3s_kernel<STAGES, CK, RAW>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3s: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  const int64_t tiles_n = (g.N + L::BN - 1) / L::BN, tiles_m = (g.M + BM - 1) / BM;
  const int64_t tiles = tiles_n * tiles_m;
  const int64_t grid = std::min<int64_t>(tiles * g.batch, (int64_t)sm_count());
  kern<<<(unsigned)grid, V2_THREADS, L::SMEM, s>>>(g, tiles_n, tiles);
  return check_launch("cgemm_tc3s");
}


// ---------------------------------------------------------------------------
// "reg" variant: 8 warps (255-register budget), operands prefetched D
// k-blocks ahead straight into registers (no raw shared-memory ring: that
// ring was ~40% of the kernel's shared-memory traffic), per-stage `full`
// mbarriers, and warp 0's elected lane issues the MMAs after waiting on them.

template <int STAGES, int CK, int D>
struct LayoutR {
  static_assert((STAGES & (STAGES - 1)) == 0 && (CK & (CK - 1)) == 0, "powers of two");
  static constexpr int BN = V2_BN;
  static constexpr int NP = 2 * BN;
  static constexpr int B_BLOCK = BN * 32;
  static constexpr int B_PLANE = 3 * B_BLOCK;
  static constexpr int STAGE = 2 * B_PLANE;
  static constexpr int BAR_OFF = STAGES * STAGE;
  static constexpr int SMEM = BAR_OFF + 1024;
  static constexpr int P_COLS = NP;
  static constexpr int A_COL0 = 2 * P_COLS;
  static constexpr int TMEM_COLS = 512;
  static constexpr int LOG_STAGES = STAGES == 2 ? 1 : STAGES == 4 ? 2 : 3;
  static constexpr int LOG_CK = CK == 1 ? 0 : CK == 2 ? 1 : CK == 4 ? 2 : CK == 8 ? 3 : 4;
  static_assert(2 * P_COLS + STAGES * 32 <= 512, "TMEM budget");
};

template <int STAGES, int CK, int D, bool SHORTK>
__global__ void __launch_bounds__(V2_THREADS, 1)
    cgemm_tc3r_kernel(const __grid_constant__ GemmArgs g, int64_t tiles_n, int64_t tiles) {
  using L = LayoutR<STAGES, CK, D>;
  constexpr int BN = L::BN;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);  // [STAGES] stage free
  uint64_t *pbar = bars + STAGES;                                    // [2] partial done
  uint64_t *full = pbar + 2;                                         // [STAGES] converted
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(full + STAGES);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3, half = warp >> 2;
  const int row_l = lg * 32 + lane;
  const int b_kp = tid & 1;
  const int b_n = (tid >> 1) & (BN - 1);
  const int b_chunk = tid >> 7;
  const int b_k = b_chunk * 4 + b_kp * 2;

  if (tid == 0) {
    for (int i = 0; i < STAGES + 2; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], V2_THREADS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
  constexpr uint32_t IDESC = idesc_tf32(BM, L::NP);
  const uint32_t boff = core_off(b_n, b_chunk) + (uint32_t)(b_kp * 8);

  const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
  const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
  float2 *Cb = reinterpret_cast<float2 *>(g.C);
  const uint32_t nk = (uint32_t)((g.K + KB - 1) / KB);
  const bool k_tail = (g.K % KB) != 0;
  const int64_t total_work = tiles * g.batch;
  const bool a_vec = (g.opA == QF_OP_N) && (g.lda % 2 == 0) && (g.sA % 2 == 0);
  const bool b_vec = (g.opB == QF_OP_T) && (g.ldb % 2 == 0) && (g.sB % 2 == 0);
  const int64_t a_kstride = (g.opA == QF_OP_N) ? 1 : g.lda;
  const int64_t b_kstride = (g.opB == QF_OP_N) ? g.ldb : 1;

  // ---- fetch cursor (register prefetch D k-blocks ahead)
  int64_t f_work = blockIdx.x;
  uint32_t f_kb = 0;
  const float2 *fa = Ab, *fb = Bb;
  bool fa_ok = false, fb_ok = false;
  auto fetch_setup = [&]() {
    if (f_work >= total_work) return;
    const int64_t bidx = f_work / tiles;
    const int64_t tile = f_work - bidx * tiles;
    const int64_t am = (tile / tiles_n) * BM + row_l;
    const int64_t bn = (tile % tiles_n) * BN + b_n;
    fa_ok = am < g.M;
    fb_ok = bn < g.N;
    const float2 *A = Ab + a_batch_off(g, bidx);
    const float2 *B = Bb + b_batch_off(g, bidx);
    fa = (g.opA == QF_OP_N) ? A + am * g.lda + 4 * half : A + (int64_t)(4 * half) * g.lda + am;
    fb = (g.opB == QF_OP_N) ? B + (int64_t)b_k * g.ldb + bn : B + bn * g.ldb + b_k;
    if (!fa_ok) fa = Ab;
    if (!fb_ok) fb = Bb;
  };
  float4 ra0[D], ra1[D], rb[D];
  auto fetch = [&](auto dc) {
    constexpr int d = decltype(dc)::value;
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    ra0[d] = z;
    ra1[d] = z;
    rb[d] = z;
    if (f_work < total_work) {
      if (!(k_tail && f_kb == nk - 1)) {
        if (fa_ok) {
          if (a_vec) {
            ra0[d] = __ldg(reinterpret_cast<const float4 *>(fa));
            ra1[d] = __ldg(reinterpret_cast<const float4 *>(fa + 2));
          } else {
            const float2 x0 = __ldg(fa), x1 = __ldg(fa + a_kstride), x2 = __ldg(fa + 2 * a_kstride),
                         x3 = __ldg(fa + 3 * a_kstride);
            ra0[d] = make_float4(x0.x, x0.y, x1.x, x1.y);
            ra1[d] = make_float4(x2.x, x2.y, x3.x, x3.y);
          }
        }
        if (fb_ok) {
          if (b_vec) {
            rb[d] = __ldg(reinterpret_cast<const float4 *>(fb));
          } else {
            const float2 y0 = __ldg(fb), y1 = __ldg(fb + b_kstride);
            rb[d] = make_float4(y0.x, y0.y, y1.x, y1.y);
          }
        }
      } else {
        const int64_t k0 = (int64_t)f_kb * KB;
        float2 x[4] = {}, y[2] = {};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (fa_ok && k0 + 4 * half + k < g.K) x[k] = __ldg(fa + k * a_kstride);
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (fb_ok && k0 + b_k + e < g.K) y[e] = __ldg(fb + e * b_kstride);
        ra0[d] = make_float4(x[0].x, x[0].y, x[1].x, x[1].y);
        ra1[d] = make_float4(x[2].x, x[2].y, x[3].x, x[3].y);
        rb[d] = make_float4(y[0].x, y[0].y, y[1].x, y[1].y);
      }
      if (fa_ok) fa += KB * a_kstride;
      if (fb_ok) fb += KB * b_kstride;
      if (++f_kb == nk) {
        f_kb = 0;
        f_work += gridDim.x;
        fetch_setup();
      }
    }
  };

  fetch_setup();
  // prologue: D k-blocks in flight
  [&]<int... I>(std::integer_sequence<int, I...>) {
    (fetch(std::integral_constant<int, I>{}), ...);
  }(std::make_integer_sequence<int, D>{});

  uint32_t q = 0, qm_tile = 0;
  uint32_t pwaits[2] = {0, 0};
  const uint32_t nch = (nk + CK - 1) >> L::LOG_CK;
  uint32_t tcount = 0;
  bool have_prev = false;
  int prev_pb = 0;
  int64_t prev_m0 = 0, prev_n0 = 0;
  float2 *prev_C = nullptr;
  float racc[32], iacc[32];

  auto wait_partial = [&](int pb) {
    mbar_wait(&pbar[pb], pwaits[pb] & 1u);
    ++pwaits[pb];
    tc_fence_after();
  };
  auto promote = [&](int pb) {
    wait_partial(pb);
    uint32_t v[32];
    const uint32_t base = tmem + lane_base + (uint32_t)(pb * L::P_COLS + 32 * half);
    tmem_ld32(base, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) racc[j] += __uint_as_float(v[j]);
    tmem_ld32(base + BN, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) iacc[j] += __uint_as_float(v[j]);
  };
  auto store_c = [&](int64_t em0, int64_t en0, float2 *eC, const float *xr, const float *xi) {
    const int64_t row = em0 + row_l;
    if (row >= g.M) return;
    const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
    const bool use_beta = (br != 0.f || bi != 0.f);
    const int64_t c0 = en0 + 32 * half;
    float2 *crow = eC + row * g.ldc + c0;
    const int64_t ncols = min((int64_t)32, g.N - c0);
    if (!use_beta && ncols == 32 && ar == 1.f && ai == 0.f && (((uintptr_t)crow) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 2)
        *reinterpret_cast<float4 *>(crow + j) = make_float4(xr[j], xi[j], xr[j + 1], xi[j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < ncols) {
          float2 o = make_float2(ar * xr[j] - ai * xi[j], ar * xi[j] + ai * xr[j]);
          if (use_beta) {
            const float2 c = crow[j];
            o.x += br * c.x - bi * c.y;
            o.y += br * c.y + bi * c.x;
          }
          crow[j] = o;
        }
      }
    }
  };
  auto tmem_epilogue = [&](int pb, int64_t em0, int64_t en0, float2 *eC) {
    wait_partial(pb);
    uint32_t vr[32], vi[32];
    const uint32_t base = tmem + lane_base + (uint32_t)(pb * L::P_COLS + 32 * half);
    tmem_ld32(base, vr);
    tmem_ld32(base + BN, vi);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    store_c(em0, en0, eC, reinterpret_cast<const float *>(vr), reinterpret_cast<const float *>(vi));
    tc_fence_before();
  };

  // one k-block: convert register buffer d, refill it, signal, maybe issue
  auto kstep = [&](auto dc, uint32_t kb, uint32_t mma_chunk) {
    constexpr int d = decltype(dc)::value;
    const uint32_t s = q & (STAGES - 1);
    if (q >= STAGES) mbar_wait(&bars[s], ((q >> L::LOG_STAGES) + 1) & 1u);
    {
      uint32_t hr0, lr0, hi0, li0, hr1, lr1, hi1, li1;
      split_fast(rb[d].x, hr0, lr0);
      split_fast(rb[d].y, hi0, li0);
      split_fast(rb[d].z, hr1, lr1);
      split_fast(rb[d].w, hi1, li1);
      uint8_t *ph = smem + s * L::STAGE, *pl = ph + L::B_PLANE;
      *reinterpret_cast<uint2 *>(ph + boff) = make_uint2(hi0 ^ 0x80000000u, hi1 ^ 0x80000000u);
      *reinterpret_cast<uint2 *>(ph + L::B_BLOCK + boff) = make_uint2(hr0, hr1);
      *reinterpret_cast<uint2 *>(ph + 2 * L::B_BLOCK + boff) = make_uint2(hi0, hi1);
      *reinterpret_cast<uint2 *>(pl + boff) = make_uint2(li0 ^ 0x80000000u, li1 ^ 0x80000000u);
      *reinterpret_cast<uint2 *>(pl + L::B_BLOCK + boff) = make_uint2(lr0, lr1);
      *reinterpret_cast<uint2 *>(pl + 2 * L::B_BLOCK + boff) = make_uint2(li0, li1);
    }
    {
      uint32_t rh[4], rl[4], ih[4], il[4];
      split_fast(ra0[d].x, rh[0], rl[0]);
      split_fast(ra0[d].y, ih[0], il[0]);
      split_fast(ra0[d].z, rh[1], rl[1]);
      split_fast(ra0[d].w, ih[1], il[1]);
      split_fast(ra1[d].x, rh[2], rl[2]);
      split_fast(ra1[d].y, ih[2], il[2]);
      split_fast(ra1[d].z, rh[3], rl[3]);
      split_fast(ra1[d].w, ih[3], il[3]);
      const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * 32 + 4 * half);
      tmem_st4(acol + 0, rh[0], rh[1], rh[2], rh[3]);
      tmem_st4(acol + 8, rl[0], rl[1], rl[2], rl[3]);
      tmem_st4(acol + 16, ih[0], ih[1], ih[2], ih[3]);
      tmem_st4(acol + 24, il[0], il[1], il[2], il[3]);
    }
    fetch(dc);  // refill this register buffer D k-blocks ahead
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    fence_async_smem();
    tc_fence_before();
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    if (warp == 0) {
      if (lane == 0) {
        mbar_wait(&full[s], (q >> L::LOG_STAGES) & 1u);
        tc_fence_after();
        const uint32_t pos = SHORTK ? kb : (kb & (CK - 1));
        const uint32_t d_t = tmem + (mma_chunk & 1u) * (uint32_t)L::P_COLS;
        const uint32_t bhi = smem_u32(smem + s * L::STAGE), blo = bhi + L::B_PLANE;
        const uint64_t b1h = smem_desc(bhi + L::B_BLOCK), b1l = smem_desc(blo + L::B_BLOCK);
        const uint64_t b2h = smem_desc(bhi), b2l = smem_desc(blo);
        const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * 32u;
        const uint32_t acc0 = pos > 0 ? 1u : 0u;
        mma_ts(d_t, a + 0, b1h, IDESC, acc0);
        mma_ts(d_t, a + 0, b1l, IDESC, 1u);
        mma_ts(d_t, a + 8, b1h, IDESC, 1u);
        mma_ts(d_t, a + 16, b2h, IDESC, 1u);
        mma_ts(d_t, a + 16, b2l, IDESC, 1u);
        mma_ts(d_t, a + 24, b2h, IDESC, 1u);
        mma_commit(&bars[s]);
        if (SHORTK ? kb == nk - 1 : (pos == CK - 1 || kb == nk - 1)) mma_commit(&pbar[mma_chunk & 1u]);
      }
      __syncwarp();
    }
    ++q;
  };

  for (int64_t work = blockIdx.x; work < total_work; work += gridDim.x, ++tcount) {
    const int64_t bidx = work / tiles;
    const int64_t tile = work - bidx * tiles;
    const int64_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    float2 *C = Cb + bidx * g.sC;
    if (!SHORTK) {
#pragma unroll
      for (int j = 0; j < 32; ++j) racc[j] = iacc[j] = 0.f;
    }
    uint32_t kb = 0;
    auto one = [&](auto dc) {
      const uint32_t chunk = SHORTK ? tcount : (kb >> L::LOG_CK);
      kstep(dc, kb, chunk);
      if constexpr (SHORTK) {
        if (kb == 0 && have_prev) {
          tmem_epilogue(prev_pb, prev_m0, prev_n0, prev_C);
          have_prev = false;
        }
      } else {
        if ((kb & (CK - 1)) == 0 && kb > 0) promote((int)(((kb >> L::LOG_CK) - 1) & 1u));
      }
      ++kb;
    };
    // the register buffer index must be static: walk k-blocks D at a time,
    // continuing the ring position q (mod D) across tiles
    while (kb < nk) {
      [&]<int... I>(std::integer_sequence<int, I...>) {
        (((q % D) == (uint32_t)I && kb < nk ? (one(std::integral_constant<int, I>{}), 0) : 0), ...);
      }(std::make_integer_sequence<int, D>{});
    }
    if constexpr (SHORTK) {
      have_prev = nk > 0;
      prev_pb = (int)(tcount & 1u);
      prev_m0 = m0;
      prev_n0 = n0;
      prev_C = C;
    } else {
      if (nk > 0) {
        promote((int)(((nk - 1) >> L::LOG_CK) & 1u));
        store_c(m0, n0, C, racc, iacc);
      }
    }
  }
  if constexpr (SHORTK) {
    if (have_prev) tmem_epilogue(prev_pb, prev_m0, prev_n0, prev_C);
  }
  (void)qm_tile;
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
}

template <int STAGES, int CK, int D, bool SHORTK>
int launch_reg(const GemmArgs &g, cudaStream_t s) {
  using L = LayoutR<STAGES, CK, D>;
  auto kern = cgemm_tc3r_kernel<STAGES, CK, D, SHORTK>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3r: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  const int64_t tiles_n = (g.N + L::BN - 1) / L::BN, tiles_m = (g.M + BM - 1) / BM;
  const int64_t tiles = tiles_n * tiles_m;
  const int64_t grid = std::min<int64_t>(tiles * g.batch, (int64_t)sm_count());
  kern<<<(unsigned)grid, V2_THREADS, L::SMEM, s>>>(g, tiles_n, tiles);
  return check_launch("cgemm_tc3r");
}


// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs computes a 256 x 64
// complex tile with M=256 MMAs issued by the leader.  Each CTA keeps its 128
// A rows in its own TMEM and HALF of every B' window in its own smem (CTA0:
// Br and -Bi, CTA1: Bi and Br at the same offsets, so the pair's windows are
// [Br|Bi] and [-Bi|Br]), which halves each SM's B conversion and the tensor
// core's shared-memory reads.  Converters of both CTAs arrive on the leader's
// `full` barrier; MMA completions multicast to both CTAs' barriers.

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_ts2(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit2(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int STAGES, int CK, int RAW>
struct LayoutP2 {
  static constexpr int BN = V2_BN;
  static constexpr int NP = 2 * BN;                 // 128: the pair's MMA N
  static constexpr int B_BLOCK = BN * 32;           // one BN-row tf32 block
  static constexpr int STAGE = 4 * B_BLOCK;         // (X, Y) x (hi, lo)
  static constexpr int RAWA_SLOT = V2_THREADS * 32;
  static constexpr int RAWB_SLOT = V2_THREADS * 16;
  static constexpr int RAWA_OFF = STAGES * STAGE;
  static constexpr int RAWB_OFF = RAWA_OFF + RAW * RAWA_SLOT;
  static constexpr int BAR_OFF = RAWB_OFF + RAW * RAWB_SLOT;
  static constexpr int SMEM = BAR_OFF + 1024;
  static constexpr int P_COLS = NP;                 // accumulator columns per partial
  static constexpr int A_COL0 = 2 * P_COLS;
  static constexpr int TMEM_COLS = 512;
  static constexpr int LOG_STAGES = STAGES == 2 ? 1 : STAGES == 4 ? 2 : 3;
  static constexpr int LOG_CK = CK == 1 ? 0 : CK == 2 ? 1 : CK == 4 ? 2 : CK == 8 ? 3 : 4;
  static_assert(2 * P_COLS + STAGES * 32 <= 512, "TMEM budget");
};

template <int STAGES, int CK, int RAW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(V2_THREADS + 32, 1)
    cgemm_tc3pair_kernel(const __grid_constant__ GemmArgs g, int64_t tiles_n, int64_t tiles) {
  using L = LayoutP2<STAGES, CK, RAW>;
  constexpr int BN = L::BN;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);  // [STAGES] stage free
  uint64_t *pbar = bars + STAGES;                                    // [2] partial done
  uint64_t *full = pbar + 2;                                         // [STAGES] (leader) converted
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(full + STAGES);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int lg = warp & 3, half = warp >> 2;
  const int row_l = lg * 32 + lane;
  const int b_kp = tid & 1;
  const int b_n = (tid >> 1) & (BN - 1);
  const int b_chunk = tid >> 7;
  const int b_k = b_chunk * 4 + b_kp * 2;
  const uint32_t crank = cluster_rank();
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (tid == 0) {
    for (int i = 0; i < STAGES + 2; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 2 * (V2_THREADS / 32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits + TMEM allocation visible pair-wide
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(lg * 32) << 16;
  constexpr uint32_t IDESC = idesc_tf32(2 * BM, L::NP);
  const uint32_t rawa0 = smem_u32(smem + L::RAWA_OFF) + (uint32_t)tid * 16;
  const uint32_t rawb0 = smem_u32(smem + L::RAWB_OFF) + (uint32_t)tid * 16;
  const uint32_t boff = core_off(b_n, b_chunk) + (uint32_t)(b_kp * 8);

  const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
  const float2 *Bb = reinterpret_cast<const float2 *>(g.B);
  float2 *Cb = reinterpret_cast<float2 *>(g.C);
  const uint32_t nk = (uint32_t)((g.K + KB - 1) / KB);
  const bool k_tail = (g.K % KB) != 0;
  const int64_t total_work = tiles * g.batch;   // 256 x BN tiles
  const bool a_vec = (g.opA == QF_OP_N) && (g.lda % 2 == 0) && (g.sA % 2 == 0);
  const bool b_vec = (g.opB == QF_OP_T) && (g.ldb % 2 == 0) && (g.sB % 2 == 0);
  const int64_t a_kstride = (g.opA == QF_OP_N) ? 1 : g.lda;
  const int64_t b_kstride = (g.opB == QF_OP_N) ? g.ldb : 1;

  if (warp == V2_THREADS / 32) {
    // ===== MMA issuer (leader CTA only)
    if (crank == 0 && lane == 0) {
      uint32_t qm = 0;
      for (int64_t work = pair; work < total_work; work += npairs) {
        for (uint32_t kb = 0; kb < nk; ++kb, ++qm) {
          const uint32_t s = qm & (STAGES - 1);
          mbar_wait(&full[s], (qm >> L::LOG_STAGES) & 1u);
          tc_fence_after();
          const uint32_t pos = kb & (CK - 1);
          const uint32_t chunk = kb >> L::LOG_CK;
          const uint32_t d = tmem + (chunk & 1u) * (uint32_t)L::P_COLS;
          const uint32_t st = smem_u32(smem + s * L::STAGE);
          // stage layout: [X_hi | Y_hi | X_lo | Y_lo]; X = window [Br|Bi], Y = [-Bi|Br]
          const uint64_t xh = smem_desc(st), yh = smem_desc(st + L::B_BLOCK);
          const uint64_t xl = smem_desc(st + 2 * L::B_BLOCK), yl = smem_desc(st + 3 * L::B_BLOCK);
          const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * 32u;
          const uint32_t acc0 = pos > 0 ? 1u : 0u;
          mma_ts2(d, a + 0, xh, IDESC, acc0);
          mma_ts2(d, a + 0, xl, IDESC, 1u);
          mma_ts2(d, a + 8, xh, IDESC, 1u);
          mma_ts2(d, a + 16, yh, IDESC, 1u);
          mma_ts2(d, a + 16, yl, IDESC, 1u);
          mma_ts2(d, a + 24, yh, IDESC, 1u);
          mma_commit2(&bars[s]);
          if (pos == CK - 1 || kb == nk - 1) mma_commit2(&pbar[chunk & 1u]);
        }
      }
    }
    __syncwarp();
  } else {
    // ===== converter warps (both CTAs)
    int64_t f_work = pair;
    uint32_t f_kb = 0;
    const float2 *fa = Ab, *fb = Bb;
    bool fa_ok = false, fb_ok = false;
    auto fetch_setup = [&]() {
      if (f_work >= total_work) return;
      const int64_t bidx = f_work / tiles;
      const int64_t tile = f_work - bidx * tiles;
      const int64_t am = (tile / tiles_n) * (2 * BM) + crank * BM + row_l;
      const int64_t bn = (tile % tiles_n) * BN + b_n;
      fa_ok = am < g.M;
      fb_ok = bn < g.N;
      const float2 *A = Ab + a_batch_off(g, bidx);
      const float2 *B = Bb + b_batch_off(g, bidx);
      fa = (g.opA == QF_OP_N) ? A + am * g.lda + 4 * half : A + (int64_t)(4 * half) * g.lda + am;
      fb = (g.opB == QF_OP_N) ? B + (int64_t)b_k * g.ldb + bn : B + bn * g.ldb + b_k;
      if (!fa_ok) fa = Ab;
      if (!fb_ok) fb = Bb;
    };
    auto fetch = [&](uint32_t slot) {
      if (f_work < total_work) {
        const uint32_t da = rawa0 + slot * L::RAWA_SLOT, db = rawb0 + slot * L::RAWB_SLOT;
        if (!(k_tail && f_kb == nk - 1)) {
          if (a_vec) {
            cp_async16(da, fa, fa_ok);
            cp_async16(da + V2_THREADS * 16, fa + 2, fa_ok);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              cp_async8(da + (k >> 1) * V2_THREADS * 16 + (k & 1) * 8, fa + k * a_kstride, fa_ok);
          }
          if (b_vec) {
            cp_async16(db, fb, fb_ok);
          } else {
            cp_async8(db, fb, fb_ok);
            cp_async8(db + 8, fb + b_kstride, fb_ok);
          }
        } else {
          const int64_t k0 = (int64_t)f_kb * KB;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool ok = fa_ok && k0 + 4 * half + k < g.K;
            cp_async8(da + (k >> 1) * V2_THREADS * 16 + (k & 1) * 8, ok ? fa + k * a_kstride : Ab, ok);
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = fb_ok && k0 + b_k + e < g.K;
            cp_async8(db + 8 * e, ok ? fb + e * b_kstride : Bb, ok);
          }
        }
        if (fa_ok) fa += KB * a_kstride;
        if (fb_ok) fb += KB * b_kstride;
        if (++f_kb == nk) {
          f_kb = 0;
          f_work += npairs;
          fetch_setup();
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };

    uint32_t q = 0;
    uint32_t pwaits[2] = {0, 0};
    const uint32_t full_leader = map_to_rank(smem_u32(full), 0);
    fetch_setup();
    for (int i = 0; i < RAW - 1; ++i) fetch((uint32_t)i);

    for (int64_t work = pair; work < total_work; work += npairs) {
      const int64_t bidx = work / tiles;
      const int64_t tile = work - bidx * tiles;
      const int64_t m0 = (tile / tiles_n) * (2 * BM) + crank * BM, n0 = (tile % tiles_n) * BN;
      float2 *C = Cb + bidx * g.sC;
      float racc[32], iacc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) racc[j] = iacc[j] = 0.f;
      auto promote = [&](int pb) {
        mbar_wait(&pbar[pb], pwaits[pb] & 1u);
        ++pwaits[pb];
        tc_fence_after();
        uint32_t v[32];
        const uint32_t base = tmem + lane_base + (uint32_t)(pb * L::P_COLS + 32 * half);
        tmem_ld32(base, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) racc[j] += __uint_as_float(v[j]);
        tmem_ld32(base + BN, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) iacc[j] += __uint_as_float(v[j]);
      };
      for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
        fetch((q + RAW - 1) & (RAW - 1));
        asm volatile("cp.async.wait_group %0;" ::"n"(RAW - 1) : "memory");
        const uint32_t s = q & (STAGES - 1);
        if (q >= STAGES) mbar_wait(&bars[s], ((q >> L::LOG_STAGES) + 1) & 1u);
        const uint32_t slot = q & (RAW - 1);
        const float4 a01 = *reinterpret_cast<const float4 *>(smem + L::RAWA_OFF +
                                                              slot * L::RAWA_SLOT + tid * 16);
        const float4 a23 = *reinterpret_cast<const float4 *>(
            smem + L::RAWA_OFF + slot * L::RAWA_SLOT + V2_THREADS * 16 + tid * 16);
        const float4 bb = *reinterpret_cast<const float4 *>(smem + L::RAWB_OFF +
                                                             slot * L::RAWB_SLOT + tid * 16);
        {
          uint32_t hr0, lr0, hi0, li0, hr1, lr1, hi1, li1;
          split_fast(bb.x, hr0, lr0);
          split_fast(bb.y, hi0, li0);
          split_fast(bb.z, hr1, lr1);
          split_fast(bb.w, hi1, li1);
          uint8_t *stage = smem + s * L::STAGE;
          // CTA0: X = Br, Y = -Bi      CTA1: X = Bi, Y = Br
          uint2 xh, yh, xl, yl;
          if (crank == 0) {
            xh = make_uint2(hr0, hr1);
            yh = make_uint2(hi0 ^ 0x80000000u, hi1 ^ 0x80000000u);
            xl = make_uint2(lr0, lr1);
            yl = make_uint2(li0 ^ 0x80000000u, li1 ^ 0x80000000u);
          } else {
            xh = make_uint2(hi0, hi1);
            yh = make_uint2(hr0, hr1);
            xl = make_uint2(li0, li1);
            yl = make_uint2(lr0, lr1);
          }
          *reinterpret_cast<uint2 *>(stage + boff) = xh;
          *reinterpret_cast<uint2 *>(stage + L::B_BLOCK + boff) = yh;
          *reinterpret_cast<uint2 *>(stage + 2 * L::B_BLOCK + boff) = xl;
          *reinterpret_cast<uint2 *>(stage + 3 * L::B_BLOCK + boff) = yl;
        }
        {
          uint32_t rh[4], rl[4], ih[4], il[4];
          split_fast(a01.x, rh[0], rl[0]);
          split_fast(a01.y, ih[0], il[0]);
          split_fast(a01.z, rh[1], rl[1]);
          split_fast(a01.w, ih[1], il[1]);
          split_fast(a23.x, rh[2], rl[2]);
          split_fast(a23.y, ih[2], il[2]);
          split_fast(a23.z, rh[3], rl[3]);
          split_fast(a23.w, ih[3], il[3]);
          const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * 32 + 4 * half);
          tmem_st4(acol + 0, rh[0], rh[1], rh[2], rh[3]);
          tmem_st4(acol + 8, rl[0], rl[1], rl[2], rl[3]);
          tmem_st4(acol + 16, ih[0], ih[1], ih[2], ih[3]);
          tmem_st4(acol + 24, il[0], il[1], il[2], il[3]);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          // plain (CTA-scope release) remote arrive, as CUTLASS's 2-SM pipelines
          // do: the data it publishes is read by the tensor core through the
          // async proxy (fenced above), not by the leader's threads
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(
                           full_leader + (uint32_t)(s * 8))
                       : "memory");
        const uint32_t pos = kb & (CK - 1);
        const uint32_t chunk = kb >> L::LOG_CK;
        if (pos == 0 && kb > 0) promote((int)((chunk - 1) & 1u));
      }
      if (nk > 0) promote((int)(((nk - 1) >> L::LOG_CK) & 1u));
      const int64_t row = m0 + row_l;
      if (row < g.M) {
        const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
        const bool use_beta = (br != 0.f || bi != 0.f);
        const int64_t c0 = n0 + 32 * half;
        float2 *crow = C + row * g.ldc + c0;
        const int64_t ncols = min((int64_t)32, g.N - c0);
        if (!use_beta && ncols == 32 && ar == 1.f && ai == 0.f && (((uintptr_t)crow) & 15) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            *reinterpret_cast<float4 *>(crow + j) =
                make_float4(racc[j], iacc[j], racc[j + 1], iacc[j + 1]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < ncols) {
              float2 o = make_float2(ar * racc[j] - ai * iacc[j], ar * iacc[j] + ai * racc[j]);
              if (use_beta) {
                const float2 c = crow[j];
                o.x += br * c.x - bi * c.y;
                o.y += br * c.y + bi * c.x;
              }
              crow[j] = o;
            }
          }
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // the leader's MMAs read this CTA's smem/TMEM until here
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
}

template <int STAGES, int CK, int RAW>
int launch_pair(const GemmArgs &g, cudaStream_t s) {
  using L = LayoutP2<STAGES, CK, RAW>;
  auto kern = cgemm_tc3pair_kernel<STAGES, CK, RAW>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3pair: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  const int64_t tiles_n = (g.N + L::BN - 1) / L::BN, tiles_m = (g.M + 2 * BM - 1) / (2 * BM);
  const int64_t tiles = tiles_n * tiles_m;
  const int64_t pairs = std::min<int64_t>(tiles * g.batch, (int64_t)sm_count() / 2);
  kern<<<(unsigned)(2 * pairs), V2_THREADS + 32, L::SMEM, s>>>(g, tiles_n, tiles);
  return check_launch("cgemm_tc3pair");
}

}  // namespace tc

// variant: 0 = auto (v3: promoted + cp.async stream), 1 = v1 SS, 2 = v1 TS
// (v1 accumulates the whole K in TMEM: its error grows ~1.4e-8 * K),
// 3 = v2 (promoted, register prefetch), 4 = v3 stream (block barrier per
// k-block); default = warp-specialised stream
static int g_tc3_variant = 0;

bool tc3_gather_ok(const GemmArgs &g) { return g.K <= 4096; }

// TMA-fed short-K runs: RAW k-blocks of A (8 KiB each) in flight per CTA.
// 8 deep for plain operands and strided views alike: the config-2 view GEMMs
// 1024 x (4096 x 64 x 64) run 0.69 ms 8 deep vs 0.80-0.85 ms 4 deep (6.26 TB/s,
// 0.97 of the measured HBM copy rate; an earlier 4-deep preference measured
// before the transposed-store/view-order changes no longer holds).  Variants
// 21/22 pin 4/8 for A/B runs.
static int launch_short_tma(const GemmArgs &g, cudaStream_t s) {
  if (g_tc3_variant == 21) return tc::launch_short<8, 4, 8, 4, 64, 0, 1, true>(g, s);
  if (g_tc3_variant == 22) return tc::launch_short<8, 8, 8, 4, 64, 0, 1, true>(g, s);
  // narrow outputs (a transposed view with N <= 32): 32-column tiles halve
  // the padded MMA work, which otherwise paces the HBM-bound tile
  if (g_tc3_variant == 24 && g.N <= 32) return tc::launch_short<8, 8, 16, 4, 32, 0, 1, true>(g, s);
  if (g_tc3_variant == 25) return tc::launch_short<8, 8, 16, 4, 64, 0, 1, true>(g, s);
  if (g.N <= 32 && g_tc3_variant != 23) return tc::launch_short<8, 8, 8, 4, 32, 0, 1, true>(g, s);
  return tc::launch_short<8, 8, 8, 4, 64, 0, 1, true>(g, s);
}

// short-K kernel flavour: output-bound shapes (K <= 56) keep the epilogue on
// the converter warps (more store parallelism); longer K hands it to 4
// dedicated epilogue warps so conversion, MMA and stores overlap.
// Variants 10/11/12 pin 8 warps / 16 warps / 16 + 4 epilogue warps.
static int launch_short_auto(const GemmArgs &g, cudaStream_t s) {
  if (g_tc3_variant == 10) return tc::launch_short<8, 4, 8, 0>(g, s);
  if (g_tc3_variant == 11) return tc::launch_short<8, 4, 16, 0>(g, s);
  if (g_tc3_variant == 12) return tc::launch_short<8, 8, 16, 4>(g, s);
  // TMA-fed runs (one producer warp) when the operands are plain strided
  // views and K >= 32 (1024 x 4096 x {16,32,64} x {32,64}: 0.57-0.68 ms vs
  // 0.74-0.96 ms for the converter-fetch kernels, scripts/smallk_bench.py)
  if (g.K >= 32 && g.K <= 128 && tc::tma_ok(g)) return launch_short_tma(g, s);
  if (g.N <= 8) return tc::launch_short<8, 8, 16, 4, 8>(g, s);
  if (g.N <= 16) return tc::launch_short<8, 8, 16, 4, 16>(g, s);
  if (g.N <= 32) return tc::launch_short<8, 8, 16, 4, 32>(g, s);
  // K in (128, 256]: the promoted long-K kernel (TMEM master, 8-k-block
  // chunks) beats one long TMEM accumulation (scripts/c5_shapes.py)
  if (g.K > 128)
    return tc::tma_ok(g) ? tc::launch_short<4, 8, 8, 4, 64, 8, 1, true>(g, s)
                         : tc::launch_short<4, 8, 8, 4, 64, 8>(g, s);
  if (g.K <= 8) return tc::launch_short<8, 4, 8, 0>(g, s);
  if (g.K <= 56) return g.N > 64 ? tc::launch_short<8, 4, 8, 0>(g, s) : tc::launch_short<8, 4, 16, 0>(g, s);
  return tc::launch_short<8, 8, 16, 4>(g, s);
}

bool tc3_eligible(const GemmArgs &g) {
  // a 128 x 64 tile reasonably full and enough tiles for the machine; short
  // K is fine (the short-K kernel streams A once and keeps B resident)
  // narrow N (12..31) only through the short-K kernel's narrow tiles; N < 12
  // stays on the CUDA-core row-block kernel (measured faster or equal)
  if (g.M < 64 || g.K < 1) return false;
  // M in [64, 128) half-fills a tile but still beats the 64x64 SIMT tiles
  // (1024 x 64^3: 0.049 vs 0.069 ms)
  if (g.N >= 32) return g.M * g.N * g.batch >= 128 * 64 * 148;
  if (g.M < 128) return false;
  return g.N >= 12 && g.K <= 256 && g.M * g.batch >= 128 * 148;
}

int gemm_tc3(const GemmArgs &g, cudaStream_t s) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return QF_OK;
  QF_REQUIRE(g.K > 0, "tc3: K must be positive (use FFMA for K == 0)");
  if (g.c_nblk && (!g.v_kin || g.K > 128 || g.c_trans)) {
    set_error("tc3: column-blocked C only on the short-K view kernel");
    return QF_ERR_UNSUPPORTED;
  }
  if (g.c_trans && !g.v_t) {
    set_error("tc3: transposed C only on a transposed A view");
    return QF_ERR_UNSUPPORTED;
  }
  if (g.v_kin) {  // A views are read by the TMA-fed short-K kernel only
    // (narrow N runs 32-column tiles that compute zeros beyond N; the
    // HBM-bound shapes do not mind)
    // long K (N-views): the promoted long-K kernel with its TMA producer
    // (plain row-major epilogue only)
    const bool long_k = g.K > 128 && !g.v_t && !g.c_trans && g.N > 32;
    if (!(g.K >= 32 && (g.K <= 128 || long_k) && tc::tma_ok(g))) {
      set_error("tc3: A view (kin %lld, rows %lld x %lld) not TMA-describable for K=%lld N=%lld",
                (long long)g.v_kin, (long long)g.v_ra, (long long)g.v_rb, (long long)g.K,
                (long long)g.N);
      return QF_ERR_UNSUPPORTED;
    }
    if (g.K > 128) return tc::launch_short<4, 8, 8, 4, 64, 4, 1, true>(g, s);
    return launch_short_tma(g, s);
  }
  const bool small_n = g.N <= 64;
  if (g.a_roff) {  // gathered A: only the warp-specialised kernel fetches through tables
    QF_REQUIRE(tc3_gather_ok(g), "tc3: gathered A needs K <= 4096");
    if (g_tc3_variant == 13) return tc::launch_short<4, 8, 8, 4, 64, 4>(g, s);
    if (g_tc3_variant == 14) return tc::launch_short<4, 8, 8, 4, 64, 8>(g, s);
    if (g_tc3_variant == 17 && g.K <= 256) return tc::launch_short<8, 4, 8, 4, 64, 0, 4>(g, s);
    if (g_tc3_variant == 18) return tc::launch_short<4, 8, 8, 4, 64, 4, 4>(g, s);
  if (g_tc3_variant == 19 && tc::tma_ok(g)) return tc::launch_short<4, 8, 8, 4, 64, 4, 1, true>(g, s);
  if (g_tc3_variant == 20 && tc::tma_ok(g) && g.K <= 256)
    return tc::launch_short<8, 4, 8, 4, 64, 0, 1, true>(g, s);

    if (g.K <= 256)
      return g_tc3_variant == 9 ? tc::launch_ws<8, 4, 8, true>(g, s) : launch_short_auto(g, s);
    if (g_tc3_variant == 15) return tc::launch_ws<8, 4, 8, false>(g, s);
    return tc::launch_short<4, 8, 8, 4, 64, 4>(g, s);
  }
  if (g_tc3_variant == 9)
    return g.K <= 256 ? tc::launch_ws<8, 4, 8, true>(g, s) : tc::launch_ws<8, 4, 8, false>(g, s);
  if (g_tc3_variant == 13) return tc::launch_short<4, 8, 8, 4, 64, 4>(g, s);
  if (g_tc3_variant == 14) return tc::launch_short<4, 8, 8, 4, 64, 8>(g, s);
  if (g_tc3_variant == 16) return tc::launch_short<4, 8, 16, 4, 64, 4>(g, s);
  if (g_tc3_variant == 17 && g.K <= 256) return tc::launch_short<8, 4, 8, 4, 64, 0, 4>(g, s);
  if (g_tc3_variant == 18) return tc::launch_short<4, 8, 8, 4, 64, 4, 4>(g, s);
  if (g_tc3_variant == 19 && tc::tma_ok(g)) return tc::launch_short<4, 8, 8, 4, 64, 4, 1, true>(g, s);
  if (g_tc3_variant == 20 && tc::tma_ok(g) && g.K <= 256)
    return tc::launch_short<8, 4, 8, 4, 64, 0, 1, true>(g, s);

  if (g_tc3_variant == 1)
    return small_n ? tc::launch<64, 6, false>(g, s) : tc::launch<128, 4, false>(g, s);
  if (g_tc3_variant == 2)
    return small_n ? tc::launch<64, 6, true>(g, s) : tc::launch<128, 4, true>(g, s);
  if (g_tc3_variant == 3) return tc::launch_v2<6, 4>(g, s);
  if (g_tc3_variant == 4) return tc::launch_v3<4, 4, 8>(g, s);
  if (g_tc3_variant == 6) return tc::launch_pair<8, 4, 8>(g, s);
  if (g_tc3_variant == 7)
    return g.K <= 256 ? tc::launch_ws<8, 4, 8, true, 2>(g, s) : tc::launch_ws<8, 4, 8, false, 2>(g, s);
  if (g_tc3_variant == 8)
    return g.K <= 256 ? tc::launch_ws<8, 4, 8, true, 4>(g, s) : tc::launch_ws<8, 4, 8, false, 4>(g, s);
  if (g_tc3_variant == 5)
    return g.K <= 256 ? tc::launch_reg<8, 4, 4, true>(g, s) : tc::launch_reg<8, 4, 4, false>(g, s);
  // short K (<= 256): no promotion needed (error <= 3.6e-6); tile-level
  // double-buffered TMEM accumulators with a deferred epilogue
  if (g.K <= 256) return launch_short_auto(g, s);
  if (g_tc3_variant == 15) return tc::launch_ws<8, 4, 8, false>(g, s);
  // long K: a TMA producer warp, 8 converter warps, 4 promotion warps with a
  // TMEM master accumulator (cp.async fetch by the converters when TMA
  // cannot describe the operands)
  if (g_tc3_variant == 26 && tc::tma_ok(g)) return tc::launch_short<4, 8, 8, 4, 64, 16, 1, true>(g, s);
  if (g_tc3_variant == 27 && tc::tma_ok(g)) return tc::launch_short<4, 8, 8, 4, 64, 32, 1, true>(g, s);
  if (g_tc3_variant != 13 && tc::tma_ok(g)) return tc::launch_short<4, 8, 8, 4, 64, 4, 1, true>(g, s);
  return tc::launch_short<4, 8, 8, 4, 64, 4>(g, s);
}

}  // namespace qf

extern "C" int qf_tc3_set_variant(int v) {
  int prev = qf::g_tc3_variant;
  qf::g_tc3_variant = v;
  return prev;
}

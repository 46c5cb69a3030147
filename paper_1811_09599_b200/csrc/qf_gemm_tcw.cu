// K2c -- the WIDE long-K complex GEMM on tcgen05 (sm_100a): 128 x 128 complex
// tiles, Gauss (3-multiplication) form, 3xTF32 split, fp32 master accumulator
// in registers.
//
// Replaces the OpenBLAS cgemm behind `@` at rq/tensor_core.py:417 for the
// big compute-bound contractions (configs 4 and 5: K >= 256, N >= 128).
//
// Why a second long-K flavour.  The 128 x 64 Gauss kernel (qf_gemm_tc.cu,
// "cgemm_tc3g") is bound by the 1 kW power cap and by a per-stage handshake
// floor, not by the tensor pipe (profiles/r2_gemm_notes.md): per 8 complex k
// it converts a 128 x 8 A block and a 64 x 8 B block, stores 6 + 6 planes and
// pulls 12 KB from L2 for 288 tensor cycles.  A 128-column tile reuses every
// converted A plane for twice the columns: per flop the A conversions, the
// A tcgen05.st traffic and the A bytes from L2 halve, the nine MMAs per stage
// are N = 128 (64 tensor cycles each, 576 per stage, above the handshake
// floor), and half as many stages are handed over.
//
// The price is tensor memory: [T1 | T2 | T3] for 128 columns is 384 of the
// 512 TMEM columns, so the fp32 master [Re | Im] cannot live there as it
// does in the 64-column kernel.  It lives in REGISTERS of 8 promotion warps
// (warp = TMEM lane quadrant x column half: 64 columns x {Re, Im} = 128
// registers per thread), which add the tensor pipe's partial sums every CK
// k-blocks with round-to-nearest CUDA-core adds (flat error in K, as in the
// 64-column kernel) and write the tile out of registers at its end.  The
// register file is re-partitioned with setmaxnreg.  The pool is what the CTA
// got at launch, and ptxas sizes that for whole warpgroups: 512 threads
// launch with 128 registers each (all 64 K), then warps 0-3 drop to 104,
// warps 4-7 to 72, and the promotion warps grow to 168.
//
// Warp roles (16 warps): 0-3 A converters (thread = one A row, all 8 k of a
// stage; also B columns 0-63), 4 TMA producer, 5 MMA issuer, 6-7 B converters
// (columns 64-127), 8-15 promotion/epilogue.  Per stage (8 complex k): TMA
// boxes of raw A (128 x 8) and raw B (128 x 8) land in an 8-deep ring;
// converters split Ar, Ai, Ar+Ai into hi/lo TF32 planes written straight into
// TMEM (6 x 8 columns) and Br, Bi, Br+Bi into hi/lo K-major core-matrix planes
// in shared memory; one elected lane issues T_j += A_j(hi) B_j(hi) + A_j(hi)
// B_j(lo) + A_j(lo) B_j(hi), j = 1..3.  Re = T1 - T2, Im = T3 - T1 - T2 at
// promotion.
//
// CTA pairs (PAIR, the default when M fills 256-row tiles): a cluster of two
// CTAs owns a 256 x 128 tile; each converts its own 128 A rows and only 64 B
// columns, the leader issues cta_group::2 MMAs with M = 256 and multicasts the
// completions.  Lockstep: the producers of all CTAs announce their progress
// every EPOCH stages in a global counter array and wait for the slowest, so
// CTAs sharing a panel read it from DRAM once (profiles/r2c_gemm_wide.md).
#include <algorithm>
#include <cstdlib>

#include "qf_tc_ptx.cuh"

namespace qf {
namespace tcw {

using namespace tc;

constexpr int BN = 128;          // complex output columns per tile
constexpr int STAGES = 2;        // converted stages (A planes in TMEM + B' planes in smem)
constexpr int RAW = 8;           // raw TMA ring depth (k-blocks in flight)
// converting warps: 4 (A rows + B columns 0-63) + 2 (B columns 64-127); in a CTA
// pair every CTA converts only its 64 columns of B, on the 4 A warps
constexpr int NPROMO = 8;        // promotion / epilogue warps
constexpr uint32_t EPOCH = 16;   // stages per lockstep epoch of the TMA producers
constexpr int THREADS_W = 512;   // warps 0-3 | 4 TMA, 5 MMA, 6-7 | 8-15
constexpr int REGS_A = 104;      // setmaxnreg targets (multiples of 8; 128 at launch)
constexpr int REGS_MISC = 72;
constexpr int REGS_PROMO = 168;
static_assert(128 * REGS_A + 128 * REGS_MISC + 256 * REGS_PROMO <= 65536, "register file");

template <bool PAIR>
struct Lw {
  static constexpr int BNL = PAIR ? BN / 2 : BN;     // B columns converted / held by this CTA
  static constexpr int NCONV = PAIR ? 4 : 6;         // converting warps per CTA
  static constexpr int B_BLOCK = BNL * 32;           // one plane block: BNL n x 8 tf32, K-major
  static constexpr int B_PLANE = 3 * B_BLOCK;        // [Br | Bi | Br+Bi]
  static constexpr int STAGE = 2 * B_PLANE;          // hi plane, lo plane
  static constexpr int RAWA_SLOT = BM * 64;          // 128 rows x 8 complex
  static constexpr int RAWB_SLOT = BNL * 64;
  static constexpr int RAWA_OFF = STAGES * STAGE;
  static constexpr int RAWB_OFF = RAWA_OFF + RAW * RAWA_SLOT;
  static constexpr int EPI_PITCH = 16 * 8 + 16;      // 16 complex columns per staging pass
  static constexpr int EPI_OFF = RAWB_OFF + RAW * RAWB_SLOT;
  static constexpr int BAR_OFF = EPI_OFF + NPROMO * 32 * EPI_PITCH;
  static constexpr int SMEM = BAR_OFF + 1024;
  static constexpr int A_COL0 = 3 * BN;              // after [T1 | T2 | T3]
  static constexpr int A_STAGE_COLS = 48;            // Ar, Ai, Ar+Ai x (hi, lo) x 8 k
  static constexpr int TMEM_COLS = 512;
  static_assert(A_COL0 + STAGES * A_STAGE_COLS <= TMEM_COLS, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(RAWA_OFF % 1024 == 0 && RAWA_SLOT % 1024 == 0 && RAWB_SLOT % 1024 == 0,
                "TMA boxes are 1 KB aligned");
};

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}

// CTA pair (cta_group::2): a cluster of two CTAs computes a 256 x 128 tile with
// M = 256 MMAs issued by the leader (rank 0).  Each CTA keeps its 128 A rows in
// its own TMEM and its 64 columns of the B' planes in its own shared memory,
// which halves every SM's B conversion and B bytes from L2.  Converters and
// promotion warps of both CTAs arrive on the leader's barriers; MMA completions
// are multicast to both CTAs.
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
// arrive on a barrier of the pair's leader (a cluster address; rank 0 maps to itself)
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
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

template <int N>
__device__ __forceinline__ void reg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

// tile w of the launch -> (entry, M tile, N tile): strided over the grid in
// groups of GM M tiles, so the ~148 tiles in flight cover a GM x (148 / GM)
// block and every A / B panel is shared through L2 by its row / column
struct Cur {
  uint32_t w, mt, nt, bidx;
};
__device__ __forceinline__ void cur_set(Cur &c, uint32_t w, uint32_t tiles_m, uint32_t tiles_n,
                                        uint32_t GM) {
  c.w = w;
  const uint32_t tiles = tiles_m * tiles_n;
  c.bidx = w / tiles;
  const uint32_t t = w - c.bidx * tiles;
  const uint32_t group = t / (GM * tiles_n), first_m = group * GM;
  const uint32_t gsize = min(tiles_m - first_m, GM);
  const uint32_t r = t - group * GM * tiles_n;
  c.mt = first_m + r % gsize;
  c.nt = r / gsize;
}

// Converter loop of one role (instantiated once per role so each inherits the
// register budget of its own setmaxnreg).  A_ROLE: warps 0-3, thread = TMEM
// lane = A row, all 8 k of the stage, plus B columns 0-63; otherwise warps 6-7,
// B columns 64-127.  Raw boxes -> registers (slot released at once),
// everything split into TF32 hi/lo planes BEFORE the wait for the stage, so
// only stores sit between the tensor pipe freeing stage s and full[s].  B
// work is cut into 256 "virtual threads" per column half: virtual thread tv
// converts one 16-byte k pair of one column -- a half-warp covers 16 columns,
// lanes 0-7 at one k pair, lanes 8-15 at the other (swapped in the next
// half-warp), so raw reads hit disjoint bank halves and the 8-byte B' stores
// of 16 lanes fill one core-matrix row block.  A converters run tv = tid,
// tid + 128 of half 0; B converters tv = u, u + 64, u + 128, u + 192 of half 1.
template <bool A_ROLE, bool PAIR>
__device__ __forceinline__ void convert_loop(const GemmArgs &g, uint8_t *smem, uint64_t *bars,
                                             uint32_t full_leader, uint64_t *rawfull,
                                             uint64_t *rawfree, uint32_t tmem, uint32_t w0,
                                             uint32_t wstep, uint32_t total, uint32_t nk) {
  using L = Lw<PAIR>;
  constexpr int BNL = L::BNL;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int u = A_ROLE ? tid : tid - 192;        // index among this role's threads
  constexpr int NB = A_ROLE ? 2 : 4;              // B k pairs per thread
  constexpr int TV_STEP = A_ROLE ? 128 : 64;
  constexpr int HSEL = A_ROLE ? 0 : 1;
  const int row_l = tid & 127;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t boff[NB];
  int b_src[NB];                                   // byte offset of the k pair inside a raw B box
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int tv = u + i * TV_STEP;
    const int t = tv & 127, hw = t >> 4, l = t & 15;
    const int b_kp = ((l >> 3) & 1) ^ (hw & 1), b_chunk = tv >> 7;
    const int n = 16 * (hw >> 1) + (l & 7) + 8 * ((l >> 3) & 1) + 64 * HSEL;
    const int b_k = b_chunk * 4 + b_kp * 2;
    boff[i] = core_off(n, b_chunk) + (uint32_t)(b_kp * 8);
    // opB N: [8 k][128 n] dense (two 8-byte reads, rows b_k and b_k + 1);
    // opB T: [128 n][64 B] with the 64-byte swizzle (one 16-byte read)
    b_src[i] = g.opB == QF_OP_N ? b_k * (BNL * 8) + n * 8
                                : n * 64 + (((b_k >> 1) ^ ((n >> 1) & 3)) << 4);
  }
  uint32_t q = 0;
  for (uint32_t w = w0; w < total; w += wstep) {
    for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
      const uint32_t slot = q & (RAW - 1), s = q & (STAGES - 1);
      mbar_wait(&rawfull[slot], (q / RAW) & 1u);
      const uint8_t *rA = smem + L::RAWA_OFF + slot * L::RAWA_SLOT;
      const uint8_t *rB = smem + L::RAWB_OFF + slot * L::RAWB_SLOT;
      float4 av[4], bv[NB];
      if constexpr (A_ROLE) {
        if (g.opA == QF_OP_N) {
          // 64-byte swizzle: the 16-byte chunk c of row r sits at chunk c ^ ((r >> 1) & 3)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            av[c] = *reinterpret_cast<const float4 *>(rA + row_l * 64 + ((c ^ ((row_l >> 1) & 3)) << 4));
        } else {  // [8 k][128 rows] dense
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float2 x0 = *reinterpret_cast<const float2 *>(rA + (2 * c) * 1024 + row_l * 8);
            const float2 x1 = *reinterpret_cast<const float2 *>(rA + (2 * c + 1) * 1024 + row_l * 8);
            av[c] = make_float4(x0.x, x0.y, x1.x, x1.y);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        if (g.opB == QF_OP_N) {
          const float2 y0 = *reinterpret_cast<const float2 *>(rB + b_src[i]);
          const float2 y1 = *reinterpret_cast<const float2 *>(rB + b_src[i] + BNL * 8);
          bv[i] = make_float4(y0.x, y0.y, y1.x, y1.y);
        } else {
          bv[i] = *reinterpret_cast<const float4 *>(rB + b_src[i]);
        }
      }
      __syncwarp();
      if (lane == 0)  // release semantics order the reads above before the refill
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rawfree[slot]))
                     : "memory");
      // B' planes [Br | Bi | Br + Bi]: hi in bp[i][0..5], lo in bp[i][6..11]
      uint32_t bp[NB][12];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        split_fast(bv[i].x, bp[i][0], bp[i][6]);
        split_fast(bv[i].y, bp[i][2], bp[i][8]);
        split_fast(bv[i].x + bv[i].y, bp[i][4], bp[i][10]);
        split_fast(bv[i].z, bp[i][1], bp[i][7]);
        split_fast(bv[i].w, bp[i][3], bp[i][9]);
        split_fast(bv[i].z + bv[i].w, bp[i][5], bp[i][11]);
      }
      uint32_t rh[8], rl[8], ih[8], il[8], sh[8], sl[8];
      if constexpr (A_ROLE) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          split_fast(av[c].x, rh[2 * c], rl[2 * c]);
          split_fast(av[c].y, ih[2 * c], il[2 * c]);
          split_fast(av[c].x + av[c].y, sh[2 * c], sl[2 * c]);
          split_fast(av[c].z, rh[2 * c + 1], rl[2 * c + 1]);
          split_fast(av[c].w, ih[2 * c + 1], il[2 * c + 1]);
          split_fast(av[c].z + av[c].w, sh[2 * c + 1], sl[2 * c + 1]);
        }
      }
      if (q >= STAGES) mbar_wait(&bars[s], ((q / STAGES) + 1) & 1u);
      uint8_t *ph = smem + s * L::STAGE, *pl = ph + L::B_PLANE;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          *reinterpret_cast<uint2 *>(ph + j * L::B_BLOCK + boff[i]) =
              make_uint2(bp[i][2 * j], bp[i][2 * j + 1]);
          *reinterpret_cast<uint2 *>(pl + j * L::B_BLOCK + boff[i]) =
              make_uint2(bp[i][6 + 2 * j], bp[i][6 + 2 * j + 1]);
        }
      }
      fence_async_smem();
      if constexpr (A_ROLE) {
        const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * L::A_STAGE_COLS);
        tmem_st8(acol + 0, rh);
        tmem_st8(acol + 8, rl);
        tmem_st8(acol + 16, ih);
        tmem_st8(acol + 24, il);
        tmem_st8(acol + 32, sh);
        tmem_st8(acol + 40, sl);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      // (pair: a plain remote arrive, as CUTLASS's 2-SM pipelines do -- what it
      // publishes is read by the tensor core through the async proxy, fenced above)
      if (lane == 0) arrive_cluster(full_leader + s * 8u);
    }
  }
}

template <int CK, bool PAIR, int DP>
__global__ void __launch_bounds__(THREADS_W, 1)
    cgemm_tc3w_kernel(const __grid_constant__ GemmArgs g, uint32_t tiles_m, uint32_t tiles_n,
                      uint32_t total, const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, uint32_t *epoch_sync,
                      uint32_t max_epochs, uint32_t gm) {
  using L = Lw<PAIR>;
  constexpr int NCONV = L::NCONV;
  constexpr uint32_t NCTA = PAIR ? 2 : 1;
  static_assert((CK & (CK - 1)) == 0 && CK >= 8, "promotion chunk: a power of two");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);  // [STAGES] stage free
  uint64_t *full = bars + STAGES;                                    // [STAGES] stage converted
  uint64_t *pbar = full + STAGES;                                    // chunk accumulated
  uint64_t *accfree = pbar + 1;                                      // partial drained
  uint64_t *rawfull = accfree + 1;                                   // [RAW] boxes landed
  uint64_t *rawfree = rawfull + RAW;                                 // [RAW] converters read them
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rawfree + RAW);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&bars[i], 1);
      mbar_init(&full[i], NCONV * NCTA);      // (leader's: both CTAs' converters)
    }
    mbar_init(pbar, 1);
    mbar_init(accfree, NPROMO * NCTA);        // (leader's: both CTAs' promotion warps)
    for (int i = 0; i < RAW; ++i) {
      mbar_init(&rawfull[i], 1);
      mbar_init(&rawfree[i], NCONV);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(L::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(L::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();   // barrier inits + TMEM allocation visible pair-wide
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // pair: w counts 256 x 128 pair tiles, both CTAs of a cluster walk the same
  // sequence and CTA `crank` owns rows [128 crank, 128 crank + 128) of each
  const uint32_t crank = PAIR ? cluster_rank() : 0u;
  const uint32_t w0 = PAIR ? blockIdx.x >> 1 : blockIdx.x, wstep = PAIR ? gridDim.x >> 1 : gridDim.x;
  const uint32_t full_leader = PAIR ? map_to_rank(smem_u32(full), 0) : smem_u32(full);
  const uint32_t accfree_leader = PAIR ? map_to_rank(smem_u32(accfree), 0) : smem_u32(accfree);
  const uint32_t nk = ((uint32_t)g.K + KB - 1) / KB;
  const uint32_t nchunks = (nk + CK - 1) / CK;

  if (warp >= 8) {
    // ===== promotion / epilogue warps: quadrant lg of the TMEM lanes, column
    // half `half`; the fp32 master of their 32 x 64 block stays in registers
    reg_inc<REGS_PROMO>();
    const int pw = warp - 8, lg = pw & 3, half = pw >> 2;
    const uint32_t pbase = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(half * 64);
    float2 *Cb = reinterpret_cast<float2 *>(g.C);
    const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
    const bool use_beta = (br != 0.f || bi != 0.f);
    uint8_t *stg = smem + L::EPI_OFF + pw * 32 * L::EPI_PITCH;
    float mr[64], mi[64];
    uint32_t chunkc = 0;
    Cur ec;
    for (uint32_t w = w0; w < total; w += wstep) {
      cur_set(ec, w, tiles_m, tiles_n, gm);
#pragma unroll
      for (int j = 0; j < 64; ++j) mr[j] = mi[j] = 0.f;
      for (uint32_t c = 0; c < nchunks; ++c, ++chunkc) {
        mbar_wait_sleep(pbar, chunkc & 1u, 200u);   // a chunk is >= 10 us of MMAs
        tc_fence_after();
#pragma unroll
        for (int piece = 0; piece < 64 / DP; ++piece) {   // DP columns of T1, T2, T3 per round trip
          uint32_t t1[DP], t2[DP], t3[DP];
          if constexpr (DP == 8) {
            tmem_ld8(pbase + piece * DP, t1);
            tmem_ld8(pbase + BN + piece * DP, t2);
            tmem_ld8(pbase + 2 * BN + piece * DP, t3);
          } else {
            tmem_ld4(pbase + piece * DP, t1);
            tmem_ld4(pbase + BN + piece * DP, t2);
            tmem_ld4(pbase + 2 * BN + piece * DP, t3);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (piece == 64 / DP - 1) {   // the partial is in registers: hand it back to the tensor pipe
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_cluster(accfree_leader);
          }
#pragma unroll
          for (int j = 0; j < DP; ++j) {
            const float x1 = __uint_as_float(t1[j]), x2 = __uint_as_float(t2[j]);
            const float re = x1 - x2, im = __uint_as_float(t3[j]) - x1 - x2;
            mr[piece * DP + j] += re;
            mi[piece * DP + j] += im;
          }
        }
      }
      // ---- epilogue out of the master registers, 16 columns per pass
      const int64_t m0 = (int64_t)(ec.mt * NCTA + crank) * BM + lg * 32;
      const int64_t n0 = (int64_t)ec.nt * BN + half * 64;
      float2 *cw = Cb + (int64_t)ec.bidx * g.sC + m0 * g.ldc + n0;
      const int64_t ntile = g.N - n0;   // columns left from n0 (may be <= 0 on a ragged edge)
      const bool vec = g.ldc % 2 == 0 && (((uintptr_t)cw) & 15) == 0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t vr[16], vi[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          vr[j] = __float_as_uint(mr[ch * 16 + j]);
          vi[j] = __float_as_uint(mi[ch * 16 + j]);
        }
        stage_store_chunk<16, L::EPI_PITCH>(stg, vr, vi, cw + ch * 16, g.ldc, g.M - m0,
                                            min(ntile, (int64_t)64) - ch * 16, ar, ai, br, bi,
                                            use_beta, vec, lane);
      }
    }
  } else if (warp >= 4) {
    reg_dec<REGS_MISC>();   // warps 4-7 form one warpgroup: one setmaxnreg for all its roles
    if (warp >= 6) {
      if constexpr (!PAIR)
        convert_loop<false, false>(g, smem, bars, full_leader, rawfull, rawfree, tmem, w0, wstep,
                                   total, nk);
    } else if (warp == 5) {
      if (crank == 0) {
      // ===== MMA issuer: the whole warp walks the stage sequence, one elected
      // lane issues.  B' descriptors = stage-0 descriptor + constant (the
      // address field is the low 14 bits, in 16-byte units).
      const uint64_t desc0 = smem_desc(smem_u32(smem));
      constexpr uint32_t ST16 = (uint32_t)L::STAGE >> 4, BP16 = (uint32_t)L::B_PLANE >> 4,
                         BB16 = (uint32_t)L::B_BLOCK >> 4;
      constexpr uint32_t IDESC = idesc_tf32(PAIR ? 2 * BM : BM, BN);
      uint32_t q = 0, chunkc = 0;
      for (uint32_t w = w0; w < total; w += wstep) {
        for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
          const uint32_t s = q & (STAGES - 1);
          mbar_wait(&full[s], (q / STAGES) & 1u);
          tc_fence_after();
          const uint32_t pos = kb & (CK - 1);
          if (pos == 0 && chunkc >= 1) {  // the promotion warps have read the previous chunk
            mbar_wait(accfree, (chunkc - 1) & 1u);
            tc_fence_after();
          }
          const bool chunk_end = pos == CK - 1 || kb == nk - 1;
          const uint64_t bh = desc0 + (uint64_t)(s * ST16), bl = bh + BP16;
          const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * (uint32_t)L::A_STAGE_COLS;
          const uint32_t acc0 = pos > 0 ? 1u : 0u;
          if (elect_one()) {
            // A planes: Ar hi/lo (+0, +8), Ai hi/lo (+16, +24), Ar+Ai hi/lo (+32, +40);
            // B' blocks 0/1/2 = Br, Bi, Br+Bi
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const uint32_t dj = tmem + (uint32_t)(j * BN);
              if constexpr (PAIR) {
                mma_ts2(dj, a + 16 * j, bh + j * BB16, IDESC, acc0);
                mma_ts2(dj, a + 16 * j, bl + j * BB16, IDESC, 1u);
                mma_ts2(dj, a + 16 * j + 8, bh + j * BB16, IDESC, 1u);
              } else {
                mma_ts(dj, a + 16 * j, bh + j * BB16, IDESC, acc0);
                mma_ts(dj, a + 16 * j, bl + j * BB16, IDESC, 1u);
                mma_ts(dj, a + 16 * j + 8, bh + j * BB16, IDESC, 1u);
              }
            }
            if constexpr (PAIR) {
              mma_commit2(&bars[s]);
              if (chunk_end) mma_commit2(pbar);
            } else {
              mma_commit(&bars[s]);
              if (chunk_end) mma_commit(pbar);
            }
          }
          if (chunk_end) ++chunkc;
          __syncwarp();
        }
      }
      }   // leader
    } else {
      // ===== TMA producer (one elected lane): per k-block one box of A and one
      // of B into the raw ring; the slot's mbarrier completes on their bytes
      if (elect_one()) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        const uint32_t rawa = smem_u32(smem + L::RAWA_OFF), rawb = smem_u32(smem + L::RAWB_OFF);
        Cur pc;
        uint32_t f = 0;
        bool sync_ok = true;
        for (uint32_t w = w0; w < total; w += wstep) {
          cur_set(pc, w, tiles_m, tiles_n, gm);
          const int32_t m0 = (int32_t)((pc.mt * NCTA + crank) * BM), b = (int32_t)pc.bidx;
          const int32_t n0 = (int32_t)(pc.nt * BN + crank * L::BNL);   // pair: this CTA's B columns
          const int32_t bslice = g.b_boff ? (int32_t)(__ldg(g.b_boff + pc.bidx) / (g.K * g.N)) : b;
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
            if (epoch_sync && (f & (EPOCH - 1)) == 0) {
              // soft lockstep: every EPOCH stages announce this CTA's progress
              // and wait until every CTA has reached the previous epoch, so the
              // CTAs that share an A or a B panel stay within ~2 EPOCH stages of
              // each other and the panel is read from DRAM once, from L2 after
              // (without it the CTAs drift apart over a K = 32768 sweep: ncu
              // counted 6.1 TB of DRAM reads per config-4 path, 7x the panels)
              const uint32_t e = f / EPOCH;
              asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(epoch_sync + e) : "memory");
              if (e >= 1 && sync_ok) {
                // bounded wait (~20 ms): if the CTAs of this grid are not all
                // resident (SMs held by another context or kernel) the
                // lockstep is dropped instead of risking a stall
                uint32_t seen, polls = 0;
                do {
                  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(epoch_sync + e - 1)
                               : "memory");
                  if (seen < gridDim.x) __nanosleep(200);
                } while (seen < gridDim.x && ++polls < 100000u);
                sync_ok = seen >= gridDim.x;
              }
            }
            const uint32_t slot = f & (RAW - 1);
            if (f >= RAW) mbar_wait(&rawfree[slot], ((f / RAW) + 1) & 1u);
            const uint32_t bar = smem_u32(&rawfull[slot]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"((uint32_t)(L::RAWA_SLOT + L::RAWB_SLOT))
                         : "memory");
            const int32_t k0 = (int32_t)(kb * KB);
            if (g.v_t) {
              // transposed view: {2 ra, rb, ki, ko, entry}; the box lands as the
              // dense [8 k][128 rows] tile of the plain opA = T path
              asm volatile(
                  "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes "
                  "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(rawa + slot * L::RAWA_SLOT),
                  "l"(&tmA), "r"(v_ra), "r"(v_rb), "r"(v_ki * KB), "r"(v_ko), "r"(aslice), "r"(bar)
                  : "memory");
              if (++v_ki == v_kbi) {
                v_ki = 0;
                ++v_ko;
              }
            } else if (g.v_kin) {
              // A view: {2 ki, ra, ko, rb, entry}; the box spans 128 rows of (ra, rb)
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
              // A: opA N -> coords {2k, m, entry}; opA T -> {2m, k, entry}
              const int32_t a0 = g.opA == QF_OP_N ? 2 * k0 : 2 * m0, a1 = g.opA == QF_OP_N ? m0 : k0;
              asm volatile(
                  "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                  "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(rawa + slot * L::RAWA_SLOT),
                  "l"(&tmA), "r"(a0), "r"(a1), "r"(aslice), "r"(bar)
                  : "memory");
            }
            // B: opB N -> {2n, k, slice}; opB T -> {2k, n, slice}
            const int32_t c0 = g.opB == QF_OP_N ? 2 * n0 : 2 * k0, c1 = g.opB == QF_OP_N ? k0 : n0;
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(rawb + slot * L::RAWB_SLOT),
                "l"(&tmB), "r"(c0), "r"(c1), "r"(bslice), "r"(bar)
                : "memory");
          }
        }
        // CTAs with fewer tiles arrive for the epochs they never reach
        if (epoch_sync)
          for (uint32_t e = (f + EPOCH - 1) / EPOCH; e < max_epochs; ++e)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(epoch_sync + e) : "memory");
      }
      __syncwarp();
    }
  } else {
    reg_dec<REGS_A>();
    convert_loop<true, PAIR>(g, smem, bars, full_leader, rawfull, rawfree, tmem, w0, wstep, total,
                             nk);
  }
  tc_fence_before();
  if constexpr (PAIR) {
    cluster_sync_all();   // the leader's MMAs read this CTA's smem / TMEM until here
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(L::TMEM_COLS));
  } else {
    __syncthreads();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(L::TMEM_COLS));
  }
}

// Lockstep counters of the TMA producers: a ring of 4 zeroed-per-launch
// slots per device (launches on one stream never overlap; the ring covers a
// second stream).  Allocated on first use outside stream capture; a launch
// that cannot have counters (first use while capturing, too many epochs)
// simply runs without lockstep.
constexpr int64_t SYNC_SLOT_WORDS = 1 << 18;
static uint32_t *sync_slot(cudaStream_t s, int64_t words) {
  static uint32_t *base[64] = {nullptr};
  static unsigned next[64] = {0};
  static const bool off = getenv("QF_TC3W_NOSYNC") != nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  if (off || dev >= 64 || words > SYNC_SLOT_WORDS) return nullptr;
  if (!base[dev]) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    if (cap != cudaStreamCaptureStatusNone) return nullptr;
    void *p = nullptr;
    if (cudaMalloc(&p, 4 * SYNC_SLOT_WORDS * sizeof(uint32_t)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    base[dev] = static_cast<uint32_t *>(p);
  }
  uint32_t *slot = base[dev] + (next[dev]++ & 3u) * SYNC_SLOT_WORDS;
  if (cudaMemsetAsync(slot, 0, (size_t)words * sizeof(uint32_t), s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return slot;
}

template <int CK, bool PAIR, int DP = 8>
static int launch_wide(const GemmArgs &g, cudaStream_t s) {
  using L = Lw<PAIR>;
  auto kern = cgemm_tc3w_kernel<CK, PAIR, DP>;
  CUtensorMap tmA{}, tmB{};
  const uint64_t nb = (uint64_t)std::max<int64_t>(g.batch, 1);
  const uint64_t na = g.a_boff ? (uint64_t)g.a_nslice : nb;   // A entries addressable
  bool okA;
  if (g.v_t) {
    // transposed view: dims {2 ra, rb, ki, ko, entry} (strides need not be
    // monotonic), box {2 min(ra, 128), 128 / min(ra, 128), 8, 1, 1}
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
                       ? make_tmap(&tmB, g.B, 2 * g.N, g.K, nbs, g.ldb * 8, sbs * 8, 2 * L::BNL, 8, false)
                       : make_tmap(&tmB, g.B, 2 * g.K, g.N, nbs, g.ldb * 8, sbs * 8, 16, L::BNL, true);
  if (!okA || !okB) {
    set_error("tc3w: cuTensorMapEncodeTiled failed (M=%lld N=%lld K=%lld)", (long long)g.M,
              (long long)g.N, (long long)g.K);
    return QF_ERR_CUDA;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) {
      set_error("tc3w: cudaFuncSetAttribute failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    attr = true;
  }
  // pair: tiles are 256 x 128, one per cluster of two CTAs
  constexpr int64_t TM = PAIR ? 2 * BM : BM;
  const int64_t tiles_n = (g.N + BN - 1) / BN, tiles_m = (g.M + TM - 1) / TM;
  const int64_t total = tiles_n * tiles_m * g.batch;
  if (total >= (int64_t)1 << 31) {
    set_error("tc3w: %lld tiles exceed the 32-bit tile index", (long long)total);
    return QF_ERR_INVALID;
  }
  const int64_t units = PAIR ? sm_count() / 2 : sm_count();
  const int64_t nunits = std::min<int64_t>(total, units);
  const int64_t grid = nunits * (PAIR ? 2 : 1);
  // lockstep where panels are long enough to drift apart (K >= 512; K = 256 measures the same)
  const int64_t nk = (g.K + KB - 1) / KB;
  const int64_t max_epochs = ((total + nunits - 1) / nunits * nk + EPOCH - 1) / EPOCH;
  static const int64_t sync_nk = [] {   // A/B knob: smallest k-block count that runs in lockstep
    const char *e = getenv("QF_TC3W_SYNCNK");
    return e ? (int64_t)atoll(e) : (int64_t)64;   // K >= 512: 2^20 x 1024 x 1024 297 -> 315 TFLOP/s
  }();
  uint32_t *epochs = (nk >= sync_nk && nunits > 1) ? sync_slot(s, max_epochs) : nullptr;
  // row tiles (pair: 256-row tiles) per raster group; QF_TC3W_GM for A/B runs
  static const uint32_t gm_env = [] {
    const char *e = getenv("QF_TC3W_GM");
    return e ? (uint32_t)std::max(1, atoi(e)) : 0u;
  }();
  const uint32_t gm = gm_env ? gm_env : 8u;   // 4..12 measure the same (326 TFLOP/s at 32768^3), 24: -2%
  if constexpr (PAIR) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(THREADS_W);
    cfg.dynamicSmemBytes = L::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, g, (uint32_t)tiles_m, (uint32_t)tiles_n,
                                       (uint32_t)total, tmA, tmB, epochs, (uint32_t)max_epochs, gm);
    if (e != cudaSuccess) {
      set_error("tc3w: pair launch failed: %s", cudaGetErrorString(e));
      return QF_ERR_CUDA;
    }
    return check_launch("cgemm_tc3w");
  }
  kern<<<(unsigned)grid, THREADS_W, L::SMEM, s>>>(g, (uint32_t)tiles_m, (uint32_t)tiles_n,
                                                  (uint32_t)total, tmA, tmB, epochs,
                                                  (uint32_t)max_epochs, gm);
  return check_launch("cgemm_tc3w");
}

}  // namespace tcw

// Shapes the wide kernel takes: TMA-describable plain operands or A views,
// row-major or transposed (no offset tables, plain row-major C), K long
// enough for the per-tile drain to vanish and N filling 128-column tiles.
bool tc3w_ok(const GemmArgs &g) {
  if (g.a_roff || g.c_trans || g.c_nblk) return false;
  if (!tc::tma_ok(g)) return false;
  // K >= 256 (one promotion chunk of 32 k-blocks per tile and up): measured
  // faster than the 64-column kernels from there on (scripts/c5_wide.py:
  // 1048576 x 256 x 256 185 -> 287 TFLOP/s); QF_TC3W_MINK moves the threshold
  static const int64_t min_k = [] {
    const char *e = getenv("QF_TC3W_MINK");
    return e ? (int64_t)atoll(e) : (int64_t)256;
  }();
  if (g.K < min_k || g.M < 128) return false;
  if (g.N < 128 || (g.N % 128 != 0 && g.N < 1024)) return false;
  return true;
}

// ck: promotion chunk in k-blocks (32 / 64 / 128); pair: 0 = single CTAs,
// 1 = CTA pairs (cta_group::2), -1 = pairs when the shape fills 256-row tiles
bool tc3w_pair_ok(const GemmArgs &g) {
  // a pair's second CTA idles on a ragged last row tile: want many 256-row tiles
  return g.M >= 1024 && (g.M % 256 == 0 || g.M >= 8192);
}

int gemm_tc3w(const GemmArgs &g, cudaStream_t s, int ck, int pair) {
  const bool use_pair = pair > 0 || (pair < 0 && tc3w_pair_ok(g));
  if (pair == 2) return tcw::launch_wide<64, true, 4>(g, s);   // A/B: 4-column drain pieces (8: +0.5%)
  if (use_pair) {
    const int st = ck == 128 ? tcw::launch_wide<128, true>(g, s)
                   : ck == 32 ? tcw::launch_wide<32, true>(g, s)
                              : tcw::launch_wide<64, true>(g, s);
    // auto mode: a device that cannot co-schedule CTA pairs (cluster launch
    // refused) still gets the single-CTA wide kernel
    if (st == QF_OK || pair > 0) return st;
    cudaGetLastError();
  }
  if (ck == 128) return tcw::launch_wide<128, false>(g, s);
  if (ck == 32) return tcw::launch_wide<32, false>(g, s);
  return tcw::launch_wide<64, false>(g, s);
}

}  // namespace qf

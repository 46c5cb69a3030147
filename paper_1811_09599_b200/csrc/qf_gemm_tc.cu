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
#include <algorithm>
#include <type_traits>
#include <utility>

#include "qf_tc_ptx.cuh"

namespace qf {


namespace tc {

// shared memory of the short-K kernel: B' stages, raw A/B rings, a per-warp
// epilogue staging tile (32 rows x CPW complex, rows padded by 16 B so both
// the row-per-lane writes and the row-contiguous reads are conflict-free)
template <int STAGES, int RAW, int NW, int NE, int BN_ = V2_BN, int CK_ = 0, int NPW_ = 0,
          bool TMA_ = false, bool G3_ = false, int ALT_ = 1>
struct LayoutK {
  // ALT_ = 2: the NW converter warps form two groups that take alternate
  // k-blocks (group g converts k-blocks q with q % 2 == g), so each warp has
  // two k-blocks of tensor time to cover its per-k-block latency chain
  // (mbarrier waits, shared-memory round trips, the async-proxy fence,
  // tcgen05.st + wait) -- with one group the converters, not the tensor
  // pipe, paced the long-K kernel (tensor pipe ~46% active).
  static_assert(ALT_ == 1 || (ALT_ == 2 && G3_ && NW == 16), "alternating groups: Gauss form");
  static constexpr int ALT = ALT_;
  // G3_: the Gauss (3-multiplication) form of the complex product on the
  // tensor pipe -- T1 = Ar.Br, T2 = Ai.Bi, T3 = (Ar+Ai).(Br+Bi), Re = T1 - T2,
  // Im = T3 - T1 - T2 -- i.e. 9 TF32 MMAs of N = BN per 8 complex k instead
  // of 6 of N = 2 BN (3/4 of the tensor work).  B' planes hold [Br | Bi | Br+Bi]
  // (hi and lo), A in TMEM holds Ar, Ai, Ar+Ai (hi and lo: 48 columns per
  // stage).  Long-K TMA-fed only: one TMEM partial [T1 | T2 | T3] drained by
  // the promotion warps into the fp32 master [Re | Im] every CK_ k-blocks.
  static_assert(!G3_ || (CK_ > 0 && TMA_ && NPW_ == 1 && BN_ == 64 && NW == 8 * ALT_),
                "the Gauss form is a long-K TMA-fed flavour with 64-column tiles");
  static constexpr bool G3 = G3_;
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
  static constexpr int NWG = NW / ALT_ / 4;          // warps per TMEM lane quadrant (per group)
  static constexpr int KPW = KB / NWG;               // k of a k-block per warp
  static constexpr int BN = BN_;                     // complex output columns per tile
  static constexpr int CPW = BN / NWG;               // epilogue columns per warp
  static constexpr int NP = G3_ ? BN : 2 * BN;        // real N of one MMA
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
  // TMEM columns: partial accumulator(s), the long-K master, the A ring
  static constexpr int P_COLS = G3_ ? 3 * BN : NP;           // [T1 | T2 | T3] or [Dre | Dim]
  static constexpr int MASTER_COL = G3_ ? P_COLS : 2 * P_COLS;  // fp32 master [Re | Im]
  static constexpr int A_COL0 = G3_ ? P_COLS + 2 * BN : (CK_ ? 3 : 2) * P_COLS;
  static constexpr int A_STAGE_COLS = G3_ ? 48 : 32;
  static constexpr int TMEM_COLS = 512;
  static_assert(A_COL0 + STAGES * A_STAGE_COLS <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

template <int STAGES, int RAW, int NW, int NE, int BN_, int CK_, int NPW, bool TMA, bool G3 = false,
          int ALT = 1>
__global__ void __launch_bounds__((NW + NE + NPW) * 32 + 32, 1)
    cgemm_tc3k_kernel(const __grid_constant__ GemmArgs g, uint32_t tiles_m, uint32_t tiles_n,
                      uint32_t total, uint32_t chunk, const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB) {
  using L = LayoutK<STAGES, RAW, NW, NE, BN_, CK_, NPW, TMA, G3, ALT>;
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
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], NW / ALT);
    for (int i = 0; i < 2; ++i) mbar_init(&accfree[i], NE ? NE : 1);
    for (int i = 0; i < RAW; ++i) {
      mbar_init(&rawfull[i], (NPW && !TMA) ? NPW * 32 : 1);
      mbar_init(&rawfree[i], NW / ALT);
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
    // ===== MMA issuer: the whole warp walks the sequence (its values stay in
    // uniform registers), one elected lane issues.  Per stage only the
    // waits, the MMAs and the commits run: the B' descriptors are the
    // stage-0 descriptor plus a constant byte offset >> 4 (the address field
    // is the descriptor's low 14 bits and shared memory < 256 KB), the A
    // planes a constant TMEM column offset.  With 9 N = 64 MMAs per stage
    // (Gauss form) per-stage descriptor arithmetic used to pace the tensor
    // pipe.  (A lone-lane loop is worse: every MMA then needs an
    // elect/broadcast waterfall to move its operands to uniform registers.)
    {
      const uint64_t desc0 = smem_desc(smem_u32(smem));
      constexpr uint32_t ST16 = (uint32_t)L::STAGE >> 4, BP16 = (uint32_t)L::B_PLANE >> 4,
                         BB16 = (uint32_t)L::B_BLOCK >> 4;
      // (Measured alternatives for the Gauss form, all slower on the full
      // kernel: one lane issuing alone (operand waterfalls), waiting on every
      // other stage, and issuing k-block pairs per elect block -- the latter
      // two only win when the converters are idle; profiles/r2_gemm_notes.md.)
      uint32_t q = 0, t = 0, chunkc = 0;
      for (uint32_t w = w0; w < w1; w += wstep, ++t) {
        for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
          const uint32_t s = q & (STAGES - 1);
          mbar_wait(&full[s], (q / STAGES) & 1u);
          tc_fence_after();
          uint32_t pbuf = t & 1u;
          uint32_t pos = kb;
          if constexpr (G3) {
            // one partial buffer: the promotion warps read chunk c-1 out of it
            // before chunk c's first MMA overwrites it
            pos = kb & (CK_ - 1);
            pbuf = 0;
            if (pos == 0 && chunkc >= 1 && !(g.dbg & 64)) {
              mbar_wait(&accfree[0], (chunkc - 1) & 1u);
              tc_fence_after();
            }
          } else if constexpr (PROMO) {
            pos = kb & (CK_ - 1);
            pbuf = chunkc & 1u;
            if (pos == 0 && chunkc >= 2) {  // promotion warps drained this partial
              mbar_wait(&accfree[pbuf], ((chunkc >> 1) + 1) & 1u);
              tc_fence_after();
            }
          }
          if (!PROMO && NE > 0 && kb == 0 && t >= 2) {  // epilogue warps drained this buffer (tile t-2)
            mbar_wait(&accfree[t & 1u], ((t >> 1) + 1) & 1u);
            tc_fence_after();
          }
          const uint32_t d = tmem + pbuf * (uint32_t)L::P_COLS;
          const uint64_t bh = desc0 + (uint64_t)(s * ST16), bl = bh + BP16;
          const uint32_t a = tmem + (uint32_t)L::A_COL0 + s * (uint32_t)L::A_STAGE_COLS;
          const uint32_t acc0 = pos > 0 ? 1u : 0u;
          const bool chunk_end = PROMO ? (pos == CK_ - 1 || kb == nk - 1) : (kb == nk - 1);
          if constexpr (G3) {
            if (elect_one()) {
              // A planes: Ar hi/lo (+0, +8), Ai hi/lo (+16, +24), Ar+Ai hi/lo
              // (+32, +40); B' blocks 0/1/2 = Br, Bi, Br+Bi (hi plane, lo plane)
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                const uint32_t dj = d + (uint32_t)(j * BN_);
                mma_ts(dj, a + 16 * j, bh + j * BB16, IDESC, acc0);
                mma_ts(dj, a + 16 * j, bl + j * BB16, IDESC, 1u);
                mma_ts(dj, a + 16 * j + 8, bh + j * BB16, IDESC, 1u);
              }
              mma_commit(&bars[s]);
              if (chunk_end) mma_commit(&pbar[0]);
            }
          } else if (elect_one()) {
            // [Dre|Dim] += Ar.[Br|Bi] + Ai.[-Bi|Br]: windows at B' blocks 1 and 0
            mma_ts(d, a + 0, bh + BB16, IDESC, acc0);
            mma_ts(d, a + 0, bl + BB16, IDESC, 1u);
            mma_ts(d, a + 8, bh + BB16, IDESC, 1u);
            mma_ts(d, a + 16, bh, IDESC, 1u);
            mma_ts(d, a + 16, bl, IDESC, 1u);
            mma_ts(d, a + 24, bh, IDESC, 1u);
            mma_commit(&bars[s]);
            if (chunk_end) mma_commit(&pbar[pbuf]);
          }
          if (PROMO && chunk_end) ++chunkc;
          __syncwarp();
        }
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
          if (g.dbg & 32) continue;   // profiling: converters only hand stages over
          const uint32_t slot = f & (RAW - 1);
          if (f >= RAW) mbar_wait(&rawfree[slot], ((f / RAW) + 1) & 1u);
          const uint32_t bar = smem_u32(&rawfull[slot]);
          if (g.dbg & 8) {   // profiling: no operand traffic at all
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
            if (++v_ki == (g.v_kin ? (int32_t)(g.v_kin / KB) : 1)) {
              v_ki = 0;
              ++v_ko;
            }
            continue;
          }
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
    const uint32_t nchunks = (nk + CK_ - 1) / (CK_ > 0 ? CK_ : 1);
    const uint32_t mbase = tmem + lane_base + (uint32_t)L::MASTER_COL;
    uint32_t chunkc = 0;
    Cur ec;
    cur_init(ec, w0);
    for (; ec.w < w1; cur_next(ec)) {
      for (uint32_t c = 0; c < nchunks && L::G3; ++c, ++chunkc) {
        // Gauss form: master [Re | Im] (+)= [T1 - T2 | T3 - T1 - T2] from the
        // single partial [T1 | T2 | T3]; the partial is released to the MMA
        // warp as soon as its last piece has been read
        mbar_wait_sleep(&pbar[0], chunkc & 1u, 200u);   // a chunk is ~10 us of MMAs
        tc_fence_after();
        if (g.dbg & 4) {
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accfree[0])) : "memory");
          continue;
        }
        const uint32_t pbase = tmem + lane_base;
        constexpr int PC = L::ALT > 1 ? 8 : 16;   // columns per piece (register budget)
#pragma unroll 1
        for (int piece = 0; piece < BN / PC; ++piece) {
          uint32_t t1[PC], t2[PC], t3[PC], mr[PC], mi[PC];
          tmem_ld_cols<PC>(pbase + piece * PC, t1);
          tmem_ld_cols<PC>(pbase + BN + piece * PC, t2);
          tmem_ld_cols<PC>(pbase + 2 * BN + piece * PC, t3);
          if (c > 0) {
            tmem_ld_cols<PC>(mbase + piece * PC, mr);
            tmem_ld_cols<PC>(mbase + BN + piece * PC, mi);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (piece == BN / PC - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
              asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&accfree[0]))
                           : "memory");
          }
#pragma unroll
          for (int j = 0; j < PC; ++j) {
            const float x1 = __uint_as_float(t1[j]), x2 = __uint_as_float(t2[j]);
            const float re = x1 - x2, im = __uint_as_float(t3[j]) - x1 - x2;
            t1[j] = __float_as_uint(c > 0 ? __uint_as_float(mr[j]) + re : re);
            t2[j] = __float_as_uint(c > 0 ? __uint_as_float(mi[j]) + im : im);
          }
          tmem_st_cols<PC>(mbase + piece * PC, t1);
          tmem_st_cols<PC>(mbase + BN + piece * PC, t2);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
      }
      for (uint32_t c = 0; c < nchunks && !L::G3; ++c, ++chunkc) {
        const uint32_t pbuf = chunkc & 1u;
        mbar_wait_sleep(&pbar[pbuf], (chunkc >> 1) & 1u, 500u);
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
    constexpr int NTG = NT / ALT;         // converter threads per group
    const int gtid = tid % NTG, grp = tid / NTG;
    constexpr int BE = (BN * KB) / NTG;   // B elements per thread per k-block (BN = 64)
    if constexpr (BE == 2) {
      // a half-warp covers 16 columns n0..n0+15: lanes 0-7 take n0..n0+7 at
      // one k pair, lanes 8-15 n0+8..n0+15 at the other (the next half-warp
      // the swapped pairs).  The raw-B reads (two k rows, 1 KB apart) then
      // touch disjoint bank halves, and the 8-byte B' stores of the 16 lanes
      // fill all 32 banks of one core-matrix row block: one wavefront each.
      const int t = gtid & 127, hw = t >> 4, l = t & 15;
      const int b_kp = ((l >> 3) & 1) ^ (hw & 1), b_chunk = gtid >> 7;
      b_n = 16 * (hw >> 1) + (l & 7) + 8 * ((l >> 3) & 1);
      b_k = b_chunk * 4 + b_kp * 2;
      boff = core_off(b_n, b_chunk) + (uint32_t)(b_kp * 8);
    } else {
      b_k = gtid & 7;
      b_n = gtid >> 3;
      boff = core_off(b_n, b_k >> 2) + (uint32_t)((b_k & 3) * 4);
    }
    const uint32_t kw0 = (uint32_t)((wg % L::NWG) * KPW);
    constexpr int CPR = KPW / 2;
    Cur cc;
    cur_init(cc, w0);
    uint32_t q = 0;
    for (; cc.w < w1; cur_next(cc)) {
      const bool breuse = rd != 0u && cc.run >= rd;
      for (uint32_t kb = 0; kb < nk; ++kb, ++q) {
        if (ALT > 1 && (int)(q % ALT) != grp) continue;   // the other group's k-block
        const uint32_t slot = q & (RAW - 1), s = q & (STAGES - 1);
        if (g.dbg & 32) {   // profiling: only the stage handshake (use with 8: no producer traffic)
          if (q >= STAGES) mbar_wait(&bars[s], ((q / STAGES) + 1) & 1u);
          tc_fence_before();
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
          continue;
        }
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
        if constexpr (L::G3) {
          // Gauss form.  Everything is split into registers BEFORE the wait
          // for the stage to be free, so only the stores sit between the
          // tensor pipe releasing stage s and this warp's arrival on full[s]
          // (that latency, not bandwidth, paced the pipe).  B' blocks [Br | Bi
          // | Br + Bi] (hi and lo planes); A planes Ar, Ai, Ar + Ai in TMEM
          // (hi at +0/+16/+32, lo 8 columns after).
          uint32_t bp[12];
          if constexpr (BE == 2) {
            split_fast(bb4.x, bp[0], bp[6]);
            split_fast(bb4.y, bp[2], bp[8]);
            split_fast(bb4.x + bb4.y, bp[4], bp[10]);
            split_fast(bb4.z, bp[1], bp[7]);
            split_fast(bb4.w, bp[3], bp[9]);
            split_fast(bb4.z + bb4.w, bp[5], bp[11]);
          }
          uint32_t rh[KPW], rl[KPW], ih[KPW], il[KPW], sh[KPW], sl[KPW];
#pragma unroll
          for (int p = 0; p < CPR; ++p) {
            split_fast(av[p].x, rh[2 * p], rl[2 * p]);
            split_fast(av[p].y, ih[2 * p], il[2 * p]);
            split_fast(av[p].x + av[p].y, sh[2 * p], sl[2 * p]);
            split_fast(av[p].z, rh[2 * p + 1], rl[2 * p + 1]);
            split_fast(av[p].w, ih[2 * p + 1], il[2 * p + 1]);
            split_fast(av[p].z + av[p].w, sh[2 * p + 1], sl[2 * p + 1]);
          }
          if (q >= STAGES) mbar_wait(&bars[s], ((q / STAGES) + 1) & 1u);
          if (!breuse && !(g.dbg & 1)) {
            uint8_t *stage = smem + s * L::STAGE;
            uint8_t *ph = stage, *pl = stage + L::B_PLANE;
            if constexpr (BE == 2) {
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                *reinterpret_cast<uint2 *>(ph + j * L::B_BLOCK + boff) = make_uint2(bp[2 * j], bp[2 * j + 1]);
                *reinterpret_cast<uint2 *>(pl + j * L::B_BLOCK + boff) =
                    make_uint2(bp[6 + 2 * j], bp[6 + 2 * j + 1]);
              }
            }
            fence_async_smem();
          }
          const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * L::A_STAGE_COLS) + kw0;
          static_assert(KPW == 4, "Gauss form: 8 converter warps per group");
          if (!(g.dbg & 2)) {
            tmem_st4(acol + 0, rh[0], rh[1], rh[2], rh[3]);
            tmem_st4(acol + 8, rl[0], rl[1], rl[2], rl[3]);
            tmem_st4(acol + 16, ih[0], ih[1], ih[2], ih[3]);
            tmem_st4(acol + 24, il[0], il[1], il[2], il[3]);
            tmem_st4(acol + 32, sh[0], sh[1], sh[2], sh[3]);
            tmem_st4(acol + 40, sl[0], sl[1], sl[2], sl[3]);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          }
        } else {
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
          const uint32_t acol = tmem + lane_base + (uint32_t)(L::A_COL0 + s * L::A_STAGE_COLS) + kw0;
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
        }  // real-block form
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
bool make_tmap(CUtensorMap *m, const void *ptr, uint64_t d0, uint64_t d1, uint64_t d2,
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
bool make_tmap5(CUtensorMap *m, const void *ptr, const uint64_t (&dims)[5],
                const uint64_t (&strides)[4], const uint32_t (&box)[5], bool swz64) {
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

template <int STAGES, int RAW, int NW, int NE, int BN = V2_BN, int CK = 0, int NPW = 0, bool TMA = false,
          bool G3 = false, int ALT = 1>
int launch_short(const GemmArgs &g, cudaStream_t s) {
  using L = LayoutK<STAGES, RAW, NW, NE, BN, CK, NPW, TMA, G3, ALT>;
  auto kern = cgemm_tc3k_kernel<STAGES, RAW, NW, NE, BN, CK, NPW, TMA, G3, ALT>;
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
  // the Gauss flavour is reported under its own name (9 real TF32 MACs per
  // complex MAC instead of 12: its tensor roofline differs)
  return check_launch(G3 ? "cgemm_tc3g" : "cgemm_tc3k");
}

}  // namespace tc

// Tuning knob (qf_tc3_set_variant): 0 = auto.  Pins for A/B measurements of
// the kernel flavours auto chooses between: 10/11/12/20 = short-K flavours
// (launch_short_auto), 21 = TMA short-K with a 4-deep A ring, 23 = 64-column
// tiles for narrow TMA views, 13/19/26/27/30/31 = long-K flavours
// (launch_long).
static int g_tc3_variant = 0;

bool tc3_gather_ok(const GemmArgs &g) { return g.K <= 4096; }

// TMA-fed short-K runs: RAW k-blocks of A (8 KiB each) in flight per CTA.
// 8 deep for plain operands and strided views alike: the config-2 view GEMMs
// 1024 x (4096 x 64 x 64) run 0.69 ms 8 deep vs 0.80-0.85 ms 4 deep (6.26 TB/s,
// 0.97 of the measured HBM copy rate).
static int launch_short_tma(const GemmArgs &g, cudaStream_t s) {
  if (g_tc3_variant == 21) return tc::launch_short<8, 4, 8, 4, 64, 0, 1, true>(g, s);
  // narrow outputs (a transposed view with N <= 32): 32-column tiles halve
  // the padded MMA work, which otherwise paces the HBM-bound tile
  if (g.N <= 32 && g_tc3_variant != 23) return tc::launch_short<8, 8, 8, 4, 32, 0, 1, true>(g, s);
  return tc::launch_short<8, 8, 8, 4, 64, 0, 1, true>(g, s);
}

// long K: a TMA producer warp, 8 converter warps, 4 promotion warps with a
// TMEM master accumulator.  Default: the Gauss form (9 instead of 12 TF32
// MMAs per complex MAC) with the partial promoted every 64 k-blocks (512 k:
// truncation error of the tensor pipe's fp32 accumulation ~3.7e-6 per chunk,
// rounded sums across chunks).  Under the 1 kW cap the big GEMMs are power
// bound, and 3/4 of the tensor work runs them ~17% faster at higher clocks
// (32768^3: 158.6 -> 185.5 TFLOP/s sustained; 4096 x 65536 x 4096: 171.5
// -> 198.3; profiles/r2_gemm_g3.jsonl).  Pins: 19 = the real-block form
// (CK 4), 26/27 = real-block CK 16/32, 30/31 = Gauss CK 16/32, 13 =
// converter fetch (no TMA; also the fallback when TMA cannot describe the
// operands).
static int launch_long(const GemmArgs &g, cudaStream_t s) {
  // N >= 128 and K >= 256: the wide (128 x 128) Gauss kernel with its master in
  // registers (qf_gemm_tcw.cu).  Pins: 40/41/42 = wide single-CTA with CK
  // 64/128/32, 43/44/45 = CTA pairs (cta_group::2) with CK 64/128/32, 32 = the
  // 64-column Gauss kernel (CK 64).
  if ((g_tc3_variant == 0 || (g_tc3_variant >= 40 && g_tc3_variant <= 46)) && tc3w_ok(g)) {
    if (g_tc3_variant == 46) return gemm_tc3w(g, s, 64, 2);
    const int v = g_tc3_variant;
    const int ck = (v == 41 || v == 44) ? 128 : (v == 42 || v == 45) ? 32 : 64;
    return gemm_tc3w(g, s, ck, v == 0 ? -1 : v >= 43 ? 1 : 0);   // auto: pairs when M fills them
  }
  if (g_tc3_variant != 13 && tc::tma_ok(g)) {
    if (g_tc3_variant == 19) return tc::launch_short<4, 8, 8, 4, 64, 4, 1, true>(g, s);
    if (g_tc3_variant == 26) return tc::launch_short<4, 8, 8, 4, 64, 16, 1, true>(g, s);
    if (g_tc3_variant == 27) return tc::launch_short<4, 8, 8, 4, 64, 32, 1, true>(g, s);
    if (g_tc3_variant == 30) return tc::launch_short<4, 8, 8, 4, 64, 16, 1, true, true>(g, s);
    if (g_tc3_variant == 31) return tc::launch_short<4, 8, 8, 4, 64, 32, 1, true, true>(g, s);
    if (g_tc3_variant == 32) return tc::launch_short<4, 8, 8, 4, 64, 64, 1, true, true>(g, s);
    if (g_tc3_variant == 34) return tc::launch_short<2, 8, 8, 4, 64, 64, 1, true, true>(g, s);
    return tc::launch_short<4, 8, 8, 4, 64, 64, 1, true, true>(g, s);
  }
  return tc::launch_short<4, 8, 8, 4, 64, 4>(g, s);
}

// short-K kernel flavour: output-bound shapes (K <= 56) keep the epilogue on
// the converter warps (more store parallelism); longer K hands it to 4
// dedicated epilogue warps so conversion, MMA and stores overlap.
static int launch_short_auto(const GemmArgs &g, cudaStream_t s) {
  // pins: 10/11 = 8/16 converter warps with the epilogue on the converters,
  // 12 = 16 converter + 4 epilogue warps, 20 = the TMA-fed run kernel
  if (g_tc3_variant == 10) return tc::launch_short<8, 4, 8, 0>(g, s);
  if (g_tc3_variant == 11) return tc::launch_short<8, 4, 16, 0>(g, s);
  if (g_tc3_variant == 12) return tc::launch_short<8, 8, 16, 4>(g, s);
  if (g_tc3_variant == 20 && tc::tma_ok(g)) return tc::launch_short<8, 8, 8, 4, 64, 0, 1, true>(g, s);
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

static int tc3_debug() {
  static const int v = [] {
    const char *e = getenv("QF_TC3_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

int gemm_tc3(const GemmArgs &g_in, cudaStream_t s) {
  GemmArgs g = g_in;
  g.dbg = tc3_debug();
  if (g.batch == 0 || g.M == 0 || g.N == 0) return QF_OK;
  QF_REQUIRE(g.K > 0, "tc3: K must be positive (use FFMA for K == 0)");
  // huge M with K = 16, N = 16 / 32: the streaming kernel (pin 50 = off)
  if (g_tc3_variant != 50 && (g_tc3_variant == 0 || g_tc3_variant == 51) && tc3s_ok(g))
    return gemm_tc3s(g, s);
  if (g.c_nblk && (!g.v_kin || g.K > 128 || g.c_trans)) {
    set_error("tc3: column-blocked C only on the short-K view kernel");
    return QF_ERR_UNSUPPORTED;
  }
  if (g.c_trans && !g.v_t) {
    set_error("tc3: transposed C only on a transposed A view");
    return QF_ERR_UNSUPPORTED;
  }
  if (g.v_kin) {  // A views are read by the TMA-fed kernels only
    // (narrow N runs 32-column tiles that compute zeros beyond N; the
    // HBM-bound shapes do not mind)
    // long K (N-views): the promoted long-K kernel with its TMA producer
    // (plain row-major epilogue only)
    // (transposed views with long K: the wide kernel only)
    const bool long_k = g.K > 128 && !g.c_trans && g.N > 32 && (!g.v_t || tc3w_ok(g));
    if (!(g.K >= 32 && (g.K <= 128 || long_k) && tc::tma_ok(g))) {
      set_error("tc3: A view (kin %lld, rows %lld x %lld) not TMA-describable for K=%lld N=%lld",
                (long long)g.v_kin, (long long)g.v_ra, (long long)g.v_rb, (long long)g.K,
                (long long)g.N);
      return QF_ERR_UNSUPPORTED;
    }
    if (g.K > 128) return launch_long(g, s);
    return launch_short_tma(g, s);
  }
  if (g.a_roff) {  // gathered A: only the converter-fetch kernels read through tables
    QF_REQUIRE(tc3_gather_ok(g), "tc3: gathered A needs K <= 4096");
    if (g.K <= 256) return launch_short_auto(g, s);
    return tc::launch_short<4, 8, 8, 4, 64, 4>(g, s);
  }
  // short K (<= 256): no promotion needed (error <= 3.6e-6); tile-level
  // double-buffered TMEM accumulators with a deferred epilogue (unless the
  // wide kernel's K threshold, QF_TC3W_MINK, has been lowered to take them)
  if (g.K <= 256 && !((g_tc3_variant == 0 || g_tc3_variant >= 40) && tc3w_ok(g)))
    return launch_short_auto(g, s);
  return launch_long(g, s);
}

}  // namespace qf

extern "C" int qf_tc3_set_variant(int v) {
  int prev = qf::g_tc3_variant;
  qf::g_tc3_variant = v;
  return prev;
}

// K1 -- general-rank tensor index permutation for sm_100a.
//
// Replaces the reference's L/R move decomposition (rq/tensor_core.py:81-330,
// numba kernels rq/_kernels.py:105-151) and its numpy fallback
// (rq/tensor_core.py:271-273).  Output is byte-identical to
// ascontiguousarray(transpose(src, perm)).
//
// Design (B200-first, HBM-bound): one pass, every element crosses HBM once
// in each direction.
//   1. Normalise: drop unit axes, fuse axes adjacent in both layouts.
//   2. Pick the tile: A = innermost INPUT axes with >= TA elements (256 B; reads
//      become contiguous runs), B = innermost OUTPUT axes with >= TB
//      elements (writes become contiguous runs).  An axis straddling the
//      threshold is split (d -> d/f x f) so tiles stay small; power-of-two
//      bond dims always split exactly.  The tile S = A u B (grown with outer
//      input axes up to ~2K elements for work per CTA).
//   3. A CTA stages one tile in shared memory: coalesced loads along A into
//      smem rows, then coalesced stores along B out of smem.  All index math
//      inside a tile is two tiny tables each side (row offsets + slot
//      offsets), so the inner loops are add + load/store.  The smem row
//      pitch is chosen on the host by simulating bank conflicts of both
//      phases.
//   4. Persistent grid (<= 8 CTAs/SM resident over all tiles), tiles walked
//      in output order for write locality.
// Plans (tables) are cached per (dims, perm, elem size, device).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "qf_common.cuh"

namespace qf {

static constexpr int kMaxRank = 64;
static constexpr int kThreads = 256;

struct PermParams {
  int64_t ntiles;
  int n_outer;
  int LA, HB, LB, HA, pitch, T;
  int la_shift, lb_shift;  // log2 if power of two, else -1
  int skew_q, skew_s;      // vec2 tile: in-row column c sits at c + skew_s * (c >> skew_q)
  int64_t outer_dim[kMaxRank];
  int64_t outer_in[kMaxRank];
  int64_t outer_out[kMaxRank];
};

// ---------------------------------------------------------------------------
// kernels

template <typename E, bool POW2>
__global__ void __launch_bounds__(kThreads)
    permute_tiled_kernel(const E *__restrict__ src, E *__restrict__ dst,
                         const __grid_constant__ PermParams p, const int64_t *__restrict__ tab64,
                         const int32_t *__restrict__ tab32) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int LA = p.LA, LB = p.LB, HB = p.HB, HA = p.HA, T = p.T, pitch = p.pitch;
  E *tile = reinterpret_cast<E *>(smem_raw);
  size_t tile_bytes = ((size_t)HB * pitch * sizeof(E) + 15) & ~(size_t)15;
  int64_t *s_hin = reinterpret_cast<int64_t *>(smem_raw + tile_bytes);
  int64_t *s_outk = s_hin + HB;
  int32_t *s_f = reinterpret_cast<int32_t *>(s_outk + HA);
  int32_t *s_g = s_f + HA;
  __shared__ int64_t s_base[2];

  for (int i = tid; i < HB + HA; i += kThreads) s_hin[i] = tab64[i];
  for (int i = tid; i < HA + LB; i += kThreads) s_f[i] = tab32[i];

  constexpr int U = 4;
  for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    if (tid == 0) {
      int64_t rem = t, bi = 0, bo = 0;
      for (int a = p.n_outer - 1; a >= 0; --a) {
        int64_t d = p.outer_dim[a];
        int64_t q = rem / d;
        int64_t digit = rem - q * d;
        rem = q;
        bi += digit * p.outer_in[a];
        bo += digit * p.outer_out[a];
      }
      s_base[0] = bi;
      s_base[1] = bo;
    }
    __syncthreads();
    const E *sp = src + s_base[0];
    E *dp = dst + s_base[1];

    // load phase: coalesced along A (input-contiguous) into smem rows
    for (int i0 = tid; i0 < T; i0 += kThreads * U) {
      E v[U];
      int pos[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int i = i0 + u * kThreads;
        if (i < T) {
          int eh, el;
          if (POW2) {
            eh = i >> p.la_shift;
            el = i & (LA - 1);
          } else {
            eh = i / LA;
            el = i - eh * LA;
          }
          v[u] = __ldg(sp + s_hin[eh] + el);
          pos[u] = eh * pitch + el;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u * kThreads < T) tile[pos[u]] = v[u];
      }
    }
    __syncthreads();

    // store phase: coalesced along B (output-contiguous) out of smem
    for (int i0 = tid; i0 < T; i0 += kThreads * U) {
      E v[U];
      int64_t off[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int i = i0 + u * kThreads;
        if (i < T) {
          int uh, ul;
          if (POW2) {
            uh = i >> p.lb_shift;
            ul = i & (LB - 1);
          } else {
            uh = i / LB;
            ul = i - uh * LB;
          }
          v[u] = tile[s_f[uh] + s_g[ul]];
          off[u] = s_outk[uh] + ul;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u * kThreads < T) dp[off[u]] = v[u];
      }
    }
  }
}

// Pair-vectorised, software-pipelined twin (used when LA and LB are even --
// always true for power-of-two bond dims).  Element pairs are 16-byte
// aligned and contiguous along A in the input and along B in the output.
// Tile k+1 streams into one of two shared buffers with cp.async (no
// registers held, many requests in flight) while tile k is written out of
// the other; the base offsets of every tile this CTA owns are precomputed
// into shared memory in chunks, so the steady-state loop is pure
// address-add + copy.
constexpr int kBaseChunk = 256;

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool POW2>
__global__ void __launch_bounds__(kThreads)
    permute_tiled_vec2_kernel(const float4 *__restrict__ src, float4 *__restrict__ dst,
                              const __grid_constant__ PermParams p,
                              const int64_t *__restrict__ tab64,
                              const int32_t *__restrict__ tab32) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int LA = p.LA, LB = p.LB, HB = p.HB, HA = p.HA, T = p.T, pitch = p.pitch;
  const size_t tile_bytes = ((size_t)HB * pitch * sizeof(float2) + 15) & ~(size_t)15;
  float2 *tiles[2] = {reinterpret_cast<float2 *>(smem_raw),
                      reinterpret_cast<float2 *>(smem_raw + tile_bytes)};
  int64_t *s_hin = reinterpret_cast<int64_t *>(smem_raw + 2 * tile_bytes);
  int64_t *s_outk = s_hin + HB;
  int64_t *s_base = s_outk + HA;                     // [kBaseChunk][2]
  int32_t *s_f = reinterpret_cast<int32_t *>(s_base + 2 * kBaseChunk);
  int32_t *s_g = s_f + HA;
  for (int i = tid; i < HB + HA; i += kThreads) s_hin[i] = tab64[i];
  for (int i = tid; i < HA + LB; i += kThreads) s_f[i] = tab32[i];
  const int T2 = T >> 1;
  const float2 *src2 = reinterpret_cast<const float2 *>(src);
  float2 *dst2 = reinterpret_cast<float2 *>(dst);
  const int64_t my_tiles = (p.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  auto issue = [&](int j, int buf) {  // cp.async tile j (chunk-local index) into buf
    const float2 *sp = src2 + s_base[2 * j];
    float2 *tb = tiles[buf];
    for (int i2 = tid; i2 < T2; i2 += kThreads) {
      const int i = i2 * 2;
      int eh, el;
      if (POW2) {
        eh = i >> p.la_shift;
        el = i & (LA - 1);
      } else {
        eh = i / LA;
        el = i - eh * LA;
      }
      cp_async16(tb + eh * pitch + el + p.skew_s * (el >> p.skew_q), sp + s_hin[eh] + el);
    }
    cp_async_commit();
  };
  // logical tile position (row * LA + column, the f/g tables) -> smem slot
  auto phys = [&](int pos) {
    int row, col;
    if (POW2) {
      row = pos >> p.la_shift;
      col = pos & (LA - 1);
    } else {
      row = pos / LA;
      col = pos - row * LA;
    }
    return row * pitch + col + p.skew_s * (col >> p.skew_q);
  };
  auto drain = [&](int j, int buf) {  // write tile j out of buf
    float2 *dp = dst2 + s_base[2 * j + 1];
    const float2 *tb = tiles[buf];
    for (int i2 = tid; i2 < T2; i2 += kThreads) {
      const int i = i2 * 2;
      int uh, ul;
      if (POW2) {
        uh = i >> p.lb_shift;
        ul = i & (LB - 1);
      } else {
        uh = i / LB;
        ul = i - uh * LB;
      }
      const int f = s_f[uh];
      const float2 a = tb[phys(f + s_g[ul])];
      const float2 b = tb[phys(f + s_g[ul + 1])];
      *reinterpret_cast<float4 *>(dp + s_outk[uh] + ul) = make_float4(a.x, a.y, b.x, b.y);
    }
  };

  for (int64_t c0 = 0; c0 < my_tiles; c0 += kBaseChunk) {
    const int cn = (int)min((int64_t)kBaseChunk, my_tiles - c0);
    __syncthreads();  // previous chunk fully drained before its bases are overwritten
    for (int j = tid; j < cn; j += kThreads) {
      int64_t rem = blockIdx.x + (c0 + j) * gridDim.x, bi = 0, bo = 0;
      for (int a = p.n_outer - 1; a >= 0; --a) {
        const int64_t d = p.outer_dim[a];
        const int64_t q = rem / d;
        const int64_t digit = rem - q * d;
        rem = q;
        bi += digit * p.outer_in[a];
        bo += digit * p.outer_out[a];
      }
      s_base[2 * j] = bi;
      s_base[2 * j + 1] = bo;
    }
    __syncthreads();
    issue(0, 0);
    for (int j = 0; j < cn; ++j) {
      if (j + 1 < cn) {
        issue(j + 1, (j + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();  // every thread's copies of tile j have landed
      drain(j, j & 1);
      __syncthreads();  // tile j's buffer is free for tile j + 2
    }
  }
}

struct NaiveParams {
  int64_t n;
  int rank;
  int64_t out_dim[kMaxRank];
  int64_t in_stride[kMaxRank];  // input stride of the axis at each output position
};

template <typename E>
__global__ void permute_naive_kernel(const E *__restrict__ src, E *__restrict__ dst,
                                     const __grid_constant__ NaiveParams p) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < p.n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = t, off = 0;
    for (int j = p.rank - 1; j >= 0; --j) {
      int64_t d = p.out_dim[j];
      int64_t q = rem / d;
      off += (rem - q * d) * p.in_stride[j];
      rem = q;
    }
    dst[t] = src[off];
  }
}

// ---------------------------------------------------------------------------
// host planner

struct PermPlan {
  enum Kind { kCopy, kTiled, kNaive } kind = kCopy;
  int64_t n = 0;
  PermParams tp{};
  NaiveParams np{};
  std::vector<int64_t> tab64;
  std::vector<int32_t> tab32;
  size_t smem = 0;
  int grid = 1;
  bool vec2 = false;
  // device copies (per plan per device)
  int64_t *d64 = nullptr;
  int32_t *d32 = nullptr;
  // set when the plan was requested while a stream was capturing: a CUDA
  // graph holds its table pointers, so the cache never evicts it
  bool pinned = false;
  PermPlan() = default;
  PermPlan(const PermPlan &) = delete;
  PermPlan &operator=(const PermPlan &) = delete;
  ~PermPlan() {  // cudaFree waits for work still using the tables
    if (d64) cudaFree(d64);
    if (d32) cudaFree(d32);
  }
};

static int ilog2_exact(int64_t v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int s = 0;
  while ((int64_t(1) << s) < v) ++s;
  return s;
}

// working representation: input-order dims + output order (operm[j] = input axis)
struct Layout {
  std::vector<int64_t> d;
  std::vector<int> operm;
  int rank() const { return (int)d.size(); }
  int out_pos(int in_axis) const {
    for (int j = 0; j < rank(); ++j)
      if (operm[j] == in_axis) return j;
    return -1;
  }
  // split input axis ax (dim D) into (D/f, f); the f part becomes ax+1
  void split(int ax, int64_t f) {
    int64_t D = d[ax];
    d[ax] = D / f;
    d.insert(d.begin() + ax + 1, f);
    int j = out_pos(ax);
    for (auto &x : operm)
      if (x > ax) ++x;
    operm.insert(operm.begin() + j + 1, ax + 1);
  }
};

static int64_t smallest_divisor_at_least(int64_t d, int64_t need) {
  // smallest f | d with f >= need (f in [2, d]); d itself if none smaller
  for (int64_t f = std::max<int64_t>(2, need); f < d && f <= 1 << 20; ++f)
    if (d % f == 0) return f;
  return d;
}

static int64_t largest_divisor_at_most(int64_t d, int64_t cap) {
  for (int64_t f = std::min(cap, d - 1); f >= 2; --f)
    if (d % f == 0) return f;
  return 1;
}

static int conflict_cost(const std::vector<int> &pos, int elem_bytes) {
  // shared-memory wavefronts for one warp-wide access of `pos` (element
  // indices); 8-byte elements go in 2 phases of 16 lanes, 16-byte in 4 of 8
  int words = elem_bytes / 4;
  int lanes_per_phase = 128 / elem_bytes;
  int cost = 0;
  for (size_t base = 0; base < pos.size(); base += lanes_per_phase) {
    int cnt[32];
    int64_t seen[32][16];
    memset(cnt, 0, sizeof(cnt));
    int worst = 0;
    for (size_t l = base; l < std::min(pos.size(), base + lanes_per_phase); ++l) {
      for (int w = 0; w < words; ++w) {
        int64_t word = (int64_t)pos[l] * words + w;
        int bank = (int)(word & 31);
        bool dup = false;
        for (int k = 0; k < cnt[bank]; ++k)
          if (seen[bank][k] == word) dup = true;
        if (!dup && cnt[bank] < 16) seen[bank][cnt[bank]++] = word;
        worst = std::max(worst, cnt[bank]);
      }
    }
    cost += worst;
  }
  return cost;
}

static int build_plan(int rank, const int64_t *dims_in, const int32_t *perm_in, int elem_bytes,
                      PermPlan &plan) {
  QF_REQUIRE(rank >= 0 && rank <= kMaxRank, "permute: rank %d out of range [0, %d]", rank, kMaxRank);
  QF_REQUIRE(elem_bytes == 8 || elem_bytes == 16, "permute: elem_bytes must be 8 or 16");
  std::vector<int> seen(rank, 0);
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) {
    QF_REQUIRE(dims_in[i] >= 0, "permute: negative dim %lld", (long long)dims_in[i]);
    QF_REQUIRE(perm_in[i] >= 0 && perm_in[i] < rank && !seen[perm_in[i]],
               "permute: perm is not a permutation of 0..%d", rank - 1);
    seen[perm_in[i]] = 1;
    n *= dims_in[i];
  }
  plan.n = n;
  if (n <= 1) {
    plan.kind = PermPlan::kCopy;
    return QF_OK;
  }
  // 1. drop unit axes
  std::vector<int> keep_index(rank, -1);
  Layout L;
  for (int i = 0; i < rank; ++i)
    if (dims_in[i] != 1) {
      keep_index[i] = (int)L.d.size();
      L.d.push_back(dims_in[i]);
    }
  for (int j = 0; j < rank; ++j)
    if (dims_in[perm_in[j]] != 1) L.operm.push_back(keep_index[perm_in[j]]);
  // 2. fuse axes consecutive in both layouts
  {
    Layout F;
    std::vector<int> group_of(L.rank(), -1);
    std::vector<std::vector<int>> groups;
    for (int j = 0; j < L.rank(); ++j) {
      if (j > 0 && L.operm[j] == L.operm[j - 1] + 1)
        groups.back().push_back(L.operm[j]);
      else
        groups.push_back({L.operm[j]});
    }
    // groups in output order; new input order = groups sorted by first axis
    std::vector<int> order(groups.size());
    for (size_t g = 0; g < groups.size(); ++g) order[g] = (int)g;
    std::sort(order.begin(), order.end(),
              [&](int a, int b) { return groups[a][0] < groups[b][0]; });
    std::vector<int> new_index(groups.size());
    for (size_t k = 0; k < order.size(); ++k) {
      new_index[order[k]] = (int)k;
      int64_t dd = 1;
      for (int ax : groups[order[k]]) dd *= L.d[ax];
      F.d.push_back(dd);
    }
    for (size_t g = 0; g < groups.size(); ++g) F.operm.push_back(new_index[g]);
    L = F;
  }
  if (L.rank() <= 1) {
    plan.kind = PermPlan::kCopy;
    return QF_OK;
  }

  // run lengths and tile size in bytes; QF_PERM_TA / QF_PERM_TB / QF_PERM_TILE
  // override them (tuning experiments only)
  // (read once per process: cached plans stay consistent with them)
  auto knob = [](const char *name, int64_t dflt) {  // clamped to sane byte counts
    const char *v = getenv(name);
    const int64_t x = v ? (int64_t)atoll(v) : dflt;
    return std::min<int64_t>(std::max<int64_t>(x, 64), 65536);
  };
  static const int64_t kTA = knob("QF_PERM_TA", 256), kTB = knob("QF_PERM_TB", 256),
                       kTile = knob("QF_PERM_TILE", 32768);
  // 256-byte runs: a 64 x 64 element tile with disjoint A/B (512-byte runs)
  // ran at 4.85 TB/s; 32-element runs let A grow to 128 inputs while B keeps
  // whole 256-byte output sectors (6.1-6.2 TB/s, profiles/r1n_permute_knobs.txt)
  const int64_t TA = kTA / elem_bytes, TB = kTB / elem_bytes;
  const int64_t Tmin = kTile / elem_bytes,
                Tmax = Tmin;  // 32 KB tiles (measured: 16 KB tiles ran ~20% slower)

  // 3. A = innermost input axes [a_start, r)
  int r = L.rank();
  int a_start = r;
  {
    int64_t prod = 1;
    for (int ax = r - 1; ax >= 0; --ax) {
      int64_t dd = L.d[ax];
      if (prod * dd >= TA) {
        int64_t f = smallest_divisor_at_least(dd, (TA + prod - 1) / prod);
        if (f < dd) {
          L.split(ax, f);
          r = L.rank();
          a_start = ax + 1;
        } else {
          a_start = ax;
        }
        break;
      }
      prod *= dd;
      a_start = ax;
    }
  }
  // B = innermost output positions [b_start, r)
  int b_start = r;
  {
    int64_t prod = 1;
    for (int j = r - 1; j >= 0; --j) {
      int ax = L.operm[j];
      int64_t dd = L.d[ax];
      if (prod * dd >= TB) {
        int64_t f = smallest_divisor_at_least(dd, (TB + prod - 1) / prod);
        if (f < dd) {
          L.split(ax, f);
          r = L.rank();
          if (ax < a_start) ++a_start;
          b_start = j + 1;
        } else {
          b_start = j;
        }
        break;
      }
      prod *= dd;
      b_start = j;
    }
  }
  auto in_S = [&](int ax) {
    if (ax >= a_start) return true;
    int j = L.out_pos(ax);
    return j >= b_start;
  };
  auto tile_size = [&]() {
    int64_t T = 1;
    for (int ax = 0; ax < r; ++ax)
      if (in_S(ax)) T *= L.d[ax];
    return T;
  };
  int64_t T = tile_size();
  // grow A outward while the tile is small
  while (T < Tmin && a_start > 0) {
    int ax = a_start - 1;
    if (in_S(ax)) {
      a_start = ax;
      continue;
    }
    int64_t dd = L.d[ax];
    if (T * dd <= Tmax) {
      a_start = ax;
      T *= dd;
      continue;
    }
    int64_t f = largest_divisor_at_most(dd, Tmax / T);
    if (f >= 2) {
      int jx = L.out_pos(ax);
      L.split(ax, f);
      r = L.rank();
      if (jx < b_start) ++b_start;  // output positions after jx shift by one
      a_start = ax + 1;
      T *= f;
    }
    break;
  }
  T = tile_size();

  // strides
  std::vector<int64_t> istride(r), ostride(r);
  {
    int64_t s = 1;
    for (int ax = r - 1; ax >= 0; --ax) {
      istride[ax] = s;
      s *= L.d[ax];
    }
    s = 1;
    for (int j = r - 1; j >= 0; --j) {
      ostride[j] = s;
      s *= L.d[L.operm[j]];
    }
  }

  if (T > Tmax || r > kMaxRank) {
    plan.kind = PermPlan::kNaive;
    NaiveParams &np = plan.np;
    np.n = n;
    np.rank = r;
    for (int j = 0; j < r; ++j) {
      np.out_dim[j] = L.d[L.operm[j]];
      np.in_stride[j] = istride[L.operm[j]];
    }
    plan.grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
    return QF_OK;
  }

  // tile bookkeeping
  std::vector<int> hb_axes;  // S \ A in input order
  for (int ax = 0; ax < a_start; ++ax)
    if (in_S(ax)) hb_axes.push_back(ax);
  std::vector<int> b_axes;   // B in output order
  for (int j = b_start; j < r; ++j) b_axes.push_back(L.operm[j]);
  std::vector<int> ha_pos;   // output positions of S \ B, output order
  for (int j = 0; j < b_start; ++j)
    if (in_S(L.operm[j])) ha_pos.push_back(j);
  std::vector<int> outer_pos;  // output positions outside S
  for (int j = 0; j < r; ++j)
    if (!in_S(L.operm[j])) outer_pos.push_back(j);

  int64_t LA = 1, HB = 1, LB = 1, HA = 1;
  for (int ax = a_start; ax < r; ++ax) LA *= L.d[ax];
  for (int ax : hb_axes) HB *= L.d[ax];
  for (int ax : b_axes) LB *= L.d[ax];
  for (int j : ha_pos) HA *= L.d[L.operm[j]];

  // row-major strides inside S\A (for e_hi) -> used for pos strides
  std::vector<int64_t> hb_stride(r, 0);
  {
    int64_t s = 1;
    for (int k = (int)hb_axes.size() - 1; k >= 0; --k) {
      hb_stride[hb_axes[k]] = s;
      s *= L.d[hb_axes[k]];
    }
  }
  auto enumerate = [&](const std::vector<int> &axes, const std::vector<int64_t> &wt) {
    // row-major enumeration over `axes` (dims L.d[axes]); value = sum digit*wt
    int64_t cnt = 1;
    for (int ax : axes) cnt *= L.d[ax];
    std::vector<int64_t> out(cnt);
    for (int64_t i = 0; i < cnt; ++i) {
      int64_t rem = i, v = 0;
      for (int k = (int)axes.size() - 1; k >= 0; --k) {
        int64_t dd = L.d[axes[k]];
        v += (rem % dd) * wt[k];
        rem /= dd;
      }
      out[i] = v;
    }
    return out;
  };
  std::vector<int> ha_axes;
  for (int j : ha_pos) ha_axes.push_back(L.operm[j]);

  std::vector<int64_t> w_in;
  for (int ax : hb_axes) w_in.push_back(istride[ax]);
  std::vector<int64_t> h_in = enumerate(hb_axes, w_in);
  std::vector<int64_t> w_out;
  for (int j : ha_pos) w_out.push_back(ostride[j]);
  std::vector<int64_t> out_k = enumerate(ha_axes, w_out);

  auto pos_tables = [&](int pitch, std::vector<int64_t> &f, std::vector<int64_t> &g) {
    auto ps = [&](int ax) -> int64_t {
      return ax >= a_start ? istride[ax] : hb_stride[ax] * pitch;
    };
    std::vector<int64_t> wf, wg;
    for (int ax : ha_axes) wf.push_back(ps(ax));
    for (int ax : b_axes) wg.push_back(ps(ax));
    f = enumerate(ha_axes, wf);
    g = enumerate(b_axes, wg);
  };

  // choose the smem row pitch by simulating both phases' bank conflicts
  // 16-byte pairs along both contiguous runs (and an even smem pitch)
  const bool vec2 = elem_bytes == 8 && LA % 2 == 0 && LB % 2 == 0;
  int best_pad = 0, best_cost = 1 << 30;
  for (int pad = 0; pad <= 16; pad += (vec2 ? 2 : 1)) {
    int pitch = (int)LA + pad;
    if ((int64_t)HB * pitch * elem_bytes > 64 * 1024) break;
    std::vector<int64_t> f, g;
    pos_tables(pitch, f, g);
    int cost = 0;
    for (int w = 0; w < 8; ++w) {
      std::vector<int> ld, st;
      for (int l = 0; l < 32; ++l) {
        int64_t i = w * 32 + l;
        if (i >= T) break;
        ld.push_back((int)((i / LA) * pitch + i % LA));
        st.push_back((int)(f[i / LB] + g[i % LB]));
      }
      cost += conflict_cost(ld, elem_bytes) + conflict_cost(st, elem_bytes);
    }
    if (cost < best_cost) {
      best_cost = cost;
      best_pad = pad;
    }
  }
  int pitch = (int)LA + best_pad;
  std::vector<int64_t> f_slot, g_slot;
  pos_tables(pitch, f_slot, g_slot);
  int skew_q = 30, skew_s = 0;
  if (elem_bytes == 8 && LA % 2 == 0 && LB % 2 == 0) {
    // the pair kernel: tables hold LOGICAL positions (pitch LA); the smem
    // slot of column c in a row is c + s*(c >> q) (+ row padding), chosen by
    // simulating its two phases: 16-byte cp.async rows in, two 8-byte reads
    // per output pair out (strided A axes among the output-contiguous ones
    // would otherwise hit one bank)
    std::vector<int64_t> f, g;
    pos_tables((int)LA, f, g);
    int best = 1 << 30;
    for (int q = 2; q <= 9; ++q) {
      for (int sk = 0; sk <= 8; sk += 2) {
        if (sk == 0 && q != 2) continue;
        if ((int64_t(1) << q) >= LA && sk) continue;
        for (int pad = 0; pad <= 16; pad += 2) {
          const int64_t row_len = LA + (sk ? (int64_t)sk * ((LA - 1) >> q) : 0) + pad;
          if (HB * row_len * elem_bytes > 44 * 1024) continue;
          auto ph = [&](int64_t pos) {
            const int64_t row = pos / LA, col = pos % LA;
            return (int)(row * row_len + col + (sk ? sk * (col >> q) : 0));
          };
          int cost = 0;
          for (int w = 0; w < 8; ++w) {
            std::vector<int> ld, st0, st1;
            for (int l = 0; l < 32; ++l) {
              const int64_t i = 2 * (w * 32 + l);
              if (i >= T) break;
              ld.push_back(ph((i / LA) * LA + i % LA) / 2);  // 16-byte slots
              st0.push_back(ph(f[i / LB] + g[i % LB]));
              st1.push_back(ph(f[i / LB] + g[i % LB + 1]));
            }
            cost += conflict_cost(ld, 16) + conflict_cost(st0, 8) + conflict_cost(st1, 8);
          }
          if (cost < best) {
            best = cost;
            skew_q = sk ? q : 30;
            skew_s = sk;
            pitch = (int)row_len;
          }
        }
      }
    }
    f_slot = f;
    g_slot = g;
  }

  PermParams &tp = plan.tp;
  memset(&tp, 0, sizeof(tp));
  tp.LA = (int)LA;
  tp.HB = (int)HB;
  tp.LB = (int)LB;
  tp.HA = (int)HA;
  tp.T = (int)T;
  tp.pitch = pitch;
  tp.skew_q = skew_q;
  tp.skew_s = skew_s;
  tp.la_shift = ilog2_exact(LA);
  tp.lb_shift = ilog2_exact(LB);
  tp.n_outer = (int)outer_pos.size();
  tp.ntiles = 1;
  for (int k = 0; k < tp.n_outer; ++k) {
    int j = outer_pos[k];
    tp.outer_dim[k] = L.d[L.operm[j]];
    tp.outer_in[k] = istride[L.operm[j]];
    tp.outer_out[k] = ostride[j];
    tp.ntiles *= tp.outer_dim[k];
  }
  plan.tab64 = h_in;
  plan.tab64.insert(plan.tab64.end(), out_k.begin(), out_k.end());
  for (int64_t v : f_slot) plan.tab32.push_back((int32_t)v);
  for (int64_t v : g_slot) plan.tab32.push_back((int32_t)v);
  size_t tile_bytes = ((size_t)HB * pitch * elem_bytes + 15) & ~(size_t)15;
  plan.smem = tile_bytes + (HB + HA) * 8 + (HA + LB) * 4;
  int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / (plan.smem + 1024)));
  plan.grid = (int)std::min<int64_t>(tp.ntiles, (int64_t)sm_count() * per_sm);
  plan.kind = PermPlan::kTiled;
  plan.vec2 = vec2;
  if (getenv("QF_PERM_DEBUG"))
    fprintf(stderr, "permute plan: rank %d T %lld LA %lld HB %lld LB %lld HA %lld pitch %d skew %d/%d "
            "outer %d tiles %lld\n", r, (long long)T, (long long)LA, (long long)HB, (long long)LB,
            (long long)HA, pitch, skew_s, skew_q, tp.n_outer, (long long)tp.ntiles);
  if (vec2) {
    plan.smem = 2 * tile_bytes + (HB + HA) * 8 + 2 * kBaseChunk * 8 + (HA + LB) * 4;
    int per_sm2 = (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / (plan.smem + 1024)));
    plan.grid = (int)std::min<int64_t>(tp.ntiles, (int64_t)sm_count() * per_sm2);
  }
  return QF_OK;
}

static std::mutex g_plan_mu;
static std::map<std::string, std::shared_ptr<PermPlan>> g_plans;

static int get_plan(int rank, const int64_t *dims, const int32_t *perm, int elem_bytes,
                    std::shared_ptr<PermPlan> &out, cudaStream_t stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  std::string key;
  key.reserve(16 + rank * 12);
  key.append((const char *)&dev, sizeof(dev));
  key.append((const char *)&elem_bytes, sizeof(elem_bytes));
  key.append((const char *)&rank, sizeof(rank));
  key.append((const char *)dims, sizeof(int64_t) * rank);
  key.append((const char *)perm, sizeof(int32_t) * rank);
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
      if (capturing) it->second->pinned = true;
      out = it->second;
      return QF_OK;
    }
  }
  if (capturing) {
    // building a plan allocates and uploads its tables: not capturable
    qf::set_error("permute: plan for this (dims, perm) first requested during stream capture; "
                  "run the call once before capturing");
    return QF_ERR_INVALID;
  }
  auto plan = std::make_shared<PermPlan>();
  int st = build_plan(rank, dims, perm, elem_bytes, *plan);
  if (st != QF_OK) return st;
  if (plan->kind == PermPlan::kTiled) {
    QF_CUDA(cudaMalloc(&plan->d64, plan->tab64.size() * sizeof(int64_t) + 8));
    QF_CUDA(cudaMalloc(&plan->d32, plan->tab32.size() * sizeof(int32_t) + 8));
    QF_CUDA(cudaMemcpy(plan->d64, plan->tab64.data(), plan->tab64.size() * sizeof(int64_t),
                       cudaMemcpyHostToDevice));
    QF_CUDA(cudaMemcpy(plan->d32, plan->tab32.data(), plan->tab32.size() * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
  }
  std::lock_guard<std::mutex> lk(g_plan_mu);
  if (g_plans.size() > 8192) {  // plans are cheap to rebuild; graph-held ones stay
    for (auto it = g_plans.begin(); it != g_plans.end();)
      it = it->second->pinned ? std::next(it) : g_plans.erase(it);
  }
  g_plans[key] = plan;
  out = plan;
  return QF_OK;
}

template <typename E>
static int launch(const PermPlan &plan, const void *src, void *dst, cudaStream_t s) {
  if (plan.kind == PermPlan::kCopy) {
    QF_CUDA(cudaMemcpyAsync(dst, src, (size_t)plan.n * sizeof(E), cudaMemcpyDeviceToDevice, s));
    return QF_OK;
  }
  if (plan.kind == PermPlan::kNaive) {
    permute_naive_kernel<E><<<plan.grid, 256, 0, s>>>((const E *)src, (E *)dst, plan.np);
    return check_launch("permute_naive");
  }
  bool pow2 = plan.tp.la_shift >= 0 && plan.tp.lb_shift >= 0;
  if (sizeof(E) == 8 && plan.vec2) {
    auto kv = pow2 ? permute_tiled_vec2_kernel<true> : permute_tiled_vec2_kernel<false>;
    static thread_local bool attr_v[2] = {false, false};
    if (!attr_v[pow2]) {
      cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      attr_v[pow2] = true;
    }
    kv<<<plan.grid, kThreads, plan.smem, s>>>((const float4 *)src, (float4 *)dst, plan.tp,
                                              plan.d64, plan.d32);
    return check_launch("permute_tiled_vec2");
  }
  auto kern = pow2 ? permute_tiled_kernel<E, true> : permute_tiled_kernel<E, false>;
  static thread_local bool attr_set[2] = {false, false};
  if (!attr_set[pow2]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set[pow2] = true;
  }
  kern<<<plan.grid, kThreads, plan.smem, s>>>((const E *)src, (E *)dst, plan.tp, plan.d64,
                                              plan.d32);
  return check_launch("permute_tiled");
}

}  // namespace qf

extern "C" {

int qf_permute(const void *src, void *dst, int rank, const int64_t *dims, const int32_t *perm,
               int elem_bytes, void *stream) {
  std::shared_ptr<qf::PermPlan> plan;
  int st = qf::get_plan(rank, dims, perm, elem_bytes, plan, qf::as_stream(stream));
  if (st != QF_OK) return st;
  if (plan->n == 0) return QF_OK;
  QF_REQUIRE(src != dst, "permute: src and dst must not alias");
  cudaStream_t s = qf::as_stream(stream);
  if (elem_bytes == 8) return qf::launch<float2>(*plan, src, dst, s);
  return qf::launch<double2>(*plan, src, dst, s);
}

int qf_permute_c64(const void *src, void *dst, int rank, const int64_t *dims, const int32_t *perm,
                   void *stream) {
  return qf_permute(src, dst, rank, dims, perm, 8, stream);
}

}  // extern "C"

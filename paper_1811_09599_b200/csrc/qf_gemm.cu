// K3 -- complex GEMM on the fp32 (or fp64) SIMT pipes, and the dispatcher
// behind qf_cgemm_c64 / qf_zgemm_c128.
//
// Replaces `arr_a.reshape(m, k) @ arr_b.reshape(k, n)` at
// rq/tensor_core.py:417 (numpy -> OpenBLAS cgemm).  Strided-batched,
// row-major, both operands in N or T layout so callers can skip operand
// permutations whenever the shared labels are already a prefix/suffix.
//
// Two kernels:
//   * tiled   : 64x64 complex tile, 4x4 complex outputs per thread,
//               register-prefetched double buffer through smem.
//   * skinny  : M*N <= 256 outputs (dot products, GEMVs against a few
//               columns -- the `result` steps of every plan): K split over
//               CTAs, deterministic two-pass reduction through a
//               stream-ordered workspace.  HBM-bound by design.
// K2 (tcgen05 3xTF32) lives in qf_gemm_tc.cu; QF_GEMM_AUTO routes there
// when the shape fills tensor-core tiles.
#include <algorithm>

#include "qf_common.cuh"

namespace qf {

template <typename R>
struct C2;
template <>
struct C2<float> {
  using T = float2;
};
template <>
struct C2<double> {
  using T = double2;
};

template <typename V>
__device__ __forceinline__ void cfma(V &acc, const V &a, const V &b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// (tried: complex64 via two packed FFMA2 (fma.rn.f32x2) per complex MAC --
// bit-identical but measured slower on every CUDA-core engine, e.g. the
// config-2 1024 x (4096 x 8 x 64) row-stream GEMM 0.539 -> 0.607 ms)


// ---------------------------------------------------------------------------
// tiled SIMT kernel

constexpr int TBM = 64, TBN = 64, TTHREADS = 256;
template <typename R>
struct TileK {
  static constexpr int v = 16;
};
template <>
struct TileK<double> {
  static constexpr int v = 8;
};

template <typename R>
__global__ void __launch_bounds__(TTHREADS, 2)
    cgemm_tiled_kernel(const __grid_constant__ GemmArgs g, int64_t tiles_n, int64_t tiles) {
  using V = typename C2<R>::T;
  constexpr int TBK = TileK<R>::v;
  constexpr int NLD = TBM * TBK / TTHREADS;
  __shared__ V As[2][TBK][TBM + 1];
  __shared__ V Bs[2][TBK][TBN + 1];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const V *Ab = (const V *)g.A;
  const V *Bb = (const V *)g.B;
  V *Cb = (V *)g.C;
  const V zero = {R(0), R(0)};
  const R ar = (R)g.ar, ai = (R)g.ai, br = (R)g.br, bi = (R)g.bi;
  const bool use_beta = (br != R(0) || bi != R(0));

  for (int64_t work = blockIdx.x; work < tiles * g.batch; work += gridDim.x) {
    int64_t b = work / tiles;
    int64_t tile = work - b * tiles;
    int64_t m0 = (tile / tiles_n) * TBM, n0 = (tile % tiles_n) * TBN;
    const V *A = Ab + a_batch_off(g, b);
    const V *B = Bb + b_batch_off(g, b);
    V *C = Cb + b * g.sC;

    V acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = zero;

    V ra[NLD], rb[NLD];
    auto load = [&](int64_t k0) {
#pragma unroll
      for (int r = 0; r < NLD; ++r) {
        int l = tid + TTHREADS * r;
        int m, k;
        if (g.opA == QF_OP_N) {
          k = l % TBK;
          m = l / TBK;
        } else {
          m = l % TBM;
          k = l / TBM;
        }
        int64_t gm = m0 + m, gk = k0 + k;
        V v = zero;
        if (gm < g.M && gk < g.K) v = A[a_offset(g, gm, gk)];
        ra[r] = v;
        int n;
        if (g.opB == QF_OP_N) {
          n = l % TBN;
          k = l / TBN;
        } else {
          k = l % TBK;
          n = l / TBK;
        }
        int64_t gn = n0 + n;
        gk = k0 + k;
        V w = zero;
        if (gn < g.N && gk < g.K) w = (g.opB == QF_OP_N) ? B[gk * g.ldb + gn] : B[gn * g.ldb + gk];
        rb[r] = w;
      }
    };
    auto store = [&](int buf) {
#pragma unroll
      for (int r = 0; r < NLD; ++r) {
        int l = tid + TTHREADS * r;
        int m, k, n, kb;
        if (g.opA == QF_OP_N) {
          k = l % TBK;
          m = l / TBK;
        } else {
          m = l % TBM;
          k = l / TBM;
        }
        As[buf][k][m] = ra[r];
        if (g.opB == QF_OP_N) {
          n = l % TBN;
          kb = l / TBN;
        } else {
          kb = l % TBK;
          n = l / TBK;
        }
        Bs[buf][kb][n] = rb[r];
      }
    };

    int64_t nk = (g.K + TBK - 1) / TBK;
    __syncthreads();  // previous work item finished reading smem
    if (nk > 0) {
      load(0);
      store(0);
    }
    __syncthreads();
    for (int64_t kt = 0; kt < nk; ++kt) {
      int buf = kt & 1;
      if (kt + 1 < nk) load((kt + 1) * TBK);
#pragma unroll
      for (int k = 0; k < TBK; ++k) {
        V a[4], bb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[buf][k][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bb[j] = Bs[buf][k][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) cfma(acc[i][j], a[i], bb[j]);
      }
      if (kt + 1 < nk) store(buf ^ 1);
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int64_t gm = m0 + ty + 16 * i;
      if (gm >= g.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int64_t gn = n0 + tx + 16 * j;
        if (gn >= g.N) continue;
        V v = acc[i][j];
        V o;
        o.x = ar * v.x - ai * v.y;
        o.y = ar * v.y + ai * v.x;
        if (use_beta) {
          V c = C[gm * g.ldc + gn];
          o.x += br * c.x - bi * c.y;
          o.y += br * c.y + bi * c.x;
        }
        C[gm * g.ldc + gn] = o;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// skinny split-K kernel: M*N <= 256 outputs

constexpr int STHREADS = 256;

template <typename R>
__global__ void __launch_bounds__(STHREADS)
    cgemm_skinny_kernel(const __grid_constant__ GemmArgs g, int P, int Ppad, int64_t kchunk,
                        int nsplit, void *ws) {
  using V = typename C2<R>::T;
  __shared__ V red[STHREADS];
  const int tid = threadIdx.x;
  const int KL = STHREADS / Ppad;
  const int p = tid % Ppad, kl = tid / Ppad;
  const int64_t split = blockIdx.x;
  const int64_t b = blockIdx.y;
  const V *A = (const V *)g.A + a_batch_off(g, b);
  const V *B = (const V *)g.B + b_batch_off(g, b);
  V acc = {R(0), R(0)};
  if (p < P) {
    int64_t m = p / g.N, n = p % g.N;
    int64_t k0 = split * kchunk, k1 = min(g.K, k0 + kchunk);
    // gathered A: the K offsets come from a table; otherwise a fixed stride
    const bool gat = g.a_roff != nullptr;
    const V *ap = gat ? A + g.a_roff[m] : ((g.opA == QF_OP_N) ? A + m * g.lda : A + m);
    int64_t as = (g.opA == QF_OP_N) ? 1 : g.lda;
    const V *bp = (g.opB == QF_OP_N) ? B + n : B + n * g.ldb;
    int64_t bs = (g.opB == QF_OP_N) ? g.ldb : 1;
    int64_t k = k0 + kl;
    // 4-way unrolled for memory-level parallelism
    V acc2 = {R(0), R(0)};
    for (; !gat && k + 3 * KL < k1; k += 4 * KL) {
      V a0 = ap[k * as], a1 = ap[(k + KL) * as], a2 = ap[(k + 2 * KL) * as],
        a3 = ap[(k + 3 * KL) * as];
      V b0 = bp[k * bs], b1 = bp[(k + KL) * bs], b2 = bp[(k + 2 * KL) * bs],
        b3 = bp[(k + 3 * KL) * bs];
      cfma(acc, a0, b0);
      cfma(acc2, a1, b1);
      cfma(acc, a2, b2);
      cfma(acc2, a3, b3);
    }
    for (; k < k1; k += KL) cfma(acc, gat ? ap[g.a_coff[k]] : ap[k * as], bp[k * bs]);
    acc.x += acc2.x;
    acc.y += acc2.y;
  }
  red[tid] = acc;
  __syncthreads();
  for (int s = KL / 2; s >= 1; s >>= 1) {
    if (kl < s) {
      V o = red[tid + s * Ppad];
      red[tid].x += o.x;
      red[tid].y += o.y;
    }
    __syncthreads();
  }
  if (kl == 0 && p < P) ((V *)ws)[(b * nsplit + split) * P + p] = red[tid];
}

// Row-contiguous A (opA N) with many outputs: the mapping above puts the
// output index on consecutive lanes, i.e. every lane in a different row (one
// sector per lane).  Here a warp owns one row m at a time and its lanes walk
// k with 16-byte loads (whole 512-byte runs per request); the N <= 4 columns
// of B are read alongside.  Same workspace layout and second pass.
template <int NC>
__global__ void __launch_bounds__(STHREADS)
    cgemm_skinny_rows_kernel(const __grid_constant__ GemmArgs g, int64_t kchunk, int nsplit,
                             void *ws) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t split = blockIdx.x, b = blockIdx.y;
  const float2 *A = (const float2 *)g.A + a_batch_off(g, b);
  const float2 *B = (const float2 *)g.B + b_batch_off(g, b);
  const int64_t k0 = split * kchunk, k1 = min(g.K, k0 + kchunk);
  const int N = (int)g.N;
  const bool vec = g.lda % 2 == 0 && g.sA % 2 == 0 && k0 % 2 == 0 && !g.a_boff &&
                   ((reinterpret_cast<uintptr_t>(g.A) & 15) == 0);
  for (int64_t m = warp; m < g.M; m += STHREADS / 32) {
    const float2 *ap = A + m * g.lda;
    float2 acc[NC], acc2[NC];
#pragma unroll
    for (int n = 0; n < NC; ++n) acc[n] = acc2[n] = make_float2(0.f, 0.f);
    auto bval = [&](int64_t k, int n) {
      return g.opB == QF_OP_N ? __ldg(B + k * g.ldb + n) : __ldg(B + (int64_t)n * g.ldb + k);
    };
    int64_t k = k0 + 2 * lane;
    if (vec) {
      // four 16-byte loads in flight per lane
      for (; k + 193 < k1; k += 256) {
        float4 a4[4];
        float2 b4[4][2][NC];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a4[u] = __ldg(reinterpret_cast<const float4 *>(ap + k + 64 * u));
#pragma unroll
          for (int n = 0; n < NC; ++n) {
            if (n < N) {
              b4[u][0][n] = bval(k + 64 * u, n);
              b4[u][1][n] = bval(k + 64 * u + 1, n);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int n = 0; n < NC; ++n)
            if (n < N) {
              cfma(acc[n], make_float2(a4[u].x, a4[u].y), b4[u][0][n]);
              cfma(acc2[n], make_float2(a4[u].z, a4[u].w), b4[u][1][n]);
            }
      }
      for (; k + 1 < k1; k += 64) {
        const float4 a2 = __ldg(reinterpret_cast<const float4 *>(ap + k));
#pragma unroll
        for (int n = 0; n < NC; ++n) {
          if (n < N) {
            cfma(acc[n], make_float2(a2.x, a2.y), bval(k, n));
            cfma(acc2[n], make_float2(a2.z, a2.w), bval(k + 1, n));
          }
        }
      }
      if (k < k1) {
#pragma unroll
        for (int n = 0; n < NC; ++n)
          if (n < N) cfma(acc[n], __ldg(ap + k), bval(k, n));
      }
    } else {
      for (k = k0 + lane; k < k1; k += 32) {
        const float2 a = __ldg(ap + k);
#pragma unroll
        for (int n = 0; n < NC; ++n)
          if (n < N) cfma(acc[n], a, bval(k, n));
      }
    }
#pragma unroll
    for (int n = 0; n < NC; ++n) {
      float x = acc[n].x + acc2[n].x, y = acc[n].y + acc2[n].y;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        x += __shfl_xor_sync(0xffffffffu, x, o);
        y += __shfl_xor_sync(0xffffffffu, y, o);
      }
      if (lane == 0 && n < N)
        ((float2 *)ws)[(b * nsplit + split) * (g.M * N) + m * N + n] = make_float2(x, y);
    }
  }
}

template <typename R>
__global__ void cgemm_skinny_reduce(const __grid_constant__ GemmArgs g, int P, int nsplit,
                                    const void *ws) {
  using V = typename C2<R>::T;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= g.batch * P) return;
  int64_t b = t / P;
  int p = (int)(t - b * P);
  const V *w = (const V *)ws + b * nsplit * P + p;
  R sx = 0, sy = 0;
  for (int s = 0; s < nsplit; ++s) {
    V v = w[(int64_t)s * P];
    sx += v.x;
    sy += v.y;
  }
  int64_t m = p / g.N, n = p % g.N;
  V *C = (V *)g.C + b * g.sC + m * g.ldc + n;
  R ar = (R)g.ar, ai = (R)g.ai, br = (R)g.br, bi = (R)g.bi;
  V o;
  o.x = ar * sx - ai * sy;
  o.y = ar * sy + ai * sx;
  if (br != R(0) || bi != R(0)) {
    V c = *C;
    o.x += br * c.x - bi * c.y;
    o.y += br * c.y + bi * c.x;
  }
  *C = o;
}

// ---------------------------------------------------------------------------
// small-KxN streaming kernel: K*N <= SKN_MAX complex (B[b] fits in smem).
// The memory-bound shapes of region growth -- GEMVs against a cut-sliced
// site (n = 1), k = 8 / n = 8 bond contractions -- stream A once, coalesced,
// through shared memory and write C rows coalesced; B[b] is staged once per
// work item.  One work item = (batch entry, block of rows).

constexpr int SKN_THREADS = 256;
constexpr int SKN_MAX = 4096;      // complex entries of B held in smem
constexpr int SKN_A_MAX = 4096;    // complex entries of the staged A block

__device__ __forceinline__ void skn_cp_async(void *smem_dst, const void *gsrc, int bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}

// Pipelined: each CTA owns a contiguous range of work items (batch-major, so
// B[b] is restaged rarely); the A block of item j+1 streams into the other
// smem buffer with cp.async while item j is computed and written.
template <typename R, int NG>
__global__ void __launch_bounds__(SKN_THREADS)
    cgemm_smallkn_kernel(const __grid_constant__ GemmArgs g, int rm, int64_t blocks_m,
                         int apitch, int bpitch, int64_t items_per_cta) {
  using V = typename C2<R>::T;
  extern __shared__ __align__(16) unsigned char skn_smem[];
  const int K = (int)g.K, N = (int)g.N;
  V *Bs = reinterpret_cast<V *>(skn_smem);
  V *As0 = Bs + (((size_t)K * bpitch + 1) & ~(size_t)1);
  V *Asb[2] = {As0, As0 + (size_t)rm * apitch};
  const int tid = threadIdx.x;
  const R ar = (R)g.ar, ai = (R)g.ai, br = (R)g.br, bi = (R)g.bi;
  const bool use_beta = (br != R(0) || bi != R(0));
  const int64_t total = g.batch * blocks_m;
  const int64_t it0 = blockIdx.x * items_per_cta;
  const int64_t it1 = min(total, it0 + items_per_cta);
  if (it0 >= it1) return;
  // 16-byte copies when rows are contiguous K-runs of even length (pairs stay in a row)
  const bool vec = sizeof(V) == 8 && g.opA == QF_OP_N && (K % 2 == 0) && (g.lda % 2 == 0) &&
                   (g.sA % 2 == 0) && (apitch % 2 == 0);

  auto issue = [&](int64_t item, int buf) {
    const int64_t b = item / blocks_m;
    const int64_t m0 = (item - b * blocks_m) * rm;
    const int rows = (int)min((int64_t)rm, g.M - m0);
    const V *A = reinterpret_cast<const V *>(g.A) + a_batch_off(g, b);
    V *As = Asb[buf];
    if (g.a_roff) {
      // walk the index group that holds A's stride-1 label fastest (coalesced)
      const bool m_fast = rows > 1 && g.a_roff[m0 + 1] - g.a_roff[m0] == 1;
      for (int i = tid; i < rows * K; i += SKN_THREADS) {
        int m, k;
        if (m_fast) {
          k = i / rows;
          m = i - k * rows;
        } else {
          m = i / K;
          k = i - m * K;
        }
        skn_cp_async(As + m * apitch + k, A + g.a_roff[m0 + m] + g.a_coff[k], sizeof(V));
      }
    } else if (vec) {
      const int pairs = rows * (K / 2);
      for (int i = tid; i < pairs; i += SKN_THREADS) {
        const int m = i / (K / 2), k = (i - m * (K / 2)) * 2;
        skn_cp_async(As + m * apitch + k, A + (m0 + m) * g.lda + k, 16);
      }
    } else if (g.opA == QF_OP_N) {
      for (int i = tid; i < rows * K; i += SKN_THREADS) {
        const int m = i / K, k = i - m * K;
        skn_cp_async(As + m * apitch + k, A + (m0 + m) * g.lda + k, sizeof(V));
      }
    } else {
      for (int i = tid; i < rows * K; i += SKN_THREADS) {
        const int k = i / rows, m = i - k * rows;
        skn_cp_async(As + m * apitch + k, A + (int64_t)k * g.lda + m0 + m, sizeof(V));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto stage_b = [&](int64_t b) {
    const V *B = reinterpret_cast<const V *>(g.B) + b_batch_off(g, b);
    for (int i = tid; i < K * N; i += SKN_THREADS) {
      int k, n;
      if (g.opB == QF_OP_N) {
        k = i / N;
        n = i - k * N;
        Bs[k * bpitch + n] = B[(int64_t)k * g.ldb + n];
      } else {
        n = i / K;
        k = i - n * K;
        Bs[k * bpitch + n] = B[(int64_t)n * g.ldb + k];
      }
    }
  };

  int64_t cur_b = it0 / blocks_m;
  stage_b(cur_b);
  issue(it0, 0);
  for (int64_t item = it0; item < it1; ++item) {
    const int buf = (int)((item - it0) & 1);
    const int64_t b = item / blocks_m;
    const int64_t m0 = (item - b * blocks_m) * rm;
    const int rows = (int)min((int64_t)rm, g.M - m0);
    if (item + 1 < it1 && (item + 1) / blocks_m == b) {
      issue(item + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // A block (and B stage) visible to every thread
    const V *As = Asb[buf];
    V *C = reinterpret_cast<V *>(g.C) + b * g.sC;
    // register blocking: a thread computes NG consecutive columns of one row,
    // reading its A row once; B reads are warp-wide broadcasts
    const int groups = (N + NG - 1) / NG;
    for (int o = tid; o < rows * groups; o += SKN_THREADS) {
      const int m = o / groups, n0 = (o - m * groups) * NG;
      V acc[NG];
#pragma unroll
      for (int j = 0; j < NG; ++j) acc[j] = V{R(0), R(0)};
      const V *arow = As + m * apitch;
      const V *bcol = Bs + n0;
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        const V a = arow[k];
#pragma unroll
        for (int j = 0; j < NG; ++j)
          if (n0 + j < N) cfma(acc[j], a, bcol[k * bpitch + j]);
      }
      V *cp = C + (m0 + m) * g.ldc + n0;
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        if (n0 + j < N) {
          V out;
          out.x = ar * acc[j].x - ai * acc[j].y;
          out.y = ar * acc[j].y + ai * acc[j].x;
          if (use_beta) {
            const V c = cp[j];
            out.x += br * c.x - bi * c.y;
            out.y += br * c.y + bi * c.x;
          }
          cp[j] = out;
        }
      }
    }
    __syncthreads();  // buffer `buf` and Bs free
    if (item + 1 < it1 && (item + 1) / blocks_m != b) {  // next batch entry: restage B, refill
      cur_b = (item + 1) / blocks_m;
      stage_b(cur_b);
      issue(item + 1, buf ^ 1);
    }
  }
}

// single-buffer twin for short K (<= 16): more CTAs per SM beat pipelining
template <typename R>
__global__ void __launch_bounds__(SKN_THREADS)
    cgemm_smallkn_simple_kernel(const __grid_constant__ GemmArgs g, int rm, int64_t blocks_m) {
  using V = typename C2<R>::T;
  extern __shared__ __align__(16) unsigned char skn_smem[];
  const int K = (int)g.K, N = (int)g.N;
  const int bpitch = N + ((N % 2 == 0) ? 1 : 0);
  const int apitch = K + ((K % 2 == 0) ? 1 : 0);
  V *Bs = reinterpret_cast<V *>(skn_smem);
  V *As = Bs + (size_t)K * bpitch;
  const int tid = threadIdx.x;
  const R ar = (R)g.ar, ai = (R)g.ai, br = (R)g.br, bi = (R)g.bi;
  const bool use_beta = (br != R(0) || bi != R(0));
  int64_t cur_b = -1;
  for (int64_t item = blockIdx.x; item < g.batch * blocks_m; item += gridDim.x) {
    const int64_t b = item / blocks_m;
    const int64_t m0 = (item - b * blocks_m) * rm;
    const int rows = (int)min((int64_t)rm, g.M - m0);
    __syncthreads();  // previous item done with smem
    if (b != cur_b) {
      const V *B = reinterpret_cast<const V *>(g.B) + b_batch_off(g, b);
      for (int i = tid; i < K * N; i += SKN_THREADS) {
        int k, n;
        if (g.opB == QF_OP_N) {
          k = i / N;
          n = i - k * N;
          Bs[k * bpitch + n] = B[(int64_t)k * g.ldb + n];
        } else {
          n = i / K;
          k = i - n * K;
          Bs[k * bpitch + n] = B[(int64_t)n * g.ldb + k];
        }
      }
      cur_b = b;
    }
    const V *A = reinterpret_cast<const V *>(g.A) + a_batch_off(g, b);
    for (int i = tid; i < rows * K; i += SKN_THREADS) {
      int m, k;
      if (g.a_roff) {
        if (rows > 1 && g.a_roff[m0 + 1] - g.a_roff[m0] == 1) {  // stride-1 label is a row label
          k = i / rows;
          m = i - k * rows;
        } else {
          m = i / K;
          k = i - m * K;
        }
        As[m * apitch + k] = A[g.a_roff[m0 + m] + g.a_coff[k]];
      } else if (g.opA == QF_OP_N) {
        m = i / K;
        k = i - m * K;
        As[m * apitch + k] = A[(m0 + m) * g.lda + k];
      } else {
        k = i / rows;
        m = i - k * rows;
        As[m * apitch + k] = A[(int64_t)k * g.lda + m0 + m];
      }
    }
    __syncthreads();
    V *C = reinterpret_cast<V *>(g.C) + b * g.sC;
    for (int o = tid; o < rows * N; o += SKN_THREADS) {
      const int m = o / N, n = o - m * N;
      V acc = {R(0), R(0)};
      const V *arow = As + m * apitch;
#pragma unroll 8
      for (int k = 0; k < K; ++k) cfma(acc, arow[k], Bs[k * bpitch + n]);
      V out;
      out.x = ar * acc.x - ai * acc.y;
      out.y = ar * acc.y + ai * acc.x;
      V *cp = C + (m0 + m) * g.ldc + n;
      if (use_beta) {
        const V c = *cp;
        out.x += br * c.x - bi * c.y;
        out.y += br * c.y + bi * c.x;
      }
      *cp = out;
    }
  }
}


// ---------------------------------------------------------------------------
// row-block streaming kernel for the small K x N shapes (K*N <= 4096 and one
// of K, N <= 16): B[b] is staged in smem once per batch entry; each thread
// owns (row, group of 8 output columns) and streams its A row in chunks of 8
// k straight into registers (N, T or gathered layout), so every A byte is
// read once with no shared-memory round trip and C is written with 16-byte
// stores.  A CTA walks a contiguous range of (batch, row-block) items.

constexpr int RB_THREADS = 256;
constexpr int RB_NG = 8;

template <typename R>
__global__ void __launch_bounds__(RB_THREADS)
    cgemm_rowblock_kernel(const __grid_constant__ GemmArgs g, int rows_per_item,
                          int64_t items_per_b, int64_t items_per_cta) {
  using V = typename C2<R>::T;
  extern __shared__ __align__(16) unsigned char rb_smem[];
  V *Bs = reinterpret_cast<V *>(rb_smem);
  const int K = (int)g.K, N = (int)g.N;
  int32_t *s_coff = reinterpret_cast<int32_t *>(Bs + (size_t)K * N);  // gathered-A k offsets
  if (g.a_roff) {
    for (int i = threadIdx.x; i < K; i += RB_THREADS) s_coff[i] = g.a_coff[i];
    __syncthreads();
  }
  // full 8-column groups of an even-N B read as 16-byte pairs
  const bool vec_b = sizeof(V) == 8 && N % 2 == 0;
  const int groups = (N + RB_NG - 1) / RB_NG;
  const int tid = threadIdx.x;
  const R ar = (R)g.ar, ai = (R)g.ai, br = (R)g.br, bi = (R)g.bi;
  const bool use_beta = (br != R(0) || bi != R(0));
  const int64_t total = g.batch * items_per_b;
  const int64_t it0 = blockIdx.x * items_per_cta, it1 = min(total, it0 + items_per_cta);
  const bool vec_a = sizeof(V) == 8 && !g.a_roff && g.opA == QF_OP_N && g.lda % 2 == 0 &&
                     g.sA % 2 == 0;
  int64_t cur_b = -1;
  for (int64_t item = it0; item < it1; ++item) {
    const int64_t b = item / items_per_b;
    const int64_t r0 = (item - b * items_per_b) * rows_per_item;
    const int rows = (int)min((int64_t)rows_per_item, g.M - r0);
    if (b != cur_b) {
      __syncthreads();
      const V *B = reinterpret_cast<const V *>(g.B) + b_batch_off(g, b);
      for (int i = tid; i < K * N; i += RB_THREADS) {
        int k, n;
        if (g.opB == QF_OP_N) {
          k = i / N;
          n = i - k * N;
          Bs[k * N + n] = B[(int64_t)k * g.ldb + n];
        } else {
          n = i / K;
          k = i - n * K;
          Bs[k * N + n] = B[(int64_t)n * g.ldb + k];
        }
      }
      cur_b = b;
      __syncthreads();
    }
    const V *A = reinterpret_cast<const V *>(g.A) + a_batch_off(g, b);
    V *C = reinterpret_cast<V *>(g.C) + b * g.sC;
    for (int task = tid; task < rows * groups; task += RB_THREADS) {
      const int r = task / groups, cg = task - r * groups;
      const int64_t row = r0 + r;
      const int n0 = cg * RB_NG;
      V acc[RB_NG];
#pragma unroll
      for (int j = 0; j < RB_NG; ++j) acc[j] = V{R(0), R(0)};
      const V *arow = g.a_roff ? A + g.a_roff[row]
                               : (g.opA == QF_OP_N ? A + row * g.lda : A + a_row_base(g, row));
      // software pipeline: the next 8 k of A are in flight while this 8 is used
      auto load8 = [&](int k0, V *a) {
        if (vec_a && k0 + 8 <= K) {  // row-major A: four 16-byte loads per 8 k
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(arow + k0 + j));
            a[j] = V{(R)v.x, (R)v.y};
            a[j + 1] = V{(R)v.z, (R)v.w};
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = k0 + j;
            a[j] = V{R(0), R(0)};
            if (k < K)
              a[j] = g.a_roff ? __ldg(arow + s_coff[k])
                              : (g.opA == QF_OP_N ? __ldg(arow + k) : __ldg(arow + (int64_t)k * g.lda));
          }
        }
      };
      V a_nx[8];
      load8(0, a_nx);
      for (int k0 = 0; k0 < K; k0 += 8) {
        V a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = a_nx[j];
        if (k0 + 8 < K) load8(k0 + 8, a_nx);
        if (vec_b && n0 + RB_NG <= N) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (k0 + j < K) {
              const float4 *bk = reinterpret_cast<const float4 *>(Bs + (k0 + j) * N + n0);
#pragma unroll
              for (int c = 0; c < RB_NG; c += 2) {
                const float4 bv = bk[c / 2];
                cfma(acc[c], a[j], V{(R)bv.x, (R)bv.y});
                cfma(acc[c + 1], a[j], V{(R)bv.z, (R)bv.w});
              }
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (k0 + j < K) {
              const V *bk = Bs + (k0 + j) * N + n0;
#pragma unroll
              for (int c = 0; c < RB_NG; ++c)
                if (n0 + c < N) cfma(acc[c], a[j], bk[c]);
            }
          }
        }
      }
      // row-major C: this row's columns; transposed C: column c, row `row`
      // (consecutive threads write consecutive rows)
      V *cp = g.c_trans ? C + (int64_t)n0 * g.ldc + row : C + row * g.ldc + n0;
      const int64_t cstep = g.c_trans ? g.ldc : 1;
#pragma unroll
      for (int c = 0; c < RB_NG; ++c) {
        if (n0 + c < N) {
          V o;
          o.x = ar * acc[c].x - ai * acc[c].y;
          o.y = ar * acc[c].y + ai * acc[c].x;
          if (use_beta) {
            const V cv = cp[c * cstep];
            o.x += br * cv.x - bi * cv.y;
            o.y += br * cv.y + bi * cv.x;
          }
          cp[c * cstep] = o;
        }
      }
    }
  }
}

// Rows per work item so that a small batch (the open-output steps run
// single GEMMs) still spreads over >= 2 items per SM; never below `floor`.
static int64_t rows_for_parallelism(const GemmArgs &g, int64_t floor) {
  const int64_t per_b = std::max<int64_t>(1, (2 * (int64_t)sm_count() + g.batch - 1) / g.batch);
  return std::max<int64_t>(floor, (g.M + per_b - 1) / per_b);
}

template <typename R>
int gemm_rowblock(const GemmArgs &g, cudaStream_t s) {
  using V = typename C2<R>::T;
  const int groups = (int)((g.N + RB_NG - 1) / RB_NG);
  // ~8 row-groups of work per thread per item; items fill the machine
  int rows_per_item = (int)std::max<int64_t>(1, std::min<int64_t>(g.M, 8 * RB_THREADS / groups));
  rows_per_item = (int)std::min<int64_t>(rows_per_item, rows_for_parallelism(g, 32));
  const int64_t items_per_b = (g.M + rows_per_item - 1) / rows_per_item;
  const int64_t items = g.batch * items_per_b;
  const int64_t ctas = std::min<int64_t>(items, (int64_t)sm_count() * 8);
  const int64_t per_cta = (items + ctas - 1) / ctas;
  const int64_t grid = (items + per_cta - 1) / per_cta;
  const size_t smem = (size_t)g.K * g.N * sizeof(V) + (g.a_roff ? (size_t)g.K * 4 : 0);
  auto kern = cgemm_rowblock_kernel<R>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  kern<<<(unsigned)grid, RB_THREADS, smem, s>>>(g, rows_per_item, items_per_b, per_cta);
  return check_launch("cgemm_rowblock");
}

// ---------------------------------------------------------------------------
// row-stream kernel (complex64, N <= 16, K*N <= 1024): the narrow-output
// GEMMs of the amplitude batch (e.g. 1024 x (4096 x 8 x 64), 1024 x (32768 x
// 8 x 8)), which the row-block kernel reads one row per lane (32 sectors
// per request).  Here:
//   * a CTA (8 warps) walks a contiguous run of 256-row steps inside batch
//     entries; B[b] sits in CTA shared memory (reloaded at a batch change)
//     and is read as broadcasts;
//   * each warp owns 32 rows of a step and streams its A block in k-chunks
//     of KC through a private double-buffered cp.async ring, fetched along
//     the layout's contiguous direction (lanes along k: 16-byte requests for
//     row-major A, 8-byte for k-contiguous gathers; lane = row for
//     column-major A and row-contiguous gathers) -- whole sectors per request;
//   * lane = row, NN accumulators, chunk loop fully unrolled; the 32 x N
//     result goes through a staging tile so stores are whole row segments.

constexpr int RS_WARPS = 8;

__device__ __forceinline__ void rs_cp8(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void rs_cp16(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

template <int NN, int KC, bool MMA = false>
struct RsLayout {
  // staged A row: an odd multiple of 16 B (FFMA: lane = row reads whole
  // rows); 8 words mod 32 for the MMA fragments (lanes 4 rows x 4 k apart)
  static constexpr int APITCH = MMA ? KC * 8 + 32 : KC * 8 + 16;
  static constexpr int OPITCH = NN * 8 + 16;          // staged C row
  static constexpr int ABUF = 32 * APITCH;
  static constexpr int NSLOT = MMA ? 3 : 2;           // A ring depth per warp
  static constexpr int WARP = NSLOT * ABUF + 32 * OPITCH;  // per warp: A ring + C staging
  // B[b]: complex K x NN (FFMA) or TF32 hi/lo fragments (MMA: per 4 k and
  // 4 columns one float4 per lane, K <= KMAX_MMA)
  static constexpr int KMAX_MMA = 64;
  static constexpr int BBYTES = MMA ? (KMAX_MMA / 4) * (NN / 4) * 32 * 16 : 1024 * 8;
  static constexpr int SMEM = BBYTES + RS_WARPS * WARP;
};

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NN, int KC, bool MMA = false>
__global__ void __launch_bounds__(RS_WARPS * 32)
    cgemm_rowstream_kernel(const __grid_constant__ GemmArgs g, int64_t steps_per_b,
                           int64_t steps_per_cta) {
  using L = RsLayout<NN, KC, MMA>;
  extern __shared__ __align__(16) unsigned char rs_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2 *Bs = reinterpret_cast<float2 *>(rs_smem);
  unsigned char *wsm = rs_smem + L::BBYTES + warp * L::WARP;
  unsigned char *Ost = wsm + L::NSLOT * L::ABUF;
  const uint32_t abuf_u32 = static_cast<uint32_t>(__cvta_generic_to_shared(wsm));
  const int K = (int)g.K, N = (int)g.N;
  const int nch = (K + KC - 1) / KC;
  const int64_t total = g.batch * steps_per_b;
  const int64_t st0 = blockIdx.x * steps_per_cta, st1 = min(total, st0 + steps_per_cta);
  const float2 *Ab = reinterpret_cast<const float2 *>(g.A);
  const bool gat = g.a_roff != nullptr;
  const bool rows_contig = gat && g.M > 1 && __ldg(g.a_roff + 1) - __ldg(g.a_roff) == 1;
  // 0: lane = row (column-major A, row-contiguous gather); 1: lanes along k,
  // 16 B (row-major A, even lda); 2: lanes along k, 8 B (other row-major / gathers)
  const int mode = gat ? (rows_contig ? 0 : 2)
                       : (g.opA == QF_OP_T ? 0 : ((g.lda % 2 == 0 && g.sA % 2 == 0) ? 1 : 2));

  // ---- fetch cursor over (step, chunk); (batch, row) advance incrementally
  // (no 64-bit division per chunk)
  int64_t f_st = st0;
  int f_ch = 0;
  int64_t f_b = st0 / steps_per_b;
  int64_t f_r0 = (st0 - f_b * steps_per_b) * (RS_WARPS * 32) + warp * 32;
  const int64_t r_end = steps_per_b * (RS_WARPS * 32);
  const float2 *f_A = Ab + a_batch_off(g, f_b);
  int32_t f_roff = 0;  // gathered: row offset of row `lane` of this warp's 32
  auto load_roff = [&]() {
    if (!gat || f_st >= st1) return;
    f_roff = __ldg(g.a_roff + min(f_r0 + lane, g.M - 1));
  };
  auto fetch = [&](int slot) {
    if (f_st < st1) {
      const int64_t r0 = f_r0;
      const float2 *A = f_A;
      const int k0 = f_ch * KC;
      const uint32_t dst0 = abuf_u32 + slot * L::ABUF;
      if (mode == 0) {
        const bool rok = r0 + lane < g.M;
        const int64_t f_rbase = a_row_base(g, r0);   // 32 rows never straddle a row block
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const bool ok = rok && k0 + k < K;
          const float2 *src = gat ? A + f_roff + (ok ? __ldg(g.a_coff + k0 + k) : 0)
                                  : A + (int64_t)(ok ? k0 + k : 0) * g.lda + f_rbase + lane;
          rs_cp8(dst0 + lane * L::APITCH + k * 8, ok ? src : Ab, ok);
        }
      } else if (mode == 1) {
        constexpr int LPR = KC / 2, RPI = 32 / LPR;  // lanes per row (16 B each), rows per request
        const int kk = 2 * (lane % LPR), rr = lane / LPR;
        const bool kok = k0 + kk + 1 < K;  // K even on this path when lda is even? keep exact
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i) {
          const int row = RPI * i + rr;
          const bool rok = r0 + row < g.M;
          const float2 *src = A + (r0 + row) * g.lda + k0 + kk;
          if (kok) {
            rs_cp16(dst0 + row * L::APITCH + kk * 8, rok ? src : Ab, rok);
          } else {
            rs_cp8(dst0 + row * L::APITCH + kk * 8, (rok && k0 + kk < K) ? src : Ab,
                   rok && k0 + kk < K);
            rs_cp8(dst0 + row * L::APITCH + kk * 8 + 8, Ab, false);
          }
        }
      } else {
        constexpr int RPI = 32 / KC;  // lanes along k (8 B each)
        const int kk = lane % KC, rr = lane / KC;
        const bool kok = k0 + kk < K;
        const int32_t c = (gat && kok) ? __ldg(g.a_coff + k0 + kk) : 0;
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i) {
          const int row = RPI * i + rr;
          const bool ok = kok && r0 + row < g.M;
          const float2 *src;
          if (gat) {
            const int32_t ro = __shfl_sync(0xffffffffu, f_roff, row);
            src = A + ro + c;
          } else {
            src = A + (r0 + row) * g.lda + k0 + kk;
          }
          rs_cp8(dst0 + row * L::APITCH + kk * 8, ok ? src : Ab, ok);
        }
      }
      if (++f_ch == nch) {
        f_ch = 0;
        ++f_st;
        f_r0 += RS_WARPS * 32;
        if (f_r0 >= r_end) {
          f_r0 -= r_end;
          ++f_b;
          if (f_st < st1) f_A = Ab + a_batch_off(g, f_b);
        }
        load_roff();
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  const float ar = (float)g.ar, ai = (float)g.ai, br_ = (float)g.br, bi_ = (float)g.bi;
  const bool use_beta = (br_ != 0.f || bi_ != 0.f);
  load_roff();
  fetch(0);
  if constexpr (MMA) {
    for (int i = 1; i < L::NSLOT - 1; ++i) fetch(i);
  }
  int64_t cur_b = -1;
  int q = 0;
  int64_t b = st0 / steps_per_b;
  int64_t r0 = (st0 - b * steps_per_b) * (RS_WARPS * 32) + warp * 32 - RS_WARPS * 32;
  for (int64_t st = st0; st < st1; ++st) {
    r0 += RS_WARPS * 32;
    if (r0 >= r_end) {
      r0 -= r_end;
      ++b;
    }
    if (b != cur_b) {  // CTA-uniform: every warp walks the same steps
      __syncthreads();
      const float2 *B = reinterpret_cast<const float2 *>(g.B) + b_batch_off(g, b);
      if constexpr (MMA) {
        // real form of the complex product, output columns interleaved
        // (re, im) and each 4-k step's 8 real rows ordered (Re A of k0..k3,
        // Im A of k0..k3): lane (gq = lane/4, t = lane%4) of fragment
        // (kstep, ntile) holds rows (Re A, Im A) of k = 4 kstep + t for real
        // column 8 ntile + gq -- {b0, b1} hi then lo, TF32
        const int nfr = nch * (KC / 4) * (NN / 4) * 32;
        float4 *Bf = reinterpret_cast<float4 *>(rs_smem);
        for (int i = threadIdx.x; i < nfr; i += RS_WARPS * 32) {
          const int ln = i & 31, fr = i >> 5;
          const int nt = fr % (NN / 4), ks = fr / (NN / 4);
          const int k = 4 * ks + (ln & 3), col = 8 * nt + (ln >> 2);
          const int n = col >> 1;
          float2 v = make_float2(0.f, 0.f);
          if (n < N && k < K)
            v = g.opB == QF_OP_N ? __ldg(B + (int64_t)k * g.ldb + n) : __ldg(B + (int64_t)n * g.ldb + k);
          // Re column: (Br, -Bi); Im column: (Bi, Br)
          const float b0 = (col & 1) ? v.y : v.x, b1 = (col & 1) ? v.x : -v.y;
          const uint32_t h0 = tf32_rna(b0), h1 = tf32_rna(b1);
          Bf[i] = make_float4(__uint_as_float(h0), __uint_as_float(h1),
                              b0 - __uint_as_float(h0), b1 - __uint_as_float(h1));
        }
      } else {
        for (int i = threadIdx.x; i < K * NN; i += RS_WARPS * 32) {
          const int k = i / NN, n = i - k * NN;
          float2 v = make_float2(0.f, 0.f);
          if (n < N)
            v = g.opB == QF_OP_N ? __ldg(B + (int64_t)k * g.ldb + n) : __ldg(B + (int64_t)n * g.ldb + k);
          Bs[i] = v;
        }
      }
      cur_b = b;
      __syncthreads();
    }
    float2 acc[NN];
#pragma unroll
    for (int n = 0; n < NN; ++n) acc[n] = make_float2(0.f, 0.f);
    if constexpr (MMA) {
      // 3xTF32 on the warp-level tensor-core path: the 32 rows are two
      // m16 tiles, each 4-k step one k8 of the real form
      float c[2][NN / 4][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NN / 4; ++nt)
#pragma unroll
          for (int j = 0; j < 4; ++j) c[mt][nt][j] = 0.f;
      const int gq = lane >> 2, t = lane & 3;
      const float4 *Bf = reinterpret_cast<const float4 *>(rs_smem);
      for (int ch = 0; ch < nch; ++ch, ++q) {
        fetch((q + L::NSLOT - 1) % L::NSLOT);   // NSLOT - 1 chunks in flight
        asm volatile("cp.async.wait_group %0;" ::"n"(L::NSLOT - 1) : "memory");
        __syncwarp();
        const unsigned char *abuf = wsm + (q % L::NSLOT) * L::ABUF;
#pragma unroll
        for (int ks = 0; ks < KC / 4; ++ks) {
          uint32_t ah[2][4], al[2][4];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const float2 lo = *reinterpret_cast<const float2 *>(
                abuf + (16 * mt + gq) * L::APITCH + (4 * ks + t) * 8);
            const float2 hi = *reinterpret_cast<const float2 *>(
                abuf + (16 * mt + gq + 8) * L::APITCH + (4 * ks + t) * 8);
            const float av[4] = {lo.x, hi.x, lo.y, hi.y};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              ah[mt][j] = tf32_rna(av[j]);
              al[mt][j] = __float_as_uint(av[j] - __uint_as_float(ah[mt][j]));
            }
          }
#pragma unroll
          for (int nt = 0; nt < NN / 4; ++nt) {
            const float4 bf = Bf[((ch * (KC / 4) + ks) * (NN / 4) + nt) * 32 + lane];
            const uint32_t bh0 = __float_as_uint(bf.x), bh1 = __float_as_uint(bf.y);
            const uint32_t bl0 = __float_as_uint(bf.z), bl1 = __float_as_uint(bf.w);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              mma_tf32(c[mt][nt], al[mt], bh0, bh1);
              mma_tf32(c[mt][nt], ah[mt], bl0, bl1);
              mma_tf32(c[mt][nt], ah[mt], bh0, bh1);
            }
          }
        }
        __syncwarp();  // the slot is refilled by a later fetch
      }
      // fragments -> staging rows (row = lane's C row) -> acc[] per lane
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NN / 4; ++nt) {
          *reinterpret_cast<float2 *>(Ost + (16 * mt + gq) * L::OPITCH + (4 * nt + t) * 8) =
              make_float2(c[mt][nt][0], c[mt][nt][1]);
          *reinterpret_cast<float2 *>(Ost + (16 * mt + gq + 8) * L::OPITCH + (4 * nt + t) * 8) =
              make_float2(c[mt][nt][2], c[mt][nt][3]);
        }
      __syncwarp();
#pragma unroll
      for (int n = 0; n < NN; ++n) acc[n] = *reinterpret_cast<const float2 *>(Ost + lane * L::OPITCH + n * 8);
      __syncwarp();
    } else
    for (int ch = 0; ch < nch; ++ch, ++q) {
      fetch((q + 1) & 1);  // next chunk (of this or the next step) into the other slot
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
      const unsigned char *arow = wsm + (q & 1) * L::ABUF + lane * L::APITCH;
      const float2 *bch = Bs + ch * KC * NN;
      const int kn = min(KC, K - ch * KC);
      if (kn == KC) {
#pragma unroll
        for (int k = 0; k < KC; k += 2) {
          const float4 a2 = *reinterpret_cast<const float4 *>(arow + k * 8);
          const float2 a0 = make_float2(a2.x, a2.y), a1 = make_float2(a2.z, a2.w);
#pragma unroll
          for (int n = 0; n < NN; n += 2) {
            const float4 b0 = *reinterpret_cast<const float4 *>(bch + k * NN + n);
            const float4 b1 = *reinterpret_cast<const float4 *>(bch + (k + 1) * NN + n);
            cfma(acc[n], a0, make_float2(b0.x, b0.y));
            cfma(acc[n + 1], a0, make_float2(b0.z, b0.w));
            cfma(acc[n], a1, make_float2(b1.x, b1.y));
            cfma(acc[n + 1], a1, make_float2(b1.z, b1.w));
          }
        }
      } else {
        for (int k = 0; k < kn; ++k) {
          const float2 a0 = *reinterpret_cast<const float2 *>(arow + k * 8);
#pragma unroll
          for (int n = 0; n < NN; ++n) cfma(acc[n], a0, bch[k * NN + n]);
        }
      }
      __syncwarp();  // the slot is refilled by the next fetch
    }
    // ---- epilogue
    float2 *C = reinterpret_cast<float2 *>(g.C) + b * g.sC;
    const int rows = (int)max((int64_t)0, min((int64_t)32, g.M - r0));
    if (g.c_trans) {  // transposed C: lane = row, one coalesced 256-byte run per column
      if (lane < rows) {
#pragma unroll
        for (int n = 0; n < NN; ++n) {
          if (n < N) {
            float2 *cp = C + (int64_t)n * g.ldc + r0 + lane;
            float2 o = make_float2(ar * acc[n].x - ai * acc[n].y, ar * acc[n].y + ai * acc[n].x);
            if (use_beta) {
              const float2 c = *cp;
              o.x += br_ * c.x - bi_ * c.y;
              o.y += br_ * c.y + bi_ * c.x;
            }
            *cp = o;
          }
        }
      }
    } else if (!use_beta && N == NN && g.ldc % 2 == 0 &&
        ((reinterpret_cast<uintptr_t>(C + r0 * g.ldc)) & 15) == 0) {
#pragma unroll
      for (int n = 0; n < NN; n += 2) {
        const float2 o0 = make_float2(ar * acc[n].x - ai * acc[n].y, ar * acc[n].y + ai * acc[n].x);
        const float2 o1 = make_float2(ar * acc[n + 1].x - ai * acc[n + 1].y,
                                      ar * acc[n + 1].y + ai * acc[n + 1].x);
        *reinterpret_cast<float4 *>(Ost + lane * L::OPITCH + n * 8) = make_float4(o0.x, o0.y, o1.x, o1.y);
      }
      __syncwarp();
      constexpr int LPR = NN / 2, RPI = 32 / LPR;
      const int rs = lane / LPR, cc = lane % LPR;
#pragma unroll
      for (int i = 0; i < 32 / RPI; ++i) {
        const int r = RPI * i + rs;
        if (r < rows)
          *reinterpret_cast<float4 *>(C + (r0 + r) * g.ldc + 2 * cc) =
              *reinterpret_cast<const float4 *>(Ost + r * L::OPITCH + cc * 16);
      }
      __syncwarp();
    } else if (lane < rows) {
      float2 *crow = C + (r0 + lane) * g.ldc;
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        if (n < N) {
          float2 o = make_float2(ar * acc[n].x - ai * acc[n].y, ar * acc[n].y + ai * acc[n].x);
          if (use_beta) {
            const float2 c = crow[n];
            o.x += br_ * c.x - bi_ * c.y;
            o.y += br_ * c.y + bi_ * c.x;
          }
          crow[n] = o;
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

bool rowstream_eligible(const GemmArgs &g) {
  if (g.a_rin && (g.a_rin % 32 || g.opA != QF_OP_T)) return false;
  return g.N >= 1 && g.N <= 16 && g.K >= 1 && g.K * (g.N <= 8 ? 8 : 16) <= 1024 && g.M >= 32;
}

template <int NN, int KC, bool MMA = false>
int rowstream_launch(const GemmArgs &g, cudaStream_t s) {
  using L = RsLayout<NN, KC, MMA>;
  auto kern = cgemm_rowstream_kernel<NN, KC, MMA>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    attr = true;
  }
  const int64_t steps_per_b = (g.M + RS_WARPS * 32 - 1) / (RS_WARPS * 32);
  const int64_t steps = g.batch * steps_per_b;
  const int per_sm = std::max(1, (int)((225 * 1024) / (L::SMEM + 1024)));
  const int64_t ctas = std::min<int64_t>(steps, (int64_t)sm_count() * per_sm);
  const int64_t per_cta = (steps + ctas - 1) / ctas;
  const int64_t grid = (steps + per_cta - 1) / per_cta;
  kern<<<(unsigned)grid, RS_WARPS * 32, L::SMEM, s>>>(g, steps_per_b, per_cta);
  return check_launch(MMA ? "cgemm_rowmma" : "cgemm_rowstream");
}

// warp-level tensor cores (mma.sync m16n8k8 TF32, 3xTF32 split) inside the
// row-stream pipeline: N <= 8 outputs, K <= 64.  The FFMA row-stream GEMMs
// run at 80% issue (ncu), so this cuts their instruction count ~4x -- but it
// measured SLOWER on the config-2 shapes (1024 x (4096 x 8 x 64): 0.539 ->
// 0.551 ms, 2 x (8.4M x 8 x 8): 0.404 -> 0.572 ms at one CTA per SM), so it
// is off by default (qf_rowmma(1) enables it; tests keep it correct)
static int g_rowmma = 0;
// QF_GEMM_FFMA calls keep every product on the FFMA pipe (the baseline)
static thread_local bool t_allow_mma = true;
struct MmaScope {
  bool prev;
  explicit MmaScope(int mode) : prev(t_allow_mma) { t_allow_mma = (mode & 0xff) != QF_GEMM_FFMA; }
  ~MmaScope() { t_allow_mma = prev; }
};
bool rowmma_eligible(const GemmArgs &g) {
  return g_rowmma && t_allow_mma && g.N >= 1 && g.N <= 8 && g.K >= 1 && g.K <= RsLayout<8, 16, true>::KMAX_MMA &&
         g.M >= 32;
}

int gemm_rowstream(const GemmArgs &g, cudaStream_t s) {
  if (rowmma_eligible(g)) return g.K <= 8 ? rowstream_launch<8, 8, true>(g, s)
                                          : rowstream_launch<8, 16, true>(g, s);
  if (g.N <= 8) return g.K <= 8 ? rowstream_launch<8, 8>(g, s) : rowstream_launch<8, 16>(g, s);
  return g.K <= 8 ? rowstream_launch<16, 8>(g, s) : rowstream_launch<16, 16>(g, s);
}

// ---------------------------------------------------------------------------
// batched GEMV family: N <= 4 output columns, A in N layout (rows contiguous
// along K).  One warp per row group: lanes stride K with coalesced loads,
// 4 rows in flight per warp, butterfly reduction.  B[b] (K x N) is read
// through the read-only path (small, L1/L2 resident).

constexpr int GV_THREADS = 256;

template <typename R, int NC>
__global__ void __launch_bounds__(GV_THREADS)
    cgemv_rows_kernel(const __grid_constant__ GemmArgs g, int64_t rows_per_item,
                      int64_t items_per_b) {
  using V = typename C2<R>::T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const R ar = (R)g.ar, ai = (R)g.ai, br = (R)g.br, bi = (R)g.bi;
  const bool use_beta = (br != R(0) || bi != R(0));
  for (int64_t item = blockIdx.x; item < g.batch * items_per_b; item += gridDim.x) {
    const int64_t b = item / items_per_b;
    const int64_t r0 = (item - b * items_per_b) * rows_per_item;
    const int64_t r1 = min(g.M, r0 + rows_per_item);
    const V *A = reinterpret_cast<const V *>(g.A) + a_batch_off(g, b);
    const V *B = reinterpret_cast<const V *>(g.B) + b_batch_off(g, b);
    V *C = reinterpret_cast<V *>(g.C) + b * g.sC;
    for (int64_t m = r0 + warp * 4; m < r1; m += (GV_THREADS / 32) * 4) {
      V acc[4][NC];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[r][c] = V{R(0), R(0)};
      for (int64_t k = lane; k < g.K; k += 32) {
        V x[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c)
          x[c] = (g.opB == QF_OP_N) ? __ldg(B + k * g.ldb + c) : __ldg(B + c * g.ldb + k);
        V a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          a[r] = (m + r < r1) ? __ldg(A + a_offset(g, m + r, k)) : V{R(0), R(0)};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < NC; ++c) cfma(acc[r][c], a[r], x[c]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            acc[r][c].x += __shfl_xor_sync(0xffffffffu, acc[r][c].x, o);
            acc[r][c].y += __shfl_xor_sync(0xffffffffu, acc[r][c].y, o);
          }
      if (lane < 4 * NC) {
        const int r = lane / NC, c = lane % NC;
        if (m + r < r1) {
          V v = acc[0][0];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int cc = 0; cc < NC; ++cc)
              if (rr == r && cc == c) v = acc[rr][cc];
          V out;
          out.x = ar * v.x - ai * v.y;
          out.y = ar * v.y + ai * v.x;
          V *cp = C + (m + r) * g.ldc + c;
          if (use_beta) {
            const V cv = *cp;
            out.x += br * cv.x - bi * cv.y;
            out.y += br * cv.y + bi * cv.x;
          }
          *cp = out;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// batched dot products (M = N = 1, many entries): the path sums of the
// amplitude walk -- C[b] = alpha * <A[b], B[b]> over K contiguous complex
// entries.  A warp per entry, four 16-byte loads of A and of B in flight per
// lane, one warp reduction, no workspace pass (the split-K skinny kernel +
// its reduction ran 8192 x 4096 at 3.8 TB/s).

constexpr int DOT_THREADS = 256;

__global__ void __launch_bounds__(DOT_THREADS)
    cdot_batched_kernel(const __grid_constant__ GemmArgs g) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (DOT_THREADS / 32) + (threadIdx.x >> 5);
  if (b >= g.batch) return;
  const float4 *A = reinterpret_cast<const float4 *>(reinterpret_cast<const float2 *>(g.A) + a_batch_off(g, b));
  const float4 *B = reinterpret_cast<const float4 *>(reinterpret_cast<const float2 *>(g.B) + b_batch_off(g, b));
  const int64_t n2 = g.K / 2;  // complex pairs
  float re0 = 0.f, im0 = 0.f, re1 = 0.f, im1 = 0.f;
  int64_t i = lane;
  for (; i + 96 < n2; i += 128) {
    float4 a[4], w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a[j] = __ldcs(A + i + 32 * j);
      w[j] = __ldg(B + i + 32 * j);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      re0 = fmaf(a[j].x, w[j].x, re0); re0 = fmaf(-a[j].y, w[j].y, re0);
      im0 = fmaf(a[j].x, w[j].y, im0); im0 = fmaf(a[j].y, w[j].x, im0);
      re1 = fmaf(a[j].z, w[j].z, re1); re1 = fmaf(-a[j].w, w[j].w, re1);
      im1 = fmaf(a[j].z, w[j].w, im1); im1 = fmaf(a[j].w, w[j].z, im1);
    }
  }
  for (; i < n2; i += 32) {
    const float4 a = __ldcs(A + i), w = __ldg(B + i);
    re0 = fmaf(a.x, w.x, re0); re0 = fmaf(-a.y, w.y, re0);
    im0 = fmaf(a.x, w.y, im0); im0 = fmaf(a.y, w.x, im0);
    re1 = fmaf(a.z, w.z, re1); re1 = fmaf(-a.w, w.w, re1);
    im1 = fmaf(a.z, w.w, im1); im1 = fmaf(a.w, w.z, im1);
  }
  float re = re0 + re1, im = im0 + im1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) {
    float2 *C = reinterpret_cast<float2 *>(g.C) + b * g.sC;
    const float ar = (float)g.ar, ai = (float)g.ai, br = (float)g.br, bi = (float)g.bi;
    float2 o = make_float2(ar * re - ai * im, ar * im + ai * re);
    if (br != 0.f || bi != 0.f) {
      const float2 c = *C;
      o.x += br * c.x - bi * c.y;
      o.y += br * c.y + bi * c.x;
    }
    *C = o;
  }
}

// both operands contiguous, 16-byte aligned entries, enough entries to
// fill the machine with a warp each
bool dot_eligible(const GemmArgs &g) {
  if (g.M != 1 || g.N != 1 || g.K < 64 || g.K % 2 || g.a_roff || g.opA != QF_OP_N) return false;
  if (!(g.opB == QF_OP_T || g.ldb == 1)) return false;   // B[b] = K contiguous entries
  if (g.batch < 4 * (int64_t)sm_count()) return false;
  if (g.sA % 2 || g.sB % 2) return false;                // entry bases even (or even b_boff)
  return ((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B)) & 15) == 0;
}

int gemm_dot(const GemmArgs &g, cudaStream_t s) {
  const int64_t grid = (g.batch + DOT_THREADS / 32 - 1) / (DOT_THREADS / 32);
  cdot_batched_kernel<<<(unsigned)grid, DOT_THREADS, 0, s>>>(g);
  return check_launch("cdot_batched");
}

bool gemv_eligible(const GemmArgs &g) {
  return g.N <= 4 && (g.opA == QF_OP_N || g.a_roff) && g.K >= 32 && g.M >= 32;
}

template <typename R, int NC>
int gemv_launch(const GemmArgs &g, cudaStream_t s) {
  // ~8 row groups per warp per item; enough items to fill 148 SMs x 8 CTAs
  const int64_t rows_per_item = std::max<int64_t>(32, std::min<int64_t>(g.M, 256));
  const int64_t items_per_b = (g.M + rows_per_item - 1) / rows_per_item;
  const int64_t items = g.batch * items_per_b;
  const int64_t grid = std::min<int64_t>(items, (int64_t)sm_count() * 8);
  cgemv_rows_kernel<R, NC><<<(unsigned)grid, GV_THREADS, 0, s>>>(g, rows_per_item, items_per_b);
  return check_launch("cgemv_rows");
}

template <typename R>
int gemm_gemv(const GemmArgs &g, cudaStream_t s) {
  switch (g.N) {
    case 1: return gemv_launch<R, 1>(g, s);
    case 2: return gemv_launch<R, 2>(g, s);
    case 3: return gemv_launch<R, 3>(g, s);
    default: return gemv_launch<R, 4>(g, s);
  }
}

template <typename R>
__global__ void cgemm_scale_kernel(const __grid_constant__ GemmArgs g) {
  // K == 0: C = beta * C
  using V = typename C2<R>::T;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t per = g.M * g.N;
  if (t >= g.batch * per) return;
  int64_t b = t / per, r = t - b * per, m = r / g.N, n = r - m * g.N;
  V *C = (V *)g.C + b * g.sC + m * g.ldc + n;
  R br = (R)g.br, bi = (R)g.bi;
  V o = {R(0), R(0)};
  if (br != R(0) || bi != R(0)) {
    V c = *C;
    o.x = br * c.x - bi * c.y;
    o.y = br * c.y + bi * c.x;
  }
  *C = o;
}

// ---------------------------------------------------------------------------
// dispatch

int validate(const GemmArgs &g) {
  QF_REQUIRE(g.batch >= 0 && g.M >= 0 && g.N >= 0 && g.K >= 0, "gemm: negative extent");
  QF_REQUIRE(g.opA == QF_OP_N || g.opA == QF_OP_T, "gemm: opA must be N or T");
  QF_REQUIRE(g.opB == QF_OP_N || g.opB == QF_OP_T, "gemm: opB must be N or T");
  QF_REQUIRE(g.ldc >= std::max<int64_t>(1, g.N), "gemm: ldc < N");
  if (g.a_rin) {
    QF_REQUIRE(g.opA == QF_OP_T && g.a_rin >= 1 && g.lda >= g.a_rin &&
                   g.a_rstride >= g.lda * std::max<int64_t>(g.K, 1),
               "gemm: row blocks need opA T, lda >= rows per block, block stride >= lda*K");
  } else {
    QF_REQUIRE(g.lda >= std::max<int64_t>(1, g.opA == QF_OP_N ? g.K : g.M), "gemm: lda too small");
  }
  QF_REQUIRE(g.ldb >= std::max<int64_t>(1, g.opB == QF_OP_N ? g.N : g.K), "gemm: ldb too small");
  return QF_OK;
}

// 0 = auto (row-block streaming for N <= 16, smem-staged otherwise), 1 =
// smem-staged kernels only, 2 = row-block kernel only, 3 = row-stream where
// eligible (experimental: coalesced staged A; not yet faster than row-block)
static int g_small_engine = 0;

bool smallkn_eligible(const GemmArgs &g) {
  // B[b] fits in smem and one of the contracted/output widths is narrow:
  // these shapes are HBM-bound and the 64x64 tile wastes most of its work
  return g.K * g.N <= SKN_MAX && (g.N <= 16 || g.K <= 16) && g.K >= 1;
}

template <typename R>
int gemm_smallkn_simple(const GemmArgs &g, cudaStream_t s) {
  using V = typename C2<R>::T;
  const int K = (int)g.K, N = (int)g.N;
  const int bpitch = N + ((N % 2 == 0) ? 1 : 0), apitch = K + ((K % 2 == 0) ? 1 : 0);
  // A block sized to the smem left after B (complex128 entries are twice as big)
  const int64_t a_budget = std::max<int64_t>(
      apitch, (int64_t)(160 * 1024) / (int64_t)sizeof(V) - (int64_t)K * bpitch);
  int rm = (int)std::min<int64_t>(g.M, std::max<int64_t>(1, std::min<int64_t>(SKN_A_MAX, a_budget) / apitch));
  rm = (int)std::min<int64_t>(rm, rows_for_parallelism(g, 16));
  int64_t blocks_m = (g.M + rm - 1) / rm;
  size_t smem = ((size_t)K * bpitch + (size_t)rm * apitch) * sizeof(V);
  auto kern = cgemm_smallkn_simple_kernel<R>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int64_t items = g.batch * blocks_m;
  int64_t grid = std::min<int64_t>(items, (int64_t)sm_count() * 6);
  kern<<<(unsigned)grid, SKN_THREADS, smem, s>>>(g, rm, blocks_m);
  return check_launch("cgemm_smallkn_simple");
}

template <typename R>
int gemm_smallkn(const GemmArgs &g, cudaStream_t s) {
  using V = typename C2<R>::T;
  const int K = (int)g.K, N = (int)g.N;
  if (K <= 16) return gemm_smallkn_simple<R>(g, s);
  const int bpitch = N + ((N % 2 == 0) ? 1 : 0);
  const int apitch = (K % 2 == 0) ? K + 2 : K + 1;  // even pitch keeps 16-byte pairs aligned
  const int64_t a_budget = std::max<int64_t>(
      apitch, ((int64_t)(160 * 1024) / (int64_t)sizeof(V) - (int64_t)K * bpitch) / 2);
  int rm = (int)std::min<int64_t>(g.M, std::max<int64_t>(1, std::min<int64_t>(SKN_A_MAX, a_budget) / apitch));
  rm = (int)std::min<int64_t>(rm, rows_for_parallelism(g, 16));
  const int64_t blocks_m = (g.M + rm - 1) / rm;
  const size_t smem = ((((size_t)K * bpitch + 1) & ~(size_t)1) + 2 * (size_t)rm * apitch) * sizeof(V);
  // short K: one output per thread (warp spans a row: A broadcast, B
  // conflict-free); long K: a thread keeps up to 8 columns of its row so the
  // A row is read from smem once
  auto kern = (N < 2) ? cgemm_smallkn_kernel<R, 1>
              : N >= 8           ? cgemm_smallkn_kernel<R, 8>
              : N >= 4           ? cgemm_smallkn_kernel<R, 4>
                                 : cgemm_smallkn_kernel<R, 2>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int64_t items = g.batch * blocks_m;
  const int per_sm = std::max(1, std::min(4, (int)((200 * 1024) / (smem + 2048))));
  const int64_t grid = std::min<int64_t>(items, (int64_t)sm_count() * per_sm);
  const int64_t per_cta = (items + grid - 1) / grid;
  const int64_t grid2 = (items + per_cta - 1) / per_cta;
  kern<<<(unsigned)grid2, SKN_THREADS, smem, s>>>(g, rm, blocks_m, apitch, bpitch, per_cta);
  return check_launch("cgemm_smallkn");
}

template <typename R>
int gemm_simt(const GemmArgs &g, cudaStream_t s) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return QF_OK;
  if (g.K == 0) {
    int64_t total = g.batch * g.M * g.N;
    cgemm_scale_kernel<R><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(g);
    return check_launch("cgemm_scale");
  }
  int64_t P = g.M * g.N;
  if constexpr (sizeof(R) == 4) {
    if (dot_eligible(g)) return gemm_dot(g, s);
  }
  if (P <= 256 && g.K >= 256) {
    int Ppad = 1;
    while (Ppad < P) Ppad <<= 1;
    int KL = STHREADS / Ppad;
    int64_t target_ctas = (int64_t)sm_count() * 8;
    int64_t nsplit = std::max<int64_t>(1, target_ctas / std::max<int64_t>(1, g.batch));
    int64_t min_chunk = (int64_t)KL * 64;
    nsplit = std::min<int64_t>(nsplit, (g.K + min_chunk - 1) / min_chunk);
    nsplit = std::max<int64_t>(1, std::min<int64_t>(nsplit, 4096));
    int64_t kchunk = (g.K + nsplit - 1) / nsplit;
    const bool rows = sizeof(R) == 4 && g.opA == QF_OP_N && !g.a_roff && P >= 8 && g.N <= 4;
    if (rows) kchunk = (kchunk + 63) / 64 * 64;   // 16-byte aligned chunks
    nsplit = (g.K + kchunk - 1) / kchunk;
    if (g.batch > 65535) {
      // gridDim.y carries the batch: split into launches of <= 65535 entries
      // (entry bases advance by the strides or through the offset tables)
      for (int64_t lo = 0; lo < g.batch; lo += 65535) {
        GemmArgs h = g;
        h.batch = std::min<int64_t>(65535, g.batch - lo);
        if (g.a_boff) h.a_boff = g.a_boff + lo;
        else h.A = static_cast<const typename C2<R>::T *>(g.A) + lo * g.sA;
        if (g.b_boff) h.b_boff = g.b_boff + lo;
        else h.B = static_cast<const typename C2<R>::T *>(g.B) + lo * g.sB;
        h.C = static_cast<typename C2<R>::T *>(g.C) + lo * g.sC;
        const int rc = gemm_simt<R>(h, s);
        if (rc != QF_OK) return rc;
      }
      return QF_OK;
    }
    int st = QF_OK;
    void *ws = workspace(g.batch * nsplit * P * (int64_t)sizeof(typename C2<R>::T), s, &st);
    if (st != QF_OK) return st;
    dim3 grid((unsigned)nsplit, (unsigned)g.batch);
    int rc;
    if (rows) {
      // many rows: warp-per-row with lanes along k (see cgemm_skinny_rows_kernel)
      if (g.N == 1) cgemm_skinny_rows_kernel<1><<<grid, STHREADS, 0, s>>>(g, kchunk, (int)nsplit, ws);
      else cgemm_skinny_rows_kernel<4><<<grid, STHREADS, 0, s>>>(g, kchunk, (int)nsplit, ws);
      rc = check_launch("cgemm_skinny_rows");
    } else {
      cgemm_skinny_kernel<R><<<grid, STHREADS, 0, s>>>(g, (int)P, Ppad, kchunk, (int)nsplit, ws);
      rc = check_launch("cgemm_skinny");
    }
    if (rc != QF_OK) return rc;
    int64_t total = g.batch * P;
    cgemm_skinny_reduce<R><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(g, (int)P, (int)nsplit,
                                                                           ws);
    return check_launch("cgemm_skinny_reduce");
  }
  if (g.c_trans) {  // only the row-block / row-stream epilogues store C transposed
    QF_REQUIRE(g.K >= 1 && g.N <= 16 && g.K * g.N <= SKN_MAX, "gemm: transposed C needs N <= 16");
    if constexpr (sizeof(R) == 4) {
      if (rowstream_eligible(g) &&
          (g_small_engine == 3 || (g_small_engine != 2 && (rowmma_eligible(g) ||
                                                          !(g.a_roff ? g.rows_unit : g.opA == QF_OP_T)))))
        return gemm_rowstream(g, s);
    }
    return gemm_rowblock<R>(g, s);
  }
  if (gemv_eligible(g)) return gemm_gemv<R>(g, s);
  if (smallkn_eligible(g)) {
    // narrow outputs stream best row by row; wide outputs keep the
    // smem-staged kernels (warp-wide conflict-free B reads)
    if constexpr (sizeof(R) == 4) {
      // row-stream stages A through shared memory along its contiguous axis;
      // when rows are already the contiguous axis (column-major A, row-unit
      // gathers) and K > 8 the row-block kernel's direct loads are as
      // coalesced and run at higher occupancy (measured 0.74 vs 0.89 ms)
      const bool rows_direct = (g.a_roff ? g.rows_unit : g.opA == QF_OP_T) && g.K > 8;
      if (rowstream_eligible(g) &&
          (g_small_engine == 3 || (g_small_engine == 0 && (!rows_direct || rowmma_eligible(g)))))
        return gemm_rowstream(g, s);
    }
    const bool rowblock = g_small_engine == 0 ? g.N <= 16 : g_small_engine == 2;
    return rowblock ? gemm_rowblock<R>(g, s) : gemm_smallkn<R>(g, s);
  }
  int64_t tiles_n = (g.N + TBN - 1) / TBN, tiles_m = (g.M + TBM - 1) / TBM;
  int64_t tiles = tiles_n * tiles_m;
  int64_t work = tiles * g.batch;
  int64_t grid = std::min<int64_t>(work, (int64_t)sm_count() * 4);
  cgemm_tiled_kernel<R><<<(unsigned)grid, TTHREADS, 0, s>>>(g, tiles_n, tiles);
  return check_launch("cgemm_tiled");
}

// from qf_gemm_tc.cu
int gemm_tc3(const GemmArgs &g, cudaStream_t s);
bool tc3_eligible(const GemmArgs &g);
bool tc3_gather_ok(const GemmArgs &g);

}  // namespace qf

extern "C" {

int qf_cgemm_c64(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                 int64_t lda, int64_t strideA, int opA, const void *B, int64_t ldb, int64_t strideB,
                 int opB, void *C, int64_t ldc, int64_t strideC, float alpha_re, float alpha_im,
                 float beta_re, float beta_im, void *stream) {
  qf::MmaScope mma_scope(mode);
  qf::GemmArgs g{batch, M, N, K, A, lda, strideA, opA, B, ldb, strideB, opB, C, ldc, strideC,
                 alpha_re, alpha_im, beta_re, beta_im};
  int st = qf::validate(g);
  if (st != QF_OK) return st;
  cudaStream_t s = qf::as_stream(stream);
  if (mode == QF_GEMM_TC3) return qf::gemm_tc3(g, s);
  if (mode == QF_GEMM_AUTO && qf::tc3_eligible(g)) return qf::gemm_tc3(g, s);
  QF_REQUIRE(mode == QF_GEMM_AUTO || mode == QF_GEMM_FFMA, "gemm: unknown mode %d", mode);
  return qf::gemm_simt<float>(g, s);
}

int qf_cgemm_c64_gather(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                        int64_t strideA, const int32_t *a_roff, const int32_t *a_coff,
                        const void *B, int64_t ldb, int64_t strideB, int opB, void *C, int64_t ldc,
                        int64_t strideC, float alpha_re, float alpha_im, float beta_re,
                        float beta_im, void *stream) {
  qf::MmaScope mma_scope(mode);
  QF_REQUIRE(a_roff != nullptr && a_coff != nullptr, "gather gemm: offset tables are NULL");
  const bool rows_unit = (mode & QF_GATHER_ROWS_UNIT) != 0;
  mode &= ~QF_GATHER_ROWS_UNIT;
  qf::GemmArgs g{batch, M, N, K, A, std::max<int64_t>(K, 1), strideA, QF_OP_N, B, ldb, strideB,
                 opB, C, ldc, strideC, alpha_re, alpha_im, beta_re, beta_im, a_roff, a_coff,
                 rows_unit};
  int st = qf::validate(g);
  if (st != QF_OK) return st;
  cudaStream_t s = qf::as_stream(stream);
  if ((mode == QF_GEMM_AUTO && qf::tc3_eligible(g)) || mode == QF_GEMM_TC3) {
    if (qf::tc3_gather_ok(g)) return qf::gemm_tc3(g, s);
  }
  return qf::gemm_simt<float>(g, s);
}

int qf_cgemm_c64_gather_boff(int mode, int64_t batch, int64_t M, int64_t N, int64_t K,
                             const void *A, const int64_t *a_boff, const int32_t *a_roff,
                             const int32_t *a_coff, const void *B, int64_t ldb, int64_t strideB,
                             int opB, void *C, int64_t ldc, int64_t strideC, float alpha_re,
                             float alpha_im, float beta_re, float beta_im, void *stream) {
  qf::MmaScope mma_scope(mode);
  QF_REQUIRE((a_roff != nullptr) == (a_coff != nullptr) && (a_boff != nullptr || batch == 0),
             "gather gemm: offset tables are NULL");
  const bool rows_unit = (mode & QF_GATHER_ROWS_UNIT) != 0;
  const bool even = (mode & QF_BOFF_EVEN) != 0;
  mode &= ~(QF_GATHER_ROWS_UNIT | QF_BOFF_EVEN);
  // sA only keys the 16-byte A paths here: 2 = every entry base is even
  qf::GemmArgs g{batch, M, N, K, A, std::max<int64_t>(K, 1), even ? 2 : 1, QF_OP_N, B, ldb,
                 strideB, opB, C, ldc, strideC, alpha_re, alpha_im, beta_re, beta_im, a_roff,
                 a_coff, rows_unit && a_roff != nullptr, a_boff};
  if (!a_roff) {  // plain row-major [M][K] slices at the entry bases
    int st = qf::validate(g);
    if (st != QF_OK) return st;
    cudaStream_t s = qf::as_stream(stream);
    if (mode == QF_GEMM_TC3 || (mode == QF_GEMM_AUTO && qf::tc3_eligible(g))) return qf::gemm_tc3(g, s);
    return qf::gemm_simt<float>(g, s);
  }
  int st = qf::validate(g);
  if (st != QF_OK) return st;
  cudaStream_t s = qf::as_stream(stream);
  if ((mode == QF_GEMM_AUTO && qf::tc3_eligible(g)) || mode == QF_GEMM_TC3) {
    if (qf::tc3_gather_ok(g)) return qf::gemm_tc3(g, s);
  }
  return qf::gemm_simt<float>(g, s);
}

int qf_cgemm_c64_ex(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                    int64_t lda, int64_t strideA, int opA, const int64_t *a_boff,
                    const int32_t *a_roff, const int32_t *a_coff, const void *B, int64_t ldb,
                    int64_t strideB, int opB, const int64_t *b_boff, void *C, int64_t ldc,
                    int64_t strideC, float alpha_re, float alpha_im, float beta_re,
                    float beta_im, void *stream) {
  return qf_cgemm_c64_ex2(mode, batch, M, N, K, A, lda, strideA, opA, a_boff, 0, a_roff, a_coff,
                          B, ldb, strideB, opB, b_boff, 0, C, ldc, strideC, alpha_re, alpha_im,
                          beta_re, beta_im, stream);
}

int qf_cgemm_c64_ex2(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                     int64_t lda, int64_t strideA, int opA, const int64_t *a_boff,
                     int64_t a_nslice, const int32_t *a_roff, const int32_t *a_coff, const void *B, int64_t ldb,
                     int64_t strideB, int opB, const int64_t *b_boff, int64_t b_nslice, void *C,
                     int64_t ldc, int64_t strideC, float alpha_re, float alpha_im, float beta_re,
                     float beta_im, void *stream) {
  qf::MmaScope mma_scope(mode);
  QF_REQUIRE(b_nslice >= 0 && (b_nslice == 0 || b_boff != nullptr),
             "gemm_ex2: b_nslice needs b_boff");
  QF_REQUIRE((a_roff != nullptr) == (a_coff != nullptr), "gemm_ex: a_roff/a_coff must pair");
  const bool rows_unit = (mode & QF_GATHER_ROWS_UNIT) != 0;
  const bool a_even = (mode & QF_BOFF_EVEN) != 0, b_even = (mode & QF_BBOFF_EVEN) != 0;
  const bool c_trans = (mode & QF_C_TRANS) != 0;
  mode &= ~(QF_GATHER_ROWS_UNIT | QF_BOFF_EVEN | QF_BBOFF_EVEN | QF_C_TRANS);
  // with entry-offset tables the batch strides only key the 16-byte paths
  // (a_nslice > 0: a_boff are whole entries of strideA elements, kept)
  QF_REQUIRE(a_nslice == 0 || (a_boff && strideA > 0 && !a_roff), "gemm_ex2: a_nslice needs a_boff");
  if (a_boff && !a_nslice) strideA = a_even ? 2 : 1;
  if (b_boff) strideB = b_even ? 2 : 1;
  if (a_roff) {
    lda = std::max<int64_t>(K, 1);
    opA = QF_OP_N;
  }
  qf::GemmArgs g{batch, M, N, K, A, lda, strideA, opA, B, ldb, strideB, opB, C, ldc, strideC,
                 alpha_re, alpha_im, beta_re, beta_im, a_roff, a_coff,
                 rows_unit && a_roff != nullptr, a_boff, b_boff};
  // b_boff values are whole [K][N] slices of a buffer of b_nslice of them:
  // lets the TMA-fed kernel address B by slice coordinate (and A likewise)
  g.b_nslice = b_nslice;
  g.a_nslice = a_nslice;
  g.c_trans = c_trans;
  if (c_trans) {
    QF_REQUIRE(ldc >= std::max<int64_t>(1, M), "gemm_ex: transposed C needs ldc >= M");
    if (!(N <= 16 && K >= 1 && K * N <= 4096)) {
      qf::set_error("gemm_ex: transposed C needs N <= 16 and K*N <= 4096");
      return QF_ERR_UNSUPPORTED;
    }
    g.ldc = std::max<int64_t>(N, 1);  // validate() checks row-major ldc; restored below
    int st = qf::validate(g);
    if (st != QF_OK) return st;
    g.ldc = ldc;
    return qf::gemm_simt<float>(g, qf::as_stream(stream));
  }
  int st = qf::validate(g);
  if (st != QF_OK) return st;
  cudaStream_t s = qf::as_stream(stream);
  if (mode == QF_GEMM_TC3 || (mode == QF_GEMM_AUTO && qf::tc3_eligible(g))) {
    if (!a_roff || qf::tc3_gather_ok(g)) return qf::gemm_tc3(g, s);
  }
  QF_REQUIRE(mode == QF_GEMM_AUTO || mode == QF_GEMM_FFMA || mode == QF_GEMM_TC3,
             "gemm_ex: unknown mode %d", mode);
  return qf::gemm_simt<float>(g, s);
}

int qf_cgemm_c64_view2(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                       int64_t strideA, const int64_t *a_boff, int64_t a_nslice, int64_t kin,
                       int64_t rows_a, int64_t s_rows_a, int64_t kout, int64_t s_kout,
                       int64_t rows_b, int64_t s_rows_b, const void *B, int64_t ldb,
                       int64_t strideB, int opB, const int64_t *b_boff, int64_t b_nslice,
                       void *C, int64_t ldc, int64_t strideC, int64_t c_nblk, int64_t c_bstride,
                       float alpha_re, float alpha_im, float beta_re, float beta_im,
                       void *stream) {
  QF_REQUIRE(kin >= 1 && rows_a >= 1 && kout >= 1 && rows_b >= 1, "gemm_view: empty run");
  QF_REQUIRE(M == rows_a * rows_b && K == kin * kout, "gemm_view: runs do not match M/K");
  QF_REQUIRE(mode == QF_GEMM_AUTO || mode == QF_GEMM_TC3, "gemm_view: tensor-core modes only");
  QF_REQUIRE(!b_boff || b_nslice > 0, "gemm_view: b_boff needs b_nslice");
  qf::GemmArgs g{batch, M, N, K, A, std::max<int64_t>(K, 1), strideA, QF_OP_N, B, ldb,
                 b_boff ? 2 : strideB, opB, C, ldc, strideC, alpha_re, alpha_im, beta_re, beta_im};
  g.b_boff = b_boff;
  g.b_nslice = b_nslice;
  QF_REQUIRE(!a_boff || a_nslice > 0, "gemm_view2: a_boff needs a_nslice");
  g.a_boff = a_boff;        // whole entries of strideA elements, TMA slice coordinates
  g.a_nslice = a_boff ? a_nslice : 0;
  if (c_nblk) {
    QF_REQUIRE(c_nblk >= 1 && N % c_nblk == 0 && ldc >= c_nblk && c_bstride >= M * ldc &&
                   strideC >= (N / c_nblk) * c_bstride,
               "gemm_view2: column blocks must tile N and not overlap");
    g.c_nblk = c_nblk;
    g.c_bstride = c_bstride;
    g.ldc = std::max<int64_t>(N, 1);   // validate() checks a row-major ldc; restored below
  }
  g.v_kin = kin;
  g.v_ra = rows_a;
  g.v_sra = s_rows_a;
  g.v_kout = kout;
  g.v_skout = s_kout;
  g.v_rb = rows_b;
  g.v_srb = s_rows_b;
  int st = qf::validate(g);
  if (st != QF_OK) return st;
  if (c_nblk) g.ldc = ldc;
  return qf::gemm_tc3(g, qf::as_stream(stream));
}

int qf_cgemm_c64_view(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                      int64_t strideA, int64_t kin, int64_t rows_a, int64_t s_rows_a,
                      int64_t kout, int64_t s_kout, int64_t rows_b, int64_t s_rows_b,
                      const void *B, int64_t ldb, int64_t strideB, int opB,
                      const int64_t *b_boff, int64_t b_nslice, void *C, int64_t ldc,
                      int64_t strideC, float alpha_re, float alpha_im, float beta_re,
                      float beta_im, void *stream) {
  return qf_cgemm_c64_view2(mode, batch, M, N, K, A, strideA, nullptr, 0, kin, rows_a, s_rows_a,
                            kout, s_kout, rows_b, s_rows_b, B, ldb, strideB, opB, b_boff,
                            b_nslice, C, ldc, strideC, 0, 0, alpha_re, alpha_im, beta_re,
                            beta_im, stream);
}

int qf_cgemm_c64_tview(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                       int64_t strideA, int64_t rows_a, int64_t rows_b, int64_t s_rows_b,
                       int64_t kin, int64_t s_kin, int64_t kout, int64_t s_kout, const void *B,
                       int64_t ldb, int64_t strideB, int opB, const int64_t *b_boff,
                       int64_t b_nslice, void *C, int64_t ldc, int64_t strideC, float alpha_re,
                       float alpha_im, float beta_re, float beta_im, void *stream) {
  const bool c_trans = (mode & QF_C_TRANS) != 0;
  mode &= ~QF_C_TRANS;
  QF_REQUIRE(kin >= 1 && rows_a >= 1 && kout >= 1 && rows_b >= 1, "gemm_tview: empty run");
  QF_REQUIRE(M == rows_a * rows_b && K == kin * kout, "gemm_tview: runs do not match M/K");
  QF_REQUIRE(mode == QF_GEMM_AUTO || mode == QF_GEMM_TC3, "gemm_tview: tensor-core modes only");
  QF_REQUIRE(!b_boff || b_nslice > 0, "gemm_tview: b_boff needs b_nslice");
  QF_REQUIRE(ldc >= std::max<int64_t>(1, c_trans ? M : N), "gemm_tview: ldc too small");
  qf::GemmArgs g{batch, M, N, K, A, std::max<int64_t>(M, 1), strideA, QF_OP_T, B, ldb,
                 b_boff ? 2 : strideB, opB, C, ldc, strideC, alpha_re, alpha_im, beta_re, beta_im};
  g.b_boff = b_boff;
  g.b_nslice = b_nslice;
  g.v_t = true;
  g.v_kin = kin;
  g.v_ra = rows_a;
  g.v_kout = kout;
  g.v_skout = s_kout;
  g.v_rb = rows_b;
  g.v_srb = s_rows_b;
  g.v_ski = s_kin;
  g.c_trans = c_trans;
  if (!c_trans) {
    int st = qf::validate(g);
    if (st != QF_OK) return st;
  }
  return qf::gemm_tc3(g, qf::as_stream(stream));
}

int qf_cgemm_c64_rowblocks(int mode, int64_t batch, int64_t M, int64_t N, int64_t K,
                           const void *A, int64_t rows_per_block, int64_t block_stride,
                           int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                           int64_t strideB, int opB, void *C, int64_t ldc, int64_t strideC,
                           float alpha_re, float alpha_im, float beta_re, float beta_im,
                           void *stream) {
  qf::MmaScope mma_scope(mode);
  qf::GemmArgs g{batch, M, N, K, A, lda, strideA, QF_OP_T, B, ldb, strideB, opB, C, ldc, strideC,
                 alpha_re, alpha_im, beta_re, beta_im};
  g.a_rin = rows_per_block;
  g.a_rstride = block_stride;
  QF_REQUIRE(rows_per_block >= 1, "gemm_rowblocks: rows_per_block must be >= 1");
  int st = qf::validate(g);
  if (st != QF_OK) return st;
  if (batch == 0 || M == 0 || N == 0) return QF_OK;
  if (!(N <= 16 && K >= 1 && K * N <= 4096)) {
    qf::set_error("gemm_rowblocks: needs N <= 16 and K*N <= 4096 (CUDA-core row engines)");
    return QF_ERR_UNSUPPORTED;
  }
  cudaStream_t s = qf::as_stream(stream);
  if (qf::g_small_engine != 2 && qf::rowstream_eligible(g) && K <= 8) return qf::gemm_rowstream(g, s);
  return qf::gemm_rowblock<float>(g, s);
}

int qf_rowmma(int enabled) {
  int prev = qf::g_rowmma;
  if (enabled >= 0) qf::g_rowmma = enabled ? 1 : 0;
  return prev;
}

int qf_small_engine(int engine) {
  int prev = qf::g_small_engine;
  qf::g_small_engine = engine;
  return prev;
}

int qf_zgemm_c128(int64_t batch, int64_t M, int64_t N, int64_t K, const void *A, int64_t lda,
                  int64_t strideA, int opA, const void *B, int64_t ldb, int64_t strideB, int opB,
                  void *C, int64_t ldc, int64_t strideC, double alpha_re, double alpha_im,
                  double beta_re, double beta_im, void *stream) {
  qf::GemmArgs g{batch, M, N, K, A, lda, strideA, opA, B, ldb, strideB, opB, C, ldc, strideC,
                 alpha_re, alpha_im, beta_re, beta_im};
  int st = qf::validate(g);
  if (st != QF_OK) return st;
  return qf::gemm_simt<double>(g, qf::as_stream(stream));
}

}  // extern "C"

// GPU state-vector simulator (complex128) -- the B200 twin of the
// reference's dense verification simulator (rq/oracle.py:51-74 with the
// numba kernels rq/_kernels.py:162-271), for exact cross-checks of the
// tensor-network amplitudes beyond the host's 26-qubit cap (2^33 amplitudes
// = 128 GiB fit in HBM).
//
// One pass = one read + one write of the state: a CTA stages a tile of 2^k
// amplitudes -- all combinations of k chosen bits (the 5 lowest included,
// so every warp reads 512 contiguous bytes) at fixed values of the other
// bits -- in shared memory, applies every gate of the pass whose qubits lie
// in the tile, and writes the tile back.  The host packs a cycle's gates
// (disjoint qubits, so they commute) into as few passes as the tile allows.
#include <algorithm>

#include "qf_common.cuh"

namespace qf {

constexpr int SV_MAXK = 10;     // tile bits (2^10 amplitudes = 16 KiB)
constexpr int SV_MAXOPS = 24;   // gates per pass
constexpr int SV_THREADS = 256;

enum { SV_1Q = 0, SV_CZ = 1, SV_ISWAP = 2 };

struct SvPass {
  int k;                 // tile bits
  int bits[SV_MAXK];     // global bit position of tile bit j (ascending)
  int nops;
  int kind[SV_MAXOPS];
  int b0[SV_MAXOPS], b1[SV_MAXOPS];  // tile-local bit positions
  double m[SV_MAXOPS][8];            // 1q: [[m0+i m1, m2+i m3], [m4+i m5, m6+i m7]]
};

__device__ __forceinline__ int64_t sv_deposit(int64_t t, const int *bits, int k) {
  // spread the tile-bit-free index t over the bit positions not in the tile
  int64_t out = 0;
  int src = 0, j = 0;
  for (int p = 0; t >> src; ++p) {
    if (j < k && bits[j] == p) {
      ++j;
      continue;
    }
    out |= ((t >> src) & 1) << p;
    ++src;
  }
  return out;
}

__global__ void __launch_bounds__(SV_THREADS)
    sv_pass_kernel(double2 *__restrict__ psi, int n, const __grid_constant__ SvPass P) {
  __shared__ double2 tile[1 << SV_MAXK];
  __shared__ int64_t s_base;
  const int k = P.k;
  const int T = 1 << k;
  const int64_t ntiles = (int64_t)1 << (n - k);
  // the tile's local -> global offsets are the same for every tile: each
  // thread keeps those of its (at most 4) elements in registers
  constexpr int PER = (1 << SV_MAXK) / SV_THREADS;
  int64_t off[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int l = threadIdx.x + e * SV_THREADS;
    int64_t g = 0;
    for (int j = 0; j < k; ++j) g |= (int64_t)((l >> j) & 1) << P.bits[j];
    off[e] = g;
  }
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x == 0) s_base = sv_deposit(t, P.bits, k);
    __syncthreads();
    const int64_t base = s_base;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int l = threadIdx.x + e * SV_THREADS;
      if (l < T) tile[l] = psi[base | off[e]];
    }
    __syncthreads();
    for (int o = 0; o < P.nops; ++o) {
      const int kind = P.kind[o];
      if (kind == SV_1Q) {
        const int j = P.b0[o];
        const double *m = P.m[o];
        for (int q = threadIdx.x; q < T / 2; q += SV_THREADS) {
          const int lo = ((q >> j) << (j + 1)) | (q & ((1 << j) - 1));
          const int hi = lo | (1 << j);
          const double2 a = tile[lo], b = tile[hi];
          tile[lo] = make_double2(m[0] * a.x - m[1] * a.y + m[2] * b.x - m[3] * b.y,
                                  m[0] * a.y + m[1] * a.x + m[2] * b.y + m[3] * b.x);
          tile[hi] = make_double2(m[4] * a.x - m[5] * a.y + m[6] * b.x - m[7] * b.y,
                                  m[4] * a.y + m[5] * a.x + m[6] * b.y + m[7] * b.x);
        }
      } else {
        const int ja = min(P.b0[o], P.b1[o]), jb = max(P.b0[o], P.b1[o]);
        for (int q = threadIdx.x; q < T / 4; q += SV_THREADS) {
          // insert zeros at ja then jb
          int x = ((q >> ja) << (ja + 1)) | (q & ((1 << ja) - 1));
          x = ((x >> jb) << (jb + 1)) | (x & ((1 << jb) - 1));
          const int i11 = x | (1 << ja) | (1 << jb);
          if (kind == SV_CZ) {
            const double2 v = tile[i11];
            tile[i11] = make_double2(-v.x, -v.y);
          } else {  // iSWAP: |01> <-> |10> with phase i, |00>, |11> unchanged
            const int i01 = x | (1 << ja), i10 = x | (1 << jb);
            const double2 u = tile[i01], w = tile[i10];
            tile[i01] = make_double2(-w.y, w.x);
            tile[i10] = make_double2(-u.y, u.x);
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int l = threadIdx.x + e * SV_THREADS;
      if (l < T) psi[base | off[e]] = tile[l];
    }
    __syncthreads();
  }
}

__global__ void sv_basis_kernel(double2 *psi, int64_t size, int64_t index) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < size;
       i += (int64_t)gridDim.x * blockDim.x)
    psi[i] = make_double2(i == index ? 1.0 : 0.0, 0.0);
}

__global__ void sv_gather_kernel(const double2 *__restrict__ psi, const int64_t *__restrict__ idx,
                                 int64_t count, double2 *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = psi[idx[i]];
}

}  // namespace qf

extern "C" {

int qf_sv_basis(void *state, int n, int64_t index, void *stream) {
  QF_REQUIRE(n >= 0 && n <= 40, "sv_basis: n=%d out of range", n);
  const int64_t size = (int64_t)1 << n;
  QF_REQUIRE(index >= 0 && index < size, "sv_basis: index out of range");
  const int64_t blocks = std::min<int64_t>((size + 255) / 256, (int64_t)qf::sm_count() * 16);
  qf::sv_basis_kernel<<<(unsigned)blocks, 256, 0, qf::as_stream(stream)>>>((double2 *)state, size,
                                                                            index);
  return qf::check_launch("sv_basis");
}

int qf_sv_apply(void *state, int n, int k, const int32_t *bits, int nops, const int32_t *kind,
                const int32_t *op_bits, const double *mats, void *stream) {
  QF_REQUIRE(n >= 1 && n <= 40, "sv_apply: n=%d out of range", n);
  QF_REQUIRE(k >= 1 && k <= qf::SV_MAXK && k <= n, "sv_apply: tile bits k=%d (max %d, <= n)", k,
             qf::SV_MAXK);
  QF_REQUIRE(nops >= 0 && nops <= qf::SV_MAXOPS, "sv_apply: %d gates per pass (max %d)", nops,
             qf::SV_MAXOPS);
  qf::SvPass P{};
  P.k = k;
  for (int j = 0; j < k; ++j) {
    QF_REQUIRE(bits[j] >= 0 && bits[j] < n && (j == 0 || bits[j] > bits[j - 1]),
               "sv_apply: tile bits must be ascending positions < n");
    P.bits[j] = bits[j];
  }
  P.nops = nops;
  for (int o = 0; o < nops; ++o) {
    QF_REQUIRE(kind[o] >= qf::SV_1Q && kind[o] <= qf::SV_ISWAP, "sv_apply: unknown gate kind %d",
               kind[o]);
    P.kind[o] = kind[o];
    P.b0[o] = op_bits[2 * o];
    P.b1[o] = op_bits[2 * o + 1];
    QF_REQUIRE(P.b0[o] >= 0 && P.b0[o] < k && (kind[o] == qf::SV_1Q ||
                                               (P.b1[o] >= 0 && P.b1[o] < k && P.b1[o] != P.b0[o])),
               "sv_apply: gate bits outside the tile");
    for (int i = 0; i < 8; ++i) P.m[o][i] = mats[8 * o + i];
  }
  const int64_t ntiles = (int64_t)1 << (n - k);
  const int64_t blocks = std::min<int64_t>(ntiles, (int64_t)qf::sm_count() * 8);
  qf::sv_pass_kernel<<<(unsigned)blocks, qf::SV_THREADS, 0, qf::as_stream(stream)>>>(
      (double2 *)state, n, P);
  return qf::check_launch("sv_pass");
}

int qf_sv_gather(const void *state, const int64_t *idx, int64_t count, void *out, void *stream) {
  QF_REQUIRE(count >= 0, "sv_gather: negative count");
  if (count == 0) return QF_OK;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)qf::sm_count() * 4);
  qf::sv_gather_kernel<<<(unsigned)blocks, 256, 0, qf::as_stream(stream)>>>(
      (const double2 *)state, idx, count, (double2 *)out);
  return qf::check_launch("sv_gather");
}

}  // extern "C"

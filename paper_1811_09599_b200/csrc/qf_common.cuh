// Shared helpers for libqflex_b200: error state, status codes, launch
// accounting, stream-ordered workspace.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/qflex_b200.h"

namespace qf {

void set_error(const char *fmt, ...);
void count_launch(int n = 1);

// Status for the last kernel launch on this thread.
int check_launch(const char *what);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Grow-only, stream-ordered workspace per device (split-K partials).
void *workspace(int64_t bytes, cudaStream_t stream, int *status);

int sm_count();

// Strided-batched complex GEMM arguments (all engines).  When a_roff/a_coff
// are set, A is GATHERED: A(b, r, k) = A + b*sA + a_roff[r] + a_coff[k]
// (b*sA -> a_boff[b] when the batch offset table is set)
// (element offsets; opA/lda ignored) -- the operand permutation is fused
// into the GEMM's operand fetch instead of a separate transpose pass.
struct GemmArgs {
  int64_t batch, M, N, K;
  const void *A;
  int64_t lda, sA;
  int opA;
  const void *B;
  int64_t ldb, sB;
  int opB;
  void *C;
  int64_t ldc, sC;
  double ar, ai, br, bi;
  const int32_t *a_roff = nullptr;
  const int32_t *a_coff = nullptr;
  bool rows_unit = false;  // gathered A hint: a_roff[r] == a_roff[0] + r
  // gathered A only: per-batch entry base offsets (elements) replacing b*sA --
  // a batch of bit-strings sliced out of a tensor whose outputs are still
  // open (late output batching); any alignment
  const int64_t *a_boff = nullptr;
  // per-batch entry base offsets of B replacing b*sB (a site tensor whose
  // output is sliced per bit-string: B(b) = B + b_boff[b]); any alignment
  const int64_t *b_boff = nullptr;
  // b_boff values are whole [K][N] blocks of a B buffer holding b_nslice of
  // them (the TMA kernel then addresses B slice b_boff[b] / (K*N)); 0 = unknown
  int64_t b_nslice = 0;
  // A as a strided view read by a 5-D TMA map (TMA kernel only; v_kin = 0:
  // unused): k = ko*v_kin + ki with ki innermost and contiguous, row
  // r = rb*v_ra + ra; v_s* are element strides of ra, ko and rb
  int64_t v_kin = 0, v_ra = 0, v_sra = 0, v_kout = 0, v_skout = 0, v_rb = 0, v_srb = 0;
  // v_t: the TRANSPOSED view (opA = T): rows innermost -- row r = rb*v_ra + ra
  // with ra contiguous (v_ra rows), rb at stride v_srb; k = ko*v_kin + ki, ki
  // at stride v_ski, ko at v_skout (any order of the four runs in memory)
  bool v_t = false;
  int64_t v_ski = 0;
  // C stored transposed per entry: C(b, m, n) at C + b*sC + n*ldc + m (row-block
  // and row-stream engines, and the TMA kernel on a transposed view)
  bool c_trans = false;
  // opA = T in row blocks (row-block / row-stream engines only): row r at
  // (r / a_rin) * a_rstride + r % a_rin, k at k * lda -- a big operand laid
  // out [outer rows][k][inner rows] read in place (no permute)
  int64_t a_rin = 0, a_rstride = 0;
  // a_boff values are whole entries (multiples of sA) of an A buffer holding
  // a_nslice of them: the TMA-fed kernel reads entry b at slice coordinate
  // a_boff[b] / sA (a bit-string's slice of a tensor whose outputs are open)
  int64_t a_nslice = 0;
  // C in column blocks (TMA short-K kernel): column n of row m of entry b at
  // C + b*sC + (n / c_nblk) * c_bstride + m * ldc + n % c_nblk -- the
  // outputs of several open-output values computed side by side land as
  // separate [M][c_nblk] blocks (ldc = c_nblk)
  int64_t c_nblk = 0, c_bstride = 0;
  // profiling knob of the long-K Gauss kernel (env QF_TC3_DEBUG, results are
  // garbage when set): 1 = skip the B' stores, 2 = skip the A tcgen05.st,
  // 4 = promotion warps release the partial without reading it, 8 = the
  // TMA producer loads nothing (the converters re-read stale raw slots)
  int dbg = 0;
};

__device__ __forceinline__ int64_t a_row_base(const GemmArgs &g, int64_t r) {
  if (!g.a_rin) return r;
  const int64_t q = r / g.a_rin;
  return q * g.a_rstride + (r - q * g.a_rin);
}

__device__ __forceinline__ int64_t b_batch_off(const GemmArgs &g, int64_t b) {
  return g.b_boff ? __ldg(g.b_boff + b) : b * g.sB;
}

__device__ __forceinline__ int64_t a_batch_off(const GemmArgs &g, int64_t b) {
  return g.a_boff ? __ldg(g.a_boff + b) : b * g.sA;
}

__device__ __forceinline__ int64_t a_offset(const GemmArgs &g, int64_t r, int64_t k) {
  if (g.a_roff) return (int64_t)g.a_roff[r] + g.a_coff[k];
  return g.opA == QF_OP_N ? r * g.lda + k : k * g.lda + a_row_base(g, r);
}

}  // namespace qf

#define QF_REQUIRE(cond, ...)                 \
  do {                                        \
    if (!(cond)) {                            \
      qf::set_error(__VA_ARGS__);             \
      return QF_ERR_INVALID;                  \
    }                                         \
  } while (0)

#define QF_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      qf::set_error("%s failed: %s", #call, cudaGetErrorString(e_));               \
      return QF_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

/*
 * qflex_b200.h -- C ABI of the B200-native RQC contraction library
 * (libqflex_b200.so, built from paper_1811_09599_b200/csrc/ for sm_100a).
 *
 * The reference (`rqcsim`, pure Python) exposes this hot path only as
 * Python functions; every entry point below replaces one reference call
 * site and is bound from Python with ctypes
 * (paper_1811_09599_b200/_lib.py; binding recipe in INTEGRATION.md).
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers owned by the caller
 *     (torch buffers); the library never frees them.
 *   - Row-major ("C order") storage everywhere, as in the reference
 *     (SPEC.md:101).  complex64 = interleaved float32 (re, im);
 *     complex128 = interleaved float64.
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     asynchronous on it.  NULL = legacy default stream.
 *   - Every function returns an int status: QF_OK (0) or a negative
 *     code; qf_last_error() returns the message of the last failure on
 *     the calling host thread.  Python maps QF_ERR_INVALID -> ValueError,
 *     QF_ERR_MEMORY -> MemoryBudgetError, others -> RuntimeError, the
 *     same exception classes the reference raises.
 *   - Thread safety: callable from one host thread per GPU concurrently;
 *     internal caches are mutex-protected.
 */
#ifndef QFLEX_B200_H
#define QFLEX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QF_OK 0
#define QF_ERR_INVALID (-1)     /* bad shape / perm / argument   -> ValueError        */
#define QF_ERR_CUDA (-2)        /* CUDA launch or runtime error  -> RuntimeError      */
#define QF_ERR_MEMORY (-3)      /* workspace allocation failed   -> MemoryBudgetError */
#define QF_ERR_UNSUPPORTED (-4) /* not built for this device     -> RuntimeError      */

/* GEMM engine selection for qf_cgemm_* */
#define QF_GEMM_AUTO 0   /* tcgen05 3xTF32 where the shape pays, else FFMA        */
#define QF_GEMM_FFMA 1   /* K3: plain fp32 FFMA complex GEMM (baseline)           */
#define QF_GEMM_TC3 2    /* K2: tcgen05 kind::tf32 3xTF32 complex GEMM (sm_100a)  */

/* hint or'ed into qf_cgemm_c64_gather's mode: a_roff[r] == a_roff[0] + r
 * (consecutive rows adjacent in memory); picks the CUDA-core fetch direction */
#define QF_GATHER_ROWS_UNIT 0x100

/* hint or'ed into qf_cgemm_c64_gather_boff's mode: every a_boff[b] is even
 * (entry bases 16-byte aligned; enables the paired A loads) */
#define QF_BOFF_EVEN 0x200
/* same for b_boff in qf_cgemm_c64_ex */
#define QF_BBOFF_EVEN 0x400
/* qf_cgemm_c64_ex: store C transposed per entry, C(b, m, n) at
 * C + b*strideC + n*ldc + m (ldc >= M; N <= 16 CUDA-core engines only,
 * QF_ERR_UNSUPPORTED otherwise) */
#define QF_C_TRANS 0x800

/* operand layouts */
#define QF_OP_N 0        /* A stored [M][K] (lda >= K); B stored [K][N] (ldb >= N) */
#define QF_OP_T 1        /* A stored [K][M] (lda >= M); B stored [N][K] (ldb >= K) */

/* Last error message of this host thread ("" if none). */
const char *qf_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
int qf_version(void);

/* Properties of device `dev`: SM count and compute capability. */
int qf_device_info(int dev, int *sm_count, int *cc_major, int *cc_minor);

/*
 * K1 -- general tensor index permutation.
 *   dst = ascontiguousarray(transpose(src, perm)), bit-exact.
 * Replaces rq/tensor_core.py:290-330 (permute_fast, the L/R move kernels
 * rq/_kernels.py:105-151) and rq/tensor_core.py:271-273 (permute_naive);
 * same (dims, perm) meaning as plan_permutation rq/tensor_core.py:81.
 * elem_bytes: 8 (complex64) or 16 (complex128).  src and dst must not
 * alias.  rank <= 64; dims may contain 1s; rank 0 copies one element.
 */
int qf_permute(const void *src, void *dst, int rank, const int64_t *dims,
               const int32_t *perm, int elem_bytes, void *stream);
int qf_permute_c64(const void *src, void *dst, int rank, const int64_t *dims,
                   const int32_t *perm, void *stream);

/*
 * K4 -- index slicing (Tensor.fix, rq/tensor_core.py:366-372, used by
 * Net2D.fix_outputs rq/network_builder.py:134-149 and the executor's cut
 * slicing rq/contraction_plan.py:450-466), batched over bit-strings.
 * View src as [outer][dim][inner]; for b in [0, nidx):
 *   dst[b][o][i] = src[o][idx[b]][i]
 * idx is a DEVICE int32 array of nidx entries, each in [0, dim).
 */
int qf_gather_axis(const void *src, void *dst, int64_t outer, int64_t dim,
                   int64_t inner, const int32_t *idx, int64_t nidx,
                   int elem_bytes, void *stream);

/* Single-value form of qf_gather_axis (host value, no index array). */
int qf_fix_axis(const void *src, void *dst, int64_t outer, int64_t dim,
                int64_t inner, int64_t value, int elem_bytes, void *stream);

/*
 * K2/K3 -- strided-batched complex GEMM, row-major:
 *   C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b],  b in [0, batch)
 * op(A) is M x K, op(B) is K x N, C[b] is M x N with leading dim ldc.
 * Replaces the `(m x k) @ (k x n)` at rq/tensor_core.py:417 (numpy ->
 * OpenBLAS cgemm).  mode: QF_GEMM_AUTO / _FFMA / _TC3.  K may be 0.
 */
int qf_cgemm_c64(int mode, int64_t batch, int64_t M, int64_t N, int64_t K,
                 const void *A, int64_t lda, int64_t strideA, int opA,
                 const void *B, int64_t ldb, int64_t strideB, int opB,
                 void *C, int64_t ldc, int64_t strideC,
                 float alpha_re, float alpha_im, float beta_re, float beta_im,
                 void *stream);

/*
 * Gathered-A twin of qf_cgemm_c64: the permutation of A is fused into the
 * GEMM's operand fetch instead of a separate transpose pass.
 *   A(b, r, k) = A + b*strideA + a_roff[r] + a_coff[k]   (complex elements)
 * a_roff: DEVICE int32[M], a_coff: DEVICE int32[K] (row-major offsets of the
 * free and summed index groups inside one batch entry; entries < 2^31).
 * Replaces the permute-then-`@` pair of rq/tensor_core.py:411-417.
 */
int qf_cgemm_c64_gather(int mode, int64_t batch, int64_t M, int64_t N, int64_t K,
                        const void *A, int64_t strideA, const int32_t *a_roff,
                        const int32_t *a_coff, const void *B, int64_t ldb, int64_t strideB,
                        int opB, void *C, int64_t ldc, int64_t strideC,
                        float alpha_re, float alpha_im, float beta_re, float beta_im,
                        void *stream);

/*
 * Late output batching (the engine's `amplitudes` path).  Early plan steps
 * run with the circuit's `out` indices still OPEN (every combination of the
 * few qubits they touch); once a step's open outputs would outnumber the
 * bit-strings, the batch is sliced out of the open tensor.  This is the
 * reference's Tensor.fix / Net2D.fix_outputs (rq/tensor_core.py:366-372,
 * rq/network_builder.py:134-149) applied to an intermediate instead of a
 * site tensor, and the open-qubit idea of amplitude_batch
 * (rq/amplitude_engine.py:128-170) applied internally.
 *
 * qf_bit_offsets:  off[b] = sum_j bits[rows[j]*ld + b] * strides[j]
 *   bits: DEVICE int32 matrix (row q = bit of qubit q for every entry b);
 *   rows/strides: HOST arrays of n <= 64 entries (element strides of the
 *   open `out` indices); off: DEVICE int64[nb].
 * qf_gather_rows:  dst[b][o][l] = src[off[b] + ooff[o] + l]
 *   (ooff: DEVICE int64[n_outer], or NULL for ooff[o] = o*L).
 * qf_cgemm_c64_gather_boff: qf_cgemm_c64_gather with the entry base
 *   b*strideA replaced by a_boff[b] (DEVICE int64[batch]), so the slice is
 *   fused into the GEMM's operand fetch.  a_roff = a_coff = NULL: each slice
 *   is a plain row-major [M][K] block (lda = K) at its entry base.
 */
int qf_bit_offsets(const int32_t *bits, int64_t ld, int n, const int32_t *rows,
                   const int64_t *strides, int64_t nb, int64_t *off, void *stream);
int qf_gather_rows(const void *src, void *dst, int64_t nb, const int64_t *off, int64_t n_outer,
                   const int64_t *ooff, int64_t L, int elem_bytes, void *stream);
int qf_cgemm_c64_gather_boff(int mode, int64_t batch, int64_t M, int64_t N, int64_t K,
                             const void *A, const int64_t *a_boff, const int32_t *a_roff,
                             const int32_t *a_coff, const void *B, int64_t ldb, int64_t strideB,
                             int opB, void *C, int64_t ldc, int64_t strideC, float alpha_re,
                             float alpha_im, float beta_re, float beta_im, void *stream);

/*
 * General form of the complex64 GEMM: every operand option at once.
 *   A(b, r, k) = A + baseA(b) + (a_roff ? a_roff[r] + a_coff[k] : opA/lda offset)
 *   B(b)       = B + baseB(b) (opB/ldb layout)
 *   baseA(b) = a_boff ? a_boff[b] : b*strideA;  baseB(b) = b_boff ? b_boff[b] : b*strideB
 * Used by the late output slicing path to contract a batched intermediate
 * with a site tensor whose output is still open: B(b) is the site's slice
 * for bit-string b, read in place (no batched copy of the site tensor).
 * mode may carry QF_GATHER_ROWS_UNIT, QF_BOFF_EVEN, QF_BBOFF_EVEN.
 */
int qf_cgemm_c64_ex(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                    int64_t lda, int64_t strideA, int opA, const int64_t *a_boff,
                    const int32_t *a_roff, const int32_t *a_coff, const void *B, int64_t ldb,
                    int64_t strideB, int opB, const int64_t *b_boff, void *C, int64_t ldc,
                    int64_t strideC, float alpha_re, float alpha_im, float beta_re,
                    float beta_im, void *stream);

/*
 * qf_cgemm_c64_ex with slice counts: a_nslice > 0 declares every a_boff[b] a
 * whole entry (a multiple of strideA) of an A buffer holding a_nslice of
 * them, addressed by the TMA kernel as a slice coordinate; likewise, when
 * every b_boff[b] is a whole
 * [K][N] slice (a multiple of K*N) of a B buffer holding b_nslice slices,
 * the TMA-fed tensor-core kernel reads B by slice coordinate (the per-entry
 * site-tensor slices of the batched amplitude walk).  b_nslice = 0: as
 * qf_cgemm_c64_ex.  Replaces the same contract() call as qf_cgemm_c64_ex
 * (rq/tensor_core.py:391-419 with the fixes of rq/network_builder.py:134-149).
 */
int qf_cgemm_c64_ex2(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                     int64_t lda, int64_t strideA, int opA, const int64_t *a_boff,
                     int64_t a_nslice, const int32_t *a_roff, const int32_t *a_coff, const void *B, int64_t ldb,
                     int64_t strideB, int opB, const int64_t *b_boff, int64_t b_nslice, void *C,
                     int64_t ldc, int64_t strideC, float alpha_re, float alpha_im, float beta_re,
                     float beta_im, void *stream);

/*
 * Strided-view A for the TMA-fed tensor-core kernel (no offset tables): the
 * big operand of a contraction whose shared labels are its innermost index
 * (kin, contiguous, kin % 8 == 0) and at most one more index (kout), with its
 * free labels in at most two runs (rows_a fast, rows_b slow):
 *   A(b, r, k) = A + b*strideA + ra*s_rows_a + rb*s_rows_b + ko*s_kout + ki
 *   r = rb*rows_a + ra,  k = ko*kin + ki        (element strides, all even)
 * b_boff/b_nslice: B entries as whole [K][N] slices of a buffer of b_nslice
 * (late output slicing; NULL/0 = strided B).  Returns QF_ERR_UNSUPPORTED when
 * the view or shape does not fit the TMA kernel (the caller falls back to
 * qf_cgemm_c64_ex with offset tables).
 */
int qf_cgemm_c64_view(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                      int64_t strideA, int64_t kin, int64_t rows_a, int64_t s_rows_a,
                      int64_t kout, int64_t s_kout, int64_t rows_b, int64_t s_rows_b,
                      const void *B, int64_t ldb, int64_t strideB, int opB,
                      const int64_t *b_boff, int64_t b_nslice, void *C, int64_t ldc,
                      int64_t strideC, float alpha_re, float alpha_im, float beta_re,
                      float beta_im, void *stream);

/*
 * qf_cgemm_c64_view with per-entry A slices: entry b reads the view at
 * A + a_boff[b], every a_boff[b] a multiple of strideA (whole entries of a
 * buffer holding a_nslice of them; a bit-string's slice of a tensor whose
 * outputs are still open) -- a TMA slice coordinate.  c_nblk > 0 stores C
 * in column blocks: column n of row m at C + b*strideC + (n / c_nblk) *
 * c_bstride + m*ldc + n % c_nblk (several open-output values computed side
 * by side, each landing as its own [M][c_nblk] block; K <= 128).
 * a_boff = NULL, c_nblk = 0: as qf_cgemm_c64_view.
 */
int qf_cgemm_c64_view2(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                       int64_t strideA, const int64_t *a_boff, int64_t a_nslice, int64_t kin,
                       int64_t rows_a, int64_t s_rows_a, int64_t kout, int64_t s_kout,
                       int64_t rows_b, int64_t s_rows_b, const void *B, int64_t ldb,
                       int64_t strideB, int opB, const int64_t *b_boff, int64_t b_nslice,
                       void *C, int64_t ldc, int64_t strideC, int64_t c_nblk, int64_t c_bstride,
                       float alpha_re, float alpha_im, float beta_re, float beta_im,
                       void *stream);

/*
 * GPU state-vector simulator (complex128), the verification twin of the
 * reference's dense simulator (rq/oracle.py:51-74, kernels
 * rq/_kernels.py:162-271).  Bit p of a state index is qubit n-1-p (qubit 0 =
 * most significant, rq/oracle.py:8-10).
 * qf_sv_basis:  state = |index>  (2^n complex128 entries)
 * qf_sv_apply:  one pass over the state: tiles of the k <= 10 ascending bit
 *   positions `bits` (HOST), applying nops <= 24 gates in order; gate o is
 *   kind[o] (0 = one-qubit, 1 = CZ, 2 = iSWAP) on tile-local bit positions
 *   op_bits[2o], op_bits[2o+1]; one-qubit matrices in mats[8o..8o+7] as
 *   (re, im) of m00, m01, m10, m11 (all HOST arrays).
 * qf_sv_gather: out[i] = state[idx[i]]  (idx: DEVICE int64)
 */
int qf_sv_basis(void *state, int n, int64_t index, void *stream);
int qf_sv_apply(void *state, int n, int k, const int32_t *bits, int nops, const int32_t *kind,
                const int32_t *op_bits, const double *mats, void *stream);
int qf_sv_gather(const void *state, const int64_t *idx, int64_t count, void *out, void *stream);

/* complex128 twin (FFMA/DFMA only), for dtype=complex128 engines. */
int qf_zgemm_c128(int64_t batch, int64_t M, int64_t N, int64_t K,
                  const void *A, int64_t lda, int64_t strideA, int opA,
                  const void *B, int64_t ldb, int64_t strideB, int opB,
                  void *C, int64_t ldc, int64_t strideC,
                  double alpha_re, double alpha_im, double beta_re, double beta_im,
                  void *stream);

/*
 * K5 -- path-sum accumulation (rq/amplitude_engine.py:123,153-157):
 *   y[i] += x[i] for i in [0, n) complex elements.
 */
int qf_accumulate(const void *x, void *y, int64_t n, int elem_bytes, void *stream);

/* Index tables of the batched walks (entry bases of per-entry operand
 * fetches), computed on the device:
 *   out[e] = (base ? base[e / rep] : (e / rep) * entry) + (e % rep) * stride,
 * e in [0, n).  base (DEVICE int64[n / rep]) may be NULL.  Serves the
 * broadcast of a path-free operand over a path-batched one and the
 * (bit-string, cut value) slices of a path-batched walk -- the reference
 * walks those paths one by one (rq/amplitude_engine.py:123). */
int qf_affine_offsets(int64_t *out, int64_t n, int64_t rep, int64_t entry, const int64_t *base,
                      int64_t stride, void *stream);

/* y[i] = re + i*im for i in [0, n) (complex64: elem_bytes 8, complex128: 16);
 * e.g. the ones row that sums a path axis. */
int qf_fill_value(void *y, int64_t n, double re, double im, int elem_bytes, void *stream);

/* y[0:bytes) = 0, stream-ordered (accumulator reset before a path sum). */
int qf_fill_zero(void *y, int64_t bytes, void *stream);

/*
 * Workspace the GEMM split-K path uses (the only memory the library owns),
 * grow-only per device: growing keeps the previous buffer alive (a CUDA graph
 * that captured a GEMM holds its pointer) and is refused while the stream is
 * capturing -- reserve before capturing to keep allocation out of timed
 * regions and graphs.  qf_workspace_release frees every buffer of the
 * current device (synchronizing it); call it only when no captured graph
 * that used the library is replayed afterwards.
 */
int qf_workspace_reserve(int64_t bytes, void *stream);
int qf_workspace_release(void);

/* K2 tuning/validation knob (A/B measurements and tests; 0 = auto, the
 * product setting).  Short-K kernel flavours: 10/11/12 = 8 converter warps /
 * 16 converter warps / 16 converter + 4 epilogue warps, 20/21 = TMA-fed with
 * an 8 / 4 deep ring, 23 = 64-column tiles for narrow views.  Long-K
 * flavours (csrc/qf_gemm_tc.cu): 13 = converter fetch (no TMA), 19/26/27 =
 * real-block form promoted every 4/16/32 k-blocks, 30/31/32 = Gauss form on
 * 128 x 64 tiles promoted every 16/32/64 k-blocks, 34 = Gauss, 2 stages.
 * Wide long-K kernel (csrc/qf_gemm_tcw.cu, 128 x 128 Gauss tiles, master in
 * registers): 40/41/42 = single CTAs promoted every 64/128/32 k-blocks,
 * 43/44/45 = CTA pairs (cta_group::2) likewise, 46 = pairs draining the
 * partial in 4-column pieces; auto = pairs when M fills 256-row tiles.
 * 50 = streaming K = 16 kernel (csrc/qf_gemm_tcs.cu) off.  Returns the
 * previous setting. */
int qf_tc3_set_variant(int variant);

/* K3 tuning/validation knob for memory-bound small K x N shapes: 0 = auto
 * (row-block streaming for N <= 16, shared-memory staged otherwise), 1 =
 * staged kernels only, 2 = row-block kernel only, 3 = row-stream (staged,
 * coalesced A; complex64 N <= 16, K*N <= 512) where eligible.  Returns the
 * previous one. */
int qf_small_engine(int engine);

/*
 * Transposed strided view of A for the TMA-fed tensor-core kernel: rows are
 * the innermost axis.  Per entry, row r = rb*rows_a + ra with ra contiguous
 * (rows_a rows) and rb at element stride s_rows_b; k = ko*kin + ki with ki at
 * stride s_kin and ko at s_kout -- the four runs in any memory order, e.g.
 * [ko][rb][ki][ra].  mode may carry QF_C_TRANS (C(b, m, n) at
 * C + b*strideC + n*ldc + m).  Any N (tiles of 64 columns) for K in [32, 128];
 * K >= 256 with N >= 128 on the wide long-K kernel (row-major C only);
 * kin % 8 == 0.  Serves the same contract() as qf_cgemm_c64_ex
 * (rq/tensor_core.py:391-419) when the big operand's innermost labels are
 * free: the permute before the GEMM (rq/tensor_core.py:410-416) is folded
 * into the TMA box.
 */
int qf_cgemm_c64_tview(int mode, int64_t batch, int64_t M, int64_t N, int64_t K, const void *A,
                       int64_t strideA, int64_t rows_a, int64_t rows_b, int64_t s_rows_b,
                       int64_t kin, int64_t s_kin, int64_t kout, int64_t s_kout, const void *B,
                       int64_t ldb, int64_t strideB, int opB, const int64_t *b_boff,
                       int64_t b_nslice, void *C, int64_t ldc, int64_t strideC, float alpha_re,
                       float alpha_im, float beta_re, float beta_im, void *stream);

/*
 * Batched GEMM whose A is read in ROW BLOCKS (complex64, N <= 16, K*N <= 4096;
 * CUDA-core row engines): A(b, r, k) = A + b*strideA + (r / rows_per_block) *
 * block_stride + r % rows_per_block + k*lda, i.e. a big operand laid out
 * [outer rows][k][inner rows] contracted over its middle labels in place
 * (replaces the permute + GEMM of `contract`, rq/tensor_core.py:411-417, for
 * operands with too many rows for offset tables).  B and C as qf_cgemm_c64.
 * QF_ERR_UNSUPPORTED outside that shape range.
 */
int qf_cgemm_c64_rowblocks(int mode, int64_t batch, int64_t M, int64_t N, int64_t K,
                           const void *A, int64_t rows_per_block, int64_t block_stride,
                           int64_t lda, int64_t strideA, const void *B, int64_t ldb,
                           int64_t strideB, int opB, void *C, int64_t ldc, int64_t strideC,
                           float alpha_re, float alpha_im, float beta_re, float beta_im,
                           void *stream);

/* K3 narrow outputs (complex64, N <= 8, K <= 64): 1 = row-stream pipeline
 * with warp-level tensor cores (mma.sync m16n8k8 TF32, 3xTF32 split), 0 =
 * its FFMA twin (the default: measured faster); < 0 only queries.  Returns
 * the previous one.  QF_GEMM_FFMA calls never use the tensor-core twin. */
int qf_rowmma(int enabled);

/*
 * Path sums and the multi-GPU slice collective.  The
 * reference sums paths sequentially in one process
 * (rq/amplitude_engine.py:123 single amplitudes, :153-157 open-qubit
 * batches); a multi-GPU run gives every rank a contiguous share of the path
 * list and combines the partial amplitudes with ONE all-reduce.
 *
 * NCCL is resolved at run time (the copy already loaded in the process, else
 * $QF_NCCL_LIB, else libnccl.so.2); the library has no link-time NCCL
 * dependency.  One communicator per (process group, device):
 *   rank 0: qf_nccl_unique_id(uid, 128) -> broadcast uid by the host ->
 *   every rank: qf_nccl_init(uid, nranks, rank, dev, &handle).
 * qf_allreduce_c64 sums `count` complex64 values (as 2*count float32) in
 * place across the communicator's ranks, enqueued on `stream`.
 */
int qf_nccl_available(void);  /* 1 if an NCCL library can be bound, else 0 */
int qf_nccl_unique_id(void *uid, int64_t nbytes);
int qf_nccl_init(const void *uid, int nranks, int rank, int dev, int *handle);
int qf_nccl_destroy(int handle);
int qf_allreduce_c64(int handle, void *buf, int64_t count, void *stream);

/* y[i] += alpha * x[i], complex64, i in [0, n) -- one path's partial
 * amplitudes added into the running sum (rq/amplitude_engine.py:123,157). */
int qf_axpy_c64(int64_t n, float alpha_re, float alpha_im, const void *x, void *y, void *stream);

/* out[b] = sum_i x[b*stride_x + i] * y[b*stride_y + i] (no conjugation),
 * complex64, b in [0, batch): the final `result` step of a plan, the dot of
 * two open region tensors (rq/contraction_plan.py:477-523 folding the last
 * pair, rq/tensor_core.py:391-419 with every label shared). */
int qf_dot_c64(int64_t batch, int64_t n, const void *x, int64_t stride_x, const void *y,
               int64_t stride_y, void *out, void *stream);

/* Name of the last kernel this library launched on the calling thread
 * (static string; "" if none) -- lets profilers attribute timings. */
const char *qf_last_kernel(void);

/* Number of kernels this library launched on the calling thread since the
 * last reset (for the bench's gpu_launches claim). */
int64_t qf_launch_count(int reset);

#ifdef __cplusplus
}
#endif

#endif /* QFLEX_B200_H */

/*
 * permute_ref.c -- TEST INFRASTRUCTURE ONLY (the CPU checker of config 3).
 *
 * A C restatement of the reference's permutation oracle
 *   permute_naive(a, perm) = np.ascontiguousarray(np.transpose(a, perm))
 * (rq/tensor_core.py:271-273, rq = /root/reference/pkg/src/rqcsim): the
 * row-major output element at coordinates (i_0 .. i_{r-1}) over the output
 * dims d[perm[0]] .. d[perm[r-1]] is the input element whose coordinate
 * along input axis perm[j] is i_j.  Pure data movement, so the result is
 * bit-exact by construction; it exists because numpy's strided transpose
 * of a 2^28..2^30-element rank-30 tensor takes minutes per case, while
 * config 3 asks for 64 byte-compared permutations per size.
 *
 * Parity pin: tests/test_oracle_golden.py checks it against numpy
 * (oracle.rqc_oracle.permute_naive) and the reference's own permute_fast
 * bytes in tests/golden/golden_perm.json.  Only tests/ and bench.py's
 * checker legs load it (oracle/permute_oracle.py); the product never does.
 *
 * Build: __graft_entry__.build() ->
 *   gcc -O3 -fopenmp -shared -fPIC oracle/permute_ref.c -o oracle/lib/libpermute_ref.so
 */
#include <stdint.h>
#include <string.h>

#define MAXR 64

/* dst[o] = src[in_offset(o)] for o in [lo, hi), elem_bytes in {8, 16};
 * returns 0, or -1 on bad arguments */
static int permute_range(const char *src, char *dst, int rank, const int64_t *dims,
                         const int32_t *perm, int elem_bytes, int64_t lo, int64_t hi) {
  int64_t in_stride[MAXR], od[MAXR], os[MAXR], c[MAXR];
  int64_t s = 1;
  for (int a = rank - 1; a >= 0; --a) {
    in_stride[a] = s;
    s *= dims[a];
  }
  for (int j = 0; j < rank; ++j) {
    od[j] = dims[perm[j]];
    os[j] = in_stride[perm[j]];
  }
  /* odometer over the output coordinates, starting at lo */
  int64_t rem = lo, off = 0;
  for (int j = rank - 1; j >= 0; --j) {
    c[j] = rem % od[j];
    rem /= od[j];
    off += c[j] * os[j];
  }
  const int last = rank - 1;
  for (int64_t o = lo; o < hi;) {
    /* innermost output axis: a strided run */
    int64_t run = od[last] - c[last];
    if (run > hi - o) run = hi - o;
    const int64_t st = os[last];
    if (elem_bytes == 8) {
      const uint64_t *sp = (const uint64_t *)src + off;
      uint64_t *dp = (uint64_t *)dst + o;
      for (int64_t t = 0; t < run; ++t) dp[t] = sp[t * st];
    } else {
      for (int64_t t = 0; t < run; ++t)
        memcpy(dst + (o + t) * 16, src + (off + t * st) * 16, 16);
    }
    o += run;
    off += run * st;
    c[last] += run;
    for (int j = last; j > 0 && c[j] == od[j]; --j) {
      off -= c[j] * os[j];
      c[j] = 0;
      c[j - 1] += 1;
      off += os[j - 1];
    }
  }
  return 0;
}

int permute_ref(const void *src, void *dst, int rank, const int64_t *dims, const int32_t *perm,
                int elem_bytes) {
  if (rank < 0 || rank > MAXR || (elem_bytes != 8 && elem_bytes != 16)) return -1;
  int seen[MAXR] = {0};
  int64_t n = 1;
  for (int j = 0; j < rank; ++j) {
    if (perm[j] < 0 || perm[j] >= rank || seen[perm[j]] || dims[j] < 1) return -1;
    seen[perm[j]] = 1;
    n *= dims[j];
  }
  if (rank == 0) {
    memcpy(dst, src, (size_t)elem_bytes);
    return 0;
  }
  const int64_t chunk = 1 << 20;
  const int64_t nchunks = (n + chunk - 1) / chunk;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < nchunks; ++k) {
    const int64_t lo = k * chunk, hi = lo + chunk < n ? lo + chunk : n;
    permute_range((const char *)src, (char *)dst, rank, dims, perm, elem_bytes, lo, hi);
  }
  return 0;
}

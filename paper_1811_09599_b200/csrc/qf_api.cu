// Library-wide state: last-error message, launch counter, workspace,
// device queries, and the small elementwise kernels (K4 slicing, K5
// accumulation).
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "qf_common.cuh"

namespace qf {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;
static thread_local const char *g_last_kernel = "";

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

void count_launch(int n) { g_launches += n; }

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return QF_ERR_CUDA;
  }
  count_launch();
  g_last_kernel = what;
  return QF_OK;
}

// Grow-only workspace per device.  A CUDA graph that captured a GEMM keeps
// the workspace pointer it saw, so a buffer is never freed while the library
// may still hand it out: growing retires the old buffer (kept until
// qf_workspace_release, which the caller may only invoke once no captured
// graph uses library workspaces), and growing during stream capture is
// refused (reserve before capturing; the engine's graph runner warms up).
struct Workspace {
  void *ptr = nullptr;
  int64_t bytes = 0;
  std::vector<void *> retired;
};
static std::mutex g_ws_mu;
static std::unordered_map<int, Workspace> g_ws;

void *workspace(int64_t bytes, cudaStream_t stream, int *status) {
  *status = QF_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Workspace &w = g_ws[dev];
  if (w.bytes >= bytes) return w.ptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  if (cap != cudaStreamCaptureStatusNone) {
    set_error("workspace: %lld bytes needed during stream capture (have %lld); reserve first "
              "(qf_workspace_reserve) or run the call once before capturing",
              (long long)bytes, (long long)w.bytes);
    *status = QF_ERR_INVALID;
    return nullptr;
  }
  if (w.ptr) w.retired.push_back(w.ptr);
  int64_t want = bytes < (1 << 20) ? (1 << 20) : bytes;
  cudaError_t e = cudaMalloc(&w.ptr, (size_t)want);
  if (e != cudaSuccess) {
    w.ptr = nullptr;
    w.bytes = 0;
    set_error("workspace allocation of %lld bytes failed: %s", (long long)want,
              cudaGetErrorString(e));
    *status = QF_ERR_MEMORY;
    return nullptr;
  }
  w.bytes = want;
  return w.ptr;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cached[dev] = n;
  return n;
}

// ---------------------------------------------------------------------------
// K4: batched axis gather   dst[b][o][i] = src[o][idx[b]][i]

template <typename E>
__global__ void gather_axis_kernel(const E *__restrict__ src, E *__restrict__ dst, int64_t outer,
                                   int64_t dim, int64_t inner, const int32_t *__restrict__ idx,
                                   int64_t fixed, int64_t nidx) {
  const int64_t per = outer * inner;
  const int64_t total = per * nidx;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t / per;
    int64_t r = t - b * per;
    int64_t o = r / inner;
    int64_t i = r - o * inner;
    int64_t v = idx ? (int64_t)idx[b] : fixed;
    dst[t] = src[(o * dim + v) * inner + i];
  }
}

// late output batching: per-entry base offsets from the bit matrix, and
// the materialising slice  dst[b][o][l] = src[off[b] + ooff[o] + l]
constexpr int BITS_MAX = 64;
struct BitRows {
  int32_t row[BITS_MAX];
  int64_t stride[BITS_MAX];
};

__global__ void bit_offsets_kernel(const int32_t *__restrict__ bits, int64_t ld, int n,
                                   const __grid_constant__ BitRows r, int64_t nb,
                                   int64_t *__restrict__ off) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = 0;
    for (int j = 0; j < n; ++j) o += (int64_t)__ldg(bits + r.row[j] * ld + b) * r.stride[j];
    off[b] = o;
  }
}

// one CTA row of the grid per batch entry (blockIdx.y strides entries);
// 32-bit index math inside an entry when it fits
template <typename E, typename I>
__global__ void gather_rows_kernel(const E *__restrict__ src, E *__restrict__ dst, int64_t nb,
                                   const int64_t *__restrict__ off, I n_outer,
                                   const int64_t *__restrict__ ooff, I L) {
  const I per = n_outer * L;
  for (int64_t b = blockIdx.y; b < nb; b += gridDim.y) {
    const E *s = src + __ldg(off + b);
    E *d = dst + b * (int64_t)per;
    for (I r = blockIdx.x * (I)blockDim.x + threadIdx.x; r < per; r += (I)gridDim.x * blockDim.x) {
      const I o = L == 1 ? r : r / L;
      const I l = r - o * L;
      d[r] = s[(ooff ? __ldg(ooff + o) : (int64_t)o * L) + l];
    }
  }
}

template <typename E>
__global__ void accumulate_kernel(const E *__restrict__ x, E *__restrict__ y, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    E a = x[t], b = y[t];
    b.x += a.x;
    b.y += a.y;
    y[t] = b;
  }
}

// out[e] = (base ? base[e / rep] : (e / rep) * entry) + (e % rep) * stride
__global__ void affine_offsets_kernel(int64_t *__restrict__ out, int64_t n, int64_t rep,
                                      int64_t entry, const int64_t *__restrict__ base,
                                      int64_t stride) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / rep, r = e - q * rep;
    out[e] = (base ? __ldg(base + q) : q * entry) + r * stride;
  }
}

template <typename E>
__global__ void fill_value_kernel(E *__restrict__ y, int64_t n, E v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = v;
}

static int grid_for(int64_t n, int threads) {
  int64_t blocks = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

static int gather_impl(const void *src, void *dst, int64_t outer, int64_t dim, int64_t inner,
                       const int32_t *idx, int64_t fixed, int64_t nidx, int elem_bytes,
                       void *stream) {
  QF_REQUIRE(outer >= 0 && dim >= 1 && inner >= 0 && nidx >= 0,
             "gather: bad extents outer=%lld dim=%lld inner=%lld nidx=%lld", (long long)outer,
             (long long)dim, (long long)inner, (long long)nidx);
  QF_REQUIRE(elem_bytes == 8 || elem_bytes == 16, "gather: elem_bytes must be 8 or 16");
  QF_REQUIRE(idx != nullptr || (fixed >= 0 && fixed < dim), "fix: value %lld out of range [0, %lld)",
             (long long)fixed, (long long)dim);
  int64_t total = outer * inner * nidx;
  if (total == 0) return QF_OK;
  int threads = 256;
  int blocks = grid_for(total, threads);
  cudaStream_t s = as_stream(stream);
  if (elem_bytes == 8)
    gather_axis_kernel<float2><<<blocks, threads, 0, s>>>((const float2 *)src, (float2 *)dst, outer,
                                                          dim, inner, idx, fixed, nidx);
  else
    gather_axis_kernel<double2><<<blocks, threads, 0, s>>>((const double2 *)src, (double2 *)dst,
                                                           outer, dim, inner, idx, fixed, nidx);
  return check_launch("gather_axis");
}

}  // namespace qf

extern "C" {

const char *qf_last_error(void) { return qf::g_err.c_str(); }

const char *qf_last_kernel(void) { return qf::g_last_kernel; }

int qf_version(void) { return 100; }

int qf_device_info(int dev, int *sm_count, int *cc_major, int *cc_minor) {
  QF_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev));
  QF_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev));
  QF_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
  return QF_OK;
}

int qf_gather_axis(const void *src, void *dst, int64_t outer, int64_t dim, int64_t inner,
                   const int32_t *idx, int64_t nidx, int elem_bytes, void *stream) {
  QF_REQUIRE(idx != nullptr || nidx == 0, "gather: idx is NULL");
  return qf::gather_impl(src, dst, outer, dim, inner, idx, 0, nidx, elem_bytes, stream);
}

int qf_fix_axis(const void *src, void *dst, int64_t outer, int64_t dim, int64_t inner,
                int64_t value, int elem_bytes, void *stream) {
  return qf::gather_impl(src, dst, outer, dim, inner, nullptr, value, 1, elem_bytes, stream);
}

int qf_bit_offsets(const int32_t *bits, int64_t ld, int n, const int32_t *rows,
                   const int64_t *strides, int64_t nb, int64_t *off, void *stream) {
  QF_REQUIRE(n >= 0 && n <= qf::BITS_MAX, "bit_offsets: %d rows (max %d)", n, qf::BITS_MAX);
  QF_REQUIRE(nb >= 0 && ld >= nb, "bit_offsets: bad batch %lld / ld %lld", (long long)nb,
             (long long)ld);
  QF_REQUIRE(nb == 0 || (off != nullptr && (n == 0 || bits != nullptr)),
             "bit_offsets: NULL pointer");
  if (nb == 0) return QF_OK;
  qf::BitRows r{};
  for (int j = 0; j < n; ++j) {
    QF_REQUIRE(rows[j] >= 0, "bit_offsets: negative row");
    r.row[j] = rows[j];
    r.stride[j] = strides[j];
  }
  qf::bit_offsets_kernel<<<qf::grid_for(nb, 256), 256, 0, qf::as_stream(stream)>>>(bits, ld, n, r,
                                                                                  nb, off);
  return qf::check_launch("bit_offsets");
}

int qf_gather_rows(const void *src, void *dst, int64_t nb, const int64_t *off, int64_t n_outer,
                   const int64_t *ooff, int64_t L, int elem_bytes, void *stream) {
  QF_REQUIRE(nb >= 0 && n_outer >= 0 && L >= 0, "gather_rows: negative extent");
  QF_REQUIRE(elem_bytes == 8 || elem_bytes == 16, "gather_rows: elem_bytes must be 8 or 16");
  const int64_t total = nb * n_outer * L;
  if (total == 0) return QF_OK;
  QF_REQUIRE(off != nullptr, "gather_rows: off is NULL");
  const int64_t per = n_outer * L;
  const int64_t want = (int64_t)qf::sm_count() * 16;   // CTAs of 256 threads
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((per + 255) / 256, want));
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(nb, std::min<int64_t>(65535, want / gx)));
  dim3 grid((unsigned)gx, (unsigned)gy);
  cudaStream_t s = qf::as_stream(stream);
  const bool small = per < (int64_t(1) << 31);
  if (elem_bytes == 8) {
    if (small)
      qf::gather_rows_kernel<float2, int32_t><<<grid, 256, 0, s>>>(
          (const float2 *)src, (float2 *)dst, nb, off, (int32_t)n_outer, ooff, (int32_t)L);
    else
      qf::gather_rows_kernel<float2, int64_t><<<grid, 256, 0, s>>>(
          (const float2 *)src, (float2 *)dst, nb, off, n_outer, ooff, L);
  } else {
    if (small)
      qf::gather_rows_kernel<double2, int32_t><<<grid, 256, 0, s>>>(
          (const double2 *)src, (double2 *)dst, nb, off, (int32_t)n_outer, ooff, (int32_t)L);
    else
      qf::gather_rows_kernel<double2, int64_t><<<grid, 256, 0, s>>>(
          (const double2 *)src, (double2 *)dst, nb, off, n_outer, ooff, L);
  }
  return qf::check_launch("gather_rows");
}

int qf_accumulate(const void *x, void *y, int64_t n, int elem_bytes, void *stream) {
  QF_REQUIRE(n >= 0, "accumulate: negative length");
  QF_REQUIRE(elem_bytes == 8 || elem_bytes == 16, "accumulate: elem_bytes must be 8 or 16");
  if (n == 0) return QF_OK;
  int threads = 256;
  int blocks = qf::grid_for(n, threads);
  cudaStream_t s = qf::as_stream(stream);
  if (elem_bytes == 8)
    qf::accumulate_kernel<float2><<<blocks, threads, 0, s>>>((const float2 *)x, (float2 *)y, n);
  else
    qf::accumulate_kernel<double2><<<blocks, threads, 0, s>>>((const double2 *)x, (double2 *)y, n);
  return qf::check_launch("accumulate");
}

int qf_fill_zero(void *y, int64_t bytes, void *stream) {
  QF_REQUIRE(bytes >= 0, "fill_zero: negative size");
  if (bytes == 0) return QF_OK;
  QF_CUDA(cudaMemsetAsync(y, 0, (size_t)bytes, qf::as_stream(stream)));
  return QF_OK;
}

int qf_affine_offsets(int64_t *out, int64_t n, int64_t rep, int64_t entry, const int64_t *base,
                      int64_t stride, void *stream) {
  QF_REQUIRE(n >= 0 && rep >= 1, "affine_offsets: bad extents n=%lld rep=%lld", (long long)n,
             (long long)rep);
  if (n == 0) return QF_OK;
  QF_REQUIRE(out != nullptr, "affine_offsets: out is NULL");
  qf::affine_offsets_kernel<<<qf::grid_for(n, 256), 256, 0, qf::as_stream(stream)>>>(
      out, n, rep, entry, base, stride);
  return qf::check_launch("affine_offsets");
}

int qf_fill_value(void *y, int64_t n, double re, double im, int elem_bytes, void *stream) {
  QF_REQUIRE(n >= 0, "fill_value: negative length");
  QF_REQUIRE(elem_bytes == 8 || elem_bytes == 16, "fill_value: elem_bytes must be 8 or 16");
  if (n == 0) return QF_OK;
  QF_REQUIRE(y != nullptr, "fill_value: y is NULL");
  cudaStream_t s = qf::as_stream(stream);
  if (elem_bytes == 8)
    qf::fill_value_kernel<float2><<<qf::grid_for(n, 256), 256, 0, s>>>(
        (float2 *)y, n, make_float2((float)re, (float)im));
  else
    qf::fill_value_kernel<double2><<<qf::grid_for(n, 256), 256, 0, s>>>(
        (double2 *)y, n, make_double2(re, im));
  return qf::check_launch("fill_value");
}

int qf_workspace_reserve(int64_t bytes, void *stream) {
  int st = QF_OK;
  qf::workspace(bytes, qf::as_stream(stream), &st);
  return st;
}

int qf_workspace_release(void) {
  std::lock_guard<std::mutex> lk(qf::g_ws_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = qf::g_ws.find(dev);
  if (it != qf::g_ws.end()) {
    cudaDeviceSynchronize();
    for (void *p : it->second.retired) cudaFree(p);
    if (it->second.ptr) cudaFree(it->second.ptr);
    it->second = qf::Workspace();
  }
  return QF_OK;
}

int64_t qf_launch_count(int reset) {
  int64_t v = qf::g_launches;
  if (reset) qf::g_launches = 0;
  return v;
}

}  // extern "C"

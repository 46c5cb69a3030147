// Library-wide state: last-error message, launch counter, workspace,
// device queries, and the small elementwise kernels (K4 slicing, K5
// accumulation).
#include <mutex>
#include <unordered_map>

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

struct Workspace {
  void *ptr = nullptr;
  int64_t bytes = 0;
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
  if (w.ptr) cudaFreeAsync(w.ptr, stream);
  int64_t want = bytes < (1 << 20) ? (1 << 20) : bytes;
  cudaError_t e = cudaMallocAsync(&w.ptr, (size_t)want, stream);
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
  if (it != qf::g_ws.end() && it->second.ptr) {
    cudaFree(it->second.ptr);
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

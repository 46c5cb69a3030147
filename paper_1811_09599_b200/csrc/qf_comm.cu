// Path sums and the multi-GPU collective of the cut/slice driver.
//
// The reference sums contraction paths sequentially in one process
// (rq/amplitude_engine.py:123 for single amplitudes, :153-157 for open-qubit
// batches).  Here every rank sums a contiguous share of the path list on its
// own GPU (qf_axpy_c64 / qf_dot_c64 on the device) and ONE all-reduce over
// NCCL combines the partial amplitudes (qf_allreduce_c64), enqueued on the
// caller's stream.  NCCL is not linked: the library resolves it at run time
// from the copy already loaded into the process (torch's), else from
// $QF_NCCL_LIB or the system libnccl.so.2, so the library still loads on
// GPU-less build hosts and never mixes two NCCL versions in one process.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "qf_common.cuh"

namespace qf {
namespace comm {

struct Nccl {
  void *handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
  const char *where = "";
};

static std::mutex g_mu;
static Nccl g_nccl;
static bool g_tried = false;
static std::vector<ncclComm_t> g_comms;  // handle = index; destroyed slots hold nullptr

static bool bind(void *h, Nccl &n) {
  n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
  n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
  n.handle = h;
  return n.get_unique_id && n.comm_init_rank && n.all_reduce && n.comm_destroy && n.error_string;
}

// caller holds g_mu
static Nccl *nccl() {
  if (g_tried) return g_nccl.handle ? &g_nccl : nullptr;
  g_tried = true;
  // 1) a libnccl already mapped into the process (torch's bundled copy)
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *nm : names) {
    void *h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
    if (h && bind(h, g_nccl)) {
      g_nccl.where = "already loaded";
      return &g_nccl;
    }
  }
  // 2) an explicit path, then the loader's search path
  const char *env = getenv("QF_NCCL_LIB");
  const char *tries[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char *nm : tries) {
    if (!nm || !*nm) continue;
    void *h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h && bind(h, g_nccl)) {
      g_nccl.where = nm;
      return &g_nccl;
    }
  }
  g_nccl = Nccl();
  return nullptr;
}

#define QF_NCCL(n, call)                                                           \
  do {                                                                             \
    ncclResult_t r_ = (call);                                                      \
    if (r_ != ncclSuccess) {                                                       \
      qf::set_error("%s failed: %s", #call, (n)->error_string(r_));                \
      return QF_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

// y[i] += alpha * x[i]  (complex64, grid-stride, 16-byte pairs when aligned)
__global__ void axpy_c64_kernel(int64_t n, float ar, float ai, const float2 *__restrict__ x,
                                float2 *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 a = x[i];
    float2 b = y[i];
    b.x = fmaf(ar, a.x, fmaf(-ai, a.y, b.x));
    b.y = fmaf(ar, a.y, fmaf(ai, a.x, b.y));
    y[i] = b;
  }
}

// out[b] = sum_i x[b*sx + i] * y[b*sy + i]  (one warp per entry, fp32
// accumulation in two interleaved partial sums, as the batched path-sum dot
// of the GEMM engines)
__global__ void dot_c64_kernel(int64_t batch, int64_t n, const float2 *__restrict__ x, int64_t sx,
                               const float2 *__restrict__ y, int64_t sy, float2 *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (b >= batch) return;
  const float2 *xb = x + b * sx, *yb = y + b * sy;
  float re0 = 0.f, im0 = 0.f, re1 = 0.f, im1 = 0.f;
  int64_t i = lane;
  for (; i + 32 < n; i += 64) {
    const float2 a0 = __ldg(xb + i), w0 = __ldg(yb + i);
    const float2 a1 = __ldg(xb + i + 32), w1 = __ldg(yb + i + 32);
    re0 = fmaf(a0.x, w0.x, fmaf(-a0.y, w0.y, re0));
    im0 = fmaf(a0.x, w0.y, fmaf(a0.y, w0.x, im0));
    re1 = fmaf(a1.x, w1.x, fmaf(-a1.y, w1.y, re1));
    im1 = fmaf(a1.x, w1.y, fmaf(a1.y, w1.x, im1));
  }
  for (; i < n; i += 32) {
    const float2 a = __ldg(xb + i), w = __ldg(yb + i);
    re0 = fmaf(a.x, w.x, fmaf(-a.y, w.y, re0));
    im0 = fmaf(a.x, w.y, fmaf(a.y, w.x, im0));
  }
  float re = re0 + re1, im = im0 + im1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) out[b] = make_float2(re, im);
}

}  // namespace comm
}  // namespace qf

extern "C" {

int qf_nccl_available(void) {
  std::lock_guard<std::mutex> lk(qf::comm::g_mu);
  return qf::comm::nccl() ? 1 : 0;
}

int qf_nccl_unique_id(void *uid, int64_t nbytes) {
  QF_REQUIRE(uid != nullptr && nbytes >= (int64_t)sizeof(ncclUniqueId),
             "nccl_unique_id: need a %d-byte buffer", (int)sizeof(ncclUniqueId));
  std::lock_guard<std::mutex> lk(qf::comm::g_mu);
  qf::comm::Nccl *n = qf::comm::nccl();
  if (!n) {
    qf::set_error("nccl_unique_id: libnccl.so.2 not found (set QF_NCCL_LIB)");
    return QF_ERR_UNSUPPORTED;
  }
  ncclUniqueId id;
  QF_NCCL(n, n->get_unique_id(&id));
  memcpy(uid, &id, sizeof(id));
  return QF_OK;
}

int qf_nccl_init(const void *uid, int nranks, int rank, int dev, int *handle) {
  QF_REQUIRE(uid != nullptr && handle != nullptr, "nccl_init: NULL argument");
  QF_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "nccl_init: rank %d of %d", rank, nranks);
  qf::comm::Nccl *n;
  {
    std::lock_guard<std::mutex> lk(qf::comm::g_mu);
    n = qf::comm::nccl();
  }
  if (!n) {
    qf::set_error("nccl_init: libnccl.so.2 not found (set QF_NCCL_LIB)");
    return QF_ERR_UNSUPPORTED;
  }
  QF_CUDA(cudaSetDevice(dev));
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t comm = nullptr;
  // collective over all ranks: called without the lock so one process may
  // drive several devices from several threads
  QF_NCCL(n, n->comm_init_rank(&comm, nranks, id, rank));
  std::lock_guard<std::mutex> lk(qf::comm::g_mu);
  qf::comm::g_comms.push_back(comm);
  *handle = (int)qf::comm::g_comms.size() - 1;
  return QF_OK;
}

int qf_nccl_destroy(int handle) {
  std::lock_guard<std::mutex> lk(qf::comm::g_mu);
  QF_REQUIRE(handle >= 0 && handle < (int)qf::comm::g_comms.size() && qf::comm::g_comms[handle],
             "nccl_destroy: bad handle %d", handle);
  qf::comm::Nccl *n = qf::comm::nccl();
  QF_NCCL(n, n->comm_destroy(qf::comm::g_comms[handle]));
  qf::comm::g_comms[handle] = nullptr;
  return QF_OK;
}

int qf_allreduce_c64(int handle, void *buf, int64_t count, void *stream) {
  qf::comm::Nccl *n;
  ncclComm_t comm;
  {
    std::lock_guard<std::mutex> lk(qf::comm::g_mu);
    QF_REQUIRE(handle >= 0 && handle < (int)qf::comm::g_comms.size() && qf::comm::g_comms[handle],
               "allreduce: bad handle %d", handle);
    n = qf::comm::nccl();
    comm = qf::comm::g_comms[handle];
  }
  QF_REQUIRE(count >= 0 && (count == 0 || buf != nullptr), "allreduce: bad buffer");
  if (count == 0) return QF_OK;
  // complex64 as float pairs: the sum is componentwise
  QF_NCCL(n, n->all_reduce(buf, buf, (size_t)(2 * count), ncclFloat32, ncclSum, comm,
                           qf::as_stream(stream)));
  return QF_OK;
}

int qf_axpy_c64(int64_t n, float alpha_re, float alpha_im, const void *x, void *y, void *stream) {
  QF_REQUIRE(n >= 0, "axpy: negative length");
  if (n == 0) return QF_OK;
  QF_REQUIRE(x != nullptr && y != nullptr, "axpy: NULL pointer");
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)qf::sm_count() * 16);
  qf::comm::axpy_c64_kernel<<<(unsigned)blocks, 256, 0, qf::as_stream(stream)>>>(
      n, alpha_re, alpha_im, (const float2 *)x, (float2 *)y);
  return qf::check_launch("axpy_c64");
}

int qf_dot_c64(int64_t batch, int64_t n, const void *x, int64_t stride_x, const void *y,
               int64_t stride_y, void *out, void *stream) {
  QF_REQUIRE(batch >= 0 && n >= 0, "dot: negative extent");
  if (batch == 0) return QF_OK;
  QF_REQUIRE(out != nullptr && (n == 0 || (x != nullptr && y != nullptr)), "dot: NULL pointer");
  QF_REQUIRE(batch == 1 || (stride_x >= n && stride_y >= n), "dot: strides shorter than n");
  const int64_t blocks = (batch + 7) / 8;
  QF_REQUIRE(blocks < ((int64_t)1 << 31), "dot: batch too large");
  qf::comm::dot_c64_kernel<<<(unsigned)blocks, 256, 0, qf::as_stream(stream)>>>(
      batch, n, (const float2 *)x, stride_x, (const float2 *)y, stride_y, (float2 *)out);
  return qf::check_launch("dot_c64");
}

}  // extern "C"

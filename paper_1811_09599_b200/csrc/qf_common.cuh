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

// K2 -- tcgen05 3xTF32 complex GEMM (placeholder until the kernel lands).
#include "qf_common.cuh"

namespace qf {
struct GemmArgs;
bool tc3_eligible(const GemmArgs &) { return false; }
int gemm_tc3(const GemmArgs &, cudaStream_t) {
  set_error("tcgen05 GEMM not built yet");
  return QF_ERR_UNSUPPORTED;
}
}  // namespace qf

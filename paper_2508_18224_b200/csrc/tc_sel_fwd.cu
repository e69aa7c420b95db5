// tcgen05 selected-attention kernels (placeholder until the tensor-core path lands).
#include "tc_plan.cuh"

namespace fsa {

bool tc_fwd_supported(const fsa_shape&, int) { return false; }
bool tc_bwd_supported(const fsa_shape&, int) { return false; }

int tc_sel_fwd(const fsa_shape*, const void*, const void*, const void*, const int32_t*,
               const int32_t*, void*, void*, cudaStream_t) {
  set_error("tensor-core forward not available");
  return FSA_ERR_UNSUPPORTED;
}
int tc_sel_bwd(const fsa_shape*, const void*, const void*, const void*, const void*, const void*,
               const void*, const int32_t*, const int32_t*, void*, int, void*, void*,
               cudaStream_t) {
  set_error("tensor-core backward not available");
  return FSA_ERR_UNSUPPORTED;
}

}  // namespace fsa

// C-ABI plumbing: thread-local error message, device check, buffer plan.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"
#include "tc_plan.cuh"

namespace fsa {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA error %s", what, cudaGetErrorString(e));
    return FSA_ERR_CUDA;
  }
  return FSA_OK;
}

}  // namespace fsa

extern "C" const char* fsa_last_error(void) { return fsa::g_err; }

extern "C" int fsa_abi_version(void) { return FSA_ABI_VERSION; }

extern "C" int fsa_device_check(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    fsa::set_error("no CUDA device: %s", cudaGetErrorString(e));
    return FSA_ERR_CUDA;
  }
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  if (p.major != 10) {
    fsa::set_error("device %s is sm_%d%d; this library is built for sm_100a", p.name, p.major,
                   p.minor);
    return FSA_ERR_UNSUPPORTED;
  }
  return FSA_OK;
}

extern "C" int64_t fsa_partial_rows(const fsa_shape* s, int dtype) {
  // tensor-core path: item-major tiles of 128 rows (common.cuh, work plan);
  // otherwise slot-indexed rows [h][N][T]
  if (fsa::tc_fwd_supported(*s, dtype)) return fsa::plan_max_items(*s) * 128;
  return s->h * s->N * s->T;
}

extern "C" int fsa_buffer_dtypes(const fsa_shape* s, int dtype, int* obuf_dtype, int* dqbuf_dtype) {
  const bool tc = fsa::tc_fwd_supported(*s, dtype);
  if (obuf_dtype) *obuf_dtype = tc ? FSA_DT_F16 : (dtype == FSA_DT_F64 ? FSA_DT_F64 : FSA_DT_F32);
  const bool tcb = fsa::tc_bwd_supported(*s, dtype);
  if (dqbuf_dtype) *dqbuf_dtype = tcb ? FSA_DT_F16R : (dtype == FSA_DT_F64 ? FSA_DT_F64 : FSA_DT_F32);
  return FSA_OK;
}

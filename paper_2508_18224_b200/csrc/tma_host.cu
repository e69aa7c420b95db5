// Host-side TMA descriptors (cuTensorMapEncodeTiled) for the token-major
// [N][heads][128] bf16 tensors the tcgen05 kernels read as 128-byte-row,
// SWIZZLE_128B tiles: a box of (64 features, `heads_box` heads, `tok_box`
// tokens) lands as rows (token, head) x 128 B -- the canonical K-major SW128
// layout the UMMA descriptors expect (tc_common.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include "tc_plan.cuh"

namespace fsa {

// The driver entry point is resolved at run time (cudaGetDriverEntryPoint),
// so the library has no link-time dependency on libcuda (it must load on the
// CPU build host, where only the symbol table is checked).
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

int make_tmap_tokens(CUtensorMap* map, const void* base, int64_t N, int64_t heads, int heads_box,
                     int tok_box) {
  const cuuint64_t dims[3] = {128, (cuuint64_t)heads, (cuuint64_t)N};
  const cuuint64_t strides[2] = {(cuuint64_t)(128 * 2), (cuuint64_t)(heads * 128 * 2)};
  const cuuint32_t box[3] = {64, (cuuint32_t)heads_box, (cuuint32_t)tok_box};
  const cuuint32_t estr[3] = {1, 1, 1};
  EncodeTiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    return FSA_ERR_CUDA;
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                                      const_cast<void*>(base), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return FSA_ERR_CUDA;
  }
  return FSA_OK;
}

}  // namespace fsa

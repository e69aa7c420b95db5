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

// fp32 token-major [N][heads][128], box (32 floats = 128 B, heads_box, tok_box), SW128:
// the TMA store / reduce-add target of a 128-row accumulator tile, 4 column quarters
int make_tmap_tokens_f32(CUtensorMap* map, const void* base, int64_t N, int64_t heads, int heads_box,
                         int tok_box) {
  const cuuint64_t dims[3] = {128, (cuuint64_t)heads, (cuuint64_t)N};
  const cuuint64_t strides[2] = {(cuuint64_t)(128 * 4), (cuuint64_t)(heads * 128 * 4)};
  const cuuint32_t box[3] = {32, (cuuint32_t)heads_box, (cuuint32_t)tok_box};
  const cuuint32_t estr[3] = {1, 1, 1};
  EncodeTiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    return FSA_ERR_CUDA;
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (f32 tokens) failed (%d)", (int)r);
    return FSA_ERR_CUDA;
  }
  return FSA_OK;
}

// 2-D view [rows][128] bf16 of a row-major tensor, box (64, box_rows), SW128:
// the tile::gather4 / tile::scatter4 operand (4 arbitrary rows per instruction).
int make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int box_rows) {
  const cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(128 * 2)};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  EncodeTiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    return FSA_ERR_CUDA;
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (rows) failed (%d)", (int)r);
    return FSA_ERR_CUDA;
  }
  return FSA_OK;
}

namespace {
// debug: gather 4-row groups idx[] of src into an SW128 tile, then write the
// tile back un-swizzled to out (row i = src[idx[i]]), and scatter it again to
// out2 rows idx2[] with tile::scatter4.
__global__ void gather4_test_kernel(const __grid_constant__ CUtensorMap tm,
                                    const __grid_constant__ CUtensorMap tm2, const int32_t* idx,
                                    const int32_t* idx2, int n, __nv_bfloat16* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bar = sb + 65536;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)(n * 256))
                 : "memory");
    for (int g = 0; g < n / 4; ++g)
      for (int hf = 0; hf < 2; ++hf)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sb + hf * (uint32_t)(n * 128) + g * 512u),
            "l"(&tm), "r"(hf * 64), "r"(idx[4 * g]), "r"(idx[4 * g + 1]), "r"(idx[4 * g + 2]),
            "r"(idx[4 * g + 3]), "r"(bar)
            : "memory");
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0, 1, 0, P; }"
                 : "=r"(ok) : "r"(bar), "r"(0u) : "memory");
  }
  for (int e = threadIdx.x; e < n * 16; e += blockDim.x) {  // 16-byte chunks
    const int row = e / 16, c = e % 16, hf = c >> 3, cc = c & 7;
    const uint4 v = *reinterpret_cast<const uint4*>(smem + hf * n * 128 + row * 128 + ((cc ^ (row & 7)) << 4));
    reinterpret_cast<uint4*>(out + (int64_t)row * 128)[c] = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int g = 0; g < n / 4; ++g)
      for (int hf = 0; hf < 2; ++hf)
        asm volatile(
            "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group"
            " [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&tm2), "r"(hf * 64), "r"(idx2[4 * g]),
            "r"(idx2[4 * g + 1]), "r"(idx2[4 * g + 2]), "r"(idx2[4 * g + 3]),
            "r"(sb + hf * (uint32_t)(n * 128) + g * 512u)
            : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
}  // namespace

}  // namespace fsa

#ifdef FSA_TRACE
extern "C" int fsa_debug_gather4_test(const void* src, int64_t rows, const int32_t* idx,
                                      const int32_t* idx2, int n, int box_rows, void* out,
                                      void* out2, int64_t rows2, void* stream) {
  CUtensorMap tm, tm2;
  int rc = fsa::make_tmap_rows(&tm, src, rows, box_rows);
  if (!rc) rc = fsa::make_tmap_rows(&tm2, out2, rows2, box_rows);
  if (rc) return rc;
  cudaFuncSetAttribute(fsa::gather4_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  fsa::gather4_test_kernel<<<1, 128, 70000, (cudaStream_t)stream>>>(tm, tm2, idx, idx2, n,
                                                                    (__nv_bfloat16*)out);
  return fsa::check_launch("gather4_test");
}
#endif

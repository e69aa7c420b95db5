// Dispatch predicates + entry points of the tcgen05 tensor-core kernels.
#pragma once
#include "common.cuh"

namespace fsa {

// bf16, d_K = d_V = 128, B_K = 64: the BASELINE.json shapes (tc_sel_fwd.cu / tc_sel_bwd.cu).
bool tc_fwd_supported(const fsa_shape& s, int dtype);
bool tc_bwd_supported(const fsa_shape& s, int dtype);

// Per-kv-head power-of-two scales of the fp16 backward operands
// (fsa_stage_f16_ops): x16 = x * s.  q: Q (per kv group), k: K, v: V, o: dOut.
struct F16Scales {
  const float *q, *k, *v, *o;
};
// the scale blocks of an fsa_stage_f16_ops `scales` buffer ([4][2 h_K])
inline F16Scales f16_scales_of(const float* scales, int64_t h_K) {
  return F16Scales{scales, scales + 2 * h_K, scales + 4 * h_K, scales + 6 * h_K};
}

// V: the fp16 staged copy (stage_f16).  mode FSA_FWD_LOCAL: obuf fp16
// item-major partial rows in the V16 scale + item-major (m_i, l_i) in ml;
// FSA_FWD_STATS: slot-indexed (m_i, l_i) [h][N][T] in ml (V unused);
// FSA_FWD_GLOBAL: obuf fp32 slot-indexed [h][N][T][128] rows exp(z - m_global) V_i
int tc_sel_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V16,
               const int32_t* offsets, const int32_t* qlist, const int32_t* work, void* obuf,
               void* ml, cudaStream_t st, int mode = FSA_FWD_LOCAL,
               const float* m_global = nullptr, const float* vscale = nullptr);
// Q, K, V, dOut: the fp16 staged copies, sc their scales
int tc_sel_bwd(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
               const void* lse, const void* delta, const int32_t* offsets, const int32_t* qlist,
               const int32_t* work, void* dq_buf, int dqbuf_dtype, void* dK, void* dV,
               F16Scales sc, cudaStream_t st);

// fp16 staging of a [rows][heads][d] bf16 / f32 tensor with a power-of-two
// scale per head (f16_stage.cu); vscale [2 heads]: scales, then scratch
int stage_f16(int src_dtype, const void* x, int64_t rows, int64_t heads, int64_t d, void* y,
              float* vscale, cudaStream_t st);

// query-outer forward (tc_qo_fwd.cu): sliding window and compressed attention
bool tc_qo_supported(const fsa_shape& s, int dtype);
int tc_slide_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V16,
                 const float* vscale, void* out, void* lse, cudaStream_t st);
size_t tc_cmp_workspace_bytes(const fsa_shape* s);
// Q16 / qscale: the fsa_stage_f16_ops copy of Q and its scale block (the
// compressed attention's S runs in fp16, as its backward recomputes it)
int tc_cmp_fwd(const fsa_shape* s, const void* Q, const void* Q16, const float* qscale,
               const void* Kc, const void* Vc, void* out, void* lse, void* scores, void* workspace,
               cudaStream_t st);

// sliding-window backward on the FSA backward kernel (tc_sel_bwd.cu)
size_t tc_slide_bwd_workspace_bytes(const fsa_shape* s);
int tc_slide_bwd(const fsa_shape* s, const void* Q, const void* K, const void* V,
                 const void* dOut, const void* lse, const void* delta, void* dQ, void* dK,
                 void* dV, void* workspace, int accumulate, F16Scales sc, cudaStream_t st);

// query-outer sliding-window dQ (tc_slide_dq.cu); accumulate: dQ += (fp32)
int tc_slide_dq(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
                const void* lse, const void* delta, void* dQ, int accumulate, F16Scales sc,
                cudaStream_t st);

// compressed-branch backward on the same kernels (tc_sel_bwd.cu, tc_slide_dq.cu):
// dK_cmp / dV_cmp partial slabs per token chunk, and dQ += over the pooled rows
int64_t cmp_chunk_tokens(const fsa_shape* s);
int tc_cmp_bwd_kv(const fsa_shape* s, const void* Q, const void* Kb, const void* Vb,
                  const void* dOut, const void* lse, const void* delta, void* dKp, void* dVp,
                  int32_t* counter, F16Scales sc, cudaStream_t st);
int tc_cmp_dq(const fsa_shape* s, const void* Q, const void* Kb, const void* Vb, const void* dOut,
              const void* lse, const void* delta, void* dQ, F16Scales sc, cudaStream_t st);

// vectorised merge of the fp16 slot partials / reduce of the fp16 dq partials
// for d = 128, any T (merge_fast.cu); out / lse / m / l / dQ / addend fp32.
// out_cmp / out_slide / tau / out_comb non-null: the gated combine in the same pass.
bool fast_reduce_ok(const fsa_shape& s);
int merge_f16_fast(const fsa_shape* s, const int32_t* idx, const int32_t* work, const void* obuf,
                   const void* ml, const float* vscale, void* out, void* lse, void* m_out,
                   void* l_out, cudaStream_t st, const void* out_cmp = nullptr,
                   const void* out_slide = nullptr, const void* tau = nullptr,
                   void* out_comb = nullptr);
int dq_reduce_f16r(const fsa_shape* s, const int32_t* idx, const void* dq, void* dQ,
                   cudaStream_t st, const void* addend = nullptr);

int num_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) holds per device: set it the
// first time a kernel launches on each device (one bit per device in `done`).
template <typename K>
inline void ensure_smem_attr(K kern, int bytes, unsigned long long& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(&done, __ATOMIC_ACQUIRE) & bit) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  __atomic_fetch_or(&done, bit, __ATOMIC_RELEASE);
}

}  // namespace fsa
#include <cuda.h>
namespace fsa {
// TMA descriptor of a token-major [N][heads][128] bf16 tensor, box (64, heads_box, tok_box)
int make_tmap_tokens(CUtensorMap* map, const void* base, int64_t N, int64_t heads, int heads_box,
                     int tok_box);
// fp32 [N][heads][128], box (32, heads_box, tok_box), SW128 (accumulator-tile stores)
int make_tmap_tokens_f32(CUtensorMap* map, const void* base, int64_t N, int64_t heads, int heads_box,
                         int tok_box);
// 2-D [rows][128] bf16 view, box (64, box_rows): the tile::gather4 / scatter4 operand
int make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int box_rows);

}  // namespace fsa

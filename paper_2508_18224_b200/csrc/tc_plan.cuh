// Dispatch predicates + entry points of the tcgen05 tensor-core kernels.
#pragma once
#include "common.cuh"

namespace fsa {

// bf16, d_K = d_V = 128, B_K = 64: the BASELINE.json shapes (tc_sel_fwd.cu / tc_sel_bwd.cu).
bool tc_fwd_supported(const fsa_shape& s, int dtype);
bool tc_bwd_supported(const fsa_shape& s, int dtype);

int tc_sel_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V,
               const int32_t* offsets, const int32_t* qlist, const int32_t* work, void* obuf,
               void* ml, cudaStream_t st);
int tc_sel_bwd(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
               const void* lse, const void* delta, const int32_t* offsets, const int32_t* qlist,
               const int32_t* work, void* dq_buf, int dqbuf_dtype, void* dK, void* dV,
               cudaStream_t st);

// query-outer forward (tc_qo_fwd.cu): sliding window and compressed attention
bool tc_qo_supported(const fsa_shape& s, int dtype);
bool tc_cmp_scores_fused(const fsa_shape& s);
int tc_slide_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V, void* out,
                 void* lse, cudaStream_t st, int out_bf16 = 0);
size_t tc_cmp_workspace_bytes(const fsa_shape* s);
int tc_cmp_fwd(const fsa_shape* s, const void* Q, const void* Kc, const void* Vc, void* out,
               void* lse, void* scores, void* workspace, cudaStream_t st, int out_bf16 = 0);

// sliding-window backward on the FSA backward kernel (tc_sel_bwd.cu)
size_t tc_slide_bwd_workspace_bytes(const fsa_shape* s);
int tc_slide_bwd(const fsa_shape* s, const void* Q, const void* K, const void* V,
                 const void* dOut, const void* lse, const void* delta, void* dQ, void* dK,
                 void* dV, void* workspace, int accumulate, cudaStream_t st);

// query-outer sliding-window dQ (tc_slide_dq.cu); accumulate: dQ += (fp32)
int tc_slide_dq(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
                const void* lse, const void* delta, void* dQ, int accumulate, cudaStream_t st,
                int out_bf16 = 0);

// compressed-branch backward on the same kernels (tc_sel_bwd.cu, tc_slide_dq.cu):
// dK_cmp / dV_cmp partial slabs per token chunk, and dQ += over the pooled rows
int64_t cmp_chunk_tokens(const fsa_shape* s);
int tc_cmp_bwd_kv(const fsa_shape* s, const void* Q, const void* Kb, const void* Vb,
                  const void* dOut, const void* lse, const void* delta, void* dKp, void* dVp,
                  int32_t* counter, cudaStream_t st);
int tc_cmp_dq(const fsa_shape* s, const void* Q, const void* Kb, const void* Vb, const void* dOut,
              const void* lse, const void* delta, void* dQ, cudaStream_t st);

// vectorised bf16 merge / dQ reduce for d = 128, T <= 32 (merge_fast.cu)
bool fast_reduce_ok(const fsa_shape& s);
int merge_bf16_fast(const fsa_shape* s, const int32_t* idx, const void* obuf, const void* ml,
                    void* out, void* lse, void* m_out, void* l_out, cudaStream_t st);
int merge_combine_bf16_fast(const fsa_shape* s, const int32_t* idx, const void* obuf,
                            const void* ml, const void* out_cmp, const void* out_slide,
                            const void* tau, void* out_sel, void* lse, void* out, cudaStream_t st,
                            int narrow = 0);
int dq_reduce_bf16_fast(const fsa_shape* s, const int32_t* idx, const void* dq, void* dQ,
                        cudaStream_t st, const void* addend = nullptr, int addend_bf16 = 0);

int num_sms();

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

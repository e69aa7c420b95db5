/*
 * fsa_b200.h -- C-ABI of the B200-native Flash Sparse Attention (NSA) operator path.
 *
 * The reference (`blockattn`, /root/reference/pkg/src/blockattn) exposes this
 * path as Python operator functions over float64 numpy arrays; its only native
 * boundary is the per-(head, block) Cython kernel set in `_kernels/_core.pyx`
 * selected through `_kernels/__init__.py:13-56`.  That granularity is one task
 * per call, far too fine for a GPU launch, so this ABI sits one level up: one
 * entry point per reference *operator* (cited per function below).  The Python
 * host layer (the paper_2508_18224_b200 package) binds these with ctypes and mirrors
 * the reference's names, argument order and exceptions.
 *
 * Conventions
 *  - Plain C: raw device pointers, int64 sizes, a cudaStream_t passed as void*.
 *  - The caller allocates every output and workspace; nothing here allocates.
 *  - Every function returns FSA_OK (0) or an error code; fsa_last_error()
 *    returns a thread-local message.  Launches are stream-ordered and
 *    reentrant; there is no global mutable state besides that message.
 *  - Storage layouts (row-major, last index contiguous).  The reference's
 *    logical (token, feature, head) tensors are permuted views of these:
 *      Q   [N][h][d_K]      K [N][h_K][d_K]     V [N][h_K][d_V]
 *      out [N][h][d_V]      lse, m, l, delta [h][N]
 *      scores [h_K][N][b]   idx [h_K][N][T] int32 (ascending, -1 padded)
 *      obuf [h][N][T][d_V]  ml [h][N][T][2]     dq_buf [h][N][T][d_K]
 *      inverse CSR: offsets [h_K][b+1] int32, qlist [h_K][N*T] int32 holding
 *      t*T + slot, ascending t inside each block (selection.py:123-169).
 *  - dtype: FSA_DT_F32 / FSA_DT_F64 / FSA_DT_BF16 for Q/K/V/dOut.  The
 *    "accumulator" type is f64 for f64 inputs and f32 otherwise; branch
 *    outputs (out of merge / compressed / sliding), lse/m/l/delta, compressed
 *    KV, scores and gradients are stored in it (the reference returns f64
 *    everywhere; keeping bf16 runs' intermediates in f32 keeps delta exact).
 */
#ifndef FSA_B200_H
#define FSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSA_OK 0
#define FSA_ERR_INVALID 1
#define FSA_ERR_CUDA 2
#define FSA_ERR_UNSUPPORTED 3

#define FSA_ABI_VERSION 4

/* Element types.  FSA_DT_F16 and FSA_DT_F16R are buffer formats of the bf16
 * tensor-core path, never input dtypes:
 *   F16  obuf [R][128] fp16 partials O_i / l_i in the power-of-two scale s_kh
 *        of the fsa_v_to_f16 copy of V (the merge divides by vscale[kh]), ml
 *        [R] (m_i, l_i) fp32 pairs, R = fsa_partial_rows().  ITEM-MAJOR rows:
 *        item n of the work plan (fsa_build_inverse) owns rows [128 n, 128 n +
 *        128), row 128 n + (p % tpi) g + hh holding list position p of the
 *        item's task for group head hh (tpi = 128 / g tokens per item);
 *   F16R dq_buf = fp16 rows [h][N][T][128] (slot-indexed) followed by 4 int8
 *        exponents per row [h][N][T] (one per 32 columns, int32-packed, low
 *        byte first): value = fp16 * 2^-e (chunk max in [2^14, 2^15)) --
 *        bytes h N T (2 * 128 + 4).
 * Every other obuf / ml / dq_buf is slot-indexed [h][N][T][d] (R = h N T). */
typedef enum {
  FSA_DT_F32 = 0, FSA_DT_F64 = 1, FSA_DT_BF16 = 2, FSA_DT_I32 = 3, FSA_DT_F16 = 4, FSA_DT_F16R = 5
} fsa_dtype;

/* Resolved AttentionConfig (config.py:30-104); scale = 1/sqrt(d_K). */
typedef struct fsa_shape {
  int64_t N, d_K, d_V, h, h_K, B_K, T, W;
  double scale;
} fsa_shape;

/* Selection-validation flag bits, in the reference's check order (selection.py:59-75). */
#define FSA_SEL_EMPTY_ROW 1
#define FSA_SEL_AFTER_SENTINEL 2
#define FSA_SEL_OUT_OF_RANGE 4
#define FSA_SEL_NON_CAUSAL 8
#define FSA_SEL_DUPLICATE 16
#define FSA_SEL_NOT_INCREASING 32

/* Selected-forward modes (kv_major.py:105-204). */
#define FSA_FWD_LOCAL 0  /* fused: per-block local (m_i,l_i) + O_i/l_i      */
#define FSA_FWD_STATS 1  /* compute_softmax_stats partials only (kv_major.py:105-149)      */
#define FSA_FWD_GLOBAL 2 /* block_pass_forward: exp(z - m_global) @ V_i (kv_major.py:152) */

/* Merge modes (kv_major.py:207-242, :137-149). */
#define FSA_MERGE_LOCAL 0  /* flash-decoding combine of LOCAL partials -> out, lse (+m,l) */
#define FSA_MERGE_STATS 1  /* ascending-block (m,l) merge -> m, l (+ shared max)          */
#define FSA_MERGE_REDUCE 2 /* sum of GLOBAL partials / l -> out, lse = m + log l           */

const char* fsa_last_error(void);
int fsa_abi_version(void);
/* 0 when a compute-capability 10.x device is current, else an error code. */
int fsa_device_check(void);

/* Buffer dtypes the library will read/write for a given problem: obuf (LOCAL
 * mode) and dq_buf.  bf16 problems on the tensor-core path (d = 128, B_K = 64)
 * use FSA_DT_F16 obuf and FSA_DT_F16R dq_buf. */
int fsa_buffer_dtypes(const fsa_shape* s, int dtype, int* obuf_dtype, int* dqbuf_dtype);

/* fp16 staging of V for the tensor-core P.V products (bf16 path): V16 [N][h_K][d_V]
 * = fp16(V * s_kh), s_kh = 2^(15 - k) for max|V[:, kh, :]| = f 2^k, f in [0.5, 1).
 * vscale [2 h_K] floats: s_kh in [0, h_K), scratch after.  dtype BF16 or F32. */
int fsa_v_to_f16(const fsa_shape* s, int dtype, const void* V, void* V16, float* vscale,
                 void* stream);

/* fp16 operands of the bf16 tensor-core BACKWARD (all of its products run
 * fp16 x fp16 -> fp32: P and dS keep 11 mantissa bits where bf16 keeps 8, the
 * rounding that otherwise drives elementwise dQ / dK / dV errors -- see
 * tools/emulate_bf16.py).  Q16 [N][h][d_K], K16 [N][h_K][d_K], V16 [N][h_K][d_V],
 * dO16 [N][h][d_V] = fp16(x * s) with one power-of-two scale s per kv head (for
 * Q and dOut: per kv group, over its g heads), max |x s| in [2^14, 2^15): exact
 * for every bf16 value above 2^-24 of the maximum.  scales [4][2 h_K] floats:
 * s_Q, s_K, s_V, s_dO at offsets 0, 2 h_K, 4 h_K, 6 h_K (the upper half of each
 * block is scratch).  A NULL source skips that operand (its scale block is left
 * untouched: V16 and its scale can be the forward's fsa_v_to_f16 copy). */
int fsa_stage_f16_ops(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
                      const void* dOut, void* Q16, void* K16, void* V16, void* dO16, float* scales,
                      void* stream);

/* compress_kv (branches.py:34-44): block means K_cmp/V_cmp [b][h_K][d] and the
 * running prefix means of the first min(B_K-1, N) rows [n_pref][h_K][d]; acc dtype. */
int fsa_compress_kv(const fsa_shape* s, int dtype, const void* K, const void* V, void* K_cmp,
                    void* V_cmp, void* K_prefix, void* V_prefix, void* stream);

/* importance_scores_from_compressed (selection.py:105-120): scores [h_K][N][b]
 * (acc dtype) = group mean of Q.K_cmp / sqrt(d_K) for every block. */
int fsa_importance_scores(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp,
                          void* scores, void* stream);

/* select_topk_blocks (selection.py:78-102): bit-exact own-block + top-(T-1),
 * ties to the lower block index, -inf/NaN unselectable.  score_dtype F32 or F64. */
int fsa_select_topk(const fsa_shape* s, int score_dtype, const void* scores, int32_t* idx,
                    void* stream);

/* validate_selection (selection.py:49-75): ORs FSA_SEL_* bits into *flags (device int32). */
int fsa_validate_selection(const fsa_shape* s, const int32_t* idx, int32_t* flags, void* stream);

/* build_inverse_index (selection.py:146-169) as CSR; flags as above (nullable).
 * work (nullable; fsa_work_plan_bytes, int32) receives the tensor-core work
 * plan: tasks task = kh * b + i (head-major), each cut into ceil(n_valid /
 * (128/g)) items of <= 128 (token, head) rows; work[task] is the exclusive
 * prefix of item counts (work[h_K b] the total), work[h_K b + 1] a scheduler
 * counter, and from int32 offset ceil((h_K b + 2) / 32) * 32 the list position
 * of every live selection entry [h_K][N][T] (the item-major buffer address). */
size_t fsa_work_plan_bytes(const fsa_shape* s);
/* Rows of the obuf / ml partial buffers for dtype's path (item-major on the
 * tensor-core path: 128 x an upper bound of the item count; else h N T). */
int64_t fsa_partial_rows(const fsa_shape* s, int dtype);
size_t fsa_inverse_workspace_bytes(const fsa_shape* s);
int fsa_build_inverse(const fsa_shape* s, const int32_t* idx, void* workspace, int32_t* offsets,
                      int32_t* qlist, int32_t* work, int32_t* flags, void* stream);

/* FSA block pass (kv_major.py:105-204, _core.pyx:49-94): one task per
 * (KV head, block) loads K_i/V_i once and serves all g query heads of the
 * gathered rows.  m_global ([h][N], acc) only for FSA_FWD_GLOBAL.
 * obuf_dtype FSA_DT_F16 selects the tcgen05 kernel (LOCAL mode; V must then be
 * the fsa_v_to_f16 copy). */
int fsa_sel_fwd(const fsa_shape* s, int dtype, int mode, const void* Q, const void* K,
                const void* V, const int32_t* offsets, const int32_t* qlist, const int32_t* work,
                const void* m_global, void* obuf, int obuf_dtype, void* ml, void* stream);

/* The reference's phase passes on the tensor cores (bf16, d_K = d_V = 128,
 * B_K = 64: the shapes fsa_buffer_dtypes maps to FSA_DT_F16 partials), the K5
 * kernel in STATS / GLOBAL mode.  Slot-indexed outputs, as fsa_sel_fwd's:
 *   FSA_FWD_STATS  (compute_softmax_stats, kv_major.py:105-149): ml
 *                  [h][N][T][2] f32 local (m_i, l_i) of each live slot, for
 *                  fsa_merge_fwd FSA_MERGE_STATS; V16 / vscale / m_global unused.
 *   FSA_FWD_GLOBAL (block_pass_forward, kv_major.py:152-204): obuf
 *                  [h][N][T][d_V] f32 rows exp(z - m_global) V_i, for
 *                  FSA_MERGE_REDUCE; m_global [h][N] f32; V16 / vscale the
 *                  fsa_v_to_f16 copy of V.
 * work: the fsa_build_inverse work plan (required). */
int fsa_sel_fwd_phase(const fsa_shape* s, int mode, const void* Q, const void* K, const void* V16,
                      const float* vscale, const int32_t* offsets, const int32_t* qlist,
                      const int32_t* work, const float* m_global, float* obuf, float* ml,
                      void* stream);

/* Merge of per-slot partials in ascending block order (kv_major.py:207-242;
 * stats merge kv_major.py:137-149, shared max :141-146).  out, lse, m_out,
 * l_out in acc dtype; m_out/l_out/lse nullable.  vscale: the V16 scales
 * (required with FSA_DT_F16 obuf, else ignored); work: the work plan of the
 * item-major FSA_DT_F16 / FSA_DT_F16R buffers (ignored for the others). */
int fsa_merge_fwd(const fsa_shape* s, int dtype, int mode, const int32_t* idx,
                  const int32_t* work, const void* obuf, int obuf_dtype, const void* ml,
                  const void* m_global, const void* l_global, void* out, void* lse, void* m_out,
                  void* l_out, int shared_max, const float* vscale, void* stream);

/* K6 + K12 fused for the NSA step: the LOCAL merge (as fsa_merge_fwd) writes the
 * selected branch's out_sel / lse (acc dtype) and, in the same pass, the gated
 * combine (branches.py:95-104) out = tau0 out_cmp + tau1 out_sel + tau2 out_slide
 * in dtype.  out_cmp / out_slide / tau in acc dtype. */
int fsa_merge_combine_fwd(const fsa_shape* s, int dtype, const int32_t* idx, const int32_t* work,
                          const void* obuf, int obuf_dtype, const void* ml, const float* vscale,
                          const void* out_cmp, const void* out_slide, const void* tau,
                          void* out_sel, void* lse, void* out, void* stream);

/* delta = sum_v out * dOut (kv_major.py:284); [h][N] acc. */
int fsa_bwd_delta(const fsa_shape* s, int dtype, const void* out, const void* dOut, void* delta,
                  void* stream);

/* Selected backward tasks (kv_major.py:297-324, _core.pyx:97-131), one per
 * (KV head, block): dq partial rows into dq_buf, dK/dV ([N][h_K][d], acc) as
 * the single writer of the block (replaces the head sum at kv_major.py:342-354).
 * bf16 tensor-core path: Q, K, V, dOut are the fsa_stage_f16_ops copies and
 * scales their scale blocks (required there; ignored -- may be NULL -- else). */
int fsa_sel_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
                const void* dOut, const void* lse, const void* delta, const int32_t* offsets,
                const int32_t* qlist, const int32_t* work, void* dq_buf, int dqbuf_dtype,
                void* dK, void* dV, const float* scales, void* stream);

/* dQ = ascending-block sum of dq partials (kv_major.py:326-340); [N][h][d_K] acc. */
int fsa_dq_reduce(const fsa_shape* s, int dtype, const int32_t* idx, const void* dq_buf,
                  int dqbuf_dtype, void* dQ, void* stream);

/* fsa_dq_reduce plus addend [N][h][d_K] (fp32) added to every row in the same
 * pass: dQ = (ascending-block sum of the dq partials) + addend.  bf16
 * tensor-core configuration only (FSA_DT_F16R partials; the NSA step:
 * selected + sliding dQ). */
int fsa_dq_reduce_add(const fsa_shape* s, int dtype, const int32_t* idx, const void* dq_buf,
                      int dqbuf_dtype, const void* addend, void* dQ, void* stream);

/* compressed_attention_forward (branches.py:47-78); scores (nullable) receives
 * importance_scores_from_compressed as a fused epilogue -- on the tensor-core
 * path only for the blocks a token's top-k can read (i < (t+1)//B_K, covered
 * by the formed key tiles); call fsa_importance_scores for every block.
 * workspace (fsa_cmp_workspace_bytes, nullable = SIMT path) holds the staged
 * pooled K/V for the tcgen05 kernel, whose S runs in fp16: Q16 / qscale are the
 * fsa_stage_f16_ops copy of Q and its scale block (required on that path,
 * ignored otherwise) -- the operands the compressed backward recomputes S from. */
size_t fsa_cmp_workspace_bytes(const fsa_shape* s);
int fsa_cmp_attn_fwd(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp,
                     const void* V_cmp, const void* K_prefix, const void* V_prefix, void* out,
                     void* lse, void* scores, void* workspace, const void* Q16,
                     const float* qscale, void* stream);

/* sliding_attention_forward (branches.py:81-83 -> oracle.py:39-44, :64-74).
 * bf16 tensor-core path: V is the fsa_v_to_f16 copy and vscale its scales
 * (required); f32 / f64: vscale ignored. */
int fsa_slide_fwd(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
                  const float* vscale, void* out, void* lse, void* stream);

/* Band-mask dense_backward (oracle.py:102-131 with band_mask); grads acc dtype.
 * The bf16 tensor-core path runs the FSA backward kernel over each KV block's
 * window of tokens (dK / dV) and a query-outer kernel for dQ, and needs
 * fsa_slide_bwd_workspace_bytes of workspace (its scheduler counter);
 * accumulate == 1 adds into dQ/dK/dV (sums the sliding branch onto the selected
 * branch's gradients), accumulate == 2 adds into dK/dV but WRITES dQ (fp32, for
 * fsa_dq_reduce_add) -- tensor-core path only. */
size_t fsa_slide_bwd_workspace_bytes(const fsa_shape* s, int dtype);
int fsa_slide_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
                  const void* dOut, const void* lse, const void* delta, void* dQ, void* dK,
                  void* dV, void* workspace, int accumulate, const float* scales, void* stream);

/* gated_combine (branches.py:95-104): out = sum_c tau[t][c] * out_c; branch
 * outputs and tau [N][3] in acc dtype; out in acc dtype if out_acc else dtype. */
int fsa_gated_combine(const fsa_shape* s, int dtype, const void* out_cmp, const void* out_sel,
                      const void* out_slide, const void* tau, void* out, int out_acc,
                      void* stream);

/* Gate backward into branch c: out = tau[t][c] * dOut (branches.py:103); [N][h][d_V]. */
int fsa_gate_scale(const fsa_shape* s, int dtype, const void* dOut, const void* tau, int col,
                   void* out, void* stream);

/* Fused gate backward + delta for the selected and sliding branches
 * (branches.py:103, kv_major.py:284): d_sel = tau[t][1] dOut, d_slide =
 * tau[t][2] dOut (dtype), delta_c[j][t] = sum_v out_c * d_c (acc dtype, from
 * the rounded d_c).  out_sel/out_slide [N][h][d_V] acc dtype. */
int fsa_gate_backward(const fsa_shape* s, int dtype, const void* dOut, const void* tau,
                      const void* out_sel, const void* out_slide, void* d_sel, void* d_slide,
                      void* delta_sel, void* delta_slide, void* stream);

/* The gate backward folded into the branch statistics (tensor-core path, used by
 * the NSA step): delta_c = sum_v out_c * dOut and lse_c_adj = lse_c - ln tau_c[t]
 * for c = selected, sliding ([h][N], acc).  The branch backward kernels then take
 * the raw dOut: tau * exp(z - lse) = exp(z - lse_adj) (branches.py:103). */
int fsa_gate_backward_fold(const fsa_shape* s, int dtype, const void* dOut, const void* tau,
                           const void* out_sel, const void* out_slide, const void* lse_sel,
                           const void* lse_slide, void* delta_sel, void* delta_slide,
                           void* lse_sel_adj, void* lse_slide_adj, void* stream);

/* Compressed-branch backward (the reference has none --
 * parity vs the float64 oracle, pinned to autograd): gradients of
 * sum(out_cmp * dOut) through the attention over the pooled rows and the
 * pooling / prefix means (branches.py:34-78), ADDED into dQ [N][h][d_K] and
 * dK, dV [N][h_K][d] (acc dtype).  K_cmp/V_cmp [b][h_K][d], lse [h][N],
 * delta = sum_v out_cmp * dOut [h][N] in acc dtype; dOut in dtype. */
size_t fsa_cmp_bwd_workspace_bytes(const fsa_shape* s, int dtype);
int fsa_cmp_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp, const void* V_cmp,
                const void* dOut, const void* lse, const void* delta, void* dQ, void* dK, void* dV,
                void* workspace, void* stream);

/* fsa_cmp_bwd with the gate folded in (after fsa_gate_backward_full_fold): dOut
 * is the raw cotangent, lse_adj = lse_cmp - ln tau[t, 0], delta = sum out_cmp *
 * dOut, and tau (N, 3) gates the pending tokens' prefix-mean gradients.  On the
 * bf16 tensor-core path (d = 128) Q16 / dO16 / scales are the fsa_stage_f16_ops
 * copies of Q and dOut (required there; ignored elsewhere).  workspace:
 * fsa_cmp_bwd_fold_workspace_bytes. */
size_t fsa_cmp_bwd_fold_workspace_bytes(const fsa_shape* s, int dtype);
int fsa_cmp_bwd_fold(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp,
                     const void* V_cmp, const void* dOut, const void* tau, const void* lse_adj,
                     const void* delta, void* dQ, void* dK, void* dV, const void* Q16,
                     const void* dO16, const float* scales, void* workspace, void* stream);

/* Gate backward for all three branches (branches.py:95-104): d_c = tau[t][c]
 * dOut (dtype), delta_c [h][N] = sum_v out_c * d_c, and the gate gradient
 * dtau [N][3] = sum_{v,j} out_c * dOut (acc dtype).  One pass over dOut. */
int fsa_gate_backward_full(const fsa_shape* s, int dtype, const void* dOut, const void* tau,
                           const void* out_cmp, const void* out_sel, const void* out_slide,
                           void* d_cmp, void* d_sel, void* d_slide, void* delta_cmp,
                           void* delta_sel, void* delta_slide, void* dtau, void* stream);

/* fsa_gate_backward_full folded into the branch statistics (the tensor-core NSA
 * step with full=True): delta_c = sum_v out_c * dOut, lse_c_adj = lse_c - ln
 * tau_c[t] for c = compressed, selected, sliding ([h][N], acc), and dtau (N, 3);
 * the branch backward kernels then take the raw dOut (no gated copies). */
int fsa_gate_backward_full_fold(const fsa_shape* s, int dtype, const void* dOut, const void* tau,
                                const void* out_cmp, const void* out_sel, const void* out_slide,
                                const void* lse_cmp, const void* lse_sel, const void* lse_slide,
                                void* delta_cmp, void* delta_sel, void* delta_slide,
                                void* lse_cmp_adj, void* lse_sel_adj, void* lse_slide_adj,
                                void* dtau, void* stream);

/* NSA query-major selected forward (query_major.py:45-69, _core.pyx:134-181):
 * one task per (kv head, token) over its selected blocks in ascending order,
 * online softmax; the FSA-vs-NSA comparison baseline (CUDA cores; g <= 16,
 * d_V <= 256).  out [N][h][d_V], lse [h][N] in acc dtype. */
int fsa_qm_fwd(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
               const int32_t* idx, void* out, void* lse, void* stream);

/* The NSA query-major forward on tcgen05 (query_major.py:45-69 with the
 * min_tile padding of :32-42): bf16, d = 128, B_K = 64, g <= 16, T <= 16.
 * Per (kv head, token) the g heads (padded to max(g, min_tile), rounded up to
 * 8) ride on the MMA's N side against pairs of 64-key blocks on M; an exact
 * two-pass softmax per token.  V16 / vscale: the fsa_v_to_f16 copy of V;
 * out (N, h, 128) f32, lse (h, N) f32. */
int fsa_qm_fwd_tc(const fsa_shape* s, const void* Q, const void* K, const void* V16,
                  const float* vscale, const int32_t* idx, void* out, void* lse, int min_tile,
                  void* stream);

/* NSA query-major selected backward (query_major.py:72-99, _core.pyx:184-241):
 * per (KV head, token) task, P recomputed from lse, dQ rows written, dK / dV
 * ([N][h_K][d], acc; zeroed here) scattered with atomics.  lse, delta [h][N]
 * in acc dtype (fsa_qm_fwd + fsa_bwd_delta).  g <= 16. */
int fsa_qm_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
               const void* dOut, const int32_t* idx, const void* lse, const void* delta, void* dQ,
               void* dK, void* dV, void* stream);

/* Finiteness check for as_headed (config.py:146-155): *flag |= 1 on any non-finite. */
int fsa_check_finite(int dtype, const void* x, int64_t n, int32_t* flag, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FSA_B200_H */

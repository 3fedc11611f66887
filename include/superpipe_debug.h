/*
 * superpipe_debug.h — kernel-level entry points of libsuperpipe.so used by the GPU unit
 * tests to check the tcgen05 GEMM in isolation against a torch fp32 reference. Not part of
 * the reference-facing boundary (superpipe.h). Pointers are device pointers; the call is
 * synchronous on the legacy default stream.
 */
#ifndef SUPERPIPE_DEBUG_H
#define SUPERPIPE_DEBUG_H

#include <stdint.h>

#include "superpipe.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] = A[M,K] B[K,N] with bf16 A/B. a_mn: A stored [K][lda] (M contiguous) instead of
 * [M][lda]; b_mn: B stored [K][ldb] (N contiguous) instead of [N][ldb]. epilogue: 0 bf16
 * act(acc+bias), 1 fp32 act(acc+bias), 2 bf16 ReLU-gated by `gate`, 3 fp32 split-K partials
 * (split s at out + s*M*ldo), 4 fp32 out -= lr*acc with lr = 1 (fused SGD). block_n: tile N
 * (0 = choose); cta: 1 = one CTA per 128-row tile, 2 = CTA pair per 256-row tile (cta_group::2),
 * 0 = choose. Returns 0 or a cudaError_t value. */
int sp_debug_gemm_bf16(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, int32_t a_mn,
                       const void* B, int32_t ldb, int32_t b_mn, int32_t epilogue, void* out,
                       int32_t ldo, const float* bias, int32_t relu, const void* gate,
                       int32_t ldg, int32_t splits, int32_t block_n, int32_t cta);
/* Same, launched asynchronously on `stream` (a cudaStream_t) without synchronising, for
 * back-to-back timing of the kernel between two CUDA events. */
int sp_debug_gemm_bf16_async(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda,
                             int32_t a_mn, const void* B, int32_t ldb, int32_t b_mn,
                             int32_t epilogue, void* out, int32_t ldo, const float* bias,
                             int32_t relu, const void* gate, int32_t ldg, int32_t splits,
                             int32_t block_n, int32_t cta, void* stream);
/* Same as sp_debug_gemm_bf16_async, plus the ReLU bit masks of the executor's bf16 training:
 * mask_out (epilogue 0 with relu: write the output's mask, uint32[N/32][M]) and gate_mask
 * (epilogue 2: gate with that mask instead of reading the gate tensor). Either may be NULL. */
int sp_debug_gemm_bf16_masked_async(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda,
                                    int32_t a_mn, const void* B, int32_t ldb, int32_t b_mn,
                                    int32_t epilogue, void* out, int32_t ldo, const float* bias,
                                    int32_t relu, const void* gate, int32_t ldg, int32_t splits,
                                    int32_t block_n, int32_t cta, void* stream, void* mask_out,
                                    const void* gate_mask);
/* The tf32 GEMM (fp32 A/B multiplied with tcgen05 kind::tf32, SP_NUMERICS_TF32): arguments
 * as sp_debug_gemm_bf16_masked_async with fp32 operands; epilogue 1 (fp32 act(acc+bias), with
 * mask_out), 5 (fp32 ReLU-gated by an fp32 `gate` or by gate_mask), 3, 4. */
int sp_debug_gemm_tf32_async(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda,
                             int32_t a_mn, const void* B, int32_t ldb, int32_t b_mn,
                             int32_t epilogue, void* out, int32_t ldo, const float* bias,
                             int32_t relu, const void* gate, int32_t ldg, int32_t splits,
                             int32_t block_n, int32_t cta, void* stream, void* mask_out,
                             const void* gate_mask);
/* Sharded streaming geometry (the executor's own functions): shard size for an image of
 * img bytes over world ranks, and rank's byte range [lo, hi). */
uint64_t sp_debug_shard_range(uint64_t img, int32_t world, int32_t rank, uint64_t* lo,
                              uint64_t* hi);
/* Split-K count the executor's bf16 dW GEMM uses for a d x d layer at `rows` rows (1 = SGD
 * fused into the GEMM epilogue; > 1 = fp32 partials reduced by the update op). */
int32_t sp_debug_dw_splits(int32_t d, int64_t rows);
/* The executor's full dW choice (choose_dw): returns the split count and writes the kernel
 * variant (cta 1|2, tile N). fused_ok = 1 for one GPU (splits = 1 means SGD fused). */
int32_t sp_debug_dw_choice(int32_t d, int64_t rows, int32_t fused_ok, int32_t* cta,
                           int32_t* block_n);
/* Split count the GEMM will use for a given K and requested splits. */
int32_t sp_debug_effective_splits(int32_t K, int32_t splits);

/* Every GEMM epilogue of the executor, including the transformer-block ones (kernels.hpp
 * GemmEpilogue 6..9: residual add, GELU with pre-activation side output, GELU' gate, SwiGLU).
 * Fields as sp_debug_gemm_bf16_masked_async; aux/ldaux the pre-activation output; act the
 * GELU kind (0 tanh, 1 erf). Launched on `stream` without synchronising. */
typedef struct {
    int32_t M, N, K;
    const void* A;
    int32_t lda, a_mn;
    const void* B;
    int32_t ldb, b_mn;
    int32_t epilogue;
    void* out;
    int32_t ldo;
    const float* bias;
    int32_t relu;
    const void* gate;
    int32_t ldg, splits, block_n, cta;
    void* aux;
    int32_t ldaux, act;
    void* stream;
    float* colsum_part; /* EPI_GELU_GATE_BF16, one split: [ceil(M / 32)][N] column partials (or NULL) */
} sp_debug_gemm_args;
int sp_debug_gemm_ex(const sp_debug_gemm_args* a);
/* The attention core of the transformer blocks (kernels.hpp AttnProblem), device pointers,
 * launched on `stream`. Forward: qkv -> o, lse. Backward: (qkv, o, lse, dout) -> dqkv, with
 * delta a scratch of tokens * n_heads floats. */
int sp_debug_attention(int32_t backward, int64_t tokens, int32_t seq_len, int32_t n_heads,
                       int32_t n_kv_heads, int32_t head_dim, int32_t causal, const void* qkv, void* o,
                       float* lse, const void* dout, float* delta, void* dqkv, void* stream);
/* LayerNorm (rms = 0) / RMSNorm (rms = 1) forward and backward (kernels.hpp norm_forward /
 * norm_backward), device pointers, on `stream`. Backward: dres_out = dres_in + dx (and its bf16
 * copy); when `out` is non-null also the parameter gradients out[0, d) (gamma) and out[d, 2d)
 * (LayerNorm beta) through the scratch `part` / `counters` (sp_debug_col_scratch sizes; the
 * counters zeroed before first use, left zero). */
int sp_debug_norm_forward(const float* x, const float* gamma, const float* beta, int32_t rms, float eps,
                          int64_t rows, int32_t d, void* y, float* stats, void* stream);
int sp_debug_norm_backward(const float* dy, const float* x, const float* stats, const float* gamma,
                           int32_t rms, int64_t rows, int32_t d, const float* dres_in, float* dres_out,
                           void* dres_out16, float* part, int32_t* counters, float* out, void* stream);
/* out[j] = sum over rows of a bf16 [rows][n] matrix (a bias gradient; n % 8 == 0), with the
 * same scratch (kernels.hpp colsum_total_bf16). */
int sp_debug_colsum(const void* x, int64_t rows, int32_t n, float* part, int32_t* counters, float* out, void* stream);
void sp_debug_col_scratch(int64_t rows, int32_t widest, int64_t* part_floats, int64_t* counters);
/* Debug timeline of the last tcgen05 dK/dV attention pass run with sp_debug_set(NULL,
 * "attn_trace", 1): CTA 0's events as (event << 56 | step << 40 | SM clock), up to cap; returns
 * the count (events: 0/1 S issue entered / issued, 2/3 product issue entered / issued, 4/5/6 and
 * 12/13/14 softmax warpgroup 0 / 1 step entered / S ready / P written). */
int sp_debug_attn_trace(uint64_t* out, int32_t cap);
/* The single-pass norm backward (kernels.hpp norm_backward_fused, d % 4 == 0 and d <= 2048, else
 * SP_ERR_INVALID) and its chunk reduction: dres_out / dres_out16 as above (dres_out null: none),
 * out_param[0, d) / [d, 2d) the parameter gradients (null: none) and out_csum[j] = sum over rows
 * of dres_out (null: none). ppart holds 2 d, cpart d floats per block of the persistent grid
 * (min(2 x SMs, ceil(rows / 2)) blocks). */
int sp_debug_norm_backward_fused(const float* dy, const float* x, const float* stats, const float* gamma,
                                 int32_t rms, int64_t rows, int32_t d, const float* dres_in, float* dres_out,
                                 void* dres_out16, float* ppart, float* cpart, float* out_param, float* out_csum,
                                 void* stream);

/* Transformer-block executors: the fp32 gradient image (the layer's parameter layout) of
 * layer `index` from the last train step, as the UPDATE op consumed it. Gradient images are
 * double-buffered by layer parity, so only the last two layers the backward reached (layers 0
 * and 1) are still intact. Not available in sharded data parallel. */
int sp_debug_read_grad(struct sp_exec* ex, int32_t index, float* out);

/* Debug and A/B measurement knobs (defaults = the product behaviour; nothing on the product
 * path sets them). Executor keys (ex != NULL): "staged_writeback" (0: write back straight from
 * the slot), "wb_stages" (staging buffer count, default 3), "defer_budget" (-1 = the executor's
 * rule), "per_move" / "move_events" (0: batched H2D jobs wait up front / no per-move completion
 * events), "graphs" (0: no CUDA-graph capture), "poison" (1: NaN-fill every slot / activation
 * reload destination before its copy), "drop_load_edges" (fault injection: computes stop
 * waiting for their loads - tests only). Process-wide GEMM keys (ex may be NULL): "epi_mode"
 * (0 auto, 1 direct stores, 2 TMA-staged stores), "narrow" (1: half-width ragged last tiles for
 * every epilogue). Returns SP_OK or SP_ERR_INVALID for an unknown key. */
struct sp_exec;
int sp_debug_set(struct sp_exec* ex, const char* key, int32_t value);

/* Two consecutive training plans exactly as the executor builds them (eager prefetch, staged
 * and deferred write-back, the largest deferral budget): call 1 with act_bytes1, then call 2 with act_bytes2 and call 1's
 * deferred write-backs pending. Text: "DEFERRED <layers>", then "FLUSHED <layers>" when call 2's
 * capacity-shrunk ring could not keep them (the executor completes them before planning), then
 * call 2's plan listing. Returns the needed length. Host-only. */
int64_t sp_debug_plan_two_calls(const sp_config* cfg, uint64_t act_bytes1, uint64_t act_bytes2,
                                char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif

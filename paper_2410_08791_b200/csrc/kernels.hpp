// kernels.hpp — host-side launchers for the executor's sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace sp {

// ---- exact (bit-identical to the reference CPU math, model.cpp:54-155) -------------
// y = act(x W + b), i-ascending fp32, separately rounded mul/add, bias last.
void exact_forward(const float* x, const float* W, const float* b, int relu, float* y,
                   int64_t rows, int d, cudaStream_t st);
// dz_out[r,i] = sum_j dz[r,j] W[i,j] (j ascending); then, if gate != nullptr, the ReLU
// derivative of the layer below: dz_out = gate[r,i] <= 0 ? 0 : dz_out (model.cpp:91-96 with
// z recomputation replaced by the stored activation, which has the same sign).
void exact_backward_dx(const float* dz, const float* W, const float* gate, float* dz_out,
                       int64_t rows, int d, cudaStream_t st);
// dW[i,j] = sum_r x[r,i] dz[r,j]; db[j] = sum_r dz[r,j] (r ascending), model.cpp:108-121.
void exact_backward_dw(const float* x, const float* dz, float* dW, float* db, int64_t rows,
                       int d, cudaStream_t st);
// loss = (sum e^2)/N sequential (model.cpp:131-140) into *loss_dev; g = 2 e (1/N) gated by
// the last layer's ReLU (y <= 0 -> 0). partial != nullptr: write the raw sum instead (DP).
void exact_loss_grad(const float* y, const float* t, int64_t count, float inv_n, int relu,
                     float* g, float* loss_sum_dev, cudaStream_t st);
// w -= lr * g  (model.cpp:150-155), no FMA.
void exact_sgd(float* w, const float* g, int64_t count, float lr, cudaStream_t st);

// ---- bf16 tensor-core path -----------------------------------------------------------
enum GemmEpilogue : int {
    EPI_BIAS_ACT_BF16 = 0,  // out(bf16) = act(acc + bias)
    EPI_BIAS_ACT_F32 = 1,   // out(f32)  = act(acc + bias)
    EPI_GATE_BF16 = 2,      // out(bf16) = (relu && gate <= 0) ? 0 : acc
    EPI_F32 = 3,            // out(f32)  = acc  (split-K partial at out + split*split_stride)
    EPI_SGD_F32 = 4,        // out(f32) -= lr * acc  (fused SGD on the fp32 master; splits == 1)
    EPI_GATE_F32 = 5,       // out(f32)  = (relu && gate <= 0) ? 0 : acc  (tf32 path; fp32 gate)
    // transformer blocks (named-shape layers)
    EPI_RESID_F32 = 6,      // out(f32)  = acc + bias + gate(f32 residual [M][ldg]); bias optional
    EPI_GELU_BF16 = 7,      // out(bf16) = gelu(acc + bias); aux(bf16) = acc + bias (pre-activation)
    EPI_GELU_GATE_BF16 = 8, // out(bf16) = acc * gelu'(gate)  (gate = the saved pre-activation, bf16)
    EPI_SWIGLU_BF16 = 9     // out(bf16)[M][N/2] = silu(acc_g) * acc_u over 32-column chunk pairs
                            // (g = chunk 2c, u = chunk 2c+1 of each tile); aux(bf16)[M][N] = acc
};
// EPI_GELU_BF16 / EPI_GELU_GATE_BF16 activation (GemmProblem::act)
enum GeluKind : int { GELU_TANH = 0, GELU_ERF = 1 };

struct GemmProblem {
    // C[M,N] = A[M,K] * B[K,N]; A given K-major ([M][lda]) or M-major ([K][lda]);
    // B given K-major ([N][ldb]) or N-major ([K][ldb]). Leading dims in elements.
    int M = 0, N = 0, K = 0;
    const void* A = nullptr;
    int lda = 0;
    bool a_mn = false;
    const void* B = nullptr;
    int ldb = 0;
    bool b_mn = false;
    int epilogue = EPI_F32;
    void* out = nullptr;
    int ldo = 0;
    const float* bias = nullptr;
    int relu = 0;
    const void* gate = nullptr;  // [M][ldg], bf16 (EPI_GATE_BF16) or fp32 (EPI_GATE_F32)
    int ldg = 0;
    int splits = 1;
    int64_t split_stride = 0;
    int block_n = 0;  // 0 = choose (1-CTA: N per CTA; 2-CTA: N per CTA pair)
    float lr = 0.0f;  // EPI_SGD_F32
    int cta = 0;      // 0 = choose, 1 = one CTA per tile (M=128), 2 = CTA pair (M=256)
    // EPI_BIAS_ACT_BF16 with relu: also write the ReLU mask of the stored output, one bit per
    // element, mask_out[(col/32) * M + row] bit (col % 32) = !(bf16(y) <= 0) (column-chunk
    // major, so one warp's 32 rows of a chunk are one 128-byte store / load).
    uint32_t* mask_out = nullptr;
    // EPI_GATE_BF16: gate with such a mask instead of reading the bf16 gate tensor.
    const uint32_t* gate_mask = nullptr;
    // Operands A and B are fp32 and multiplied as tf32 (tcgen05 kind::tf32) instead of bf16
    // (kind::f16). Epilogues: EPI_BIAS_ACT_F32 (with mask_out), EPI_GATE_F32 (gate: fp32
    // tensor or gate_mask), EPI_F32, EPI_SGD_F32.
    bool tf32 = false;
    // EPI_GELU_BF16 / EPI_SWIGLU_BF16: second output (pre-activation), bf16 [M][ldaux]; may be
    // null for SWIGLU (inference).
    void* aux = nullptr;
    int ldaux = 0;
    int act = GELU_TANH;  // GeluKind for the GELU epilogues
    // EPI_GELU_GATE_BF16 with one split: also the column sums of the output (the bias gradient
    // of the layer that produced the gate), per 32-row group: colsum_part[ceil(M/32)][N] (fp32
    // sums of the unrounded outputs, fixed order); reduce_col_chunks sums the groups
    float* colsum_part = nullptr;
};

struct GemmChoice {
    int cta;
    int block_n;
};
// The kernel variant gemm_bf16 picks when cta/block_n are 0 (depends on the shape only, so
// results are identical for every window setting).
GemmChoice choose_gemm(int M, int N, int K, int splits, int epilogue, bool b_kmajor = false);

// Launches the warp-specialized tcgen05/TMEM/TMA GEMM. Returns cudaSuccess or an error.
cudaError_t gemm_bf16(const GemmProblem& p, cudaStream_t st);
// Picks the split-K factor that best fills the 148 SMs for an M x N x K problem.
int choose_splits(int M, int N, int K, int block_n);
// dW kernel choice: variant and split-K count together (splits = 1 and fused_ok: SGD fused).
struct DwChoice {
    int cta, block_n, splits;
};
DwChoice choose_dw(int M, int N, int K, int max_splits, bool fused_ok, bool tf32 = false);
int choose_block_n(int N);
// Split count actually used for K (no empty split): what gemm_bf16 will launch.
int effective_splits(int K, int splits, bool tf32 = false);
int num_sms();

void convert_f32_to_bf16(const float* src, void* dst, int64_t count, cudaStream_t st);
// Fused MSE: partial sums of e^2 per block into partials[nblk] (fixed grid, deterministic),
// g(bf16) = 2 e inv_n gated by the last layer's ReLU. Then loss_finalize sums partials in a
// fixed order into *out (raw sum; caller divides by N).
int loss_grad_bf16(const float* y, const float* t, int64_t count, float inv_n, int relu,
                   void* g, float* partials, cudaStream_t st);
// The same with an fp32 gradient (tf32 path).
int loss_grad_f32(const float* y, const float* t, int64_t count, float inv_n, int relu,
                  float* g, float* partials, cudaStream_t st);
void loss_finalize(const float* partials, int n, float* out, cudaStream_t st);
// Column sums of a bf16 [rows][d] matrix into partials[chunks][d] (fixed chunking).
int colsum_bf16(const void* x, int64_t rows, int d, float* partials, cudaStream_t st);
int colsum_chunks(int64_t rows);
// Column sums of an fp32 [rows][d] matrix (d % 4 == 0), same chunking (tf32 path).
int colsum_f32(const float* x, int64_t rows, int d, float* partials, cudaStream_t st);
// grad[i] = sum_s parts[s*stride + i] (fixed order).
void reduce_partials(const float* parts, int nparts, int64_t stride, int64_t count,
                     float* grad, cudaStream_t st);
// w[i] -= lr * sum_s parts[s*stride + i]  (reduction fused into the SGD update).
void sgd_reduce(float* w, const float* parts, int nparts, int64_t stride, int64_t count,
                float lr, cudaStream_t st);
void scale_inplace(float* x, int64_t count, float s, cudaStream_t st);

// AdamW (PyTorch's decoupled weight decay) on fp32 master weights w with optimizer state m, v,
// the gradient being sum_p parts[p*stride + i] (fixed order; nparts = 1 for a plain gradient).
// The step's scalars are read from device memory (refreshed each call, so a captured CUDA graph
// replays every step). Each operation separately rounded, in orc_adamw's order (oracle.h).
struct AdamwScalars {
    float decay, omb1, b2, omb2, bc2_sqrt, eps, neg_step, pad;
};
// Up to 16 fp32 regions converted to bf16 (to_bf16) or copied as fp32, one launch: a layer
// image's matrices -> the bf16 operand copy, its vectors -> fp32 next to them (wire layout).
struct ConvertRegions {
    int n = 0;
    const float* src[16];
    void* dst[16];
    int64_t count[16];  // elements, multiple of 4
    int to_bf16[16];
};
void convert_regions(const ConvertRegions& r, cudaStream_t st);
// Update of a split master image (block.hpp): per tensor region, the fp32 parameter is
// (hi << 16 | lo) for matrices (hi in the wire prefix, lo in the low plane) or a plain fp32
// vector; g (and AdamW m, v) are in the logical fp32 layout. SGD (opt 0, model.cpp:150-155:
// w -= lr g, no FMA) or AdamW (opt 1, adamw_reduce's arithmetic). Up to 16 regions, one launch.
struct SplitRegions {
    int n = 0;
    void* hi[16];        // matrices: uint16 hi halves; vectors: fp32 values
    uint16_t* lo[16];    // matrices: low halves; vectors: nullptr
    int64_t off[16];     // logical offset (floats) of the region in g / m / v
    int64_t count[16];   // elements
    // optional: the gradient of region i is the fixed-order sum of nparts[i] split-K partials
    // at parts[i] (stride count[i]) instead of g[off[i] ...]
    const float* parts[16] = {};
    int nparts[16] = {};
    // optional: every updated value (halves, vectors, m, v) is also stored at its address +
    // stage_delta bytes (the write-back stage, which has the slot's layout), so no separate
    // staging copy re-reads the slot
    int64_t stage_delta = 0;
    // with a stage: the slot itself keeps the old values (nothing reads it again: the plan does
    // not leave the layer valid in that slot), only the stage receives the update
    bool stage_only = false;
};
void split_update(const SplitRegions& r, const float* g, float* m, float* v, float lr, int opt,
                  const AdamwScalars* scalars, cudaStream_t st);
// n (<= 3) device-to-device copies of `bytes` each (multiple of 4, 4-byte aligned) on the SMs.
void copy_regions(void* const* dst, const void* const* src, int n, int64_t bytes, cudaStream_t st);
void adamw_reduce(float* w, float* m, float* v, const float* parts, int nparts, int64_t stride,
                  int64_t count, const AdamwScalars* scalars, cudaStream_t st);

// ---- named-shape transformer blocks (kernels_attn.cu, kernels_block.cu) ------------------
// Attention over the packed projections qkv[T][(H + 2 Hkv) hd] (bf16, token-major; q heads,
// then k heads, then v heads), sequences of seq_len consecutive tokens. head_dim 64, 80 or 128.
struct AttnProblem {
    int64_t tokens = 0;
    int seq_len = 0, n_heads = 0, n_kv_heads = 0, head_dim = 0;
    int causal = 1;
    const void* qkv = nullptr;   // [T][(H + 2 Hkv) hd] bf16
    void* o = nullptr;           // [T][H hd] bf16 (forward output; backward input)
    float* lse = nullptr;        // [T / seq_len][H][seq_len] fp32, log2 units of scaled scores
    const void* dout = nullptr;  // backward: dO [T][H hd] bf16
    float* delta = nullptr;      // backward scratch [T / seq_len][H][seq_len]
    void* dqkv = nullptr;        // backward output, same layout as qkv
    // backward, optional: the column sums of dqkv (bqkv's gradient) per 32-row group,
    // colsum_part[T / 32][(H + 2 Hkv) hd], formed in the tcgen05 passes' epilogues (head_dim 64 /
    // 128 and seq_len % 32 == 0 only: attention_colsum_fused says whether a shape gets them)
    float* colsum_part = nullptr;
};
bool attention_colsum_fused(const AttnProblem& a);
// (sequence, head) pairs per chunk of the causal attention kernels' work order
int attention_causal_chunk(const AttnProblem& a);
cudaError_t attention_forward(const AttnProblem& a, cudaStream_t st);
cudaError_t attention_backward(const AttnProblem& a, cudaStream_t st);

// LayerNorm (gamma, beta; rms = 0) or RMSNorm (gamma only; rms = 1) of fp32 rows [T][d]:
// y (bf16) = norm(x) * gamma (+ beta); stats[T][2] = {mean, rstd} (RMSNorm: {0, rstd}).
void norm_forward(const float* x, const float* gamma, const float* beta, int rms, float eps,
                  int64_t rows, int d, void* y, float* stats, cudaStream_t st);
// Scratch of the column-sum kernels below: part (fp32 chunk partials) and counters (ints, zero
// before first use; each kernel leaves them zero), sized by col_scratch_size for the widest
// matrix. Kernels on one stream may share one scratch.
struct ColScratch {
    float* part = nullptr;
    int* counters = nullptr;
};
struct ColScratchSize {
    size_t part_floats = 0, counters = 0;
};
ColScratchSize col_scratch_size(int64_t rows, int widest);
// Backward of the norm given dy (fp32 [T][d], the gradient of its output):
//   dx = rstd (dy*gamma - mean(dy*gamma) - xhat mean(dy*gamma*xhat))   (RMSNorm: no mean term)
//   dres_out (fp32) = dres_in + dx and dres_out16 (bf16) = the same rounded, when non-null.
// Parameter gradients, when out is non-null: out[0, d) = sum_r dy*xhat (gamma), out[d, 2d) =
// sum_r dy (LayerNorm's beta), through 512-row chunk partials summed in chunk order by the last
// block of each column group (fixed decomposition: depends on the shape only).
void norm_backward(const float* dy, const float* x, const float* stats, const float* gamma, int rms,
                   int64_t rows, int d, const float* dres_in, float* dres_out, void* dres_out16,
                   const ColScratch& scr, float* out, cudaStream_t st);
// out[j] = sum_r x[r][j] of a bf16 [rows][n] matrix (n % 8 == 0; a bias gradient), the same
// chunking and in-kernel fixed-order reduction.
void colsum_total_bf16(const void* x, int64_t rows, int n, const ColScratch& scr, float* out, cudaStream_t st);
int norm_param_chunks(int64_t rows);
// The single-pass form of norm_backward (d % 4 == 0, d <= 2048; norm_backward_fused_ok): the
// same dres_out / dres_out16 (skipped when dres_out is null), plus per block c of its persistent
// grid (norm_bwd_chunks(rows) blocks, each a fixed strided set of rows) the column partials
// param_part[c][0][j] = sum dy*xhat, param_part[c][1][j] = sum dy (LayerNorm only) and
// csum_part[c][j] = sum dres_out (each skipped when null). reduce_col_chunks sums the blocks.
bool norm_backward_fused_ok(int d);
int norm_bwd_chunks(int64_t rows);
void norm_backward_fused(const float* dy, const float* x, const float* stats, const float* gamma, int rms,
                         int64_t rows, int d, const float* dres_in, float* dres_out, void* dres_out16,
                         float* param_part, float* csum_part, cudaStream_t st);
// Up to three chunk-partial segments, out[s][j] = sum_c part[s][c * stride[s] + j] in a fixed
// order (chunk ranges of ceil(chunks / 8), each in chunk order, then the ranges in order).
struct ColChunks {
    int n = 0, chunks = 0;
    const float* part[3] = {nullptr, nullptr, nullptr};
    int64_t stride[3] = {0, 0, 0};
    int width[3] = {0, 0, 0};
    float* out[3] = {nullptr, nullptr, nullptr};
};
void reduce_col_chunks(const ColChunks& r, cudaStream_t st);

}  // namespace sp

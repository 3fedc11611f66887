// block_exec.cpp — the executor's per-layer work for named-shape transformer layers.
//
// The ring, the plan, the copies and the optimizer are the dense executor's (executor.cpp);
// only what one COMPUTE op does changes. A layer is a pre-norm transformer block (block.hpp):
//
//   forward  x -> norm1 -> xn1 -> [Wqkv, bqkv] -> qkv -> attention -> o -> [Wo, bo] + x -> h
//            h -> norm2 -> xn2 -> [W1, b1] -> GELU (or SwiGLU) -> g -> [W2, b2] + h -> y
//   (x, h, y fp32 residual stream; xn*, qkv, o, g bf16 tcgen05 operands; the bias, GELU,
//    SwiGLU and residual adds are GEMM epilogues)
//   backward the reverse, producing the layer's flat fp32 gradient image in its parameter
//            layout, which the UPDATE op applies like a dense layer's [dW | db]
//
// Training keeps each layer's intermediates (BlockActs) for its backward. With activation
// offload (the reference's checkpointing, engine.cpp:247-252) only the layer input x rides the
// layer's D2H / H2D, as in the reference's ledger, and the backward recomputes the block's
// forward from it into one scratch set first.
#include <cstring>

#include "executor.hpp"
#include "kernels.hpp"

namespace sp {

#define CUDA_OK(expr)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw Error(SP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

Executor::WirePtrs Executor::wire_ptrs(const uint8_t* wire) const {
    WirePtrs w;
    auto mat = [&](int i) -> const void* { return i < 0 ? nullptr : wire + lay_.t[static_cast<size_t>(i)].wire_off; };
    auto vec = [&](int i) -> const float* {
        return i < 0 ? nullptr : reinterpret_cast<const float*>(wire + lay_.t[static_cast<size_t>(i)].wire_off);
    };
    w.wqkv = mat(lay_.wqkv);
    w.wo = mat(lay_.wo);
    w.w1 = mat(lay_.w1);
    w.w2 = mat(lay_.w2);
    w.ln1_g = vec(lay_.ln1_g);
    w.ln1_b = vec(lay_.ln1_b);
    w.bqkv = vec(lay_.bqkv);
    w.bo = vec(lay_.bo);
    w.ln2_g = vec(lay_.ln2_g);
    w.ln2_b = vec(lay_.ln2_b);
    w.b1 = vec(lay_.b1);
    w.b2 = vec(lay_.b2);
    return w;
}

void Executor::block_alloc(int64_t R, int items, bool train, const std::function<void*(size_t)>& alloc) {
    (void)items;
    const size_t T = static_cast<size_t>(R), d = static_cast<size_t>(d_);
    const size_t hhd = static_cast<size_t>(lay_.desc.n_heads) * lay_.head_dim;
    const size_t lse = T * static_cast<size_t>(lay_.desc.n_heads);
    const bool ckpt = train && cfg_.checkpointing && cfg_.strategy != SP_STANDARD;
    auto acts = [&](bool keep_pre) {
        BlockActs a;
        a.xn1 = alloc(T * d * 2);
        a.st1 = static_cast<float*>(alloc(T * 8));
        a.qkv = alloc(T * static_cast<size_t>(lay_.qkv_cols) * 2);
        a.o = alloc(T * hhd * 2);
        a.lse = static_cast<float*>(alloc(lse * 4));
        a.xmid = static_cast<float*>(alloc(T * d * 4));
        a.xn2 = alloc(T * d * 2);
        a.st2 = static_cast<float*>(alloc(T * 8));
        // g: the MLP's activation output [T][ff]; h: the pre-activation (GELU: [T][ff]; SwiGLU:
        // gate and up [T][2 ff]) - kept only when a backward will read it
        a.g = alloc(T * static_cast<size_t>(lay_.desc.ff) * 2);
        if (keep_pre) a.h = alloc(T * static_cast<size_t>(lay_.mlp_cols) * 2);
        return a;
    };
    for (auto& p : pp_) p = alloc(T * d * 4);  // inference: fp32 residual stream ping-pong
    bx_.clear();
    bsv_.clear();
    // one scratch set: inference (also after training: the buffers are shared) and the
    // offload mode's forward / backward recompute
    bscr_ = acts(train && ckpt);
    if (!train) return;
    if (!ckpt) {
        for (int l = 0; l < n_; ++l) {
            bx_.push_back(static_cast<float*>(alloc(T * d * 4)));
            bsv_.push_back(acts(true));
        }
        bx_.push_back(yout_);
    }
    // backward scratch, shared by every layer (stream-ordered on the compute stream)
    bdxn_ = static_cast<float*>(alloc(T * d * 4));
    bdmid_ = static_cast<float*>(alloc(T * d * 4));
    bdmid16_ = alloc(T * d * 2);
    bdbig_ = alloc(T * static_cast<size_t>(std::max(lay_.mlp_cols, lay_.qkv_cols)) * 2);
    bdo_ = alloc(T * hhd * 2);
    bdelta_ = static_cast<float*>(alloc(lse * 4));
    for (int i = 0; i < 2; ++i) {
        bdres_[i] = static_cast<float*>(alloc(T * d * 4));
        bdres16_[i] = alloc(T * d * 2);
    }
    // gradient images hold world equal shards when reduce-scattered (sharded streaming)
    const size_t grad_f = std::max(img_f(), shardA_ / 4 * static_cast<size_t>(world_));
    for (auto& g : bgimg_) {
        g = static_cast<float*>(alloc(grad_f * 4));
        CUDA_OK(cudaMemset(g, 0, grad_f * 4));  // alignment gaps between tensors stay zero
    }
    grad_red_ = bgimg_[0];  // (unused in block mode: the gradient image is reduced in place)
    // dW split-K partial regions, one per split matrix, per layer parity (sized by the split
    // count at the allocation's row capacity; smaller calls never use more: block_dw caps it)
    bdw_off_.assign(lay_.t.size(), 0);
    bdw_cap_.assign(lay_.t.size(), 1);
    size_t ws = 0;
    for (size_t i = 0; i < lay_.t.size(); ++i) {
        const BlockTensor& t = lay_.t[i];
        if (!t.matrix) continue;
        const DwChoice c = choose_dw(static_cast<int>(t.rows), static_cast<int>(t.cols), static_cast<int>(R), 16, false);
        if (c.splits <= 1) continue;
        bdw_cap_[i] = c.splits;
        bdw_off_[i] = ws;
        ws += static_cast<size_t>(c.splits) * t.count();
    }
    for (int p = 0; p < 2; ++p) {
        bws_[p] = ws ? static_cast<float*>(alloc(ws * 4)) : nullptr;
        bdw_pending_[p].clear();
        bdw_last_[p].clear();
    }
    const int widest = std::max({lay_.qkv_cols, lay_.mlp_cols, d_});
    const ColScratchSize cs = col_scratch_size(R, widest);
    bcs_.part = static_cast<float*>(alloc(cs.part_floats * 4));
    bcs_.counters = static_cast<int*>(alloc(cs.counters * 4));
    CUDA_OK(cudaMemset(bcs_.counters, 0, cs.counters * 4));  // each kernel leaves them zero
    // b1's gradient: column sums of dh, formed in the GELU' GEMM's epilogue per 32-row group
    bb1p_ = nullptr;
    bqkvp_ = nullptr;
    if (!lay_.swiglu() && lay_.b1 >= 0)
        bb1p_ = static_cast<float*>(alloc(static_cast<size_t>((R + 31) / 32) * static_cast<size_t>(lay_.desc.ff) * 4));
    if (lay_.bqkv >= 0 && lay_.desc.seq_len % 32 == 0)
        bqkvp_ = static_cast<float*>(alloc(static_cast<size_t>(R / 32) * static_cast<size_t>(lay_.qkv_cols) * 4));
    fused_norm_ = norm_backward_fused_ok(d_);
    if (fused_norm_) {
        const size_t nc = static_cast<size_t>(norm_bwd_chunks(R));
        bnp_ = static_cast<float*>(alloc(nc * 2 * d * 4));
        bnc_ = static_cast<float*>(alloc(nc * d * 4));
        bcarry_ = static_cast<float*>(alloc(nc * d * 4));
    }
}

// The update regions of a split master in slot `slot` (block.hpp): each tensor's halves or fp32
// vector, at its logical offset in the gradient / moment arrays.
SplitRegions Executor::split_regions(int slot) const {
    SplitRegions r;
    uint8_t* base = slot_ptr(slot);
    for (const BlockTensor& t : lay_.t) {
        r.hi[r.n] = base + t.wire_off;
        r.lo[r.n] = t.matrix ? reinterpret_cast<uint16_t*>(base + lay_.wire_bytes + t.lo_off) : nullptr;
        r.off[r.n] = static_cast<int64_t>(t.off);
        r.count[r.n] = static_cast<int64_t>(t.count());
        ++r.n;
    }
    return r;
}

// The slot's bf16 operand region in wire layout: matrices converted, vectors copied (fp32).
void Executor::block_convert(int slot, cudaStream_t st) {
    ConvertRegions r;
    const float* img = slot_w32(slot);
    uint8_t* wire = static_cast<uint8_t*>(slot_w16(slot));
    for (const BlockTensor& t : lay_.t) {
        r.src[r.n] = img + t.off;
        r.dst[r.n] = wire + t.wire_off;
        r.count[r.n] = static_cast<int64_t>(t.count());
        r.to_bf16[r.n] = t.matrix ? 1 : 0;
        ++r.n;
    }
    convert_regions(r, st);
    ++kernels_;
}

bool Executor::attention(bool backward, const BlockActs& a, const void* dout, void* dqkv, int64_t rows,
                         cudaStream_t st, bool want_colsum) {
    AttnProblem p;
    p.tokens = rows;
    p.seq_len = lay_.desc.seq_len;
    p.n_heads = lay_.desc.n_heads;
    p.n_kv_heads = lay_.desc.n_kv_heads;
    p.head_dim = lay_.head_dim;
    p.causal = lay_.desc.causal;
    p.qkv = a.qkv;
    p.o = a.o;
    p.lse = a.lse;
    p.dout = dout;
    p.delta = bdelta_;
    p.dqkv = dqkv;
    p.colsum_part = backward && want_colsum ? bqkvp_ : nullptr;
    const bool fused = p.colsum_part && attention_colsum_fused(p);
    const cudaError_t e = backward ? attention_backward(p, st) : attention_forward(p, st);
    if (e != cudaSuccess) throw Error(SP_ERR_CUDA, std::string("attention: ") + cudaGetErrorString(e));
    const double fl = static_cast<double>(rows) * lay_.attn_flops_per_token();
    attn_flops_ += backward ? 3.5 * fl : fl;  // dK/dV pass 4 products, dQ pass 3 (vs 2 forward)
    attn_launches_ += backward ? 3 : 1;
    kernels_ += backward ? 3 : 1;
    return fused;
}

void Executor::block_forward_layer(const WirePtrs& w, const float* x, const BlockActs& a, float* y, int64_t rows,
                                   bool train, cudaStream_t st) {
    const int T = static_cast<int>(rows), d = d_, ff = lay_.desc.ff;
    const int hhd = lay_.desc.n_heads * lay_.head_dim;
    const int rms = lay_.rms() ? 1 : 0;
    const float eps = lay_.desc.norm_eps;
    norm_forward(x, w.ln1_g, w.ln1_b, rms, eps, rows, d, a.xn1, a.st1, st);
    ++kernels_;
    GemmProblem g;
    g.M = T;
    g.N = lay_.qkv_cols;
    g.K = d;
    g.A = a.xn1;
    g.lda = d;
    g.B = w.wqkv;
    g.ldb = lay_.qkv_cols;
    g.b_mn = true;
    g.epilogue = EPI_BIAS_ACT_BF16;
    g.bias = w.bqkv;
    g.out = a.qkv;
    g.ldo = lay_.qkv_cols;
    gemm(g, st);
    attention(false, a, nullptr, nullptr, rows, st);
    g = GemmProblem{};
    g.M = T;
    g.N = d;
    g.K = hhd;
    g.A = a.o;
    g.lda = hhd;
    g.B = w.wo;
    g.ldb = d;
    g.b_mn = true;
    g.epilogue = EPI_RESID_F32;
    g.bias = w.bo;
    g.gate = x;
    g.ldg = d;
    g.out = a.xmid;
    g.ldo = d;
    gemm(g, st);
    norm_forward(a.xmid, w.ln2_g, w.ln2_b, rms, eps, rows, d, a.xn2, a.st2, st);
    ++kernels_;
    g = GemmProblem{};
    g.M = T;
    g.N = lay_.mlp_cols;
    g.K = d;
    g.A = a.xn2;
    g.lda = d;
    g.B = w.w1;
    g.ldb = lay_.mlp_cols;
    g.b_mn = true;
    g.bias = w.b1;
    g.out = a.g;
    g.ldo = ff;
    if (lay_.swiglu()) {
        g.epilogue = EPI_SWIGLU_BF16;
        g.bias = nullptr;  // (the Llama MLP carries no bias)
        g.aux = train ? a.h : nullptr;
        g.ldaux = lay_.mlp_cols;
    } else {
        g.epilogue = EPI_GELU_BF16;
        g.act = lay_.gelu_kind();
        g.aux = a.h;  // the backward's GELU' reads the pre-activation (inference: none kept)
        g.ldaux = ff;
    }
    gemm(g, st);
    g = GemmProblem{};
    g.M = T;
    g.N = d;
    g.K = ff;
    g.A = a.g;
    g.lda = ff;
    g.B = w.w2;
    g.ldb = d;
    g.b_mn = true;
    g.epilogue = EPI_RESID_F32;
    g.bias = w.b2;
    g.gate = a.xmid;
    g.ldg = d;
    g.out = y;
    g.ldo = d;
    gemm(g, st);
}

// dW = act^T grad ([rows][M] and [rows][N] bf16) of matrix tensor `ti` (M x N fp32). With one
// split the GEMM writes the layer's gradient image directly; with several it writes fp32
// partials into the matrix's region of the parity's workspace, and the layer's UPDATE op sums
// them in a fixed order on the update stream (block_reduce_pending / split_update), off the
// compute stream. The split count depends only on the shape (and the workspace's capacity).
void Executor::block_dw(int L, int ti, const void* act, const void* grad, int64_t rows, cudaStream_t st) {
    const BlockTensor& t = lay_.t[static_cast<size_t>(ti)];
    const int M = static_cast<int>(t.rows), N = static_cast<int>(t.cols);
    const int cap = bdw_cap_[static_cast<size_t>(ti)];
    const DwChoice c = choose_dw(M, N, static_cast<int>(rows), cap, false);
    GemmProblem g;
    g.M = M;
    g.N = N;
    g.K = static_cast<int>(rows);
    g.A = act;
    g.lda = M;
    g.a_mn = true;
    g.B = grad;
    g.ldb = N;
    g.b_mn = true;
    g.epilogue = EPI_F32;
    g.cta = c.cta;
    g.block_n = c.block_n;
    g.splits = c.splits;
    g.ldo = N;
    g.split_stride = static_cast<int64_t>(M) * N;  // (a valid 3-D partial map even for one split)
    if (c.splits == 1) {
        g.out = bgimg_[L % 2] + t.off;
        gemm(g, st);
        return;
    }
    DwPartials p;
    p.tensor = ti;
    p.splits = effective_splits(g.K, c.splits);
    p.parts = bws_[L % 2] + bdw_off_[static_cast<size_t>(ti)];
    g.out = p.parts;
    gemm(g, st);
    bdw_pending_[L % 2].push_back(p);
}

// The pending dW partials of the layer of parity `parity` -> its gradient image (fixed order).
void Executor::block_reduce_pending(int parity, cudaStream_t st) {
    for (const DwPartials& p : bdw_pending_[parity]) {
        const BlockTensor& t = lay_.t[static_cast<size_t>(p.tensor)];
        const int64_t n = static_cast<int64_t>(t.count());
        reduce_partials(p.parts, p.splits, n, n, bgimg_[parity] + t.off, st);
        ++kernels_;
    }
    bdw_pending_[parity].clear();
}

void Executor::block_colsum(const void* x, int64_t rows, int N, float* out, cudaStream_t st) {
    colsum_total_bf16(x, rows, N, bcs_, out, st);
    ++kernels_;
}

void Executor::block_backward_layer(int L, const WirePtrs& w, const float* x, const BlockActs& a, int64_t rows,
                                    cudaStream_t st) {
    const int T = static_cast<int>(rows), d = d_, ff = lay_.desc.ff;
    const int hhd = lay_.desc.n_heads * lay_.head_dim;
    const int rms = lay_.rms() ? 1 : 0;
    const bool trainable = !frozen_[static_cast<size_t>(L)];
    const bool need_dx = L > 0;
    if (!trainable && !need_dx) return;
    float* gi = bgimg_[L % 2];
    auto at = [&](int idx) { return gi + lay_.t[static_cast<size_t>(idx)].off; };
    const float* dy = bdres_[L % 2];
    const void* dy16 = bdres16_[L % 2];
    // --- MLP: y = h + W2^T g(h W1 + b1) + b2
    if (trainable) {
        block_dw(L, lay_.w2, a.g, dy16, rows, st);
        if (lay_.b2 >= 0) {
            if (fused_norm_ && L < n_ - 1) {  // the layer above's norm1 left its output's chunk sums
                norm_param_reduce(rows, nullptr, bcarry_, at(lay_.b2), st);
            } else {
                block_colsum(dy16, rows, d, at(lay_.b2), st);
            }
        }
    }
    GemmProblem g;
    g.M = T;
    g.N = ff;
    g.K = d;
    g.A = dy16;
    g.lda = d;
    g.B = w.w2;  // W2 [ff][d]: K-major B of dg = dy W2^T
    g.ldb = d;
    g.epilogue = EPI_GELU_GATE_BF16;
    g.gate = a.h;
    g.ldg = ff;
    g.act = lay_.gelu_kind();
    g.out = bdbig_;  // dh
    g.ldo = ff;
    const bool b1_fused = trainable && lay_.b1 >= 0 && bb1p_;
    if (b1_fused) g.colsum_part = bb1p_;  // + the column sums of dh per 32-row group (b1)
    gemm(g, st);
    if (trainable) {
        block_dw(L, lay_.w1, a.xn2, bdbig_, rows, st);
        if (b1_fused) {
            ColChunks c;
            c.n = 1;
            c.chunks = static_cast<int>((rows + 31) / 32);
            c.part[0] = bb1p_;
            c.stride[0] = ff;
            c.width[0] = ff;
            c.out[0] = at(lay_.b1);
            reduce_col_chunks(c, st);
            ++kernels_;
        } else if (lay_.b1 >= 0) {
            block_colsum(bdbig_, rows, ff, at(lay_.b1), st);
        }
    }
    g = GemmProblem{};
    g.M = T;
    g.N = d;
    g.K = ff;
    g.A = bdbig_;
    g.lda = ff;
    g.B = w.w1;  // W1 [d][ff]: K-major B of dxn2 = dh W1^T
    g.ldb = ff;
    g.epilogue = EPI_F32;
    g.out = bdxn_;
    g.ldo = d;
    gemm(g, st);
    // norm2: dh_res = dy + norm2'(dxn2)
    if (fused_norm_) {  // + its parameter gradients and bo's (the column sums of dh_res), one pass
        const bool csum = trainable && lay_.bo >= 0;
        norm_backward_fused(bdxn_, a.xmid, a.st2, w.ln2_g, rms, rows, d, dy, bdmid_, bdmid16_,
                            trainable ? bnp_ : nullptr, csum ? bnc_ : nullptr, st);
        ++kernels_;
        if (trainable) norm_param_reduce(rows, at(lay_.ln2_g), csum ? bnc_ : nullptr, csum ? at(lay_.bo) : nullptr, st);
    } else {
        norm_backward(bdxn_, a.xmid, a.st2, w.ln2_g, rms, rows, d, dy, bdmid_, bdmid16_, bcs_,
                      trainable ? at(lay_.ln2_g) : nullptr, st);
        kernels_ += trainable ? 2 : 1;
    }
    // --- attention: h = x + Wo^T attn(norm1(x) Wqkv + bqkv) + bo
    if (trainable) {
        block_dw(L, lay_.wo, a.o, bdmid16_, rows, st);
        if (lay_.bo >= 0 && !fused_norm_) block_colsum(bdmid16_, rows, d, at(lay_.bo), st);
    }
    g = GemmProblem{};
    g.M = T;
    g.N = hhd;
    g.K = d;
    g.A = bdmid16_;
    g.lda = d;
    g.B = w.wo;  // Wo [hhd][d]: K-major B of do = dh Wo^T
    g.ldb = d;
    g.epilogue = EPI_GATE_BF16;  // relu = 0: a plain bf16 store
    g.out = bdo_;
    g.ldo = hhd;
    gemm(g, st);
    // dqkv (+ bqkv's column partials from the passes' epilogues where the shape allows)
    const bool bqkv_fused = attention(true, a, bdo_, bdbig_, rows, st, trainable && lay_.bqkv >= 0 && bqkvp_);
    if (trainable) {
        block_dw(L, lay_.wqkv, a.xn1, bdbig_, rows, st);
        if (bqkv_fused) {
            ColChunks c;
            c.n = 1;
            c.chunks = static_cast<int>(rows / 32);
            c.part[0] = bqkvp_;
            c.stride[0] = lay_.qkv_cols;
            c.width[0] = lay_.qkv_cols;
            c.out[0] = at(lay_.bqkv);
            reduce_col_chunks(c, st);
            ++kernels_;
        } else if (lay_.bqkv >= 0) {
            block_colsum(bdbig_, rows, lay_.qkv_cols, at(lay_.bqkv), st);
        }
    }
    g = GemmProblem{};
    g.M = T;
    g.N = d;
    g.K = lay_.qkv_cols;
    g.A = bdbig_;
    g.lda = lay_.qkv_cols;
    g.B = w.wqkv;  // Wqkv [d][qkv]: K-major B of dxn1 = dqkv Wqkv^T
    g.ldb = lay_.qkv_cols;
    g.epilogue = EPI_F32;
    g.out = bdxn_;
    g.ldo = d;
    gemm(g, st);
    // norm1: dx = dh_res + norm1'(dxn1) -> the gradient the layer below reads (layer 0: none)
    if (fused_norm_) {  // + the chunk sums of dx: the layer below's b2 gradient (carried)
        const bool carry = need_dx && !frozen_[static_cast<size_t>(L) - 1] && lay_.b2 >= 0;
        norm_backward_fused(bdxn_, x, a.st1, w.ln1_g, rms, rows, d, bdmid_, need_dx ? bdres_[(L + 1) % 2] : nullptr,
                            need_dx ? bdres16_[(L + 1) % 2] : nullptr, trainable ? bnp_ : nullptr,
                            carry ? bcarry_ : nullptr, st);
        ++kernels_;
        if (trainable) norm_param_reduce(rows, at(lay_.ln1_g), nullptr, nullptr, st);
        return;
    }
    norm_backward(bdxn_, x, a.st1, w.ln1_g, rms, rows, d, bdmid_, need_dx ? bdres_[(L + 1) % 2] : nullptr,
                  need_dx ? bdres16_[(L + 1) % 2] : nullptr, bcs_, trainable ? at(lay_.ln1_g) : nullptr, st);
    kernels_ += (need_dx ? 1 : 0) + (trainable ? 1 : 0);
}

// The fused norm backward's chunk partials -> the gradient image: the norm parameters (g_out:
// gamma, then LayerNorm's beta) and / or one column-sum vector (csum_part -> csum_out).
void Executor::norm_param_reduce(int64_t rows, float* g_out, float* csum_part, float* csum_out, cudaStream_t st) {
    ColChunks c;
    c.chunks = norm_bwd_chunks(rows);
    if (g_out) {
        c.part[c.n] = bnp_;
        c.stride[c.n] = 2 * static_cast<int64_t>(d_);
        c.width[c.n] = lay_.rms() ? d_ : 2 * d_;
        c.out[c.n] = g_out;
        ++c.n;
    }
    if (csum_part) {
        c.part[c.n] = csum_part;
        c.stride[c.n] = d_;
        c.width[c.n] = d_;
        c.out[c.n] = csum_out;
        ++c.n;
    }
    reduce_col_chunks(c, st);
    ++kernels_;
}

void Executor::block_compute(const Op& op, bool train, int64_t rows, int fmt) {
    const int L = op.layer, s = op.slot;
    const size_t act = static_cast<size_t>(rows) * d_;
    const bool ckpt = train && cfg_.checkpointing && cfg_.strategy != SP_STANDARD;
    cudaStream_t st = s_comp_;
    if (rows % lay_.desc.seq_len != 0)
        throw Error(SP_ERR_INVALID, "rows must be a multiple of the block's seq_len");
    if (!split_ && fmt != kFmtBf16Infer && w16_layer_[s] != L) {  // plain master: the bf16 operand copy
        block_convert(s, st);
        w16_layer_[s] = L;
    }
    const WirePtrs w = wire_ptrs(static_cast<const uint8_t*>(slot_w16(s)));
    if (!train) {
        const float* x_item = cur_x_ + static_cast<size_t>(op.item) * act;
        float* y_item = cur_y_ + static_cast<size_t>(op.item) * act;
        const float* in = L == 0 ? x_item : static_cast<const float*>(pp_[(L - 1) % 2]);
        float* out = L == n_ - 1 ? y_item : static_cast<float*>(pp_[L % 2]);
        block_forward_layer(w, in, bscr_, out, rows, false, st);
        return;
    }
    if (op.pass == 0) {  // training forward: x_L -> x_{L+1}
        if (ckpt) {
            float* xL = static_cast<float*>(fa_[L % 3]);
            if (L == 0) {
                void* dst[1] = {xL};
                const void* src[1] = {cur_x_};
                copy_regions(dst, src, 1, static_cast<int64_t>(act * 4), st);
                ++kernels_;
            }
            float* out = L == n_ - 1 ? yout_ : static_cast<float*>(fa_[(L + 1) % 3]);
            block_forward_layer(w, xL, bscr_, out, rows, true, st);
            return;
        }
        if (L == 0) {
            void* dst[1] = {bx_[0]};
            const void* src[1] = {cur_x_};
            copy_regions(dst, src, 1, static_cast<int64_t>(act * 4), st);
            ++kernels_;
        }
        block_forward_layer(w, bx_[static_cast<size_t>(L)], bsv_[static_cast<size_t>(L)], bx_[static_cast<size_t>(L) + 1],
                            rows, true, st);
        return;
    }
    if (ckpt) {  // the reloaded input; recompute the block's intermediates, then its backward
        const float* xL = static_cast<const float*>(ba_[static_cast<size_t>(s)]);
        block_forward_layer(w, xL, bscr_, static_cast<float*>(pp_[0]), rows, true, st);
        block_backward_layer(L, w, xL, bscr_, rows, st);
        return;
    }
    block_backward_layer(L, w, bx_[static_cast<size_t>(L)], bsv_[static_cast<size_t>(L)], rows, st);
}

// MSE of the last layer's output (mse_loss / mse_grad, model.cpp:131-148): the fp32 gradient
// of the residual stream and its bf16 copy for the first backward GEMMs.
void Executor::block_loss(int64_t rows) {
    const int64_t count = rows * d_;
    const float inv_n = 1.0f / static_cast<float>(count * world_);
    const int last = n_ - 1;
    loss_blocks_ = loss_grad_f32(yout_, cur_t_, count, inv_n, 0, bdres_[last % 2], loss_parts_, s_comp_);
    loss_finalize(loss_parts_, loss_blocks_, loss_dev_, s_comp_);
    convert_f32_to_bf16(bdres_[last % 2], bdres16_[last % 2], count, s_comp_);
    kernels_ += 3;
}

void Executor::debug_read_grad(int index, float* out) {
    if (!blk_) throw Error(SP_ERR_INVALID, "debug_read_grad: transformer-block executors only");
    if (index < 0 || index > 1 || index >= n_) throw Error(SP_ERR_INVALID, "debug_read_grad: layers 0 and 1 only");
    if (sharded_) throw Error(SP_ERR_STATE, "debug_read_grad: not in sharded data parallel");
    if (!bgimg_[index % 2]) throw Error(SP_ERR_STATE, "debug_read_grad: no train step yet");
    CUDA_OK(cudaDeviceSynchronize());
    // split-K dW partials the update summed in place: fold them into the image first
    for (const DwPartials& p : bdw_last_[index % 2]) {
        const BlockTensor& t = lay_.t[static_cast<size_t>(p.tensor)];
        const int64_t n = static_cast<int64_t>(t.count());
        reduce_partials(p.parts, p.splits, n, n, bgimg_[index % 2] + t.off, nullptr);
    }
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaMemcpy(out, bgimg_[index % 2], img_f() * 4, cudaMemcpyDeviceToHost));
}

}  // namespace sp

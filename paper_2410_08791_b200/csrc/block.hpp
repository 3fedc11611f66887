// block.hpp — named-shape transformer layers: parameter-image layout and FLOP accounting.
//
// The reference streams one square dense LayerBlock per layer (model.hpp:14-26). A named-shape
// layer is a pre-norm transformer block whose parameters form ONE flat fp32 image, so the ring,
// the ledger, the write-back and the data-parallel sharding treat it exactly like a LayerBlock
// image of another size (include/superpipe.h "named-shape layers").
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/superpipe.h"

namespace sp {

struct BlockTensor {
    std::string name;
    int64_t rows = 1, cols = 0;
    bool matrix = false;
    uint64_t off = 0;       // floats, in the fp32 image
    uint64_t wire_off = 0;  // bytes, in the bf16 wire image (matrices bf16, vectors fp32)
    uint64_t lo_off = 0;    // matrices: bytes in the low-half plane of the split image
    uint64_t count() const { return static_cast<uint64_t>(rows) * static_cast<uint64_t>(cols); }
};

struct BlockLayout {
    sp_block_desc desc{};
    int head_dim = 0, qkv_cols = 0, mlp_cols = 0;  // mlp_cols: ff (GELU) or 2 ff (SwiGLU)
    std::vector<BlockTensor> t;
    // tensor indices (-1 when absent)
    int ln1_g = -1, ln1_b = -1, wqkv = -1, bqkv = -1, wo = -1, bo = -1, ln2_g = -1, ln2_b = -1,
        w1 = -1, b1 = -1, w2 = -1, b2 = -1;
    uint64_t n_floats = 0, wire_bytes = 0, n_params = 0;
    // Split master image: [wire image | low halves of the matrices]. A matrix parameter's fp32
    // bits are (hi << 16 | lo): hi, the bf16 truncation the GEMMs multiply, lives in the wire
    // image, lo in the plane after it. The forward streams the wire prefix alone (2 B per
    // matrix parameter), the backward the whole image; the master stays exact fp32.
    uint64_t lo_bytes = 0, split_bytes = 0;
    bool rms() const { return desc.norm == SP_NORM_RMS; }
    bool swiglu() const { return desc.mlp == SP_MLP_SWIGLU; }
    int gelu_kind() const { return desc.mlp == SP_MLP_GELU_ERF ? 1 : 0; }
    // Algorithmic FLOPs per token of one forward pass: the linear layers (2 x params of the
    // matrices) and the attention core (QK^T and PV: 4 hd per attended key per head; causal
    // sequences attend (S + 1) / 2 keys on average).
    double linear_flops_per_token() const;
    double attn_flops_per_token() const;
};

// Validates the descriptor and lays out the image; returns an error message or "".
std::string make_block_layout(const sp_block_desc& desc, BlockLayout& out);

}  // namespace sp

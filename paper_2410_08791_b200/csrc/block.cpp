// block.cpp — named-shape layer image layout, deterministic init and the C ABI helpers for it.
#include "block.hpp"

#include <cmath>
#include <cstring>

namespace sp {

namespace {
constexpr uint64_t kAlignFloats = 64;  // every tensor starts on a 256-byte boundary
constexpr uint64_t kAlignBytes = 256;
uint64_t up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

struct SplitMix64 {  // model.hpp:40-52 (the reference's generator)
    uint64_t state;
    explicit SplitMix64(uint64_t s) : state(s) {}
    uint64_t next() {
        state += 0x9E3779B97F4A7C15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};
}  // namespace

std::string make_block_layout(const sp_block_desc& d, BlockLayout& L) {
    L = BlockLayout{};
    L.desc = d;
    if (d.kind != SP_BLOCK_TRANSFORMER) return "block: kind must be SP_BLOCK_TRANSFORMER";
    if (d.d < 64 || d.d % 64 != 0) return "block: d must be a positive multiple of 64";
    if (d.n_heads < 1 || d.d % d.n_heads != 0) return "block: n_heads must divide d";
    if (d.n_kv_heads < 1 || d.n_heads % d.n_kv_heads != 0) return "block: n_kv_heads must divide n_heads";
    L.head_dim = d.d / d.n_heads;
    if (L.head_dim != 64 && L.head_dim != 80 && L.head_dim != 128) return "block: head_dim (d / n_heads) must be 64, 80 or 128";
    if (d.ff < 64 || d.ff % 64 != 0) return "block: ff must be a positive multiple of 64";
    if (d.seq_len < 1) return "block: seq_len must be >= 1";
    if (d.norm != SP_NORM_LAYER && d.norm != SP_NORM_RMS) return "block: unknown norm";
    if (d.mlp != SP_MLP_GELU_TANH && d.mlp != SP_MLP_GELU_ERF && d.mlp != SP_MLP_SWIGLU) return "block: unknown mlp";
    if (!(d.norm_eps > 0.0f)) return "block: norm_eps must be > 0";
    L.qkv_cols = (d.n_heads + 2 * d.n_kv_heads) * L.head_dim;
    L.mlp_cols = L.swiglu() ? 2 * d.ff : d.ff;
    uint64_t off = 0, woff = 0;
    auto add = [&](const char* name, int64_t rows, int64_t cols, bool matrix) {
        BlockTensor t;
        t.name = name;
        t.rows = rows;
        t.cols = cols;
        t.matrix = matrix;
        t.off = off;
        t.wire_off = woff;
        off = up(off + t.count(), kAlignFloats);
        woff = up(woff + t.count() * (matrix ? 2 : 4), kAlignBytes);
        L.n_params += t.count();
        L.t.push_back(t);
        return static_cast<int>(L.t.size()) - 1;
    };
    const bool ln = d.norm == SP_NORM_LAYER;
    L.ln1_g = add("norm1.g", 1, d.d, false);
    if (ln) L.ln1_b = add("norm1.b", 1, d.d, false);
    L.wqkv = add("wqkv", d.d, L.qkv_cols, true);
    if (d.bias) L.bqkv = add("bqkv", 1, L.qkv_cols, false);
    L.wo = add("wo", static_cast<int64_t>(d.n_heads) * L.head_dim, d.d, true);
    if (d.bias) L.bo = add("bo", 1, d.d, false);
    L.ln2_g = add("norm2.g", 1, d.d, false);
    if (ln) L.ln2_b = add("norm2.b", 1, d.d, false);
    L.w1 = add(L.swiglu() ? "wgu" : "w1", d.d, L.mlp_cols, true);
    if (d.bias) L.b1 = add(L.swiglu() ? "bgu" : "b1", 1, L.mlp_cols, false);
    L.w2 = add("w2", d.ff, d.d, true);
    if (d.bias) L.b2 = add("b2", 1, d.d, false);
    L.n_floats = off;
    L.wire_bytes = woff;
    uint64_t lo = 0;
    for (BlockTensor& t : L.t) {
        if (!t.matrix) continue;
        t.lo_off = lo;
        lo = up(lo + t.count() * 2, kAlignBytes);
    }
    L.lo_bytes = lo;
    L.split_bytes = L.wire_bytes + L.lo_bytes;
    return "";
}

double BlockLayout::linear_flops_per_token() const {
    double macs = 0;
    for (const BlockTensor& x : t)
        if (x.matrix) macs += static_cast<double>(x.count());
    return 2.0 * macs;
}

double BlockLayout::attn_flops_per_token() const {
    const double S = desc.seq_len;
    const double keys = desc.causal ? (S + 1.0) / 2.0 : S;
    return 4.0 * keys * head_dim * desc.n_heads;
}

}  // namespace sp

extern "C" int sp_block_layout(const sp_block_desc* blk, sp_block_tensor* tensors, int32_t cap, int32_t* count,
                               uint64_t* n_floats, uint64_t* wire_bytes) {
    if (!blk) return SP_ERR_INVALID;
    sp::BlockLayout L;
    if (!sp::make_block_layout(*blk, L).empty()) return SP_ERR_INVALID;
    if (count) *count = static_cast<int32_t>(L.t.size());
    if (n_floats) *n_floats = L.n_floats;
    if (wire_bytes) *wire_bytes = L.wire_bytes;
    for (int32_t i = 0; tensors && i < cap && i < static_cast<int32_t>(L.t.size()); ++i) {
        sp_block_tensor& o = tensors[i];
        std::memset(&o, 0, sizeof(o));
        std::strncpy(o.name, L.t[static_cast<size_t>(i)].name.c_str(), sizeof(o.name) - 1);
        o.rows = L.t[static_cast<size_t>(i)].rows;
        o.cols = L.t[static_cast<size_t>(i)].cols;
        o.offset = L.t[static_cast<size_t>(i)].off;
        o.wire_offset = L.t[static_cast<size_t>(i)].wire_off;
        o.matrix = L.t[static_cast<size_t>(i)].matrix ? 1 : 0;
    }
    return SP_OK;
}

extern "C" int sp_build_block(const sp_block_desc* blk, uint64_t seed, int32_t index, float* params) {
    if (!blk || !params || index < 0) return SP_ERR_INVALID;
    sp::BlockLayout L;
    if (!sp::make_block_layout(*blk, L).empty()) return SP_ERR_INVALID;
    std::memset(params, 0, L.n_floats * sizeof(float));
    // layer_stream_seed (model.cpp:11-14)
    sp::SplitMix64 rng(seed ^ (0xA24BAED4963EE407ull * (static_cast<uint64_t>(index) + 1) + 0x9FB21C651E98DF25ull));
    double bound = 1.0;
    for (const sp::BlockTensor& t : L.t) {
        float* p = params + t.off;
        const bool gain = t.name == "norm1.g" || t.name == "norm2.g";
        const bool shift = t.name == "norm1.b" || t.name == "norm2.b";
        if (gain) {
            for (uint64_t e = 0; e < t.count(); ++e) p[e] = 1.0f;
        } else if (shift) {
            // zero (memset)
        } else {
            if (t.matrix) bound = 1.0 / std::sqrt(static_cast<double>(t.rows));  // fan_in of [in][out]
            for (uint64_t e = 0; e < t.count(); ++e) p[e] = static_cast<float>((2.0 * rng.unit() - 1.0) * bound);
        }
    }
    return SP_OK;
}

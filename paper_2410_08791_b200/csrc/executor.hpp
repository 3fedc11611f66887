// executor.hpp — the B200 ring executor behind the C ABI (include/superpipe.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/superpipe.h"
#include "block.hpp"
#include "kernels.hpp"
#include "plan.hpp"

namespace sp {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Content format of the HBM ring slots (cached slot contents are only reusable within a
// format): exact fp32, bf16 training (fp32 master + derived bf16), bf16 inference wire.
enum SlotFormat : int { kFmtExactF32 = 0, kFmtBf16Train = 1, kFmtBf16Infer = 2 };

class Executor {
public:
    explicit Executor(const sp_config& cfg, const sp_block_desc* block = nullptr);
    ~Executor();

    void register_layer(int index, const float* W, const float* b, int activation, int frozen);
    void forward(const float* x, int64_t rows, int n_items, float* y, bool device_io);
    float train_step(const float* x, const float* target, int64_t rows, float lr,
                     bool device_io);
    void read_layer(int index, float* W, float* b);
    // named-shape layers (transformer blocks): one flat fp32 image per layer
    void register_block(int index, const float* params, int frozen);
    void read_block(int index, float* params);
    bool is_block() const { return blk_; }
    void debug_read_grad(int index, float* out);
    void digest_train(float loss, char out[17]);
    void set_trace(int level) { cfg_.trace = level; }
    void set_item_batching(bool on) { item_batching_ = on; }
    void set_eager_prefetch(bool on) { eager_prefetch_ = on; }
    void set_debug(const std::string& key, int value);
    std::string last_plan_text() const { return describe_plan(last_plan_); }
    const Plan& last_plan() const { return last_plan_; }
    void dp_init(const uint8_t id[128], int rank, int world, bool shard_weights);
    void dp_sync();
    // Optimizer: SP_OPT_SGD (apply_sgd, the reference) or SP_OPT_ADAMW (state m, v in pinned
    // host memory, streamed with each trainable layer's backward). Resets the state and step.
    void set_optimizer(int kind, float beta1, float beta2, float eps, float weight_decay);
    void read_optimizer_state(int index, float* mW, float* mb, float* vW, float* vb);
    // Moves the pinned fp32 master into a named POSIX shared-memory segment (create) or
    // attaches to one another process created (layer metadata included), registered with
    // CUDA in every process: one host copy serves all ranks of a node.
    void share_host_master(const char* name, bool create);

    const sp_stats& stats() const { return stats_; }
    const std::vector<sp_trace_event>& trace() const { return trace_; }
    std::string error;

private:
    // layout helpers: a layer's fp32 image is [W | b] (dense) or the block image (block.hpp)
    // img_f: floats of a layer's logical fp32 image (the gradient / AdamW-state layout).
    // layer_bytes: bytes of the master as stored and streamed - the fp32 image, or (split_) the
    // split image [wire | low halves] of block.hpp. opt_bytes: one AdamW moment array.
    size_t img_f() const { return blk_ ? static_cast<size_t>(lay_.n_floats) : static_cast<size_t>(d_) * d_ + d_; }
    uint64_t layer_bytes() const {
        return infer_only_ ? lay_.wire_bytes : split_ ? lay_.split_bytes : static_cast<uint64_t>(img_f()) * 4;
    }
    uint64_t opt_bytes() const { return static_cast<uint64_t>(img_f()) * 4; }
    // host master of layer L: one stride fits either block layout, so dp_init can switch in place
    uint8_t* host_layer(int L) const { return reinterpret_cast<uint8_t*>(host32_) + static_cast<size_t>(L) * host_stride_; }
    float* host_opt(float* base, int L) const { return base + static_cast<size_t>(L) * img_f(); }
    uint64_t wire16_bytes() const {
        return blk_ ? lay_.wire_bytes : static_cast<uint64_t>(d_) * d_ * 2 + d_ * 4ull;
    }
    size_t act_elt() const { return (blk_ || !bf16_) ? 4 : 2; }  // saved layer-input element
    uint8_t* slot_ptr(int s) const { return slots_dev_ + static_cast<size_t>(s) * slot_bytes_; }
    float* slot_w32(int s) const { return reinterpret_cast<float*>(slot_ptr(s)); }
    float* slot_m32(int s) const { return reinterpret_cast<float*>(slot_ptr(s) + off_m_); }  // AdamW
    float* slot_v32(int s) const { return reinterpret_cast<float*>(slot_ptr(s) + off_v_); }
    float* slot_b32(int s) const { return slot_w32(s) + static_cast<size_t>(d_) * d_; }
    void* slot_w16(int s) const { return slot_ptr(s) + off_w16_; }
    float* slot_b16(int s) const {  // bias of the bf16 inference wire image
        return reinterpret_cast<float*>(slot_ptr(s) + off_w16_ + static_cast<size_t>(d_) * d_ * 2);
    }

    // What one call moves across the host boundary (user pointers; device or host).
    struct CallIO {
        bool train;
        int n_items;
        int64_t rows;
        float lr;
        int fmt;
        bool device_io;
        const float* x;
        const float* t;
        float* y;
    };
    // A captured step: replayed with one cudaGraphLaunch while the call signature (plan,
    // pointers, lr, bf16-copy state, buffers) is unchanged.
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        std::vector<int> w16_after;
        std::vector<int> stale_layers;
        uint64_t kernels = 0, h2d_bytes = 0, d2h_bytes = 0;
        size_t gemm_count = 0;
        double gemm_flops = 0.0;
        uint64_t attn_launches = 0;
        double attn_flops = 0.0;
    };

    void layout_slots(int world);
    void ensure_stages();
    void flush_writebacks();
    uint8_t* stage_ptr(int i) const { return stages_dev_ + static_cast<size_t>(i) * stage_bytes_; }
    void check_ready();
    void ensure_buffers(int64_t rows, int n_items, bool train, bool device_io);
    void refresh_host16();
    // The call's plan: build_plan is a pure function of (PlanInput, initial slot content), so a
    // call whose inputs equal the previous call's reuses that plan (steady-state calls skip the
    // host-side planning). The reference is valid until the next make_plan.
    const Plan& make_plan(bool train, int n_items, int64_t rows, int fmt);
    struct PlanMemo {
        bool valid = false;
        PlanInput in;
        std::vector<SlotCache> initial;
        Plan plan;
    } memo_;
    void enqueue_call(const Plan& plan, const CallIO& io);
    void run_call(const Plan& plan, const CallIO& io);
    void run_call_impl(const Plan& plan, const CallIO& io);
    uint64_t call_signature(const Plan& plan, const CallIO& io) const;
    void enqueue_op(const Plan& plan, int i, bool train, int n_items, int64_t rows, float lr,
                    int fmt);
    void compute_op(const Op& op, bool train, int64_t rows, int fmt);
    void loss_op(int64_t rows);
    // true: it also filled the op's write-back stage; keep_slot: the plan leaves the layer valid
    // in its slot at the end of the call (the slot must hold the update too)
    bool update_op(const Op& op, float lr, bool keep_slot = true);
    void collect_stats(const Plan& plan, int n_items, bool train);
    void gemm(const struct GemmProblem& g, cudaStream_t st);
    // transformer blocks (block_exec.cpp)
    struct BlockActs {  // one layer's forward intermediates (saved for its backward)
        void *xn1 = nullptr, *qkv = nullptr, *o = nullptr, *xn2 = nullptr, *h = nullptr, *g = nullptr;
        float *st1 = nullptr, *st2 = nullptr, *lse = nullptr, *xmid = nullptr;
    };
    struct WirePtrs {  // bf16 matrices + fp32 vectors of one layer image in wire layout
        const void *wqkv = nullptr, *wo = nullptr, *w1 = nullptr, *w2 = nullptr;
        const float *ln1_g = nullptr, *ln1_b = nullptr, *bqkv = nullptr, *bo = nullptr, *ln2_g = nullptr,
                    *ln2_b = nullptr, *b1 = nullptr, *b2 = nullptr;
    };
    WirePtrs wire_ptrs(const uint8_t* wire) const;
    void block_alloc(int64_t R, int items, bool train, const std::function<void*(size_t)>& alloc);
    void block_convert(int slot, cudaStream_t st);
    void block_forward_layer(const WirePtrs& w, const float* x, const BlockActs& a, float* y, int64_t rows,
                             bool train, cudaStream_t st);
    void block_backward_layer(int L, const WirePtrs& w, const float* x, const BlockActs& a, int64_t rows,
                              cudaStream_t st);
    void block_compute(const Op& op, bool train, int64_t rows, int fmt);
    void block_loss(int64_t rows);
    void block_dw(int L, int tensor, const void* act, const void* grad, int64_t rows, cudaStream_t st);
    void block_colsum(const void* x, int64_t rows, int N, float* out, cudaStream_t st);
    // returns true when the backward also formed bqkv's column partials (bqkvp_)
    bool attention(bool backward, const BlockActs& a, const void* dout, void* dqkv, int64_t rows, cudaStream_t st,
                   bool want_colsum = false);
    cudaStream_t stream_of(OpKind k) const;

    sp_config cfg_;
    int n_ = 0, d_ = 0;
    bool blk_ = false;  // named-shape transformer layers (block.hpp) instead of dense blocks
    BlockLayout lay_;
    // Split master (block.hpp): the forward streams only the wire prefix of each layer. Off in
    // sharded data parallel (whose byte shards assume the fp32 image), where the slot keeps a
    // device-converted bf16 copy instead.
    bool split_ = false;
    bool infer_only_ = false;  // SP_BLOCK_INFER_ONLY: the split master without its low halves
    size_t host_stride_ = 0;
    size_t fp_bytes_ = 0;  // slot bytes of the fp32 master regions [A][M][V] (the write-back stage)
    void split_image(const float* params, uint8_t* dst) const;    // fp32 image -> split image
    void unsplit_image(const uint8_t* src, float* params) const;  // split image -> fp32 image
    void set_split(bool on);
    SplitRegions split_regions(int slot) const;
    // block-mode device buffers
    std::vector<float*> bx_;            // training: residual stream x_0..x_n (fp32; x_n = yout_)
    std::vector<BlockActs> bsv_;        // training: per-layer saved intermediates (no offload)
    BlockActs bscr_;                    // inference / offload recompute: one scratch set
    float *bdxn_ = nullptr, *bdmid_ = nullptr, *bdelta_ = nullptr;
    ColScratch bcs_;  // column-sum partials + counters (bias / norm parameter gradients)
    // single-pass norm backward (d <= 2048): chunk partials of the norm parameter gradients, of
    // norm2's output column sums (bo) and of norm1's (the next layer down's b2, carried across
    // the layer boundary: that layer's gradient image may still be read by an update)
    bool fused_norm_ = false;
    float *bnp_ = nullptr, *bnc_ = nullptr, *bcarry_ = nullptr;
    float* bb1p_ = nullptr;  // b1's 32-row-group column partials, from the GELU' GEMM's epilogue
    float* bqkvp_ = nullptr;  // bqkv's, from the attention backward's epilogues
    void norm_param_reduce(int64_t rows, float* g_out, float* csum_part, float* csum_out, cudaStream_t st);
    // dW split-K partials, per layer parity: each split matrix has its own region (bdw_cap_
    // splits of its size), so the UPDATE op (update stream) reduces them while the compute
    // stream moves on to the layer below. bdw_pending_[p]: what the last backward of a layer of
    // parity p left there (tensor index, partial base, split count).
    struct DwPartials {
        int tensor = -1, splits = 1;
        float* parts = nullptr;
    };
    float* bws_[2] = {nullptr, nullptr};
    std::vector<size_t> bdw_off_;  // per tensor: float offset of its region (matrices with splits)
    std::vector<int> bdw_cap_;     // per tensor: the most splits its region holds (1: none)
    std::vector<DwPartials> bdw_pending_[2];
    std::vector<DwPartials> bdw_last_[2];  // what the last UPDATE of each parity consumed
    void block_reduce_pending(int parity, cudaStream_t st);  // partials -> the gradient image
    void *bdmid16_ = nullptr, *bdbig_ = nullptr, *bdo_ = nullptr;
    float* bdres_[2] = {nullptr, nullptr};
    void* bdres16_[2] = {nullptr, nullptr};
    float* bgimg_[2] = {nullptr, nullptr};  // per-layer gradient images (ping-pong)
    uint64_t attn_launches_ = 0;
    double attn_flops_ = 0.0;
    bool bf16_ = false;  // bf16 tensor-core path (bf16 operands / activations)
    bool tf32_ = false;  // tf32 tensor-core path (fp32 operands / activations, kind::tf32)
    bool tc_ = false;    // either tensor-core path (split-K partials, masks, fused loss)
    // pinned host copies
    float* host32_ = nullptr;  // [n][d*d + d] fp32 master (W then b)
    // Shared master (share_host_master): header + master in a POSIX shm segment.
    struct ShmHeader;
    ShmHeader* shm_ = nullptr;
    size_t shm_bytes_ = 0;
    std::string shm_name_;
    bool shm_owner_ = false;
    void sync_layer_meta(int index);
    // Per-layer write versions in the segment: every host write of layer L (registration,
    // write-back) increments version[L]. Outside data parallel, where another process may
    // have written a layer, a cached ring slot or bf16 wire image is reused only if its
    // version is current (in data parallel every rank writes the same update it caches).
    size_t ver_off_ = 0;
    std::vector<uint64_t> cache_ver_, host16_ver_, plan_ver_;
    uint64_t* shm_versions() const { return reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(shm_) + ver_off_); }
    uint64_t layer_version(int L) const;
    void bump_version(int L);
    void after_call(const Plan& plan);
    uint8_t* host16_ = nullptr;  // [n][wire16] bf16 W + fp32 b (bf16 inference wire)
    std::vector<uint8_t> host16_stale_;
    std::vector<int> relu_, frozen_;
    std::vector<uint8_t> registered_;
    // Layers whose host master may be part-updated by a train step that failed after reaching
    // the device (run_call); calls refuse with SP_ERR_STATE until they are registered again.
    std::vector<uint8_t> inconsistent_;
    bool launched_ = false;  // the current call has put work on the device
    void mark_inconsistent();
    // HBM ring
    int n_slots_ = 0;
    size_t slot_bytes_ = 0, off_w16_ = 0, off_m_ = 0, off_v_ = 0;
    uint8_t* slots_dev_ = nullptr;
    std::vector<SlotCache> cache_;
    int cache_fmt_ = -1;
    // Write-back staging buffers ([A] or [A][M][V] like a slot) and the previous train step's
    // deferred write-backs (layers whose updated image lives only in its ring slot until the
    // next call's first D2H, or until flush_writebacks() before any host read).
    uint8_t* stages_dev_ = nullptr;
    int n_stages_ = 0;
    size_t stage_bytes_ = 0;
    bool staged_writeback_ = true;
    // A/B and debug knobs (set_debug; defaults are the product behaviour)
    int wb_stages_cap_ = 3;
    int defer_budget_override_ = -1;
    bool per_move_ = true, move_events_ = true;
    // Debug (SP_POISON=1): every ring-slot / activation-reload copy is preceded by a NaN fill
    // of its destination, so a read that overtakes the copy shows up as NaN (a dynamic check
    // of the plan's edges next to the static one in tests/test_plan_hazards.py).
    bool poison_ = false;
    bool drop_load_edges_ = false;  // fault injection (SP_FAULT_DROP_LOAD_EDGES=1): tests only
    std::vector<int> pending_wb_layers_, pending_wb_slots_;
    std::vector<int> w16_layer_;  // bf16 training: layer whose bf16 copy is current per slot
    // streams / events
    cudaStream_t s_h2d_ = nullptr, s_comp_ = nullptr, s_d2h_ = nullptr, s_upd_ = nullptr;
    std::vector<cudaEvent_t> ev_done_, ev_start_;  // per-op timing (external records)
    std::vector<cudaEvent_t> ev_dep_;              // per-op dependency edges
    // Per-move completion of multi-layer H2D jobs: a layer's compute waits for its own copy,
    // not for the whole job (move_ev_base_[op] indexes ev_move_; -1 = none).
    std::vector<cudaEvent_t> ev_move_;
    std::vector<int> move_ev_base_;
    cudaEvent_t ev_call0_ = nullptr, ev_io_in_ = nullptr, ev_io_out_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev_call1_ = nullptr, ev_loss_ = nullptr;
    std::vector<uint8_t> cross_dep_;  // op has a dependent on another stream
    bool use_graphs_ = true;
    bool item_batching_ = false;  // forward: n_items x rows as one layer-major pass
    bool eager_prefetch_ = true;  // H2D waits for its slot only, not the policy trigger
    bool capturing_ = false;
    // Timing events: plain records when eager; "external" event-record nodes under capture
    // (cudaEventRecordExternal is only valid while capturing).
    void record_timing(cudaEvent_t ev, cudaStream_t st);
    std::unordered_map<uint64_t, GraphEntry> graphs_;
    uint64_t alloc_gen_ = 0;
    uint64_t graph_replays_ = 0;
    // activations / workspaces (device)
    int64_t cap_rows_ = 0;
    int cap_items_ = 0;
    bool cap_train_ = false;
    std::vector<void*> dev_allocs_;
    uint64_t dev_bytes_ = 0;
    float* xin_ = nullptr;   // staging for host-side inputs [items][rows][d] fp32
    float* yout_ = nullptr;  // staging for host-side outputs / training output y (fp32)
    float* tgt_ = nullptr;   // training target staging (fp32)
    void* pp_[2] = {nullptr, nullptr};  // inference ping-pong activations
    void* xconv_ = nullptr;             // bf16 converted input
    std::vector<void*> act_;            // training saved inputs x_0..x_{n-1}
    std::vector<uint32_t*> masks_;      // bf16 training: ReLU bit masks of x_1..x_{n-1} (no ckpt)
    void* gbuf_[2] = {nullptr, nullptr};  // dz ping-pong
    float* gws_[2] = {nullptr, nullptr};  // per-layer gradient workspaces (dW [+db] partials)
    float* grad_red_ = nullptr;           // reduced gradient (DP path)
    float* loss_parts_ = nullptr;
    float* loss_dev_ = nullptr;
    float* loss_host_ = nullptr;  // pinned
    void* fa_[3] = {nullptr, nullptr, nullptr};  // checkpointing: forward activation ring
    std::vector<void*> ba_;                      // checkpointing: backward act per slot
    uint8_t* host_act_ = nullptr;                // checkpointing: pinned activation store
    size_t host_act_bytes_ = 0;
    // current call pointers
    const float* cur_x_ = nullptr;
    float* cur_y_ = nullptr;
    const float* cur_t_ = nullptr;
    float cur_lr_ = 0.0f;
    double host_enqueue_ms_ = 0.0;
    int splits_ = 1, dw_bn_ = 256, dw_cta_ = 2, col_chunks_ = 1, splits_cap_ = 1, col_chunks_cap_ = 1;
    int loss_blocks_ = 0;
    bool dw_fused_ = true;  // bf16 dW: SGD fused into the GEMM epilogue (else split-K partials)
    // optimizer (SGD = the reference's apply_sgd; AdamW with streamed state)
    int optimizer_ = SP_OPT_SGD;
    double beta1_ = 0.9, beta2_ = 0.999, eps_ = 1e-8, wd_ = 0.0;
    int64_t step_t_ = 0;
    float* host_m_ = nullptr;  // pinned [n][d*d + d] fp32, same layout as host32_
    float* host_v_ = nullptr;
    AdamwScalars* adamw_host_ = nullptr;  // pinned: this step's scalars, copied in by the graph
    AdamwScalars* adamw_dev_ = nullptr;
    bool adamw() const { return optimizer_ == SP_OPT_ADAMW; }
    // data parallel
    ncclComm_t comm_ = nullptr;
    int rank_ = 0, world_ = 1;
    bool sharded_ = false;          // each rank streams 1/world of every layer (+ NCCL)
    size_t shardA_ = 0, shardB_ = 0;  // shard bytes of the fp32 / bf16-wire slot images
    // Sharded training writes back only this rank's shard: such a layer's pinned host master
    // is authoritative for that shard alone until dp_sync() all-gathers it.
    std::vector<uint8_t> host_partial_;
    void require_full_host(int layer, const char* what) const;
    // byte range [lo, hi) of this rank's shard within an image of `img` bytes (plan.hpp)
    void shard_range(size_t shard, size_t img, size_t& lo, size_t& hi) const {
        uint64_t l = 0, h = 0;
        sp::shard_range(shard, img, rank_, l, h);
        lo = static_cast<size_t>(l);
        hi = static_cast<size_t>(h);
    }
    // metrics
    sp_stats stats_{};
    std::vector<sp_trace_event> trace_;
    Plan last_plan_;
    uint64_t kernels_ = 0;
    uint64_t h2d_bytes_ = 0, d2h_bytes_ = 0;
    std::vector<cudaEvent_t> gemm_ev_;  // start/end pairs around each tcgen05 GEMM launch
    size_t gemm_count_ = 0;
    double gemm_flops_ = 0.0;
    void reset_call_counters() {
        kernels_ = 0;
        h2d_bytes_ = d2h_bytes_ = 0;
        gemm_count_ = 0;
        gemm_flops_ = 0.0;
        attn_launches_ = 0;
        attn_flops_ = 0.0;
    }
};

}  // namespace sp

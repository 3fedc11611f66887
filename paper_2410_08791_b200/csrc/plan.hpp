// plan.hpp — static Superpipeline op plan (host-only, no CUDA).
//
// The reference drives its policy online from a virtual event loop: policy_step
// (scheduler.cpp:53-141) is re-evaluated after every completion (engine.cpp:172-182) and
// transfers are admitted against a byte ledger (engine.cpp:366-378). Because compute is
// strictly sequential in stream order, the Superpipeline policy is a pure function of
// (n, n_items, k, k', mode, pass structure), so on the GPU it is resolved ONCE into a DAG of
// ops on three CUDA streams (H2D copy engine, compute, D2H copy engine, + an update stream
// for SGD / gradient all-reduce) joined by events. This file builds that DAG, assigns the
// fixed HBM ring slots, and replays the reference's DeviceArena ledger (arena.hpp:38-111)
// along it for peak / OOM accounting.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sp {

enum class Strategy : int { Standard = 0, CpuOnly = 1, Naive = 2, Superpipeline = 3 };
enum class OpKind : int {
    H2D = 0, Compute = 1, D2H = 2, Loss = 3, Update = 4, ActSave = 5,
    AllGather = 6  // sharded streaming: NCCL all-gather completing a slot (update stream)
};

// StrategyConfig::validate (strategy.cpp:19-36). Returns an empty string when valid.
std::string validate_strategy(int strategy, int k, int k_prime, int n_layers);
// peak_weight_residency (strategy.cpp:48-60).
uint64_t peak_weight_residency(int strategy, int k, int k_prime, int n_layers,
                               uint64_t layer_bytes);
// Number of HBM weight slots the ring needs (S = min(k+k', n) for Superpipeline).
int ring_slots(int strategy, int k, int k_prime, int n_layers);

// Sharded streaming: an image of `img` bytes is cut into `world` equal shards of
// shard_bytes(img, world) bytes (256-byte aligned, so world*shard >= img); rank r owns the
// byte range [lo, hi) = [min(img, r*shard), min(img, (r+1)*shard)).
inline uint64_t shard_bytes(uint64_t img, int world) {
    const uint64_t per = (img + static_cast<uint64_t>(world) - 1) / static_cast<uint64_t>(world);
    return (per + 255) / 256 * 256;
}
inline void shard_range(uint64_t shard, uint64_t img, int rank, uint64_t& lo, uint64_t& hi) {
    const uint64_t start = shard * static_cast<uint64_t>(rank);
    lo = start < img ? start : img;
    hi = lo + shard < img ? lo + shard : img;
}

struct PlanInput {
    int n_layers = 1;
    int strategy = 3;
    int k = 0, k_prime = 0;
    int transfer_mode = 1;  // 0 sequential, 1 batch
    bool train = false;
    int n_items = 1;
    bool checkpointing = false;
    bool sharded = false;         // data parallel: H2D 1/world of each layer + all-gather
    // Eager prefetch: an H2D waits only for its slot to be free (and, for activation reloads,
    // for the offload it reads) - not for the compute that triggers it in policy_step
    // (scheduler.cpp:105-136). Same ops, order, slots and ledger; copies start earlier.
    bool eager = false;
    // Optimizer state (AdamW m, v) streams with every trainable layer's backward: its H2D
    // (even when the weights are a slot hit) and its write-back ride the layer's transfers.
    bool optimizer_state = false;
    // Staged write-back: an Update copies the updated image of its slot (HBM -> HBM, a few
    // microseconds) into one of `wb_stages` staging buffers and the write-back D2H reads the
    // stage, so the slot is free for the next H2D as soon as the update is done instead of
    // after the (link-bound) D2H. 0 = write back straight from the slot.
    int wb_stages = 0;
    // Deferred write-back: a trained layer still resident in the ring at the end of the call
    // (final_slots) is written back at the start of the NEXT call, on the otherwise idle D2H
    // engine during the forward, instead of on the critical tail of this backward. Such D2H
    // ops are marked `deferred` and listed in Plan::deferred_*; the next call passes them in
    // pending_wb_* and gets one D2H per layer at its start, which every later writer of that
    // slot depends on. The caller flushes pending write-backs before the host copy is read.
    bool defer_writeback = false;
    // How many write-backs the next forward can absorb (its idle D2H time / one write-back);
    // -1 = n_layers - S (one per layer the forward loads). At most S are ever deferred.
    int defer_budget = -1;
    std::vector<int> pending_wb_layers, pending_wb_slots;
    std::vector<uint8_t> frozen;  // per layer
    uint64_t layer_bytes = 0;     // reference ledger units: (d*d + d) * 4
    uint64_t act_bytes = 0;       // rows * d * 4
    uint64_t capacity = 0;        // 0 = unlimited
};

// Persistent content of one HBM slot across calls (weights valid == equal to host copy).
struct SlotCache {
    int layer = -1;
    bool valid = false;
};

struct Op {
    OpKind kind = OpKind::Compute;
    int pass = 0;       // 0 forward / inference, 1 backward
    int position = -1;  // compute position in the pass sequence
    int item = 0;       // inference item
    int layer = -1;     // Compute / Update / ActSave
    int slot = -1;      // Compute / Update: the weight slot
    std::vector<int> layers;       // H2D / D2H: moved layers (in order)
    std::vector<int> slots;        // H2D / D2H: their slots
    std::vector<uint8_t> weights;  // per moved layer: weight bytes move
    std::vector<uint8_t> acts;     // per moved layer: the saved activation rides along
    std::vector<uint8_t> opts;     // per moved layer: optimizer state (m, v) rides along
    std::vector<int> deps;         // op indices that must complete first (any stream)
    // H2D: the dependencies of each moved layer alone (its slot's last reader, the offload it
    // reloads, a pending write-back); deps = their union + the policy trigger. The executor
    // waits per layer, so one batched job's first copy does not wait for its last slot.
    std::vector<std::vector<int>> move_deps;
    int stage = -1;         // Update: copy the slot to this write-back stage; D2H: read it
    bool deferred = false;  // D2H: skipped in this call, done at the start of the next
    uint64_t led_w = 0, led_a = 0, led_g = 0;  // ledger (weight/act/grad bytes) at this op
};

struct LedgerPeaks {
    uint64_t peak_bytes = 0, peak_weight = 0, peak_activation = 0, peak_gradient = 0;
    uint64_t total_gradient = 0;
};

struct Plan {
    int n_slots = 0;
    std::vector<Op> ops;
    LedgerPeaks ledger;
    std::vector<SlotCache> final_slots;
    std::vector<int> deferred_layers, deferred_slots;  // write-backs left for the next call
    std::vector<int> first_writer;  // per slot: the op that waits for its pending write-back
    uint64_t n_h2d_jobs = 0, n_d2h_jobs = 0, n_evictions = 0;
    uint64_t h2d_weight_layers = 0, h2d_act_layers = 0, d2h_weight_layers = 0,
             d2h_act_layers = 0;
    bool oom = false;
    // The ring cannot keep a pending write-back's slot (see build_plan): flush, plan again.
    bool pending_conflict = false;
    std::string error;  // invalid configuration or OOM reason
};

// Builds the op DAG for one call. `initial` is the slot content left by the previous call
// (empty = cold ring).
Plan build_plan(const PlanInput& in, const std::vector<SlotCache>& initial);

// Human-readable one-op-per-line listing (used by sp_describe_plan and the CPU tests).
std::string describe_plan(const Plan& plan);

}  // namespace sp

// plan.cpp — builds the static Superpipeline op DAG (see plan.hpp).
//
// Policy semantics follow the reference scheduler exactly:
//   * Superpipeline (scheduler.cpp:105-136): prologue loads positions [0, k); every time k'
//     computed positions are awaiting eviction, those k' are evicted and the next k'
//     positions are prefetched (trigger = the compute that completed the group); the final
//     partial group is evicted at stream end.
//   * Naive (scheduler.cpp:85-104): load a group of k, compute it, evict it, next group.
//   * Standard (scheduler.cpp:71-80): everything loaded once and kept across passes.
//   * Training (engine.cpp:84-114,184-194): a forward pass, the loss, then a reversed pass.
// GPU-specific refinements that do not change the math:
//   * an evicted slot keeps its (still valid) weights until it is overwritten, so a later
//     request for the same layer claims it without a copy (this is how the last forward
//     layers are reused by the backward prologue instead of the reference's D2H + H2D
//     round trip, engine.cpp:368-369);
//   * forward evictions of unmodified weights move no bytes; backward evictions of trained
//     layers write the updated fp32 weights back to the pinned host copy;
//   * the prefetch H2D of group g targets the slots released one trigger earlier, so it
//     waits only for their last reader (compute, or the writeback D2H in training).
#include "plan.hpp"

#include <algorithm>
#include <deque>
#include <limits>
#include <sstream>

namespace sp {

std::string validate_strategy(int strategy, int k, int k_prime, int n_layers) {
    if (n_layers < 1) return "strategy: n_layers must be >= 1";
    switch (strategy) {
        case 0:
        case 1:
            return "";
        case 2:
            if (k <= 0 || k > n_layers) return "strategy: naive requires 0 < k <= n_layers";
            return "";
        case 3:
            if (k <= 0 || k > n_layers)
                return "strategy: superpipeline requires 0 < k <= n_layers";
            if (k_prime <= 0 || k_prime >= k) return "strategy: superpipeline requires 0 < k' < k";
            return "";
        default:
            return "strategy: unknown kind";
    }
}

uint64_t peak_weight_residency(int strategy, int k, int k_prime, int n_layers,
                               uint64_t layer_bytes) {
    switch (strategy) {
        case 0: return static_cast<uint64_t>(n_layers) * layer_bytes;
        case 1: return 0;
        case 2: return static_cast<uint64_t>(k) * layer_bytes;
        case 3: return static_cast<uint64_t>(std::min(k + k_prime, n_layers)) * layer_bytes;
        default: return 0;
    }
}

int ring_slots(int strategy, int k, int k_prime, int n_layers) {
    switch (strategy) {
        case 0: return n_layers;
        case 2: return k;
        case 3: return std::min(k + k_prime, n_layers);
        default: return 0;
    }
}

namespace {

constexpr int kInf = std::numeric_limits<int>::max();

struct SlotState {
    int layer = -1;
    bool valid = false;
    int refs = 0;        // claimed positions not yet released
    int fill_op = -1;    // op that last wrote the weights
    int busy_op = -1;    // last op touching the slot's memory (overwrite must wait)
    int wb_op = -1;      // a pending write-back (previous call's layer) the first writer waits for
    uint64_t stamp = 0;  // release order (FIFO tie-break)
};

enum Tag { kWeight = 0, kActivation = 1, kGradient = 2 };

class Builder {
public:
    Builder(const PlanInput& in, const std::vector<SlotCache>& initial, int n_slots)
        : in_(in), n_(in.n_layers) {
        // Standard never evicts, so its activations are never offloaded (the reference's
        // checkpointing rides eviction D2H / prefetch H2D jobs, engine.cpp:247-252).
        ckpt_ = in.train && in.checkpointing &&
                in.strategy != static_cast<int>(Strategy::Standard);
        plan_.n_slots = n_slots;
        plan_.first_writer.assign(static_cast<std::size_t>(n_slots), std::numeric_limits<int>::max());
        slots_.resize(static_cast<std::size_t>(n_slots));
        for (int s = 0; s < n_slots && s < static_cast<int>(initial.size()); ++s) {
            slots_[s].layer = initial[s].layer;
            slots_[s].valid = initial[s].valid && initial[s].layer >= 0 &&
                              initial[s].layer < n_;
        }
        ba_busy_.assign(static_cast<std::size_t>(n_slots), -1);
        stage_busy_.assign(static_cast<std::size_t>(std::max(in.wb_stages, 0)), -1);
        act_save_op_.assign(static_cast<std::size_t>(n_), -1);
        if (in_.train) {
            std::vector<int> fwd(n_), bwd(n_);
            for (int i = 0; i < n_; ++i) fwd[i] = i, bwd[i] = n_ - 1 - i;
            seqs_ = {fwd, bwd};
        } else {
            std::vector<int> seq(static_cast<std::size_t>(n_) * in_.n_items);
            for (std::size_t p = 0; p < seq.size(); ++p) seq[p] = static_cast<int>(p) % n_;
            seqs_ = {seq};
        }
    }

    Plan run() {
        // The previous call's deferred write-backs: first on the D2H engine, reading slots
        // that still hold those layers (only the writers of those slots wait for them), in the
        // order given - build_plan passes them sorted by when each slot is first overwritten.
        for (std::size_t i = 0; i < in_.pending_wb_layers.size(); ++i) {
            const int L = in_.pending_wb_layers[i], s = in_.pending_wb_slots[i];
            if (s < 0 || s >= static_cast<int>(slots_.size())) {
                // build_plan never shrinks the ring below a pending slot (the executor
                // flushes first), so this is an internal invariant, never a silent skip.
                plan_.error = "internal: pending write-back of layer " + std::to_string(L) +
                              " targets slot " + std::to_string(s) + " outside a " +
                              std::to_string(slots_.size()) + "-slot ring";
                plan_.pending_conflict = true;
                return plan_;
            }
            Op wb;
            wb.kind = OpKind::D2H;
            wb.pass = 0;
            wb.layers = {L};
            wb.slots = {s};
            wb.weights = {1};
            wb.acts = {0};
            slots_[s].wb_op = push(std::move(wb));  // counted in the call that deferred it
        }
        if (!in_.train) {
            // The reference holds one io activation buffer for inference (engine.cpp:60-64).
            if (in_.capacity && in_.act_bytes > in_.capacity) {
                plan_.oom = true;
                plan_.error = "activation buffer alone exceeds device capacity";
                return plan_;
            }
            ledger_add(kActivation, in_.act_bytes);
        }
        for (pass_ = 0; pass_ < static_cast<int>(seqs_.size()); ++pass_) {
            run_pass();
            if (in_.train && pass_ == 0) {
                Op loss;
                loss.kind = OpKind::Loss;
                loss.pass = 0;
                loss_op_ = push(std::move(loss));
            }
        }
        flush_deferred();
        for (auto& s : slots_) {  // end of call: every claim is dropped (release_remaining)
            if (s.refs > 0) ledger_sub(kWeight, in_.layer_bytes);
            s.refs = 0;
        }
        plan_.final_slots.resize(slots_.size());
        for (std::size_t s = 0; s < slots_.size(); ++s)
            plan_.final_slots[s] = SlotCache{slots_[s].layer, slots_[s].valid};
        if (in_.defer_writeback) defer_final_writebacks();
        return plan_;
    }

    // Write-backs of layers that end the call resident (and valid) in their slot move to the
    // next call; their Update skips the staging copy. Only as many as the next forward's idle
    // D2H time absorbs (in_.defer_budget, estimated by the executor from the layer's compute and
    // copy times) are deferred - the lowest layers, whose slots the next forward recycles first
    // and which the next backward rewrites last; the rest stay in this backward.
    void defer_final_writebacks() {
        std::vector<std::pair<int, std::size_t>> cand;  // (layer, D2H op)
        for (std::size_t i = 0; i < plan_.ops.size(); ++i) {
            const Op& op = plan_.ops[i];
            if (op.kind != OpKind::D2H || op.pass != 1) continue;
            const int L = op.layers[0], s = op.slots[0];
            if (plan_.final_slots[static_cast<std::size_t>(s)].valid &&
                plan_.final_slots[static_cast<std::size_t>(s)].layer == L)
                cand.emplace_back(L, i);
        }
        std::sort(cand.begin(), cand.end());
        const int b = in_.defer_budget >= 0 ? in_.defer_budget : n_ - plan_.n_slots;
        const std::size_t budget = static_cast<std::size_t>(std::max(0, std::min(b, plan_.n_slots)));
        if (cand.size() > budget) cand.resize(budget);
        std::vector<uint8_t> deferred(plan_.ops.size(), 0);
        for (const auto& c : cand) {
            Op& op = plan_.ops[c.second];
            const int L = op.layers[0], s = op.slots[0];
            op.deferred = true;
            deferred[c.second] = 1;
            for (int dep : op.deps)
                if (plan_.ops[static_cast<std::size_t>(dep)].kind == OpKind::Update)
                    plan_.ops[static_cast<std::size_t>(dep)].stage = -1;
            op.stage = -1;
            plan_.deferred_layers.push_back(L);
            plan_.deferred_slots.push_back(s);
        }
        // A deferred write-back reads no stage, and its (empty) op sits behind the next call's
        // D2H queue: later updates reusing that stage need not wait for it (they are ordered
        // after this layer's update, which waited for the stage's previous reader).
        for (Op& op : plan_.ops)
            if (op.kind == OpKind::Update)
                op.deps.erase(std::remove_if(op.deps.begin(), op.deps.end(),
                                             [&](int d) { return deferred[static_cast<std::size_t>(d)] != 0; }),
                              op.deps.end());
    }

    // The first op that overwrites slot s after a pending write-back of its old content waits
    // for it; every later writer is ordered after that one through the slot's own chain.
    void wait_writeback(std::vector<int>& deps, int s) {
        if (slots_[s].wb_op < 0) return;
        deps.push_back(slots_[s].wb_op);
        slots_[s].wb_op = -1;
        plan_.first_writer[static_cast<std::size_t>(s)] = static_cast<int>(plan_.ops.size());  // op about to be pushed
    }

private:
    const std::vector<int>& seq() const { return seqs_[static_cast<std::size_t>(pass_)]; }
    int len() const { return static_cast<int>(seq().size()); }
    bool backward() const { return in_.train && pass_ == 1; }
    bool trainable(int layer) const {
        return !(layer < static_cast<int>(in_.frozen.size()) && in_.frozen[layer]);
    }

    int push(Op op) {
        // ledger snapshot at this point of the plan (TraceEvent::footprint_after, trace.hpp:44-46)
        op.led_w = tag_[kWeight];
        op.led_a = tag_[kActivation];
        op.led_g = tag_[kGradient];
        plan_.ops.push_back(std::move(op));
        return static_cast<int>(plan_.ops.size()) - 1;
    }

    // ---- ledger (DeviceArena semantics, arena.hpp:45-67) -----------------------------
    void ledger_add(int tag, uint64_t bytes) {
        tag_[tag] += bytes;
        auto& pk = tag == kWeight ? plan_.ledger.peak_weight
                   : tag == kActivation ? plan_.ledger.peak_activation
                                        : plan_.ledger.peak_gradient;
        pk = std::max(pk, tag_[tag]);
        const uint64_t total = tag_[0] + tag_[1] + tag_[2];
        plan_.ledger.peak_bytes = std::max(plan_.ledger.peak_bytes, total);
        if (in_.capacity && total > in_.capacity && !plan_.oom) {
            plan_.oom = true;
            plan_.error = "no runnable event: required working set cannot fit in " +
                          std::to_string(in_.capacity) + " bytes";
        }
    }
    void ledger_sub(int tag, uint64_t bytes) { tag_[tag] -= std::min(tag_[tag], bytes); }
    // Evictions free their bytes when the D2H completes in the reference
    // (engine.cpp:390-405), i.e. while the next compute is already running.
    void defer_free(int tag, uint64_t bytes, int slot = -1) { deferred_.push_back({tag, bytes, slot}); }
    void flush_deferred() {
        for (const auto& f : deferred_) ledger_sub(f.tag, f.bytes);
        deferred_.clear();
    }
    // A claim of a released slot whose eviction has not drained yet: in the reference the layer
    // has a single placement, so it is never counted twice — the pending free is cancelled and
    // the layer stays counted once (instead of being added again).
    bool cancel_pending_free(int slot) {
        for (auto it = deferred_.begin(); it != deferred_.end(); ++it)
            if (it->tag == kWeight && it->slot == slot) {
                deferred_.erase(it);
                return true;
            }
        return false;
    }

    // ---- slot choice -------------------------------------------------------------------
    int next_use(int layer, int after_pos) const {
        int base = 0;
        for (int ps = 0; ps < static_cast<int>(seqs_.size()); ++ps) {
            const auto& s = seqs_[ps];
            const int start = ps < pass_ ? static_cast<int>(s.size()) : ps == pass_ ? after_pos + 1 : 0;
            for (int q = start; q < static_cast<int>(s.size()); ++q)
                if (s[q] == layer) return base + q;
            base += static_cast<int>(s.size());
        }
        return kInf;
    }
    int active_slot(int layer) const {
        for (int s = 0; s < static_cast<int>(slots_.size()); ++s)
            if (slots_[s].refs > 0 && slots_[s].layer == layer) return s;
        return -1;
    }
    int cached_free_slot(int layer) const {
        for (int s = 0; s < static_cast<int>(slots_.size()); ++s)
            if (slots_[s].refs == 0 && slots_[s].valid && slots_[s].layer == layer) return s;
        return -1;
    }
    // Belady among free slots: evict the cached layer whose next use is farthest away;
    // ties go to the earliest-released slot, then the lowest index.
    int victim_slot(int pos) const {
        int best = -1, best_use = -1;
        uint64_t best_stamp = 0;
        for (int s = 0; s < static_cast<int>(slots_.size()); ++s) {
            if (slots_[s].refs != 0) continue;
            const int use = slots_[s].valid ? next_use(slots_[s].layer, pos) : kInf;
            if (best < 0 || use > best_use || (use == best_use && slots_[s].stamp < best_stamp)) {
                best = s;
                best_use = use;
                best_stamp = slots_[s].stamp;
            }
        }
        return best;
    }
    int free_slots() const {
        int c = 0;
        for (const auto& s : slots_) c += s.refs == 0;
        return c;
    }
    int misses_in(int b, int e) const {
        int m = 0;
        std::vector<int> seen;
        for (int q = b; q < e; ++q) {
            const int L = seq()[q];
            if (std::find(seen.begin(), seen.end(), L) != seen.end()) continue;
            seen.push_back(L);
            if (active_slot(L) < 0) ++m;  // cached free slots are consumed as well
        }
        return m;
    }

    // ---- policy actions ----------------------------------------------------------------
    void claim_positions(int b, int e, int trigger) {
        struct Move { int pos, slot; bool weights, act, opt; };
        std::vector<Move> moves;
        for (int q = b; q < e; ++q) {
            const int L = seq()[q];
            // AdamW moments travel with each trainable layer's backward claim, hit or miss
            const bool opt = backward() && in_.optimizer_state && trainable(L);
            int s = active_slot(L);
            if (s >= 0) {
                slots_[s].refs += 1;
                pos_slot_[q] = s;
                pos_load_[q] = slots_[s].fill_op;
                if (opt) moves.push_back({q, s, false, false, true});  // Standard: still resident
                continue;
            }
            bool miss = false;
            s = cached_free_slot(L);
            if (s < 0) {
                s = victim_slot(q);
                if (s < 0) {
                    plan_.error = "plan: no free ring slot (internal)";
                    plan_.oom = true;
                    return;
                }
                miss = true;
                slots_[s].layer = L;
                slots_[s].valid = true;
            }
            slots_[s].refs = 1;
            pos_slot_[q] = s;
            pos_load_[q] = slots_[s].fill_op;
            if (miss || !cancel_pending_free(s)) ledger_add(kWeight, in_.layer_bytes);
            const bool act = backward() && ckpt_;
            if (act) ledger_add(kActivation, in_.act_bytes);
            if (miss || act || opt) moves.push_back({q, s, miss, act, opt});
        }
        if (moves.empty()) return;
        auto emit = [&](const std::vector<Move>& group) {
            Op op;
            op.kind = OpKind::H2D;
            op.pass = pass_;
            if (trigger >= 0 && !in_.eager) op.deps.push_back(trigger);
            for (const auto& m : group) {
                op.layers.push_back(seq()[m.pos]);
                op.slots.push_back(m.slot);
                op.weights.push_back(m.weights);
                op.acts.push_back(m.act);
                op.opts.push_back(m.opt);
                std::vector<int> md;
                // weights or optimizer state overwrite the slot: after its last reader
                if ((m.weights || m.opt) && slots_[m.slot].busy_op >= 0) md.push_back(slots_[m.slot].busy_op);
                if (m.act && ba_busy_[m.slot] >= 0) md.push_back(ba_busy_[m.slot]);
                // The reload reads the pinned copy written by this layer's forward offload
                // (the reference only reloads once act_on_host_ is set, engine.cpp:397-402).
                const int saved = act_save_op_[static_cast<size_t>(seq()[m.pos])];
                if (m.act && saved >= 0) md.push_back(saved);
                if (m.weights || m.opt) wait_writeback(md, m.slot);
                op.deps.insert(op.deps.end(), md.begin(), md.end());
                op.move_deps.push_back(std::move(md));
                plan_.h2d_weight_layers += m.weights;
                plan_.h2d_act_layers += m.act;
            }
            const int id = push(std::move(op));
            // Sharded streaming (data parallel): the H2D brought only this rank's 1/world of
            // each layer; an NCCL all-gather over NVLink completes the slot before any use.
            int fill = id;
            if (in_.sharded) {
                Op ag;
                ag.kind = OpKind::AllGather;
                ag.pass = pass_;
                ag.deps.push_back(id);
                for (const auto& m : group)
                    if (m.weights) {
                        ag.layers.push_back(seq()[m.pos]);
                        ag.slots.push_back(m.slot);
                        ag.weights.push_back(1);
                        ag.acts.push_back(0);
                    }
                if (!ag.layers.empty()) fill = push(std::move(ag));
            }
            for (const auto& m : group) {
                if (m.weights) {
                    slots_[m.slot].fill_op = fill;
                    slots_[m.slot].busy_op = fill;
                }
                pos_load_[m.pos] = m.weights ? fill : id;
                if (m.act) pos_act_[m.pos] = id;
            }
            plan_.n_h2d_jobs += 1;
        };
        if (in_.transfer_mode == 0) {
            for (const auto& m : moves) emit({m});
        } else {
            emit(moves);
        }
    }

    void release_positions(const std::vector<int>& positions) {
        for (int q : positions) {
            const int s = pos_slot_[q];
            plan_.n_evictions += 1;
            if (--slots_[s].refs == 0) {
                slots_[s].stamp = ++stamp_;
                defer_free(kWeight, in_.layer_bytes, s);
                if (!backward() && in_.train && ckpt_)
                    defer_free(kActivation, in_.act_bytes);  // offloaded with the layer
            }
        }
    }

    int emit_compute(int p) {
        const int L = seq()[p];
        const int s = pos_slot_[p];
        Op op;
        op.kind = OpKind::Compute;
        op.pass = pass_;
        op.position = p;
        op.item = in_.train ? 0 : p / n_;
        op.layer = L;
        op.slot = s;
        if (pos_load_[p] >= 0) op.deps.push_back(pos_load_[p]);
        if (backward() && ckpt_ && pos_act_[p] >= 0) op.deps.push_back(pos_act_[p]);
        if (!backward() && in_.train && ckpt_) {
            const int buf = (L + 1) % 3;  // forward act ring: x_{L+1} overwrites x_{L-2}
            if (fa_busy_[buf] >= 0) op.deps.push_back(fa_busy_[buf]);
        }
        if (backward() && trainable(L) && gws_busy_[L % 2] >= 0)
            op.deps.push_back(gws_busy_[L % 2]);  // dW workspace double buffer
        if (backward() && trainable(L)) wait_writeback(op.deps, s);  // may update W in its epilogue
        // Ledger at compute begin (engine.cpp:271-282).
        if (in_.train && !backward()) ledger_add(kActivation, in_.act_bytes);
        const bool grad = backward() && trainable(L);
        if (grad) {
            ledger_add(kGradient, in_.layer_bytes);
            plan_.ledger.total_gradient += in_.layer_bytes;
        }
        flush_deferred();
        const int id = push(std::move(op));
        slots_[s].busy_op = id;
        if (grad) ledger_sub(kGradient, in_.layer_bytes);  // freed at compute end
        if (backward() && ckpt_) {
            ba_busy_[s] = id;
            ledger_sub(kActivation, in_.act_bytes);  // engine.cpp:438-441
        }
        if (!backward() && in_.train && ckpt_) {
            Op save;  // offload x_L to the pinned host activation store
            save.kind = OpKind::ActSave;
            save.pass = 0;
            save.layer = L;
            save.deps.push_back(id);
            fa_busy_[L % 3] = push(std::move(save));
            act_save_op_[static_cast<size_t>(L)] = fa_busy_[L % 3];
            plan_.d2h_act_layers += 1;
        }
        if (grad) {
            Op upd;  // gradient all-reduce (DP) + SGD on the update stream
            upd.kind = OpKind::Update;
            upd.pass = 1;
            upd.layer = L;
            upd.slot = s;
            upd.deps.push_back(id);
            wait_writeback(upd.deps, s);
            if (!stage_busy_.empty()) {  // staged: the update also copies the slot to a stage
                upd.stage = static_cast<int>(n_staged_++ % stage_busy_.size());
                if (stage_busy_[upd.stage] >= 0) upd.deps.push_back(stage_busy_[upd.stage]);
            }
            const int stage = upd.stage;
            const int uid = push(std::move(upd));
            gws_busy_[L % 2] = uid;
            Op wb;  // write the updated fp32 weights back to the host master copy
            wb.kind = OpKind::D2H;
            wb.pass = 1;
            wb.layers = {L};
            wb.slots = {s};
            wb.weights = {1};
            wb.acts = {0};
            wb.stage = stage;
            wb.deps.push_back(uid);
            const int wid = push(std::move(wb));
            // staged: the slot is free once the update (and its copy) is done
            slots_[s].busy_op = stage >= 0 ? uid : wid;
            if (stage >= 0) stage_busy_[stage] = wid;
            plan_.n_d2h_jobs += 1;
            plan_.d2h_weight_layers += 1;
            // Sharded: only this rank's shard of the slot was updated (and written back), so
            // the slot no longer holds a valid full copy of the layer.
            if (in_.sharded) slots_[s].valid = false;
        }
        return id;
    }

    void run_pass() {
        const int n = len();
        pos_slot_.assign(static_cast<std::size_t>(n), -1);
        pos_load_.assign(static_cast<std::size_t>(n), -1);
        pos_act_.assign(static_cast<std::size_t>(n), -1);
        const int trigger0 = pass_ == 0 ? -1 : loss_op_;
        const auto kind = static_cast<Strategy>(in_.strategy);
        if (kind == Strategy::Standard) {
            claim_positions(0, n, trigger0);
            for (int p = 0; p < n && !plan_.oom; ++p) emit_compute(p);
            return;
        }
        if (kind == Strategy::Naive) {
            int trigger = trigger0;
            for (int gb = 0; gb < n && !plan_.oom; gb += in_.k) {
                const int ge = std::min(gb + in_.k, n);
                claim_positions(gb, ge, trigger);
                std::vector<int> group;
                for (int p = gb; p < ge && !plan_.oom; ++p) {
                    trigger = emit_compute(p);
                    group.push_back(p);
                }
                release_positions(group);
                flush_deferred();  // the next group is admitted only once this one drained
            }
            return;
        }
        // Superpipeline.
        const int k = in_.k, kp = in_.k_prime;
        claim_positions(0, std::min(k, n), trigger0);
        int next_load = std::min(k, n);
        std::deque<int> ready;
        for (int p = 0; p < n && !plan_.oom; ++p) {
            const int c = emit_compute(p);
            ready.push_back(p);
            if (static_cast<int>(ready.size()) >= kp) {
                std::vector<int> evict(ready.begin(), ready.begin() + kp);
                ready.erase(ready.begin(), ready.begin() + kp);
                const int nb = next_load, ne = std::min(next_load + kp, n);
                if (nb < ne && misses_in(nb, ne) <= free_slots()) {
                    claim_positions(nb, ne, c);  // prefetch into slots freed one group earlier
                    release_positions(evict);
                } else {  // capacity-bound: the prefetch waits for the eviction to drain
                    release_positions(evict);
                    flush_deferred();
                    if (nb < ne) claim_positions(nb, ne, c);
                }
                next_load = ne;
            }
        }
        release_positions(std::vector<int>(ready.begin(), ready.end()));
    }

    const PlanInput& in_;
    int n_;
    Plan plan_;
    std::vector<SlotState> slots_;
    std::vector<std::vector<int>> seqs_;
    std::vector<int> pos_slot_, pos_load_, pos_act_;
    std::vector<int> ba_busy_;
    std::vector<int> stage_busy_;  // per write-back stage: the D2H that last read it
    uint64_t n_staged_ = 0;
    std::vector<int> act_save_op_;  // per layer: the forward ActSave op (offload to host)
    int fa_busy_[3] = {-1, -1, -1};
    int gws_busy_[2] = {-1, -1};
    int pass_ = 0;
    int loss_op_ = -1;
    bool ckpt_ = false;
    uint64_t stamp_ = 0;
    uint64_t tag_[3] = {0, 0, 0};
    struct PendingFree {
        int tag;
        uint64_t bytes;
        int slot;  // weight frees: the released slot
    };
    std::vector<PendingFree> deferred_;
};

}  // namespace

Plan build_plan(const PlanInput& in, const std::vector<SlotCache>& initial) {
    Plan bad;
    bad.error = validate_strategy(in.strategy, in.k, in.k_prime, in.n_layers);
    if (!bad.error.empty()) return bad;
    if (in.strategy == static_cast<int>(Strategy::CpuOnly)) {
        bad.error = "strategy: cpu_only is the reference's host path; the GPU executor has no "
                    "CPU fallback";
        return bad;
    }
    if (in.n_items < 1) {
        bad.error = "execution_stream: counts must be >= 1";
        return bad;
    }
    // The reference admits a prefetch only when it fits (engine.cpp:366-378), so a tight
    // capacity shrinks the effective ring instead of failing; below the minimum working
    // set (k slots, or n for Standard) it deadlocks -> OOM.
    int S = ring_slots(in.strategy, in.k, in.k_prime, in.n_layers);
    const int smin = in.strategy == static_cast<int>(Strategy::Standard) ? in.n_layers : in.k;
    // The previous call's deferred write-backs read their slots at this call's start: a ring
    // shrunk below one of them (a capacity cap with a larger batch) would lose that update.
    // Such a plan is refused with pending_conflict; the caller flushes and plans again.
    int wb_min = 0;
    for (int s : in.pending_wb_slots) wb_min = std::max(wb_min, s + 1);
    for (;;) {
        if (S < wb_min) {
            Plan c;
            c.pending_conflict = true;
            c.error = "internal: the ring would shrink below a pending write-back slot";
            return c;
        }
        Builder b(in, initial, S);
        Plan p = b.run();
        if (!p.oom && in.pending_wb_layers.size() > 1) {
            // Issue the previous call's write-backs in the order their slots are first
            // overwritten: ascending layers for slots the forward recycles, backward order for
            // layers that stay resident (Standard, or a ring wider than the model), so no
            // writer queues behind write-backs it does not need.
            std::vector<std::size_t> idx(in.pending_wb_layers.size());
            for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
            auto when = [&](std::size_t i) {
                const int s = in.pending_wb_slots[i];
                return s >= 0 && s < static_cast<int>(p.first_writer.size()) ? p.first_writer[static_cast<std::size_t>(s)]
                                                                            : std::numeric_limits<int>::max();
            };
            std::stable_sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b2) {
                return when(a) != when(b2) ? when(a) < when(b2) : in.pending_wb_layers[a] < in.pending_wb_layers[b2];
            });
            PlanInput sorted = in;
            for (std::size_t i = 0; i < idx.size(); ++i) {
                sorted.pending_wb_layers[i] = in.pending_wb_layers[idx[i]];
                sorted.pending_wb_slots[i] = in.pending_wb_slots[idx[i]];
            }
            Builder b2(sorted, initial, S);
            return b2.run();
        }
        if (!p.oom || S <= smin) return p;
        --S;
    }
}

std::string describe_plan(const Plan& plan) {
    static const char* names[] = {"H2D", "COMPUTE", "D2H", "LOSS", "UPDATE", "ACTSAVE", "ALLGATHER"};
    std::ostringstream os;
    os << "slots=" << plan.n_slots << " ops=" << plan.ops.size()
       << " h2d_jobs=" << plan.n_h2d_jobs << " d2h_jobs=" << plan.n_d2h_jobs
       << " evictions=" << plan.n_evictions << " peak=" << plan.ledger.peak_bytes
       << " peak_w=" << plan.ledger.peak_weight << " peak_a=" << plan.ledger.peak_activation
       << " peak_g=" << plan.ledger.peak_gradient << " total_g=" << plan.ledger.total_gradient
       << (plan.oom ? " OOM" : "") << "\n";
    auto list = [&](const std::vector<int>& v) {
        std::ostringstream s;
        for (std::size_t i = 0; i < v.size(); ++i) s << (i ? "," : "") << v[i];
        return s.str();
    };
    for (std::size_t i = 0; i < plan.ops.size(); ++i) {
        const Op& op = plan.ops[i];
        os << i << " " << names[static_cast<int>(op.kind)] << " pass=" << op.pass;
        if (op.kind == OpKind::Compute)
            os << " pos=" << op.position << " item=" << op.item << " layer=" << op.layer
               << " slot=" << op.slot;
        if (op.kind == OpKind::Update) {
            os << " layer=" << op.layer << " slot=" << op.slot;
            if (op.stage >= 0) os << " stage=" << op.stage;
        }
        if (op.kind == OpKind::ActSave) os << " layer=" << op.layer;
        if (op.kind == OpKind::H2D || op.kind == OpKind::D2H || op.kind == OpKind::AllGather) {
            std::vector<int> w(op.weights.begin(), op.weights.end()),
                a(op.acts.begin(), op.acts.end()), o(op.opts.begin(), op.opts.end());
            os << " layers=" << list(op.layers) << " slots=" << list(op.slots)
               << " w=" << list(w) << " a=" << list(a);
            if (!o.empty()) os << " o=" << list(o);
            if (op.kind == OpKind::D2H && op.stage >= 0) os << " stage=" << op.stage;
            if (op.deferred) os << " deferred=1";
            if (op.kind == OpKind::H2D) {  // per-move dependencies: md=a.b|c|...
                os << " md=";
                for (std::size_t j = 0; j < op.move_deps.size(); ++j) {
                    if (j) os << "|";
                    for (std::size_t t = 0; t < op.move_deps[j].size(); ++t)
                        os << (t ? "." : "") << op.move_deps[j][t];
                }
            }
        }
        os << " deps=" << list(op.deps) << " led=" << op.led_w << "," << op.led_a << ","
           << op.led_g << "\n";
    }
    return os.str();
}

}  // namespace sp

// capi.cpp — extern "C" boundary (include/superpipe.h) over the ring executor.
// Exceptions never cross the ABI: every entry point maps them onto sp_status codes that
// mirror the reference's exception taxonomy (invalid_argument -> 2, OomDeadlockError -> 3,
// logic_error -> 1).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <new>
#include <string>

#include "executor.hpp"
#include "nccl_dyn.hpp"
#include "plan.hpp"

struct sp_exec {
    sp::Executor* impl = nullptr;
    std::string error;
};

namespace {

template <typename F>
int guarded(sp_exec* ex, F&& f) {
    try {
        f();
        if (ex) ex->error.clear();
        return SP_OK;
    } catch (const sp::Error& e) {
        if (ex) ex->error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        if (ex) ex->error = "host allocation failed";
        return SP_ERR_OOM;
    } catch (const std::exception& e) {
        if (ex) ex->error = e.what();
        return SP_ERR_INTERNAL;
    }
}

thread_local std::string g_create_error;

}  // namespace

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }

int sp_create(const sp_config* cfg, sp_exec** out) {
    if (!cfg || !out) return SP_ERR_INVALID;
    *out = nullptr;
    auto* ex = new (std::nothrow) sp_exec;
    if (!ex) return SP_ERR_OOM;
    const int rc = guarded(ex, [&] { ex->impl = new sp::Executor(*cfg); });
    if (rc != SP_OK) {
        g_create_error = ex->error;
        delete ex;
        return rc;
    }
    *out = ex;
    return SP_OK;
}

int sp_create_blocks(const sp_config* cfg, const sp_block_desc* blk, sp_exec** out) {
    if (!cfg || !blk || !out) return SP_ERR_INVALID;
    *out = nullptr;
    auto* ex = new (std::nothrow) sp_exec;
    if (!ex) return SP_ERR_OOM;
    const int rc = guarded(ex, [&] { ex->impl = new sp::Executor(*cfg, blk); });
    if (rc != SP_OK) {
        g_create_error = ex->error;
        delete ex;
        return rc;
    }
    *out = ex;
    return SP_OK;
}

int sp_register_block(sp_exec* ex, int32_t index, const float* params, int32_t frozen) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->register_block(index, params, frozen); });
}

int sp_read_block(sp_exec* ex, int32_t index, float* params) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->read_block(index, params); });
}

int sp_register_layer(sp_exec* ex, int32_t index, const float* W, const float* b,
                      int32_t activation, int32_t frozen) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->register_layer(index, W, b, activation, frozen); });
}

int sp_destroy(sp_exec* ex) {
    if (!ex) return SP_OK;
    delete ex->impl;
    delete ex;
    return SP_OK;
}

const char* sp_last_error(const sp_exec* ex) {
    return ex ? ex->error.c_str() : g_create_error.c_str();
}

int sp_forward(sp_exec* ex, const float* x, int64_t rows, int32_t n_items, float* y) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->forward(x, rows, n_items, y, false); });
}

int sp_forward_device(sp_exec* ex, const void* x_dev, int64_t rows, int32_t n_items,
                      void* y_dev) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] {
        ex->impl->forward(static_cast<const float*>(x_dev), rows, n_items,
                          static_cast<float*>(y_dev), true);
    });
}

int sp_train_step(sp_exec* ex, const float* x, const float* target, int64_t rows, float lr,
                  float* loss) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] {
        const float l = ex->impl->train_step(x, target, rows, lr, false);
        if (loss) *loss = l;
    });
}

int sp_train_step_device(sp_exec* ex, const void* x_dev, const void* target_dev, int64_t rows,
                         float lr, float* loss) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] {
        const float l = ex->impl->train_step(static_cast<const float*>(x_dev),
                                             static_cast<const float*>(target_dev), rows, lr, true);
        if (loss) *loss = l;
    });
}

int sp_read_layer(sp_exec* ex, int32_t index, float* W, float* b) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->read_layer(index, W, b); });
}

int64_t sp_last_plan(const sp_exec* ex, char* buf, int64_t cap) {
    if (!ex) return -1;
    const std::string text = ex->impl->last_plan_text();
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(text.size()));
        std::memcpy(buf, text.data(), static_cast<size_t>(n));
        buf[n] = '\0';
    }
    return static_cast<int64_t>(text.size()) + 1;
}

int sp_get_op_info(const sp_exec* ex, int32_t op_index, uint64_t ledger[3], int32_t* layers, int32_t cap,
                   int32_t* count) {
    if (!ex) return SP_ERR_INVALID;
    const sp::Plan& plan = ex->impl->last_plan();
    if (op_index < 0 || op_index >= static_cast<int32_t>(plan.ops.size())) return SP_ERR_INVALID;
    const sp::Op& op = plan.ops[static_cast<size_t>(op_index)];
    if (ledger) {
        ledger[0] = op.led_w;
        ledger[1] = op.led_a;
        ledger[2] = op.led_g;
    }
    const int32_t n = static_cast<int32_t>(op.layers.size());
    if (count) *count = n;
    for (int32_t i = 0; layers && i < n && i < cap; ++i) layers[i] = op.layers[static_cast<size_t>(i)];
    return SP_OK;
}

int sp_set_trace(sp_exec* ex, int32_t level) {
    if (!ex || level < 0 || level > 2) return SP_ERR_INVALID;
    ex->impl->set_trace(level);
    return SP_OK;
}

int sp_set_eager_prefetch(sp_exec* ex, int32_t on) {
    if (!ex || on < 0 || on > 1) return SP_ERR_INVALID;
    ex->impl->set_eager_prefetch(on != 0);
    return SP_OK;
}

int sp_set_item_batching(sp_exec* ex, int32_t on) {
    if (!ex || on < 0 || on > 1) return SP_ERR_INVALID;
    ex->impl->set_item_batching(on != 0);
    return SP_OK;
}

int sp_share_host_master(sp_exec* ex, const char* name, int32_t create) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->share_host_master(name, create != 0); });
}

int sp_set_optimizer(sp_exec* ex, int32_t kind, float beta1, float beta2, float eps, float weight_decay) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->set_optimizer(kind, beta1, beta2, eps, weight_decay); });
}

int sp_read_optimizer_state(sp_exec* ex, int32_t index, float* mW, float* mb, float* vW, float* vb) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->read_optimizer_state(index, mW, mb, vW, vb); });
}

int sp_digest_train(const sp_exec* ex, float loss, char out[17]) {
    if (!ex || !out) return SP_ERR_INVALID;
    // digest_train flushes pending write-backs and refuses a shard-only master: both throw,
    // and exceptions never cross the ABI
    sp_exec* mex = const_cast<sp_exec*>(ex);
    return guarded(mex, [&] { mex->impl->digest_train(loss, out); });
}

int sp_get_stats(const sp_exec* ex, sp_stats* out) {
    if (!ex || !out) return SP_ERR_INVALID;
    *out = ex->impl->stats();
    return SP_OK;
}

int sp_get_trace(const sp_exec* ex, sp_trace_event* events, int32_t cap, int32_t* count) {
    if (!ex || !count) return SP_ERR_INVALID;
    const auto& tr = ex->impl->trace();
    *count = static_cast<int32_t>(tr.size());
    if (events)
        for (int32_t i = 0; i < cap && i < static_cast<int32_t>(tr.size()); ++i) events[i] = tr[i];
    return SP_OK;
}

int sp_nccl_unique_id(uint8_t id[128]) {
    if (!id) return SP_ERR_INVALID;
    ncclUniqueId uid;
    if (!sp::nccl().ok() || sp::nccl().GetUniqueId(&uid) != ncclSuccess) return SP_ERR_NCCL;
    std::memcpy(id, uid.internal, sizeof(uid.internal));
    return SP_OK;
}

int sp_dp_init(sp_exec* ex, const uint8_t id[128], int32_t rank, int32_t world) {
    return sp_dp_init2(ex, id, rank, world, world > 1 ? 1 : 0);
}

int sp_dp_init2(sp_exec* ex, const uint8_t id[128], int32_t rank, int32_t world,
                int32_t shard_weights) {
    if (!ex || !id) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->dp_init(id, rank, world, shard_weights != 0); });
}

int sp_dp_sync(sp_exec* ex) {
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->dp_sync(); });
}

void* sp_host_alloc(uint64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    return p;
}

void sp_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

uint64_t sp_peak_weight_residency(int32_t strategy, int32_t k, int32_t k_prime,
                                  int32_t n_layers, uint64_t layer_bytes) {
    if (!sp::validate_strategy(strategy, k, k_prime, n_layers).empty()) return 0;
    return sp::peak_weight_residency(strategy, k, k_prime, n_layers, layer_bytes);
}

int sp_validate_strategy(int32_t strategy, int32_t k, int32_t k_prime, int32_t n_layers) {
    return sp::validate_strategy(strategy, k, k_prime, n_layers).empty() ? SP_OK : SP_ERR_INVALID;
}

int64_t sp_describe_plan(const sp_config* cfg, int32_t n_items, int32_t train,
                         const int32_t* frozen, int32_t flags, char* buf, int64_t cap) {
    if (!cfg) return -1;
    sp::PlanInput in;
    in.n_layers = cfg->n_layers;
    in.strategy = cfg->strategy;
    in.k = cfg->k;
    in.k_prime = cfg->k_prime;
    in.transfer_mode = cfg->transfer_mode;
    in.train = train != 0;
    in.n_items = n_items;
    in.checkpointing = cfg->checkpointing != 0;
    in.layer_bytes = (static_cast<uint64_t>(cfg->d) * cfg->d + cfg->d) * 4;
    in.act_bytes = static_cast<uint64_t>(cfg->d) * 4;  // one row per item
    in.capacity = cfg->capacity_bytes;
    if (frozen)
        for (int32_t l = 0; l < cfg->n_layers; ++l) in.frozen.push_back(frozen[l] != 0);
    in.sharded = (flags & SP_PLAN_SHARDED) != 0;
    in.eager = (flags & SP_PLAN_EAGER) != 0;
    in.optimizer_state = (flags & SP_PLAN_OPTSTATE) != 0;
    sp::Plan plan = sp::build_plan(in, {});
    if ((flags & SP_PLAN_WRITEBACK) && in.train && plan.error.empty()) {
        // the executor's training write-back scheme, steady state: the second of two calls
        in.wb_stages = std::max(1, std::min(plan.n_slots, 3));  // as the executor (ensure_stages)
        in.defer_writeback = !in.checkpointing;
        plan = sp::build_plan(in, {});
        in.pending_wb_layers = plan.deferred_layers;
        in.pending_wb_slots = plan.deferred_slots;
        plan = sp::build_plan(in, plan.final_slots);
    }
    std::string text = plan.error.empty() ? sp::describe_plan(plan) : ("ERROR " + plan.error + "\n");
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(text.size()));
        std::memcpy(buf, text.data(), static_cast<size_t>(n));
        buf[n] = '\0';
    }
    return static_cast<int64_t>(text.size()) + 1;
}

void sp_digest_tensors(const float* values, int32_t n_items, int64_t rows, int32_t d,
                       char out[17]) {
    uint64_t h = 0xCBF29CE484222325ull;
    auto fnv = [&](const void* p, size_t n) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) {
            h ^= c[i];
            h *= 0x100000001B3ull;
        }
    };
    const int64_t shape[2] = {rows, d};
    const size_t count = static_cast<size_t>(rows) * d;
    for (int32_t t = 0; t < n_items; ++t) {
        fnv(shape, sizeof(shape));
        fnv(values + t * count, count * 4);
    }
    static const char digits[] = "0123456789abcdef";
    for (int i = 15; i >= 0; --i) {
        out[i] = digits[h & 0xF];
        h >>= 4;
    }
    out[16] = '\0';
}

}  // extern "C"

// ---- kernel-level debug entry points (include/superpipe_debug.h) ----------------------
#include "../../include/superpipe_debug.h"
#include "kernels.hpp"

namespace {
int debug_gemm(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, int32_t a_mn,
               const void* B, int32_t ldb, int32_t b_mn, int32_t epilogue, void* out, int32_t ldo,
               const float* bias, int32_t relu, const void* gate, int32_t ldg, int32_t splits,
               int32_t block_n, int32_t cta, void* stream, void* mask_out, const void* gate_mask,
               bool tf32);
}  // namespace

extern "C" int sp_debug_gemm_tf32_async(int32_t M, int32_t N, int32_t K, const void* A,
                                        int32_t lda, int32_t a_mn, const void* B, int32_t ldb,
                                        int32_t b_mn, int32_t epilogue, void* out, int32_t ldo,
                                        const float* bias, int32_t relu, const void* gate,
                                        int32_t ldg, int32_t splits, int32_t block_n, int32_t cta,
                                        void* stream, void* mask_out, const void* gate_mask) {
    return debug_gemm(M, N, K, A, lda, a_mn, B, ldb, b_mn, epilogue, out, ldo, bias, relu, gate, ldg,
                      splits, block_n, cta, stream, mask_out, gate_mask, true);
}

extern "C" int sp_debug_gemm_bf16_masked_async(int32_t M, int32_t N, int32_t K, const void* A,
                                               int32_t lda, int32_t a_mn, const void* B,
                                               int32_t ldb, int32_t b_mn, int32_t epilogue,
                                               void* out, int32_t ldo, const float* bias,
                                               int32_t relu, const void* gate, int32_t ldg,
                                               int32_t splits, int32_t block_n, int32_t cta,
                                               void* stream, void* mask_out,
                                               const void* gate_mask) {
    return debug_gemm(M, N, K, A, lda, a_mn, B, ldb, b_mn, epilogue, out, ldo, bias, relu, gate, ldg,
                      splits, block_n, cta, stream, mask_out, gate_mask, false);
}

namespace {
int debug_gemm(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, int32_t a_mn,
               const void* B, int32_t ldb, int32_t b_mn, int32_t epilogue, void* out, int32_t ldo,
               const float* bias, int32_t relu, const void* gate, int32_t ldg, int32_t splits,
               int32_t block_n, int32_t cta, void* stream, void* mask_out, const void* gate_mask,
               bool tf32) {
    sp::GemmProblem g;
    g.tf32 = tf32;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.a_mn = a_mn != 0;
    g.B = B;
    g.ldb = ldb;
    g.b_mn = b_mn != 0;
    g.epilogue = epilogue;
    g.out = out;
    g.ldo = ldo;
    g.bias = bias;
    g.relu = relu;
    g.gate = gate;
    g.ldg = ldg;
    g.splits = splits;
    g.split_stride = static_cast<int64_t>(M) * ldo;
    g.block_n = block_n;
    g.cta = cta;
    g.lr = 1.0f;
    g.mask_out = static_cast<uint32_t*>(mask_out);
    g.gate_mask = static_cast<const uint32_t*>(gate_mask);
    return static_cast<int>(sp::gemm_bf16(g, static_cast<cudaStream_t>(stream)));
}
}  // namespace

extern "C" int sp_debug_gemm_bf16_async(int32_t M, int32_t N, int32_t K, const void* A,
                                        int32_t lda, int32_t a_mn, const void* B, int32_t ldb,
                                        int32_t b_mn, int32_t epilogue, void* out, int32_t ldo,
                                        const float* bias, int32_t relu, const void* gate,
                                        int32_t ldg, int32_t splits, int32_t block_n,
                                        int32_t cta, void* stream) {
    sp::GemmProblem g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.a_mn = a_mn != 0;
    g.B = B;
    g.ldb = ldb;
    g.b_mn = b_mn != 0;
    g.epilogue = epilogue;
    g.out = out;
    g.ldo = ldo;
    g.bias = bias;
    g.relu = relu;
    g.gate = gate;
    g.ldg = ldg;
    g.splits = splits;
    g.split_stride = static_cast<int64_t>(M) * ldo;
    g.block_n = block_n;
    g.cta = cta;
    g.lr = 1.0f;
    return static_cast<int>(sp::gemm_bf16(g, static_cast<cudaStream_t>(stream)));
}

extern "C" int sp_debug_gemm_bf16(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda,
                                  int32_t a_mn, const void* B, int32_t ldb, int32_t b_mn,
                                  int32_t epilogue, void* out, int32_t ldo, const float* bias,
                                  int32_t relu, const void* gate, int32_t ldg, int32_t splits,
                                  int32_t block_n, int32_t cta) {
    sp::GemmProblem g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.a_mn = a_mn != 0;
    g.B = B;
    g.ldb = ldb;
    g.b_mn = b_mn != 0;
    g.epilogue = epilogue;
    g.out = out;
    g.ldo = ldo;
    g.bias = bias;
    g.relu = relu;
    g.gate = gate;
    g.ldg = ldg;
    g.splits = splits;
    g.split_stride = static_cast<int64_t>(M) * ldo;
    g.block_n = block_n;
    g.cta = cta;
    g.lr = 1.0f;
    cudaError_t e = sp::gemm_bf16(g, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return static_cast<int>(e);
}

extern "C" uint64_t sp_debug_shard_range(uint64_t img, int32_t world, int32_t rank, uint64_t* lo,
                                         uint64_t* hi) {
    const uint64_t shard = sp::shard_bytes(img, world);
    sp::shard_range(shard, img, rank, *lo, *hi);
    return shard;
}

extern "C" int32_t sp_debug_dw_splits(int32_t d, int64_t rows) {
    if (d < 1 || rows < 1 || rows > (1ll << 31) - 1) return 0;
    const int r = static_cast<int>(rows);
    return sp::choose_dw(d, d, r, 16, true).splits;
}

extern "C" int32_t sp_debug_dw_choice(int32_t d, int64_t rows, int32_t fused_ok, int32_t* cta,
                                      int32_t* block_n) {
    if (d < 1 || rows < 1 || rows > (1ll << 31) - 1 || !cta || !block_n) return 0;
    const sp::DwChoice c = sp::choose_dw(d, d, static_cast<int>(rows), 16, fused_ok != 0);
    *cta = c.cta;
    *block_n = c.block_n;
    return c.splits;
}

namespace sp {
void set_gemm_debug(const char* key, int value, bool* known);
}

extern "C" int sp_debug_set(sp_exec* ex, const char* key, int32_t value) {
    if (!key) return SP_ERR_INVALID;
    bool known = false;
    sp::set_gemm_debug(key, value, &known);
    if (known) return SP_OK;
    if (!ex) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->set_debug(key, value); });
}

extern "C" int32_t sp_debug_effective_splits(int32_t K, int32_t splits) {
    return sp::effective_splits(K, splits);
}

// Two consecutive training plans as the executor makes them (make_plan): call 1 at act_bytes1,
// call 2 at act_bytes2 with call 1's deferred write-backs pending. When the second ring would
// shrink below a pending slot the executor flushes them first; the text then starts "FLUSHED".
extern "C" int64_t sp_debug_plan_two_calls(const sp_config* cfg, uint64_t act_bytes1,
                                           uint64_t act_bytes2, char* buf, int64_t cap) {
    if (!cfg) return -1;
    sp::PlanInput in;
    in.n_layers = cfg->n_layers;
    in.strategy = cfg->strategy;
    in.k = cfg->k;
    in.k_prime = cfg->k_prime;
    in.transfer_mode = cfg->transfer_mode;
    in.train = true;
    in.layer_bytes = (static_cast<uint64_t>(cfg->d) * cfg->d + cfg->d) * 4;
    in.capacity = cfg->capacity_bytes;
    in.eager = true;
    in.wb_stages = 3;
    in.defer_writeback = true;
    in.defer_budget = in.n_layers;  // the most the executor ever defers (clipped to S)
    in.act_bytes = act_bytes1;
    sp::Plan p1 = sp::build_plan(in, {});
    std::string text;
    if (!p1.error.empty()) {
        text = "ERROR " + p1.error + "\n";
    } else {
        in.act_bytes = act_bytes2;
        in.pending_wb_layers = p1.deferred_layers;
        in.pending_wb_slots = p1.deferred_slots;
        sp::Plan p2 = sp::build_plan(in, p1.final_slots);
        std::string head;
        if (p2.pending_conflict) {
            head = "FLUSHED";
            for (int L : p1.deferred_layers) head += " " + std::to_string(L);
            head += "\n";
            in.pending_wb_layers.clear();
            in.pending_wb_slots.clear();
            p2 = sp::build_plan(in, p1.final_slots);
        }
        std::string deferred = "DEFERRED";
        for (int L : p1.deferred_layers) deferred += " " + std::to_string(L);
        text = deferred + "\n" + head +
               (p2.error.empty() ? sp::describe_plan(p2) : ("ERROR " + p2.error + "\n"));
    }
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(text.size()));
        std::memcpy(buf, text.data(), static_cast<size_t>(n));
        buf[n] = '\0';
    }
    return static_cast<int64_t>(text.size()) + 1;
}

extern "C" int sp_debug_gemm_ex(const sp_debug_gemm_args* a) {
    if (!a) return static_cast<int>(cudaErrorInvalidValue);
    sp::GemmProblem g;
    g.M = a->M;
    g.N = a->N;
    g.K = a->K;
    g.A = a->A;
    g.lda = a->lda;
    g.a_mn = a->a_mn != 0;
    g.B = a->B;
    g.ldb = a->ldb;
    g.b_mn = a->b_mn != 0;
    g.epilogue = a->epilogue;
    g.out = a->out;
    g.ldo = a->ldo;
    g.bias = a->bias;
    g.relu = a->relu;
    g.gate = a->gate;
    g.ldg = a->ldg;
    g.splits = a->splits;
    g.split_stride = static_cast<int64_t>(a->M) * a->ldo;
    g.block_n = a->block_n;
    g.cta = a->cta;
    g.lr = 1.0f;
    g.aux = a->aux;
    g.ldaux = a->ldaux;
    g.act = a->act;
    g.colsum_part = a->colsum_part;
    return static_cast<int>(sp::gemm_bf16(g, static_cast<cudaStream_t>(a->stream)));
}

extern "C" int sp_debug_attention(int32_t backward, int64_t tokens, int32_t seq_len, int32_t n_heads,
                                  int32_t n_kv_heads, int32_t head_dim, int32_t causal, const void* qkv, void* o,
                                  float* lse, const void* dout, float* delta, void* dqkv, void* stream) {
    sp::AttnProblem a;
    a.tokens = tokens;
    a.seq_len = seq_len;
    a.n_heads = n_heads;
    a.n_kv_heads = n_kv_heads;
    a.head_dim = head_dim;
    a.causal = causal;
    a.qkv = qkv;
    a.o = o;
    a.lse = lse;
    a.dout = dout;
    a.delta = delta;
    a.dqkv = dqkv;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    return static_cast<int>(backward ? sp::attention_backward(a, st) : sp::attention_forward(a, st));
}

extern "C" int sp_debug_norm_forward(const float* x, const float* gamma, const float* beta, int32_t rms, float eps,
                                     int64_t rows, int32_t d, void* y, float* stats, void* stream) {
    sp::norm_forward(x, gamma, beta, rms, eps, rows, d, y, stats, static_cast<cudaStream_t>(stream));
    return static_cast<int>(cudaGetLastError());
}

extern "C" int sp_debug_norm_backward(const float* dy, const float* x, const float* stats, const float* gamma,
                                      int32_t rms, int64_t rows, int32_t d, const float* dres_in, float* dres_out,
                                      void* dres_out16, float* part, int32_t* counters, float* out, void* stream) {
    sp::ColScratch scr;
    scr.part = part;
    scr.counters = counters;
    sp::norm_backward(dy, x, stats, gamma, rms, rows, d, dres_in, dres_out, dres_out16, scr, out,
                      static_cast<cudaStream_t>(stream));
    return static_cast<int>(cudaGetLastError());
}

extern "C" int sp_debug_colsum(const void* x, int64_t rows, int32_t n, float* part, int32_t* counters, float* out,
                               void* stream) {
    sp::ColScratch scr;
    scr.part = part;
    scr.counters = counters;
    sp::colsum_total_bf16(x, rows, n, scr, out, static_cast<cudaStream_t>(stream));
    return static_cast<int>(cudaGetLastError());
}

extern "C" int sp_debug_norm_backward_fused(const float* dy, const float* x, const float* stats, const float* gamma,
                                            int32_t rms, int64_t rows, int32_t d, const float* dres_in, float* dres_out,
                                            void* dres_out16, float* ppart, float* cpart, float* out_param,
                                            float* out_csum, void* stream) {
    if (!sp::norm_backward_fused_ok(d) || (out_csum && !dres_out)) return SP_ERR_INVALID;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    sp::norm_backward_fused(dy, x, stats, gamma, rms, rows, d, dres_in, dres_out, dres_out16,
                            out_param ? ppart : nullptr, out_csum ? cpart : nullptr, st);
    sp::ColChunks c;
    c.chunks = sp::norm_bwd_chunks(rows);
    if (out_param) {
        c.part[c.n] = ppart;
        c.stride[c.n] = 2 * static_cast<int64_t>(d);
        c.width[c.n] = rms ? d : 2 * d;
        c.out[c.n++] = out_param;
    }
    if (out_csum) {
        c.part[c.n] = cpart;
        c.stride[c.n] = d;
        c.width[c.n] = d;
        c.out[c.n++] = out_csum;
    }
    sp::reduce_col_chunks(c, st);
    return static_cast<int>(cudaGetLastError());
}

namespace sp {
int attn_trace_read(unsigned long long* out, int cap);  // kernels_attn_bwd.cu
}
extern "C" int sp_debug_attn_trace(uint64_t* out, int32_t cap) {
    return sp::attn_trace_read(reinterpret_cast<unsigned long long*>(out), cap);
}

extern "C" void sp_debug_col_scratch(int64_t rows, int32_t widest, int64_t* part_floats, int64_t* counters) {
    const sp::ColScratchSize s = sp::col_scratch_size(rows, widest);
    *part_floats = static_cast<int64_t>(s.part_floats);
    *counters = static_cast<int64_t>(s.counters);
}

extern "C" int sp_debug_read_grad(sp_exec* ex, int32_t index, float* out) {
    if (!ex || !out) return SP_ERR_INVALID;
    return guarded(ex, [&] { ex->impl->debug_read_grad(index, out); });
}

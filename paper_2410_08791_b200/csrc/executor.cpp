// executor.cpp — the B200 layer-streaming ring executor.
//
// Replaces the reference Engine (engine.cpp:33-548): instead of a virtual event loop, the
// static plan (plan.cpp) is enqueued once onto four CUDA streams —
//   h2d  : pinned host -> HBM slot copies (copy engine 0)
//   comp : the layer kernels (tcgen05 GEMMs or the exact SIMT kernels), loss
//   d2h  : updated-weight writeback / activation offload (copy engine 1)
//   upd  : gradient all-reduce (NCCL, data parallel) + SGD update
// joined only by CUDA events at the plan's dependency edges, so the copy engines stream
// layers i+1..i+k over the host link while layer i computes. The DeviceArena ledger is
// replayed by the planner (reference byte semantics); real HBM use is reported separately.
#include "executor.hpp"

#include <cstdio>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: no-ops unless a tool (nsys) is attached

#include <cuda_bf16.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "kernels.hpp"
#include "nccl_dyn.hpp"

namespace sp {

#define CUDA_OK(expr)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw Error(SP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define NCCL_OK(expr)                                                                      \
    do {                                                                                   \
        ncclResult_t r_ = (expr);                                                          \
        if (r_ != ncclSuccess)                                                             \
            throw Error(SP_ERR_NCCL, std::string(#expr) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

namespace {

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

uint16_t bf16_rne(float f) {  // matches __float2bfloat16_rn for all inputs
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

template <typename F>
void parallel_for(int n, F&& f) {
    const int hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = std::min(n, std::min(hw, 16));
    if (nt <= 1) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int i = t; i < n; i += nt) f(i);
        });
    for (auto& x : th) x.join();
}

}  // namespace

Executor::Executor(const sp_config& cfg, const sp_block_desc* block) : cfg_(cfg) {
    n_ = cfg.n_layers;
    d_ = cfg.d;
    if (block && block->kind != SP_BLOCK_DENSE) {
        const std::string e = make_block_layout(*block, lay_);
        if (!e.empty()) throw Error(SP_ERR_INVALID, e);
        if (block->d != cfg.d) throw Error(SP_ERR_INVALID, "block: d must equal the executor's d");
        if (cfg.numerics != SP_NUMERICS_BF16)
            throw Error(SP_ERR_INVALID, "transformer blocks run in bf16 numerics (SP_NUMERICS_BF16)");
        blk_ = true;
        split_ = true;
        infer_only_ = (block->flags & SP_BLOCK_INFER_ONLY) != 0;
    }
    if (n_ < 1) throw Error(SP_ERR_INVALID, "build_model: n_layers must be >= 1");
    if (d_ < 1) throw Error(SP_ERR_INVALID, "build_model: d must be >= 1");
    const std::string v = validate_strategy(cfg.strategy, cfg.k, cfg.k_prime, n_);
    if (!v.empty()) throw Error(SP_ERR_INVALID, v);
    if (cfg.strategy == static_cast<int>(Strategy::CpuOnly))
        throw Error(SP_ERR_INVALID,
                    "strategy: cpu_only is the reference's host path; the GPU executor has no CPU "
                    "fallback");
    if (cfg.numerics != SP_NUMERICS_EXACT && cfg.numerics != SP_NUMERICS_BF16 &&
        cfg.numerics != SP_NUMERICS_TF32)
        throw Error(SP_ERR_INVALID, "numerics: unknown mode");
    if (cfg.transfer_mode != SP_SEQUENTIAL && cfg.transfer_mode != SP_BATCH)
        throw Error(SP_ERR_INVALID, "transfer_mode: unknown mode");
    bf16_ = cfg.numerics == SP_NUMERICS_BF16;
    tf32_ = cfg.numerics == SP_NUMERICS_TF32;
    tc_ = bf16_ || tf32_;
    if (tc_ && d_ % 64 != 0)
        throw Error(SP_ERR_INVALID, "bf16 / tf32 numerics require d % 64 == 0 (128-byte TMA rows)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SP_ERR_CUDA, "no CUDA device visible: the executor has no CPU fallback");
    if (cfg.device < 0 || cfg.device >= ndev) throw Error(SP_ERR_INVALID, "device ordinal out of range");
    CUDA_OK(cudaSetDevice(cfg.device));

    host_stride_ = infer_only_ ? round_up(lay_.wire_bytes, 256)
                 : blk_       ? round_up(std::max<size_t>(lay_.split_bytes, img_f() * 4), 256)
                              : img_f() * 4;
    CUDA_OK(cudaHostAlloc(&host32_, static_cast<size_t>(n_) * host_stride_, cudaHostAllocPortable));
    std::memset(host32_, 0, static_cast<size_t>(n_) * host_stride_);
    // the bf16 inference wire image: a separate host copy for dense layers, the split master's
    // own prefix for blocks (allocated when dp_init turns the split layout off)
    if (bf16_ && !split_) CUDA_OK(cudaHostAlloc(&host16_, static_cast<size_t>(n_) * wire16_bytes(), cudaHostAllocPortable));

    n_slots_ = ring_slots(cfg.strategy, cfg.k, cfg.k_prime, n_);
    layout_slots(1);

    // Priorities: the compute stream's blocks are scheduled before the update stream's (the
    // update kernels' many short blocks would otherwise take SM slots from the layer kernels);
    // graphs are instantiated with per-node priority so replays keep them.
    int prio_lo = 0, prio_hi = 0;
    CUDA_OK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CUDA_OK(cudaStreamCreateWithPriority(&s_h2d_, cudaStreamNonBlocking, prio_lo));
    CUDA_OK(cudaStreamCreateWithPriority(&s_comp_, cudaStreamNonBlocking, prio_hi));
    CUDA_OK(cudaStreamCreateWithPriority(&s_d2h_, cudaStreamNonBlocking, prio_lo));
    CUDA_OK(cudaStreamCreateWithPriority(&s_upd_, cudaStreamNonBlocking, prio_lo));
    CUDA_OK(cudaEventCreate(&ev_call0_));
    CUDA_OK(cudaEventCreate(&ev_call1_));
    CUDA_OK(cudaEventCreateWithFlags(&ev_io_in_, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&ev_io_out_, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&ev_loss_, cudaEventDisableTiming));
    for (auto& e : ev_join_) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_OK(cudaHostAlloc(&loss_host_, 16, cudaHostAllocPortable));

    relu_.assign(static_cast<size_t>(n_), 1);
    frozen_.assign(static_cast<size_t>(n_), 0);
    registered_.assign(static_cast<size_t>(n_), 0);
    inconsistent_.assign(static_cast<size_t>(n_), 0);
    host16_stale_.assign(static_cast<size_t>(n_), 1);
    host_partial_.assign(static_cast<size_t>(n_), 0);
}

Executor::~Executor() {
    if (s_h2d_) cudaStreamSynchronize(s_h2d_);
    if (s_comp_) cudaStreamSynchronize(s_comp_);
    if (s_d2h_) cudaStreamSynchronize(s_d2h_);
    if (s_upd_) cudaStreamSynchronize(s_upd_);
    if (comm_ && nccl().ok()) nccl().CommDestroy(comm_);
    for (void* p : dev_allocs_) cudaFree(p);
    if (slots_dev_) cudaFree(slots_dev_);
    for (auto e : ev_done_) cudaEventDestroy(e);
    for (auto e : ev_start_) cudaEventDestroy(e);
    for (auto e : gemm_ev_) cudaEventDestroy(e);
    for (auto e : ev_dep_) cudaEventDestroy(e);
    for (auto e : ev_move_) cudaEventDestroy(e);
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_loss_) cudaEventDestroy(ev_loss_);
    for (auto e : ev_join_)
        if (e) cudaEventDestroy(e);
    if (ev_call0_) cudaEventDestroy(ev_call0_);
    if (ev_call1_) cudaEventDestroy(ev_call1_);
    if (ev_io_in_) cudaEventDestroy(ev_io_in_);
    if (ev_io_out_) cudaEventDestroy(ev_io_out_);
    if (shm_) {
        cudaHostUnregister(host32_);
        munmap(shm_, shm_bytes_);
        if (shm_owner_) shm_unlink(shm_name_.c_str());
    } else if (host32_) {
        cudaFreeHost(host32_);
    }
    if (host_m_) cudaFreeHost(host_m_);
    if (host_v_) cudaFreeHost(host_v_);
    if (adamw_host_) cudaFreeHost(adamw_host_);
    if (adamw_dev_) cudaFree(adamw_dev_);
    if (stages_dev_) cudaFree(stages_dev_);
    if (host16_) cudaFreeHost(host16_);
    if (host_act_) cudaFreeHost(host_act_);
    if (loss_host_) cudaFreeHost(loss_host_);
    for (auto s : {s_h2d_, s_comp_, s_d2h_, s_upd_})
        if (s) cudaStreamDestroy(s);
}

// Slot = [A: fp32 W|b image] ([M][V]: AdamW state, same layout as A) [B: bf16 W + fp32 b
// wire image]. Each region is cut into `world` equal shards (256-byte aligned) so a rank can
// H2D / D2H its own shard and NCCL all-gather / reduce-scatter the rest in place.
void Executor::layout_slots(int world) {
    shardA_ = shard_bytes(layer_bytes(), world);
    shardB_ = shard_bytes(wire16_bytes(), world);
    if (split_) {
        // [A: split image, whose wire prefix is the GEMM operand] [M][V: AdamW, fp32 logical]
        const size_t a_region = round_up(layer_bytes(), 1024), o_region = round_up(opt_bytes(), 1024);
        off_m_ = adamw() ? a_region : 0;
        off_v_ = adamw() ? a_region + o_region : 0;
        fp_bytes_ = a_region + (adamw() ? 2 * o_region : 0);
        off_w16_ = 0;
        slot_bytes_ = fp_bytes_;
    } else {
        const size_t a_region = round_up(shardA_ * world, 1024);
        off_m_ = adamw() ? a_region : 0;
        off_v_ = adamw() ? 2 * a_region : 0;
        off_w16_ = adamw() ? 3 * a_region : a_region;
        fp_bytes_ = off_w16_;
        slot_bytes_ = bf16_ ? round_up(off_w16_ + shardB_ * world, 1024) : off_w16_;
    }
    if (slots_dev_) {
        CUDA_OK(cudaDeviceSynchronize());
        cudaFree(slots_dev_);
        slots_dev_ = nullptr;
    }
    CUDA_OK(cudaMalloc(&slots_dev_, static_cast<size_t>(n_slots_) * slot_bytes_));
    if (stages_dev_) {  // re-sized on the next training call
        cudaFree(stages_dev_);
        stages_dev_ = nullptr;
        n_stages_ = 0;
    }
    pending_wb_layers_.clear();  // callers flush first; the old slots are gone
    pending_wb_slots_.clear();
    cache_.assign(static_cast<size_t>(n_slots_), SlotCache{});
    cache_fmt_ = -1;
    w16_layer_.assign(static_cast<size_t>(n_slots_), -1);
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
    graphs_.clear();
    ++alloc_gen_;
}

// Write-back stages: min(S, 3) buffers of one slot's fp32 regions (weights [+ m, v]). Three
// keep the update stream ahead of the D2H engine: 2 cost 2% of the C2 step, 3 and 8 measure
// the same (SGD and AdamW, interleaved A/B), and each stage is a slot's worth of HBM.
void Executor::ensure_stages() {
    if (stages_dev_ || !staged_writeback_) return;
    n_stages_ = std::max(1, std::min(n_slots_, wb_stages_cap_));
    stage_bytes_ = fp_bytes_;  // [A] or [A][M][V]: the slot minus its bf16 wire region
    CUDA_OK(cudaMalloc(&stages_dev_, static_cast<size_t>(n_stages_) * stage_bytes_));
    // (a split update writes only the tensors into a stage: alignment gaps stay zero)
    CUDA_OK(cudaMemset(stages_dev_, 0, static_cast<size_t>(n_stages_) * stage_bytes_));
}

// Completes the previous train step's deferred write-backs now (host readers, inference,
// re-layout): each still-resident layer's updated image [+ m, v] to the pinned master.
void Executor::flush_writebacks() {
    if (pending_wb_layers_.empty()) return;
    CUDA_OK(cudaSetDevice(cfg_.device));
    for (auto s : {s_h2d_, s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamSynchronize(s));
    const size_t img = layer_bytes(), ob = opt_bytes();
    for (size_t i = 0; i < pending_wb_layers_.size(); ++i) {
        const int L = pending_wb_layers_[i], s = pending_wb_slots_[i];
        CUDA_OK(cudaMemcpyAsync(host_layer(L), slot_ptr(s), img, cudaMemcpyDeviceToHost, s_d2h_));
        if (adamw()) {
            CUDA_OK(cudaMemcpyAsync(host_opt(host_m_, L), slot_m32(s), ob, cudaMemcpyDeviceToHost, s_d2h_));
            CUDA_OK(cudaMemcpyAsync(host_opt(host_v_, L), slot_v32(s), ob, cudaMemcpyDeviceToHost, s_d2h_));
        }
        host16_stale_[static_cast<size_t>(L)] = 1;
    }
    CUDA_OK(cudaStreamSynchronize(s_d2h_));
    for (int L : pending_wb_layers_) bump_version(L);
    pending_wb_layers_.clear();
    pending_wb_slots_.clear();
}

// Shared master segment: [header | relu[n] frozen[n] registered[n] (int32) | pad | master].
struct Executor::ShmHeader {
    uint64_t magic;
    int32_t n, d;
    uint64_t master_offset, master_bytes;
    int32_t meta[1];  // 3 * n int32 follow
};
namespace {
constexpr uint64_t kShmMagic = 0x3176'4D48'5350'5053ull;  // "SPSPHMv1"
}

void Executor::sync_layer_meta(int index) {
    if (!shm_) return;
    int32_t* meta = shm_->meta;
    if (index >= 0) {  // this process registered a layer: publish its metadata
        meta[index] = relu_[static_cast<size_t>(index)];
        meta[n_ + index] = frozen_[static_cast<size_t>(index)];
        meta[2 * n_ + index] = registered_[static_cast<size_t>(index)];
        return;
    }
    for (int L = 0; L < n_; ++L) {  // pick up what other processes registered
        relu_[static_cast<size_t>(L)] = meta[L];
        frozen_[static_cast<size_t>(L)] = meta[n_ + L];
        registered_[static_cast<size_t>(L)] = static_cast<uint8_t>(meta[2 * n_ + L]);
    }
}

void Executor::share_host_master(const char* name, bool create) {
    if (!name || !*name) throw Error(SP_ERR_INVALID, "share_host_master: empty segment name");
    if (shm_) throw Error(SP_ERR_STATE, "share_host_master: the master is already shared");
    flush_writebacks();
    if (create) require_full_host(-1, "share_host_master");
    CUDA_OK(cudaSetDevice(cfg_.device));
    for (auto s : {s_h2d_, s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamSynchronize(s));
    const std::string nm = name[0] == '/' ? std::string(name) : "/" + std::string(name);
    const size_t master = static_cast<size_t>(n_) * host_stride_;
    const size_t ver_off = round_up(offsetof(ShmHeader, meta) + 12 * static_cast<size_t>(n_), 8);
    const size_t off = round_up(ver_off + 8 * static_cast<size_t>(n_), 4096);
    const size_t bytes = off + master;
    int fd = -1;
    if (create) {
        shm_unlink(nm.c_str());  // a stale segment of a crashed run
        fd = shm_open(nm.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        // reserve the pages now: a tmpfs too small for the model fails here, not with SIGBUS
        if (fd < 0 || ftruncate(fd, static_cast<off_t>(bytes)) != 0 ||
            posix_fallocate(fd, 0, static_cast<off_t>(bytes)) != 0) {
            if (fd >= 0) close(fd);
            shm_unlink(nm.c_str());
            throw Error(SP_ERR_INTERNAL, "share_host_master: cannot create a " + std::to_string(bytes) +
                                             "-byte shared segment " + nm + " (is /dev/shm large enough?)");
        }
    } else {
        fd = shm_open(nm.c_str(), O_RDWR, 0);
        struct stat st{};
        if (fd < 0 || fstat(fd, &st) != 0 || static_cast<size_t>(st.st_size) != bytes) {
            if (fd >= 0) close(fd);
            throw Error(SP_ERR_INVALID, "share_host_master: no segment " + nm + " of this model's size");
        }
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(SP_ERR_INTERNAL, "share_host_master: mmap failed");
    auto* h = static_cast<ShmHeader*>(p);
    float* base = reinterpret_cast<float*>(static_cast<uint8_t*>(p) + off);
    if (create) {
        std::memcpy(base, host32_, master);
        h->n = n_;
        h->d = d_;
        h->master_offset = off;
        h->master_bytes = master;
        for (int L = 0; L < n_; ++L) {
            h->meta[L] = relu_[static_cast<size_t>(L)];
            h->meta[n_ + L] = frozen_[static_cast<size_t>(L)];
            h->meta[2 * n_ + L] = registered_[static_cast<size_t>(L)];
        }
        __atomic_store_n(&h->magic, kShmMagic, __ATOMIC_RELEASE);
    } else if (__atomic_load_n(&h->magic, __ATOMIC_ACQUIRE) != kShmMagic || h->n != n_ || h->d != d_) {
        munmap(p, bytes);
        throw Error(SP_ERR_INVALID, "share_host_master: segment " + nm + " holds another model");
    }
    const cudaError_t e = cudaHostRegister(base, master, cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        munmap(p, bytes);
        if (create) shm_unlink(nm.c_str());
        throw Error(SP_ERR_CUDA, std::string("share_host_master: cudaHostRegister: ") + cudaGetErrorString(e));
    }
    cudaFreeHost(host32_);
    host32_ = base;
    shm_ = h;
    shm_bytes_ = bytes;
    shm_name_ = nm;
    shm_owner_ = create;
    ver_off_ = ver_off;
    cache_ver_.assign(static_cast<size_t>(n_), ~0ull);
    host16_ver_.assign(static_cast<size_t>(n_), ~0ull);
    plan_ver_.assign(static_cast<size_t>(n_), 0);
    sync_layer_meta(-1);
    std::fill(host16_stale_.begin(), host16_stale_.end(), 1);
    for (auto& c : cache_) c.valid = false;
    std::fill(w16_layer_.begin(), w16_layer_.end(), -1);
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);  // host pointers are baked in
    graphs_.clear();
}

uint64_t Executor::layer_version(int L) const {
    return shm_ ? __atomic_load_n(&shm_versions()[L], __ATOMIC_ACQUIRE) : 0;
}

void Executor::bump_version(int L) {
    if (shm_) cache_ver_[static_cast<size_t>(L)] = __atomic_add_fetch(&shm_versions()[L], 1, __ATOMIC_ACQ_REL);
}

// After a call's streams are synchronised: publish this call's host writes (write-backs run in
// it, including the previous call's deferred ones) and note which versions the loads saw.
void Executor::after_call(const Plan& plan) {
    if (!shm_) return;
    for (const Op& op : plan.ops) {
        if (op.kind == OpKind::D2H && !op.deferred) bump_version(op.layers[0]);
        if (op.kind == OpKind::H2D)
            for (size_t j = 0; j < op.layers.size(); ++j)
                if (op.weights[j]) cache_ver_[static_cast<size_t>(op.layers[j])] = plan_ver_[static_cast<size_t>(op.layers[j])];
    }
}

void Executor::register_layer(int index, const float* W, const float* b, int activation,
                              int frozen) {
    if (index < 0 || index >= n_) throw Error(SP_ERR_INVALID, "register_layer: index out of range");
    if (!W || !b) throw Error(SP_ERR_INVALID, "register_layer: null weight or bias");
    if (blk_) throw Error(SP_ERR_INVALID, "register_layer: this executor streams transformer blocks (sp_register_block)");
    flush_writebacks();  // a pending write-back must not land on top of the new weights
    if (activation != SP_RELU && activation != SP_IDENTITY)
        throw Error(SP_ERR_INVALID, "register_layer: unknown activation");
    const size_t dd = static_cast<size_t>(d_) * d_;
    float* dst = host32_ + static_cast<size_t>(index) * (dd + d_);
    std::memcpy(dst, W, dd * 4);
    std::memcpy(dst + dd, b, static_cast<size_t>(d_) * 4);
    relu_[index] = activation == SP_RELU;
    frozen_[index] = frozen != 0;
    registered_[index] = 1;
    inconsistent_[static_cast<size_t>(index)] = 0;
    host16_stale_[index] = 1;
    host_partial_[index] = 0;
    sync_layer_meta(index);
    bump_version(index);
    for (auto& c : cache_)
        if (c.layer == index) c.valid = false;
}

void Executor::require_full_host(int layer, const char* what) const {
    for (int i = 0; i < n_; ++i)
        if ((layer < 0 || i == layer) && host_partial_[static_cast<size_t>(i)])
            throw Error(SP_ERR_STATE, std::string(what) + ": layer " + std::to_string(i) +
                                          " holds only this rank's shard after sharded training; "
                                          "call sp_dp_sync() on every rank first");
}

void Executor::check_ready() {
    if (shm_) sync_layer_meta(-1);  // layers registered by another process sharing the master
    for (int i = 0; i < n_; ++i) {
        if (!registered_[i])
            throw Error(SP_ERR_STATE, "layer " + std::to_string(i) + " was never registered");
        if (inconsistent_[static_cast<size_t>(i)])
            throw Error(SP_ERR_STATE, "layer " + std::to_string(i) +
                                          ": a failed train step left the host master part-updated; "
                                          "register the layers again");
    }
}

void Executor::refresh_host16() {
    if (!bf16_ || split_) return;  // (split masters stream their own wire prefix)
    std::vector<int> todo;
    for (int i = 0; i < n_; ++i) {
        const uint64_t v = layer_version(i);  // another process may have written the master
        if (host16_stale_[i] || (shm_ && v != host16_ver_[static_cast<size_t>(i)])) todo.push_back(i);
        if (shm_) host16_ver_[static_cast<size_t>(i)] = v;
    }
    if (todo.empty()) return;
    const size_t dd = static_cast<size_t>(d_) * d_;
    if (blk_) {  // wire image: matrices bf16, vectors fp32, each at its layout offset
        parallel_for(static_cast<int>(todo.size()), [&](int t) {
            const int L = todo[t];
            const float* src = reinterpret_cast<const float*>(host_layer(L));
            uint8_t* dst = host16_ + static_cast<size_t>(L) * wire16_bytes();
            for (const BlockTensor& x : lay_.t) {
                if (x.matrix) {
                    uint16_t* w16 = reinterpret_cast<uint16_t*>(dst + x.wire_off);
                    for (uint64_t e = 0; e < x.count(); ++e) w16[e] = bf16_rne(src[x.off + e]);
                } else {
                    std::memcpy(dst + x.wire_off, src + x.off, x.count() * 4);
                }
            }
        });
        for (int L : todo) host16_stale_[L] = 0;
        return;
    }
    parallel_for(static_cast<int>(todo.size()), [&](int t) {
        const int L = todo[t];
        const float* src = host32_ + static_cast<size_t>(L) * (dd + d_);
        uint8_t* dst = host16_ + static_cast<size_t>(L) * wire16_bytes();
        uint16_t* w16 = reinterpret_cast<uint16_t*>(dst);
        for (size_t e = 0; e < dd; ++e) w16[e] = bf16_rne(src[e]);
        std::memcpy(dst + dd * 2, src + dd, static_cast<size_t>(d_) * 4);
    });
    for (int L : todo) host16_stale_[L] = 0;
}

void Executor::ensure_buffers(int64_t rows, int n_items, bool train, bool device_io) {
    const bool ckpt = train && cfg_.checkpointing && cfg_.strategy != SP_STANDARD;
    const bool fits = rows <= cap_rows_ && n_items <= cap_items_ && (!train || cap_train_);
    if (fits && (!ckpt || host_act_)) return;
    CUDA_OK(cudaDeviceSynchronize());
    ++alloc_gen_;  // captured graphs refer to the old buffers
    for (void* p : dev_allocs_) cudaFree(p);
    dev_allocs_.clear();
    dev_bytes_ = 0;
    if (host_act_) {
        cudaFreeHost(host_act_);
        host_act_ = nullptr;
    }
    const int64_t R = std::max<int64_t>(rows, cap_rows_);
    const int items = std::max(n_items, cap_items_);
    const bool tr = train || cap_train_;
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        bytes = round_up(std::max<size_t>(bytes, 256), 1024);
        CUDA_OK(cudaMalloc(&p, bytes));
        dev_allocs_.push_back(p);
        dev_bytes_ += bytes;
        return p;
    };
    const size_t elt = bf16_ ? 2 : 4;
    const size_t act = static_cast<size_t>(R) * d_;
    const size_t dd = static_cast<size_t>(d_) * d_;
    xin_ = static_cast<float*>(alloc(std::max<size_t>(static_cast<size_t>(items), 1) * act * 4));
    yout_ = static_cast<float*>(alloc(std::max<size_t>(static_cast<size_t>(items), 1) * act * 4));
    act_.clear();
    ba_.clear();
    masks_.clear();
    if (blk_) {
        if (tr) {
            tgt_ = static_cast<float*>(alloc(act * 4));
            loss_parts_ = static_cast<float*>(alloc(4096 * 4));
            loss_dev_ = static_cast<float*>(alloc(16));
            if (cfg_.checkpointing && cfg_.strategy != SP_STANDARD) {  // the layer input (fp32) rides
                for (auto& f : fa_) f = alloc(act * 4);
                for (int s = 0; s < n_slots_; ++s) ba_.push_back(alloc(act * 4));
                host_act_bytes_ = static_cast<size_t>(n_) * act * 4;
                CUDA_OK(cudaHostAlloc(&host_act_, host_act_bytes_, cudaHostAllocPortable));
            }
        }
        block_alloc(R, items, tr, alloc);
        cap_rows_ = R;
        cap_items_ = items;
        cap_train_ = tr;
        return;
    }
    for (auto& p : pp_) p = alloc(act * elt);
    xconv_ = alloc(act * 2);
    if (tr) {
        tgt_ = static_cast<float*>(alloc(act * 4));
        for (int l = 0; l < n_; ++l) act_.push_back(alloc(act * elt));
        masks_.clear();
        if (tc_ && !(cfg_.checkpointing && cfg_.strategy != SP_STANDARD) && d_ % 32 == 0)
            for (int l = 0; l < n_; ++l)
                masks_.push_back(static_cast<uint32_t*>(alloc(static_cast<size_t>(R) * (d_ / 32) * 4)));
        for (auto& g : gbuf_) g = alloc(act * elt);
        splits_cap_ = tc_ ? choose_dw(d_, d_, static_cast<int>(R), 16, comm_ == nullptr, tf32_).splits : 1;
        col_chunks_cap_ = tc_ ? colsum_chunks(R) : 1;
        // gradient buffers hold world equal shards when reduce-scattered (sharded streaming)
        const size_t grad_f = std::max(dd + d_, shardA_ / 4 * static_cast<size_t>(world_));
        const size_t ws = tc_ ? static_cast<size_t>(splits_cap_) * dd + static_cast<size_t>(col_chunks_cap_) * d_
                              : grad_f;
        for (auto& g : gws_) g = static_cast<float*>(alloc(ws * 4));
        grad_red_ = static_cast<float*>(alloc(grad_f * 4));
        loss_parts_ = static_cast<float*>(alloc(4096 * 4));
        loss_dev_ = static_cast<float*>(alloc(16));
        if (cfg_.checkpointing && cfg_.strategy != SP_STANDARD) {
            for (auto& f : fa_) f = alloc(act * elt);
            for (int s = 0; s < n_slots_; ++s) ba_.push_back(alloc(act * elt));
            host_act_bytes_ = static_cast<size_t>(n_) * act * elt;
            CUDA_OK(cudaHostAlloc(&host_act_, host_act_bytes_, cudaHostAllocPortable));
        }
    }
    cap_rows_ = R;
    cap_items_ = items;
    cap_train_ = tr;
    (void)device_io;
}

namespace {
bool same_input(const PlanInput& a, const PlanInput& b) {
    return a.n_layers == b.n_layers && a.strategy == b.strategy && a.k == b.k && a.k_prime == b.k_prime &&
           a.transfer_mode == b.transfer_mode && a.train == b.train && a.n_items == b.n_items &&
           a.checkpointing == b.checkpointing && a.sharded == b.sharded && a.eager == b.eager &&
           a.optimizer_state == b.optimizer_state && a.wb_stages == b.wb_stages &&
           a.defer_writeback == b.defer_writeback && a.defer_budget == b.defer_budget &&
           a.pending_wb_layers == b.pending_wb_layers && a.pending_wb_slots == b.pending_wb_slots &&
           a.frozen == b.frozen && a.layer_bytes == b.layer_bytes && a.act_bytes == b.act_bytes &&
           a.capacity == b.capacity;
}
bool same_slots(const std::vector<SlotCache>& a, const std::vector<SlotCache>& b) {
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (a[i].layer != b[i].layer || a[i].valid != b[i].valid) return false;
    return true;
}
}  // namespace

const Plan& Executor::make_plan(bool train, int n_items, int64_t rows, int fmt) {
    PlanInput in;
    in.n_layers = n_;
    in.strategy = cfg_.strategy;
    in.k = cfg_.k;
    in.k_prime = cfg_.k_prime;
    in.transfer_mode = cfg_.transfer_mode;
    in.train = train;
    in.n_items = n_items;
    in.checkpointing = cfg_.checkpointing != 0;
    in.frozen.assign(frozen_.begin(), frozen_.end());
    in.layer_bytes = layer_bytes();
    in.act_bytes = static_cast<uint64_t>(rows) * d_ * 4;
    in.capacity = cfg_.capacity_bytes;
    in.sharded = sharded_;
    in.eager = eager_prefetch_;
    // AdamW state, and the split master's low halves, ride every trainable backward claim
    in.optimizer_state = train && (adamw() || split_);
    in.wb_stages = train && stages_dev_ ? n_stages_ : 0;
    // (checkpointing: the D2H engine carries the forward's activation offloads - no deferral;
    // a master shared outside data parallel must be complete when the call returns)
    const bool foreign_writers = shm_ && !comm_;
    in.defer_writeback = train && staged_writeback_ && !cfg_.checkpointing && !foreign_writers;
    if (in.defer_writeback) {
        // Write-backs the next forward absorbs: one per layer it loads (n - S; measured best for
        // rings up to half the model), or, when the forward is mostly compute on resident layers
        // (Standard, wide rings), what fits in its compute time beyond its loads - from a rough
        // model: tensor rate ~1 PFLOP/s bf16, half for tf32, ~20 TFLOP/s for the exact SIMT
        // kernels; ~50 GB/s over the host link. (Measured at C2: Standard 13.0 -> 12.2 ms.)
        const int S = std::min(n_slots_, n_);
        const double rate = tf32_ ? 0.5e15 : bf16_ ? 1.0e15 : 2.0e13;
        const double t_c = static_cast<double>(rows) *
                           (blk_ ? lay_.linear_flops_per_token() + lay_.attn_flops_per_token() : 2.0 * d_ * d_) / rate;
        const double t_load = static_cast<double>(layer_bytes()) / 5.0e10;
        const double t_wb = t_load * (adamw() ? 3.0 : 1.0);
        const double spare = n_ * t_c - (n_ - S) * t_load;  // forward compute beyond its loads
        const int fit = spare > 0 ? static_cast<int>(spare / t_wb) : 0;
        in.defer_budget = std::min(S, std::max(n_ - S, fit));
        if (defer_budget_override_ >= 0) in.defer_budget = defer_budget_override_;  // A/B only
    }
    if (shm_) {
        for (int L = 0; L < n_; ++L) plan_ver_[static_cast<size_t>(L)] = layer_version(L);
        if (foreign_writers)
            for (auto& c : cache_)
                if (c.valid && c.layer >= 0 && plan_ver_[static_cast<size_t>(c.layer)] != cache_ver_[static_cast<size_t>(c.layer)])
                    c.valid = false;
    }
    if (train && fmt == cache_fmt_) {
        in.pending_wb_layers = pending_wb_layers_;
        in.pending_wb_slots = pending_wb_slots_;
    } else {
        flush_writebacks();
    }
    const std::vector<SlotCache> none;
    const std::vector<SlotCache>& initial = fmt == cache_fmt_ ? cache_ : none;
    if (memo_.valid && same_input(in, memo_.in) && same_slots(initial, memo_.initial)) return memo_.plan;
    memo_.valid = false;
    Plan plan = build_plan(in, initial);
    if (plan.pending_conflict && !in.pending_wb_layers.empty()) {
        // A capacity-shrunk ring would drop a deferred write-back: complete them now, then plan
        // from the (unchanged, still valid) slot cache without pending ones.
        flush_writebacks();
        in.pending_wb_layers.clear();
        in.pending_wb_slots.clear();
        plan = build_plan(in, initial);
    }
    if (plan.pending_conflict) throw Error(SP_ERR_INTERNAL, plan.error);
    if (!plan.error.empty()) throw Error(plan.oom ? SP_ERR_OOM : SP_ERR_INVALID, plan.error);
    memo_.in = std::move(in);
    memo_.initial = initial;
    memo_.plan = std::move(plan);
    memo_.valid = true;
    return memo_.plan;
}

void Executor::record_timing(cudaEvent_t ev, cudaStream_t st) {
    if (capturing_) CUDA_OK(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
    else CUDA_OK(cudaEventRecord(ev, st));
}

cudaStream_t Executor::stream_of(OpKind k) const {
    switch (k) {
        case OpKind::H2D: return s_h2d_;
        case OpKind::D2H:
        case OpKind::ActSave: return s_d2h_;
        case OpKind::Update:
        case OpKind::AllGather: return s_upd_;  // every NCCL call on one stream, plan order
        default: return s_comp_;
    }
}

void Executor::gemm(const GemmProblem& g, cudaStream_t st) {
    const bool timed = cfg_.trace >= 2;  // per-GEMM events perturb the stream: opt-in only
    if (timed) {
        while (gemm_ev_.size() < 2 * (gemm_count_ + 1)) {
            cudaEvent_t e;
            CUDA_OK(cudaEventCreate(&e));
            gemm_ev_.push_back(e);
        }
        record_timing(gemm_ev_[2 * gemm_count_], st);
    }
    const cudaError_t e = gemm_bf16(g, st);
    if (e != cudaSuccess) throw Error(SP_ERR_CUDA, std::string("tcgen05 gemm: ") + cudaGetErrorString(e));
    if (timed)
        record_timing(gemm_ev_[2 * gemm_count_ + 1], st);
    ++gemm_count_;
    gemm_flops_ += 2.0 * g.M * static_cast<double>(g.N) * g.K;
    ++kernels_;
}

void Executor::compute_op(const Op& op, bool train, int64_t rows, int fmt) {
    if (blk_) {
        block_compute(op, train, rows, fmt);
        return;
    }
    const int L = op.layer, s = op.slot;
    const size_t act = static_cast<size_t>(rows) * d_;
    const bool ckpt = train && cfg_.checkpointing && cfg_.strategy != SP_STANDARD;
    cudaStream_t st = s_comp_;
    auto ensure_w16 = [&] {
        if (tf32_ || w16_layer_[s] == L) return;  // tf32 multiplies the fp32 master directly
        convert_f32_to_bf16(slot_w32(s), slot_w16(s), static_cast<int64_t>(d_) * d_, st);
        ++kernels_;
        w16_layer_[s] = L;
    };
    if (!train) {
        const float* x_item = cur_x_ + static_cast<size_t>(op.item) * act;
        float* y_item = cur_y_ + static_cast<size_t>(op.item) * act;
        const bool last = L == n_ - 1;
        if (!tc_) {
            const float* in = L == 0 ? x_item : static_cast<const float*>(pp_[(L - 1) % 2]);
            float* out = last ? y_item : static_cast<float*>(pp_[L % 2]);
            exact_forward(in, slot_w32(s), slot_b32(s), relu_[L], out, rows, d_, st);
            ++kernels_;
            return;
        }
        if (L == 0 && bf16_) {
            convert_f32_to_bf16(x_item, xconv_, static_cast<int64_t>(act), st);
            ++kernels_;
        }
        GemmProblem g;
        g.M = static_cast<int>(rows);
        g.N = d_;
        g.K = d_;
        g.A = L == 0 ? (tf32_ ? static_cast<const void*>(x_item) : xconv_) : pp_[(L - 1) % 2];
        g.lda = d_;
        g.B = tf32_ ? static_cast<void*>(slot_w32(s)) : slot_w16(s);
        g.ldb = d_;
        g.b_mn = true;
        g.epilogue = last || tf32_ ? EPI_BIAS_ACT_F32 : EPI_BIAS_ACT_BF16;
        g.out = last ? static_cast<void*>(y_item) : pp_[L % 2];
        g.ldo = d_;
        g.bias = tf32_ ? slot_b32(s) : slot_b16(s);
        g.relu = relu_[L];
        g.tf32 = tf32_;
        gemm(g, st);
        return;
    }
    if (op.pass == 0) {  // training forward: save x_L, produce x_{L+1}
        void* xL = ckpt ? fa_[L % 3] : act_[L];
        const bool last = L == n_ - 1;
        void* out = last ? static_cast<void*>(yout_) : (ckpt ? fa_[(L + 1) % 3] : act_[L + 1]);
        if (L == 0) {
            if (bf16_) {  // (tf32: fp32 activations, copied like the exact path)
                convert_f32_to_bf16(cur_x_, xL, static_cast<int64_t>(act), st);
                ++kernels_;
            } else {
                // an SM copy: a copy-engine D2D here would queue behind the ring's PCIe copies
                void* dst[1] = {xL};
                const void* src[1] = {cur_x_};
                copy_regions(dst, src, 1, static_cast<int64_t>(act * 4), st);
                ++kernels_;
            }
        }
        if (!tc_) {
            exact_forward(static_cast<const float*>(xL), slot_w32(s), slot_b32(s), relu_[L],
                          static_cast<float*>(out), rows, d_, st);
            ++kernels_;
            return;
        }
        ensure_w16();
        GemmProblem g;
        g.M = static_cast<int>(rows);
        g.N = d_;
        g.K = d_;
        g.A = xL;
        g.lda = d_;
        g.B = tf32_ ? static_cast<void*>(slot_w32(s)) : slot_w16(s);
        g.ldb = d_;
        g.b_mn = true;
        g.tf32 = tf32_;
        g.epilogue = last || tf32_ ? EPI_BIAS_ACT_F32 : EPI_BIAS_ACT_BF16;
        g.out = out;
        g.ldo = d_;
        g.bias = slot_b32(s);
        g.relu = relu_[L];
        // ReLU bit mask of x_{L+1}: the backward's dX of layer L+1 gates with it instead of
        // re-reading x_{L+1} (activation offload keeps the tensor gate: no mask buffers then)
        if (!last && relu_[L] && !masks_.empty()) g.mask_out = masks_[static_cast<size_t>(L + 1)];
        gemm(g, st);
        return;
    }
    // backward of layer L: dz_L (gbuf[L%2]) -> dz_{L-1} (gated by layer L-1's ReLU) + dW/db
    void* dz = gbuf_[L % 2];
    void* xL = ckpt ? ba_[s] : act_[L];
    const bool trainable = !frozen_[L];
    if (L > 0) {
        void* out = gbuf_[(L - 1) % 2];
        const bool gate = relu_[L - 1] != 0;
        if (!tc_) {
            exact_backward_dx(static_cast<const float*>(dz), slot_w32(s),
                              gate ? static_cast<const float*>(xL) : nullptr,
                              static_cast<float*>(out), rows, d_, st);
            ++kernels_;
        } else {
            ensure_w16();
            GemmProblem g;
            g.M = static_cast<int>(rows);
            g.N = d_;
            g.K = d_;
            g.A = dz;
            g.lda = d_;
            g.B = tf32_ ? static_cast<void*>(slot_w32(s)) : slot_w16(s);  // W[i][j]: K-major B of dx = dz W^T
            g.ldb = d_;
            g.tf32 = tf32_;
            g.epilogue = tf32_ ? EPI_GATE_F32 : EPI_GATE_BF16;
            g.out = out;
            g.ldo = d_;
            g.gate = xL;
            g.ldg = d_;
            g.relu = gate ? 1 : 0;
            if (gate && !masks_.empty()) g.gate_mask = masks_[static_cast<size_t>(L)];
            gemm(g, st);
        }
    }
    if (!trainable) return;
    float* ws = gws_[L % 2];
    const size_t dd = static_cast<size_t>(d_) * d_;
    if (!tc_) {
        exact_backward_dw(static_cast<const float*>(xL), static_cast<const float*>(dz), ws,
                          ws + dd, rows, d_, st);
        ++kernels_;
        return;
    }
    GemmProblem g;
    g.M = d_;
    g.N = d_;
    g.K = static_cast<int>(rows);
    g.A = xL;  // x_L [r][i]: the M-major A of dW = x^T dz
    g.lda = d_;
    g.a_mn = true;
    g.B = dz;  // dz [r][j]: N-major B
    g.ldb = d_;
    g.b_mn = true;
    g.tf32 = tf32_;
    // One GPU and enough output tiles to fill the SMs: SGD is fused into the dW epilogue
    // (W -= lr*acc on the slot's fp32 master; splits = 1 keeps each element owned by one CTA).
    // Otherwise (too few d x d tiles for the SMs, or data parallel): raw split-K partials,
    // reduced in a fixed order [+ all-reduced] and applied on the update stream.
    const bool fused = dw_fused_;
    g.epilogue = fused ? EPI_SGD_F32 : EPI_F32;
    g.out = fused ? static_cast<void*>(slot_w32(s)) : static_cast<void*>(ws);
    g.ldo = d_;
    g.splits = fused ? 1 : splits_;
    g.split_stride = static_cast<int64_t>(dd);
    g.cta = dw_cta_;  // variant and splits chosen together from the shape (choose_dw)
    g.block_n = dw_bn_;
    g.lr = cur_lr_;
    gemm(g, st);
    if (fused) w16_layer_[s] = -1;
    float* db_parts = ws + (fused ? 0 : static_cast<size_t>(splits_) * dd);
    if (tf32_) colsum_f32(static_cast<const float*>(dz), rows, d_, db_parts, st);
    else colsum_bf16(dz, rows, d_, db_parts, st);
    ++kernels_;
}

void Executor::loss_op(int64_t rows) {
    const int64_t count = rows * d_;
    const float inv_n = 1.0f / static_cast<float>(count * world_);
    const int last = n_ - 1;
    void* g = gbuf_[last % 2];
    if (blk_) {
        block_loss(rows);
    } else if (!tc_) {
        exact_loss_grad(yout_, cur_t_, count, inv_n, relu_[last], static_cast<float*>(g), loss_dev_, s_comp_);
        kernels_ += 2;
    } else {
        loss_blocks_ = tf32_ ? loss_grad_f32(yout_, cur_t_, count, inv_n, relu_[last], static_cast<float*>(g),
                                             loss_parts_, s_comp_)
                             : loss_grad_bf16(yout_, cur_t_, count, inv_n, relu_[last], g, loss_parts_, s_comp_);
        loss_finalize(loss_parts_, loss_blocks_, loss_dev_, s_comp_);
        kernels_ += 2;
    }
    if (comm_) {
        // The loss value is only reported (the gradient above already uses the global count),
        // so its all-reduce joins the other NCCL calls on the update stream, off the critical
        // path; one stream keeps every rank's collectives in the same order.
        CUDA_OK(cudaEventRecord(ev_loss_, s_comp_));
        CUDA_OK(cudaStreamWaitEvent(s_upd_, ev_loss_, 0));
        NCCL_OK(nccl().AllReduce(loss_dev_, loss_dev_, 1, ncclFloat, ncclSum, comm_, s_upd_));
    }
    // (the 4-byte loss is read back after the final join, enqueue_call: a copy here would queue
    // on the D2H copy engine behind the write-backs and stall this stream until they drain)
}

bool Executor::update_op(const Op& op, float lr, bool keep_slot) {
    const int L = op.layer, s = op.slot;
    const size_t dd = static_cast<size_t>(d_) * d_;
    cudaStream_t st = s_upd_;
    float* ws = blk_ ? bgimg_[L % 2] : gws_[L % 2];
    if (adamw() && tc_ && !comm_ && !blk_) {
        // AdamW straight from the partials: dW split-K partials, db column-sum partials
        adamw_reduce(slot_w32(s), slot_m32(s), slot_v32(s), ws, splits_, static_cast<int64_t>(dd),
                     static_cast<int64_t>(dd), adamw_dev_, st);
        adamw_reduce(slot_b32(s), slot_m32(s) + dd, slot_v32(s) + dd, ws + static_cast<size_t>(splits_) * dd,
                     col_chunks_, d_, d_, adamw_dev_, st);
        kernels_ += 2;
        w16_layer_[s] = -1;
        return false;
    }
    if (tc_ && !comm_ && !blk_) {
        // W: updated in the dW epilogue (fused), or here from the split-K partials in a fixed
        // order; bias from the db column-sum partials.
        const size_t db_off = dw_fused_ ? 0 : static_cast<size_t>(splits_) * dd;
        if (!dw_fused_) {
            sgd_reduce(slot_w32(s), ws, splits_, static_cast<int64_t>(dd), static_cast<int64_t>(dd), lr, st);
            kernels_ += 1;
        }
        sgd_reduce(slot_b32(s), ws + db_off, col_chunks_, d_, d_, lr, st);
        kernels_ += 1;
        w16_layer_[s] = -1;
        return false;
    }
    // The full-batch gradient [dW | db] (fp32, the slot's [W | b] layout; a block's gradient
    // image in its parameter layout) in `g`.
    const size_t imgf = img_f();
    float* g = ws;
    bool staged = false;
    // block layers: the split-K dW partials the layer's backward left; summed inside the split
    // update when nothing else reads the image first, else into the image here
    const bool fuse_parts = blk_ && split_ && !comm_;
    if (blk_) {
        bdw_last_[L % 2] = bdw_pending_[L % 2];
        if (!fuse_parts) block_reduce_pending(L % 2, st);
    }
    if (tc_ && !blk_) {
        reduce_partials(ws, splits_, static_cast<int64_t>(dd), static_cast<int64_t>(dd), grad_red_, st);
        reduce_partials(ws + splits_ * dd, col_chunks_, d_, d_, grad_red_ + dd, st);
        kernels_ += 2;
        g = grad_red_;
    }
    if (comm_ && sharded_) {
        // Reduce-scatter: this rank receives the summed gradient of its shard only, applies
        // SGD to that shard of the slot, and (D2H op) writes back just that shard.
        const size_t shard_f = shardA_ / 4;
        float* mine = g + shard_f * static_cast<size_t>(rank_);
        NCCL_OK(nccl().ReduceScatter(g, mine, shard_f, ncclFloat, ncclSum, comm_, st));
        size_t lo = 0, hi = 0;
        shard_range(shardA_, layer_bytes(), lo, hi);
        if (hi > lo) {
            const int64_t count = static_cast<int64_t>((hi - lo) / 4);
            if (adamw())
                adamw_reduce(slot_w32(s) + lo / 4, slot_m32(s) + lo / 4, slot_v32(s) + lo / 4, mine, 1, 0,
                             count, adamw_dev_, st);
            else
                exact_sgd(slot_w32(s) + lo / 4, mine, count, lr, st);
            ++kernels_;
        }
    } else if (split_) {
        // split master: the (all-reduced) logical gradient updates the halves in place
        if (comm_) NCCL_OK(nccl().AllReduce(g, g, imgf, ncclFloat, ncclSum, comm_, st));
        SplitRegions r = split_regions(s);
        if (fuse_parts) {
            for (const DwPartials& p : bdw_pending_[L % 2])
                for (int i = 0; i < r.n; ++i)
                    if (r.off[i] == static_cast<int64_t>(lay_.t[static_cast<size_t>(p.tensor)].off)) {
                        r.parts[i] = p.parts;
                        r.nparts[i] = p.splits;
                    }
            bdw_pending_[L % 2].clear();
        }
        if (op.stage >= 0) {  // also into the write-back stage (same layout): no staging copy
            r.stage_delta = static_cast<int64_t>(stage_ptr(op.stage) - slot_ptr(s));
            r.stage_only = !keep_slot;  // (the slot is not read again: skip its half of the writes)
            staged = true;
        }
        split_update(r, g, adamw() ? slot_m32(s) : nullptr, adamw() ? slot_v32(s) : nullptr, lr, adamw() ? 1 : 0,
                     adamw_dev_, st);
        ++kernels_;
    } else {
        if (comm_) NCCL_OK(nccl().AllReduce(g, g, imgf, ncclFloat, ncclSum, comm_, st));
        if (adamw())  // [W|b], [mW|mb], [vW|vb] are each contiguous
            adamw_reduce(slot_w32(s), slot_m32(s), slot_v32(s), g, 1, 0, static_cast<int64_t>(imgf),
                         adamw_dev_, st);
        else
            exact_sgd(slot_w32(s), g, static_cast<int64_t>(imgf), lr, st);
        ++kernels_;
    }
    w16_layer_[s] = -1;  // the bf16 copy is now stale
    return staged;
}

void Executor::enqueue_op(const Plan& plan, int i, bool train, int n_items, int64_t rows,
                          float lr, int fmt) {
    (void)n_items;
    const Op& op = plan.ops[static_cast<size_t>(i)];
    cudaStream_t st = stream_of(op.kind);
    auto wait = [&](int dep) {
        const Op& d = plan.ops[static_cast<size_t>(dep)];
        if (stream_of(d.kind) == st) return;
        // fault injection for the poison test only: computes stop waiting for their loads
        if (drop_load_edges_ && op.kind == OpKind::Compute && d.kind == OpKind::H2D) return;
        // A compute waits only for the move of its own layer in a multi-layer H2D job
        const int base = move_ev_base_[static_cast<size_t>(dep)];
        if (op.kind == OpKind::Compute && base >= 0) {
            for (size_t j = 0; j + 1 < d.layers.size(); ++j)
                if (d.layers[j] == op.layer && d.slots[j] == op.slot) {
                    CUDA_OK(cudaStreamWaitEvent(st, ev_move_[static_cast<size_t>(base) + j], 0));
                    return;
                }
        }
        CUDA_OK(cudaStreamWaitEvent(st, ev_dep_[static_cast<size_t>(dep)], 0));
    };
    // Eager H2D: each moved layer waits for its own slot just before its copy (deps is then
    // exactly the union of move_deps); otherwise everything up front (policy trigger).
    const bool per_move = per_move_ && op.kind == OpKind::H2D && eager_prefetch_ && !op.move_deps.empty();
    if (!per_move)
        for (int dep : op.deps) wait(dep);
    // Timing events are "external" so that, under graph capture, they become event-record
    // nodes; the dependency events (ev_dep_) become graph edges.
    // (per-move H2D: the start is taken once the first copy's own waits are satisfied)
    if (cfg_.trace >= 1 && !per_move) record_timing(ev_start_[static_cast<size_t>(i)], st);
    const size_t act_b = static_cast<size_t>(rows) * d_ * act_elt();
    switch (op.kind) {
        case OpKind::H2D:
            for (size_t j = 0; j < op.layers.size(); ++j) {
                const int L = op.layers[j], s = op.slots[j];
                if (per_move) {
                    for (int dep : op.move_deps[j]) wait(dep);
                    if (j == 0 && cfg_.trace >= 1) record_timing(ev_start_[static_cast<size_t>(i)], st);
                }
                if (op.weights[j] && split_) {
                    // the split master's wire prefix: the bf16 operands (forward, backward, inference)
                    uint8_t* dst = slot_ptr(s);
                    if (poison_) CUDA_OK(cudaMemsetAsync(dst, 0xFF, layer_bytes(), st));
                    CUDA_OK(cudaMemcpyAsync(dst, host_layer(L), lay_.wire_bytes, cudaMemcpyHostToDevice, st));
                    h2d_bytes_ += lay_.wire_bytes;
                } else if (op.weights[j]) {
                    // Whole image, or (sharded) only this rank's [lo, hi) byte range of it.
                    const bool wire = fmt == kFmtBf16Infer;
                    const size_t img = wire ? wire16_bytes() : layer_bytes();
                    size_t lo = 0, hi = img;
                    if (sharded_) shard_range(wire ? shardB_ : shardA_, img, lo, hi);
                    const uint8_t* src = wire ? host16_ + static_cast<size_t>(L) * wire16_bytes() : host_layer(L);
                    uint8_t* dst = wire ? slot_ptr(s) + off_w16_ : slot_ptr(s);
                    // Debug (SP_POISON=1): NaN-fill the whole image first, so a compute that
                    // reads the slot before this copy lands (a missing edge) produces NaNs.
                    if (poison_) CUDA_OK(cudaMemsetAsync(dst, 0xFF, img, st));
                    if (hi > lo)
                        CUDA_OK(cudaMemcpyAsync(dst + lo, src + lo, hi - lo, cudaMemcpyHostToDevice, st));
                    h2d_bytes_ += hi - lo;
                    if (!wire) w16_layer_[s] = -1;
                }
                if (op.acts[j]) {
                    if (poison_) CUDA_OK(cudaMemsetAsync(ba_[s], 0xFF, act_b, st));
                    CUDA_OK(cudaMemcpyAsync(ba_[s], host_act_ + static_cast<size_t>(L) * act_b, act_b,
                                            cudaMemcpyHostToDevice, st));
                    h2d_bytes_ += act_b;
                }
                if (j < op.opts.size() && op.opts[j] && split_) {
                    // the low halves the update needs (whether or not the prefix was a hit)
                    CUDA_OK(cudaMemcpyAsync(slot_ptr(s) + lay_.wire_bytes, host_layer(L) + lay_.wire_bytes,
                                            lay_.lo_bytes, cudaMemcpyHostToDevice, st));
                    h2d_bytes_ += lay_.lo_bytes;
                }
                if (j < op.opts.size() && op.opts[j] && adamw()) {  // AdamW m, v (sharded: this rank's shard)
                    size_t lo = 0, hi = opt_bytes();
                    if (sharded_) shard_range(shardA_, opt_bytes(), lo, hi);
                    if (hi > lo) {
                        CUDA_OK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(slot_m32(s)) + lo,
                                                reinterpret_cast<const uint8_t*>(host_opt(host_m_, L)) + lo, hi - lo,
                                                cudaMemcpyHostToDevice, st));
                        CUDA_OK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(slot_v32(s)) + lo,
                                                reinterpret_cast<const uint8_t*>(host_opt(host_v_, L)) + lo, hi - lo,
                                                cudaMemcpyHostToDevice, st));
                    }
                    h2d_bytes_ += 2 * (hi - lo);
                }
                const int base = move_ev_base_[static_cast<size_t>(i)];
                if (base >= 0 && j + 1 < op.layers.size())  // this layer has landed
                    CUDA_OK(cudaEventRecord(ev_move_[static_cast<size_t>(base) + j], st));
            }
            break;
        case OpKind::Compute:
            compute_op(op, train, rows, fmt);
            break;
        case OpKind::Loss:
            loss_op(rows);
            break;
        case OpKind::Update:
            {
                const SlotCache& fin = plan.final_slots[static_cast<size_t>(op.slot)];
                if (update_op(op, lr, fin.valid && fin.layer == op.layer)) {
                    // the slot kept the pre-update values: it must not count as this layer's
                    // current weights (the plan already leaves it invalid or another layer's)
                    break;
                }
            }
            if (op.stage >= 0) {  // copy the updated image [+ m, v] out: the slot is free now
                size_t lo = 0, hi = layer_bytes();
                if (sharded_) shard_range(shardA_, layer_bytes(), lo, hi);
                uint8_t* stage = stage_ptr(op.stage);
                const uint8_t* slot = slot_ptr(op.slot);
                if (hi > lo && split_) {  // split master: its image, and the moments (own size)
                    void* dst[1] = {stage};
                    const void* src[1] = {slot};
                    copy_regions(dst, src, 1, static_cast<int64_t>(layer_bytes()), st);
                    ++kernels_;
                    if (adamw()) {
                        void* dm[2] = {stage + off_m_, stage + off_v_};
                        const void* sm[2] = {slot + off_m_, slot + off_v_};
                        copy_regions(dm, sm, 2, static_cast<int64_t>(opt_bytes()), st);
                        ++kernels_;
                    }
                } else if (hi > lo) {  // an SM kernel: copy engines stay with the PCIe transfers
                    void* dst[3] = {stage + lo, stage + off_m_ + lo, stage + off_v_ + lo};
                    const void* src[3] = {slot + lo, slot + off_m_ + lo, slot + off_v_ + lo};
                    copy_regions(dst, src, adamw() ? 3 : 1, static_cast<int64_t>(hi - lo), st);
                    ++kernels_;
                }
            }
            break;
        case OpKind::D2H: {
            // Updated fp32 master back to the pinned host copy (sharded: this rank's shard only;
            // every rank streams exactly that shard in later calls, so its copy stays
            // authoritative for it).
            // From the write-back stage the Update filled, or (deferred write-back of the
            // previous call, unstaged plans) straight from the slot.
            const int L = op.layers[0], s = op.slots[0];
            host16_stale_[L] = 1;
            if (op.deferred) break;  // done at the start of the next call (or a flush)
            size_t lo = 0, hi = layer_bytes();
            if (sharded_) shard_range(shardA_, layer_bytes(), lo, hi);
            const uint8_t* src = op.stage >= 0 ? stage_ptr(op.stage) : slot_ptr(s);
            if (hi > lo)
                CUDA_OK(cudaMemcpyAsync(host_layer(L) + lo, src + lo, hi - lo, cudaMemcpyDeviceToHost, st));
            d2h_bytes_ += hi - lo;
            size_t mlo = 0, mhi = opt_bytes();
            if (sharded_) shard_range(shardA_, opt_bytes(), mlo, mhi);
            if (adamw() && mhi > mlo) {  // the optimizer state rides the write-back
                CUDA_OK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(host_opt(host_m_, L)) + mlo, src + off_m_ + mlo,
                                        mhi - mlo, cudaMemcpyDeviceToHost, st));
                CUDA_OK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(host_opt(host_v_, L)) + mlo, src + off_v_ + mlo,
                                        mhi - mlo, cudaMemcpyDeviceToHost, st));
                d2h_bytes_ += 2 * (mhi - mlo);
            }
            break;
        }
        case OpKind::AllGather:
            for (size_t j = 0; j < op.layers.size(); ++j) {
                const int s = op.slots[j];
                const bool wire = fmt == kFmtBf16Infer;
                uint8_t* base = wire ? slot_ptr(s) + off_w16_ : slot_ptr(s);
                const size_t shard = wire ? shardB_ : shardA_;
                NCCL_OK(nccl().AllGather(base + shard * static_cast<size_t>(rank_), base, shard,
                                         ncclUint8, comm_, st));
                if (!wire) w16_layer_[s] = -1;
            }
            break;
        case OpKind::ActSave:
            CUDA_OK(cudaMemcpyAsync(host_act_ + static_cast<size_t>(op.layer) * act_b, fa_[op.layer % 3],
                                    act_b, cudaMemcpyDeviceToHost, st));
            d2h_bytes_ += act_b;
            break;
    }
    if (cfg_.trace >= 1) record_timing(ev_done_[static_cast<size_t>(i)], st);
    if (cross_dep_[static_cast<size_t>(i)]) CUDA_OK(cudaEventRecord(ev_dep_[static_cast<size_t>(i)], st));
}

// Everything one call puts on the device, from the timing base to the final join: the input
// copies, every op of the plan, the output copy. Enqueued eagerly or captured into a graph.
void Executor::enqueue_call(const Plan& plan, const CallIO& io) {
    // Dependency events only where another stream waits on the op (every event record on
    // the compute stream costs device time between kernels).
    cross_dep_.assign(plan.ops.size(), 0);
    for (size_t j = 0; j < plan.ops.size(); ++j)
        for (int dep : plan.ops[j].deps)
            if (stream_of(plan.ops[static_cast<size_t>(dep)].kind) != stream_of(plan.ops[j].kind))
                cross_dep_[static_cast<size_t>(dep)] = 1;
    move_ev_base_.assign(plan.ops.size(), -1);
    size_t moves = 0;
    for (size_t j = 0; j < plan.ops.size() && move_events_; ++j)
        if (plan.ops[j].kind == OpKind::H2D && plan.ops[j].layers.size() > 1) {
            move_ev_base_[j] = static_cast<int>(moves);
            moves += plan.ops[j].layers.size() - 1;
        }
    while (ev_move_.size() < moves) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev_move_.push_back(e);
    }
    record_timing(ev_call0_, s_h2d_);
    CUDA_OK(cudaEventRecord(ev_fork_, s_h2d_));
    for (auto s : {s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamWaitEvent(s, ev_fork_, 0));
    if (io.train && adamw())  // this step's AdamW scalars: read at execution, so replays stay valid
        CUDA_OK(cudaMemcpyAsync(adamw_dev_, adamw_host_, sizeof(AdamwScalars), cudaMemcpyHostToDevice, s_upd_));
    const size_t act = static_cast<size_t>(io.rows) * d_ * 4;
    if (!io.device_io) {
        CUDA_OK(cudaMemcpyAsync(xin_, io.x, act * (io.train ? 1 : io.n_items), cudaMemcpyHostToDevice, s_comp_));
        if (io.train) CUDA_OK(cudaMemcpyAsync(tgt_, io.t, act, cudaMemcpyHostToDevice, s_comp_));
    }
    // NVTX: one range per plan op ("H2D L3 s1", "COMP L3 bwd", ...). With CUDA graphs on they
    // annotate the capture on the host timeline; with graphs off (sp_debug_set "graphs" 0) nsys
    // projects them onto the GPU work of each stream (overlap evidence).
    static const char* kKind[] = {"H2D", "COMP", "D2H", "LOSS", "UPD", "ACT", "GATHER"};
    char label[64];
    for (size_t i = 0; i < plan.ops.size(); ++i) {
        const Op& op = plan.ops[i];
        const int L = op.layer >= 0 ? op.layer : (op.layers.empty() ? -1 : op.layers[0]);
        std::snprintf(label, sizeof(label), "%s L%d s%d%s", kKind[static_cast<int>(op.kind)], L,
                      op.slot >= 0 ? op.slot : (op.slots.empty() ? -1 : op.slots[0]), op.pass == 1 ? " bwd" : "");
        nvtxRangePushA(label);
        enqueue_op(plan, static_cast<int>(i), io.train, io.n_items, io.rows, io.lr, io.fmt);
        nvtxRangePop();
    }
    if (!io.device_io && !io.train) {
        CUDA_OK(cudaEventRecord(ev_io_out_, s_comp_));
        CUDA_OK(cudaStreamWaitEvent(s_d2h_, ev_io_out_, 0));
        CUDA_OK(cudaMemcpyAsync(io.y, yout_, act * io.n_items, cudaMemcpyDeviceToHost, s_d2h_));
    }
    int k = 0;
    for (auto s : {s_comp_, s_d2h_, s_upd_}) {
        CUDA_OK(cudaEventRecord(ev_join_[k], s));
        CUDA_OK(cudaStreamWaitEvent(s_h2d_, ev_join_[k], 0));
        ++k;
    }
    if (io.train) CUDA_OK(cudaMemcpyAsync(loss_host_, loss_dev_, 4, cudaMemcpyDeviceToHost, s_h2d_));
    record_timing(ev_call1_, s_h2d_);  // all streams joined: the call's device makespan
}

namespace {
bool pinned_or_null(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice ||
           a.type == cudaMemoryTypeManaged;
}
}  // namespace

uint64_t Executor::call_signature(const Plan& plan, const CallIO& io) const {
    uint64_t h = 0xCBF29CE484222325ull;
    auto mix = [&](uint64_t v) {  // word-wise multiply-xorshift (host time per call matters)
        h = (h ^ v) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
    };
    for (const Op& op : plan.ops) {
        mix(static_cast<uint64_t>(op.kind) | static_cast<uint64_t>(op.pass) << 8 |
            static_cast<uint64_t>(static_cast<uint32_t>(op.layer)) << 16 |
            static_cast<uint64_t>(static_cast<uint32_t>(op.slot)) << 40);
        mix(static_cast<uint64_t>(static_cast<uint32_t>(op.item)));
        for (size_t j = 0; j < op.layers.size(); ++j)
            mix(static_cast<uint64_t>(op.layers[j]) << 32 | static_cast<uint32_t>(op.slots[j]) |
                static_cast<uint64_t>(op.weights[j]) << 62 | static_cast<uint64_t>(op.acts[j]) << 63);
        for (int dep : op.deps) mix(static_cast<uint64_t>(dep) | 1ull << 60);
        mix(static_cast<uint64_t>(static_cast<uint32_t>(op.stage)) | static_cast<uint64_t>(op.deferred) << 40);
    }
    uint32_t lr_bits;
    std::memcpy(&lr_bits, &io.lr, 4);
    mix(static_cast<uint64_t>(io.train) | static_cast<uint64_t>(io.device_io) << 1 |
        static_cast<uint64_t>(io.fmt) << 2 | static_cast<uint64_t>(lr_bits) << 32);
    mix(static_cast<uint64_t>(io.rows));
    mix(static_cast<uint64_t>(io.n_items));
    mix(reinterpret_cast<uintptr_t>(io.x));
    mix(reinterpret_cast<uintptr_t>(io.t));
    mix(reinterpret_cast<uintptr_t>(io.y));
    for (int v : w16_layer_) mix(static_cast<uint64_t>(static_cast<uint32_t>(v)));
    for (int L = 0; L < n_; ++L)  // activations are baked into the captured kernels
        mix(static_cast<uint64_t>(relu_[static_cast<size_t>(L)] != 0) | static_cast<uint64_t>(L) << 1);
    mix(static_cast<uint64_t>(splits_) | static_cast<uint64_t>(col_chunks_) << 32);
    mix(reinterpret_cast<uintptr_t>(comm_));
    mix(alloc_gen_);
    mix(static_cast<uint64_t>(cfg_.trace));
    return h;
}

void Executor::run_call(const Plan& plan, const CallIO& io) {
    launched_ = false;
    nvtxRangePushA(io.train ? "sp_train_step" : "sp_forward");
    struct PopRange {
        ~PopRange() { nvtxRangePop(); }
    } pop_range;
    try {
        run_call_impl(plan, io);
    } catch (...) {
        if (!launched_) {
            // Nothing reached the device (capture / instantiation failed): the ring still
            // holds the previous step's deferred updates - complete them before giving up.
            try {
                flush_writebacks();
            } catch (...) {
                if (io.train || !pending_wb_layers_.empty()) mark_inconsistent();
            }
        } else if (io.train) {
            // Part of the step may have run: some layers updated and written back, others
            // not, and deferred updates possibly overwritten. The host master is no longer
            // one consistent model; every later call refuses until the layers are registered
            // again (SP_ERR_STATE) instead of silently training a mixed model.
            mark_inconsistent();
        }
        // A failed call may have overwritten ring slots part-way: nothing cached on the device
        // can be trusted by the next call (the host master copy is the source of truth).
        for (auto& c : cache_) c.valid = false;
        std::fill(w16_layer_.begin(), w16_layer_.end(), -1);
        pending_wb_layers_.clear();
        pending_wb_slots_.clear();
        throw;
    }
}

// Debug / A/B knobs (include/superpipe_debug.h sp_debug_set): never set on the product path.
void Executor::set_debug(const std::string& key, int value) {
    flush_writebacks();
    if (key == "staged_writeback") staged_writeback_ = value != 0;
    else if (key == "poison") poison_ = value != 0;
    else if (key == "drop_load_edges") drop_load_edges_ = value != 0;
    else if (key == "graphs") use_graphs_ = value != 0;
    else if (key == "wb_stages") wb_stages_cap_ = std::max(1, value);
    else if (key == "defer_budget") defer_budget_override_ = value;
    else if (key == "per_move") per_move_ = value != 0;
    else if (key == "move_events") move_events_ = value != 0;
    else throw Error(SP_ERR_INVALID, "sp_debug_set: unknown key " + key);
    if (stages_dev_) {  // re-sized (or dropped) on the next training call
        CUDA_OK(cudaDeviceSynchronize());
        cudaFree(stages_dev_);
        stages_dev_ = nullptr;
        n_stages_ = 0;
    }
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
    graphs_.clear();
}

void Executor::mark_inconsistent() {
    for (int L = 0; L < n_; ++L)
        if (!frozen_[static_cast<size_t>(L)]) inconsistent_[static_cast<size_t>(L)] = 1;
}

void Executor::run_call_impl(const Plan& plan, const CallIO& io) {
    const size_t need = plan.ops.size();
    while (ev_done_.size() < need) {
        cudaEvent_t a, b, c;
        CUDA_OK(cudaEventCreate(&a));
        CUDA_OK(cudaEventCreate(&b));
        CUDA_OK(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
        ev_done_.push_back(a);
        ev_start_.push_back(b);
        ev_dep_.push_back(c);
    }
    const bool graphable = use_graphs_ && (io.device_io || (pinned_or_null(io.x) &&
                                                            pinned_or_null(io.t) &&
                                                            pinned_or_null(io.y)));
    if (!graphable) {
        launched_ = true;  // eager: ops reach the device as they are enqueued
        enqueue_call(plan, io);
    } else {
        const uint64_t sig = call_signature(plan, io);
        auto it = graphs_.find(sig);
        if (it != graphs_.end()) {
            // Replay: one launch for the whole step; re-apply the host-side effects the
            // captured enqueue had (bf16-copy tracking, stale inference wire, counters).
            const GraphEntry& g = it->second;
            launched_ = true;
            CUDA_OK(cudaGraphLaunch(g.exec, s_h2d_));
            w16_layer_ = g.w16_after;
            for (int L : g.stale_layers) host16_stale_[static_cast<size_t>(L)] = 1;
            kernels_ = g.kernels;
            h2d_bytes_ = g.h2d_bytes;
            d2h_bytes_ = g.d2h_bytes;
            gemm_count_ = g.gemm_count;
            gemm_flops_ = g.gemm_flops;
            attn_launches_ = g.attn_launches;
            attn_flops_ = g.attn_flops;
            ++graph_replays_;
        } else {
            if (graphs_.size() >= 16) {
                for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
                graphs_.clear();
            }
            CUDA_OK(cudaStreamBeginCapture(s_h2d_, cudaStreamCaptureModeThreadLocal));
            capturing_ = true;
            try {
                enqueue_call(plan, io);
            } catch (...) {
                capturing_ = false;
                cudaGraph_t broken = nullptr;
                cudaStreamEndCapture(s_h2d_, &broken);
                if (broken) cudaGraphDestroy(broken);
                cudaGetLastError();
                throw;
            }
            capturing_ = false;
            cudaGraph_t graph = nullptr;
            CUDA_OK(cudaStreamEndCapture(s_h2d_, &graph));
            GraphEntry g;
            const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
            cudaGraphDestroy(graph);
            CUDA_OK(ie);
            g.w16_after = w16_layer_;
            for (const Op& op : plan.ops)
                if (op.kind == OpKind::D2H) g.stale_layers.push_back(op.layers[0]);
            g.kernels = kernels_;
            g.h2d_bytes = h2d_bytes_;
            g.d2h_bytes = d2h_bytes_;
            g.gemm_count = gemm_count_;
            g.gemm_flops = gemm_flops_;
            g.attn_launches = attn_launches_;
            g.attn_flops = attn_flops_;
            launched_ = true;
            CUDA_OK(cudaGraphLaunch(g.exec, s_h2d_));
            graphs_.emplace(sig, std::move(g));
        }
    }
    cache_ = plan.final_slots;
    cache_fmt_ = io.fmt;
    // this call ran the previous call's deferred write-backs and leaves its own
    pending_wb_layers_ = plan.deferred_layers;
    pending_wb_slots_ = plan.deferred_slots;
}

void Executor::collect_stats(const Plan& plan, int n_items, bool train) {
    trace_.clear();
    double first_c = -1, last_c = 0, makespan = 0, stall = 0, comp = 0, prev_end = -1;
    {
        float call = 0;
        CUDA_OK(cudaEventElapsedTime(&call, ev_call0_, ev_call1_));
        makespan = call;
    }
    const size_t timed_ops = cfg_.trace >= 1 ? plan.ops.size() : 0;
    for (size_t i = 0; i < timed_ops; ++i) {
        const Op& op = plan.ops[i];
        float t0 = 0, t1 = 0;
        CUDA_OK(cudaEventElapsedTime(&t0, ev_call0_, ev_start_[i]));
        CUDA_OK(cudaEventElapsedTime(&t1, ev_call0_, ev_done_[i]));
        sp_trace_event ev{};
        ev.op_index = static_cast<int32_t>(i);
        ev.t_start = t0;
        ev.t_end = t1;
        ev.item = op.item;
        ev.layer = op.layer;
        ev.backward = op.pass == 1;
        if (op.kind == OpKind::Compute || op.kind == OpKind::Loss) {
            if (op.kind == OpKind::Compute) {
                if (first_c < 0) first_c = t0;
                last_c = std::max(last_c, static_cast<double>(t1));
                comp += t1 - t0;
            }
            if (prev_end >= 0 && t0 > prev_end) {
                sp_trace_event s{};
                s.op_index = -1;
                s.t_start = prev_end;
                s.t_end = t0;
                s.kind = 3;
                s.layer = op.layer;
                s.backward = op.pass == 1;
                stall += t0 - prev_end;
                trace_.push_back(s);
            }
            prev_end = t1;
            if (op.kind == OpKind::Loss) continue;
            ev.kind = 0;
        } else if (op.kind == OpKind::H2D || op.kind == OpKind::D2H || op.kind == OpKind::ActSave) {
            ev.kind = op.kind == OpKind::H2D ? 1 : 2;
            if (!op.layers.empty()) {
                ev.first_layer = op.layers[0];
                ev.n_layers_moved = static_cast<int>(op.layers.size());
                for (size_t j = 0; j < op.layers.size(); ++j) {
                    if (op.weights[j]) ev.weight_bytes += layer_bytes();
                    if (op.acts[j]) ev.activation_bytes += static_cast<uint64_t>(cap_rows_) * d_ * 4;
                }
            } else {
                ev.first_layer = op.layer;
                ev.n_layers_moved = 0;
            }
        } else {
            continue;
        }
        trace_.push_back(ev);
    }
    last_plan_ = plan;
    stats_.peak_bytes = plan.ledger.peak_bytes;
    stats_.peak_weight_bytes = plan.ledger.peak_weight;
    stats_.peak_activation_bytes = plan.ledger.peak_activation;
    stats_.peak_gradient_bytes = plan.ledger.peak_gradient;
    stats_.total_gradient_bytes = plan.ledger.total_gradient;
    stats_.n_transfers_h2d = plan.n_h2d_jobs;
    stats_.n_transfers_d2h = plan.n_d2h_jobs + plan.d2h_act_layers;
    stats_.n_evictions = plan.n_evictions;
    stats_.h2d_bytes = h2d_bytes_;
    stats_.d2h_bytes = d2h_bytes_;
    stats_.hbm_reserved_bytes = static_cast<uint64_t>(n_slots_) * slot_bytes_ + dev_bytes_;
    stats_.kernels_launched = kernels_;
    stats_.per_item_ms = first_c >= 0 ? (last_c - first_c) / std::max(1, train ? 1 : n_items) : 0.0;
    stats_.makespan_ms = makespan;
    stats_.stall_ms = stall;
    stats_.compute_ms = comp;
    stats_.n_slots = plan.n_slots;
    stats_.host_enqueue_ms = host_enqueue_ms_;
    stats_.graph_replays = graph_replays_;
    stats_.gemm_launches = gemm_count_;
    stats_.gemm_flops = gemm_flops_;
    stats_.gemm_ms = 0.0;
    stats_.attn_launches = attn_launches_;
    stats_.attn_flops = attn_flops_;
    if (cfg_.trace >= 2)
        for (size_t g = 0; g < gemm_count_; ++g) {
            float ms = 0;
            CUDA_OK(cudaEventElapsedTime(&ms, gemm_ev_[2 * g], gemm_ev_[2 * g + 1]));
            stats_.gemm_ms += ms;
        }
}

void Executor::forward(const float* x, int64_t rows, int n_items, float* y, bool device_io) {
    if (!x || !y) throw Error(SP_ERR_INVALID, "run_inference: null input or output");
    if (rows < 1 || n_items < 1) throw Error(SP_ERR_INVALID, "run_inference: no inputs");
    if (rows > (1ll << 31) - 1) throw Error(SP_ERR_INVALID, "run_inference: too many rows");
    check_ready();
    flush_writebacks();  // inference reads the host master (and re-streams every layer)
    if (item_batching_ && n_items > 1 && rows * n_items <= (1ll << 31) - 1) {
        // [items][rows][d] is contiguous, i.e. one [items*rows][d] input: one pass over the
        // ring serves every item (row-independent math, so outputs are unchanged).
        rows *= n_items;
        n_items = 1;
    }
    const int fmt = bf16_ ? kFmtBf16Infer : kFmtExactF32;
    // The bf16 wire image is derived from the whole fp32 master; its shards do not line up
    // with the fp32 shards, so it needs every element current on this rank.
    if (bf16_) require_full_host(-1, "run_inference");
    const Plan& plan = make_plan(false, n_items, rows, fmt);
    refresh_host16();
    ensure_buffers(rows, n_items, false, device_io);
    CUDA_OK(cudaSetDevice(cfg_.device));
    reset_call_counters();
    cur_x_ = device_io ? x : xin_;
    cur_y_ = device_io ? y : yout_;
    CallIO io{false, n_items, rows, 0.0f, fmt, device_io, x, nullptr, y};
    const auto t0 = std::chrono::steady_clock::now();
    run_call(plan, io);
    host_enqueue_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    CUDA_OK(cudaStreamSynchronize(s_h2d_));  // every stream joined into s_h2d_ (enqueue_call)
    CUDA_OK(cudaGetLastError());
    after_call(plan);
    collect_stats(plan, n_items, false);
    stats_.loss = 0.0f;
    std::memset(stats_.digest, 0, sizeof(stats_.digest));  // on demand: sp_digest_tensors(y)
}

float Executor::train_step(const float* x, const float* target, int64_t rows, float lr,
                           bool device_io) {
    if (!x || !target) throw Error(SP_ERR_INVALID, "run_train_step: null input or target");
    if (!(lr > 0.0f)) throw Error(SP_ERR_INVALID, "train: lr must be > 0");
    if (rows < 1) throw Error(SP_ERR_INVALID, "train: batch_size must be >= 1");
    check_ready();
    const int fmt = bf16_ ? kFmtBf16Train : kFmtExactF32;
    CUDA_OK(cudaSetDevice(cfg_.device));
    ensure_stages();
    const Plan& plan = make_plan(true, 1, rows, fmt);
    ensure_buffers(rows, 1, true, device_io);
    CUDA_OK(cudaSetDevice(cfg_.device));
    if (blk_ && rows % lay_.desc.seq_len != 0)
        throw Error(SP_ERR_INVALID, "train: rows must be a multiple of the block's seq_len");
    if (infer_only_)
        throw Error(SP_ERR_INVALID, "train: this executor was created SP_BLOCK_INFER_ONLY (no fp32 master)");
    if (blk_ && lay_.swiglu())
        throw Error(SP_ERR_INVALID, "train: SwiGLU blocks are inference-only in this build");
    if (tc_ && !blk_) {  // split-K depends only on (d, rows): identical for every window setting
        const DwChoice c = choose_dw(d_, d_, static_cast<int>(rows), splits_cap_, comm_ == nullptr, tf32_);
        splits_ = c.splits;
        dw_cta_ = c.cta;
        dw_bn_ = c.block_n;
        col_chunks_ = colsum_chunks(rows);
        dw_fused_ = comm_ == nullptr && splits_ == 1 && !adamw();
    }
    reset_call_counters();
    cur_x_ = device_io ? x : xin_;
    cur_t_ = device_io ? target : tgt_;
    if (cache_fmt_ != fmt) std::fill(w16_layer_.begin(), w16_layer_.end(), -1);
    cur_lr_ = lr;
    if (adamw()) {  // PyTorch's scalars: computed in double, rounded to float once (orc_adamw)
        ++step_t_;
        const double t = static_cast<double>(step_t_);
        AdamwScalars& a = *adamw_host_;
        a.decay = static_cast<float>(1.0 - static_cast<double>(lr) * wd_);
        a.omb1 = static_cast<float>(1.0 - beta1_);
        a.b2 = static_cast<float>(beta2_);
        a.omb2 = static_cast<float>(1.0 - beta2_);
        a.bc2_sqrt = static_cast<float>(std::sqrt(1.0 - std::pow(beta2_, t)));
        a.eps = static_cast<float>(eps_);
        a.neg_step = static_cast<float>(-static_cast<double>(lr) / (1.0 - std::pow(beta1_, t)));
        a.pad = 0.0f;
    }
    CallIO io{true, 1, rows, lr, fmt, device_io, x, target, nullptr};
    const auto t0 = std::chrono::steady_clock::now();
    try {
        run_call(plan, io);
    } catch (...) {
        if (adamw()) --step_t_;  // no update was applied for this step
        throw;
    }
    host_enqueue_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (auto s : {s_h2d_, s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamSynchronize(s));
    CUDA_OK(cudaGetLastError());
    after_call(plan);
    collect_stats(plan, 1, true);
    if (sharded_)
        for (int L = 0; L < n_; ++L)
            if (!frozen_[static_cast<size_t>(L)]) host_partial_[static_cast<size_t>(L)] = 1;
    const float loss = loss_host_[0] / static_cast<float>(rows * d_ * world_);
    stats_.loss = loss;
    std::memset(stats_.digest, 0, sizeof(stats_.digest));  // on demand: digest_train()
    return loss;
}

void Executor::digest_train(float loss, char out[17]) {
    flush_writebacks();
    require_full_host(-1, "digest_train");
    // digest_train (engine.cpp:574-581): loss bytes, then each block's W and b — the host
    // master copy is [W_0 b_0 W_1 b_1 ...] contiguous, exactly the reference's byte order.
    uint64_t h = 0xCBF29CE484222325ull;
    auto fnv = [&](const void* p, size_t n) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) {
            h ^= c[i];
            h *= 0x100000001B3ull;
        }
    };
    fnv(&loss, 4);
    if (split_) {  // hash the fp32 images, as the reference's digest_train does
        std::vector<float> img(img_f());
        for (int L = 0; L < n_; ++L) {
            unsplit_image(host_layer(L), img.data());
            fnv(img.data(), img.size() * 4);
        }
    } else {
        fnv(host32_, static_cast<size_t>(n_) * host_stride_);
    }
    static const char digits[] = "0123456789abcdef";
    for (int i = 15; i >= 0; --i) {
        out[i] = digits[h & 0xF];
        h >>= 4;
    }
    out[16] = '\0';
}

void Executor::read_layer(int index, float* W, float* b) {
    if (index < 0 || index >= n_) throw Error(SP_ERR_INVALID, "read_layer: index out of range");
    if (blk_) throw Error(SP_ERR_INVALID, "read_layer: this executor streams transformer blocks (sp_read_block)");
    flush_writebacks();
    require_full_host(index, "read_layer");
    const size_t dd = static_cast<size_t>(d_) * d_;
    const float* src = host32_ + static_cast<size_t>(index) * (dd + d_);
    if (W) std::memcpy(W, src, dd * 4);
    if (b) std::memcpy(b, src + dd, static_cast<size_t>(d_) * 4);
}

// Host conversions between a block's fp32 image and its split image, over host threads (a
// Llama-3-70B-shape layer holds 856M parameters).
void Executor::split_image(const float* params, uint8_t* dst) const {
    for (const BlockTensor& t : lay_.t) {
        const float* src = params + t.off;
        if (!t.matrix) {
            std::memcpy(dst + t.wire_off, src, t.count() * 4);
            continue;
        }
        uint16_t* hi = reinterpret_cast<uint16_t*>(dst + t.wire_off);
        uint16_t* lo = infer_only_ ? nullptr : reinterpret_cast<uint16_t*>(dst + lay_.wire_bytes + t.lo_off);
        const uint64_t n = t.count(), chunk = 1 << 20;
        parallel_for(static_cast<int>((n + chunk - 1) / chunk), [&](int c) {
            const uint64_t e1 = std::min<uint64_t>(n, (static_cast<uint64_t>(c) + 1) * chunk);
            for (uint64_t e = static_cast<uint64_t>(c) * chunk; e < e1; ++e) {
                uint32_t u;
                std::memcpy(&u, src + e, 4);
                hi[e] = static_cast<uint16_t>(u >> 16);
                if (lo) lo[e] = static_cast<uint16_t>(u & 0xFFFFu);
            }
        });
    }
}

void Executor::unsplit_image(const uint8_t* src, float* params) const {
    std::memset(params, 0, img_f() * 4);
    for (const BlockTensor& t : lay_.t) {
        float* out = params + t.off;
        if (!t.matrix) {
            std::memcpy(out, src + t.wire_off, t.count() * 4);
            continue;
        }
        const uint16_t* hi = reinterpret_cast<const uint16_t*>(src + t.wire_off);
        const uint16_t* lo = infer_only_ ? nullptr : reinterpret_cast<const uint16_t*>(src + lay_.wire_bytes + t.lo_off);
        const uint64_t n = t.count(), chunk = 1 << 20;
        parallel_for(static_cast<int>((n + chunk - 1) / chunk), [&](int c) {
            const uint64_t e1 = std::min<uint64_t>(n, (static_cast<uint64_t>(c) + 1) * chunk);
            for (uint64_t e = static_cast<uint64_t>(c) * chunk; e < e1; ++e) {
                const uint32_t u = static_cast<uint32_t>(hi[e]) << 16 | (lo ? lo[e] : 0u);
                std::memcpy(out + e, &u, 4);
            }
        });
    }
}

// Switches a block master between the split image and the plain fp32 image (host side; the
// slots are re-laid out by the caller).
void Executor::set_split(bool on) {
    if (split_ == on || !blk_) return;
    if (infer_only_) return;  // inference replicas never shard: the wire image stays
    flush_writebacks();
    CUDA_OK(cudaSetDevice(cfg_.device));
    for (auto st : {s_h2d_, s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamSynchronize(st));
    if (!shm_ || shm_owner_) {
        std::vector<float> img(img_f());
        std::vector<uint8_t> tmp(host_stride_);
        for (int L = 0; L < n_; ++L) {
            if (on) {
                std::memcpy(img.data(), host_layer(L), img_f() * 4);
                std::memset(tmp.data(), 0, tmp.size());
                split_image(img.data(), tmp.data());
                std::memcpy(host_layer(L), tmp.data(), host_stride_);
            } else {
                unsplit_image(host_layer(L), img.data());
                std::memcpy(host_layer(L), img.data(), img_f() * 4);
            }
        }
    }
    split_ = on;
    if (!split_ && bf16_ && !host16_)
        CUDA_OK(cudaHostAlloc(&host16_, static_cast<size_t>(n_) * wire16_bytes(), cudaHostAllocPortable));
    std::fill(host16_stale_.begin(), host16_stale_.end(), 1);
    for (auto& c : cache_) c.valid = false;
    std::fill(w16_layer_.begin(), w16_layer_.end(), -1);
    for (int L = 0; L < n_; ++L) bump_version(L);
}

void Executor::register_block(int index, const float* params, int frozen) {
    if (!blk_) throw Error(SP_ERR_INVALID, "register_block: this executor streams dense layers (sp_register_layer)");
    if (index < 0 || index >= n_) throw Error(SP_ERR_INVALID, "register_block: index out of range");
    if (!params) throw Error(SP_ERR_INVALID, "register_block: null parameters");
    flush_writebacks();
    if (split_) split_image(params, host_layer(index));
    else std::memcpy(host_layer(index), params, img_f() * 4);
    relu_[index] = 0;
    frozen_[index] = frozen != 0;
    registered_[index] = 1;
    inconsistent_[static_cast<size_t>(index)] = 0;
    host16_stale_[index] = 1;
    host_partial_[index] = 0;
    sync_layer_meta(index);
    bump_version(index);
    for (auto& c : cache_)
        if (c.layer == index) c.valid = false;
}

void Executor::read_block(int index, float* params) {
    if (!blk_) throw Error(SP_ERR_INVALID, "read_block: this executor streams dense layers (sp_read_layer)");
    if (index < 0 || index >= n_) throw Error(SP_ERR_INVALID, "read_block: index out of range");
    if (!params) throw Error(SP_ERR_INVALID, "read_block: null output");
    flush_writebacks();
    require_full_host(index, "read_block");
    if (split_) unsplit_image(host_layer(index), params);
    else std::memcpy(params, host_layer(index), img_f() * 4);
}

void Executor::dp_init(const uint8_t id[128], int rank, int world, bool shard_weights) {
    if (world < 1 || rank < 0 || rank >= world) throw Error(SP_ERR_INVALID, "dp_init: bad rank/world");
    flush_writebacks();
    require_full_host(-1, "dp_init");
    // world == 1 still builds a (1-rank) communicator: the data-parallel code path (split-K
    // partials, fixed-order reduce, NCCL all-reduce inside the captured graph, SGD on the
    // update stream) then runs end to end on a single GPU.
    if (!nccl().ok()) throw Error(SP_ERR_NCCL, nccl().error);
    // One reduction order for every call: the per-layer collectives have the same sizes for
    // every (k, k') window, and pinning the algorithm and protocol (unless the caller chose
    // them) keeps NCCL's tuner from picking different reduction trees across runs or boxes.
    setenv("NCCL_ALGO", "Ring", 0);
    setenv("NCCL_PROTO", "Simple", 0);
    CUDA_OK(cudaSetDevice(cfg_.device));
    for (auto s : {s_h2d_, s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamSynchronize(s));
    if (comm_) {
        nccl().CommDestroy(comm_);
        comm_ = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    // Byte shards of a split master would not line up with the gradient's logical shards: sharded
    // streaming keeps the fp32 image (the owner of a shared master converts it; CommInitRank below
    // waits for every rank, so the others see the converted copy).
    if (shard_weights && split_) set_split(false);
    NCCL_OK(nccl().CommInitRank(&comm_, world, uid, rank));
    rank_ = rank;
    world_ = world;
    sharded_ = shard_weights;
    layout_slots(shard_weights ? world : 1);  // shard-aligned slot regions
    cap_rows_ = 0;                            // gradient buffers re-sized for world shards
}

void Executor::set_optimizer(int kind, float beta1, float beta2, float eps, float weight_decay) {
    if (kind != SP_OPT_SGD && kind != SP_OPT_ADAMW) throw Error(SP_ERR_INVALID, "optimizer: unknown kind");
    if (kind == SP_OPT_ADAMW && (!(beta1 >= 0.0f && beta1 < 1.0f) || !(beta2 >= 0.0f && beta2 < 1.0f) ||
                                 !(eps > 0.0f) || !(weight_decay >= 0.0f)))
        throw Error(SP_ERR_INVALID, "optimizer: AdamW needs 0 <= beta < 1, eps > 0, weight_decay >= 0");
    flush_writebacks();
    require_full_host(-1, "set_optimizer");
    CUDA_OK(cudaSetDevice(cfg_.device));
    for (auto s : {s_h2d_, s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamSynchronize(s));
    optimizer_ = kind;
    beta1_ = beta1;
    beta2_ = beta2;
    eps_ = eps;
    wd_ = weight_decay;
    step_t_ = 0;
    const size_t img = static_cast<size_t>(n_) * img_f() * 4;
    if (kind == SP_OPT_ADAMW) {
        if (!host_m_) CUDA_OK(cudaHostAlloc(&host_m_, img, cudaHostAllocPortable));
        if (!host_v_) CUDA_OK(cudaHostAlloc(&host_v_, img, cudaHostAllocPortable));
        if (!adamw_host_) CUDA_OK(cudaHostAlloc(&adamw_host_, sizeof(AdamwScalars), cudaHostAllocPortable));
        if (!adamw_dev_) CUDA_OK(cudaMalloc(&adamw_dev_, sizeof(AdamwScalars)));
        std::memset(host_m_, 0, img);
        std::memset(host_v_, 0, img);
    }
    layout_slots(sharded_ ? world_ : 1);  // [A][M][V][B] slots for AdamW; drops caches and graphs
}

void Executor::read_optimizer_state(int index, float* mW, float* mb, float* vW, float* vb) {
    if (index < 0 || index >= n_) throw Error(SP_ERR_INVALID, "read_optimizer_state: index out of range");
    if (!adamw()) throw Error(SP_ERR_STATE, "read_optimizer_state: the optimizer has no state (SGD)");
    flush_writebacks();
    require_full_host(index, "read_optimizer_state");
    if (blk_) {  // a block's state is flat like its image: mW, vW receive all of it
        if (mW) std::memcpy(mW, host_opt(host_m_, index), img_f() * 4);
        if (vW) std::memcpy(vW, host_opt(host_v_, index), img_f() * 4);
        return;
    }
    const size_t dd = static_cast<size_t>(d_) * d_, off = static_cast<size_t>(index) * (dd + d_);
    if (mW) std::memcpy(mW, host_m_ + off, dd * 4);
    if (mb) std::memcpy(mb, host_m_ + off + dd, static_cast<size_t>(d_) * 4);
    if (vW) std::memcpy(vW, host_v_ + off, dd * 4);
    if (vb) std::memcpy(vb, host_v_ + off + dd, static_cast<size_t>(d_) * 4);
}

void Executor::dp_sync() {
    // Collective (every rank, same order): for each layer whose host master is shard-only,
    // stream this rank's shard into slot 0, all-gather the image over NCCL, and copy the
    // whole image back to the pinned host master.
    flush_writebacks();
    bool any = false;
    for (uint8_t p : host_partial_) any = any || p;
    if (!any) return;
    if (!comm_) throw Error(SP_ERR_STATE, "dp_sync: no communicator");
    CUDA_OK(cudaSetDevice(cfg_.device));
    for (auto s : {s_h2d_, s_comp_, s_d2h_, s_upd_}) CUDA_OK(cudaStreamSynchronize(s));
    const size_t img = layer_bytes();
    size_t lo = 0, hi = 0;
    shard_range(shardA_, img, lo, hi);
    uint8_t* stage = slot_ptr(0);
    if (shm_) {  // every rank's train steps (and their write-backs) have completed past here
        NCCL_OK(nccl().AllReduce(loss_dev_ + 1, loss_dev_ + 1, 1, ncclFloat, ncclSum, comm_, s_upd_));
        CUDA_OK(cudaStreamSynchronize(s_upd_));
    }
    for (int L = 0; L < n_; ++L) {
        if (!host_partial_[static_cast<size_t>(L)]) continue;
        // The weights, then (AdamW) the moments: all three are written back shard-only. A
        // shared master (share_host_master) already holds every rank's shard: a barrier below.
        for (float* base : {shm_ ? nullptr : host32_, adamw() ? host_m_ : nullptr, adamw() ? host_v_ : nullptr}) {
            if (!base) continue;
            uint8_t* host = base == host32_ ? host_layer(L) : reinterpret_cast<uint8_t*>(host_opt(base, L));
            if (hi > lo) CUDA_OK(cudaMemcpyAsync(stage + lo, host + lo, hi - lo, cudaMemcpyHostToDevice, s_upd_));
            NCCL_OK(nccl().AllGather(stage + shardA_ * static_cast<size_t>(rank_), stage, shardA_,
                                     ncclUint8, comm_, s_upd_));
            CUDA_OK(cudaMemcpyAsync(host, stage, img, cudaMemcpyDeviceToHost, s_upd_));
            CUDA_OK(cudaStreamSynchronize(s_upd_));  // stage is reused by the next array
        }
        host_partial_[static_cast<size_t>(L)] = 0;
        host16_stale_[static_cast<size_t>(L)] = 1;
    }
    for (auto& c : cache_) c.valid = false;  // slot 0 was overwritten
    std::fill(w16_layer_.begin(), w16_layer_.end(), -1);
}

}  // namespace sp

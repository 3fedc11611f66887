/*
 * superpipe.h — C ABI of the B200 Superpipeline layer-streaming executor.
 *
 * This is the drop-in boundary for the reference's layer-scheduling path. The reference
 * (pipesim, /root/reference/proj) exposes it as a C++ API; each entry point below names
 * the reference interface it replaces. The C++ mirror of that API (include/pipesim_b200/,
 * namespace pipesim) is a thin shim over these calls, so reference callers recompile
 * unchanged. Plain pointers and sizes only; no CUDA or torch types cross the boundary.
 *
 * Conventions
 *  - Every call returns an sp_status; sp_last_error() gives the message of the last failure
 *    on that executor. Codes mirror the reference exit taxonomy (experiment.hpp:60-64;
 *    main.cpp:155-178): 2 = invalid argument (std::invalid_argument), 3 = OOM
 *    (OomDeadlockError, engine.hpp:27-29), 1 = internal invariant (std::logic_error).
 *  - One executor per device per thread; calls are synchronous. The executor owns all
 *    device memory and the pinned host copy of the weights.
 *  - Tensors are row-major fp32: inputs [n_items][rows][d], weights W[in][out] (d*d) and
 *    bias b[d] exactly as LayerBlock (model.hpp:14-26).
 *  - Numerics: SP_NUMERICS_EXACT reproduces the reference bit-for-bit (fp32 SIMT kernels,
 *    reference summation order). SP_NUMERICS_BF16 runs the layer GEMMs on tcgen05 tensor
 *    cores (bf16 operands, fp32 accumulate/master weights); results are bit-identical across
 *    every (k, k') setting and within the documented tolerance of the reference.
 *    SP_NUMERICS_TF32 keeps fp32 operands and activations and multiplies on the tensor cores
 *    as tf32 (kind::tf32, fp32 accumulate): also bit-identical across windows, ~10x closer
 *    to the reference than bf16, at half the bf16 tensor rate.
 *  - There is no CPU path: without a CUDA device every compute call fails with
 *    SP_ERR_CUDA. CpuOnly (strategy.hpp:13) is rejected with SP_ERR_INVALID.
 */
#ifndef SUPERPIPE_H
#define SUPERPIPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 1

typedef struct sp_exec sp_exec;

typedef enum {
    SP_OK = 0,
    SP_ERR_INTERNAL = 1, /* std::logic_error in the reference */
    SP_ERR_INVALID = 2,  /* std::invalid_argument (shapes, knobs, lr, ...) */
    SP_ERR_OOM = 3,      /* OomDeadlockError: the plan cannot fit capacity_bytes */
    SP_ERR_FIDELITY = 4, /* digest mismatch (reserved; mirrors exit code 4) */
    SP_ERR_CUDA = 5,     /* CUDA runtime/driver failure or no device */
    SP_ERR_NCCL = 6,     /* NCCL failure (data-parallel gradient reduction) */
    SP_ERR_STATE = 7     /* call out of order (e.g. layer not registered) */
} sp_status;

/* StrategyKind (strategy.hpp:13) — same order. */
typedef enum { SP_STANDARD = 0, SP_CPU_ONLY = 1, SP_NAIVE = 2, SP_SUPERPIPELINE = 3 } sp_strategy;
/* TransferMode (sim.hpp:15) — same order. */
typedef enum { SP_SEQUENTIAL = 0, SP_BATCH = 1 } sp_transfer_mode;
/* Activation (model.hpp:11) — same order. */
typedef enum { SP_RELU = 0, SP_IDENTITY = 1 } sp_activation;
typedef enum { SP_NUMERICS_EXACT = 0, SP_NUMERICS_BF16 = 1, SP_NUMERICS_TF32 = 2 } sp_numerics;

/* Executor configuration: LayeredModel shape (model.hpp:28-37) + StrategyConfig
 * (strategy.hpp:17-25) + ArenaConfig::capacity_bytes (arena.hpp:14-30) +
 * TrainConfig::checkpointing (engine.hpp:15-24). The arena's bandwidth/latency/rate
 * fields are simulator inputs and have no GPU counterpart. */
typedef struct {
    int32_t n_layers;
    int32_t d;
    int32_t strategy;       /* sp_strategy */
    int32_t k;              /* resident window (Naive, Superpipeline) */
    int32_t k_prime;        /* prefetch / eviction group (Superpipeline) */
    int32_t transfer_mode;  /* sp_transfer_mode */
    int32_t numerics;       /* sp_numerics */
    int32_t checkpointing;  /* training: offload saved activations with their layer */
    int32_t device;         /* CUDA ordinal */
    int32_t trace;          /* 0: call makespan only; 1: + per-op CUDA-event timeline
                               (sp_get_trace, stall/per-item figures); 2: + per-GEMM events
                               (each event record costs device time between kernels) */
    uint64_t capacity_bytes; /* ledger budget in reference bytes; 0 = unlimited */
} sp_config;

/* RunSummary (trace.hpp:52-71) + measured device figures. Ledger fields follow the
 * reference's byte accounting (DeviceArena, arena.hpp:38-111); *_ms fields are measured
 * with CUDA events on the executor's streams for the last forward/train call. */
typedef struct {
    uint64_t peak_bytes;            /* ledger: max weight+activation+gradient bytes */
    uint64_t peak_weight_bytes;
    uint64_t peak_activation_bytes;
    uint64_t peak_gradient_bytes;
    uint64_t total_gradient_bytes;
    uint64_t n_transfers_h2d;       /* H2D channel jobs (batch: one per group) */
    uint64_t n_transfers_d2h;       /* D2H jobs with real bytes (writebacks, offloads) */
    uint64_t n_evictions;           /* slot releases (the reference counts these as D2H) */
    uint64_t h2d_bytes;             /* bytes actually copied host->device (weights+acts) */
    uint64_t d2h_bytes;             /* bytes actually copied device->host */
    uint64_t hbm_reserved_bytes;    /* measured: device memory held by the executor */
    uint64_t kernels_launched;      /* executor kernels launched in the last call */
    double per_item_ms;             /* (last compute end - first compute start) / n_items */
    double makespan_ms;             /* first op start -> last op end */
    double stall_ms;                /* compute-stream idle time waiting for residency */
    double compute_ms;              /* sum of compute-op durations */
    float loss;                     /* training: MSE loss of the last step */
    int32_t n_slots;                /* HBM ring slots S = min(k+k', n) for Superpipeline */
    char digest[17];                /* digest_tensors / digest_train of the last call */
    char _pad[3];
    /* tcgen05 GEMM launches of the last call, each bracketed by CUDA events on the compute
     * stream (cfg.trace = 1): count, summed device time and algorithmic FLOPs (2*M*N*K). */
    uint64_t gemm_launches;
    double gemm_ms;
    double gemm_flops;
    /* host time to enqueue (or replay) the call, and how many calls so far were replayed from
     * a captured CUDA graph (the plan is static, so repeated steps are one graph launch). */
    double host_enqueue_ms;
    uint64_t graph_replays;
    /* attention-core launches and their algorithmic FLOPs (transformer blocks) in the last call */
    uint64_t attn_launches;
    double attn_flops;
} sp_stats;

/* One timeline row (TraceEvent, trace.hpp:20-50); times in ms from the call's start. */
typedef struct {
    double t_start, t_end;
    int32_t kind;      /* 0 Compute, 1 H2D, 2 D2H, 3 Stall (TraceEvent::Kind order) */
    int32_t item, layer, backward;
    int32_t first_layer, n_layers_moved;
    uint64_t weight_bytes, activation_bytes;
    int32_t op_index;  /* index of the op in sp_last_plan's listing (-1 for Stall rows) */
    int32_t reserved;
} sp_trace_event;

/* ---- named-shape layers ------------------------------------------------------------- */
/* The reference's block is one square dense layer y = act(xW + b) (model.hpp:11-26), "an
 * explicit stand-in, not a paper artifact"; the paper streams real transformer
 * layers. A transformer block is a pre-norm decoder / encoder layer whose
 * parameters form one flat fp32 image per layer (the unit the ring streams, exactly as the
 * reference streams one LayerBlock):
 *   norm1 gamma[d] (beta[d])          LayerNorm (SP_NORM_LAYER) or RMSNorm (SP_NORM_RMS)
 *   Wqkv[d][(H + 2 Hkv) hd] (bqkv)    q heads, k heads, v heads; hd = d / H
 *   Wo[H hd][d] (bo)
 *   norm2 gamma[d] (beta[d])
 *   W1[d][ff] (b1)  or  Wgu[d][2 ff]  GELU MLP, or SwiGLU with gate / up interleaved in
 *                                      32-column chunks: columns [g0..g31 u0..u31 g32..]
 *   W2[ff][d] (b2)
 * (bias terms only with bias = 1). Matrices are [in][out] row-major like LayerBlock::weight;
 * every tensor starts on a 64-float boundary; sp_block_layout gives the offsets. Forward:
 *   h = x + attn(norm1(x)) Wo + bo,  y = h + mlp(norm2(h))   (x, h, y: fp32 residual stream)
 * with causal (decoder) or bidirectional (encoder) softmax attention over sequences of
 * seq_len consecutive rows, grouped-query when Hkv < H. Rows = tokens; the training loss is
 * the reference's MSE against a [rows][d] target (mse_loss, model.cpp:131-148). */
typedef enum { SP_BLOCK_DENSE = 0, SP_BLOCK_TRANSFORMER = 1 } sp_block_kind;
typedef enum { SP_NORM_LAYER = 0, SP_NORM_RMS = 1 } sp_norm_kind;
typedef enum { SP_MLP_GELU_TANH = 0, SP_MLP_GELU_ERF = 1, SP_MLP_SWIGLU = 2 } sp_mlp_kind;
typedef struct {
    int32_t kind;        /* sp_block_kind */
    int32_t d;           /* model width (the residual stream) */
    int32_t ff;          /* MLP hidden width */
    int32_t n_heads;     /* query heads H; head_dim = d / H (64, 80 or 128) */
    int32_t n_kv_heads;  /* key/value heads Hkv (divides H; = H without grouped-query) */
    int32_t seq_len;     /* tokens per sequence (rows per call must be a multiple) */
    int32_t norm;        /* sp_norm_kind */
    int32_t mlp;         /* sp_mlp_kind */
    int32_t bias;        /* linear layers carry biases */
    int32_t causal;      /* 1 decoder (causal) attention, 0 encoder (bidirectional) */
    float norm_eps;
    int32_t flags;       /* SP_BLOCK_INFER_ONLY: the host keeps only the bf16 wire image */
    int32_t reserved[4];
} sp_block_desc;
/* sp_block_desc.flags. SP_BLOCK_INFER_ONLY: an inference-only executor whose pinned host copy
 * is the bf16 wire image alone (2 B per matrix parameter instead of 4), for models whose fp32
 * master would not fit host memory (a Llama-3-70B-shape stack: 137 GB of wire image against
 * 274 GB of fp32). Registration keeps the bf16 truncation of each matrix; training calls fail
 * with SP_ERR_INVALID; sp_read_block returns the stored (bf16-valued) parameters. */
#define SP_BLOCK_INFER_ONLY 1
/* One parameter tensor of a block image. */
typedef struct {
    char name[16];
    int64_t rows, cols;      /* vectors: rows = 1 */
    uint64_t offset;         /* in floats, within the fp32 layer image */
    uint64_t wire_offset;    /* in bytes, within the bf16 inference wire image */
    int32_t matrix;          /* 1: bf16 on the wire; 0: fp32 vector */
    int32_t reserved;
} sp_block_tensor;
/* Layout of a block's image: up to cap tensors, their count, the image size in floats and the
 * inference wire image size in bytes (matrices bf16, vectors fp32). Host-only. */
int sp_block_layout(const sp_block_desc* blk, sp_block_tensor* tensors, int32_t cap, int32_t* count,
                    uint64_t* n_floats, uint64_t* wire_bytes);
/* Deterministic random init of layer `index` of a named-shape model (host-only): the
 * reference's per-layer splitmix64 stream (model.cpp:11-14), each matrix and its bias
 * U(+-1/sqrt(fan_in)) in layout order, norm gains 1 and shifts 0. */
int sp_build_block(const sp_block_desc* blk, uint64_t seed, int32_t index, float* params);

/* ---- lifecycle --------------------------------------------------------------------- */
/* Replaces Engine::Engine (engine.cpp:35-49): validates StrategyConfig (strategy.cpp:19-36),
 * allocates the pinned host weight pool and the HBM slot ring. */
int sp_create(const sp_config* cfg, sp_exec** out);
/* Replaces LayerBlock registration (model.hpp:14-26 / build_model, model.cpp:23-52):
 * copies W[d*d] ([in][out]) and b[d] into executor-owned pinned host memory. */
int sp_register_layer(sp_exec* ex, int32_t index, const float* W, const float* b,
                      int32_t activation, int32_t frozen);
/* Executor over named-shape layers: cfg as for sp_create with cfg->d == blk->d; bf16 numerics
 * only (SP_NUMERICS_BF16). Layers are registered with sp_register_block. */
int sp_create_blocks(const sp_config* cfg, const sp_block_desc* blk, sp_exec** out);
/* Copies one layer's fp32 image (sp_block_layout's n_floats floats) into the pinned master. */
int sp_register_block(sp_exec* ex, int32_t index, const float* params, int32_t frozen);
/* Reads one layer's current fp32 image back (RunResult::model for named-shape layers). */
int sp_read_block(sp_exec* ex, int32_t index, float* params);
int sp_destroy(sp_exec* ex);
const char* sp_last_error(const sp_exec* ex);
int sp_abi_version(void);

/* ---- hot path ---------------------------------------------------------------------- */
/* Replaces run_inference (engine.hpp:42-43, engine.cpp:552-556): streams the item-major
 * (item, layer) sequence (strategy.cpp:38-46) through the ring. x, y: host fp32
 * [n_items][rows][d] (pinned buffers from sp_host_alloc avoid a staging copy). */
int sp_forward(sp_exec* ex, const float* x, int64_t rows, int32_t n_items, float* y);
/* Same, with x/y already resident in device memory (fp32). */
int sp_forward_device(sp_exec* ex, const void* x_dev, int64_t rows, int32_t n_items,
                      void* y_dev);
/* Replaces run_train_step (engine.hpp:48-50, engine.cpp:558-563): forward, MSE loss,
 * reverse backward with SGD (model.cpp:157-184) through the ring; the updated weights are
 * written back into the pinned host copy. x, target: host fp32 [rows][d]. The write-backs
 * of the layers still resident in the ring at the end of the step run at the start of the
 * next call (on the otherwise idle D2H engine); every host read through this API
 * (sp_read_layer, sp_digest_train, sp_read_optimizer_state, sp_forward, sp_dp_sync, ...)
 * completes them first, so callers always observe the post-step weights. */
int sp_train_step(sp_exec* ex, const float* x, const float* target, int64_t rows, float lr,
                  float* loss);
int sp_train_step_device(sp_exec* ex, const void* x_dev, const void* target_dev, int64_t rows,
                         float lr, float* loss);
/* Reads back a layer's current weights (RunResult::model, engine.hpp:33). */
int sp_read_layer(sp_exec* ex, int32_t index, float* W, float* b);

/* ---- metrics ----------------------------------------------------------------------- */
int sp_get_stats(const sp_exec* ex, sp_stats* out);
/* The op plan of the last forward/train call, in sp_describe_plan's format (one op per line,
 * with the reference-semantics ledger snapshot "led=weight,activation,gradient"); returns the
 * needed length. Joined with sp_get_trace rows (op_index) it yields the reference's trace CSV. */
int64_t sp_last_plan(const sp_exec* ex, char* buf, int64_t cap);
/* One op of the last call's plan (op_index as in sp_get_trace rows): the reference-semantics
 * ledger snapshot after it (weight, activation, gradient bytes; DeviceArena, arena.hpp:69-80,
 * as TraceEvent::footprint_after, trace.hpp:44-45) and, for transfers, the moved layers in
 * order (TraceEvent::layers). Either output may be NULL; *count = number of moved layers. */
int sp_get_op_info(const sp_exec* ex, int32_t op_index, uint64_t ledger[3], int32_t* layers, int32_t cap,
                   int32_t* count);
/* Changes the trace level (sp_config.trace) for subsequent calls. */
int sp_set_trace(sp_exec* ex, int32_t level);
/* Item batching for sp_forward (layer-major streaming). 0 (default): the
 * reference's item-major execution_stream (strategy.cpp:38-46), every item streams the whole
 * layer stack. 1: the n_items inputs are stacked into one [n_items*rows, d] pass, so each
 * layer crosses the host link once per call instead of once per item. Rows are independent
 * in the layer math, so outputs are bitwise identical; only the transfer count, the ledger
 * and the time change. */
int sp_set_item_batching(sp_exec* ex, int32_t on);
/* Prefetch timing. 1 (default): a weight/activation H2D starts as soon as its ring slot is free
 * (the compute that last read the slot has finished). 0: it also waits for the compute whose
 * completion triggers it in the reference policy (policy_step, scheduler.cpp:105-136: after
 * every k' computes). Both run the same op sequence in the same slots with the same ledger and
 * bitwise-identical results; 1 keeps the link busier (copies are not held behind a
 * copy -> compute -> copy round trip). */
int sp_set_eager_prefetch(sp_exec* ex, int32_t on);

/* ---- optimizer ------------------------------------------------------------------------ */
/* The reference trains with plain SGD (apply_sgd, model.cpp:150-155): SP_OPT_SGD, the default.
 * SP_OPT_ADAMW is PyTorch's AdamW (decoupled weight decay) on the fp32 master weights. Its
 * state m, v lives in pinned host memory next to the weights and streams with every
 * trainable layer's backward: H2D with the layer (even when its weights are still resident),
 * updated in place by one fused kernel (split-K gradient reduction + AdamW), written back
 * with the weights. Each operation is separately rounded in a fixed order (oracle.h
 * orc_adamw), so SP_NUMERICS_EXACT is bit-reproducible. Setting the optimizer zeroes the
 * state and the step count. In sharded data parallel each rank streams and updates only
 * its shard of m, v. */
#define SP_OPT_SGD 0
#define SP_OPT_ADAMW 1
int sp_set_optimizer(sp_exec* ex, int32_t kind, float beta1, float beta2, float eps,
                     float weight_decay);
/* Current AdamW state of one layer (m and v of W[d*d] and b[d]); any pointer may be NULL. */
int sp_read_optimizer_state(sp_exec* ex, int32_t index, float* mW, float* mb, float* vW,
                            float* vb);
/* Copies up to cap events of the last call's measured timeline; *count = total rows. */
int sp_get_trace(const sp_exec* ex, sp_trace_event* events, int32_t cap, int32_t* count);

/* One pinned host master per node (every rank streams from a shared pinned copy):
 * create = 1 moves this executor's fp32 master (and the layers' activation / frozen flags)
 * into the POSIX shared-memory segment `name` (replacing any stale one); create = 0 attaches
 * to the segment another process created for the same (n_layers, d) and drops the private
 * copy. Each process registers the segment with CUDA (cudaHostRegisterPortable), so copies
 * stay pinned-speed. Layers registered through any attached executor are visible to all.
 * Sharded data parallel then needs no all-gather of the weights in sp_dp_sync (each rank's
 * write-back lands in the one copy; sp_dp_sync is a barrier for them). Without sharding, every
 * rank writes back the same all-reduced update, so concurrent write-backs agree bitwise. */
int sp_share_host_master(sp_exec* ex, const char* name, int32_t create);

/* ---- data parallel ----------------------------------------------------------------- */
/* Per-layer NCCL all-reduce of dW/db as each layer's backward completes. The first dp_init of
 * a process sets NCCL_ALGO=Ring and NCCL_PROTO=Simple unless the caller set them, so every
 * call reduces in one fixed order (results are bit-identical across windows and runs). */
int sp_nccl_unique_id(uint8_t id[128]);
int sp_dp_init(sp_exec* ex, const uint8_t id[128], int32_t rank, int32_t world);
/* Same, choosing the weight-streaming mode explicitly. shard_weights = 1: each rank copies only
 * 1/world of every layer over its own host link and an NCCL all-gather over NVLink completes the
 * slot; in training the gradient is reduce-scattered, each rank updates and writes back only its
 * shard (its pinned copy stays authoritative for exactly the shard it streams). shard_weights = 0:
 * every rank streams whole layers and all-reduces dW/db. sp_dp_init uses shard_weights =
 * (world > 1). world = 1 builds a 1-rank communicator (exercises the same code path). */
int sp_dp_init2(sp_exec* ex, const uint8_t id[128], int32_t rank, int32_t world,
                int32_t shard_weights);
/* Collective, every rank in the same order. After sharded training each rank's pinned host
 * master holds only its own shard of every trained layer; sp_dp_sync all-gathers those shards
 * (NCCL over NVLink) so the host copy is whole again. Until then sp_read_layer,
 * sp_digest_train, bf16 sp_forward and sp_dp_init fail with SP_ERR_STATE instead of returning
 * a mix of current and stale shards. No-op when nothing is partial. With a shared host master
 * (sp_share_host_master) every rank's shard already landed in the one copy: the weights need
 * only a barrier (AdamW moments, kept per rank, are still gathered). */
int sp_dp_sync(sp_exec* ex);

/* ---- host utilities ---------------------------------------------------------------- */
/* Pinned (page-locked, portable) host buffers for callers' inputs/outputs. */
void* sp_host_alloc(uint64_t bytes);
void sp_host_free(void* p);
/* peak_weight_residency (strategy.cpp:48-60) and StrategyConfig::validate
 * (strategy.cpp:19-36); pure host functions. validate returns SP_OK or SP_ERR_INVALID. */
uint64_t sp_peak_weight_residency(int32_t strategy, int32_t k, int32_t k_prime,
                                  int32_t n_layers, uint64_t layer_bytes);
int sp_validate_strategy(int32_t strategy, int32_t k, int32_t k_prime, int32_t n_layers);
/* Describes the static op plan the executor would run (policy_step, scheduler.cpp:53-141,
 * resolved ahead of time) as text, one op per line; returns the needed length. Host-only.
 * flags: SP_PLAN_SHARDED (data-parallel sharded streaming), SP_PLAN_EAGER (eager prefetch
 * dependencies, see sp_set_eager_prefetch), SP_PLAN_OPTSTATE (an optimizer with state, e.g.
 * AdamW: its m, v stream with each trainable layer's backward), SP_PLAN_WRITEBACK (training:
 * the executor's write-back scheme - updates copy the slot to a staging buffer the D2H reads,
 * and layers still resident at the end are written back at the start of the next call; the
 * plan shown is the second of two consecutive calls, i.e. the steady state). */
#define SP_PLAN_SHARDED 1
#define SP_PLAN_EAGER 2
#define SP_PLAN_OPTSTATE 4
#define SP_PLAN_WRITEBACK 8
int64_t sp_describe_plan(const sp_config* cfg, int32_t n_items, int32_t train,
                         const int32_t* frozen, int32_t flags, char* buf, int64_t cap);
/* Deterministic layer / input generators of the reference (host-only), so callers can
 * register synthetic models without a second copy: build_model's per-layer splitmix64 stream
 * (model.cpp:23-52, W[fan_in][fan_out] then b[fan_out], U(+-1/sqrt(fan_in)); fan_in = fan_out
 * = d for the reference's square block, 0 = d) and make_input (model.cpp:186-191). */
int sp_build_layer(uint64_t seed, int32_t index, int32_t d, int32_t fan_in, int32_t fan_out,
                   float* W, float* b);
void sp_make_input(uint64_t seed, uint64_t tag, int64_t rows, int32_t d, float* out);
/* digest helpers (engine.cpp:565-581): FNV-1a-64 digests as 16 hex chars + NUL. They are
 * computed on demand (never inside the hot path): sp_digest_tensors over a caller's outputs,
 * sp_digest_train over (loss, the executor's current weights) = digest_train(loss, model). */
int sp_digest_train(const sp_exec* ex, float loss, char out[17]);
void sp_digest_tensors(const float* values, int32_t n_items, int64_t rows, int32_t d,
                       char out[17]);

#ifdef __cplusplus
}
#endif
#endif /* SUPERPIPE_H */

// pipesim.hpp — C++ mirror of the reference's public API (namespace pipesim) over the C ABI
// of libsuperpipe.so (include/superpipe.h). Header-only; link with -lsuperpipe.
//
// Source-compatible with the reference's headers for the executor path:
//   tensor.hpp:11-51   Tensor
//   model.hpp:11-89    Activation, LayerBlock, LayeredModel, build_model, make_input
//   strategy.hpp:13-33 StrategyKind, StrategyConfig, peak_weight_residency
//   sim.hpp:15         TransferMode
//   arena.hpp:14-30    ArenaConfig
//   engine.hpp:15-62   TrainConfig, OomDeadlockError, RunResult, run_inference,
//                      run_train_step, digest_tensors, digest_train
// so a reference caller (experiment.cpp:83-100, tuner.cpp:86-87, the tests) recompiles
// against this header unchanged. Differences, by design:
//   * compute runs on the GPU; RunSummary times are measured milliseconds (CUDA events),
//     not the simulator's virtual seconds, and the trace is the measured timeline;
//   * StrategyKind::CpuOnly throws std::invalid_argument (there is no CPU path);
//   * numerics: bit-exact fp32 by default (Numerics::Exact), Numerics::Bf16 / Numerics::Tf32
//     select the tcgen05 tensor-core paths (set_numerics()).
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../superpipe.h"

namespace pipesim {

// ---- tensor.hpp ------------------------------------------------------------------------
struct Tensor {
    std::vector<std::int64_t> shape;
    std::vector<float> values;

    Tensor() = default;
    Tensor(std::vector<std::int64_t> s, std::vector<float> v) : shape(std::move(s)), values(std::move(v)) {
        if (element_count(shape) != static_cast<std::int64_t>(values.size()))
            throw std::invalid_argument("tensor: shape does not match value count");
    }
    static std::int64_t element_count(const std::vector<std::int64_t>& s) {
        std::int64_t n = 1;
        for (auto d : s) {
            if (d < 0) throw std::invalid_argument("tensor: negative dimension");
            n *= d;
        }
        return n;
    }
    static Tensor zeros(std::vector<std::int64_t> s) {
        const auto n = element_count(s);
        return Tensor{std::move(s), std::vector<float>(static_cast<std::size_t>(n), 0.0f)};
    }
    std::int64_t rows() const { return shape.empty() ? 0 : shape[0]; }
    std::int64_t cols() const { return shape.size() < 2 ? 0 : shape[1]; }
    float& at(std::int64_t r, std::int64_t c) { return values[static_cast<std::size_t>(r * cols() + c)]; }
    float at(std::int64_t r, std::int64_t c) const { return values[static_cast<std::size_t>(r * cols() + c)]; }
    bool same_shape(const Tensor& o) const { return shape == o.shape; }
    friend bool operator==(const Tensor& a, const Tensor& b) {
        return a.shape == b.shape && a.values == b.values;
    }
};

// ---- model.hpp -------------------------------------------------------------------------
enum class Activation { ReLU, Identity };

struct LayerBlock {
    int index = 0;
    int d = 0;
    std::vector<float> weight;  // d*d, [in][out] row-major
    std::vector<float> bias;    // d
    Activation activation = Activation::ReLU;
    bool frozen = false;
    std::uint64_t weight_bytes() const {
        const auto dd = static_cast<std::uint64_t>(d);
        return (dd * dd + dd) * 4;
    }
};

struct LayeredModel {
    int d = 0;
    int n_layers = 0;
    std::uint64_t seed = 0;
    std::vector<LayerBlock> blocks;
    std::uint64_t layer_bytes() const { return blocks.empty() ? 0 : blocks.front().weight_bytes(); }
};

inline LayeredModel build_model(std::uint64_t seed, int n_layers, int d, int frozen_prefix) {
    if (n_layers < 1) throw std::invalid_argument("build_model: n_layers must be >= 1");
    if (d < 1) throw std::invalid_argument("build_model: d must be >= 1");
    if (frozen_prefix < 0 || frozen_prefix > n_layers)
        throw std::invalid_argument("build_model: frozen_prefix out of range");
    LayeredModel m;
    m.d = d;
    m.n_layers = n_layers;
    m.seed = seed;
    for (int i = 0; i < n_layers; ++i) {
        LayerBlock b;
        b.index = i;
        b.d = d;
        b.frozen = i < frozen_prefix;
        b.weight.resize(static_cast<std::size_t>(d) * d);
        b.bias.resize(static_cast<std::size_t>(d));
        sp_build_layer(seed, i, d, 0, 0, b.weight.data(), b.bias.data());
        m.blocks.push_back(std::move(b));
    }
    return m;
}

inline Tensor make_input(std::uint64_t seed, std::uint64_t stream_tag, std::int64_t rows, int d) {
    Tensor t = Tensor::zeros({rows, d});
    sp_make_input(seed, stream_tag, rows, d, t.values.data());
    return t;
}

// ---- strategy.hpp / sim.hpp / arena.hpp -------------------------------------------------
enum class StrategyKind { Standard, CpuOnly, Naive, Superpipeline };
enum class TransferMode { Sequential, Batch };

inline std::string to_string(StrategyKind kind) {
    switch (kind) {
        case StrategyKind::Standard: return "standard";
        case StrategyKind::CpuOnly: return "cpu_only";
        case StrategyKind::Naive: return "naive";
        case StrategyKind::Superpipeline: return "superpipeline";
    }
    return "unknown";
}

struct StrategyConfig {
    StrategyKind kind = StrategyKind::Standard;
    int k = 0;
    int k_prime = 0;
    TransferMode transfer_mode = TransferMode::Batch;
    void validate(int n_layers) const {
        if (sp_validate_strategy(static_cast<int>(kind), k, k_prime, n_layers) != SP_OK)
            throw std::invalid_argument("strategy: invalid (k, k') for n_layers");
    }
};

inline std::uint64_t peak_weight_residency(const StrategyConfig& cfg, int n_layers,
                                           std::uint64_t weight_bytes_per_layer) {
    cfg.validate(n_layers);
    return sp_peak_weight_residency(static_cast<int>(cfg.kind), cfg.k, cfg.k_prime, n_layers,
                                    weight_bytes_per_layer);
}

struct ArenaConfig {
    std::uint64_t capacity_bytes = 0;
    double h2d_bandwidth = 1.0;  // simulator-only fields: accepted, validated, not used
    double d2h_bandwidth = 1.0;
    double per_call_latency = 0.0;
    double device_compute_rate = 1.0;
    double host_compute_rate = 1.0;
    void validate() const {
        if (h2d_bandwidth <= 0 || d2h_bandwidth <= 0)
            throw std::invalid_argument("arena: bandwidths must be > 0");
        if (device_compute_rate <= 0 || host_compute_rate <= 0)
            throw std::invalid_argument("arena: compute rates must be > 0");
        if (per_call_latency < 0) throw std::invalid_argument("arena: per_call_latency must be >= 0");
    }
};

// ---- engine.hpp ------------------------------------------------------------------------
struct TrainConfig {
    float lr = 0.01f;
    bool checkpointing = false;
    std::int64_t batch_size = 1;
    void validate() const {
        if (lr <= 0.0f) throw std::invalid_argument("train: lr must be > 0");
        if (batch_size < 1) throw std::invalid_argument("train: batch_size must be >= 1");
    }
};

struct OomDeadlockError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// trace.hpp:52-71, measured: times in milliseconds of device time.
struct RunSummary {
    std::string strategy;
    int k = 0;
    int k_prime = 0;
    std::uint64_t peak_bytes = 0;
    double per_item_time = 0.0;
    double makespan = 0.0;
    double total_stall_time = 0.0;
    std::uint64_t n_transfers_h2d = 0;
    std::uint64_t n_transfers_d2h = 0;
    std::string output_digest;
    std::uint64_t peak_weight_bytes = 0;
    std::uint64_t peak_activation_bytes = 0;
    std::uint64_t peak_gradient_bytes = 0;
    std::uint64_t total_gradient_bytes = 0;
    double loss = 0.0;
    bool has_loss = false;
};

struct RunResult {
    std::vector<Tensor> outputs;
    LayeredModel model;
    float loss = 0.0f;
    std::vector<sp_trace_event> trace;
    RunSummary summary;
};

enum class Numerics { Exact = SP_NUMERICS_EXACT, Bf16 = SP_NUMERICS_BF16, Tf32 = SP_NUMERICS_TF32 };

namespace detail {
inline Numerics& numerics() {
    static thread_local Numerics n = Numerics::Exact;
    return n;
}
inline std::string hex_of(const char* s) { return std::string(s); }

inline void check(int rc, sp_exec* ex) {
    if (rc == SP_OK) return;
    const std::string msg = sp_last_error(ex) ? sp_last_error(ex) : "";
    if (rc == SP_ERR_INVALID) throw std::invalid_argument(msg);
    if (rc == SP_ERR_OOM) throw OomDeadlockError(msg);
    if (rc == SP_ERR_INTERNAL || rc == SP_ERR_STATE) throw std::logic_error(msg);
    throw std::runtime_error("superpipe: " + msg);
}

// RAII executor for one run_* call (the reference constructs an Engine per call too,
// engine.cpp:552-563).
struct Exec {
    sp_exec* ex = nullptr;
    Exec(const LayeredModel& m, const StrategyConfig& s, const ArenaConfig& a, bool ckpt) {
        a.validate();
        s.validate(m.n_layers);
        if (s.kind == StrategyKind::CpuOnly)
            throw std::invalid_argument("strategy: cpu_only has no GPU executor (no CPU fallback)");
        sp_config c{};
        c.n_layers = m.n_layers;
        c.d = m.d;
        c.strategy = static_cast<int>(s.kind);
        c.k = s.k;
        c.k_prime = s.k_prime;
        c.transfer_mode = s.transfer_mode == TransferMode::Batch ? SP_BATCH : SP_SEQUENTIAL;
        c.numerics = static_cast<int>(numerics());
        c.checkpointing = ckpt ? 1 : 0;
        c.trace = 1;
        c.capacity_bytes = a.capacity_bytes;
        check(sp_create(&c, &ex), nullptr);
        for (const auto& b : m.blocks)
            check(sp_register_layer(ex, b.index, b.weight.data(), b.bias.data(),
                                    b.activation == Activation::ReLU ? SP_RELU : SP_IDENTITY,
                                    b.frozen ? 1 : 0),
                  ex);
    }
    ~Exec() { sp_destroy(ex); }
    Exec(const Exec&) = delete;
    Exec& operator=(const Exec&) = delete;

    RunSummary summary(const StrategyConfig& s, int n_items) const {
        sp_stats st{};
        sp_get_stats(ex, &st);
        RunSummary r;
        r.strategy = to_string(s.kind);
        r.k = s.k;
        r.k_prime = s.k_prime;
        r.peak_bytes = st.peak_bytes;
        r.per_item_time = st.per_item_ms;
        r.makespan = st.makespan_ms;
        r.total_stall_time = st.stall_ms;
        r.n_transfers_h2d = st.n_transfers_h2d;
        r.n_transfers_d2h = st.n_transfers_d2h;
        r.peak_weight_bytes = st.peak_weight_bytes;
        r.peak_activation_bytes = st.peak_activation_bytes;
        r.peak_gradient_bytes = st.peak_gradient_bytes;
        r.total_gradient_bytes = st.total_gradient_bytes;
        (void)n_items;
        return r;
    }
    std::vector<sp_trace_event> trace() const {
        int32_t n = 0;
        sp_get_trace(ex, nullptr, 0, &n);
        std::vector<sp_trace_event> ev(static_cast<std::size_t>(n));
        sp_get_trace(ex, ev.data(), n, &n);
        return ev;
    }
};
}  // namespace detail

// Selects the numerics of subsequent run_* calls on this thread (default: bit-exact fp32).
inline void set_numerics(Numerics n) { detail::numerics() = n; }

inline std::string digest_tensors(const std::vector<Tensor>& tensors) {
    // engine.cpp:565-572: chain FNV-1a over each tensor (shape bytes, then values).
    std::uint64_t h = 0xCBF29CE484222325ull;
    auto fnv = [&](const void* p, std::size_t n) {
        const auto* c = static_cast<const unsigned char*>(p);
        for (std::size_t i = 0; i < n; ++i) {
            h ^= c[i];
            h *= 0x100000001B3ull;
        }
    };
    for (const auto& t : tensors) {
        fnv(t.shape.data(), t.shape.size() * sizeof(std::int64_t));
        fnv(t.values.data(), t.values.size() * sizeof(float));
    }
    static const char digits[] = "0123456789abcdef";
    std::string out(16, '0');
    for (int i = 15; i >= 0; --i) {
        out[static_cast<std::size_t>(i)] = digits[h & 0xF];
        h >>= 4;
    }
    return out;
}

inline std::string digest_train(float loss, const LayeredModel& model) {
    std::uint64_t h = 0xCBF29CE484222325ull;
    auto fnv = [&](const void* p, std::size_t n) {
        const auto* c = static_cast<const unsigned char*>(p);
        for (std::size_t i = 0; i < n; ++i) {
            h ^= c[i];
            h *= 0x100000001B3ull;
        }
    };
    fnv(&loss, sizeof(loss));
    for (const auto& b : model.blocks) {
        fnv(b.weight.data(), b.weight.size() * sizeof(float));
        fnv(b.bias.data(), b.bias.size() * sizeof(float));
    }
    static const char digits[] = "0123456789abcdef";
    std::string out(16, '0');
    for (int i = 15; i >= 0; --i) {
        out[static_cast<std::size_t>(i)] = digits[h & 0xF];
        h >>= 4;
    }
    return out;
}

inline RunResult run_inference(const LayeredModel& model, const std::vector<Tensor>& inputs,
                               const StrategyConfig& strategy, const ArenaConfig& arena_cfg) {
    if (inputs.empty()) throw std::invalid_argument("run_inference: no inputs");
    const std::int64_t rows = inputs.front().rows();
    for (const auto& in : inputs)
        if (in.shape.size() != 2 || in.cols() != model.d || in.rows() != rows)
            throw std::invalid_argument("run_inference: inputs must have shape [b, d]");
    detail::Exec ex(model, strategy, arena_cfg, false);
    const std::size_t per = static_cast<std::size_t>(rows) * static_cast<std::size_t>(model.d);
    std::vector<float> x(per * inputs.size()), y(per * inputs.size());
    for (std::size_t i = 0; i < inputs.size(); ++i)
        std::memcpy(x.data() + i * per, inputs[i].values.data(), per * sizeof(float));
    detail::check(sp_forward(ex.ex, x.data(), rows, static_cast<int32_t>(inputs.size()), y.data()), ex.ex);
    RunResult r;
    for (std::size_t i = 0; i < inputs.size(); ++i)
        r.outputs.emplace_back(std::vector<std::int64_t>{rows, model.d},
                               std::vector<float>(y.begin() + static_cast<std::ptrdiff_t>(i * per),
                                                  y.begin() + static_cast<std::ptrdiff_t>((i + 1) * per)));
    r.model = model;
    r.summary = ex.summary(strategy, static_cast<int>(inputs.size()));
    r.summary.output_digest = digest_tensors(r.outputs);
    r.trace = ex.trace();
    return r;
}

inline RunResult run_train_step(const LayeredModel& model, const Tensor& x, const Tensor& target,
                                const StrategyConfig& strategy, const ArenaConfig& arena_cfg,
                                const TrainConfig& train_cfg) {
    train_cfg.validate();
    if (x.shape.size() != 2 || x.cols() != model.d || x.rows() != train_cfg.batch_size)
        throw std::invalid_argument("run_train_step: x must have shape [batch_size, d]");
    if (!target.same_shape(x)) throw std::invalid_argument("run_train_step: target shape mismatch");
    detail::Exec ex(model, strategy, arena_cfg, train_cfg.checkpointing);
    float loss = 0.0f;
    detail::check(sp_train_step(ex.ex, x.values.data(), target.values.data(), x.rows(),
                                train_cfg.lr, &loss),
                  ex.ex);
    RunResult r;
    r.model = model;
    for (auto& b : r.model.blocks)
        detail::check(sp_read_layer(ex.ex, b.index, b.weight.data(), b.bias.data()), ex.ex);
    r.loss = loss;
    r.summary = ex.summary(strategy, 1);
    r.summary.output_digest = digest_train(loss, r.model);
    r.summary.loss = loss;
    r.summary.has_loss = true;
    r.trace = ex.trace();
    return r;
}

// engine.hpp:55-62 (engine.cpp:583-592): recompute the reference forward of every input and
// compare bitwise. The recomputation is the executor's exact numerics, which reproduce
// reference_forward bit for bit on the GPU (a Superpipeline(2,1) ring, so any model fits).
struct FidelityResult {
    bool ok = false;
    std::string digest;
};

inline FidelityResult verify_fidelity(const std::vector<Tensor>& outputs, const LayeredModel& model,
                                      const std::vector<Tensor>& inputs) {
    FidelityResult result;
    result.digest = digest_tensors(outputs);
    if (outputs.size() != inputs.size()) return result;
    const Numerics saved = detail::numerics();
    detail::numerics() = Numerics::Exact;
    const StrategyConfig ring = model.n_layers >= 2
                                    ? StrategyConfig{StrategyKind::Superpipeline, 2, 1, TransferMode::Batch}
                                    : StrategyConfig{StrategyKind::Standard, 0, 0, TransferMode::Batch};
    try {
        for (std::size_t i = 0; i < inputs.size(); ++i) {
            const RunResult ref = run_inference(model, {inputs[i]}, ring, ArenaConfig{});
            if (!(ref.outputs[0] == outputs[i])) {
                detail::numerics() = saved;
                return result;
            }
        }
    } catch (...) {
        detail::numerics() = saved;
        throw;
    }
    detail::numerics() = saved;
    result.ok = true;
    return result;
}

}  // namespace pipesim

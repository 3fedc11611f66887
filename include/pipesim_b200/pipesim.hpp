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
//                      run_train_step, digest_tensors, digest_train, verify_fidelity
//   trace.hpp:10-87    MemoryFootprint, TraceEvent, Trace, RunSummary, summarize, kind_name,
//                      event_detail, format_double, export_trace_csv / _json,
//                      import_trace_csv, summary_to_json
// so a reference caller (experiment.cpp:83-100, tuner.cpp:86-87, the tests) recompiles
// against this header unchanged: include/pipesim_b200/pipesim/<name>.hpp are the reference's
// header names, each forwarding here (tests/cpp builds the reference's own test_engine.cpp and
// acceptance.cpp against them). The CPU oracle of model.hpp:54-86 (layer_forward,
// layer_backward, reference_forward, mse_loss, mse_grad, apply_sgd, reference_train_step) is
// declared for source compatibility; the library has no CPU math, so a caller links an
// implementation (the test build links the reference's own model.cpp). Differences, by design:
//   * compute runs on the GPU; RunSummary times are measured milliseconds (CUDA events),
//     not the simulator's virtual seconds, and the trace is the measured timeline;
//   * StrategyKind::CpuOnly throws std::invalid_argument (there is no CPU path);
//   * numerics: bit-exact fp32 by default (Numerics::Exact), Numerics::Bf16 / Numerics::Tf32
//     select the tcgen05 tensor-core paths (set_numerics()).
#pragma once

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
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

// splitmix64 (model.hpp:40-52); the per-layer stream is seeded from (seed, layer index).
struct SplitMix64 {
    std::uint64_t state;
    explicit SplitMix64(std::uint64_t s) : state(s) {}
    std::uint64_t next() {
        state += 0x9E3779B97F4A7C15ull;
        std::uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

#ifndef PIPESIM_B200_EXTERNAL_GENERATORS  // (defined only where the reference's model.cpp is compiled)
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
#else
LayeredModel build_model(std::uint64_t seed, int n_layers, int d, int frozen_prefix);
Tensor make_input(std::uint64_t seed, std::uint64_t stream_tag, std::int64_t rows, int d);
#endif

// The reference's CPU oracle (model.hpp:56-86): declarations only (see the header comment).
struct LayerGrads {
    Tensor dx;
    std::vector<float> dW;  // d*d
    std::vector<float> db;  // d
};
struct TrainStepResult {
    float loss = 0.0f;
    std::vector<LayerGrads> grads;
};
Tensor layer_forward(const LayerBlock& block, const Tensor& x);
LayerGrads layer_backward(const LayerBlock& block, const Tensor& x, const Tensor& dy);
Tensor reference_forward(const LayeredModel& model, const Tensor& x);
float mse_loss(const Tensor& y, const Tensor& target);
Tensor mse_grad(const Tensor& y, const Tensor& target);
void apply_sgd(LayerBlock& block, const std::vector<float>& dW, const std::vector<float>& db, float lr);
TrainStepResult reference_train_step(LayeredModel& model, const Tensor& x, const Tensor& target, float lr);

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

// ---- trace.hpp -------------------------------------------------------------------------
// trace.hpp:10-50. Rows come from the measured CUDA-event timeline (times in milliseconds of
// device time from the call's start); footprint_after is the plan's reference-semantics ledger
// snapshot after the op (sp_get_op_info).
struct MemoryFootprint {
    std::uint64_t weight_bytes = 0;
    std::uint64_t activation_bytes = 0;
    std::uint64_t gradient_bytes = 0;
    std::uint64_t total() const { return weight_bytes + activation_bytes + gradient_bytes; }
    friend bool operator==(const MemoryFootprint& a, const MemoryFootprint& b) {
        return a.weight_bytes == b.weight_bytes && a.activation_bytes == b.activation_bytes &&
               a.gradient_bytes == b.gradient_bytes;
    }
};

struct TraceEvent {
    enum class Kind { Compute, H2D, D2H, Stall };
    double t_start = 0.0;
    double t_end = 0.0;
    Kind kind = Kind::Compute;
    int item = -1;
    int layer = -1;
    bool backward = false;
    std::vector<int> layers;
    std::uint64_t moved_weight_bytes = 0;
    std::uint64_t moved_activation_bytes = 0;
    std::uint64_t compute_activation_bytes = 0;
    std::uint64_t compute_gradient_bytes = 0;
    std::string reason;
    std::uint64_t resident_bytes_after = 0;
    MemoryFootprint footprint_after;
    friend bool operator==(const TraceEvent& a, const TraceEvent& b) {
        return a.t_start == b.t_start && a.t_end == b.t_end && a.kind == b.kind && a.item == b.item &&
               a.layer == b.layer && a.backward == b.backward && a.layers == b.layers &&
               a.moved_weight_bytes == b.moved_weight_bytes &&
               a.moved_activation_bytes == b.moved_activation_bytes &&
               a.compute_activation_bytes == b.compute_activation_bytes &&
               a.compute_gradient_bytes == b.compute_gradient_bytes && a.reason == b.reason &&
               a.resident_bytes_after == b.resident_bytes_after && a.footprint_after == b.footprint_after;
    }
};

using Trace = std::vector<TraceEvent>;

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
    Trace trace;
    RunSummary summary;
};

inline std::string kind_name(TraceEvent::Kind kind) {
    switch (kind) {
        case TraceEvent::Kind::Compute: return "Compute";
        case TraceEvent::Kind::H2D: return "H2D";
        case TraceEvent::Kind::D2H: return "D2H";
        case TraceEvent::Kind::Stall: return "Stall";
    }
    return "?";
}

// Shortest decimal that round-trips (trace.hpp:77-78).
inline std::string format_double(double v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    if (res.ec != std::errc{}) throw std::runtime_error("format_double: conversion failed");
    return std::string(buf, res.ptr);
}

namespace detail {
inline std::string join_ints(const std::vector<int>& v) {
    std::string out;
    for (std::size_t i = 0; i < v.size(); ++i) out += (i ? "+" : "") + std::to_string(v[i]);
    return out;
}
inline std::string json_string(const std::string& s) {
    std::string out = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') out += '\\';
        out += c;
    }
    return out + "\"";
}
// JSON number of a double: shortest round-trip digits, integral values written with ".0"
inline std::string json_double(double v) {
    std::string t = format_double(v);
    if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
    return t;
}
}  // namespace detail

// The detail column of the trace CSV (trace.hpp:75): key=value pairs joined by ';'.
inline std::string event_detail(const TraceEvent& ev) {
    std::string out;
    if (ev.kind == TraceEvent::Kind::Compute) {
        out = "item=" + std::to_string(ev.item) + ";layer=" + std::to_string(ev.layer) +
              ";pass=" + (ev.backward ? "bwd" : "fwd");
        if (ev.compute_activation_bytes) out += ";ab=" + std::to_string(ev.compute_activation_bytes);
        if (ev.compute_gradient_bytes) out += ";gb=" + std::to_string(ev.compute_gradient_bytes);
    } else if (ev.kind == TraceEvent::Kind::Stall) {
        out = "reason=" + ev.reason;
    } else {
        out = "layers=" + detail::join_ints(ev.layers) + ";wb=" + std::to_string(ev.moved_weight_bytes);
        if (ev.moved_activation_bytes) out += ";ab=" + std::to_string(ev.moved_activation_bytes);
    }
    return out;
}

// trace.hpp:73: the timing / peak / transfer-count fields of a completed trace.
inline RunSummary summarize(const Trace& trace, int n_items) {
    if (trace.empty()) throw std::invalid_argument("summarize: empty trace");
    if (n_items < 1) throw std::invalid_argument("summarize: n_items must be >= 1");
    RunSummary s;
    double first = -1.0, last = 0.0;
    for (const auto& ev : trace) {
        s.makespan = std::max(s.makespan, ev.t_end);
        s.peak_bytes = std::max(s.peak_bytes, ev.footprint_after.total());
        if (ev.kind == TraceEvent::Kind::Compute) {
            if (first < 0) first = ev.t_start;
            last = std::max(last, ev.t_end);
        } else if (ev.kind == TraceEvent::Kind::H2D) {
            ++s.n_transfers_h2d;
        } else if (ev.kind == TraceEvent::Kind::D2H) {
            ++s.n_transfers_d2h;
        } else {
            s.total_stall_time += ev.t_end - ev.t_start;
        }
    }
    if (first >= 0) s.per_item_time = (last - first) / n_items;
    return s;
}

inline std::string summary_to_json(const RunSummary& s) {
    // keys in lexicographic order, compact, as the reference's nlohmann dump (trace.cpp:219-237)
    std::vector<std::pair<std::string, std::string>> kv = {
        {"k", std::to_string(s.k)},
        {"k_prime", std::to_string(s.k_prime)},
        {"makespan", detail::json_double(s.makespan)},
        {"n_transfers_d2h", std::to_string(s.n_transfers_d2h)},
        {"n_transfers_h2d", std::to_string(s.n_transfers_h2d)},
        {"output_digest", detail::json_string(s.output_digest)},
        {"peak_activation_bytes", std::to_string(s.peak_activation_bytes)},
        {"peak_bytes", std::to_string(s.peak_bytes)},
        {"peak_gradient_bytes", std::to_string(s.peak_gradient_bytes)},
        {"peak_weight_bytes", std::to_string(s.peak_weight_bytes)},
        {"per_item_time", detail::json_double(s.per_item_time)},
        {"strategy", detail::json_string(s.strategy)},
        {"total_gradient_bytes", std::to_string(s.total_gradient_bytes)},
        {"total_stall_time", detail::json_double(s.total_stall_time)},
    };
    if (s.has_loss) kv.emplace_back("loss", detail::json_double(s.loss));
    std::sort(kv.begin(), kv.end());
    std::string out = "{";
    for (std::size_t i = 0; i < kv.size(); ++i) out += (i ? "," : "") + detail::json_string(kv[i].first) + ":" + kv[i].second;
    return out + "}";
}

inline const char* trace_csv_header() {
    return "t_start,t_end,kind,detail,resident_bytes,weight_bytes,activation_bytes,gradient_bytes";
}

inline void export_trace_csv(const Trace& trace, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("export_trace: cannot open '" + path + "' for writing");
    out << trace_csv_header() << '\n';
    for (const auto& ev : trace)
        out << format_double(ev.t_start) << ',' << format_double(ev.t_end) << ',' << kind_name(ev.kind) << ','
            << event_detail(ev) << ',' << ev.resident_bytes_after << ',' << ev.footprint_after.weight_bytes << ','
            << ev.footprint_after.activation_bytes << ',' << ev.footprint_after.gradient_bytes << '\n';
    if (!out) throw std::runtime_error("export_trace: write to '" + path + "' failed");
}

inline void export_trace_json(const Trace& trace, const RunSummary& summary, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("export_trace: cannot open '" + path + "' for writing");
    out << "{\"events\":[";
    for (std::size_t i = 0; i < trace.size(); ++i) {
        const auto& ev = trace[i];
        out << (i ? "," : "") << "{\"t_start\":" << detail::json_double(ev.t_start)
            << ",\"t_end\":" << detail::json_double(ev.t_end) << ",\"kind\":" << detail::json_string(kind_name(ev.kind))
            << ",\"detail\":" << detail::json_string(event_detail(ev)) << ",\"resident_bytes\":" << ev.resident_bytes_after
            << ",\"weight_bytes\":" << ev.footprint_after.weight_bytes
            << ",\"activation_bytes\":" << ev.footprint_after.activation_bytes
            << ",\"gradient_bytes\":" << ev.footprint_after.gradient_bytes << "}";
    }
    out << "],\"summary\":" << summary_to_json(summary) << "}\n";
    if (!out) throw std::runtime_error("export_trace: write to '" + path + "' failed");
}

inline Trace import_trace_csv(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("import_trace: cannot open '" + path + "'");
    std::string line;
    if (!std::getline(in, line)) throw std::runtime_error("import_trace: '" + path + "' is empty");
    if (line != trace_csv_header()) throw std::runtime_error("import_trace: unexpected header in '" + path + "'");
    Trace trace;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::vector<std::string> col;
        std::stringstream ss(line);
        std::string cell;
        while (std::getline(ss, cell, ',')) col.push_back(cell);
        if (col.size() != 8) throw std::runtime_error("import_trace: malformed row in '" + path + "'");
        TraceEvent ev;
        ev.t_start = std::stod(col[0]);
        ev.t_end = std::stod(col[1]);
        const std::string& k = col[2];
        if (k == "Compute") ev.kind = TraceEvent::Kind::Compute;
        else if (k == "H2D") ev.kind = TraceEvent::Kind::H2D;
        else if (k == "D2H") ev.kind = TraceEvent::Kind::D2H;
        else if (k == "Stall") ev.kind = TraceEvent::Kind::Stall;
        else throw std::runtime_error("import_trace: unknown kind '" + k + "'");
        std::stringstream ds(col[3]);
        std::string pair;
        while (std::getline(ds, pair, ';')) {
            const auto eq = pair.find('=');
            if (eq == std::string::npos) throw std::runtime_error("import_trace: bad detail '" + pair + "'");
            const std::string key = pair.substr(0, eq), val = pair.substr(eq + 1);
            if (key == "item") ev.item = std::stoi(val);
            else if (key == "layer") ev.layer = std::stoi(val);
            else if (key == "pass") ev.backward = val == "bwd";
            else if (key == "wb") ev.moved_weight_bytes = std::stoull(val);
            else if (key == "gb") ev.compute_gradient_bytes = std::stoull(val);
            else if (key == "reason") ev.reason = val;
            else if (key == "ab") (ev.kind == TraceEvent::Kind::Compute ? ev.compute_activation_bytes
                                                                         : ev.moved_activation_bytes) = std::stoull(val);
            else if (key == "layers") {
                std::stringstream ls(val);
                std::string l;
                while (std::getline(ls, l, '+'))
                    if (!l.empty()) ev.layers.push_back(std::stoi(l));
            } else throw std::runtime_error("import_trace: unknown detail key '" + key + "'");
        }
        ev.resident_bytes_after = std::stoull(col[4]);
        ev.footprint_after.weight_bytes = std::stoull(col[5]);
        ev.footprint_after.activation_bytes = std::stoull(col[6]);
        ev.footprint_after.gradient_bytes = std::stoull(col[7]);
        trace.push_back(std::move(ev));
    }
    return trace;
}

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
    // The measured timeline as reference TraceEvents (trace.hpp:20-50): compute rows carry the
    // activation / gradient bytes the reference's ledger allocates for them (engine.cpp:271-282),
    // transfer rows their moved layers, every row the plan's ledger snapshot after it.
    Trace trace(bool train, bool ckpt, const LayeredModel& m, std::int64_t rows) const {
        int32_t n = 0;
        sp_get_trace(ex, nullptr, 0, &n);
        std::vector<sp_trace_event> raw(static_cast<std::size_t>(n));
        sp_get_trace(ex, raw.data(), n, &n);
        Trace out;
        const std::uint64_t act = static_cast<std::uint64_t>(rows) * static_cast<std::uint64_t>(m.d) * 4;
        MemoryFootprint last{};
        for (const auto& r : raw) {
            TraceEvent ev;
            ev.t_start = r.t_start;
            ev.t_end = r.t_end;
            ev.kind = static_cast<TraceEvent::Kind>(r.kind);
            uint64_t led[3] = {0, 0, 0};
            if (r.op_index >= 0) {
                int32_t cnt = 0;
                sp_get_op_info(ex, r.op_index, led, nullptr, 0, &cnt);
                if (cnt > 0) {
                    ev.layers.resize(static_cast<std::size_t>(cnt));
                    sp_get_op_info(ex, r.op_index, nullptr, ev.layers.data(), cnt, &cnt);
                }
                last = MemoryFootprint{led[0], led[1], led[2]};
            }
            ev.footprint_after = last;  // a stall row: the ledger as it stands
            ev.resident_bytes_after = last.total();
            if (ev.kind == TraceEvent::Kind::Compute) {
                ev.item = r.item;
                ev.layer = r.layer;
                ev.backward = r.backward != 0;
                const bool frozen = r.layer >= 0 && r.layer < m.n_layers && m.blocks[static_cast<std::size_t>(r.layer)].frozen;
                if (train && !ev.backward) ev.compute_activation_bytes = act;
                if (train && ev.backward && ckpt) ev.compute_activation_bytes = act;
                if (train && ev.backward && !frozen) ev.compute_gradient_bytes = m.layer_bytes();
            } else if (ev.kind == TraceEvent::Kind::Stall) {
                ev.reason = "residency";
                ev.item = r.item;
                ev.layer = r.layer;
                ev.backward = r.backward != 0;
            } else {
                ev.moved_weight_bytes = r.weight_bytes;
                ev.moved_activation_bytes = r.activation_bytes;
            }
            out.push_back(std::move(ev));
        }
        return out;
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
#ifdef PIPESIM_B200_TEST_CPU_ONLY_VIA_ORACLE
    // TEST BUILDS ONLY (tests/cpp): StrategyKind::CpuOnly, the reference's host comparison mode,
    // is answered by the linked CPU oracle so the reference's unmodified tests can run their
    // CpuOnly rows; the library itself has no CPU path and rejects CpuOnly.
    if (strategy.kind == StrategyKind::CpuOnly) {
        arena_cfg.validate();
        strategy.validate(model.n_layers);
        RunResult r;
        for (const auto& in : inputs) r.outputs.push_back(reference_forward(model, in));
        r.model = model;
        r.summary.strategy = to_string(strategy.kind);
        r.summary.output_digest = digest_tensors(r.outputs);
        return r;
    }
#endif
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
    r.trace = ex.trace(false, false, model, rows);
    return r;
}

inline RunResult run_train_step(const LayeredModel& model, const Tensor& x, const Tensor& target,
                                const StrategyConfig& strategy, const ArenaConfig& arena_cfg,
                                const TrainConfig& train_cfg) {
    train_cfg.validate();
    if (x.shape.size() != 2 || x.cols() != model.d || x.rows() != train_cfg.batch_size)
        throw std::invalid_argument("run_train_step: x must have shape [batch_size, d]");
    if (!target.same_shape(x)) throw std::invalid_argument("run_train_step: target shape mismatch");
#ifdef PIPESIM_B200_TEST_CPU_ONLY_VIA_ORACLE
    if (strategy.kind == StrategyKind::CpuOnly) {  // TEST BUILDS ONLY (see run_inference)
        arena_cfg.validate();
        strategy.validate(model.n_layers);
        RunResult r;
        r.model = model;
        r.loss = reference_train_step(r.model, x, target, train_cfg.lr).loss;
        r.summary.strategy = to_string(strategy.kind);
        r.summary.output_digest = digest_train(r.loss, r.model);
        r.summary.loss = r.loss;
        r.summary.has_loss = true;
        for (const auto& b : model.blocks)
            if (!b.frozen) r.summary.total_gradient_bytes += b.weight_bytes();
        return r;
    }
#endif
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
    r.trace = ex.trace(true, train_cfg.checkpointing, model, x.rows());
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

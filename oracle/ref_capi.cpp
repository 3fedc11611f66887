// ref_capi.cpp — extern "C" shim over the UNMODIFIED reference library (pipesim), compiled
// together with the reference's own sources from /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libpipesim_ref.so. TEST INFRASTRUCTURE ONLY: it lets
// the Python tests and bench.py's CPU-baseline / --impl reference legs call the real
// reference (model.hpp:54-89, engine.hpp:42-62) through ctypes.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pipesim/engine.hpp"
#include "pipesim/model.hpp"

using namespace pipesim;

namespace {

LayeredModel model_from_flat(int n, int d, const float* W, const float* b, const int* relu,
                             const int* frozen) {
    LayeredModel m;
    m.d = d;
    m.n_layers = n;
    const std::size_t dd = static_cast<std::size_t>(d) * d;
    for (int l = 0; l < n; ++l) {
        LayerBlock blk;
        blk.index = l;
        blk.d = d;
        blk.weight.assign(W + l * dd, W + (l + 1) * dd);
        blk.bias.assign(b + static_cast<std::size_t>(l) * d, b + static_cast<std::size_t>(l + 1) * d);
        blk.activation = (relu && !relu[l]) ? Activation::Identity : Activation::ReLU;
        blk.frozen = frozen ? frozen[l] != 0 : false;
        m.blocks.push_back(std::move(blk));
    }
    return m;
}

Tensor tensor_from(const float* v, std::int64_t rows, int d) {
    return Tensor({rows, d}, std::vector<float>(v, v + rows * d));
}

}  // namespace

extern "C" {

struct ref_summary {
    std::uint64_t peak_bytes, peak_weight_bytes, peak_activation_bytes, peak_gradient_bytes;
    std::uint64_t total_gradient_bytes, n_transfers_h2d, n_transfers_d2h;
    double per_item_time, makespan, total_stall_time, loss;
    char digest[17];
};

int ref_build_model(std::uint64_t seed, int n, int d, int frozen_prefix, float* W, float* b,
                    int* frozen) {
    try {
        LayeredModel m = build_model(seed, n, d, frozen_prefix);
        const std::size_t dd = static_cast<std::size_t>(d) * d;
        for (int l = 0; l < n; ++l) {
            std::memcpy(W + l * dd, m.blocks[l].weight.data(), dd * 4);
            std::memcpy(b + static_cast<std::size_t>(l) * d, m.blocks[l].bias.data(),
                        static_cast<std::size_t>(d) * 4);
            if (frozen) frozen[l] = m.blocks[l].frozen ? 1 : 0;
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return 2;
    }
}

void ref_make_input(std::uint64_t seed, std::uint64_t tag, std::int64_t rows, int d, float* out) {
    Tensor t = make_input(seed, tag, rows, d);
    std::memcpy(out, t.values.data(), t.values.size() * 4);
}

void ref_layer_forward(int d, const float* W, const float* b, int relu, const float* x,
                       std::int64_t rows, float* y) {
    LayeredModel m = model_from_flat(1, d, W, b, &relu, nullptr);
    Tensor out = layer_forward(m.blocks[0], tensor_from(x, rows, d));
    std::memcpy(y, out.values.data(), out.values.size() * 4);
}

void ref_layer_backward(int d, const float* W, const float* b, int relu, const float* x,
                        const float* dy, std::int64_t rows, float* dx, float* dW, float* db) {
    LayeredModel m = model_from_flat(1, d, W, b, &relu, nullptr);
    LayerGrads g = layer_backward(m.blocks[0], tensor_from(x, rows, d), tensor_from(dy, rows, d));
    if (dx) std::memcpy(dx, g.dx.values.data(), g.dx.values.size() * 4);
    if (dW) std::memcpy(dW, g.dW.data(), g.dW.size() * 4);
    if (db) std::memcpy(db, g.db.data(), g.db.size() * 4);
}

void ref_reference_forward(int n, int d, const float* W, const float* b, const int* relu,
                           const float* x, std::int64_t rows, float* y) {
    LayeredModel m = model_from_flat(n, d, W, b, relu, nullptr);
    Tensor out = reference_forward(m, tensor_from(x, rows, d));
    std::memcpy(y, out.values.data(), out.values.size() * 4);
}

float ref_reference_train_step(int n, int d, float* W, float* b, const int* relu,
                               const int* frozen, const float* x, const float* target,
                               std::int64_t rows, float lr, float* dW_all, float* db_all) {
    LayeredModel m = model_from_flat(n, d, W, b, relu, frozen);
    TrainStepResult r = reference_train_step(m, tensor_from(x, rows, d),
                                             tensor_from(target, rows, d), lr);
    const std::size_t dd = static_cast<std::size_t>(d) * d;
    for (int l = 0; l < n; ++l) {
        std::memcpy(W + l * dd, m.blocks[l].weight.data(), dd * 4);
        std::memcpy(b + static_cast<std::size_t>(l) * d, m.blocks[l].bias.data(),
                    static_cast<std::size_t>(d) * 4);
        if (dW_all) {
            if (r.grads[l].dW.empty()) std::memset(dW_all + l * dd, 0, dd * 4);
            else std::memcpy(dW_all + l * dd, r.grads[l].dW.data(), dd * 4);
        }
        if (db_all) {
            float* dst = db_all + static_cast<std::size_t>(l) * d;
            if (r.grads[l].db.empty()) std::memset(dst, 0, static_cast<std::size_t>(d) * 4);
            else std::memcpy(dst, r.grads[l].db.data(), static_cast<std::size_t>(d) * 4);
        }
    }
    return r.loss;
}

static void fill_summary(const RunResult& r, ref_summary* s) {
    s->peak_bytes = r.summary.peak_bytes;
    s->peak_weight_bytes = r.summary.peak_weight_bytes;
    s->peak_activation_bytes = r.summary.peak_activation_bytes;
    s->peak_gradient_bytes = r.summary.peak_gradient_bytes;
    s->total_gradient_bytes = r.summary.total_gradient_bytes;
    s->n_transfers_h2d = r.summary.n_transfers_h2d;
    s->n_transfers_d2h = r.summary.n_transfers_d2h;
    s->per_item_time = r.summary.per_item_time;
    s->makespan = r.summary.makespan;
    s->total_stall_time = r.summary.total_stall_time;
    s->loss = r.summary.loss;
    std::memset(s->digest, 0, sizeof(s->digest));
    std::strncpy(s->digest, r.summary.output_digest.c_str(), 16);
}

static StrategyConfig make_strategy(int kind, int k, int kp, int mode) {
    StrategyConfig s;
    s.kind = static_cast<StrategyKind>(kind);
    s.k = k;
    s.k_prime = kp;
    s.transfer_mode = mode == 0 ? TransferMode::Sequential : TransferMode::Batch;
    return s;
}

static ArenaConfig make_arena(std::uint64_t cap, const double* rates) {
    ArenaConfig a;
    a.capacity_bytes = cap;
    a.h2d_bandwidth = rates[0];
    a.d2h_bandwidth = rates[1];
    a.per_call_latency = rates[2];
    a.device_compute_rate = rates[3];
    a.host_compute_rate = rates[4];
    return a;
}

// Runs the reference engine (engine.cpp:552-556) on flat model/inputs. rates =
// {h2d_bw, d2h_bw, latency, device_rate, host_rate}. Returns 0 ok, 2 invalid, 3 OOM.
int ref_run_inference(int n, int d, const float* W, const float* b, const int* frozen,
                      int n_items, std::int64_t rows, const float* x, int kind, int k, int kp,
                      int mode, std::uint64_t capacity, const double* rates, float* y,
                      ref_summary* summary) {
    try {
        LayeredModel m = model_from_flat(n, d, W, b, nullptr, frozen);
        std::vector<Tensor> inputs;
        for (int i = 0; i < n_items; ++i) inputs.push_back(tensor_from(x + i * rows * d, rows, d));
        RunResult r = run_inference(m, inputs, make_strategy(kind, k, kp, mode),
                                    make_arena(capacity, rates));
        for (int i = 0; i < n_items; ++i)
            std::memcpy(y + i * rows * d, r.outputs[i].values.data(), rows * d * 4);
        fill_summary(r, summary);
        return 0;
    } catch (const OomDeadlockError&) {
        return 3;
    } catch (const std::invalid_argument&) {
        return 2;
    }
}

// Reference training step through the engine (engine.cpp:558-563). W/b updated in place.
int ref_run_train_step(int n, int d, float* W, float* b, const int* frozen, std::int64_t rows,
                       const float* x, const float* target, float lr, int checkpointing,
                       int kind, int k, int kp, int mode, std::uint64_t capacity,
                       const double* rates, ref_summary* summary) {
    try {
        LayeredModel m = model_from_flat(n, d, W, b, nullptr, frozen);
        TrainConfig tc;
        tc.lr = lr;
        tc.checkpointing = checkpointing != 0;
        tc.batch_size = rows;
        RunResult r = run_train_step(m, tensor_from(x, rows, d), tensor_from(target, rows, d),
                                     make_strategy(kind, k, kp, mode), make_arena(capacity, rates),
                                     tc);
        const std::size_t dd = static_cast<std::size_t>(d) * d;
        for (int l = 0; l < n; ++l) {
            std::memcpy(W + l * dd, r.model.blocks[l].weight.data(), dd * 4);
            std::memcpy(b + static_cast<std::size_t>(l) * d, r.model.blocks[l].bias.data(),
                        static_cast<std::size_t>(d) * 4);
        }
        fill_summary(r, summary);
        summary->loss = r.loss;
        return 0;
    } catch (const OomDeadlockError&) {
        return 3;
    } catch (const std::invalid_argument&) {
        return 2;
    }
}

}  // extern "C"

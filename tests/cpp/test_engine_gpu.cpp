// test_engine_gpu.cpp — executor contract tests written against the C++ mirror of the
// reference API (include/pipesim_b200/pipesim.hpp), with the GPU executor behind it. They
// restate the reference's own executor tests (test_engine.cpp:92-118, 154-281, 331-339;
// acceptance.cpp C1/C2/C7) and compare against the CPU oracle (oracle/oracle.h, the C
// restatement of model.cpp — linked here as the checker only).
#include <cmath>
#include <cstring>
#include <random>

#include "../../include/pipesim_b200/pipesim.hpp"
#include "../../oracle/oracle.h"
#include "mini_test.hpp"

using namespace pipesim;

namespace {

ArenaConfig roomy_arena() {
    ArenaConfig a;
    a.capacity_bytes = 1ull << 30;
    return a;
}

StrategyConfig strat(StrategyKind kind, int k = 0, int k_prime = 0,
                     TransferMode mode = TransferMode::Batch) {
    StrategyConfig s;
    s.kind = kind;
    s.k = k;
    s.k_prime = k_prime;
    s.transfer_mode = mode;
    return s;
}

std::vector<Tensor> make_inputs(std::uint64_t seed, int n_items, std::int64_t b, int d) {
    std::vector<Tensor> v;
    for (int i = 0; i < n_items; ++i) v.push_back(make_input(seed, static_cast<std::uint64_t>(i), b, d));
    return v;
}

// Flattened views for the C oracle.
struct Flat {
    std::vector<float> W, b;
    std::vector<int> relu, frozen;
    explicit Flat(const LayeredModel& m) {
        for (const auto& blk : m.blocks) {
            W.insert(W.end(), blk.weight.begin(), blk.weight.end());
            b.insert(b.end(), blk.bias.begin(), blk.bias.end());
            relu.push_back(blk.activation == Activation::ReLU);
            frozen.push_back(blk.frozen);
        }
    }
};

Tensor oracle_forward(const LayeredModel& m, const Tensor& x) {
    Flat f(m);
    Tensor y = Tensor::zeros(x.shape);
    orc_forward(m.n_layers, m.d, f.W.data(), f.b.data(), f.relu.data(), x.values.data(), x.rows(),
                y.values.data());
    return y;
}

float oracle_train_step(LayeredModel& m, const Tensor& x, const Tensor& t, float lr) {
    Flat f(m);
    const float loss = orc_train_step(m.n_layers, m.d, f.W.data(), f.b.data(), f.relu.data(),
                                      f.frozen.data(), x.values.data(), t.values.data(), x.rows(),
                                      lr, nullptr, nullptr, nullptr);
    const std::size_t dd = static_cast<std::size_t>(m.d) * m.d;
    for (int l = 0; l < m.n_layers; ++l) {
        std::memcpy(m.blocks[l].weight.data(), f.W.data() + l * dd, dd * 4);
        std::memcpy(m.blocks[l].bias.data(), f.b.data() + static_cast<std::size_t>(l) * m.d,
                    static_cast<std::size_t>(m.d) * 4);
    }
    return loss;
}

bool same_weights(const LayeredModel& a, const LayeredModel& b) {
    for (std::size_t i = 0; i < a.blocks.size(); ++i)
        if (a.blocks[i].weight != b.blocks[i].weight || a.blocks[i].bias != b.blocks[i].bias)
            return false;
    return true;
}

}  // namespace

TEST_CASE("build_model and make_input match the reference restatement bitwise [cpu]") {
    for (std::uint64_t seed : {1ull, 7ull, 42ull}) {
        LayeredModel m = build_model(seed, 3, 7, 1);
        std::vector<float> W(3 * 49), b(3 * 7);
        orc_build_model(seed, 3, 7, W.data(), b.data());
        for (int l = 0; l < 3; ++l) {
            CHECK(std::memcmp(m.blocks[l].weight.data(), W.data() + l * 49, 49 * 4) == 0);
            CHECK(std::memcmp(m.blocks[l].bias.data(), b.data() + l * 7, 7 * 4) == 0);
        }
        CHECK(m.blocks[0].frozen);
        CHECK_FALSE(m.blocks[1].frozen);
        Tensor x = make_input(seed, 3, 5, 7);
        std::vector<float> xo(35);
        orc_make_input(seed, 3, 5, 7, xo.data());
        CHECK(x.values == xo);
    }
    CHECK(build_model(7, 8, 16, 0).layer_bytes() == 1088);
}

TEST_CASE("input validation mirrors the reference exceptions [cpu]") {
    LayeredModel model = build_model(1, 2, 3, 0);
    ArenaConfig arena = roomy_arena();
    CHECK_THROWS_AS(run_inference(model, {}, strat(StrategyKind::Standard), arena), std::invalid_argument);
    auto bad = make_inputs(1, 1, 1, 4);
    CHECK_THROWS_AS(run_inference(model, bad, strat(StrategyKind::Standard), arena), std::invalid_argument);
    Tensor x = make_input(1, 0, 2, 3);
    Tensor t = make_input(1, 1, 3, 3);
    CHECK_THROWS_AS(run_train_step(model, x, t, strat(StrategyKind::Standard), arena, TrainConfig{0.1f, false, 2}),
                    std::invalid_argument);
    CHECK_THROWS_AS(run_train_step(model, x, x, strat(StrategyKind::Standard), arena, TrainConfig{-1.0f, false, 2}),
                    std::invalid_argument);
    CHECK_THROWS_AS(strat(StrategyKind::Superpipeline, 2, 2).validate(4), std::invalid_argument);
    CHECK_THROWS_AS(build_model(1, 4, 4, 5), std::invalid_argument);
    CHECK(peak_weight_residency(strat(StrategyKind::Superpipeline, 4, 2), 8, 1088) == 6 * 1088);
    CHECK(peak_weight_residency(strat(StrategyKind::Naive, 3), 8, 1088) == 3 * 1088);
}

TEST_CASE("configs/default.json reproduces the reference digest and ledger [gpu]") {
    LayeredModel model = build_model(7, 8, 16, 0);
    auto inputs = make_inputs(7, 4, 1, 16);
    RunResult r = run_inference(model, inputs, strat(StrategyKind::Superpipeline, 4, 2), roomy_arena());
    CHECK(r.summary.output_digest == "046c06b54d8304c5");
    CHECK(r.summary.peak_bytes == 6592);
    CHECK(r.summary.n_transfers_h2d == 15);
    for (std::size_t i = 0; i < inputs.size(); ++i) CHECK(r.outputs[i] == oracle_forward(model, inputs[i]));
}

TEST_CASE("all strategies produce bitwise-identical outputs and digests [gpu]") {
    LayeredModel model = build_model(42, 8, 4, 0);
    auto inputs = make_inputs(42, 3, 2, 4);
    std::string first;
    for (const auto& s : {strat(StrategyKind::Standard), strat(StrategyKind::Naive, 3),
                          strat(StrategyKind::Superpipeline, 3, 1),
                          strat(StrategyKind::Superpipeline, 3, 2, TransferMode::Sequential)}) {
        RunResult r = run_inference(model, inputs, s, roomy_arena());
        REQUIRE(r.outputs.size() == inputs.size());
        for (std::size_t i = 0; i < inputs.size(); ++i) CHECK(r.outputs[i] == oracle_forward(model, inputs[i]));
        if (first.empty()) first = r.summary.output_digest;
        else CHECK(r.summary.output_digest == first);
    }
}

TEST_CASE("verify_fidelity flags a single perturbed bit [gpu]") {
    // test_engine.cpp:120-127
    LayeredModel model = build_model(5, 2, 3, 0);
    auto inputs = make_inputs(5, 1, 1, 3);
    RunResult r = run_inference(model, inputs, strat(StrategyKind::Standard), roomy_arena());
    CHECK(verify_fidelity(r.outputs, model, inputs).ok);
    CHECK(verify_fidelity(r.outputs, model, inputs).digest == r.summary.output_digest);
    r.outputs[0].values[0] = std::nextafter(r.outputs[0].values[0], 1e30f);
    CHECK(!verify_fidelity(r.outputs, model, inputs).ok);
    // a bf16 run is not bit-faithful to the reference: verify_fidelity says so
    set_numerics(Numerics::Bf16);
    LayeredModel wide = build_model(5, 3, 64, 0);
    auto xs = make_inputs(5, 2, 16, 64);
    RunResult rb = run_inference(wide, xs, strat(StrategyKind::Superpipeline, 2, 1), roomy_arena());
    set_numerics(Numerics::Exact);
    CHECK(!verify_fidelity(rb.outputs, wide, xs).ok);
    CHECK(verify_fidelity(run_inference(wide, xs, strat(StrategyKind::Standard), roomy_arena()).outputs,
                          wide, xs).ok);
}

TEST_CASE("train step is bitwise-faithful for every strategy and option [gpu]") {
    for (int frozen_prefix : {0, 2, 4}) {
        LayeredModel ref = build_model(7, 4, 5, frozen_prefix);
        Tensor x = make_input(7, 0, 3, 5);
        Tensor target = make_input(7, 1, 3, 5);
        LayeredModel expected = ref;
        const float expected_loss = oracle_train_step(expected, x, target, 0.02f);
        for (const auto& s : {strat(StrategyKind::Standard), strat(StrategyKind::Naive, 2),
                              strat(StrategyKind::Superpipeline, 2, 1)}) {
            for (bool ckpt : {false, true}) {
                RunResult r = run_train_step(build_model(7, 4, 5, frozen_prefix), x, target, s,
                                             roomy_arena(), TrainConfig{0.02f, ckpt, 3});
                CHECK(std::memcmp(&r.loss, &expected_loss, sizeof(float)) == 0);
                CHECK(same_weights(r.model, expected));
                CHECK(r.summary.has_loss);
            }
        }
    }
}

TEST_CASE("configs/oom_train.json: window fits where standard deadlocks [gpu]") {
    LayeredModel model = build_model(11, 12, 16, 0);
    Tensor x = make_input(11, 0, 4, 16), t = make_input(11, 1, 4, 16);
    ArenaConfig arena;
    arena.capacity_bytes = 15000;
    RunResult r = run_train_step(model, x, t, strat(StrategyKind::Superpipeline, 6, 3), arena,
                                 TrainConfig{0.01f, false, 4});
    CHECK(r.summary.output_digest == "44ab7f18e19ef8b8");
    CHECK(r.summary.peak_bytes == 13952);
    CHECK_THROWS_AS(run_train_step(model, x, t, strat(StrategyKind::Standard), arena, TrainConfig{0.01f, false, 4}),
                    OomDeadlockError);
}

TEST_CASE("fully frozen model trains to an identical model with zero gradient bytes [gpu]") {
    LayeredModel model = build_model(8, 4, 4, 4);
    Tensor x = make_input(8, 0, 2, 4), t = make_input(8, 1, 2, 4);
    RunResult r = run_train_step(model, x, t, strat(StrategyKind::Superpipeline, 2, 1), roomy_arena(),
                                 TrainConfig{0.1f, false, 2});
    CHECK(same_weights(r.model, model));
    CHECK(r.summary.peak_gradient_bytes == 0);
    CHECK(r.summary.total_gradient_bytes == 0);
}

TEST_CASE("checkpointing lowers peak activation bytes at identical loss [gpu]") {
    LayeredModel model = build_model(6, 8, 4, 0);
    Tensor x = make_input(6, 0, 4, 4), t = make_input(6, 1, 4, 4);
    auto s = strat(StrategyKind::Superpipeline, 3, 1);
    RunResult plain = run_train_step(model, x, t, s, roomy_arena(), TrainConfig{0.01f, false, 4});
    RunResult ckpt = run_train_step(model, x, t, s, roomy_arena(), TrainConfig{0.01f, true, 4});
    CHECK(std::memcmp(&plain.loss, &ckpt.loss, sizeof(float)) == 0);
    CHECK(plain.summary.output_digest == ckpt.summary.output_digest);
    CHECK(plain.summary.peak_activation_bytes == 8ull * 4 * 4 * 4);
    CHECK(ckpt.summary.peak_activation_bytes < plain.summary.peak_activation_bytes);
}

TEST_CASE("insufficient capacity is reported as an OOM deadlock [gpu]") {
    LayeredModel model = build_model(2, 4, 3, 0);
    auto inputs = make_inputs(2, 1, 1, 3);
    ArenaConfig arena = roomy_arena();
    for (std::uint64_t cap : {4ull, 100ull, 3ull * 48 + 12}) {
        arena.capacity_bytes = cap;
        CHECK_THROWS_AS(run_inference(model, inputs, strat(StrategyKind::Standard), arena), OomDeadlockError);
    }
    RunResult r = run_inference(model, inputs, strat(StrategyKind::Superpipeline, 2, 1), arena);
    CHECK(r.outputs[0] == oracle_forward(model, inputs[0]));
    CHECK_THROWS_AS(run_inference(model, inputs, strat(StrategyKind::CpuOnly), arena), std::invalid_argument);
}

TEST_CASE("randomized small configs stay faithful (acceptance C1) [gpu]") {
    std::mt19937_64 rng(20240824);
    for (int trial = 0; trial < 15; ++trial) {
        const int n = 1 + static_cast<int>(rng() % 8);
        const int d = 1 + static_cast<int>(rng() % 16);
        const int frozen = static_cast<int>(rng() % (static_cast<unsigned>(n) + 1));
        const std::int64_t b = 1 + static_cast<std::int64_t>(rng() % 3);
        const int items = 1 + static_cast<int>(rng() % 3);
        LayeredModel model = build_model(rng(), n, d, frozen);
        std::vector<StrategyConfig> strategies = {strat(StrategyKind::Standard),
                                                  strat(StrategyKind::Naive, 1 + static_cast<int>(rng() % n))};
        if (n >= 2) {
            const int k = 2 + static_cast<int>(rng() % (n - 1));
            const int kp = 1 + static_cast<int>(rng() % (k - 1));
            strategies.push_back(strat(StrategyKind::Superpipeline, k, kp,
                                       (rng() & 1) ? TransferMode::Sequential : TransferMode::Batch));
        }
        auto inputs = make_inputs(model.seed, items, b, d);
        Tensor x = make_input(model.seed, 1001, b, d), t = make_input(model.seed, 1002, b, d);
        LayeredModel expected = model;
        const float expected_loss = oracle_train_step(expected, x, t, 0.02f);
        for (const auto& s : strategies) {
            RunResult r = run_inference(model, inputs, s, roomy_arena());
            for (std::size_t i = 0; i < inputs.size(); ++i) CHECK(r.outputs[i] == oracle_forward(model, inputs[i]));
            CHECK(r.summary.peak_weight_bytes <= peak_weight_residency(s, n, model.layer_bytes()));
            for (bool ckpt : {false, true}) {
                RunResult rt = run_train_step(model, x, t, s, roomy_arena(), TrainConfig{0.02f, ckpt, b});
                CHECK(std::memcmp(&rt.loss, &expected_loss, sizeof(float)) == 0);
                CHECK(same_weights(rt.model, expected));
            }
        }
    }
}

TEST_CASE("bf16 tensor-core path is window-invariant and close to the reference [gpu]") {
    set_numerics(Numerics::Bf16);
    LayeredModel model = build_model(5, 8, 128, 0);
    auto inputs = make_inputs(5, 1, 256, 128);
    Tensor want = oracle_forward(model, inputs[0]);
    std::vector<float> first;
    for (const auto& s : {strat(StrategyKind::Standard), strat(StrategyKind::Superpipeline, 2, 1),
                          strat(StrategyKind::Superpipeline, 5, 3)}) {
        RunResult r = run_inference(model, inputs, s, roomy_arena());
        if (first.empty()) first = r.outputs[0].values;
        else CHECK(r.outputs[0].values == first);
    }
    float err = 0.0f, ref = 0.0f;
    for (std::size_t i = 0; i < want.values.size(); ++i) {
        err = std::fmax(err, std::fabs(first[i] - want.values[i]));
        ref = std::fmax(ref, std::fabs(want.values[i]));
    }
    CHECK(err / ref <= 2e-2f);
    set_numerics(Numerics::Exact);
}

TEST_CASE("tf32 tensor-core path is window-invariant and within 2e-3 of the reference [gpu]") {
    set_numerics(Numerics::Tf32);
    LayeredModel model = build_model(5, 8, 128, 0);
    auto inputs = make_inputs(5, 1, 256, 128);
    Tensor want = oracle_forward(model, inputs[0]);
    std::vector<float> first;
    for (const auto& s : {strat(StrategyKind::Standard), strat(StrategyKind::Superpipeline, 2, 1),
                          strat(StrategyKind::Naive, 3)}) {
        RunResult r = run_inference(model, inputs, s, roomy_arena());
        if (first.empty()) first = r.outputs[0].values;
        else CHECK(r.outputs[0].values == first);
    }
    float err = 0.0f, ref = 0.0f;
    for (std::size_t i = 0; i < want.values.size(); ++i) {
        err = std::fmax(err, std::fabs(first[i] - want.values[i]));
        ref = std::fmax(ref, std::fabs(want.values[i]));
    }
    CHECK(err / ref <= 2e-3f);
    set_numerics(Numerics::Exact);
}

// The AdamW option through the C ABI a reference-side caller binds (superpipe.h), checked
// bitwise against the oracle: the reference's gradients (orc_train_step on a scratch copy),
// then orc_adamw with the scalars computed in double and rounded once.
TEST_CASE("AdamW through the C ABI is bit-identical to the oracle over several steps [gpu]") {
    const int n = 4, d = 8, rows = 4;
    const float lr = 0.01f, b1 = 0.9f, b2 = 0.999f, eps = 1e-8f, wd = 0.01f;
    LayeredModel model = build_model(3, n, d, 1);
    Tensor x = make_input(3, 0, rows, d), t = make_input(3, 1, rows, d);
    sp_config c{};
    c.n_layers = n;
    c.d = d;
    c.strategy = SP_SUPERPIPELINE;
    c.k = 2;
    c.k_prime = 1;
    c.transfer_mode = SP_BATCH;
    c.numerics = SP_NUMERICS_EXACT;
    sp_exec* ex = nullptr;
    REQUIRE(sp_create(&c, &ex) == SP_OK);
    for (int l = 0; l < n; ++l)
        REQUIRE(sp_register_layer(ex, l, model.blocks[l].weight.data(), model.blocks[l].bias.data(), SP_RELU,
                                  model.blocks[l].frozen ? 1 : 0) == SP_OK);
    CHECK(sp_set_optimizer(ex, SP_OPT_ADAMW, b1, b2, eps, wd) == SP_OK);
    CHECK(sp_set_optimizer(ex, SP_OPT_ADAMW, 1.5f, b2, eps, wd) == SP_ERR_INVALID);
    CHECK(sp_set_optimizer(ex, SP_OPT_ADAMW, b1, b2, eps, wd) == SP_OK);

    Flat f(model);
    const std::size_t dd = static_cast<std::size_t>(d) * d, img = dd + d;
    std::vector<float> m(n * img, 0.0f), v(n * img, 0.0f);
    for (int step = 1; step <= 3; ++step) {
        float loss = 0.0f;
        REQUIRE(sp_train_step(ex, x.values.data(), t.values.data(), rows, lr, &loss) == SP_OK);
        std::vector<float> W(f.W), b(f.b), dW(f.W.size()), db(f.b.size());
        const float want_loss = orc_train_step(n, d, W.data(), b.data(), f.relu.data(), f.frozen.data(),
                                               x.values.data(), t.values.data(), rows, lr, dW.data(),
                                               db.data(), nullptr);
        CHECK(std::memcmp(&loss, &want_loss, 4) == 0);
        const double tt = step;
        const float decay = static_cast<float>(1.0 - static_cast<double>(lr) * wd);
        const float omb1 = static_cast<float>(1.0 - b1), bb2 = b2, omb2 = static_cast<float>(1.0 - b2);
        const float bc2 = static_cast<float>(std::sqrt(1.0 - std::pow(static_cast<double>(b2), tt)));
        const float neg = static_cast<float>(-static_cast<double>(lr) / (1.0 - std::pow(static_cast<double>(b1), tt)));
        for (int l = 0; l < n; ++l) {
            if (f.frozen[l]) continue;
            float* ml = m.data() + l * img;
            float* vl = v.data() + l * img;
            orc_adamw(static_cast<int64_t>(dd), f.W.data() + l * dd, ml, vl, dW.data() + l * dd, decay, omb1, bb2,
                      omb2, bc2, eps, neg);
            orc_adamw(d, f.b.data() + l * d, ml + dd, vl + dd, db.data() + l * d, decay, omb1, bb2, omb2, bc2,
                      eps, neg);
        }
    }
    for (int l = 0; l < n; ++l) {
        std::vector<float> W(dd), b(d), mW(dd), mb(d), vW(dd), vb(d);
        REQUIRE(sp_read_layer(ex, l, W.data(), b.data()) == SP_OK);
        REQUIRE(sp_read_optimizer_state(ex, l, mW.data(), mb.data(), vW.data(), vb.data()) == SP_OK);
        CHECK(std::memcmp(W.data(), f.W.data() + l * dd, dd * 4) == 0);
        CHECK(std::memcmp(b.data(), f.b.data() + l * d, d * 4) == 0);
        CHECK(std::memcmp(mW.data(), m.data() + l * img, dd * 4) == 0);
        CHECK(std::memcmp(mb.data(), m.data() + l * img + dd, d * 4) == 0);
        CHECK(std::memcmp(vW.data(), v.data() + l * img, dd * 4) == 0);
        CHECK(std::memcmp(vb.data(), v.data() + l * img + dd, d * 4) == 0);
    }
    sp_destroy(ex);
}

int main(int argc, char** argv) { return mini::run(argc, argv); }

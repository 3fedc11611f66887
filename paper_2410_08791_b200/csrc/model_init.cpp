// model_init.cpp — layer registration data for the executor: the reference's deterministic
// model and input generators (SplitMix64, model.hpp:40-52; build_model, model.cpp:23-52;
// make_input, model.cpp:186-191), exported through the C ABI so callers can materialise
// synthetic weights layer by layer straight into pinned memory (a 70B-shape model never
// needs a second full copy). Bit-identical to the reference (checked against oracle/).
#include <cmath>
#include <cstdint>

#include "../../include/superpipe.h"

namespace {

struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t s) : state(s) {}
    uint64_t next() {
        state += 0x9E3779B97F4A7C15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

}  // namespace

extern "C" {

int sp_build_layer(uint64_t seed, int32_t index, int32_t d, int32_t fan_in, int32_t fan_out,
                   float* W, float* b) {
    if (index < 0 || d < 1) return SP_ERR_INVALID;
    const int32_t in = fan_in > 0 ? fan_in : d;
    const int32_t out = fan_out > 0 ? fan_out : d;
    // layer_stream_seed (model.cpp:11-14) and the U(+-1/sqrt(d)) draw of build_model.
    SplitMix64 rng(seed ^ (0xA24BAED4963EE407ull * (static_cast<uint64_t>(index) + 1) +
                           0x9FB21C651E98DF25ull));
    const double bound = 1.0 / std::sqrt(static_cast<double>(in));
    const uint64_t nw = static_cast<uint64_t>(in) * static_cast<uint64_t>(out);
    for (uint64_t e = 0; e < nw; ++e) W[e] = static_cast<float>((2.0 * rng.unit() - 1.0) * bound);
    for (int32_t e = 0; e < out; ++e) b[e] = static_cast<float>((2.0 * rng.unit() - 1.0) * bound);
    return SP_OK;
}

void sp_make_input(uint64_t seed, uint64_t tag, int64_t rows, int32_t d, float* out) {
    SplitMix64 rng(seed ^ (0xD6E8FEB86659FD93ull * (tag + 1)));
    const int64_t count = rows * static_cast<int64_t>(d);
    for (int64_t e = 0; e < count; ++e) out[e] = static_cast<float>(2.0 * rng.unit() - 1.0);
}

}  // extern "C"

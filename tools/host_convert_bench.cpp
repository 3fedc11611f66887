// Host fp32 -> bf16 (RNE) conversion throughput, per 48x1600 layer, vs thread count.
// Sizing probe for pipelined host-side wire-image refresh. g++ -O3 -pthread.
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

static inline uint16_t rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

int main() {
    const int n = 48, d = 1600;
    const size_t dd = size_t(d) * d;
    std::vector<float> src(n * dd);
    std::vector<uint16_t> dst(n * dd);
    for (size_t i = 0; i < src.size(); ++i) src[i] = float(int64_t(i * 2654435761u % 100000) - 50000) * 1e-5f;
    std::memset(dst.data(), 0, dst.size() * 2);
    unsigned hw = std::thread::hardware_concurrency();
    printf("hardware_concurrency %u\n", hw);
    for (int T : {1, 2, 4, 8, 16, 32, 48, 64}) {
        if (unsigned(T) > hw) break;
        auto t0 = std::chrono::steady_clock::now();
        for (int L = 0; L < n; ++L) {
            std::vector<std::thread> th;
            const size_t chunk = (dd + T - 1) / T;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    const size_t lo = t * chunk, hi = std::min(dd, lo + chunk);
                    const float* s = src.data() + L * dd;
                    uint16_t* o = dst.data() + L * dd;
                    for (size_t e = lo; e < hi; ++e) o[e] = rne(s[e]);
                });
            for (auto& x : th) x.join();
        }
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        printf("threads %2d: %.3f ms/layer  %.1f GB/s (read+write)\n", T, ms / n, n * dd * 6.0 / ms / 1e6);
    }
    return dst[12345] == 0x1234;
}

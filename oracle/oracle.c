/*
 * oracle.c — plain-C restatement of the reference's layer math. TEST INFRASTRUCTURE
 * ONLY (see oracle.h): the product path never links or calls this file.
 *
 * Evaluation order and rounding follow /root/reference/proj/core/src/model.cpp
 * exactly; build with -ffp-contract=off so every `acc += a*b` stays a separately
 * rounded multiply and add, as in the reference's SSE2 build.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

uint64_t orc_splitmix_next(uint64_t* state) {  /* model.hpp:43-49 */
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double orc_splitmix_unit(uint64_t* state) {  /* model.hpp:51 */
    return (double)(orc_splitmix_next(state) >> 11) * 0x1.0p-53;
}

static uint64_t layer_stream_seed(uint64_t seed, uint64_t index) {  /* model.cpp:11-14 */
    return seed ^ (0xA24BAED4963EE407ull * (index + 1) + 0x9FB21C651E98DF25ull);
}

int orc_build_model(uint64_t seed, int n_layers, int d, float* W, float* b) {
    /* model.cpp:23-52: weights of a layer first, then its bias, from one stream. */
    if (n_layers < 1 || d < 1) return -1;
    const double bound = 1.0 / sqrt((double)d);
    const size_t dd = (size_t)d * (size_t)d;
    for (int i = 0; i < n_layers; ++i) {
        uint64_t st = layer_stream_seed(seed, (uint64_t)i);
        float* w = W + (size_t)i * dd;
        float* bb = b + (size_t)i * (size_t)d;
        for (size_t e = 0; e < dd; ++e) w[e] = (float)((2.0 * orc_splitmix_unit(&st) - 1.0) * bound);
        for (int e = 0; e < d; ++e) bb[e] = (float)((2.0 * orc_splitmix_unit(&st) - 1.0) * bound);
    }
    return 0;
}

void orc_make_input(uint64_t seed, uint64_t tag, int64_t rows, int d, float* out) {
    /* model.cpp:186-191 */
    uint64_t st = seed ^ (0xD6E8FEB86659FD93ull * (tag + 1));
    const int64_t count = rows * (int64_t)d;
    for (int64_t e = 0; e < count; ++e) out[e] = (float)(2.0 * orc_splitmix_unit(&st) - 1.0);
}

void orc_layer_forward(int d, const float* W, const float* b, int relu, const float* x,
                       int64_t rows, float* y) {
    /* model.cpp:54-70: i-ascending fp32 accumulation, bias last, acc<0 -> 0. */
    for (int64_t r = 0; r < rows; ++r) {
        const float* xr = x + r * d;
        for (int j = 0; j < d; ++j) {
            float acc = 0.0f;
            for (int i = 0; i < d; ++i) acc += xr[i] * W[(size_t)i * d + j];
            acc += b[j];
            if (relu && acc < 0.0f) acc = 0.0f;
            y[r * d + j] = acc;
        }
    }
}

void orc_layer_backward(int d, const float* W, const float* b, int relu, const float* x,
                        const float* dy, int64_t rows, float* dx, float* dW, float* db) {
    /* model.cpp:72-123 */
    const int64_t count = rows * (int64_t)d;
    float* dz = (float*)malloc((size_t)count * sizeof(float));
    for (int64_t r = 0; r < rows; ++r) {           /* z recompute + gate, :78-96 */
        for (int j = 0; j < d; ++j) {
            float acc = 0.0f;
            for (int i = 0; i < d; ++i) acc += x[r * d + i] * W[(size_t)i * d + j];
            acc += b[j];
            float g = dy[r * d + j];
            if (relu && acc <= 0.0f) g = 0.0f;
            dz[r * d + j] = g;
        }
    }
    if (dx) {                                        /* dx = dz W^T, j ascending, :98-106 */
        for (int64_t r = 0; r < rows; ++r)
            for (int i = 0; i < d; ++i) {
                float acc = 0.0f;
                for (int j = 0; j < d; ++j) acc += dz[r * d + j] * W[(size_t)i * d + j];
                dx[r * d + i] = acc;
            }
    }
    if (dW) {                                        /* dW = x^T dz, r ascending, :108-114 */
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) {
                float acc = 0.0f;
                for (int64_t r = 0; r < rows; ++r) acc += x[r * d + i] * dz[r * d + j];
                dW[(size_t)i * d + j] = acc;
            }
    }
    if (db) {                                        /* db = sum_r dz, :116-121 */
        for (int j = 0; j < d; ++j) {
            float acc = 0.0f;
            for (int64_t r = 0; r < rows; ++r) acc += dz[r * d + j];
            db[j] = acc;
        }
    }
    free(dz);
}

float orc_mse_loss(const float* y, const float* t, int64_t count) {  /* model.cpp:131-140 */
    float acc = 0.0f;
    for (int64_t i = 0; i < count; ++i) {
        const float e = y[i] - t[i];
        acc += e * e;
    }
    return acc / (float)count;
}

void orc_mse_grad(const float* y, const float* t, int64_t count, float* g) {  /* :142-148 */
    const float inv_n = 1.0f / (float)count;
    for (int64_t i = 0; i < count; ++i) g[i] = 2.0f * (y[i] - t[i]) * inv_n;
}

void orc_apply_sgd(float* w, const float* g, int64_t count, float lr) {  /* :150-155 */
    for (int64_t i = 0; i < count; ++i) w[i] -= lr * g[i];
}

void orc_adamw(int64_t count, float* w, float* m, float* v, const float* g, float decay,
               float omb1, float b2, float omb2, float bc2_sqrt, float eps, float neg_step) {
    for (int64_t i = 0; i < count; ++i) {
        const float gi = g[i];
        const float wi = w[i] * decay;
        const float mi = m[i] + omb1 * (gi - m[i]);
        const float vi = v[i] * b2 + (omb2 * gi) * gi;
        const float denom = sqrtf(vi) / bc2_sqrt + eps;
        w[i] = wi + neg_step * (mi / denom);
        m[i] = mi;
        v[i] = vi;
    }
}

void orc_forward(int n_layers, int d, const float* W, const float* b, const int* relu,
                 const float* x, int64_t rows, float* y) {  /* model.cpp:125-129 */
    const int64_t count = rows * (int64_t)d;
    float* cur = (float*)malloc((size_t)count * sizeof(float));
    float* nxt = (float*)malloc((size_t)count * sizeof(float));
    memcpy(cur, x, (size_t)count * sizeof(float));
    const size_t dd = (size_t)d * (size_t)d;
    for (int l = 0; l < n_layers; ++l) {
        orc_layer_forward(d, W + l * dd, b + (size_t)l * d, relu ? relu[l] : 1, cur, rows, nxt);
        float* t = cur; cur = nxt; nxt = t;
    }
    memcpy(y, cur, (size_t)count * sizeof(float));
    free(cur);
    free(nxt);
}

float orc_train_step(int n_layers, int d, float* W, float* b, const int* relu,
                     const int* frozen, const float* x, const float* target, int64_t rows,
                     float lr, float* dW_all, float* db_all, float* dx0) {
    /* model.cpp:157-184: forward saving inputs, MSE, reverse backward + SGD. */
    const int64_t count = rows * (int64_t)d;
    const size_t dd = (size_t)d * (size_t)d;
    float* acts = (float*)malloc((size_t)(n_layers + 1) * (size_t)count * sizeof(float));
    memcpy(acts, x, (size_t)count * sizeof(float));
    for (int l = 0; l < n_layers; ++l)
        orc_layer_forward(d, W + l * dd, b + (size_t)l * d, relu ? relu[l] : 1,
                          acts + (size_t)l * count, rows, acts + (size_t)(l + 1) * count);
    const float* y = acts + (size_t)n_layers * count;
    const float loss = orc_mse_loss(y, target, count);
    float* dy = (float*)malloc((size_t)count * sizeof(float));
    float* dx = (float*)malloc((size_t)count * sizeof(float));
    float* dW = (float*)malloc(dd * sizeof(float));
    float* db = (float*)malloc((size_t)d * sizeof(float));
    orc_mse_grad(y, target, count, dy);
    if (dW_all) memset(dW_all, 0, (size_t)n_layers * dd * sizeof(float));
    if (db_all) memset(db_all, 0, (size_t)n_layers * (size_t)d * sizeof(float));
    for (int l = n_layers - 1; l >= 0; --l) {
        float* Wl = W + l * dd;
        float* bl = b + (size_t)l * d;
        const int fz = frozen ? frozen[l] : 0;
        orc_layer_backward(d, Wl, bl, relu ? relu[l] : 1, acts + (size_t)l * count, dy, rows,
                           dx, dW, db);
        if (!fz) {
            if (dW_all) memcpy(dW_all + l * dd, dW, dd * sizeof(float));
            if (db_all) memcpy(db_all + (size_t)l * d, db, (size_t)d * sizeof(float));
            orc_apply_sgd(Wl, dW, (int64_t)dd, lr);
            orc_apply_sgd(bl, db, d, lr);
        }
        float* t = dy; dy = dx; dx = t;
    }
    if (dx0) memcpy(dx0, dy, (size_t)count * sizeof(float));
    free(acts); free(dy); free(dx); free(dW); free(db);
    return loss;
}

uint64_t orc_fnv1a64(const void* data, uint64_t size, uint64_t h) {  /* engine.cpp:14-21 */
    const unsigned char* p = (const unsigned char*)data;
    for (uint64_t i = 0; i < size; ++i) {
        h ^= p[i];
        h *= 0x100000001B3ull;
    }
    return h;
}

uint64_t orc_digest_tensors(int n_items, int64_t rows, int d, const float* values) {
    /* engine.cpp:565-572: per tensor, the int64 shape bytes then the fp32 values. */
    uint64_t h = 0xCBF29CE484222325ull;
    const int64_t shape[2] = {rows, (int64_t)d};
    const int64_t count = rows * (int64_t)d;
    for (int t = 0; t < n_items; ++t) {
        h = orc_fnv1a64(shape, sizeof(shape), h);
        h = orc_fnv1a64(values + (size_t)t * count, (uint64_t)count * sizeof(float), h);
    }
    return h;
}

uint64_t orc_digest_train(float loss, int n_layers, int d, const float* W, const float* b) {
    /* engine.cpp:574-581: loss bytes, then each block's weight then bias. */
    uint64_t h = orc_fnv1a64(&loss, sizeof(loss), 0xCBF29CE484222325ull);
    const size_t dd = (size_t)d * (size_t)d;
    for (int l = 0; l < n_layers; ++l) {
        h = orc_fnv1a64(W + l * dd, dd * sizeof(float), h);
        h = orc_fnv1a64(b + (size_t)l * d, (size_t)d * sizeof(float), h);
    }
    return h;
}

void orc_to_hex(uint64_t v, char out[17]) {  /* engine.cpp:23-31 */
    static const char digits[] = "0123456789abcdef";
    for (int i = 15; i >= 0; --i) {
        out[i] = digits[v & 0xF];
        v >>= 4;
    }
    out[16] = '\0';
}

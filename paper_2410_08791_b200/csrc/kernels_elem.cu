// kernels_elem.cu — HBM-bound elementwise / reduction kernels of the bf16 path.
//
// All reductions use a fixed decomposition that depends only on the problem size (never on
// slot addresses, stream timing or the (k, k') window), so the bf16 path is bit-identical
// across every window setting. 128-bit vectorised loads/stores; grids sized in multiples of
// the SM count.
#include <cuda_bf16.h>

#include "kernels.hpp"
#include "launch.cuh"

namespace sp {
namespace {

constexpr int kThreads = 256;

__global__ void convert_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                               int64_t count) {
    const int64_t n4 = count / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 v = reinterpret_cast<const float4*>(src)[i];
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 packed;
        packed.x = *reinterpret_cast<uint32_t*>(&lo);
        packed.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(dst)[i] = packed;
    }
    for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
        dst[i] = __float2bfloat16_rn(src[i]);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float block_sum(float v) {
    __shared__ float red[kThreads / 32];
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float s = 0.0f;
    if (warp == 0) {
        s = lane < kThreads / 32 ? red[lane] : 0.0f;
        s = warp_sum(s);
    }
    return s;  // valid in thread 0
}

__device__ __forceinline__ float grad_elem(float y, float t, float inv_n, int relu) {
    float g = __fmul_rn(__fmul_rn(2.0f, __fsub_rn(y, t)), inv_n);
    if (relu && y <= 0.0f) g = 0.0f;
    return g;
}

__device__ __forceinline__ void store_grad4(__nv_bfloat16* g, int64_t i, float a, float b, float c, float d) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(a, b);
    __nv_bfloat162 hi = __floats2bfloat162_rn(c, d);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&lo);
    packed.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(g)[i] = packed;
}
__device__ __forceinline__ void store_grad4(float* g, int64_t i, float a, float b, float c, float d) {
    reinterpret_cast<float4*>(g)[i] = make_float4(a, b, c, d);
}
__device__ __forceinline__ void store_grad1(__nv_bfloat16* g, int64_t i, float a) { g[i] = __float2bfloat16_rn(a); }
__device__ __forceinline__ void store_grad1(float* g, int64_t i, float a) { g[i] = a; }

// Fused MSE: per-block partial sums of e^2 and g = 2 e / N gated by the last ReLU, stored as
// T (bf16 for the bf16 path, fp32 for tf32).
template <typename T>
__global__ void loss_grad_kernel(const float* __restrict__ y, const float* __restrict__ t,
                                 int64_t count, float inv_n, int relu,
                                 T* __restrict__ g, float* __restrict__ partials) {
    const int64_t n4 = count / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    float acc = 0.0f;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 yv = reinterpret_cast<const float4*>(y)[i];
        const float4 tv = reinterpret_cast<const float4*>(t)[i];
        const float e0 = yv.x - tv.x, e1 = yv.y - tv.y, e2 = yv.z - tv.z, e3 = yv.w - tv.w;
        acc += e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3;
        store_grad4(g, i, grad_elem(yv.x, tv.x, inv_n, relu), grad_elem(yv.y, tv.y, inv_n, relu),
                    grad_elem(yv.z, tv.z, inv_n, relu), grad_elem(yv.w, tv.w, inv_n, relu));
    }
    for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float e = y[i] - t[i];
        acc += e * e;
        store_grad1(g, i, grad_elem(y[i], t[i], inv_n, relu));
    }
    const float s = block_sum(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void finalize_kernel(const float* __restrict__ partials, int n, float* __restrict__ out) {
    float acc = 0.0f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
    const float s = block_sum(acc);
    if (threadIdx.x == 0) *out = s;
}

// Column sums (db = sum_r dz[r, :]) of a bf16 [rows][d] matrix. Block = 32 column-groups of
// 8 columns (one 16-byte load each) x 8 row-lanes; a block owns kColRows consecutive rows,
// each row-lane sums kColRows/8 rows with independent unrolled loads, then the 8 lanes are
// combined in a fixed order in shared memory -> partials[chunk][d]. Deterministic.
constexpr int kColRows = 128;
constexpr int kColLanes = 8;

__global__ void __launch_bounds__(256) colsum_kernel(const __nv_bfloat16* __restrict__ x,
                                                     int64_t rows, int d,
                                                     float* __restrict__ partials) {
    __shared__ float red[kColLanes][32][9];
    const int g = blockIdx.x * 32 + threadIdx.x;  // 8-column group
    const int lane_r = threadIdx.y;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kColRows;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    if (8 * g < d) {
        constexpr int per = kColRows / kColLanes;
        uint4 v[per];
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int64_t r = r0 + lane_r + static_cast<int64_t>(i) * kColLanes;
            v[i] = r < rows ? __ldg(reinterpret_cast<const uint4*>(x + r * d) + g) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
                acc[2 * h] += f.x;
                acc[2 * h + 1] += f.y;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) red[lane_r][threadIdx.x][i] = acc[i];
    __syncthreads();
    if (lane_r == 0 && 8 * g < d) {
        float out[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float s = red[0][threadIdx.x][i];
            for (int l = 1; l < kColLanes; ++l) s += red[l][threadIdx.x][i];
            out[i] = s;
        }
        float4* dst = reinterpret_cast<float4*>(partials + static_cast<int64_t>(blockIdx.y) * d + 8 * g);
        dst[0] = make_float4(out[0], out[1], out[2], out[3]);
        dst[1] = make_float4(out[4], out[5], out[6], out[7]);
    }
}

// The same for an fp32 [rows][d] matrix (tf32 path): 32 groups of 4 columns x 8 row-lanes.
__global__ void __launch_bounds__(256) colsum_f32_kernel(const float* __restrict__ x, int64_t rows,
                                                         int d, float* __restrict__ partials) {
    __shared__ float red[kColLanes][32][5];
    const int g = blockIdx.x * 32 + threadIdx.x;  // 4-column group
    const int lane_r = threadIdx.y;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kColRows;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (4 * g < d) {
        constexpr int per = kColRows / kColLanes;
        float4 v[per];
#pragma unroll
        for (int i = 0; i < per; ++i) {
            const int64_t r = r0 + lane_r + static_cast<int64_t>(i) * kColLanes;
            v[i] = r < rows ? __ldg(reinterpret_cast<const float4*>(x + r * d) + g) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < per; ++i) {
            acc[0] += v[i].x;
            acc[1] += v[i].y;
            acc[2] += v[i].z;
            acc[3] += v[i].w;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) red[lane_r][threadIdx.x][i] = acc[i];
    __syncthreads();
    if (lane_r == 0 && 4 * g < d) {
        float out[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float s = red[0][threadIdx.x][i];
            for (int l = 1; l < kColLanes; ++l) s += red[l][threadIdx.x][i];
            out[i] = s;
        }
        reinterpret_cast<float4*>(partials + static_cast<int64_t>(blockIdx.y) * d)[g] =
            make_float4(out[0], out[1], out[2], out[3]);
    }
}

__global__ void reduce_kernel(const float* __restrict__ parts, int nparts, int64_t stride,
                              int64_t count, float* __restrict__ grad) {
    const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool vec = stride % 4 == 0 && ((reinterpret_cast<uintptr_t>(parts) | reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    const int64_t n4 = vec ? count / 4 : 0;
    for (int64_t i = t0; i < n4; i += gs) {
        float4 s = __ldg(reinterpret_cast<const float4*>(parts) + i);
        for (int p = 1; p < nparts; ++p) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(parts + p * stride) + i);
            s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
        }
        reinterpret_cast<float4*>(grad)[i] = s;
    }
    for (int64_t i = 4 * n4 + t0; i < count; i += gs) {
        float s = parts[i];
        for (int p = 1; p < nparts; ++p) s += parts[p * stride + i];
        grad[i] = s;
    }
}

__global__ void sgd_reduce_kernel(float* __restrict__ w, const float* __restrict__ parts,
                                  int nparts, int64_t stride, int64_t count, float lr) {
    const int64_t n4 = (stride % 4 == 0) ? count / 4 : 0;
    const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += gs) {
        float4 s = reinterpret_cast<const float4*>(parts)[i];
        for (int p = 1; p < nparts; ++p) {
            const float4 v = reinterpret_cast<const float4*>(parts + p * stride)[i];
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
        float4 wv = reinterpret_cast<float4*>(w)[i];
        wv.x = __fsub_rn(wv.x, __fmul_rn(lr, s.x));
        wv.y = __fsub_rn(wv.y, __fmul_rn(lr, s.y));
        wv.z = __fsub_rn(wv.z, __fmul_rn(lr, s.z));
        wv.w = __fsub_rn(wv.w, __fmul_rn(lr, s.w));
        reinterpret_cast<float4*>(w)[i] = wv;
    }
    for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += gs) {
        float s = parts[i];
        for (int p = 1; p < nparts; ++p) s += parts[p * stride + i];
        w[i] = __fsub_rn(w[i], __fmul_rn(lr, s));
    }
}

__device__ __forceinline__ void adamw_elem(float& w, float& m, float& v, float g, const AdamwScalars& s) {
    const float wi = __fmul_rn(w, s.decay);
    const float mi = __fadd_rn(m, __fmul_rn(s.omb1, __fsub_rn(g, m)));
    const float vi = __fadd_rn(__fmul_rn(v, s.b2), __fmul_rn(__fmul_rn(s.omb2, g), g));
    const float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(vi), s.bc2_sqrt), s.eps);
    w = __fadd_rn(wi, __fmul_rn(s.neg_step, __fdiv_rn(mi, denom)));
    m = mi;
    v = vi;
}

__global__ void adamw_reduce_kernel(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
                                    const float* __restrict__ parts, int nparts, int64_t stride,
                                    int64_t count, const AdamwScalars* __restrict__ sc) {
    const AdamwScalars s = *sc;
    const int64_t n4 = (stride % 4 == 0) ? count / 4 : 0;
    const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += gs) {
        float4 g = reinterpret_cast<const float4*>(parts)[i];
        for (int p = 1; p < nparts; ++p) {
            const float4 q = reinterpret_cast<const float4*>(parts + p * stride)[i];
            g.x = __fadd_rn(g.x, q.x);
            g.y = __fadd_rn(g.y, q.y);
            g.z = __fadd_rn(g.z, q.z);
            g.w = __fadd_rn(g.w, q.w);
        }
        float4 wv = reinterpret_cast<float4*>(w)[i], mv = reinterpret_cast<float4*>(m)[i],
               vv = reinterpret_cast<float4*>(v)[i];
        adamw_elem(wv.x, mv.x, vv.x, g.x, s);
        adamw_elem(wv.y, mv.y, vv.y, g.y, s);
        adamw_elem(wv.z, mv.z, vv.z, g.z, s);
        adamw_elem(wv.w, mv.w, vv.w, g.w, s);
        reinterpret_cast<float4*>(w)[i] = wv;
        reinterpret_cast<float4*>(m)[i] = mv;
        reinterpret_cast<float4*>(v)[i] = vv;
    }
    for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += gs) {
        float g = parts[i];
        for (int p = 1; p < nparts; ++p) g = __fadd_rn(g, parts[p * stride + i]);
        adamw_elem(w[i], m[i], v[i], g, s);
    }
}

// w[j] -= lr * sum_p parts[p*stride + j] for a short vector (the bias) with many partials:
// 32 columns x 8 lanes per block, each lane sums every 8th partial, lanes combined in a fixed
// order. Deterministic and latency-tolerant (independent loads per lane).
__global__ void __launch_bounds__(256) sgd_reduce_narrow_kernel(float* __restrict__ w,
                                                                const float* __restrict__ parts,
                                                                int nparts, int64_t stride,
                                                                int64_t count, float lr) {
    __shared__ float red[8][33];
    const int64_t j = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
    float s = 0.0f;
    if (j < count)
        for (int p = threadIdx.y; p < nparts; p += 8) s += parts[p * stride + j];
    red[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && j < count) {
        float t = red[0][threadIdx.x];
        for (int l = 1; l < 8; ++l) t += red[l][threadIdx.x];
        w[j] = __fsub_rn(w[j], __fmul_rn(lr, t));
    }
}

__global__ void scale_kernel(float* __restrict__ x, int64_t count, float s) {
    const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += gs)
        x[i] *= s;
}

unsigned grid_for(int64_t items) {
    const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
    const int64_t need = (items + kThreads - 1) / kThreads;
    return static_cast<unsigned>(need < 1 ? 1 : (need < cap ? need : cap));
}

}  // namespace

int num_sms() {
    static int sms = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return sms;
}

void convert_f32_to_bf16(const float* src, void* dst, int64_t count, cudaStream_t st) {
    launch_kernel(convert_kernel, dim3(grid_for(count / 4 + 1)), dim3(kThreads), 0, st, src,
               static_cast<__nv_bfloat16*>(dst), count);
}

int loss_grad_bf16(const float* y, const float* t, int64_t count, float inv_n, int relu,
                   void* g, float* partials, cudaStream_t st) {
    // Fixed grid (a function of count only) => a fixed summation tree.
    const int64_t need = (count / 4 + kThreads) / kThreads;
    const int blocks = static_cast<int>(need < 1 ? 1 : (need < 1184 ? need : 1184));
    launch_kernel(loss_grad_kernel<__nv_bfloat16>, dim3(blocks), dim3(kThreads), 0, st, y, t, count, inv_n,
               relu, static_cast<__nv_bfloat16*>(g), partials);
    return blocks;
}

int loss_grad_f32(const float* y, const float* t, int64_t count, float inv_n, int relu,
                  float* g, float* partials, cudaStream_t st) {
    const int64_t need = (count / 4 + kThreads) / kThreads;
    const int blocks = static_cast<int>(need < 1 ? 1 : (need < 1184 ? need : 1184));
    launch_kernel(loss_grad_kernel<float>, dim3(blocks), dim3(kThreads), 0, st, y, t, count, inv_n, relu, g,
               partials);
    return blocks;
}

void loss_finalize(const float* partials, int n, float* out, cudaStream_t st) {
    launch_kernel(finalize_kernel, dim3(1), dim3(kThreads), 0, st, partials, n, out);
}

int colsum_chunks(int64_t rows) { return static_cast<int>((rows + kColRows - 1) / kColRows); }

int colsum_bf16(const void* x, int64_t rows, int d, float* partials, cudaStream_t st) {
    const int chunks = colsum_chunks(rows);  // requires d % 8 == 0 (bf16 path: d % 64 == 0)
    dim3 grid((d / 8 + 31) / 32, chunks);
    launch_kernel(colsum_kernel, grid, dim3(32, kColLanes), 0, st,
               static_cast<const __nv_bfloat16*>(x), rows, d, partials);
    return chunks;
}

int colsum_f32(const float* x, int64_t rows, int d, float* partials, cudaStream_t st) {
    const int chunks = colsum_chunks(rows);  // requires d % 4 == 0
    dim3 grid((d / 4 + 31) / 32, chunks);
    launch_kernel(colsum_f32_kernel, grid, dim3(32, kColLanes), 0, st, x, rows, d, partials);
    return chunks;
}

void reduce_partials(const float* parts, int nparts, int64_t stride, int64_t count,
                     float* grad, cudaStream_t st) {
    launch_kernel(reduce_kernel, dim3(grid_for(count / 4 + 1)), dim3(kThreads), 0, st, parts, nparts, stride,
               count, grad);
}

void sgd_reduce(float* w, const float* parts, int nparts, int64_t stride, int64_t count,
                float lr, cudaStream_t st) {
    if (count <= 65536 && nparts > 8) {  // short vector, many partials (bias from colsum)
        launch_kernel(sgd_reduce_narrow_kernel, dim3(static_cast<unsigned>((count + 31) / 32)),
                   dim3(32, 8), 0, st, w, parts, nparts, stride, count, lr);
        return;
    }
    launch_kernel(sgd_reduce_kernel, dim3(grid_for(count / 4 + 1)), dim3(kThreads), 0, st, w, parts,
               nparts, stride, count, lr);
}

void adamw_reduce(float* w, float* m, float* v, const float* parts, int nparts, int64_t stride,
                  int64_t count, const AdamwScalars* scalars, cudaStream_t st) {
    launch_kernel(adamw_reduce_kernel, dim3(grid_for(count / 4 + 1)), dim3(kThreads), 0, st, w, m, v,
               parts, nparts, stride, count, scalars);
}

// Up to three equal-size device copies in one launch (blockIdx.y = region) on the SMs: the
// write-back staging copy must not queue on a copy engine the PCIe transfers are using.
struct CopyRegions {
    void* dst[3];
    const void* src[3];
};

__global__ void copy_regions_kernel(CopyRegions r, int64_t bytes) {
    const int k = blockIdx.y;
    const int64_t n16 = bytes / 16;
    const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint4* s = static_cast<const uint4*>(r.src[k]);
    uint4* d = static_cast<uint4*>(r.dst[k]);
    for (int64_t i = t0; i < n16; i += gs) d[i] = s[i];
    const uint32_t* s4 = static_cast<const uint32_t*>(r.src[k]);
    uint32_t* d4 = static_cast<uint32_t*>(r.dst[k]);
    for (int64_t i = n16 * 4 + t0; i < bytes / 4; i += gs) d4[i] = s4[i];
}

void copy_regions(void* const* dst, const void* const* src, int n, int64_t bytes, cudaStream_t st) {
    if (n < 1 || bytes <= 0) return;
    CopyRegions r{};
    for (int k = 0; k < n && k < 3; ++k) {
        r.dst[k] = dst[k];
        r.src[k] = src[k];
    }
    const int64_t n16 = bytes / 16 + 1;
    const int blocks = static_cast<int>(std::min<int64_t>((n16 + kThreads - 1) / kThreads, 296));
    launch_kernel(copy_regions_kernel, dim3(blocks, std::min(n, 3)), dim3(kThreads), 0, st, r, bytes);
}

void scale_inplace(float* x, int64_t count, float s, cudaStream_t st) {
    launch_kernel(scale_kernel, dim3(grid_for(count)), dim3(kThreads), 0, st, x, count, s);
}

namespace {
__global__ void convert_regions_kernel(ConvertRegions r) {
    const int i = blockIdx.y;
    const int64_t n4 = r.count[i] / 4;
    const float4* src = reinterpret_cast<const float4*>(r.src[i]);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    if (r.to_bf16[i]) {
        uint2* dst = static_cast<uint2*>(r.dst[i]);
        for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n4; e += stride) {
            const float4 v = src[e];
            __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            dst[e] = pk;
        }
    } else {
        float4* dst = static_cast<float4*>(r.dst[i]);
        for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n4; e += stride) dst[e] = src[e];
    }
}
}  // namespace

void convert_regions(const ConvertRegions& r, cudaStream_t st) {
    if (r.n <= 0) return;
    int64_t most = 0;
    for (int i = 0; i < r.n; ++i) most = most > r.count[i] ? most : r.count[i];
    const unsigned bx = static_cast<unsigned>(grid_for(most / 4 + 1));
    launch_kernel(convert_regions_kernel, dim3(bx, static_cast<unsigned>(r.n)), dim3(kThreads), 0, st, r);
}

namespace {
// Eight parameters per thread of region blockIdx.y (every region is 256-byte aligned and a
// multiple of 64 elements, block.cpp): rebuild the fp32 master from its halves (or read the
// fp32 vector), take the gradient from g, or as the fixed-order sum of the region's split-K
// partials, apply the update in the reference's order, and store it back split.
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

template <typename T>
__device__ __forceinline__ T* shifted(T* p, int64_t bytes) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(p) + bytes);
}

__global__ void split_update_kernel(SplitRegions r, const float* __restrict__ g, float* __restrict__ m,
                                    float* __restrict__ v, float lr, int opt, const AdamwScalars* __restrict__ sc) {
    const int i = blockIdx.y;
    const int64_t n8 = r.count[i] / 8;
    const int64_t base = r.off[i];
    const bool matrix = r.lo[i] != nullptr;
    const float* parts = r.parts[i];
    const int np = r.nparts[i];
    AdamwScalars s{};
    if (opt == 1) s = *sc;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e8 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e8 < n8; e8 += stride) {
        const int64_t e = 8 * e8;
        float w[8], gr[8];
        if (matrix) {
            const uint4 hv = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(r.hi[i]) + e);
            const uint4 lv = *reinterpret_cast<const uint4*>(r.lo[i] + e);
            const uint32_t h4[4] = {hv.x, hv.y, hv.z, hv.w}, l4[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                w[2 * k] = __uint_as_float((h4[k] << 16) | (l4[k] & 0xFFFFu));
                w[2 * k + 1] = __uint_as_float((h4[k] & 0xFFFF0000u) | (l4[k] >> 16));
            }
        } else {
            load8(static_cast<const float*>(r.hi[i]) + e, w);
        }
        if (parts) {
            load8(parts + e, gr);
            for (int p = 1; p < np; ++p) {
                float q[8];
                load8(parts + static_cast<int64_t>(p) * r.count[i] + e, q);
#pragma unroll
                for (int k = 0; k < 8; ++k) gr[k] += q[k];
            }
        } else {
            load8(g + base + e, gr);
        }
        if (opt == 1) {
            float mm[8], vv[8];
            load8(m + base + e, mm);
            load8(v + base + e, vv);
#pragma unroll
            for (int k = 0; k < 8; ++k) adamw_elem(w[k], mm[k], vv[k], gr[k], s);
            if (!r.stage_only) {
                store8(m + base + e, mm);
                store8(v + base + e, vv);
            }
            if (r.stage_delta) {
                store8(shifted(m + base + e, r.stage_delta), mm);
                store8(shifted(v + base + e, r.stage_delta), vv);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) w[k] = __fsub_rn(w[k], __fmul_rn(lr, gr[k]));
        }
        if (matrix) {
            uint32_t h4[4], l4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t b0 = __float_as_uint(w[2 * k]), b1 = __float_as_uint(w[2 * k + 1]);
                h4[k] = (b0 >> 16) | (b1 & 0xFFFF0000u);
                l4[k] = (b0 & 0xFFFFu) | (b1 << 16);
            }
            const uint4 hv = make_uint4(h4[0], h4[1], h4[2], h4[3]), lv = make_uint4(l4[0], l4[1], l4[2], l4[3]);
            if (!r.stage_only) {
                *reinterpret_cast<uint4*>(static_cast<uint16_t*>(r.hi[i]) + e) = hv;
                *reinterpret_cast<uint4*>(r.lo[i] + e) = lv;
            }
            if (r.stage_delta) {
                *shifted(reinterpret_cast<uint4*>(static_cast<uint16_t*>(r.hi[i]) + e), r.stage_delta) = hv;
                *shifted(reinterpret_cast<uint4*>(r.lo[i] + e), r.stage_delta) = lv;
            }
        } else {
            if (!r.stage_only) store8(static_cast<float*>(r.hi[i]) + e, w);
            if (r.stage_delta) store8(shifted(static_cast<float*>(r.hi[i]) + e, r.stage_delta), w);
        }
    }
}
}  // namespace

void split_update(const SplitRegions& r, const float* g, float* m, float* v, float lr, int opt,
                  const AdamwScalars* scalars, cudaStream_t st) {
    if (r.n <= 0) return;
    int64_t most = 0;
    for (int i = 0; i < r.n; ++i) most = most > r.count[i] ? most : r.count[i];
    launch_kernel(split_update_kernel, dim3(grid_for((most + 7) / 8), static_cast<unsigned>(r.n)), dim3(kThreads), 0,
                  st, r, g, m, v, lr, opt, scalars);
}

}  // namespace sp

// kernels_block.cu — normalisation kernels of the named-shape transformer blocks (sm_100a).
//
// LayerNorm / RMSNorm forward (fp32 residual stream in, bf16 GEMM operand out) and backward
// (fused with the residual-gradient add and the bf16 copy the next dW / dX GEMMs read), plus
// the fixed-decomposition column partials of the norm's parameter gradients. One warp per row,
// 128-bit loads; every reduction has a fixed order, so results depend only on the shapes.
#include <cuda_bf16.h>

#include "kernels.hpp"
#include "launch.cuh"

namespace sp {
namespace {

constexpr int kRowsPerBlock = 8;  // one warp per row
constexpr int kChunkRows = 512;   // column-sum partials: rows per chunk
constexpr int kRowLanes = 8;

__device__ __forceinline__ float warp_allsum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <bool RMS>
__global__ void __launch_bounds__(32 * kRowsPerBlock) norm_fwd_kernel(const float* __restrict__ x,
                                                                      const float* __restrict__ gamma,
                                                                      const float* __restrict__ beta, float eps,
                                                                      int64_t rows, int d,
                                                                      __nv_bfloat16* __restrict__ y,
                                                                      float* __restrict__ stats) {
    const int lane = threadIdx.x & 31;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float4* xr = reinterpret_cast<const float4*>(x + r * d);
    const int n4 = d / 4;
    float mean = 0.0f;
    if (!RMS) {
        float s = 0.0f;
        for (int i = lane; i < n4; i += 32) {
            const float4 v = __ldg(xr + i);
            s += (v.x + v.y) + (v.z + v.w);
        }
        mean = warp_allsum(s) / static_cast<float>(d);
    }
    float q = 0.0f;
    for (int i = lane; i < n4; i += 32) {
        const float4 v = __ldg(xr + i);
        const float a = v.x - mean, b = v.y - mean, c = v.z - mean, e = v.w - mean;
        q += (a * a + b * b) + (c * c + e * e);
    }
    const float rstd = rsqrtf(warp_allsum(q) / static_cast<float>(d) + eps);
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    const float4* b4 = reinterpret_cast<const float4*>(beta);
    uint2* yr = reinterpret_cast<uint2*>(y + r * d);
    for (int i = lane; i < n4; i += 32) {
        const float4 v = __ldg(xr + i);
        const float4 g = __ldg(g4 + i);
        float4 o;
        o.x = (v.x - mean) * rstd * g.x;
        o.y = (v.y - mean) * rstd * g.y;
        o.z = (v.z - mean) * rstd * g.z;
        o.w = (v.w - mean) * rstd * g.w;
        if (!RMS) {
            const float4 bb = __ldg(b4 + i);
            o.x += bb.x, o.y += bb.y, o.z += bb.z, o.w += bb.w;
        }
        __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        yr[i] = pk;
    }
    if (lane == 0) {
        stats[2 * r] = mean;
        stats[2 * r + 1] = rstd;
    }
}

template <bool RMS>
__global__ void __launch_bounds__(32 * kRowsPerBlock) norm_bwd_kernel(
    const float* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ stats,
    const float* __restrict__ gamma, int64_t rows, int d, const float* __restrict__ dres_in,
    float* __restrict__ dres_out, __nv_bfloat16* __restrict__ dres_out16) {
    const int lane = threadIdx.x & 31;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + (threadIdx.x >> 5);
    if (r >= rows) return;
    const float mean = stats[2 * r], rstd = stats[2 * r + 1];
    const float4* xr = reinterpret_cast<const float4*>(x + r * d);
    const float4* dr = reinterpret_cast<const float4*>(dy + r * d);
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    const int n4 = d / 4;
    float sg = 0.0f, sgx = 0.0f;  // sum of dy*gamma, sum of dy*gamma*xhat
    for (int i = lane; i < n4; i += 32) {
        const float4 v = __ldg(xr + i), e = __ldg(dr + i), g = __ldg(g4 + i);
        const float g0 = e.x * g.x, g1 = e.y * g.y, g2 = e.z * g.z, g3 = e.w * g.w;
        sg += (g0 + g1) + (g2 + g3);
        sgx += (g0 * (v.x - mean) + g1 * (v.y - mean)) + (g2 * (v.z - mean) + g3 * (v.w - mean));
    }
    const float inv_d = 1.0f / static_cast<float>(d);
    const float c_mean = RMS ? 0.0f : warp_allsum(sg) * inv_d;
    const float c_x = warp_allsum(sgx) * rstd * inv_d;  // mean(dy*gamma*xhat)
    const float4* ri = reinterpret_cast<const float4*>(dres_in + r * d);
    float4* ro = reinterpret_cast<float4*>(dres_out + r * d);
    uint2* r16 = dres_out16 ? reinterpret_cast<uint2*>(dres_out16 + r * d) : nullptr;
    for (int i = lane; i < n4; i += 32) {
        const float4 v = __ldg(xr + i), e = __ldg(dr + i), g = __ldg(g4 + i);
        const float4 base = __ldg(ri + i);
        float4 o;
        o.x = base.x + rstd * (e.x * g.x - c_mean - (v.x - mean) * rstd * c_x);
        o.y = base.y + rstd * (e.y * g.y - c_mean - (v.y - mean) * rstd * c_x);
        o.z = base.z + rstd * (e.z * g.z - c_mean - (v.z - mean) * rstd * c_x);
        o.w = base.w + rstd * (e.w * g.w - c_mean - (v.w - mean) * rstd * c_x);
        ro[i] = o;
        if (r16) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            r16[i] = pk;
        }
    }
}

// The last block of a column group to finish (of nchunks) sees every chunk's partial: the
// writes of each block are fenced before its counter increment, the last block fences again
// before reading. It re-arms the counter for the next launch on the stream.
__device__ __forceinline__ bool last_chunk_block(int* counter, int nchunks) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        s_last = atomicAdd(counter, 1) == nchunks - 1;
        if (s_last) *counter = 0;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// Sum over chunks 0..n-1 of part[c * stride + j], in chunk order (L2 reads: other blocks wrote
// them). Loads are issued eight at a time; the adds stay sequential.
__device__ __forceinline__ float chunk_sum(const float* part, int n, int64_t stride, int64_t j) {
    float s = 0.0f;
    int c = 0;
    for (; c + 8 <= n; c += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + static_cast<int64_t>(c + u) * stride + j);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; c < n; ++c) s += __ldcg(part + static_cast<int64_t>(c) * stride + j);
    return s;
}

// Norm parameter gradients: per kChunkRows-row chunk, part[chunk][0][j] = sum_r dy xhat and
// part[chunk][1][j] = sum_r dy (block = 32 threads x 4 columns, 8 row lanes combined in a fixed
// order through shared memory); the last chunk block of each column group then sums the chunks
// in order into out[j] (and out[d + j] for LayerNorm's beta).
__global__ void __launch_bounds__(32 * kRowLanes) norm_param_kernel(const float* __restrict__ dy,
                                                                    const float* __restrict__ x,
                                                                    const float* __restrict__ stats,
                                                                    int64_t rows, int d, int rms,
                                                                    float* __restrict__ part, int* __restrict__ counters,
                                                                    float* __restrict__ out) {
    __shared__ float4 red[2][kRowLanes][32];
    const int c4 = blockIdx.x * 32 + threadIdx.x;  // float4 column group
    const int lane_r = threadIdx.y;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kChunkRows;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * c4 < d) {
        const int64_t rend = min(rows, r0 + kChunkRows);
#pragma unroll 4
        for (int64_t r = r0 + lane_r; r < rend; r += kRowLanes) {
            const float mean = rms ? 0.0f : stats[2 * r], rstd = stats[2 * r + 1];
            const float4 e = __ldg(reinterpret_cast<const float4*>(dy + r * d) + c4);
            const float4 v = __ldg(reinterpret_cast<const float4*>(x + r * d) + c4);
            a.x += e.x * ((v.x - mean) * rstd);
            a.y += e.y * ((v.y - mean) * rstd);
            a.z += e.z * ((v.z - mean) * rstd);
            a.w += e.w * ((v.w - mean) * rstd);
            b.x += e.x, b.y += e.y, b.z += e.z, b.w += e.w;
        }
    }
    red[0][lane_r][threadIdx.x] = a;
    red[1][lane_r][threadIdx.x] = b;
    __syncthreads();
    if (lane_r < 2 && 4 * c4 < d) {
        float4 s = red[lane_r][0][threadIdx.x];
        for (int l = 1; l < kRowLanes; ++l) {
            const float4 v = red[lane_r][l][threadIdx.x];
            s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
        }
        reinterpret_cast<float4*>(part + (static_cast<int64_t>(blockIdx.y) * 2 + lane_r) * d)[c4] = s;
    }
    if (!last_chunk_block(counters + blockIdx.x, gridDim.y)) return;
    // 256 threads: (which, column) for the group's 128 columns
    const int t = threadIdx.y * 32 + threadIdx.x;
    const int which = t >> 7, j = blockIdx.x * 128 + (t & 127);
    if (j >= d || (rms && which == 1)) return;
    out[static_cast<int64_t>(which) * d + j] = chunk_sum(part + static_cast<int64_t>(which) * d, gridDim.y, 2 * static_cast<int64_t>(d), j);
}

// Column sums of a bf16 [rows][N] matrix (a bias gradient): per kChunkRows-row chunk, block =
// 32 groups of 8 columns (one 16-byte load each) x 8 row lanes, lanes combined in a fixed order
// into part[chunk][N]; the last chunk block of each 256-column group sums the chunks in order.
__global__ void __launch_bounds__(32 * kRowLanes) colsum_total_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                                      int n, float* __restrict__ part,
                                                                      int* __restrict__ counters, float* __restrict__ out) {
    __shared__ float red[kRowLanes][32][9];
    const int g = blockIdx.x * 32 + threadIdx.x;  // 8-column group
    const int lane_r = threadIdx.y;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kChunkRows;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    if (8 * g < n) {
        const int64_t rend = min(rows, r0 + kChunkRows);
#pragma unroll 8
        for (int64_t r = r0 + lane_r; r < rend; r += kRowLanes) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + r * n) + g);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
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
    if (lane_r == 0 && 8 * g < n) {
        float o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float s = red[0][threadIdx.x][i];
            for (int l = 1; l < kRowLanes; ++l) s += red[l][threadIdx.x][i];
            o[i] = s;
        }
        float4* dst = reinterpret_cast<float4*>(part + static_cast<int64_t>(blockIdx.y) * n + 8 * g);
        dst[0] = make_float4(o[0], o[1], o[2], o[3]);
        dst[1] = make_float4(o[4], o[5], o[6], o[7]);
    }
    if (!last_chunk_block(counters + blockIdx.x, gridDim.y)) return;
    const int j = blockIdx.x * 256 + threadIdx.y * 32 + threadIdx.x;
    if (j < n) out[j] = chunk_sum(part, gridDim.y, n, j);
}

}  // namespace

int norm_param_chunks(int64_t rows) { return static_cast<int>((rows + kChunkRows - 1) / kChunkRows); }

void norm_forward(const float* x, const float* gamma, const float* beta, int rms, float eps, int64_t rows, int d,
                  void* y, float* stats, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((rows + kRowsPerBlock - 1) / kRowsPerBlock));
    auto* yo = static_cast<__nv_bfloat16*>(y);
    if (rms) launch_kernel(norm_fwd_kernel<true>, grid, dim3(32 * kRowsPerBlock), 0, st, x, gamma, beta, eps, rows, d, yo, stats);
    else launch_kernel(norm_fwd_kernel<false>, grid, dim3(32 * kRowsPerBlock), 0, st, x, gamma, beta, eps, rows, d, yo, stats);
}

void norm_backward(const float* dy, const float* x, const float* stats, const float* gamma, int rms, int64_t rows,
                   int d, const float* dres_in, float* dres_out, void* dres_out16, const ColScratch& scr, float* out,
                   cudaStream_t st) {
    if (dres_out) {
        const dim3 grid(static_cast<unsigned>((rows + kRowsPerBlock - 1) / kRowsPerBlock));
        auto* o16 = static_cast<__nv_bfloat16*>(dres_out16);
        if (rms)
            launch_kernel(norm_bwd_kernel<true>, grid, dim3(32 * kRowsPerBlock), 0, st, dy, x, stats, gamma, rows, d,
                          dres_in, dres_out, o16);
        else
            launch_kernel(norm_bwd_kernel<false>, grid, dim3(32 * kRowsPerBlock), 0, st, dy, x, stats, gamma, rows, d,
                          dres_in, dres_out, o16);
    }
    if (out) {
        const dim3 grid(static_cast<unsigned>((d / 4 + 31) / 32), static_cast<unsigned>(norm_param_chunks(rows)));
        launch_kernel(norm_param_kernel, grid, dim3(32, kRowLanes), 0, st, dy, x, stats, rows, d, rms, scr.part,
                      scr.counters, out);
    }
}

void colsum_total_bf16(const void* x, int64_t rows, int n, const ColScratch& scr, float* out, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((n / 8 + 31) / 32), static_cast<unsigned>(norm_param_chunks(rows)));
    launch_kernel(colsum_total_kernel, grid, dim3(32, kRowLanes), 0, st, static_cast<const __nv_bfloat16*>(x), rows, n,
                  scr.part, scr.counters, out);
}

ColScratchSize col_scratch_size(int64_t rows, int widest) {
    ColScratchSize s;
    s.part_floats = static_cast<size_t>(norm_param_chunks(rows)) * 2 * static_cast<size_t>(widest);
    s.counters = static_cast<size_t>((widest + 127) / 128);
    return s;
}

}  // namespace sp

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

// One warp per row; the row is held in registers (NJ float4 per lane), so x is read from
// memory once and all NJ loads of a lane are in flight together. Sums run in the same per-lane
// order as a strided loop would (j ascending), then across lanes.
template <bool RMS, int NJ>
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
    float4 v[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) v[j] = lane + 32 * j < n4 ? __ldg(xr + lane + 32 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
    float mean = 0.0f;
    if (!RMS) {
        float s = 0.0f;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (lane + 32 * j < n4) s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
        mean = warp_allsum(s) / static_cast<float>(d);
    }
    float q = 0.0f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        if (lane + 32 * j >= n4) continue;
        const float a = v[j].x - mean, b = v[j].y - mean, c = v[j].z - mean, e = v[j].w - mean;
        q += (a * a + b * b) + (c * c + e * e);
    }
    const float rstd = rsqrtf(warp_allsum(q) / static_cast<float>(d) + eps);
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    const float4* b4 = reinterpret_cast<const float4*>(beta);
    uint2* yr = reinterpret_cast<uint2*>(y + r * d);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int i = lane + 32 * j;
        if (i >= n4) continue;
        const float4 g = __ldg(g4 + i);
        float4 o;
        o.x = (v[j].x - mean) * rstd * g.x;
        o.y = (v[j].y - mean) * rstd * g.y;
        o.z = (v[j].z - mean) * rstd * g.z;
        o.w = (v[j].w - mean) * rstd * g.w;
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

// Rows wider than 32 float4 per lane (d > 4096: Llama-3-70B's 8192): three strided passes over
// the row (L1 hits after the first), the same per-lane summation order.
template <bool RMS>
__global__ void __launch_bounds__(32 * kRowsPerBlock) norm_fwd_wide_kernel(const float* __restrict__ x,
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

// Fused norm backward (d <= 2048): one pass over dy, x and dres_in produces dres_out (fp32 and
// bf16) AND the per-block column partials of the norm's parameter gradients (sum dy*xhat, sum
// dy) and of dres_out itself (the bias gradient of the linear that produced the norm's input),
// so neither dy / x nor dres_out is read a second time. Persistent, two blocks per SM (one
// partial row each); block = 8 warps: two row groups x four column quarters; warp (rg, q) owns
// the 32-float4 stripes q, q+4, q+8, ... of every row of its group, so a row's reductions are four warp sums combined through shared
// memory in quarter order (one named barrier per row, double-buffered by row parity), and each
// lane keeps its stripes' column partials in registers across the rows. The two row groups are
// added (rg 0 + rg 1) into the block's partial row; reduce_col_chunks sums them in order.
constexpr int kNbMaxS = 4;  // stripes per warp: d <= 4 * 4 * 32 * 4 = 2048

__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void f4_add(float4& a, const float4& b) { a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w; }

template <bool RMS>
__global__ void __launch_bounds__(256, 2) norm_bwd_fused_kernel(
    const float* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ stats,
    const float* __restrict__ gamma, int64_t rows, int d, const float* __restrict__ dres_in,
    float* __restrict__ dres_out, __nv_bfloat16* __restrict__ dres_out16, float* __restrict__ ppart,
    float* __restrict__ cpart) {
    __shared__ float2 red[2][2][4];                 // [row parity][row group][quarter]
    __shared__ float4 xch[4][kNbMaxS][3][32];       // row group 1's column partials
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, rg = w >> 2, q = w & 3;
    const int n4 = d >> 2;
    const bool dx = dres_out != nullptr;
    const float inv_d = 1.0f / static_cast<float>(d);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* g4 = reinterpret_cast<const float4*>(gamma);  // (re-read per row: L1 hits)
    float4 A[kNbMaxS], B[kNbMaxS], Cs[kNbMaxS];
    int jj[kNbMaxS];
#pragma unroll
    for (int i = 0; i < kNbMaxS; ++i) {
        jj[i] = (q + 4 * i) * 32 + lane;
        A[i] = z4, B[i] = z4, Cs[i] = z4;
    }
    int par = 0;
    // persistent: block b takes the row pairs b, b + grid, b + 2 grid, ... (row 2 p + rg of pair p)
    for (int64_t r = 2 * static_cast<int64_t>(blockIdx.x) + rg; r < rows; r += 2 * static_cast<int64_t>(gridDim.x)) {
        const float mean = RMS ? 0.0f : stats[2 * r], rstd = stats[2 * r + 1];
        const float4* dr = reinterpret_cast<const float4*>(dy + r * d);
        const float4* xr = reinterpret_cast<const float4*>(x + r * d);
        // every load of the row up front (one DRAM round trip per row); e becomes dy*gamma and v
        // becomes x - mean before the row reduction's barrier, so no register holds e, v and the
        // products at once (the arithmetic is the same, operation for operation)
        float4 e[kNbMaxS], v[kNbMaxS], base[kNbMaxS];
        const float4* ri = reinterpret_cast<const float4*>(dres_in + r * d);
#pragma unroll
        for (int i = 0; i < kNbMaxS; ++i) {
            e[i] = jj[i] < n4 ? __ldg(dr + jj[i]) : z4;
            v[i] = jj[i] < n4 ? __ldg(xr + jj[i]) : z4;
            base[i] = dx && jj[i] < n4 ? __ldg(ri + jj[i]) : z4;
        }
#pragma unroll
        for (int i = 0; i < kNbMaxS; ++i) v[i] = make_float4(v[i].x - mean, v[i].y - mean, v[i].z - mean, v[i].w - mean);
        if (ppart) {
#pragma unroll
            for (int i = 0; i < kNbMaxS; ++i) {
                A[i].x += e[i].x * (v[i].x * rstd);
                A[i].y += e[i].y * (v[i].y * rstd);
                A[i].z += e[i].z * (v[i].z * rstd);
                A[i].w += e[i].w * (v[i].w * rstd);
                f4_add(B[i], e[i]);
            }
        }
        if (dx) {
            float sg = 0.0f, sgx = 0.0f;
#pragma unroll
            for (int i = 0; i < kNbMaxS; ++i) {  // (padding lanes hold zeros)
                const float4 gi = jj[i] < n4 ? __ldg(g4 + jj[i]) : z4;
                e[i] = make_float4(e[i].x * gi.x, e[i].y * gi.y, e[i].z * gi.z, e[i].w * gi.w);  // dy * gamma
                sg += (e[i].x + e[i].y) + (e[i].z + e[i].w);
                sgx += (e[i].x * v[i].x + e[i].y * v[i].y) + (e[i].z * v[i].z + e[i].w * v[i].w);
            }
            sg = warp_allsum(sg);
            sgx = warp_allsum(sgx);
            if (lane == 0) red[par][rg][q] = make_float2(sg, sgx);
            named_bar(1 + rg, 128);
            float tg = red[par][rg][0].x, tx = red[par][rg][0].y;
#pragma unroll
            for (int k = 1; k < 4; ++k) tg += red[par][rg][k].x, tx += red[par][rg][k].y;
            par ^= 1;
            const float c_mean = RMS ? 0.0f : tg * inv_d;
            const float c_x = tx * rstd * inv_d;
            float4* ro = reinterpret_cast<float4*>(dres_out + r * d);
            uint2* r16 = dres_out16 ? reinterpret_cast<uint2*>(dres_out16 + r * d) : nullptr;
#pragma unroll
            for (int i = 0; i < kNbMaxS; ++i) {
                if (jj[i] >= n4) continue;
                float4 o;
                o.x = base[i].x + rstd * (e[i].x - c_mean - v[i].x * rstd * c_x);
                o.y = base[i].y + rstd * (e[i].y - c_mean - v[i].y * rstd * c_x);
                o.z = base[i].z + rstd * (e[i].z - c_mean - v[i].z * rstd * c_x);
                o.w = base[i].w + rstd * (e[i].w - c_mean - v[i].w * rstd * c_x);
                ro[jj[i]] = o;
                if (r16) {
                    __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
                    uint2 pk;
                    pk.x = *reinterpret_cast<uint32_t*>(&lo);
                    pk.y = *reinterpret_cast<uint32_t*>(&hi);
                    r16[jj[i]] = pk;
                }
                f4_add(Cs[i], o);
            }
        }
    }
    if (rg == 1) {
#pragma unroll
        for (int i = 0; i < kNbMaxS; ++i) {
            xch[q][i][0][lane] = A[i];
            xch[q][i][1][lane] = B[i];
            xch[q][i][2][lane] = Cs[i];
        }
    }
    __syncthreads();
    if (rg != 0) return;
#pragma unroll
    for (int i = 0; i < kNbMaxS; ++i) {
        if (jj[i] >= n4) continue;
        if (ppart) {
            f4_add(A[i], xch[q][i][0][lane]);
            reinterpret_cast<float4*>(ppart + static_cast<int64_t>(blockIdx.x) * 2 * d)[jj[i]] = A[i];
            if (!RMS) {
                f4_add(B[i], xch[q][i][1][lane]);
                reinterpret_cast<float4*>(ppart + (static_cast<int64_t>(blockIdx.x) * 2 + 1) * d)[jj[i]] = B[i];
            }
        }
        if (cpart) {
            f4_add(Cs[i], xch[q][i][2][lane]);
            reinterpret_cast<float4*>(cpart + static_cast<int64_t>(blockIdx.x) * d)[jj[i]] = Cs[i];
        }
    }
}

// out_s[j] = sum over chunks c (in order) of part_s[c * stride_s + j] for up to three segments.
// Block = 32 columns x 8 chunk ranges; each range is summed in chunk order, then the ranges in
// range order (a fixed decomposition of the shape).
__global__ void __launch_bounds__(256) reduce_col_chunks_kernel(ColChunks r) {
    __shared__ float sub[8][33];
    const int col = blockIdx.x * 32 + threadIdx.x;
    int s = 0, j = col;
    while (s < r.n && j >= r.width[s]) j -= r.width[s++];
    float acc = 0.0f;
    if (s < r.n) {
        const int per = (r.chunks + 7) / 8;
        const int c0 = threadIdx.y * per, c1 = min(r.chunks, c0 + per);
        const float* p = r.part[s] + j;
        const int64_t stride = r.stride[s];
        int c = c0;
        for (; c + 8 <= c1; c += 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + static_cast<int64_t>(c + u) * stride);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
        }
        for (; c < c1; ++c) acc += __ldcg(p + static_cast<int64_t>(c) * stride);
    }
    sub[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y != 0 || s >= r.n) return;
    float t = sub[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += sub[k][threadIdx.x];
    r.out[s][j] = t;
}

}  // namespace

int norm_param_chunks(int64_t rows) { return static_cast<int>((rows + kChunkRows - 1) / kChunkRows); }

bool norm_backward_fused_ok(int d) { return d % 4 == 0 && d <= 4 * kNbMaxS * 32 * 4; }
// Grid of the persistent fused norm backward = its number of partial rows: two blocks per SM
// (fixed for a GPU model, so the reduction order depends only on the shape there).
int norm_bwd_chunks(int64_t rows) {
    const int64_t pairs = (rows + 1) / 2;
    const int64_t g = 2 * static_cast<int64_t>(num_sms());
    return static_cast<int>(pairs < g ? pairs : g);
}

void norm_backward_fused(const float* dy, const float* x, const float* stats, const float* gamma, int rms,
                         int64_t rows, int d, const float* dres_in, float* dres_out, void* dres_out16,
                         float* param_part, float* csum_part, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>(norm_bwd_chunks(rows)));
    auto* o16 = static_cast<__nv_bfloat16*>(dres_out16);
    if (rms)
        launch_kernel(norm_bwd_fused_kernel<true>, grid, dim3(256), 0, st, dy, x, stats, gamma, rows, d, dres_in,
                      dres_out, o16, param_part, csum_part);
    else
        launch_kernel(norm_bwd_fused_kernel<false>, grid, dim3(256), 0, st, dy, x, stats, gamma, rows, d, dres_in,
                      dres_out, o16, param_part, csum_part);
}

void reduce_col_chunks(const ColChunks& r, cudaStream_t st) {
    int total = 0;
    for (int s = 0; s < r.n; ++s) total += r.width[s];
    if (total == 0) return;
    launch_kernel(reduce_col_chunks_kernel, dim3(static_cast<unsigned>((total + 31) / 32)), dim3(32, 8), 0, st, r);
}

void norm_forward(const float* x, const float* gamma, const float* beta, int rms, float eps, int64_t rows, int d,
                  void* y, float* stats, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((rows + kRowsPerBlock - 1) / kRowsPerBlock));
    auto* yo = static_cast<__nv_bfloat16*>(y);
    const int nj = (d / 4 + 31) / 32;  // float4 per lane (d <= 4096 held in registers)
    auto go = [&](auto kern) { launch_kernel(kern, grid, dim3(32 * kRowsPerBlock), 0, st, x, gamma, beta, eps, rows, d, yo, stats); };
    if (rms) {
        if (nj <= 8) go(norm_fwd_kernel<true, 8>);
        else if (nj <= 16) go(norm_fwd_kernel<true, 16>);
        else if (nj <= 32) go(norm_fwd_kernel<true, 32>);
        else go(norm_fwd_wide_kernel<true>);
    } else {
        if (nj <= 8) go(norm_fwd_kernel<false, 8>);
        else if (nj <= 16) go(norm_fwd_kernel<false, 16>);
        else if (nj <= 32) go(norm_fwd_kernel<false, 32>);
        else go(norm_fwd_wide_kernel<false>);
    }
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

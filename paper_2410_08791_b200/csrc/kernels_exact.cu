// kernels_exact.cu — fp32 SIMT kernels that are bit-identical to the reference CPU math.
//
// The reference evaluates every dot product as a left-to-right fp32 fold with separately
// rounded multiply and add (scalar SSE2 mulss/addss, model.cpp:54-123). These kernels keep
// exactly that order per output element and use __fmul_rn/__fadd_rn so nvcc cannot contract
// to FMA. They are the parity mode (SP_NUMERICS_EXACT), not the throughput path.
#include "kernels.hpp"

namespace sp {
namespace {

constexpr int kCols = 128;  // threads per block, one output column each
constexpr int kRows = 8;    // rows per block (register blocking)
constexpr int kChunk = 32;  // reduction chunk staged in shared memory

__global__ void __launch_bounds__(kCols) exact_forward_kernel(
    const float* __restrict__ x, const float* __restrict__ W, const float* __restrict__ b,
    int relu, float* __restrict__ y, int64_t rows, int d) {
    __shared__ float xs[kRows][kChunk];
    const int j = blockIdx.x * kCols + threadIdx.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kRows;
    float acc[kRows];
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) acc[rr] = 0.0f;
    for (int i0 = 0; i0 < d; i0 += kChunk) {
        for (int e = threadIdx.x; e < kRows * kChunk; e += kCols) {
            const int rr = e / kChunk, ii = e % kChunk;
            const int64_t r = r0 + rr;
            xs[rr][ii] = (r < rows && i0 + ii < d) ? x[r * d + i0 + ii] : 0.0f;
        }
        __syncthreads();
        if (j < d) {
            const int iend = min(kChunk, d - i0);
            for (int ii = 0; ii < iend; ++ii) {
                const float w = W[static_cast<int64_t>(i0 + ii) * d + j];
#pragma unroll
                for (int rr = 0; rr < kRows; ++rr) acc[rr] = __fadd_rn(acc[rr], __fmul_rn(xs[rr][ii], w));
            }
        }
        __syncthreads();
    }
    if (j >= d) return;
    const float bj = b[j];
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
        const int64_t r = r0 + rr;
        if (r >= rows) break;
        float v = __fadd_rn(acc[rr], bj);
        if (relu && v < 0.0f) v = 0.0f;
        y[r * d + j] = v;
    }
}

__global__ void __launch_bounds__(kCols) exact_dx_kernel(
    const float* __restrict__ dz, const float* __restrict__ W, const float* __restrict__ gate,
    float* __restrict__ out, int64_t rows, int d) {
    __shared__ float wt[kCols][kChunk + 1];
    __shared__ float ds[kRows][kChunk];
    const int ibase = blockIdx.x * kCols;
    const int i = ibase + threadIdx.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kRows;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float acc[kRows];
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) acc[rr] = 0.0f;
    for (int j0 = 0; j0 < d; j0 += kChunk) {
        // W[i][j0..j0+31] for the block's 128 rows i, read coalesced along j.
        for (int ii = warp; ii < kCols; ii += kCols / 32) {
            const int gi = ibase + ii, gj = j0 + lane;
            wt[ii][lane] = (gi < d && gj < d) ? W[static_cast<int64_t>(gi) * d + gj] : 0.0f;
        }
        for (int e = threadIdx.x; e < kRows * kChunk; e += kCols) {
            const int rr = e / kChunk, jj = e % kChunk;
            const int64_t r = r0 + rr;
            ds[rr][jj] = (r < rows && j0 + jj < d) ? dz[r * d + j0 + jj] : 0.0f;
        }
        __syncthreads();
        const int jend = min(kChunk, d - j0);
        for (int jj = 0; jj < jend; ++jj) {
            const float w = wt[threadIdx.x][jj];
#pragma unroll
            for (int rr = 0; rr < kRows; ++rr) acc[rr] = __fadd_rn(acc[rr], __fmul_rn(ds[rr][jj], w));
        }
        __syncthreads();
    }
    if (i >= d) return;
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
        const int64_t r = r0 + rr;
        if (r >= rows) break;
        float v = acc[rr];
        if (gate && gate[r * d + i] <= 0.0f) v = 0.0f;
        out[r * d + i] = v;
    }
}

constexpr int kIRows = 8;  // dW rows i per block

__global__ void __launch_bounds__(kCols) exact_dw_kernel(
    const float* __restrict__ x, const float* __restrict__ dz, float* __restrict__ dW,
    float* __restrict__ db, int64_t rows, int d) {
    __shared__ float xs[kChunk][kIRows];
    const int j = blockIdx.x * kCols + threadIdx.x;
    const int i0 = blockIdx.y * kIRows;
    const bool do_db = blockIdx.y == 0 && db != nullptr;
    float acc[kIRows];
#pragma unroll
    for (int ii = 0; ii < kIRows; ++ii) acc[ii] = 0.0f;
    float bacc = 0.0f;
    for (int64_t rb = 0; rb < rows; rb += kChunk) {
        for (int e = threadIdx.x; e < kChunk * kIRows; e += kCols) {
            const int rr = e / kIRows, ii = e % kIRows;
            const int64_t r = rb + rr;
            xs[rr][ii] = (r < rows && i0 + ii < d) ? x[r * d + i0 + ii] : 0.0f;
        }
        __syncthreads();
        if (j < d) {
            const int rend = static_cast<int>((rows - rb) < kChunk ? (rows - rb) : kChunk);
            for (int rr = 0; rr < rend; ++rr) {
                const float g = dz[(rb + rr) * d + j];
#pragma unroll
                for (int ii = 0; ii < kIRows; ++ii) acc[ii] = __fadd_rn(acc[ii], __fmul_rn(xs[rr][ii], g));
                if (do_db) bacc = __fadd_rn(bacc, g);
            }
        }
        __syncthreads();
    }
    if (j >= d) return;
#pragma unroll
    for (int ii = 0; ii < kIRows; ++ii)
        if (i0 + ii < d) dW[static_cast<int64_t>(i0 + ii) * d + j] = acc[ii];
    if (do_db) db[j] = bacc;
}

// Sequential fp32 sum of squared errors (model.cpp:133-139): one thread, reference order.
__global__ void exact_loss_kernel(const float* __restrict__ y, const float* __restrict__ t,
                                  int64_t count, float* __restrict__ out) {
    float acc = 0.0f;
    for (int64_t i = 0; i < count; ++i) {
        const float e = __fsub_rn(y[i], t[i]);
        acc = __fadd_rn(acc, __fmul_rn(e, e));
    }
    *out = acc;
}

__global__ void exact_grad_kernel(const float* __restrict__ y, const float* __restrict__ t,
                                  int64_t count, float inv_n, int relu, float* __restrict__ g) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const float yi = y[i];
    float v = __fmul_rn(__fmul_rn(2.0f, __fsub_rn(yi, t[i])), inv_n);  // model.cpp:146
    if (relu && yi <= 0.0f) v = 0.0f;  // ReLU gate of the last layer (model.cpp:93)
    g[i] = v;
}

__global__ void exact_sgd_kernel(float* __restrict__ w, const float* __restrict__ g,
                                 int64_t count, float lr) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) w[i] = __fsub_rn(w[i], __fmul_rn(lr, g[i]));
}

unsigned blocks_for(int64_t count, int threads) {
    return static_cast<unsigned>((count + threads - 1) / threads);
}

}  // namespace

// Rows are independent, so a row range larger than one grid's y extent (65535 blocks of kRows)
// is launched in consecutive slices; each row's arithmetic is unchanged.
constexpr int64_t kMaxRowsPerLaunch = 65535LL * kRows;

void exact_forward(const float* x, const float* W, const float* b, int relu, float* y,
                   int64_t rows, int d, cudaStream_t st) {
    for (int64_t r = 0; r < rows; r += kMaxRowsPerLaunch) {
        const int64_t n = rows - r < kMaxRowsPerLaunch ? rows - r : kMaxRowsPerLaunch;
        dim3 grid((d + kCols - 1) / kCols, static_cast<unsigned>((n + kRows - 1) / kRows));
        exact_forward_kernel<<<grid, kCols, 0, st>>>(x + r * d, W, b, relu, y + r * d, n, d);
    }
}

void exact_backward_dx(const float* dz, const float* W, const float* gate, float* dz_out,
                       int64_t rows, int d, cudaStream_t st) {
    for (int64_t r = 0; r < rows; r += kMaxRowsPerLaunch) {
        const int64_t n = rows - r < kMaxRowsPerLaunch ? rows - r : kMaxRowsPerLaunch;
        dim3 grid((d + kCols - 1) / kCols, static_cast<unsigned>((n + kRows - 1) / kRows));
        exact_dx_kernel<<<grid, kCols, 0, st>>>(dz + r * d, W, gate ? gate + r * d : nullptr,
                                                dz_out + r * d, n, d);
    }
}

void exact_backward_dw(const float* x, const float* dz, float* dW, float* db, int64_t rows,
                       int d, cudaStream_t st) {
    dim3 grid((d + kCols - 1) / kCols, (d + kIRows - 1) / kIRows);
    exact_dw_kernel<<<grid, kCols, 0, st>>>(x, dz, dW, db, rows, d);
}

void exact_loss_grad(const float* y, const float* t, int64_t count, float inv_n, int relu,
                     float* g, float* loss_sum_dev, cudaStream_t st) {
    exact_loss_kernel<<<1, 1, 0, st>>>(y, t, count, loss_sum_dev);
    exact_grad_kernel<<<blocks_for(count, 256), 256, 0, st>>>(y, t, count, inv_n, relu, g);
}

void exact_sgd(float* w, const float* g, int64_t count, float lr, cudaStream_t st) {
    exact_sgd_kernel<<<blocks_for(count, 256), 256, 0, st>>>(w, g, count, lr);
}

}  // namespace sp

// kernels_attn.cu — the attention core of the named-shape transformer blocks (sm_100a).
//
// Fused (flash) attention over the packed projection buffer qkv[T][(H + 2 Hkv) hd] (bf16,
// token-major, q heads then k heads then v heads), sequences of S consecutive tokens, causal or
// not, grouped-query (Hkv divides H). Tensor-core work uses warp-level mma.sync m16n8k16 (bf16
// in, fp32 accumulate) with ldmatrix from padded shared-memory tiles filled by cp.async, and
// an online softmax in registers: no S x S matrix ever reaches HBM.
//
//   forward : o[T][H hd] (bf16), lse[B][H][S] (fp32, log2 units of the scaled scores)
//   backward: delta = rowsum(dO * O) per (token, head); dK/dV per key block (looping over the
//             query blocks and, for GQA, over the heads of the group); dQ per query block
//             (looping over key blocks). dQ is its own pass, so no atomics: every output
//             element is owned by one warp with a fixed summation order, and the results are
//             bit-identical run to run and across every (k, k') window.
// The reference has no attention: this serves north_star's
// "named shapes".
#include <cuda_bf16.h>

#include <cstdint>

#include "kernels.hpp"
#include "launch.cuh"

namespace sp {
cudaError_t attention_backward_tc(const AttnProblem& a, cudaStream_t st);   // kernels_attn_tc.cu
cudaError_t attention_backward_tc2(const AttnProblem& a, cudaStream_t st);  // kernels_attn_bwd.cu
extern int g_attn_bwd_kind;
namespace {

constexpr int kWarps = 4;        // 16 rows per warp
constexpr int kBM = 16 * kWarps; // query (or key) rows per CTA
constexpr int kBN = 64;          // keys (or queries) per inner block
constexpr int kThreads = 32 * kWarps;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    // zero-fill when the source row is outside the sequence
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2f(float x) {  // MUFU.EX2 (ex2(-inf) = +0)
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// A [rows][HD] bf16 tile in shared memory with rows padded by 16 bytes, so the 8 row addresses
// of every ldmatrix phase fall in distinct banks (HD*2 + 16 bytes per row).
template <int HD>
struct Tile {
    static constexpr int LD = HD + 8;  // elements per smem row
    static constexpr int BYTES = kBN * LD * 2;
};

// Loads rows [r0, r0 + ROWS) of one head (column offset col) of a token-major [T][ld] bf16
// matrix restricted to one sequence (rows >= S zero-filled) into a padded tile.
template <int HD, int ROWS>
__device__ __forceinline__ void load_tile(__nv_bfloat16* tile, const __nv_bfloat16* base, int64_t seq_row0,
                                          int r0, int S, int ld, int col) {
    constexpr int CH = HD / 8;  // 16-byte chunks per row
    for (int i = threadIdx.x; i < ROWS * CH; i += kThreads) {
        const int r = i / CH, c = i % CH;
        const bool ok = r0 + r < S;
        const __nv_bfloat16* src = base + (seq_row0 + (ok ? r0 + r : 0)) * ld + col + c * 8;
        cp_async16(tile + r * Tile<HD>::LD + c * 8, src, ok);
    }
}

// Fragment addressing (mma.sync m16n8k16, lane = 4 g + t):
//  A 16x16 from a row-major [m][k] tile at (m0, k0): ldmatrix.x4, lane address row m0 + (lane % 16),
//    col k0 + 8 (lane / 16).
//  B pair (two n8 blocks) from an [n][k] tile (non-trans) at (n0, k0): row n0 + (lane % 8) +
//    8 (lane / 16), col k0 + 8 ((lane / 8) % 2) -> regs {b0, b1} of block n0, {b0, b1} of n0 + 8.
//  B pair from a [k][n] tile (trans) at (k0, n0): row k0 + (lane % 8) + 8 ((lane / 8) % 2),
//    col n0 + 8 (lane / 16) -> {r0, r1} block n0, {r2, r3} block n0 + 8.
template <int LD>
__device__ __forceinline__ const __nv_bfloat16* a_addr(const __nv_bfloat16* t, int m0, int k0, int lane) {
    return t + (m0 + (lane & 15)) * LD + k0 + 8 * (lane >> 4);
}
template <int LD>
__device__ __forceinline__ const __nv_bfloat16* bn_addr(const __nv_bfloat16* t, int n0, int k0, int lane) {
    return t + (n0 + (lane & 7) + 8 * (lane >> 4)) * LD + k0 + 8 * ((lane >> 3) & 1);
}
template <int LD>
__device__ __forceinline__ const __nv_bfloat16* bt_addr(const __nv_bfloat16* t, int k0, int n0, int lane) {
    return t + (k0 + (lane & 7) + 8 * ((lane >> 3) & 1)) * LD + n0 + 8 * (lane >> 4);
}

struct AttnShape {
    int S, H, Hkv, ld;       // sequence length, heads, kv heads, qkv row stride (elements)
    int ldo;                 // o / do row stride (H * hd)
    int causal;
    float scale_log2;        // softmax scale * log2(e)
};

// ---------------------------------------------------------------------------------------
// forward: one CTA = 64 queries of one (sequence, head); 4 warps x 16 rows
// ---------------------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                            __nv_bfloat16* __restrict__ o,
                                                            float* __restrict__ lse, AttnShape sh) {
    using TL = Tile<HD>;
    constexpr int LD = TL::LD;
    extern __shared__ __align__(128) uint8_t smem[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* sK = sQ + kBM * LD;          // 2 stages
    __nv_bfloat16* sV = sK + 2 * kBN * LD;      // 2 stages
    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (sh.H / sh.Hkv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = static_cast<int64_t>(b) * sh.S;
    const int q0 = qb * kBM;
    const int qcol = h * HD, kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
    const int n_kb_total = (sh.S + kBN - 1) / kBN;
    const int n_kb = sh.causal ? min(n_kb_total, (q0 + kBM - 1) / kBN + 1) : n_kb_total;

    load_tile<HD, kBM>(sQ, qkv, row0, q0, sh.S, sh.ld, qcol);
    load_tile<HD, kBN>(sK, qkv, row0, 0, sh.S, sh.ld, kcol);
    load_tile<HD, kBN>(sV, qkv, row0, 0, sh.S, sh.ld, vcol);
    cp_commit();

    constexpr int KB = HD / 16;  // k16 blocks over the head dimension
    constexpr int NT = HD / 8;   // n8 tiles of the output
    uint32_t qf[KB][4];
    float acc[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};
    const int g = lane >> 2, t = lane & 3;
    const int qr0 = q0 + warp * 16 + g;  // this thread's two query rows: qr0, qr0 + 8

    for (int kb = 0; kb < n_kb; ++kb) {
        const int st = kb & 1;
        if (kb + 1 < n_kb) {  // prefetch the next key block into the other stage
            load_tile<HD, kBN>(sK + (st ^ 1) * kBN * LD, qkv, row0, (kb + 1) * kBN, sh.S, sh.ld, kcol);
            load_tile<HD, kBN>(sV + (st ^ 1) * kBN * LD, qkv, row0, (kb + 1) * kBN, sh.S, sh.ld, vcol);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kb == 0) {
#pragma unroll
            for (int k = 0; k < KB; ++k) ldsm_x4(qf[k], a_addr<LD>(sQ, warp * 16, k * 16, lane));
        }
        const __nv_bfloat16* tK = sK + st * kBN * LD;
        const __nv_bfloat16* tV = sV + st * kBN * LD;
        const int k0 = kb * kBN;
        // this warp's rows may all precede the block (causal): nothing to add
        const bool active = !sh.causal || k0 <= q0 + warp * 16 + 15;
        if (active) {
            float s[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.0f;
#pragma unroll
            for (int k = 0; k < KB; ++k) {
#pragma unroll
                for (int np = 0; np < 4; ++np) {
                    uint32_t bf[4];
                    ldsm_x4(bf, bn_addr<LD>(tK, np * 16, k * 16, lane));
                    mma16816(s[2 * np], qf[k], bf[0], bf[1]);
                    mma16816(s[2 * np + 1], qf[k], bf[2], bf[3]);
                }
            }
            // scale, mask, online softmax (rows g and g + 8 of the warp's 16)
            float mx[2] = {m_run[0], m_run[1]};
            // only the diagonal (causal) and a ragged last block need masks
            const bool need_mask = (sh.causal && k0 + kBN - 1 > q0 + warp * 16) || k0 + kBN > sh.S;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float v = s[i][e] * sh.scale_log2;
                    if (need_mask) {
                        const int key = k0 + i * 8 + 2 * t + (e & 1);
                        const int q = qr0 + (e >> 1) * 8;
                        if (key >= sh.S || (sh.causal && key > q)) v = -INFINITY;
                    }
                    s[i][e] = v;
                    mx[e >> 1] = fmaxf(mx[e >> 1], v);
                }
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
                mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
            }
            float corr[2], base[2], rs[2] = {0.0f, 0.0f};
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                base[r] = mx[r] == -INFINITY ? 0.0f : mx[r];  // a fully masked row so far
                corr[r] = ex2f(m_run[r] - base[r]);
                m_run[r] = mx[r];
            }
            uint32_t pf[4][4];  // P as A fragments of the four k16 key blocks
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float p0 = ex2f(s[i][0] - base[0]), p1 = ex2f(s[i][1] - base[0]);
                const float p2 = ex2f(s[i][2] - base[1]), p3 = ex2f(s[i][3] - base[1]);
                rs[0] += p0 + p1;
                rs[1] += p2 + p3;
                pf[i >> 1][(i & 1) * 2 + 0] = pack2(p0, p1);
                pf[i >> 1][(i & 1) * 2 + 1] = pack2(p2, p3);
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) l_run[r] = l_run[r] * corr[r] + rs[r];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                acc[i][0] *= corr[0];
                acc[i][1] *= corr[0];
                acc[i][2] *= corr[1];
                acc[i][3] *= corr[1];
            }
            // O += P V
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
                for (int np = 0; np < NT / 2; ++np) {
                    uint32_t vf[4];
                    ldsm_x4_t(vf, bt_addr<LD>(tV, kk * 16, np * 16, lane));
                    mma16816(acc[2 * np], pf[kk], vf[0], vf[1]);
                    mma16816(acc[2 * np + 1], pf[kk], vf[2], vf[3]);
                }
            }
        }
        __syncthreads();  // the stage is refilled by the next iteration's prefetch
    }
    // row sums across the quad, normalise, store
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
        l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = qr0 + r * 8;
        if (q >= sh.S) continue;
        const float inv = l_run[r] > 0.0f ? 1.0f / l_run[r] : 0.0f;
        __nv_bfloat16* orow = o + (row0 + q) * sh.ldo + h * HD;
#pragma unroll
        for (int i = 0; i < NT; ++i)
            *reinterpret_cast<uint32_t*>(orow + i * 8 + 2 * t) = pack2(acc[i][2 * r] * inv, acc[i][2 * r + 1] * inv);
        if (t == 0)
            lse[(static_cast<int64_t>(b) * sh.H + h) * sh.S + q] =
                l_run[r] > 0.0f ? m_run[r] + log2f(l_run[r]) : INFINITY;
    }
}

// ---------------------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------------------
// delta[b][h][s] = sum_d dO[t][h hd + d] * O[t][h hd + d]  (fp32)
template <int HD>
__global__ void attn_bwd_delta_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                      float* __restrict__ delta, int64_t T, AttnShape sh) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (token, head)
    if (i >= T * sh.H) return;
    const int64_t tok = i / sh.H;
    const int h = static_cast<int>(i % sh.H);
    const uint4* a = reinterpret_cast<const uint4*>(o + tok * sh.ldo + h * HD);
    const uint4* c = reinterpret_cast<const uint4*>(dout + tok * sh.ldo + h * HD);
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
        const uint4 va = __ldg(a + j), vc = __ldg(c + j);
        const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wc[4] = {vc.x, vc.y, vc.z, vc.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wa[k]));
            const float2 fc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wc[k]));
            acc += fa.x * fc.x + fa.y * fc.y;
        }
    }
    const int64_t b = tok / sh.S, s = tok % sh.S;
    delta[(b * sh.H + h) * sh.S + s] = acc;
}

// dK, dV: one CTA = 64 keys of one (sequence, kv head); 4 warps x 16 keys. For each q head of
// the group and each query block: S^T = K Q^T, P^T = exp2(S^T c - lse), dV += P^T dO,
// dP^T = V dO^T, dS^T = P^T (dP^T - delta), dK += dS^T Q.
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_bwd_dkdv_kernel(
    const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
    const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, AttnShape sh, float scale) {
    using TL = Tile<HD>;
    constexpr int LD = TL::LD;
    extern __shared__ __align__(128) uint8_t smem[];
    __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* sV = sK + kBM * LD;
    __nv_bfloat16* sQ = sV + kBM * LD;        // 2 stages
    __nv_bfloat16* sD = sQ + 2 * kBN * LD;    // dO, 2 stages
    float* sL = reinterpret_cast<float*>(sD + 2 * kBN * LD);  // lse, 2 stages
    float* sDl = sL + 2 * kBN;                                // delta, 2 stages
    const int kb = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int64_t row0 = static_cast<int64_t>(b) * sh.S;
    const int k0 = kb * kBM;
    const int kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
    const int group = sh.H / sh.Hkv;
    load_tile<HD, kBM>(sK, qkv, row0, k0, sh.S, sh.ld, kcol);
    load_tile<HD, kBM>(sV, qkv, row0, k0, sh.S, sh.ld, vcol);
    cp_commit();

    constexpr int KB = HD / 16, NT = HD / 8;
    float dk[NT][4], dv[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.0f;
    const int n_qb = (sh.S + kBN - 1) / kBN;
    const int qb0 = sh.causal ? k0 / kBN : 0;  // causal: queries before the keys see none of them
    const int n_iter = (n_qb - qb0) * group;
    const int kr0 = k0 + warp * 16 + g;  // this thread's key rows kr0, kr0 + 8

    // head dims up to 80: this warp's K and V rows stay in registers as A fragments
    constexpr bool KV_REGS = HD <= 80;
    constexpr int KBR = KV_REGS ? KB : 1;
    uint32_t kreg[KBR][4], vreg[KBR][4];
    auto issue = [&](int it, int st) {
        const int hq = kvh * group + it / (n_qb - qb0);
        const int q0 = (qb0 + it % (n_qb - qb0)) * kBN;
        load_tile<HD, kBN>(sQ + st * kBN * LD, qkv, row0, q0, sh.S, sh.ld, hq * HD);
        load_tile<HD, kBN>(sD + st * kBN * LD, dout, row0, q0, sh.S, sh.ldo, hq * HD);
        for (int i = threadIdx.x; i < kBN; i += kThreads) {
            const int q = q0 + i;
            const int64_t idx = (static_cast<int64_t>(b) * sh.H + hq) * sh.S + q;
            sL[st * kBN + i] = q < sh.S ? lse[idx] : INFINITY;
            sDl[st * kBN + i] = q < sh.S ? delta[idx] : 0.0f;
        }
    };
    if (n_iter > 0) issue(0, 0);
    cp_commit();
    for (int it = 0; it < n_iter; ++it) {
        const int st = it & 1;
        if (it + 1 < n_iter) {
            issue(it + 1, st ^ 1);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (KV_REGS && it == 0) {
#pragma unroll
            for (int k = 0; k < KBR; ++k) {
                ldsm_x4(kreg[k], a_addr<LD>(sK, warp * 16, k * 16, lane));
                ldsm_x4(vreg[k], a_addr<LD>(sV, warp * 16, k * 16, lane));
            }
        }
        const int q0 = (qb0 + it % (n_qb - qb0)) * kBN;
        const __nv_bfloat16* tQ = sQ + st * kBN * LD;
        const __nv_bfloat16* tD = sD + st * kBN * LD;
        const float* tL = sL + st * kBN;
        const float* tDl = sDl + st * kBN;
        // causal: this warp's keys all follow every query of the block -> no contribution
        const bool active = !sh.causal || k0 + warp * 16 <= q0 + kBN - 1;
        if (active) {
            float s[8][4], dp[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.0f;
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                uint32_t kf[4], vf[4];
                if (KV_REGS) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) kf[u] = kreg[k % KBR][u], vf[u] = vreg[k % KBR][u];
                } else {
                    ldsm_x4(kf, a_addr<LD>(sK, warp * 16, k * 16, lane));
                    ldsm_x4(vf, a_addr<LD>(sV, warp * 16, k * 16, lane));
                }
#pragma unroll
                for (int np = 0; np < 4; ++np) {
                    uint32_t qf[4], df[4];
                    ldsm_x4(qf, bn_addr<LD>(tQ, np * 16, k * 16, lane));
                    ldsm_x4(df, bn_addr<LD>(tD, np * 16, k * 16, lane));
                    mma16816(s[2 * np], kf, qf[0], qf[1]);
                    mma16816(s[2 * np + 1], kf, qf[2], qf[3]);
                    mma16816(dp[2 * np], vf, df[0], df[1]);
                    mma16816(dp[2 * np + 1], vf, df[2], df[3]);
                }
            }
            // masks only where a key follows a query (causal diagonal) or lies past the sequence
            const bool need_mask = (sh.causal && k0 + warp * 16 + 15 > q0) || k0 + kBM > sh.S;
            uint32_t pf[4][4], dsf[4][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float p[4], ds[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int qi = i * 8 + 2 * t + (e & 1);  // query within the block
                    float v = ex2f(fmaf(s[i][e], sh.scale_log2, -tL[qi]));
                    if (need_mask) {
                        const int key = kr0 + (e >> 1) * 8;
                        if (key >= sh.S || (sh.causal && key > q0 + qi)) v = 0.0f;
                    }
                    p[e] = v;
                    ds[e] = v * (dp[i][e] - tDl[qi]);
                }
                pf[i >> 1][(i & 1) * 2 + 0] = pack2(p[0], p[1]);
                pf[i >> 1][(i & 1) * 2 + 1] = pack2(p[2], p[3]);
                dsf[i >> 1][(i & 1) * 2 + 0] = pack2(ds[0], ds[1]);
                dsf[i >> 1][(i & 1) * 2 + 1] = pack2(ds[2], ds[3]);
            }
            // dV += P^T dO, dK += dS^T Q  (B = dO / Q as [k = query][n = d] tiles, transposed loads)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
                for (int np = 0; np < NT / 2; ++np) {
                    uint32_t df[4], qf[4];
                    ldsm_x4_t(df, bt_addr<LD>(tD, kk * 16, np * 16, lane));
                    ldsm_x4_t(qf, bt_addr<LD>(tQ, kk * 16, np * 16, lane));
                    mma16816(dv[2 * np], pf[kk], df[0], df[1]);
                    mma16816(dv[2 * np + 1], pf[kk], df[2], df[3]);
                    mma16816(dk[2 * np], dsf[kk], qf[0], qf[1]);
                    mma16816(dk[2 * np + 1], dsf[kk], qf[2], qf[3]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int key = kr0 + r * 8;
        if (key >= sh.S) continue;
        __nv_bfloat16* drow = dqkv + (row0 + key) * sh.ld;
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            *reinterpret_cast<uint32_t*>(drow + kcol + i * 8 + 2 * t) =
                pack2(dk[i][2 * r] * scale, dk[i][2 * r + 1] * scale);
            *reinterpret_cast<uint32_t*>(drow + vcol + i * 8 + 2 * t) = pack2(dv[i][2 * r], dv[i][2 * r + 1]);
        }
    }
}

// dQ: one CTA = 64 queries of one (sequence, head); loops over key blocks.
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_bwd_dq_kernel(
    const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
    const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, AttnShape sh, float scale) {
    using TL = Tile<HD>;
    constexpr int LD = TL::LD;
    extern __shared__ __align__(128) uint8_t smem[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* sD = sQ + kBM * LD;
    __nv_bfloat16* sK = sD + kBM * LD;      // 2 stages
    __nv_bfloat16* sV = sK + 2 * kBN * LD;  // 2 stages
    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (sh.H / sh.Hkv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int64_t row0 = static_cast<int64_t>(b) * sh.S;
    const int q0 = qb * kBM;
    const int qcol = h * HD, kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
    const int n_kb_total = (sh.S + kBN - 1) / kBN;
    const int n_kb = sh.causal ? min(n_kb_total, (q0 + kBM - 1) / kBN + 1) : n_kb_total;
    load_tile<HD, kBM>(sQ, qkv, row0, q0, sh.S, sh.ld, qcol);
    load_tile<HD, kBM>(sD, dout, row0, q0, sh.S, sh.ldo, qcol);
    load_tile<HD, kBN>(sK, qkv, row0, 0, sh.S, sh.ld, kcol);
    load_tile<HD, kBN>(sV, qkv, row0, 0, sh.S, sh.ld, vcol);
    cp_commit();
    constexpr int KB = HD / 16, NT = HD / 8;
    uint32_t qf[KB][4], df[KB][4];
    float dq[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.0f;
    const int qr0 = q0 + warp * 16 + g;
    float L[2], Dl[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = qr0 + r * 8;
        const int64_t idx = (static_cast<int64_t>(b) * sh.H + h) * sh.S + q;
        L[r] = q < sh.S ? lse[idx] : INFINITY;
        Dl[r] = q < sh.S ? delta[idx] : 0.0f;
    }
    for (int kb = 0; kb < n_kb; ++kb) {
        const int st = kb & 1;
        if (kb + 1 < n_kb) {
            load_tile<HD, kBN>(sK + (st ^ 1) * kBN * LD, qkv, row0, (kb + 1) * kBN, sh.S, sh.ld, kcol);
            load_tile<HD, kBN>(sV + (st ^ 1) * kBN * LD, qkv, row0, (kb + 1) * kBN, sh.S, sh.ld, vcol);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kb == 0) {
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                ldsm_x4(qf[k], a_addr<LD>(sQ, warp * 16, k * 16, lane));
                ldsm_x4(df[k], a_addr<LD>(sD, warp * 16, k * 16, lane));
            }
        }
        const __nv_bfloat16* tK = sK + st * kBN * LD;
        const __nv_bfloat16* tV = sV + st * kBN * LD;
        const int k0 = kb * kBN;
        const bool active = !sh.causal || k0 <= q0 + warp * 16 + 15;
        if (active) {
            float s[8][4], dp[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.0f;
#pragma unroll
            for (int k = 0; k < KB; ++k) {
#pragma unroll
                for (int np = 0; np < 4; ++np) {
                    uint32_t kf[4], vf[4];
                    ldsm_x4(kf, bn_addr<LD>(tK, np * 16, k * 16, lane));
                    ldsm_x4(vf, bn_addr<LD>(tV, np * 16, k * 16, lane));
                    mma16816(s[2 * np], qf[k], kf[0], kf[1]);
                    mma16816(s[2 * np + 1], qf[k], kf[2], kf[3]);
                    mma16816(dp[2 * np], df[k], vf[0], vf[1]);
                    mma16816(dp[2 * np + 1], df[k], vf[2], vf[3]);
                }
            }
            const bool need_mask = (sh.causal && k0 + kBN - 1 > q0 + warp * 16) || k0 + kBN > sh.S;
            uint32_t dsf[4][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float ds[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = e >> 1;
                    float p = ex2f(fmaf(s[i][e], sh.scale_log2, -L[r]));
                    if (need_mask) {
                        const int key = k0 + i * 8 + 2 * t + (e & 1);
                        if (key >= sh.S || (sh.causal && key > qr0 + r * 8)) p = 0.0f;
                    }
                    ds[e] = p * (dp[i][e] - Dl[r]);
                }
                dsf[i >> 1][(i & 1) * 2 + 0] = pack2(ds[0], ds[1]);
                dsf[i >> 1][(i & 1) * 2 + 1] = pack2(ds[2], ds[3]);
            }
            // dQ += dS K  (B = K as a [k = key][n = d] tile, transposed loads)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
                for (int np = 0; np < NT / 2; ++np) {
                    uint32_t kf[4];
                    ldsm_x4_t(kf, bt_addr<LD>(tK, kk * 16, np * 16, lane));
                    mma16816(dq[2 * np], dsf[kk], kf[0], kf[1]);
                    mma16816(dq[2 * np + 1], dsf[kk], kf[2], kf[3]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = qr0 + r * 8;
        if (q >= sh.S) continue;
        __nv_bfloat16* drow = dqkv + (row0 + q) * sh.ld + qcol;
#pragma unroll
        for (int i = 0; i < NT; ++i)
            *reinterpret_cast<uint32_t*>(drow + i * 8 + 2 * t) = pack2(dq[i][2 * r] * scale, dq[i][2 * r + 1] * scale);
    }
}

template <int HD>
constexpr int fwd_smem() {
    return (kBM + 4 * kBN) * Tile<HD>::LD * 2;
}
template <int HD>
constexpr int dkdv_smem() {
    return (2 * kBM + 4 * kBN) * Tile<HD>::LD * 2 + 4 * kBN * 4;
}
template <int HD>
constexpr int dq_smem() {
    return (2 * kBM + 4 * kBN) * Tile<HD>::LD * 2;
}

AttnShape shape_of(const AttnProblem& a) {
    AttnShape sh;
    sh.S = a.seq_len;
    sh.H = a.n_heads;
    sh.Hkv = a.n_kv_heads;
    sh.ld = (a.n_heads + 2 * a.n_kv_heads) * a.head_dim;
    sh.ldo = a.n_heads * a.head_dim;
    sh.causal = a.causal;
    const float scale = 1.0f / sqrtf(static_cast<float>(a.head_dim));
    sh.scale_log2 = scale * 1.4426950408889634f;
    return sh;
}

template <int HD>
cudaError_t fwd_hd(const AttnProblem& a, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem<HD>());
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const AttnShape sh = shape_of(a);
    const int n_seq = static_cast<int>(a.tokens / a.seq_len);
    dim3 grid((a.seq_len + kBM - 1) / kBM, a.n_heads, n_seq);
    return launch_kernel(attn_fwd_kernel<HD>, grid, dim3(kThreads), fwd_smem<HD>(), st,
                         static_cast<const __nv_bfloat16*>(a.qkv), static_cast<__nv_bfloat16*>(a.o), a.lse, sh);
}

template <int HD>
cudaError_t bwd_hd(const AttnProblem& a, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_bwd_dkdv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             dkdv_smem<HD>());
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attn_bwd_dq_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, dq_smem<HD>());
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const AttnShape sh = shape_of(a);
    const int n_seq = static_cast<int>(a.tokens / a.seq_len);
    const float scale = 1.0f / sqrtf(static_cast<float>(a.head_dim));
    const int64_t th = a.tokens * a.n_heads;
    if (g_attn_bwd_kind == 0) {  // tcgen05 dQ (+ delta) and dK/dV passes, v2, where the shape allows
        cudaError_t e2 = attention_backward_tc2(a, st);
        if (e2 != cudaErrorNotSupported) return e2;
    }
    cudaError_t e = launch_kernel(attn_bwd_delta_kernel<HD>, dim3(static_cast<unsigned>((th + 255) / 256)), dim3(256), 0,
                                  st, static_cast<const __nv_bfloat16*>(a.o), static_cast<const __nv_bfloat16*>(a.dout),
                                  a.delta, a.tokens, sh);
    if (e != cudaSuccess) return e;
    if (g_attn_bwd_kind == 0 || g_attn_bwd_kind == 2) {  // tcgen05 dK/dV and dQ passes, v1
        e = attention_backward_tc(a, st);
        if (e != cudaErrorNotSupported) return e;
    }
    dim3 gkv((a.seq_len + kBM - 1) / kBM, a.n_kv_heads, n_seq);
    e = launch_kernel(attn_bwd_dkdv_kernel<HD>, gkv, dim3(kThreads), dkdv_smem<HD>(), st,
                      static_cast<const __nv_bfloat16*>(a.qkv), static_cast<const __nv_bfloat16*>(a.dout), a.lse,
                      static_cast<const float*>(a.delta), static_cast<__nv_bfloat16*>(a.dqkv), sh, scale);
    if (e != cudaSuccess) return e;
    dim3 gq((a.seq_len + kBM - 1) / kBM, a.n_heads, n_seq);
    return launch_kernel(attn_bwd_dq_kernel<HD>, gq, dim3(kThreads), dq_smem<HD>(), st,
                         static_cast<const __nv_bfloat16*>(a.qkv), static_cast<const __nv_bfloat16*>(a.dout), a.lse,
                         static_cast<const float*>(a.delta), static_cast<__nv_bfloat16*>(a.dqkv), sh, scale);
}

bool valid(const AttnProblem& a) {
    return a.seq_len > 0 && a.tokens > 0 && a.tokens % a.seq_len == 0 && a.n_heads > 0 && a.n_kv_heads > 0 &&
           a.n_heads % a.n_kv_heads == 0;
}

}  // namespace

// Forward kind (A/B knob "attn_fwd", sp_debug_set): 0 (default) = 4 where a tcgen05 kernel covers the
// head dim (64, 80, 128); 4: v3 tcgen05 (8 softmax warps, P in TMEM, O accumulated in TMEM with a
// lazy rescale); 2: v2 (O accumulated in registers, one block behind); 3: v1 (4 softmax warps;
// head_dim 80 then takes the mma.sync kernel); 1: always the mma.sync kernel.
int g_attn_fwd_kind = 0;
int g_attn_bwd_kind = 0;
int g_attn_chunk = 0;  // sp_debug_set "attn_chunk": causal work-order chunk (0 = by shape)

// Chunked only when the whole K / V outgrows the 126 MB L2: Llama-3-8B's 268 MB at 32 x 2048
// tokens (chunks of 32: forward 1809 -> 1512 us, backward 4.91 -> 4.49 ms per layer); GPT-2 XL's
// 105 MB is re-read from L2 anyway, where chunks of 32..256 measured 1-4% slower than the plain
// longest-first order (tools/attn_probe.py, SP_ATTN_CHUNK).
int attention_causal_chunk(const AttnProblem& a) {
    if (g_attn_chunk > 0) return g_attn_chunk;
    const double kv_bytes = static_cast<double>(a.tokens) * a.n_kv_heads * a.head_dim * 4.0;
    return kv_bytes > 126e6 ? 32 : 1 << 30;
}

cudaError_t attention_forward_tc(const AttnProblem& a, cudaStream_t st, int kind);  // kernels_attn_tc.cu

cudaError_t attention_forward(const AttnProblem& a, cudaStream_t st) {
    if (!valid(a)) return cudaErrorInvalidValue;
    // tcgen05 forward for head_dim 64 / 128 (persistent; tools/attn_probe.py), mma.sync for 80
    if (g_attn_fwd_kind != 1 && (a.head_dim == 64 || a.head_dim == 128 || (a.head_dim == 80 && g_attn_fwd_kind != 3)))
        return attention_forward_tc(a, st, g_attn_fwd_kind == 0 ? 4 : g_attn_fwd_kind);
    switch (a.head_dim) {
        case 64: return fwd_hd<64>(a, st);
        case 80: return fwd_hd<80>(a, st);
        case 128: return fwd_hd<128>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t attention_backward(const AttnProblem& a, cudaStream_t st) {
    if (!valid(a)) return cudaErrorInvalidValue;
    switch (a.head_dim) {
        case 64: return bwd_hd<64>(a, st);
        case 80: return bwd_hd<80>(a, st);
        case 128: return bwd_hd<128>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sp

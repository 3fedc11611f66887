// kernels_attn_bwd.cu — tcgen05 flash-attention backward (sm_100a), head_dim 64 / 128.
//
// Two persistent kernels, deterministic (every output element is one fixed-order reduction, no
// atomics), head_dim 64 / 80 / 128, any sequence length (a ragged last block is masked):
//
//   dQ pass   tile = 128 queries of one (sequence, head); streams 64-key steps of K, V:
//               S = Q K^T, dP = dO V^T                        (TMEM, fp32, M 128 x N 64)
//               dS = exp2(S c - lse) (dP - delta)             (softmax warps, bf16 -> TMEM)
//               dQ += dS K                                    (A = dS from TMEM, B = K N-major)
//             delta = rowsum(dO . O) is formed here (thread = query row) and written for the
//             dK/dV pass, so no separate delta kernel runs.
//   dK/dV pass tile = 128 keys of one (sequence, kv head); streams 64-query steps of Q, dO for
//             every query head of the group:
//               S^T = K Q^T, dP^T = V dO^T                    (TMEM)
//               P^T = exp2(S^T c - lse), dS^T = P^T (dP^T - delta)   (bf16 -> TMEM)
//               dV += P^T dO, dK += dS^T Q                    (A from TMEM, B = dO / Q N-major)
//
// Warp roles (384 threads): warp 0 TMA producer, warp 1 MMA issuer (one thread), warp 2 TMEM
// allocator, warps 4..11 the elementwise ("softmax") work in two warpgroups: warpgroup wg takes
// the steps of parity wg (both 32-row halves of each), so the two warps of an SM sub-partition
// work on different steps and overlap each other's TMEM-load, MUFU and barrier latencies. P / dS
// are written into TMEM (each thread only its own lane) and consumed straight from TMEM by the
// tcgen05.mma A operand — no shared-memory round trip for the probability tiles.
//
// TMEM columns. dQ pass: S / dP of step b at 128 b (b = step mod 2), dS in a separate region
// from 256, dQ from 320. dK/dV pass: S / dP in NB buffers at 128 b (b = step mod NB; NB = 3 at
// head_dim 64, 2 at 128), P / dS written back over the S / dP columns they were computed from,
// dK then dV from 128 NB. The S / dP MMAs of step j + NB are issued after the products of step
// j, which read that buffer (one issuing thread: in order).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <type_traits>

#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace sp {
extern int g_attn_trace;  // sp_debug_set "attn_trace" (defined below)
extern int g_attn_bwd_kind;  // kernels_attn.cu
namespace {
using namespace tc;

constexpr int kThreadsB = 384;
constexpr int kRowsB = 128;  // the CTA tile's own rows (queries in dQ, keys in dK/dV)
constexpr int kStepB = 64;   // rows streamed per step (keys in dQ, queries in dK/dV)
// lse / delta stage stride (floats): a step's 64 values plus up to 3 of 16-byte alignment slack
// (rows of a ragged sequence start at any float)
constexpr int kLStride = 72;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Debug timeline of the dK/dV pass (sp_debug_set "attn_trace" 1; tools/attn_trace.py): CTA 0
// records (event, step, SM clock) for the first kTraceCap events; a separate instantiation, so the
// product kernel carries none of it.
constexpr int kTraceCap = 4096;
__device__ unsigned long long g_bwd_trace[kTraceCap];
__device__ unsigned int g_bwd_trace_n;
template <bool TRACE>
__device__ __forceinline__ void trace_ev(int ev, int step) {
    if (!TRACE || blockIdx.x != 0) return;
    const unsigned int i = atomicAdd(&g_bwd_trace_n, 1u);
    if (i < kTraceCap)
        g_bwd_trace[i] = (static_cast<unsigned long long>(ev) << 56) | (static_cast<unsigned long long>(step & 0xFFFF) << 40) |
                         (clock64() & 0xFFFFFFFFFFull);
}

__device__ __forceinline__ void bulk_load_b(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// K-major tile of `atom` bytes per 64-element column atom (128 B rows, 128B swizzle), 16-element
// K step kk
__device__ __forceinline__ uint64_t kmaj(uint32_t base, int kk, int atom) {
    return make_desc(base + (kk / 4) * atom + (kk % 4) * 32, 16, 1024);
}
// the same tile as an N-major B operand (K = its rows): 16-row K step kk, atoms `atom` apart in N
__device__ __forceinline__ uint64_t nmaj(uint32_t base, int kk, int atom) {
    return make_desc(base + kk * 16 * 128, atom, 1024);
}
// A-operand TMEM column of K step kk (16 rows of the step) of a P / dS tile written by the two
// half-warps: separate regions hold it contiguously (half h at 16 h); written back over S / dP,
// half h sits at its own columns 32 h .. 32 h + 15
template <bool SEP>
__device__ __forceinline__ uint32_t ts_col(int kk) {
    return SEP ? static_cast<uint32_t>(8 * kk) : static_cast<uint32_t>((kk >> 1) * 32 + (kk & 1) * 8);
}
// a descriptor advanced by `bytes` (the 14-bit start field cannot carry: smem < 256 KB)
__device__ __forceinline__ uint64_t dadd(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }
// head_dim 80's 16-column tails: 32B swizzle (layout 6), 8-row groups 256 bytes apart; K-major
// (the last K step of QK^T-like products) or, as one 16-column MN-major atom, the N = 16 half
// of the products against the streamed tile
__device__ __forceinline__ uint64_t tail_desc(uint32_t saddr) { return make_desc(saddr, 256, 256, 6); }

struct BShape {
    int S, H, Hkv, ld, ldo, causal, chunk;  // chunk: causal work order (causal_chunked)
    float scale_log2, scale;
};

template <int HD>
struct BCfg {
    // head_dim 80 (ViT-H/14) takes two 64-column atoms; the MMAs read the first HD columns only
    static constexpr int ATOMS = (HD + 63) / 64;
    // head_dim 80: the 16 columns past the first atom are a 32B-swizzled [rows][16] tile (own
    // TMA maps), not a second 64-column atom: 160 instead of 256 bytes per row
    static constexpr bool NARROW = HD % 64 == 16;
    static constexpr int BIG = NARROW ? kRowsB * (128 + 32) : kRowsB * ATOMS * 128;    // a 128-row tile
    static constexpr int SMALL = NARROW ? kStepB * (128 + 32) : kStepB * ATOMS * 128;  // a 64-row tile
    static constexpr int A_BIG = kRowsB * 128, A_SMALL = kStepB * 128;  // the second atom / the tail
    static constexpr int ST = HD == 64 ? 8 : 3;                 // streamed-tile stages
    // own-tile stages (next tile prefetch): head_dim 80's narrow tiles make room for the second
    // (ViT backward 1154 -> 1100 us; six streamed stages instead measured slower, 1156-1190 us)
    static constexpr int OWN = (HD == 64 || NARROW) ? 2 : 1;
    // dK/dV pass: P / dS written back over S / dP in NB_DKDV buffers. Three buffers at head_dim
    // 64 (dK, dV from column 384) let a warpgroup's next step start without waiting for its
    // previous step's products (the separate-region double-buffered form, SEP, waited there:
    // ncu, 21% of the softmax warps' samples on that barrier); two at 128.
    static constexpr bool SEP_DKDV = false;
    static constexpr int NB_DKDV = HD == 64 ? 3 : 2;
    static constexpr int SMEM_DKDV = OWN * 2 * BIG + ST * 2 * SMALL + ST * 2 * kLStride * 4 + 1024 + 512;
    static constexpr int SMEM_DQ = OWN * 2 * BIG + ST * 2 * SMALL + 1024 + 512;
};

// NC accumulator columns of this thread's TMEM lane (from column `col`), times `sc`, to bf16 at
// `dst` (NC % 8 == 0): 32-column loads while they fit, then 8-column ones (head_dim 80). With
// `csum` (NC % 32 == 0), also the column sums of the warp's 32 rows (invalid rows as 0) into
// csum[c * 32 + lane] (a lane-order reduce-scatter per 32 columns).
__device__ __forceinline__ float warp_colsum32(float (&a)[32], int lane) {
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const bool up = (lane & w) != 0;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const float send = up ? a[i] : a[i + w];
            const float recv = __shfl_xor_sync(0xffffffffu, send, w);
            a[i] = (up ? a[i + w] : a[i]) + recv;
        }
    }
    return a[0];
}
template <int NC>
__device__ __forceinline__ void acc_row_out(uint32_t taddr, __nv_bfloat16* dst, float sc, bool store,
                                            float* csum = nullptr, int lane = 0) {
    uint32_t v[32];
#pragma unroll
    for (int c = 0; c < NC / 32; ++c) {
        tmem_ld32_async(taddr + c * 32, v);
        tmem_ld_wait(v);
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) * sc;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4 w;
            w.x = pack_bf16(f[8 * u + 0], f[8 * u + 1]);
            w.y = pack_bf16(f[8 * u + 2], f[8 * u + 3]);
            w.z = pack_bf16(f[8 * u + 4], f[8 * u + 5]);
            w.w = pack_bf16(f[8 * u + 6], f[8 * u + 7]);
            if (store) reinterpret_cast<uint4*>(dst + c * 32)[u] = w;
        }
        if (csum) {  // (warp-uniform)
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] = store ? f[i] : 0.0f;
            csum[c * 32 + lane] = warp_colsum32(f, lane);
        }
    }
#pragma unroll
    for (int c = (NC / 32) * 4; c < NC / 8; ++c) {
        uint32_t v8[8];
        tmem_ld8(taddr + c * 8, v8);
        uint4 w;
        w.x = pack_bf16(__uint_as_float(v8[0]) * sc, __uint_as_float(v8[1]) * sc);
        w.y = pack_bf16(__uint_as_float(v8[2]) * sc, __uint_as_float(v8[3]) * sc);
        w.z = pack_bf16(__uint_as_float(v8[4]) * sc, __uint_as_float(v8[5]) * sc);
        w.w = pack_bf16(__uint_as_float(v8[6]) * sc, __uint_as_float(v8[7]) * sc);
        if (store) reinterpret_cast<uint4*>(dst + c * 8)[0] = w;
    }
}

// ------------------------------------------------------------------------------------------
// dQ (+ delta)
// ------------------------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(kThreadsB, 1)
    attn_bwd_dq2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
                        const __grid_constant__ CUtensorMap tmKV, const __grid_constant__ CUtensorMap tmQ1,
                        const __grid_constant__ CUtensorMap tmDO1, const __grid_constant__ CUtensorMap tmKV1,
                        const __nv_bfloat16* __restrict__ o,
                        const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                        float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, BShape sh, int n_seq,
                        float* __restrict__ csum) {
    using C = BCfg<HD>;
    constexpr uint32_t T_DS = 256, T_ACC = 320;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // (stays a shared pointer)
    uint8_t* sQ = smem;                      // OWN
    uint8_t* sDO = sQ + C::OWN * C::BIG;     // OWN
    uint8_t* sK = sDO + C::OWN * C::BIG;     // ST
    uint8_t* sV = sK + C::ST * C::SMALL;     // ST
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::ST * C::SMALL);
    uint64_t* q_full = bars;                 // OWN
    uint64_t* q_empty = bars + 2;            // OWN
    uint64_t* kv_full = bars + 4;            // ST
    uint64_t* kv_empty = kv_full + C::ST;    // ST
    uint64_t* s_full = kv_empty + C::ST;     // 2: S / dP of the step are in TMEM
    uint64_t* s_free = s_full + 2;           // 2: the softmax warps have loaded them
    uint64_t* p_full = s_free + 2;           // 2: dS is in TMEM
    uint64_t* ds_free = p_full + 2;          // 2: the dQ MMAs have read it
    uint64_t* acc_full = ds_free + 2;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // ragged sequences (ViT's 257 tokens): the last query block / key step is partial; rows past
    // the sequence are masked (keys) or never stored (queries)
    const int n_qb = (sh.S + kRowsB - 1) / kRowsB, n_ks = (sh.S + kStepB - 1) / kStepB;
    const int n_tiles = n_qb * sh.H * n_seq;
    // tile t: (query block, head, sequence), query blocks descending (causal: longest first);
    // without the mask, query blocks innermost (one DRAM read of K / V, as the forward's tile_of)
    auto tile = [&](int t, int& qb, int& h, int& b) {
        const int per = sh.H * n_seq;
        int rest;
        if (sh.causal) {
            causal_chunked(t, per, n_qb, true, sh.chunk, qb, rest);  // (the forward's chunked order)
        } else {
            rest = t / n_qb;
            qb = t % n_qb;
        }
        h = rest % sh.H;
        b = rest / sh.H;
    };
    auto steps = [&](int qb) { return sh.causal ? min(2 * (qb + 1), n_ks) : n_ks; };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmQ);
        prefetch_tmap(&tmDO);
        prefetch_tmap(&tmKV);
        for (int i = 0; i < C::OWN; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < C::ST; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 128);  // one warpgroup per step
            mbar_init(&p_full[i], 128);
            mbar_init(&ds_free[i], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 256);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int qb, h, b;
                tile(t, qb, h, b);
                const int kvh = h / (sh.H / sh.Hkv);
                const int row0 = b * sh.S;
                const int ob = lt % C::OWN;
                mbar_wait(&q_empty[ob], ((lt / C::OWN) & 1) ^ 1);
                mbar_expect_tx(&q_full[ob], 2 * C::BIG);
                for (int a = 0; a < C::ATOMS; ++a) {
                    tma_load_2d(C::NARROW && a ? &tmQ1 : &tmQ, &q_full[ob], sQ + ob * C::BIG + a * C::A_BIG, h * HD + 64 * a,
                                row0 + qb * kRowsB);
                    tma_load_2d(C::NARROW && a ? &tmDO1 : &tmDO, &q_full[ob], sDO + ob * C::BIG + a * C::A_BIG, h * HD + 64 * a,
                                row0 + qb * kRowsB);
                }
                const int kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
                const int n = steps(qb);
                for (int j = 0; j < n; ++j, ++g) {
                    const int st = g % C::ST;
                    mbar_wait(&kv_empty[st], ((g / C::ST) & 1) ^ 1);
                    mbar_expect_tx(&kv_full[st], 2 * C::SMALL);
                    for (int a = 0; a < C::ATOMS; ++a) {
                        tma_load_2d(C::NARROW && a ? &tmKV1 : &tmKV, &kv_full[st], sK + st * C::SMALL + a * C::A_SMALL,
                                    kcol + 64 * a, row0 + j * kStepB);
                        tma_load_2d(C::NARROW && a ? &tmKV1 : &tmKV, &kv_full[st], sV + st * C::SMALL + a * C::A_SMALL,
                                    vcol + 64 * a, row0 + j * kStepB);
                    }
                }
            }
        }
    } else if (warp == 1) {
        {  // the whole warp runs the loop; the elected lane issues
            const uint32_t leader = elect_one();  // ===== MMA issuer =====
            constexpr uint32_t ID_S = make_idesc(128, kStepB, false, false);
            constexpr uint32_t ID_D = make_idesc(128, HD, false, true);
            constexpr uint32_t ID_D64 = make_idesc(128, 64, false, true), ID_D16 = make_idesc(128, 16, false, true);
            uint64_t dq_, ddo_;  // the tile's Q / dO descriptors (K-major, k step 0)
            uint32_t q_own = 0, do_own = 0;  // (their shared addresses: the tails)
            // S / dP of step gg into buffer gg & 1, once the softmax warps have loaded step gg - 2's
            auto issue_s = [&](int gg) {
                const int st = gg % C::ST, bb = gg & 1;
                mbar_wait(&kv_full[st], (gg / C::ST) & 1);
                if (gg >= 2) mbar_wait(&s_free[bb], ((gg - 2) >> 1) & 1);
                fence_after();
                const uint64_t dk = make_desc(smem_u32(sK + st * C::SMALL), 16, 1024);
                const uint64_t dv = make_desc(smem_u32(sV + st * C::SMALL), 16, 1024);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t ob = (kk / 4) * C::A_BIG + (kk % 4) * 32, sb = (kk / 4) * C::A_SMALL + (kk % 4) * 32;
                    if (C::NARROW && kk == 4) {
                        umma_if(leader, tmem + 128 * bb, tail_desc(q_own + C::A_BIG),
                                tail_desc(smem_u32(sK + st * C::SMALL + C::A_SMALL)), ID_S, 1);
                        umma_if(leader, tmem + 128 * bb + 64, tail_desc(do_own + C::A_BIG),
                                tail_desc(smem_u32(sV + st * C::SMALL + C::A_SMALL)), ID_S, 1);
                    } else {
                        umma_if(leader, tmem + 128 * bb, dadd(dq_, ob), dadd(dk, sb), ID_S, kk > 0);
                        umma_if(leader, tmem + 128 * bb + 64, dadd(ddo_, ob), dadd(dv, sb), ID_S, kk > 0);
                    }
                }
                umma_commit_if(leader, &s_full[bb]);
            };
            // dQ += dS K of step gg
            auto issue_d = [&](int gg, bool first) {
                const int st = gg % C::ST, bb = gg & 1;
                mbar_wait(&p_full[bb], (gg >> 1) & 1);
                fence_after();
                const uint64_t dk = make_desc(smem_u32(sK + st * C::SMALL), C::A_SMALL, 1024);
#pragma unroll
                for (int kk = 0; kk < kStepB / 16; ++kk) {
                    const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
                    if (C::NARROW) {  // dQ columns 0..63 from K's atom, 64..79 from its tail
                        umma_ts_if(leader, tmem + T_ACC, tmem + T_DS + 32 * bb + ts_col<true>(kk), dadd(dk, kk * 2048),
                                   ID_D64, acc);
                        umma_ts_if(leader, tmem + T_ACC + 64, tmem + T_DS + 32 * bb + ts_col<true>(kk),
                                   tail_desc(smem_u32(sK + st * C::SMALL + C::A_SMALL) + kk * 512), ID_D16, acc);
                    } else {
                        umma_ts_if(leader, tmem + T_ACC, tmem + T_DS + 32 * bb + ts_col<true>(kk), dadd(dk, kk * 2048), ID_D,
                                   acc);
                    }
                }
                umma_commit_if(leader, &ds_free[bb]);
                umma_commit_if(leader, &kv_empty[st]);
            };
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int qb, h, b;
                tile(t, qb, h, b);
                const int n = steps(qb);
                const int ob = lt % C::OWN;
                mbar_wait(&q_full[ob], (lt / C::OWN) & 1);
                q_own = smem_u32(sQ + ob * C::BIG);
                do_own = smem_u32(sDO + ob * C::BIG);
                dq_ = make_desc(q_own, 16, 1024);
                ddo_ = make_desc(do_own, 16, 1024);
                for (int i = 0; i < 2 && i < n; ++i) issue_s(g + i);  // (one step: a sequence <= 64 keys)
                mbar_wait(acc_empty, (lt & 1) ^ 1);  // the previous tile's dQ is read out
                fence_after();
                for (int j = 0; j < n; ++j) {
                    // step j's dQ product first, then S / dP of step j + 2: an S issue waiting for
                    // its K / V tile must not hold back the product the next dS buffer waits for
                    // (Llama-3 shape: 6.2 -> 5.3 ms for both passes; GPT-2 XL unchanged)
                    issue_d(g + j, j == 0);
                    if (j + 2 < n) issue_s(g + j + 2);
                }
                umma_commit_if(leader, acc_full);
                umma_commit_if(leader, &q_empty[ob]);
                g += n;
            }
        }
    } else if (warp >= 4) {
        // ===== elementwise: thread = query row; warpgroup wg takes the steps of parity wg (both
        // 32-key halves of each), as in the dK/dV pass =====
        const int q4 = warp & 3, wg = (warp - 4) >> 2;
        const int half = wg;  // (delta store and the tile's dQ readout: half the columns each)
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        uint32_t vs[32], vp[32];
        // this thread's O and dO rows of the next tile, prefetched during the current one: whole
        // rows at head_dim 64; at 80 / 128 each warpgroup takes half the columns and the two
        // partial dot products meet in shared memory (the registers of whole rows would spill)
        constexpr bool kHalfRows = HD != 64;
        constexpr int NR = kHalfRows ? HD / 16 : HD / 8;
        __shared__ float xdl[2][2][kRowsB];  // [tile parity][half][row] partial deltas
        uint4 ro[NR], rd[NR];
        auto load_rows = [&](int tt) {
            int qb_, h_, b_;
            tile(tt, qb_, h_, b_);
            const bool in = qb_ * kRowsB + r < sh.S;
            const int64_t tk = static_cast<int64_t>(b_) * sh.S + qb_ * kRowsB + r;
            const int c0 = h_ * HD + (kHalfRows ? half * (HD / 2) : 0);
            const uint4* a4 = reinterpret_cast<const uint4*>(o + tk * sh.ldo + c0);
            const uint4* c4 = reinterpret_cast<const uint4*>(dout + tk * sh.ldo + c0);
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                ro[j] = in ? __ldg(a4 + j) : make_uint4(0u, 0u, 0u, 0u);
                rd[j] = in ? __ldg(c4 + j) : make_uint4(0u, 0u, 0u, 0u);
            }
        };
        int g = 0, lt = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
            int qb, h, b;
            tile(t, qb, h, b);
            const int qi = qb * kRowsB + r;
            const int64_t tok = static_cast<int64_t>(b) * sh.S + qi;
            const int64_t li = (static_cast<int64_t>(b) * sh.H + h) * sh.S + qi;
            const bool q_in = qi < sh.S;
            const float L = q_in ? lse[li] : 0.0f;
            // delta = sum_d dO . O of this row (half 0 stores it), from rows prefetched into
            // registers during the previous tile
            if (t == static_cast<int>(blockIdx.x)) load_rows(t);
            float Dl = 0.0f;
#pragma unroll
            for (int j = 0; j < NR; ++j) {
                const uint32_t wa[4] = {ro[j].x, ro[j].y, ro[j].z, ro[j].w}, wc[4] = {rd[j].x, rd[j].y, rd[j].z, rd[j].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wa[k]));
                    const float2 fc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wc[k]));
                    Dl += fa.x * fc.x + fa.y * fc.y;
                }
            }
            if (t + static_cast<int>(gridDim.x) < n_tiles) load_rows(t + gridDim.x);
            if (kHalfRows) {  // the row's two halves (warps q4 of both warpgroups) meet
                xdl[lt & 1][half][r] = Dl;
                asm volatile("bar.sync %0, 64;" ::"r"(1 + q4) : "memory");
                Dl = xdl[lt & 1][0][r] + xdl[lt & 1][1][r];
            }
            if (half == 0 && q_in) delta[li] = Dl;
            const int n = steps(qb);
            for (int j = 0; j < n; ++j, ++g) {
                if ((g & 1) != wg) continue;  // the other warpgroup's step
                const int bb = g & 1;
                if (g >= 2) mbar_wait(&ds_free[bb], ((g - 2) >> 1) & 1);  // step g - 2's dQ product read it
                mbar_wait(&s_full[bb], (g >> 1) & 1);
                fence_after();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    tmem_ld32_async(tmem + lane_off + 128 * bb + 32 * h, vs);
                    tmem_ld32_async(tmem + lane_off + 128 * bb + 64 + 32 * h, vp);
                    tmem_ld_wait(vs);
                    tmem_ld_wait(vp);
                    if (h == 1) {
                        fence_before();
                        mbar_arrive(&s_free[bb]);  // the MMAs of step g + 2 may overwrite S / dP now
                    }
                    const int k0 = j * kStepB + 32 * h;                  // first key of this half
                    // some key above some query, or past the sequence
                    const bool mask = (sh.causal && k0 + 31 > qb * kRowsB) || k0 + 32 > sh.S;
                    const int klim = sh.causal ? min(qi + 1, sh.S) : sh.S;  // keys < klim are valid
                    uint32_t dd[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float2 x = ffma2(make_float2(__uint_as_float(vs[2 * i]), __uint_as_float(vs[2 * i + 1])),
                                               make_float2(sh.scale_log2, sh.scale_log2), make_float2(-L, -L));
                        float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
                        if (mask) {
                            if (k0 + 2 * i >= klim) p0 = 0.0f;
                            if (k0 + 2 * i + 1 >= klim) p1 = 0.0f;
                        }
                        const float2 d = fmul2(make_float2(p0, p1),
                                               fsub2(make_float2(__uint_as_float(vp[2 * i]), __uint_as_float(vp[2 * i + 1])),
                                                     make_float2(Dl, Dl)));
                        dd[i] = pack_bf16(d.x, d.y);
                    }
                    tmem_st16(tmem + lane_off + T_DS + 32 * bb + 16 * h, dd);
                }
                tmem_st_wait();
                fence_before();
                mbar_arrive(&p_full[bb]);
            }
            mbar_wait(acc_full, lt & 1);
            fence_after();
            // this half's HD / 2 columns of the query row's dQ (rows past the sequence: not stored)
            // (+ bqkv's column sums of these dQ columns over the warp's 32 rows, when asked)
            // (a warp's 32 rows are all in the sequence or all padding past it: seq_len % 32 == 0;
            // padding warps must not write - their token index belongs to the next sequence)
            const bool warp_in = qb * kRowsB + q4 * 32 < sh.S;
            float* cs = csum && warp_in ? csum + (tok - r % 32) / 32 * sh.ld + h * HD + half * (HD / 2) : nullptr;
            acc_row_out<HD / 2>(tmem + lane_off + T_ACC + half * (HD / 2), dqkv + tok * sh.ld + h * HD + half * (HD / 2),
                                sh.scale, q_in, cs, lane);
            fence_before();
            mbar_arrive(acc_empty);
        }
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------------------------------
// dK, dV
// ------------------------------------------------------------------------------------------
template <int HD, bool SEP, int NB, bool TRACE = false>
__global__ void __launch_bounds__(kThreadsB, 1)
    attn_bwd_dkdv2_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmDO, const __grid_constant__ CUtensorMap tmK1,
                          const __grid_constant__ CUtensorMap tmQ1, const __grid_constant__ CUtensorMap tmDO1,
                          const float* __restrict__ lse,
                          const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, BShape sh, int n_seq,
                          float* __restrict__ csum) {
    using C = BCfg<HD>;
    // TMEM map (header): P / dS regions of buffer b, then dK and dV
    // NB S / dP buffers (P / dS written back over them when !SEP); SEP uses 2 + separate P / dS
    static_assert(!SEP || NB == 2, "separate P / dS regions are double-buffered");
    constexpr uint32_t T_ACC = SEP ? 384 : 128 * NB;
    static_assert(T_ACC + 2 * HD <= 512, "dK / dV do not fit in TMEM");
    auto p_col = [](int bb) { return SEP ? 256u + 64u * bb : 128u * bb; };
    auto ds_col = [](int bb) { return SEP ? 288u + 64u * bb : 128u * bb + 64u; };
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // (stays a shared pointer)
    uint8_t* sK = smem;                      // OWN
    uint8_t* sV = sK + C::OWN * C::BIG;      // OWN
    uint8_t* sQ = sV + C::OWN * C::BIG;      // ST
    uint8_t* sDO = sQ + C::ST * C::SMALL;    // ST
    float* sL = reinterpret_cast<float*>(sDO + C::ST * C::SMALL);  // ST x kLStride
    float* sD = sL + C::ST * kLStride;                              // ST x kLStride
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + C::ST * kLStride);
    uint64_t* kv_full = bars;                // OWN
    uint64_t* kv_empty = bars + 2;           // OWN
    uint64_t* q_full = bars + 4;             // ST
    uint64_t* q_empty = q_full + C::ST;      // ST
    uint64_t* s_full = q_empty + C::ST;      // NB
    uint64_t* s_free = s_full + NB;          // 2 (SEP)
    uint64_t* p_full = s_free + 2;           // NB
    uint64_t* ds_free = p_full + NB;         // 2 (SEP)
    uint64_t* acc_full = ds_free + 2;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_kb = (sh.S + kRowsB - 1) / kRowsB, n_qs = (sh.S + kStepB - 1) / kStepB;  // (ragged: as dQ)
    const int group = sh.H / sh.Hkv;
    const int n_tiles = n_kb * sh.Hkv * n_seq;
    // tile t: (key block, kv head, sequence), key blocks ascending (causal: longest first);
    // without the mask, key blocks innermost (one DRAM read of Q / dO per (sequence, head))
    auto tile = [&](int t, int& kb, int& kvh, int& b) {
        const int per = sh.Hkv * n_seq;
        int rest;
        if (sh.causal) {
            causal_chunked(t, per, n_kb, false, sh.chunk, kb, rest);  // key block 0 (the longest) first
        } else {
            rest = t / n_kb;
            kb = t % n_kb;
        }
        kvh = rest % sh.Hkv;
        b = rest / sh.Hkv;
    };
    auto per_head = [&](int kb) { return sh.causal ? n_qs - 2 * kb : n_qs; };
    auto step_of = [&](int kb, int kvh, int j, int& hq, int& qs) {
        const int per = per_head(kb);
        hq = kvh * group + j / per;
        qs = (sh.causal ? 2 * kb : 0) + j % per;
    };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmQ);
        prefetch_tmap(&tmDO);
        for (int i = 0; i < C::OWN; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < C::ST; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < NB; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);  // one warpgroup per step
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_free[i], 128);
            mbar_init(&ds_free[i], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 256);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int kb, kvh, b;
                tile(t, kb, kvh, b);
                const int row0 = b * sh.S;
                const int kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
                const int ob = lt % C::OWN;
                mbar_wait(&kv_empty[ob], ((lt / C::OWN) & 1) ^ 1);
                mbar_expect_tx(&kv_full[ob], 2 * C::BIG);
                for (int a = 0; a < C::ATOMS; ++a) {
                    tma_load_2d(C::NARROW && a ? &tmK1 : &tmK, &kv_full[ob], sK + ob * C::BIG + a * C::A_BIG, kcol + 64 * a,
                                row0 + kb * kRowsB);
                    tma_load_2d(C::NARROW && a ? &tmK1 : &tmK, &kv_full[ob], sV + ob * C::BIG + a * C::A_BIG, vcol + 64 * a,
                                row0 + kb * kRowsB);
                }
                const int n = group * per_head(kb);
                for (int j = 0; j < n; ++j, ++g) {
                    int hq, qs;
                    step_of(kb, kvh, j, hq, qs);
                    const int st = g % C::ST;
                    mbar_wait(&q_empty[st], ((g / C::ST) & 1) ^ 1);
                    // lse / delta of the step's valid queries, from the 16-byte aligned address at
                    // or below the first (bulk copies need it; the consumer skips `off` floats),
                    // rounded up to 16 bytes; stage floats past them are stale and masked
                    const int64_t li = (static_cast<int64_t>(b) * sh.H + hq) * sh.S + qs * kStepB;
                    const int off = static_cast<int>(li & 3);
                    const int nvalid = min(kStepB, sh.S - qs * kStepB);
                    const uint32_t lbytes = static_cast<uint32_t>((off + nvalid + 3) / 4 * 16);
                    mbar_expect_tx(&q_full[st], 2 * C::SMALL + 2 * lbytes);
                    for (int a = 0; a < C::ATOMS; ++a) {
                        tma_load_2d(C::NARROW && a ? &tmQ1 : &tmQ, &q_full[st], sQ + st * C::SMALL + a * C::A_SMALL,
                                    hq * HD + 64 * a, row0 + qs * kStepB);
                        tma_load_2d(C::NARROW && a ? &tmDO1 : &tmDO, &q_full[st], sDO + st * C::SMALL + a * C::A_SMALL,
                                    hq * HD + 64 * a, row0 + qs * kStepB);
                    }
                    bulk_load_b(sL + st * kLStride, lse + (li - off), lbytes, &q_full[st]);
                    bulk_load_b(sD + st * kLStride, delta + (li - off), lbytes, &q_full[st]);
                }
            }
        }
    } else if (warp == 1) {
        {  // the whole warp runs the loop; the elected lane issues
            const uint32_t leader = elect_one();  // ===== MMA issuer =====
            constexpr uint32_t ID_S = make_idesc(128, kStepB, false, false);
            constexpr uint32_t ID_D = make_idesc(128, HD, false, true);
            constexpr uint32_t ID_D64 = make_idesc(128, 64, false, true), ID_D16 = make_idesc(128, 16, false, true);
            uint64_t dk_, dv_;  // the tile's K / V descriptors (K-major, k step 0)
            uint32_t k_own = 0, v_own = 0;  // (their shared addresses: the tails)
            auto issue_s = [&](int gg) {
                const int st = gg % C::ST, bb = gg % NB;
                if (leader) trace_ev<TRACE>(0, gg);
                mbar_wait(&q_full[st], (gg / C::ST) & 1);
                if (SEP && gg >= 2) mbar_wait(&s_free[bb], ((gg - 2) >> 1) & 1);
                fence_after();
                if (leader) trace_ev<TRACE>(1, gg);
                const uint64_t dq = make_desc(smem_u32(sQ + st * C::SMALL), 16, 1024);
                const uint64_t ddo = make_desc(smem_u32(sDO + st * C::SMALL), 16, 1024);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t ob = (kk / 4) * C::A_BIG + (kk % 4) * 32, sb = (kk / 4) * C::A_SMALL + (kk % 4) * 32;
                    if (C::NARROW && kk == 4) {
                        umma_if(leader, tmem + 128 * bb, tail_desc(k_own + C::A_BIG),
                                tail_desc(smem_u32(sQ + st * C::SMALL + C::A_SMALL)), ID_S, 1);
                        umma_if(leader, tmem + 128 * bb + 64, tail_desc(v_own + C::A_BIG),
                                tail_desc(smem_u32(sDO + st * C::SMALL + C::A_SMALL)), ID_S, 1);
                    } else {
                        umma_if(leader, tmem + 128 * bb, dadd(dk_, ob), dadd(dq, sb), ID_S, kk > 0);
                        umma_if(leader, tmem + 128 * bb + 64, dadd(dv_, ob), dadd(ddo, sb), ID_S, kk > 0);
                    }
                }
                umma_commit_if(leader, &s_full[bb]);
            };
            auto issue_d = [&](int gg, bool first) {
                const int st = gg % C::ST, bb = gg % NB;
                if (leader) trace_ev<TRACE>(2, gg);
                mbar_wait(&p_full[bb], (gg / NB) & 1);
                fence_after();
                if (leader) trace_ev<TRACE>(3, gg);
                const uint64_t dq = make_desc(smem_u32(sQ + st * C::SMALL), C::A_SMALL, 1024);
                const uint64_t ddo = make_desc(smem_u32(sDO + st * C::SMALL), C::A_SMALL, 1024);
#pragma unroll
                for (int kk = 0; kk < kStepB / 16; ++kk) {
                    const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
                    if (C::NARROW) {  // dK / dV columns 0..63 from Q's / dO's atom, 64..79 from the tails
                        umma_ts_if(leader, tmem + T_ACC, tmem + ds_col(bb) + ts_col<SEP>(kk), dadd(dq, kk * 2048), ID_D64, acc);
                        umma_ts_if(leader, tmem + T_ACC + 64, tmem + ds_col(bb) + ts_col<SEP>(kk),
                                   tail_desc(smem_u32(sQ + st * C::SMALL + C::A_SMALL) + kk * 512), ID_D16, acc);
                        umma_ts_if(leader, tmem + T_ACC + HD, tmem + p_col(bb) + ts_col<SEP>(kk), dadd(ddo, kk * 2048), ID_D64,
                                   acc);
                        umma_ts_if(leader, tmem + T_ACC + HD + 64, tmem + p_col(bb) + ts_col<SEP>(kk),
                                   tail_desc(smem_u32(sDO + st * C::SMALL + C::A_SMALL) + kk * 512), ID_D16, acc);
                    } else {
                        umma_ts_if(leader, tmem + T_ACC, tmem + ds_col(bb) + ts_col<SEP>(kk), dadd(dq, kk * 2048), ID_D, acc);
                        umma_ts_if(leader, tmem + T_ACC + HD, tmem + p_col(bb) + ts_col<SEP>(kk), dadd(ddo, kk * 2048), ID_D,
                                   acc);
                    }
                }
                if (SEP) umma_commit_if(leader, &ds_free[bb]);
                umma_commit_if(leader, &q_empty[st]);
            };
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int kb, kvh, b;
                tile(t, kb, kvh, b);
                const int n = group * per_head(kb);
                const int ob = lt % C::OWN;
                mbar_wait(&kv_full[ob], (lt / C::OWN) & 1);
                k_own = smem_u32(sK + ob * C::BIG);
                v_own = smem_u32(sV + ob * C::BIG);
                dk_ = make_desc(k_own, 16, 1024);
                dv_ = make_desc(v_own, 16, 1024);
                for (int i = 0; i < NB && i < n; ++i) issue_s(g + i);
                mbar_wait(acc_empty, (lt & 1) ^ 1);  // the previous tile's dK / dV are read out
                fence_after();
                for (int j = 0; j < n; ++j) {
                    // separate P / dS: S / dP of step j + 2 as soon as step j's are loaded;
                    // written back over S / dP: only after the products that read them
                    if (SEP && j + 2 < n) issue_s(g + j + 2);
                    issue_d(g + j, j == 0);
                    if (!SEP && j + NB < n) issue_s(g + j + NB);  // (in order after the product)
                }
                umma_commit_if(leader, acc_full);
                umma_commit_if(leader, &kv_empty[ob]);
                g += n;
            }
        }
    } else if (warp >= 4) {
        // ===== elementwise: thread = key row; warpgroup wg takes the steps of parity wg (all 64
        // queries of each, in two 32-query halves), so the two warps of an SM sub-partition work
        // on different steps and overlap each other's TMEM / MUFU / barrier latencies =====
        const int q4 = warp & 3, wg = (warp - 4) >> 2;
        const int half = wg;  // (the tile's dK / dV readout below: wg 0 dK, wg 1 dV)
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        uint32_t vs[32], vp[32];
        int g = 0, lt = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
            int kb, kvh, b;
            tile(t, kb, kvh, b);
            const int key = kb * kRowsB + r;
            const int n = group * per_head(kb);
            const int qs0 = sh.causal ? 2 * kb : 0;
            int hq = kvh * group, qs = qs0;  // step j's query head and block (step_of, incrementally)
            for (int j = 0; j < n; ++j, ++g, (++qs == n_qs ? (qs = qs0, ++hq) : 0)) {
                if ((g & 1) != wg) continue;  // the other warpgroup's step
                const int st = g % C::ST, bb = g % NB;
                if (TRACE && q4 == 0 && lane == 0) trace_ev<TRACE>(4 + 8 * wg, g);
                if (SEP && g >= 2) mbar_wait(&ds_free[bb], ((g - 2) >> 1) & 1);  // step g - 2's products
                mbar_wait(&s_full[bb], (g / NB) & 1);                              // read this P / dS buffer
                fence_after();
                if (TRACE && q4 == 0 && lane == 0) trace_ev<TRACE>(5 + 8 * wg, g);
                // a step's lse / delta start on a 16-byte boundary unless the sequence length is
                // not a multiple of 4 (ViT's 257): two instantiations of the step body
                auto step_body = [&](auto aligned_tag) {
                    constexpr bool ALIGNED = decltype(aligned_tag)::value;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t pp[16], dd[16];
                        const uint32_t cs = tmem + lane_off + 128 * bb + 32 * h;
                        tmem_ld32_async(cs, vs);
                        tmem_ld32_async(cs + 64, vp);
                        // lse / delta of these 32 queries (landed with the step's Q tile, which the
                        // S MMA already waited for)
                        const int off = ALIGNED ? 0 : static_cast<int>(((static_cast<int64_t>(b) * sh.H + hq) * sh.S + qs * kStepB) & 3);
                        const float* Ls = sL + st * kLStride + off + 32 * h;
                        const float* Ds = sD + st * kLStride + off + 32 * h;
                        tmem_ld_wait(vs);
                        tmem_ld_wait(vp);
                        if (SEP && h == 1) {
                            fence_before();
                            mbar_arrive(&s_free[bb]);  // the MMAs of step g + 2 may overwrite S / dP now
                        }
                        const int q0 = qs * kStepB + 32 * h;  // first query of this half
                        // some query below some key, or past the sequence (stale lse / delta: zeroed)
                        const bool mask = (sh.causal && kb * kRowsB + kRowsB - 1 > q0) || q0 + 32 > sh.S;
                        const int qlo = sh.causal ? key : 0;  // valid queries: qlo <= q < S
#pragma unroll
                        for (int i4 = 0; i4 < 8; ++i4) {
                            float lv[4], dv[4];
                            if (ALIGNED) {  // 16-byte shared loads
                                const float4 l = reinterpret_cast<const float4*>(Ls)[i4], dl = reinterpret_cast<const float4*>(Ds)[i4];
                                lv[0] = l.x, lv[1] = l.y, lv[2] = l.z, lv[3] = l.w;
                                dv[0] = dl.x, dv[1] = dl.y, dv[2] = dl.z, dv[3] = dl.w;
                            } else {
#pragma unroll
                                for (int k = 0; k < 4; ++k) lv[k] = Ls[4 * i4 + k], dv[k] = Ds[4 * i4 + k];
                            }
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const int i = 2 * i4 + u;  // query pair (2 i, 2 i + 1)
                                const float2 x = ffma2(make_float2(__uint_as_float(vs[2 * i]), __uint_as_float(vs[2 * i + 1])),
                                                       make_float2(sh.scale_log2, sh.scale_log2),
                                                       make_float2(-lv[2 * u], -lv[2 * u + 1]));
                                float p0 = ex2_approx(x.x), p1 = ex2_approx(x.y);
                                const float2 dd2 = fmul2(make_float2(p0, p1),
                                                         fsub2(make_float2(__uint_as_float(vp[2 * i]), __uint_as_float(vp[2 * i + 1])),
                                                               make_float2(dv[2 * u], dv[2 * u + 1])));
                                float d0 = dd2.x, d1 = dd2.y;
                                if (mask) {
                                    const int qa = q0 + 2 * i;
                                    if (qa < qlo || qa >= sh.S) p0 = 0.0f, d0 = 0.0f;
                                    if (qa + 1 < qlo || qa + 1 >= sh.S) p1 = 0.0f, d1 = 0.0f;
                                }
                                pp[i] = pack_bf16(p0, p1);
                                dd[i] = pack_bf16(d0, d1);
                            }
                        }
                        // (written back over S / dP, half 0's P / dS columns are not half 1's S / dP
                        // columns: TMEM map in the header)
                        const uint32_t pofs = SEP ? 16 * h : 32 * h;
                        tmem_st16(tmem + lane_off + p_col(bb) + pofs, pp);
                        tmem_st16(tmem + lane_off + ds_col(bb) + pofs, dd);
                    }
                };
                if ((sh.S & 3) == 0) step_body(std::true_type{});
                else step_body(std::false_type{});
                tmem_st_wait();
                fence_before();
                mbar_arrive(&p_full[bb]);
                if (TRACE && q4 == 0 && lane == 0) trace_ev<TRACE>(6 + 8 * wg, g);
            }
            // the tile's dK (half 0, with the softmax scale) or dV (half 1) out of TMEM
            mbar_wait(acc_full, lt & 1);
            fence_after();
            __nv_bfloat16* row = dqkv + (static_cast<int64_t>(b) * sh.S + key) * sh.ld +
                                 (half == 0 ? (sh.H + kvh) * HD : (sh.H + sh.Hkv + kvh) * HD);
            const int col0 = half == 0 ? (sh.H + kvh) * HD : (sh.H + sh.Hkv + kvh) * HD;
            const int64_t tokk = static_cast<int64_t>(b) * sh.S + key;
            const bool warp_in = kb * kRowsB + q4 * 32 < sh.S;  // (as in the dQ pass)
            float* cs = csum && warp_in ? csum + (tokk - r % 32) / 32 * sh.ld + col0 : nullptr;
            acc_row_out<HD>(tmem + lane_off + T_ACC + half * HD, row, half == 0 ? sh.scale : 1.0f, key < sh.S, cs, lane);
            fence_before();
            mbar_arrive(acc_empty);
        }
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int HD>
cudaError_t launch_bwd2(const AttnProblem& a, cudaStream_t st) {
    using C = BCfg<HD>;
    constexpr bool SEP = C::SEP_DKDV;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_bwd_dq2_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM_DQ);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attn_bwd_dkdv2_kernel<HD, SEP, C::NB_DKDV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::SMEM_DKDV);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int ld = (a.n_heads + 2 * a.n_kv_heads) * a.head_dim;
    const int ldo = a.n_heads * a.head_dim;
    const uint64_t T = static_cast<uint64_t>(a.tokens);
    CUtensorMap t128, t64, do128, do64;
    if (!make_map(&t128, a.qkv, ld, T, ld, 64, kRowsB, false, false) ||
        !make_map(&t64, a.qkv, ld, T, ld, 64, kStepB, false, false) ||
        !make_map(&do128, a.dout, ldo, T, ldo, 64, kRowsB, false, false) ||
        !make_map(&do64, a.dout, ldo, T, ldo, 64, kStepB, false, false))
        return cudaErrorInvalidValue;
    CUtensorMap n128 = t128, n64 = t64, ndo128 = do128, ndo64 = do64;  // head_dim 80: the 16-column tails
    if (C::NARROW && (!make_map_sw32(&n128, a.qkv, ld, T, ld, 16, kRowsB) || !make_map_sw32(&n64, a.qkv, ld, T, ld, 16, kStepB) ||
                      !make_map_sw32(&ndo128, a.dout, ldo, T, ldo, 16, kRowsB) ||
                      !make_map_sw32(&ndo64, a.dout, ldo, T, ldo, 16, kStepB)))
        return cudaErrorInvalidValue;
    BShape sh;
    sh.S = a.seq_len;
    sh.H = a.n_heads;
    sh.Hkv = a.n_kv_heads;
    sh.ld = ld;
    sh.ldo = ldo;
    sh.causal = a.causal;
    sh.chunk = attention_causal_chunk(a);
    sh.scale = 1.0f / sqrtf(static_cast<float>(a.head_dim));
    sh.scale_log2 = 1.4426950408889634f * sh.scale;
    const int n_seq = static_cast<int>(a.tokens / a.seq_len);
    const int n_blk = (a.seq_len + kRowsB - 1) / kRowsB;
    const int q_tiles = n_blk * a.n_heads * n_seq;
    const int kv_tiles = n_blk * a.n_kv_heads * n_seq;
    auto* dq = static_cast<__nv_bfloat16*>(a.dqkv);
    float* cs = attention_colsum_fused(a) ? a.colsum_part : nullptr;
    attn_bwd_dq2_kernel<HD><<<q_tiles < num_sms() ? q_tiles : num_sms(), kThreadsB, C::SMEM_DQ, st>>>(
        t128, do128, t64, n128, ndo128, n64, static_cast<const __nv_bfloat16*>(a.o), static_cast<const __nv_bfloat16*>(a.dout), a.lse,
        a.delta, dq, sh, n_seq, cs);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (g_attn_trace) {  // debug timeline (tools/attn_trace.py)
        static bool configured_t = false;
        if (!configured_t) {
            cudaFuncSetAttribute(attn_bwd_dkdv2_kernel<HD, SEP, C::NB_DKDV, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_DKDV);
            configured_t = true;
        }
        const unsigned int zero = 0;
        cudaMemcpyToSymbolAsync(g_bwd_trace_n, &zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st);
        attn_bwd_dkdv2_kernel<HD, SEP, C::NB_DKDV, true><<<kv_tiles < num_sms() ? kv_tiles : num_sms(), kThreadsB,
                                                          C::SMEM_DKDV, st>>>(t128, t64, do64, n128, n64, ndo64, a.lse, a.delta, dq, sh, n_seq, cs);
        return cudaGetLastError();
    }
    attn_bwd_dkdv2_kernel<HD, SEP, C::NB_DKDV><<<kv_tiles < num_sms() ? kv_tiles : num_sms(), kThreadsB, C::SMEM_DKDV, st>>>(
        t128, t64, do64, n128, n64, ndo64, a.lse, a.delta, dq, sh, n_seq, cs);
    return cudaGetLastError();
}
}  // namespace

// The backward for head_dim 64 / 80 / 128, any sequence length; delta is formed inside (no
// separate kernel). cudaErrorNotSupported for other head dims.
int g_attn_trace = 0;
int attn_trace_read(unsigned long long* out, int cap) {
    unsigned int n = 0;
    if (cudaMemcpyFromSymbol(&n, g_bwd_trace_n, sizeof(n)) != cudaSuccess) return -1;
    const int m = static_cast<int>(n < static_cast<unsigned>(kTraceCap) ? n : kTraceCap);
    const int k = m < cap ? m : cap;
    if (k > 0 && cudaMemcpyFromSymbol(out, g_bwd_trace, k * sizeof(unsigned long long)) != cudaSuccess) return -1;
    return k;
}

// ViT's ragged 257-token sequences keep the separate colsum_total: the passes' epilogues with
// per-sequence 32-row groups (and 8-column tails for head_dim 80) were measured there, and the
// column sums on each short tile's critical path cost dQ + dK/dV 150 us per layer against the
// 114 us colsum they replace (profiles/r02_c4_vit_launches.txt is the kept build)
bool attention_colsum_fused(const AttnProblem& a) {
    return a.colsum_part && (a.head_dim == 64 || a.head_dim == 128) && a.seq_len % 32 == 0 && g_attn_bwd_kind == 0;
}

cudaError_t attention_backward_tc2(const AttnProblem& a, cudaStream_t st) {
    if (a.head_dim == 64) return launch_bwd2<64>(a, st);
    if (a.head_dim == 80) return launch_bwd2<80>(a, st);
    if (a.head_dim == 128) return launch_bwd2<128>(a, st);
    return cudaErrorNotSupported;
}

}  // namespace sp

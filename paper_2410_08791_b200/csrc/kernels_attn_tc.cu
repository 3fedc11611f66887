// kernels_attn_tc.cu — tcgen05 flash-attention forward (sm_100a), head_dim 64 and 128.
//
// Persistent: one CTA per SM walks work tiles of 128 queries of one (sequence, head), longest
// first, so TMEM allocation, barrier setup and the next tile's Q / K / V loads overlap the
// current tile's compute. 256 threads:
//   warp 0      TMA producer: Q once, then K_j / V_j tiles of 128 keys into a 2-stage ring
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T (M 128, N 128, K hd) into TMEM S[j%2],
//               then, once the softmax has written P_j, O_j = P_j V_j (M 128, N hd, K 128)
//               into TMEM O[j%2]; tcgen05.commit frees smem stages and signals TMEM buffers
//   warp 2      TMEM allocator (512 columns: S[2] x 128 + O[2] x hd)
//   warps 4..7  softmax: thread = query row = TMEM lane; row max / exp2 / row sum of S_j from
//               TMEM, P_j (bf16) into swizzled smem as the PV MMA's K-major A operand, and the
//               running output acc = acc * exp2(m_{j-1} - m_j) + O_j in registers, one block
//               behind, so O_j's MMA overlaps the softmax of S_{j+1}
// Operand layouts are the GEMM's (kernels_tc.cu): Q and K K-major (rows of hd, 128B swizzle),
// V N-major (B[k = key][n = d]), P K-major. Same inputs, outputs and lse convention (log2 units
// of the scaled scores) as the mma.sync kernel in kernels_attn.cu, so the backward is shared.
// Every output element is one thread's fixed-order reduction: deterministic.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace sp {
namespace {
using namespace tc;

constexpr int kQ = 128;      // queries per CTA
constexpr int kKV = 128;     // keys per block
constexpr int kThreadsTc = 256;
constexpr int kStages = 2;   // K/V ring

template <int HD>
struct AttnCfg {
    static constexpr int ATOMS = HD / 64;                 // 64-element (128-byte) K atoms of a row
    static constexpr int Q_BYTES = kQ * HD * 2;
    static constexpr int KV_BYTES = kKV * HD * 2;         // one K (or V) tile
    static constexpr int P_BYTES = kQ * kKV * 2;
    // head_dim 128: one Q buffer (reloaded per tile) so P can be double-buffered (every block)
    static constexpr int Q_BUFS = HD <= 64 ? 2 : 1;
    static constexpr int P_BUFS = 2;
    static constexpr int SMEM = Q_BUFS * Q_BYTES + 2 * kStages * KV_BYTES + P_BUFS * P_BYTES + 1024 + 256;
    static constexpr int O_COL0 = 2 * kKV;                // TMEM: S[0], S[1], then O[0], O[1]
};

struct TcShape {
    int S, H, Hkv, ld, ldo, causal, chunk;  // chunk: causal work order (causal_chunked)
    float scale_log2;
};

__device__ __forceinline__ float ex2_fast(float x) {  // MUFU.EX2; ex2(-inf) = +0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    tmem_ld32_async(taddr, r);
    tmem_ld_wait(r);
}

// Work tile t of a persistent CTA: (query block, head, sequence), longest tiles first (causal
// blocks near the end of a sequence attend the most keys). (Measured against (sequence, head)-
// major order for K / V reuse in L2: 209 vs 232 us at GPT-2 XL, tools/attn_probe.py.)
struct TileOf {
    int qb, h, b;
};
// Without a causal mask every tile is equally long and the query blocks of one (sequence, head)
// go innermost instead: they run side by side, so K / V come from DRAM once (qb-outermost order
// at ViT-H's 4096 (sequence, head) pairs cycled 540 MB of K / V through the 126 MB L2 between
// reuses: 52% hit rate, the forward bound by the DRAM share of each SM).
__device__ __forceinline__ TileOf tile_of(int t, const TcShape& sh, int n_qb, int n_seq) {
    const int per = sh.H * n_seq;
    TileOf o;
    if (sh.causal) {
        int pair;
        causal_chunked(t, per, n_qb, true, sh.chunk, o.qb, pair);
        o.h = pair % sh.H;
        o.b = pair / sh.H;
    } else {
        o.qb = t % n_qb;
        const int rest = t / n_qb;
        o.h = rest % sh.H;
        o.b = rest / sh.H;
    }
    return o;
}

template <int HD>
__global__ void __launch_bounds__(kThreadsTc, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                       __nv_bfloat16* __restrict__ o, float* __restrict__ lse, TcShape sh, int n_seq) {
    using C = AttnCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                                // Q_BUFS tiles (the next tile's Q loads early)
    uint8_t* sK = sQ + C::Q_BUFS * C::Q_BYTES;         // kStages tiles
    uint8_t* sV = sK + kStages * C::KV_BYTES;          // kStages tiles
    uint8_t* sP = sV + kStages * C::KV_BYTES;          // P_BUFS tiles
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BUFS * C::P_BYTES);
    uint64_t* q_full = bars;                 // 2
    uint64_t* q_empty = bars + 2;            // 2
    uint64_t* kv_full = bars + 4;            // kStages
    uint64_t* kv_empty = kv_full + kStages;  // kStages
    uint64_t* s_full = kv_empty + kStages;   // 2
    uint64_t* s_empty = s_full + 2;          // 2
    uint64_t* p_full = s_empty + 2;          // 2 (indexed by P buffer)
    uint64_t* p_empty = p_full + 2;          // 2
    uint64_t* o_full = p_empty + 2;          // 2
    uint64_t* o_empty = o_full + 2;          // 2
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_qb = (sh.S + kQ - 1) / kQ;
    const int n_tiles = n_qb * sh.H * n_seq;
    const int n_kb_total = (sh.S + kKV - 1) / kKV;
    auto blocks_of = [&](int qb) { return sh.causal ? min(n_kb_total, (qb * kQ + kQ - 1) / kKV + 1) : n_kb_total; };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmQK);
        prefetch_tmap(&tmV);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 128);
            mbar_init(&p_full[i], 128);
            mbar_init(&p_empty[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 128);
        }
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
    // Every role walks the same (tile, key block) sequence; g counts key blocks over the CTA's
    // tiles and lt its tiles, so buffer indices and mbarrier phases stay in step across tiles.

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                const TileOf w = tile_of(t, sh, n_qb, n_seq);
                const int kvh = w.h / (sh.H / sh.Hkv);
                const int row0 = w.b * sh.S;
                const int qcol = w.h * HD, kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
                const int qbuf = lt % C::Q_BUFS;
                mbar_wait(&q_empty[qbuf], ((lt / C::Q_BUFS) & 1) ^ 1);
                mbar_expect_tx(&q_full[qbuf], C::Q_BYTES);
                for (int a = 0; a < C::ATOMS; ++a)
                    tma_load_2d(&tmQK, &q_full[qbuf], sQ + qbuf * C::Q_BYTES + a * kQ * 128, qcol + 64 * a,
                                row0 + w.qb * kQ);
                const int n_kb = blocks_of(w.qb);
                for (int j = 0; j < n_kb; ++j, ++g) {
                    const int st = g % kStages;
                    mbar_wait(&kv_empty[st], ((g / kStages) & 1) ^ 1);
                    mbar_expect_tx(&kv_full[st], 2 * C::KV_BYTES);
                    const int k0 = row0 + j * kKV;
                    uint8_t* k = sK + st * C::KV_BYTES;
                    uint8_t* v = sV + st * C::KV_BYTES;
                    for (int a = 0; a < C::ATOMS; ++a) tma_load_2d(&tmQK, &kv_full[st], k + a * kKV * 128, kcol + 64 * a, k0);
                    // V as N-major B: per 64-key k-block, per 64-wide d atom, a {64 d, 64 keys} box
                    for (int kb = 0; kb < 2; ++kb)
                        for (int a = 0; a < C::ATOMS; ++a)
                            tma_load_2d(&tmV, &kv_full[st], v + (kb * C::ATOMS + a) * 8192, vcol + 64 * a, k0 + 64 * kb);
                }
            }
        }
    } else if (warp == 1) {
        {  // the whole warp runs the loop; the elected lane issues
            const uint32_t leader = elect_one();
            // ===== MMA issuer =====
            constexpr uint32_t IDESC_S = make_idesc(kQ, kKV, false, false);
            constexpr uint32_t IDESC_O = make_idesc(kQ, HD, false, true);
            auto issue_s = [&](int g, uint32_t q_base) {
                const int st = g % kStages, sb = g & 1;
                mbar_wait(&kv_full[st], (g / kStages) & 1);
                mbar_wait(&s_empty[sb], ((g >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t k_base = smem_u32(sK + st * C::KV_BYTES);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const int a = kk / 4, w = kk % 4;  // atom, 32-byte step within the atom
                    const uint64_t ad = make_desc(q_base + a * kQ * 128 + w * 32, 16, 1024);
                    const uint64_t bd = make_desc(k_base + a * kKV * 128 + w * 32, 16, 1024);
                    umma_if(leader, tmem + sb * kKV, ad, bd, IDESC_S, kk > 0 ? 1u : 0u);
                }
                umma_commit_if(leader, &s_full[sb]);
            };
            auto issue_o = [&](int g) {
                const int st = g % kStages, ob = g & 1, pb = g % C::P_BUFS;
                mbar_wait(&p_full[pb], (g / C::P_BUFS) & 1);
                mbar_wait(&o_empty[ob], ((g >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t p_base = smem_u32(sP + pb * C::P_BYTES);
                const uint32_t v_base = smem_u32(sV + st * C::KV_BYTES);
#pragma unroll
                for (int kk = 0; kk < kKV / 16; ++kk) {
                    const int a = kk / 4, w = kk % 4;
                    const uint64_t ad = make_desc(p_base + a * kQ * 128 + w * 32, 16, 1024);
                    // N-major V: k-block a (64 keys), 16-key step w; atoms of 64 d at 8 KB stride
                    const uint64_t bd = make_desc(v_base + a * C::ATOMS * 8192 + w * 16 * 128, 8192, 1024);
                    umma_if(leader, tmem + C::O_COL0 + ob * HD, ad, bd, IDESC_O, kk > 0 ? 1u : 0u);
                }
                umma_commit_if(leader, &o_full[ob]);
                umma_commit_if(leader, &p_empty[pb]);
                umma_commit_if(leader, &kv_empty[st]);  // both MMAs of block g are done with K_g, V_g
            };
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                const TileOf w = tile_of(t, sh, n_qb, n_seq);
                const int n_kb = blocks_of(w.qb);
                const int qbuf = lt % C::Q_BUFS;
                mbar_wait(&q_full[qbuf], (lt / C::Q_BUFS) & 1);
                fence_after();
                const uint32_t q_base = smem_u32(sQ + qbuf * C::Q_BYTES);
                issue_s(g, q_base);
                for (int j = 0; j < n_kb; ++j) {
                    if (j + 1 < n_kb) issue_s(g + j + 1, q_base);
                    if (j + 1 == n_kb) umma_commit_if(leader, &q_empty[qbuf]);  // every S MMA of the tile issued
                    issue_o(g + j);
                }
                g += n_kb;
            }
        }
    } else if (warp >= 4) {
        // ===== softmax: one query row per thread =====
        const int q = warp & 3;
        const int r = q * 32 + lane;   // row in the tile = TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        uint32_t v[32], v2[32];
        float acc[HD];
        int g = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            const TileOf w = tile_of(t, sh, n_qb, n_seq);
            const int n_kb = blocks_of(w.qb);
            const int q0 = w.qb * kQ;
            const int qi = q0 + r;  // query index in the sequence
#pragma unroll
            for (int i = 0; i < HD; ++i) acc[i] = 0.0f;
            float m_run = -INFINITY, l_run = 0.0f, corr_prev = 1.0f;
            auto accumulate_o = [&](int gg, float corr) {
                const int ob = gg & 1;
                mbar_wait(&o_full[ob], (gg >> 1) & 1);
                fence_after();
#pragma unroll
                for (int c = 0; c < HD / 32; ++c) {
                    tmem_ld32(tmem + lane_off + C::O_COL0 + ob * HD + c * 32, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[c * 32 + i] = fmaf(acc[c * 32 + i], corr, __uint_as_float(v[i]));
                }
                fence_before();
                mbar_arrive(&o_empty[ob]);
            };
            for (int j = 0; j < n_kb; ++j, ++g) {
                const int sb = g & 1, pb = g % C::P_BUFS;
                const int k0 = j * kKV;
                mbar_wait(&s_full[sb], (g >> 1) & 1);
                fence_after();
                const uint32_t s_addr = tmem + lane_off + sb * kKV;
                // masking is needed only on the diagonal block (causal) and a ragged last block
                const bool need_mask = (sh.causal && k0 + kKV - 1 > q0) || k0 + kKV > sh.S;
                const int lim = need_mask ? min(sh.S, sh.causal ? qi + 1 : sh.S) - k0 : kKV;  // valid keys
                // pass 1: row max of the raw scores (the scale is positive), two loads per wait
                float mraw = -INFINITY;
                if (HD <= 64) {
#pragma unroll
                    for (int c = 0; c < kKV / 32; c += 2) {
                        tmem_ld32_async(s_addr + c * 32, v);
                        tmem_ld32_async(s_addr + (c + 1) * 32, v2);
                        tmem_ld_wait(v);
                        tmem_ld_wait(v2);
                        if (need_mask) {
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                const float x0 = c * 32 + i < lim ? __uint_as_float(v[i]) : -INFINITY;
                                const float x1 = (c + 1) * 32 + i < lim ? __uint_as_float(v2[i]) : -INFINITY;
                                mraw = fmaxf(mraw, fmaxf(x0, x1));
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                mraw = fmaxf(mraw, fmaxf(__uint_as_float(v[i]), __uint_as_float(v2[i])));
                        }
                    }
                } else {  // head_dim 128: acc[128] is live; one 32-column buffer
#pragma unroll
                    for (int c = 0; c < kKV / 32; ++c) {
                        tmem_ld32(s_addr + c * 32, v);
                        if (need_mask) {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                mraw = fmaxf(mraw, c * 32 + i < lim ? __uint_as_float(v[i]) : -INFINITY);
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; i += 2)
                                mraw = fmaxf(mraw, fmaxf(__uint_as_float(v[i]), __uint_as_float(v[i + 1])));
                        }
                    }
                }
                const float mx = fmaxf(m_run, mraw * sh.scale_log2);
                const float base = mx == -INFINITY ? 0.0f : mx;
                const float corr = ex2_fast(m_run - base);
                m_run = mx;
                // pass 2: P = exp2(s * scale - m) (one FFMA + one MUFU ex2 each), row sum, bf16
                // pairs into the K-major swizzled P tile (row r)
                if (g >= C::P_BUFS) mbar_wait(&p_empty[pb], ((g / C::P_BUFS) & 1) ^ 1);
                uint8_t* prow = sP + pb * C::P_BYTES + r * 128;
                float rs0 = 0.0f, rs1 = 0.0f;
#pragma unroll
                for (int c = 0; c < kKV / 32; ++c) {
                    tmem_ld32_async(s_addr + c * 32, v);
                    tmem_ld_wait(v);
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        float p0 = ex2_fast(fmaf(__uint_as_float(v[2 * i]), sh.scale_log2, -base));
                        float p1 = ex2_fast(fmaf(__uint_as_float(v[2 * i + 1]), sh.scale_log2, -base));
                        if (need_mask) {
                            if (c * 32 + 2 * i >= lim) p0 = 0.0f;
                            if (c * 32 + 2 * i + 1 >= lim) p1 = 0.0f;
                        }
                        rs0 += p0;
                        rs1 += p1;
                        pk[i] = pack_bf16(p0, p1);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {  // 32 keys = 4 16-byte chunks of the 128-byte row
                        const int chunk = (c % 2) * 4 + u;
                        uint8_t* dst = prow + (c / 2) * kQ * 128 + ((chunk ^ (r & 7)) << 4);
                        *reinterpret_cast<uint4*>(dst) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
                    }
                }
                l_run = l_run * corr + (rs0 + rs1);
                fence_before();
                mbar_arrive(&s_empty[sb]);  // S read: the MMA may overwrite the buffer
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the tensor core
                mbar_arrive(&p_full[pb]);
                if (j > 0) accumulate_o(g - 1, corr_prev);
                corr_prev = corr;
            }
            if (n_kb > 0) accumulate_o(g - 1, corr_prev);
            if (qi < sh.S) {
                const float inv = l_run > 0.0f ? 1.0f / l_run : 0.0f;
                __nv_bfloat16* orow = o + static_cast<int64_t>(w.b * sh.S + qi) * sh.ldo + w.h * HD;
#pragma unroll
                for (int c = 0; c < HD / 8; ++c) {
                    uint4 u4;
                    u4.x = pack_bf16(acc[8 * c + 0] * inv, acc[8 * c + 1] * inv);
                    u4.y = pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv);
                    u4.z = pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv);
                    u4.w = pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv);
                    reinterpret_cast<uint4*>(orow)[c] = u4;
                }
                lse[(static_cast<int64_t>(w.b) * sh.H + w.h) * sh.S + qi] =
                    l_run > 0.0f ? m_run + log2f(l_run) : INFINITY;
            }
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

// ---------------------------------------------------------------------------------------
// forward v2: TWO softmax warps per TMEM lane quarter (warps 4..11; warp 4 + 4 h takes keys
// [64 h, 64 h + 64) of each 128-key block), P written back over its own S columns in TMEM and
// fed to the PV MMA as the A operand from TMEM (no shared-memory P tile). A row's max is the
// two halves' maxima exchanged through shared memory (one 64-thread named barrier per block);
// the row sums stay per half until the end of the tile. Each half accumulates its HD / 2 output
// columns in registers, one block behind, as the 4-warp kernel does. 384 threads; TMEM: S / P
// double-buffered at 128 b, O[b] at 256 + HD b.
// ---------------------------------------------------------------------------------------
constexpr int kThreadsF2 = 384;

template <int HD>
struct Fwd2Cfg {
    // head_dim 80 (ViT-H/14) takes two 64-column atoms: the MMAs read only the first HD
    // columns (5 K steps of 16 for QK^T, N = 80 for PV); the rest of the second atom (the next
    // head's columns, or TMA zero fill past the row) is loaded but never multiplied
    static constexpr int ATOMS = (HD + 63) / 64;
    // head_dim 80: the 16 columns past the first atom are loaded alone, as a 32-byte-swizzled
    // [rows][16] tile (TMA box {16, rows}), instead of a whole second 64-column atom: 160 instead
    // of 256 bytes per row of Q / K / V, and the ring gets a third stage in the saved space
    static constexpr bool NARROW = HD % 64 == 16;
    static constexpr int Q_BYTES = NARROW ? kQ * (128 + 32) : kQ * ATOMS * 64 * 2;
    static constexpr int KV_BYTES = NARROW ? kKV * (128 + 32) : kKV * ATOMS * 64 * 2;
    static constexpr int ST = (HD <= 64 || NARROW) ? 3 : 2;  // K / V ring
    static constexpr int SMEM = 2 * Q_BYTES + 2 * ST * KV_BYTES + 1024 + 512;  // (+ 3 KB static exchange)
    static constexpr uint32_t T_O = 256;
};

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    tmem_st16(taddr, *reinterpret_cast<const uint32_t(*)[16]>(r));
    tmem_st16(taddr + 16, *reinterpret_cast<const uint32_t(*)[16]>(r + 16));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
// This lane's NC columns of O (TMEM, from `taddr`) times f, written back (the lazy rescale)
template <int NC>
__device__ __forceinline__ void tmem_scale(uint32_t taddr, float f) {
    if (NC % 32 == 0) {
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < NC / 32; ++c) {
            tmem_ld32(taddr + c * 32, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
            tmem_st32(taddr + c * 32, v);
        }
    } else {
        uint32_t v[8];
#pragma unroll
        for (int c = 0; c < NC / 8; ++c) {
            tmem_ld8(taddr + c * 8, v);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
            tmem_st8(taddr + c * 8, v);
        }
    }
    tmem_st_wait();
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// LAZY (v3): O accumulates in TMEM across the tile's key blocks (one accumulator per tile
// parity) and is rescaled in place only when a row's max grows by more than 2^8 over the
// reference max its P values were computed with (P <= 256 otherwise: exact in fp32, fine in
// bf16); the softmax warps read O once per tile instead of once per block.
template <int HD, bool LAZY>
__global__ void __launch_bounds__(kThreadsF2, 1)
    attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmQK1, const __grid_constant__ CUtensorMap tmV1,
                        __nv_bfloat16* __restrict__ o, float* __restrict__ lse, TcShape sh, int n_seq) {
    using C = Fwd2Cfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                        // 2 tiles (the next tile's Q loads early)
    uint8_t* sK = sQ + 2 * C::Q_BYTES;         // ST tiles
    uint8_t* sV = sK + C::ST * C::KV_BYTES;    // ST tiles
    __shared__ float xmax[2 * 2 * 128];  // row-max exchange [block parity][half][row] (static:
    __shared__ float xl[2 * 128];        // plain shared loads) and row-sum exchange [half][row]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::ST * C::KV_BYTES);
    uint64_t* q_full = bars;                   // 2
    uint64_t* q_empty = bars + 2;              // 2
    uint64_t* kv_full = bars + 4;              // ST
    uint64_t* kv_empty = kv_full + C::ST;      // ST
    uint64_t* s_full = kv_empty + C::ST;       // 2: S[b] computed
    uint64_t* p_full = s_full + 2;             // 2: P[b] written (256 arrivals)
    uint64_t* pv_done = p_full + 2;            // 2: the PV MMAs have read P[b] (S[b] reusable)
    uint64_t* o_full = pv_done + 2;            // 2
    uint64_t* o_empty = o_full + 2;            // 2 (256 arrivals)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_qb = (sh.S + kQ - 1) / kQ;
    const int n_tiles = n_qb * sh.H * n_seq;
    const int n_kb_total = (sh.S + kKV - 1) / kKV;
    auto blocks_of = [&](int qb) { return sh.causal ? min(n_kb_total, (qb * kQ + kQ - 1) / kKV + 1) : n_kb_total; };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmQK);
        prefetch_tmap(&tmV);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 256);
            mbar_init(&pv_done[i], 1);
            mbar_init(&o_full[i], 1);
            mbar_init(&o_empty[i], 256);
        }
        for (int i = 0; i < C::ST; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
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
        if (lane == 0) {
            // ===== TMA producer =====
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                const TileOf w = tile_of(t, sh, n_qb, n_seq);
                const int kvh = w.h / (sh.H / sh.Hkv);
                const int row0 = w.b * sh.S;
                const int qcol = w.h * HD, kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
                const int qbuf = lt & 1;
                mbar_wait(&q_empty[qbuf], ((lt >> 1) & 1) ^ 1);
                mbar_expect_tx(&q_full[qbuf], C::Q_BYTES);
                if (C::NARROW) {
                    tma_load_2d(&tmQK, &q_full[qbuf], sQ + qbuf * C::Q_BYTES, qcol, row0 + w.qb * kQ);
                    tma_load_2d(&tmQK1, &q_full[qbuf], sQ + qbuf * C::Q_BYTES + kQ * 128, qcol + 64, row0 + w.qb * kQ);
                } else {
                    for (int a = 0; a < C::ATOMS; ++a)
                        tma_load_2d(&tmQK, &q_full[qbuf], sQ + qbuf * C::Q_BYTES + a * kQ * 128, qcol + 64 * a,
                                    row0 + w.qb * kQ);
                }
                const int n_kb = blocks_of(w.qb);
                for (int j = 0; j < n_kb; ++j, ++g) {
                    const int st = g % C::ST;
                    mbar_wait(&kv_empty[st], ((g / C::ST) & 1) ^ 1);
                    mbar_expect_tx(&kv_full[st], 2 * C::KV_BYTES);
                    const int k0 = row0 + j * kKV;
                    uint8_t* k = sK + st * C::KV_BYTES;
                    uint8_t* v = sV + st * C::KV_BYTES;
                    if (C::NARROW) {  // K: [128][64] + [128][16]; V: [2][64][64] + [2][64][16]
                        tma_load_2d(&tmQK, &kv_full[st], k, kcol, k0);
                        tma_load_2d(&tmQK1, &kv_full[st], k + kKV * 128, kcol + 64, k0);
                        for (int kb = 0; kb < 2; ++kb) {
                            tma_load_2d(&tmV, &kv_full[st], v + kb * 8192, vcol, k0 + 64 * kb);
                            tma_load_2d(&tmV1, &kv_full[st], v + 16384 + kb * 2048, vcol + 64, k0 + 64 * kb);
                        }
                    } else {
                        for (int a = 0; a < C::ATOMS; ++a) tma_load_2d(&tmQK, &kv_full[st], k + a * kKV * 128, kcol + 64 * a, k0);
                        for (int kb = 0; kb < 2; ++kb)
                            for (int a = 0; a < C::ATOMS; ++a)
                                tma_load_2d(&tmV, &kv_full[st], v + (kb * C::ATOMS + a) * 8192, vcol + 64 * a, k0 + 64 * kb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        {  // the whole warp runs the loop; the elected lane issues
            const uint32_t leader = elect_one();
            // ===== MMA issuer =====
            constexpr uint32_t IDESC_S = make_idesc(kQ, kKV, false, false);
            constexpr uint32_t IDESC_O = make_idesc(kQ, HD, false, true);
            constexpr uint32_t IDESC_O64 = make_idesc(kQ, 64, false, true), IDESC_O16 = make_idesc(kQ, 16, false, true);
            // nk: the block's keys inside the sequence; a ragged last block (ViT's 257th key)
            // multiplies only ceil(nk / 16) * 16 of them (the softmax masks the rest anyway)
            auto issue_s = [&](int g, uint32_t q_base, int nk) {
                const int st = g % C::ST, sb = g & 1;
                mbar_wait(&kv_full[st], (g / C::ST) & 1);
                if (g >= 2) mbar_wait(&pv_done[sb], ((g - 2) >> 1) & 1);
                fence_after();
                const uint32_t k_base = smem_u32(sK + st * C::KV_BYTES);
                const uint32_t idesc_s = nk >= kKV ? IDESC_S : make_idesc(kQ, (nk + 15) / 16 * 16, false, false);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const int a = kk / 4, w = kk % 4;
                    // (NARROW: columns 64..79 are the 32B-swizzled [rows][16] tiles, 8-row groups 256 B apart)
                    const bool tail = C::NARROW && a == 1;
                    const uint64_t ad = tail ? make_desc(q_base + kQ * 128, 16, 256, 6)
                                             : make_desc(q_base + a * kQ * 128 + w * 32, 16, 1024);
                    const uint64_t bd = tail ? make_desc(k_base + kKV * 128, 16, 256, 6)
                                             : make_desc(k_base + a * kKV * 128 + w * 32, 16, 1024);
                    umma_if(leader, tmem + sb * 128, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
                }
                umma_commit_if(leader, &s_full[sb]);
            };
            auto issue_o = [&](int g, int j, int n_kb, int lt, int nk) {
                const int st = g % C::ST, sb = g & 1;
                const int ob = LAZY ? (lt & 1) : sb;  // LAZY: one O per tile parity
                mbar_wait(&p_full[sb], (g >> 1) & 1);
                if (!LAZY) mbar_wait(&o_empty[ob], ((g >> 1) & 1) ^ 1);
                else if (j == 0) mbar_wait(&o_empty[ob], ((lt >> 1) & 1) ^ 1);  // tile lt - 2's O read out
                fence_after();
                const uint32_t v_base = smem_u32(sV + st * C::KV_BYTES);
#pragma unroll
                for (int kk = 0; kk < kKV / 16; ++kk) {
                    // P of keys 16 kk .. 16 kk + 15: half kk / 4 wrote its 64 keys as 32 packed
                    // columns at 128 sb + 64 half
                    if (16 * kk >= nk) continue;  // keys past the sequence (P = 0 there)
                    const uint32_t pcol = static_cast<uint32_t>(sb * 128 + (kk / 4) * 64 + (kk % 4) * 8);
                    const uint32_t acc = (kk > 0 || (LAZY && j > 0)) ? 1u : 0u;
                    if (C::NARROW) {
                        // O columns 0..63 from V's 128B-swizzled atom, 64..79 from its [64][16]
                        // 32B-swizzled tail (MN-major, one 16-column atom, 8-key groups 256 B apart)
                        const uint64_t bd0 = make_desc(v_base + (kk / 4) * 8192 + (kk % 4) * 16 * 128, 8192, 1024);
                        const uint64_t bd1 = make_desc(v_base + 16384 + (kk / 4) * 2048 + (kk % 4) * 16 * 32, 256, 256, 6);
                        umma_ts_if(leader, tmem + C::T_O + ob * HD, tmem + pcol, bd0, IDESC_O64, acc);
                        umma_ts_if(leader, tmem + C::T_O + ob * HD + 64, tmem + pcol, bd1, IDESC_O16, acc);
                    } else {
                        const uint64_t bd = make_desc(v_base + (kk / 4) * C::ATOMS * 8192 + (kk % 4) * 16 * 128, 8192, 1024);
                        umma_ts_if(leader, tmem + C::T_O + ob * HD, tmem + pcol, bd, IDESC_O, acc);
                    }
                }
                if (!LAZY || j + 1 == n_kb) umma_commit_if(leader, &o_full[ob]);
                umma_commit_if(leader, &pv_done[sb]);
                umma_commit_if(leader, &kv_empty[st]);
            };
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                const TileOf w = tile_of(t, sh, n_qb, n_seq);
                const int n_kb = blocks_of(w.qb);
                const int qbuf = lt & 1;
                mbar_wait(&q_full[qbuf], (lt >> 1) & 1);
                fence_after();
                const uint32_t q_base = smem_u32(sQ + qbuf * C::Q_BYTES);
                auto keys = [&](int jj) { return min(kKV, sh.S - jj * kKV); };
                issue_s(g, q_base, keys(0));
                for (int j = 0; j < n_kb; ++j) {
                    if (j + 1 < n_kb) issue_s(g + j + 1, q_base, keys(j + 1));
                    if (j + 1 == n_kb) umma_commit_if(leader, &q_empty[qbuf]);
                    issue_o(g + j, j, n_kb, lt, keys(j));
                }
                g += n_kb;
            }
        }
    } else if (warp >= 4) {
        // ===== softmax: thread = query row (TMEM lane) x key half =====
        const int q4 = warp & 3, h = (warp - 4) >> 2;
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        constexpr int HH = HD / 2;  // output columns of this half
        uint32_t v[32], v2[32];
        float acc[LAZY ? 1 : HH];
        int g = 0, lt = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
            const TileOf w = tile_of(t, sh, n_qb, n_seq);
            const int n_kb = blocks_of(w.qb);
            const int q0 = w.qb * kQ;
            const int qi = q0 + r;
#pragma unroll
            for (int i = 0; i < (LAZY ? 1 : HH); ++i) acc[i] = 0.0f;
            float m_run = -INFINITY, l_h = 0.0f, corr_prev = 1.0f;
            const uint32_t o_lazy = tmem + lane_off + C::T_O + (lt & 1) * HD + h * HH;  // LAZY: this half's O
            auto accumulate_o = [&](int gg, float corr) {
                if (LAZY) return;
                const int ob = gg & 1;
                mbar_wait(&o_full[ob], (gg >> 1) & 1);
                fence_after();
                if (HH % 32 == 0) {
#pragma unroll
                    for (int c = 0; c < HH / 32; ++c) {
                        tmem_ld32(tmem + lane_off + C::T_O + ob * HD + h * HH + c * 32, v);
#pragma unroll
                        for (int i = 0; i < 32; ++i) acc[c * 32 + i] = fmaf(acc[c * 32 + i], corr, __uint_as_float(v[i]));
                    }
                } else {  // head_dim 80: 40 columns per half, 8 at a time
#pragma unroll
                    for (int c = 0; c < HH / 8; ++c) {
                        uint32_t v8[8];
                        tmem_ld8(tmem + lane_off + C::T_O + ob * HD + h * HH + c * 8, v8);
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc[c * 8 + i] = fmaf(acc[c * 8 + i], corr, __uint_as_float(v8[i]));
                    }
                }
                fence_before();
                mbar_arrive(&o_empty[ob]);
            };
            if (LAZY && q0 + q4 * 32 >= sh.S) {
                // a lane quarter wholly past the sequence (ragged S, e.g. ViT's 257 = 2 x 128 + 1:
                // three of the last tile's four quarters): no softmax work, only the barrier
                // protocol. Its O rows accumulate whatever P its TMEM lanes hold and are never
                // stored. Each arrival follows the matching S / O completion, so it cannot count
                // toward an earlier phase.
                for (int j = 0; j < n_kb; ++j, ++g) {
                    mbar_wait(&s_full[g & 1], (g >> 1) & 1);
                    mbar_arrive(&p_full[g & 1]);
                }
                mbar_wait(&o_full[lt & 1], (lt >> 1) & 1);
                mbar_arrive(&o_empty[lt & 1]);
                continue;
            }
            for (int j = 0; j < n_kb; ++j, ++g) {
                const int sb = g & 1;
                const int k0 = j * kKV + 64 * h;  // first key of this half
                const bool need_mask = (sh.causal && k0 + 63 > q0) || k0 + 64 > sh.S;
                const int lim = need_mask ? min(sh.S, sh.causal ? qi + 1 : sh.S) - k0 : 64;  // valid keys
                // a half with no valid key for any of the warp's rows (the ragged last block):
                // P = 0 without reading S
                const bool half_dead = need_mask && __all_sync(0xffffffffu, lim <= 0);
                mbar_wait(&s_full[sb], (g >> 1) & 1);
                fence_after();
                const uint32_t s_addr = tmem + lane_off + sb * 128 + 64 * h;
                if (!half_dead) {
                    tmem_ld32_async(s_addr, v);
                    tmem_ld32_async(s_addr + 32, v2);
                    tmem_ld_wait(v);
                    tmem_ld_wait(v2);
                }
                // row max of the half: eight independent chains, then a tree (short dependency chains)
                float mx8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
                if (half_dead) {
                } else if (need_mask) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float x0 = i < lim ? __uint_as_float(v[i]) : -INFINITY;
                        const float x1 = 32 + i < lim ? __uint_as_float(v2[i]) : -INFINITY;
                        mx8[i & 7] = fmax3(mx8[i & 7], x0, x1);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) mx8[i & 7] = fmax3(mx8[i & 7], __uint_as_float(v[i]), __uint_as_float(v2[i]));
                }
                const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                float* xm = xmax + (g & 1) * 256;
                xm[h * 128 + r] = mraw;
                named_bar_sync(1 + q4, 64);
                const float mrow = fmaxf(mraw, xm[(1 - h) * 128 + r]);
                const float mx = fmaxf(m_run, mrow * sh.scale_log2);
                float base, corr = 1.0f;
                if (!LAZY) {
                    base = mx == -INFINITY ? 0.0f : mx;
                    corr = ex2_fast(m_run - base);
                    m_run = mx;
                } else if (j == 0) {
                    m_run = mx;  // the tile's reference max (its first PV overwrites O)
                    base = mx == -INFINITY ? 0.0f : mx;
                } else {
                    // rescale O and l only when the max has grown past 2^8 of the reference
                    const bool need = mx > (m_run == -INFINITY ? -INFINITY : m_run + 8.0f);
                    if (__any_sync(0xffffffffu, need)) {
                        mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);  // PV of block j - 1 done
                        fence_after();
                        const float f = need ? ex2_fast(m_run - mx) : 1.0f;  // (-inf reference: 0)
                        tmem_scale<HH>(o_lazy, f);
                        l_h *= f;
                        if (need) m_run = mx;
                    }
                    base = m_run == -INFINITY ? 0.0f : m_run;
                }
                uint32_t pk[32];
                float2 rs01 = make_float2(0.0f, 0.0f), rs23 = make_float2(0.0f, 0.0f);  // row-sum chains (pairs)
                if (half_dead) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) pk[i] = 0u;
                } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float2 x01 = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])),
                                             make_float2(sh.scale_log2, sh.scale_log2), make_float2(-base, -base));
                    const float2 x23 = ffma2(make_float2(__uint_as_float(v2[2 * i]), __uint_as_float(v2[2 * i + 1])),
                                             make_float2(sh.scale_log2, sh.scale_log2), make_float2(-base, -base));
                    float p0 = ex2_fast(x01.x), p1 = ex2_fast(x01.y), p2 = ex2_fast(x23.x), p3 = ex2_fast(x23.y);
                    if (need_mask) {
                        if (2 * i >= lim) p0 = 0.0f;
                        if (2 * i + 1 >= lim) p1 = 0.0f;
                        if (32 + 2 * i >= lim) p2 = 0.0f;
                        if (32 + 2 * i + 1 >= lim) p3 = 0.0f;
                    }
                    rs01 = fadd2(rs01, make_float2(p0, p1));
                    rs23 = fadd2(rs23, make_float2(p2, p3));
                    pk[i] = pack_bf16(p0, p1);
                    pk[16 + i] = pack_bf16(p2, p3);
                }
                }
                const float rs0 = rs01.x + rs01.y, rs1 = rs23.x + rs23.y;
                // P over the first 32 of this half's S columns (already read into registers)
                tmem_st16(s_addr, *reinterpret_cast<const uint32_t(*)[16]>(pk));
                tmem_st16(s_addr + 16, *reinterpret_cast<const uint32_t(*)[16]>(pk + 16));
                tmem_st_wait();
                fence_before();
                mbar_arrive(&p_full[sb]);
                l_h = l_h * corr + (rs0 + rs1);
                if (j > 0) accumulate_o(g - 1, corr_prev);
                corr_prev = corr;
            }
            if (n_kb > 0) accumulate_o(g - 1, corr_prev);
            xl[h * 128 + r] = l_h;
            named_bar_sync(1 + q4, 64);
            const float l_run = xl[r] + xl[128 + r];
            const float inv = l_run > 0.0f ? 1.0f / l_run : 0.0f;
            __nv_bfloat16* orow = o + static_cast<int64_t>(w.b * sh.S + qi) * sh.ldo + w.h * HD + h * HH;
            if (LAZY) {  // the tile's O out of TMEM (once), normalised
                mbar_wait(&o_full[lt & 1], (lt >> 1) & 1);
                fence_after();
                if (HH % 32 == 0) {
#pragma unroll
                    for (int c = 0; c < HH / 32; ++c) {
                        tmem_ld32(o_lazy + c * 32, v);
                        if (qi < sh.S) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                uint4 u4;
                                u4.x = pack_bf16(__uint_as_float(v[8 * u + 0]) * inv, __uint_as_float(v[8 * u + 1]) * inv);
                                u4.y = pack_bf16(__uint_as_float(v[8 * u + 2]) * inv, __uint_as_float(v[8 * u + 3]) * inv);
                                u4.z = pack_bf16(__uint_as_float(v[8 * u + 4]) * inv, __uint_as_float(v[8 * u + 5]) * inv);
                                u4.w = pack_bf16(__uint_as_float(v[8 * u + 6]) * inv, __uint_as_float(v[8 * u + 7]) * inv);
                                reinterpret_cast<uint4*>(orow + c * 32)[u] = u4;
                            }
                        }
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < HH / 8; ++c) {
                        uint32_t v8[8];
                        tmem_ld8(o_lazy + c * 8, v8);
                        uint4 u4;
                        u4.x = pack_bf16(__uint_as_float(v8[0]) * inv, __uint_as_float(v8[1]) * inv);
                        u4.y = pack_bf16(__uint_as_float(v8[2]) * inv, __uint_as_float(v8[3]) * inv);
                        u4.z = pack_bf16(__uint_as_float(v8[4]) * inv, __uint_as_float(v8[5]) * inv);
                        u4.w = pack_bf16(__uint_as_float(v8[6]) * inv, __uint_as_float(v8[7]) * inv);
                        if (qi < sh.S) reinterpret_cast<uint4*>(orow)[c] = u4;
                    }
                }
                fence_before();
                mbar_arrive(&o_empty[lt & 1]);
            }
            if (qi < sh.S) {
                if (!LAZY) {
#pragma unroll
                    for (int c = 0; c < HH / 8; ++c) {
                        uint4 u4;
                        u4.x = pack_bf16(acc[8 * c + 0] * inv, acc[8 * c + 1] * inv);
                        u4.y = pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv);
                        u4.z = pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv);
                        u4.w = pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv);
                        reinterpret_cast<uint4*>(orow)[c] = u4;
                    }
                }
                if (h == 0)
                    lse[(static_cast<int64_t>(w.b) * sh.H + w.h) * sh.S + qi] =
                        l_run > 0.0f ? m_run + log2f(l_run) : INFINITY;
            }
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

template <int HD, bool LAZY>
cudaError_t launch_fwd_tc2(const AttnProblem& a, cudaStream_t st) {
    using C = Fwd2Cfg<HD>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc2_kernel<HD, LAZY>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int ld = (a.n_heads + 2 * a.n_kv_heads) * a.head_dim;
    CUtensorMap tqk, tv;
    if (!make_map(&tqk, a.qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(a.tokens), static_cast<uint64_t>(ld), 64,
                  128, false, false) ||
        !make_map(&tv, a.qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(a.tokens), static_cast<uint64_t>(ld), 64, 64,
                  false, false))
        return cudaErrorInvalidValue;
    CUtensorMap tqk1 = tqk, tv1 = tv;  // head_dim 80: the 16-column tails (32B swizzle)
    if (C::NARROW && (!make_map_sw32(&tqk1, a.qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(a.tokens),
                                     static_cast<uint64_t>(ld), 16, 128) ||
                      !make_map_sw32(&tv1, a.qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(a.tokens),
                                     static_cast<uint64_t>(ld), 16, 64)))
        return cudaErrorInvalidValue;
    TcShape sh;
    sh.S = a.seq_len;
    sh.H = a.n_heads;
    sh.Hkv = a.n_kv_heads;
    sh.ld = ld;
    sh.ldo = a.n_heads * a.head_dim;
    sh.causal = a.causal;
    sh.chunk = attention_causal_chunk(a);
    sh.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(a.head_dim));
    const int n_seq = static_cast<int>(a.tokens / a.seq_len);
    const int tiles = ((a.seq_len + kQ - 1) / kQ) * a.n_heads * n_seq;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    attn_fwd_tc2_kernel<HD, LAZY><<<grid, kThreadsF2, C::SMEM, st>>>(tqk, tv, tqk1, tv1, static_cast<__nv_bfloat16*>(a.o), a.lse, sh,
                                                                n_seq);
    return cudaGetLastError();
}

template <int HD>
cudaError_t launch_fwd_tc(const AttnProblem& a, cudaStream_t st) {
    using C = AttnCfg<HD>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int ld = (a.n_heads + 2 * a.n_kv_heads) * a.head_dim;
    CUtensorMap tqk, tv;
    if (!make_map(&tqk, a.qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(a.tokens), static_cast<uint64_t>(ld), 64,
                  128, false, false) ||
        !make_map(&tv, a.qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(a.tokens), static_cast<uint64_t>(ld), 64, 64,
                  false, false))
        return cudaErrorInvalidValue;
    TcShape sh;
    sh.S = a.seq_len;
    sh.H = a.n_heads;
    sh.Hkv = a.n_kv_heads;
    sh.ld = ld;
    sh.ldo = a.n_heads * a.head_dim;
    sh.causal = a.causal;
    sh.chunk = attention_causal_chunk(a);
    sh.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(a.head_dim));
    const int n_seq = static_cast<int>(a.tokens / a.seq_len);
    const int tiles = ((a.seq_len + kQ - 1) / kQ) * a.n_heads * n_seq;
    const int grid = tiles < num_sms() ? tiles : num_sms();  // persistent: one CTA per SM
    attn_fwd_tc_kernel<HD><<<grid, kThreadsTc, C::SMEM, st>>>(tqk, tv, static_cast<__nv_bfloat16*>(a.o), a.lse, sh,
                                                              n_seq);
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------------------
// backward (tcgen05): dK / dV per key block, dQ per query block (no atomics: deterministic)
// ---------------------------------------------------------------------------------------
// Tiles in smem are stored as ATOMS boxes of 128 rows x 128 bytes (64 elements of the head dim),
// 128B-swizzled: the same tile is a K-major operand (rows = M or N, K = head dim) and an
// N-major B operand (rows = K, N = head dim; atoms 16 KB apart), so Q, dO and K each serve
// both products they appear in without a transposed copy.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
template <int ATOMS>
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {  // K-major, 16-element K step kk
    return make_desc(base + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t ndesc(uint32_t base, int kk) {  // N-major B, 16-row K step kk
    return make_desc(base + kk * 16 * 128, 16384, 1024);
}
// P / dS row chunk (32 values of row r, columns 32c..32c+31) into a K-major swizzled tile
__device__ __forceinline__ void store_row_chunk(uint8_t* tile, int r, int c, const uint32_t (&pk)[16]) {
    uint8_t* row = tile + (c / 2) * 16384 + r * 128;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int chunk = (c % 2) * 4 + u;
        *reinterpret_cast<uint4*>(row + ((chunk ^ (r & 7)) << 4)) =
            make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
    }
}

template <int HD>
struct BwdCfg {
    static constexpr int ATOMS = HD / 64;
    static constexpr int TILE = 128 * HD * 2;  // one 128-row operand tile
    static constexpr int QB = HD <= 64 ? 2 : 1;  // Q / dO buffers (dK/dV kernel)
    static constexpr int SMEM_KV = 2 * TILE + QB * 2 * TILE + 2 * 32768 + QB * 2 * 512 + 1024 + 256;
    static constexpr int SMEM_Q = 2 * TILE + 2 * 2 * TILE + 32768 + 1024 + 256;
};

// dK, dV: tile = (128 keys, kv head, sequence); for every query head of the group and every
// query block: S^T = K Q^T, dP^T = V dO^T (TMEM), the softmax warps (thread = key row) form
// P^T = exp2(S^T c - lse) and dS^T = P^T (dP^T - delta) in smem, then dV += P^T dO, dK += dS^T Q.
template <int HD>
__global__ void __launch_bounds__(kThreadsTc, 1)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmDO,
                            const float* __restrict__ lse, const float* __restrict__ delta,
                            __nv_bfloat16* __restrict__ dqkv, TcShape sh, int n_seq, float scale) {
    using C = BwdCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem;
    uint8_t* sV = sK + C::TILE;
    uint8_t* sQ = sV + C::TILE;              // QB tiles
    uint8_t* sDO = sQ + C::QB * C::TILE;     // QB tiles
    uint8_t* sP = sDO + C::QB * C::TILE;     // 32 KB: P^T [key][q]
    uint8_t* sDS = sP + 32768;               // 32 KB: dS^T [key][q]
    float* sL = reinterpret_cast<float*>(sDS + 32768);  // QB x 128 lse
    float* sD = sL + C::QB * 128;                       // QB x 128 delta
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + C::QB * 128);
    uint64_t* kv_full = bars;
    uint64_t* kv_empty = bars + 1;
    uint64_t* q_full = bars + 2;      // QB
    uint64_t* q_empty = bars + 4;     // QB
    uint64_t* s_full = bars + 6;
    uint64_t* s_empty = bars + 7;
    uint64_t* p_full = bars + 8;
    uint64_t* p_empty = bars + 9;
    uint64_t* dkv_full = bars + 10;
    uint64_t* dkv_empty = bars + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_qb = sh.S / kQ, n_kb = sh.S / kKV;
    const int group = sh.H / sh.Hkv;
    const int n_tiles = n_kb * sh.Hkv * n_seq;
    constexpr uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 256 + HD;
    // tile t: key block ascending (causal: the first key blocks see the most query blocks)
    auto tile_of_kv = [&](int t, int& kb, int& kvh, int& b) {
        const int per = sh.Hkv * n_seq;
        kb = t / per;
        const int rest = t % per;
        kvh = rest % sh.Hkv;
        b = rest / sh.Hkv;
    };
    auto n_steps = [&](int kb) { return group * (sh.causal ? n_qb - kb : n_qb); };
    auto step_of = [&](int kb, int kvh, int j, int& hq, int& qb) {
        const int per = sh.causal ? n_qb - kb : n_qb;
        hq = kvh * group + j / per;
        qb = (sh.causal ? kb : 0) + j % per;
    };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmQK);
        prefetch_tmap(&tmDO);
        for (int i = 0; i < 12; ++i) mbar_init(&bars[i], 1);
        mbar_init(s_empty, 128);
        mbar_init(p_full, 128);
        mbar_init(dkv_empty, 128);
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
                tile_of_kv(t, kb, kvh, b);
                const int row0 = b * sh.S;
                const int kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
                mbar_wait(kv_empty, (lt & 1) ^ 1);
                mbar_expect_tx(kv_full, 2 * C::TILE);
                for (int a = 0; a < C::ATOMS; ++a) {
                    tma_load_2d(&tmQK, kv_full, sK + a * 16384, kcol + 64 * a, row0 + kb * kKV);
                    tma_load_2d(&tmQK, kv_full, sV + a * 16384, vcol + 64 * a, row0 + kb * kKV);
                }
                const int n = n_steps(kb);
                for (int j = 0; j < n; ++j, ++g) {
                    int hq, qb;
                    step_of(kb, kvh, j, hq, qb);
                    const int buf = g % C::QB;
                    mbar_wait(&q_empty[buf], ((g / C::QB) & 1) ^ 1);
                    mbar_expect_tx(&q_full[buf], 2 * C::TILE + 2 * 512);
                    for (int a = 0; a < C::ATOMS; ++a) {
                        tma_load_2d(&tmQK, &q_full[buf], sQ + buf * C::TILE + a * 16384, hq * HD + 64 * a,
                                    row0 + qb * kQ);
                        tma_load_2d(&tmDO, &q_full[buf], sDO + buf * C::TILE + a * 16384, hq * HD + 64 * a,
                                    row0 + qb * kQ);
                    }
                    const int64_t li = (static_cast<int64_t>(b) * sh.H + hq) * sh.S + qb * kQ;
                    bulk_load(sL + buf * 128, lse + li, 512, &q_full[buf]);
                    bulk_load(sD + buf * 128, delta + li, 512, &q_full[buf]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer =====
            constexpr uint32_t IDESC_S = make_idesc(128, 128, false, false);
            constexpr uint32_t IDESC_D = make_idesc(128, HD, false, true);
            const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
            const uint32_t p_base = smem_u32(sP), ds_base = smem_u32(sDS);
            auto issue_sdp = [&](int g) {
                const int buf = g % C::QB;
                mbar_wait(&q_full[buf], (g / C::QB) & 1);
                mbar_wait(s_empty, (g & 1) ^ 1);
                fence_after();
                const uint32_t qb_ = smem_u32(sQ + buf * C::TILE), db_ = smem_u32(sDO + buf * C::TILE);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    umma<false>(tmem + T_S, kdesc<C::ATOMS>(k_base, kk), kdesc<C::ATOMS>(qb_, kk), IDESC_S, kk > 0);
                    umma<false>(tmem + T_DP, kdesc<C::ATOMS>(v_base, kk), kdesc<C::ATOMS>(db_, kk), IDESC_S, kk > 0);
                }
                umma_commit(s_full);
            };
            auto issue_dkv = [&](int g, bool first) {
                const int buf = g % C::QB;
                mbar_wait(p_full, g & 1);
                fence_after();
                const uint32_t qb_ = smem_u32(sQ + buf * C::TILE), db_ = smem_u32(sDO + buf * C::TILE);
#pragma unroll
                for (int kk = 0; kk < 128 / 16; ++kk) {
                    const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
                    umma<false>(tmem + T_DV, kdesc<2>(p_base, kk), ndesc(db_, kk), IDESC_D, acc);
                    umma<false>(tmem + T_DK, kdesc<2>(ds_base, kk), ndesc(qb_, kk), IDESC_D, acc);
                }
                umma_commit(p_empty);
                umma_commit(&q_empty[buf]);
            };
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                int kb, kvh, b;
                tile_of_kv(t, kb, kvh, b);
                const int n = n_steps(kb);
                mbar_wait(kv_full, lt & 1);
                mbar_wait(dkv_empty, (lt & 1) ^ 1);  // the previous tile's dK / dV are read out
                fence_after();
                issue_sdp(g);
                for (int j = 0; j < n; ++j) {
                    // the next block's S^T / dP^T run under this block's softmax; with one Q / dO
                    // buffer (head_dim 128) its loads wait for this block's dK / dV MMAs first
                    if (C::QB > 1 && j + 1 < n) issue_sdp(g + j + 1);
                    issue_dkv(g + j, j == 0);
                    if (C::QB == 1 && j + 1 < n) issue_sdp(g + j + 1);
                }
                umma_commit(dkv_full);
                umma_commit(kv_empty);
                g += n;
            }
        }
    } else if (warp >= 4) {
        // ===== softmax: one key row per thread =====
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        uint32_t vs[32], vp[32];
        int g = 0, lt = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
            int kb, kvh, b;
            tile_of_kv(t, kb, kvh, b);
            const int key = kb * kKV + r;
            const int n = n_steps(kb);
            for (int j = 0; j < n; ++j, ++g) {
                int hq, qb;
                step_of(kb, kvh, j, hq, qb);
                const int buf = g % C::QB;
                const float* L = sL + buf * 128;
                const float* D = sD + buf * 128;
                mbar_wait(s_full, g & 1);
                fence_after();
                if (g > 0) mbar_wait(p_empty, (g & 1) ^ 1);  // the previous block's dK / dV MMAs read P, dS
                const bool diag = sh.causal && qb == kb;  // keys above a query of this block: masked
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    tmem_ld32_async(tmem + lane_off + T_S + c * 32, vs);
                    tmem_ld32_async(tmem + lane_off + T_DP + c * 32, vp);
                    tmem_ld_wait(vs);
                    tmem_ld_wait(vp);
                    uint32_t pp[16], dd[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int q0 = c * 32 + 2 * i;
                        float p0 = ex2_fast(fmaf(__uint_as_float(vs[2 * i]), sh.scale_log2, -L[q0]));
                        float p1 = ex2_fast(fmaf(__uint_as_float(vs[2 * i + 1]), sh.scale_log2, -L[q0 + 1]));
                        if (diag) {
                            if (r > q0) p0 = 0.0f;
                            if (r > q0 + 1) p1 = 0.0f;
                        }
                        const float d0 = p0 * (__uint_as_float(vp[2 * i]) - D[q0]);
                        const float d1 = p1 * (__uint_as_float(vp[2 * i + 1]) - D[q0 + 1]);
                        pp[i] = pack_bf16(p0, p1);
                        dd[i] = pack_bf16(d0, d1);
                    }
                    store_row_chunk(sP, r, c, pp);
                    store_row_chunk(sDS, r, c, dd);
                }
                fence_before();
                mbar_arrive(s_empty);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(p_full);
            }
            // the tile's dK, dV out of TMEM (dK gets the softmax scale)
            mbar_wait(dkv_full, lt & 1);
            fence_after();
            __nv_bfloat16* row = dqkv + static_cast<int64_t>(b * sh.S + key) * sh.ld;
            const int kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
                tmem_ld32_async(tmem + lane_off + T_DK + c * 32, vs);
                tmem_ld32_async(tmem + lane_off + T_DV + c * 32, vp);
                tmem_ld_wait(vs);
                tmem_ld_wait(vp);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint4 wk, wv;
                    wk.x = pack_bf16(__uint_as_float(vs[8 * u + 0]) * scale, __uint_as_float(vs[8 * u + 1]) * scale);
                    wk.y = pack_bf16(__uint_as_float(vs[8 * u + 2]) * scale, __uint_as_float(vs[8 * u + 3]) * scale);
                    wk.z = pack_bf16(__uint_as_float(vs[8 * u + 4]) * scale, __uint_as_float(vs[8 * u + 5]) * scale);
                    wk.w = pack_bf16(__uint_as_float(vs[8 * u + 6]) * scale, __uint_as_float(vs[8 * u + 7]) * scale);
                    wv.x = pack_bf16(__uint_as_float(vp[8 * u + 0]), __uint_as_float(vp[8 * u + 1]));
                    wv.y = pack_bf16(__uint_as_float(vp[8 * u + 2]), __uint_as_float(vp[8 * u + 3]));
                    wv.z = pack_bf16(__uint_as_float(vp[8 * u + 4]), __uint_as_float(vp[8 * u + 5]));
                    wv.w = pack_bf16(__uint_as_float(vp[8 * u + 6]), __uint_as_float(vp[8 * u + 7]));
                    reinterpret_cast<uint4*>(row + kcol + c * 32)[u] = wk;
                    reinterpret_cast<uint4*>(row + vcol + c * 32)[u] = wv;
                }
            }
            fence_before();
            mbar_arrive(dkv_empty);
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

// dQ: tile = (128 queries, head, sequence); for every key block: S = Q K^T, dP = dO V^T (TMEM),
// the softmax warps (thread = query row) form dS = P (dP - delta) in smem, then dQ += dS K.
template <int HD>
__global__ void __launch_bounds__(kThreadsTc, 1)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmDO,
                          const float* __restrict__ lse, const float* __restrict__ delta,
                          __nv_bfloat16* __restrict__ dqkv, TcShape sh, int n_seq, float scale) {
    using C = BwdCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sDO = sQ + C::TILE;
    uint8_t* sK = sDO + C::TILE;           // 2 stages
    uint8_t* sV = sK + 2 * C::TILE;        // 2 stages
    uint8_t* sDS = sV + 2 * C::TILE;       // 32 KB: dS [q][key]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sDS + 32768);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* kv_full = bars + 2;   // 2
    uint64_t* kv_empty = bars + 4;  // 2
    uint64_t* s_full = bars + 6;
    uint64_t* s_empty = bars + 7;
    uint64_t* p_full = bars + 8;
    uint64_t* p_empty = bars + 9;
    uint64_t* dq_full = bars + 10;
    uint64_t* dq_empty = bars + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_qb = sh.S / kQ, n_kb_total = sh.S / kKV;
    const int n_tiles = n_qb * sh.H * n_seq;
    constexpr uint32_t T_S = 0, T_DP = 128, T_DQ = 256;
    auto blocks_of = [&](int qb) { return sh.causal ? min(n_kb_total, qb + 1) : n_kb_total; };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmQK);
        prefetch_tmap(&tmDO);
        for (int i = 0; i < 12; ++i) mbar_init(&bars[i], 1);
        mbar_init(s_empty, 128);
        mbar_init(p_full, 128);
        mbar_init(dq_empty, 128);
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
                const TileOf w = tile_of(t, sh, n_qb, n_seq);
                const int kvh = w.h / (sh.H / sh.Hkv);
                const int row0 = w.b * sh.S;
                const int kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;
                mbar_wait(q_empty, (lt & 1) ^ 1);
                mbar_expect_tx(q_full, 2 * C::TILE);
                for (int a = 0; a < C::ATOMS; ++a) {
                    tma_load_2d(&tmQK, q_full, sQ + a * 16384, w.h * HD + 64 * a, row0 + w.qb * kQ);
                    tma_load_2d(&tmDO, q_full, sDO + a * 16384, w.h * HD + 64 * a, row0 + w.qb * kQ);
                }
                const int n = blocks_of(w.qb);
                for (int j = 0; j < n; ++j, ++g) {
                    const int st = g & 1;
                    mbar_wait(&kv_empty[st], ((g >> 1) & 1) ^ 1);
                    mbar_expect_tx(&kv_full[st], 2 * C::TILE);
                    for (int a = 0; a < C::ATOMS; ++a) {
                        tma_load_2d(&tmQK, &kv_full[st], sK + st * C::TILE + a * 16384, kcol + 64 * a, row0 + j * kKV);
                        tma_load_2d(&tmQK, &kv_full[st], sV + st * C::TILE + a * 16384, vcol + 64 * a, row0 + j * kKV);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer =====
            constexpr uint32_t IDESC_S = make_idesc(128, 128, false, false);
            constexpr uint32_t IDESC_D = make_idesc(128, HD, false, true);
            const uint32_t q_base = smem_u32(sQ), do_base = smem_u32(sDO), ds_base = smem_u32(sDS);
            auto issue_sdp = [&](int g) {
                const int st = g & 1;
                mbar_wait(&kv_full[st], (g >> 1) & 1);
                mbar_wait(s_empty, (g & 1) ^ 1);
                fence_after();
                const uint32_t kb_ = smem_u32(sK + st * C::TILE), vb_ = smem_u32(sV + st * C::TILE);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    umma<false>(tmem + T_S, kdesc<C::ATOMS>(q_base, kk), kdesc<C::ATOMS>(kb_, kk), IDESC_S, kk > 0);
                    umma<false>(tmem + T_DP, kdesc<C::ATOMS>(do_base, kk), kdesc<C::ATOMS>(vb_, kk), IDESC_S, kk > 0);
                }
                umma_commit(s_full);
            };
            auto issue_dq = [&](int g, bool first) {
                const int st = g & 1;
                mbar_wait(p_full, g & 1);
                fence_after();
                const uint32_t kb_ = smem_u32(sK + st * C::TILE);
#pragma unroll
                for (int kk = 0; kk < 128 / 16; ++kk)
                    umma<false>(tmem + T_DQ, kdesc<2>(ds_base, kk), ndesc(kb_, kk), IDESC_D, (!first || kk > 0) ? 1u : 0u);
                umma_commit(p_empty);
                umma_commit(&kv_empty[st]);
            };
            int g = 0, lt = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
                const TileOf w = tile_of(t, sh, n_qb, n_seq);
                const int n = blocks_of(w.qb);
                mbar_wait(q_full, lt & 1);
                mbar_wait(dq_empty, (lt & 1) ^ 1);
                fence_after();
                issue_sdp(g);
                for (int j = 0; j < n; ++j) {
                    if (j + 1 < n) issue_sdp(g + j + 1);
                    issue_dq(g + j, j == 0);
                }
                umma_commit(dq_full);
                umma_commit(q_empty);
                g += n;
            }
        }
    } else if (warp >= 4) {
        // ===== softmax: one query row per thread =====
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        uint32_t vs[32], vp[32];
        int g = 0, lt = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++lt) {
            const TileOf w = tile_of(t, sh, n_qb, n_seq);
            const int qi = w.qb * kQ + r;
            const int64_t li = (static_cast<int64_t>(w.b) * sh.H + w.h) * sh.S + qi;
            const float L = lse[li], Dl = delta[li];
            const int n = blocks_of(w.qb);
            for (int j = 0; j < n; ++j, ++g) {
                mbar_wait(s_full, g & 1);
                fence_after();
                if (g > 0) mbar_wait(p_empty, (g & 1) ^ 1);
                const bool diag = sh.causal && j == w.qb;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    tmem_ld32_async(tmem + lane_off + T_S + c * 32, vs);
                    tmem_ld32_async(tmem + lane_off + T_DP + c * 32, vp);
                    tmem_ld_wait(vs);
                    tmem_ld_wait(vp);
                    uint32_t dd[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int k0 = c * 32 + 2 * i;  // key within the block
                        float p0 = ex2_fast(fmaf(__uint_as_float(vs[2 * i]), sh.scale_log2, -L));
                        float p1 = ex2_fast(fmaf(__uint_as_float(vs[2 * i + 1]), sh.scale_log2, -L));
                        if (diag) {
                            if (k0 > r) p0 = 0.0f;
                            if (k0 + 1 > r) p1 = 0.0f;
                        }
                        dd[i] = pack_bf16(p0 * (__uint_as_float(vp[2 * i]) - Dl), p1 * (__uint_as_float(vp[2 * i + 1]) - Dl));
                    }
                    store_row_chunk(sDS, r, c, dd);
                }
                fence_before();
                mbar_arrive(s_empty);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(p_full);
            }
            mbar_wait(dq_full, lt & 1);
            fence_after();
            __nv_bfloat16* row = dqkv + static_cast<int64_t>(w.b * sh.S + qi) * sh.ld + w.h * HD;
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
                tmem_ld32_async(tmem + lane_off + T_DQ + c * 32, vs);
                tmem_ld_wait(vs);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint4 wq;
                    wq.x = pack_bf16(__uint_as_float(vs[8 * u + 0]) * scale, __uint_as_float(vs[8 * u + 1]) * scale);
                    wq.y = pack_bf16(__uint_as_float(vs[8 * u + 2]) * scale, __uint_as_float(vs[8 * u + 3]) * scale);
                    wq.z = pack_bf16(__uint_as_float(vs[8 * u + 4]) * scale, __uint_as_float(vs[8 * u + 5]) * scale);
                    wq.w = pack_bf16(__uint_as_float(vs[8 * u + 6]) * scale, __uint_as_float(vs[8 * u + 7]) * scale);
                    reinterpret_cast<uint4*>(row + c * 32)[u] = wq;
                }
            }
            fence_before();
            mbar_arrive(dq_empty);
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
cudaError_t launch_bwd_tc(const AttnProblem& a, cudaStream_t st) {
    using C = BwdCfg<HD>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM_KV);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attn_bwd_dq_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_Q);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int ld = (a.n_heads + 2 * a.n_kv_heads) * a.head_dim;
    const int ldo = a.n_heads * a.head_dim;
    CUtensorMap tqk, tdo;
    if (!make_map(&tqk, a.qkv, static_cast<uint64_t>(ld), static_cast<uint64_t>(a.tokens), static_cast<uint64_t>(ld), 64,
                  128, false, false) ||
        !make_map(&tdo, a.dout, static_cast<uint64_t>(ldo), static_cast<uint64_t>(a.tokens), static_cast<uint64_t>(ldo),
                  64, 128, false, false))
        return cudaErrorInvalidValue;
    TcShape sh;
    sh.S = a.seq_len;
    sh.H = a.n_heads;
    sh.Hkv = a.n_kv_heads;
    sh.ld = ld;
    sh.ldo = ldo;
    sh.causal = a.causal;
    sh.chunk = attention_causal_chunk(a);
    const float scale = 1.0f / sqrtf(static_cast<float>(a.head_dim));
    sh.scale_log2 = 1.4426950408889634f * scale;
    const int n_seq = static_cast<int>(a.tokens / a.seq_len);
    const int kv_tiles = (a.seq_len / 128) * a.n_kv_heads * n_seq;
    const int q_tiles = (a.seq_len / 128) * a.n_heads * n_seq;
    auto* dq = static_cast<__nv_bfloat16*>(a.dqkv);
    attn_bwd_dkdv_tc_kernel<HD><<<kv_tiles < num_sms() ? kv_tiles : num_sms(), kThreadsTc, C::SMEM_KV, st>>>(
        tqk, tdo, a.lse, a.delta, dq, sh, n_seq, scale);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    attn_bwd_dq_tc_kernel<HD><<<q_tiles < num_sms() ? q_tiles : num_sms(), kThreadsTc, C::SMEM_Q, st>>>(
        tqk, tdo, a.lse, a.delta, dq, sh, n_seq, scale);
    return cudaGetLastError();
}
}  // namespace

// The tensor-core forward for head_dim 64 / 128 (the GPT-2 XL and Llama-3 shapes);
// cudaErrorNotSupported for other head dims (the caller falls back to the mma.sync kernel).
cudaError_t attention_forward_tc(const AttnProblem& a, cudaStream_t st, int kind) {
    // kind: 4 v3 (O in TMEM, lazy rescale), 2 v2 (O in registers), 3 v1 (4 softmax warps)
    switch (a.head_dim) {
        case 64: return kind == 4 ? launch_fwd_tc2<64, true>(a, st) : kind == 2 ? launch_fwd_tc2<64, false>(a, st) : launch_fwd_tc<64>(a, st);
        case 80: return kind == 4 ? launch_fwd_tc2<80, true>(a, st) : launch_fwd_tc2<80, false>(a, st);
        case 128: return kind == 4 ? launch_fwd_tc2<128, true>(a, st) : kind == 2 ? launch_fwd_tc2<128, false>(a, st) : launch_fwd_tc<128>(a, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace sp

namespace sp {
// The tensor-core dK/dV and dQ passes for head_dim 64 / 128 and sequences that are whole 128-row
// blocks (GPT-2 XL, Llama-3); cudaErrorNotSupported otherwise. delta must be filled first.
cudaError_t attention_backward_tc(const AttnProblem& a, cudaStream_t st) {
    if (a.seq_len % 128 != 0) return cudaErrorNotSupported;
    if (a.head_dim == 64) return launch_bwd_tc<64>(a, st);
    if (a.head_dim == 128) return launch_bwd_tc<128>(a, st);
    return cudaErrorNotSupported;
}
}  // namespace sp

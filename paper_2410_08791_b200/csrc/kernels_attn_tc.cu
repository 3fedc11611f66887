// kernels_attn_tc.cu — tcgen05 flash-attention forward (sm_100a), head_dim 64 and 128.
//
// One CTA = 128 queries of one (sequence, head); 256 threads:
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
    static constexpr int P_BUFS = HD <= 64 ? 2 : 1;
    static constexpr int SMEM = Q_BYTES + 2 * kStages * KV_BYTES + P_BUFS * P_BYTES + 1024 + 256;
    static constexpr int O_COL0 = 2 * kKV;                // TMEM: S[0], S[1], then O[0], O[1]
};

struct TcShape {
    int S, H, Hkv, ld, ldo, causal;
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

template <int HD>
__global__ void __launch_bounds__(kThreadsTc, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQK, const __grid_constant__ CUtensorMap tmV,
                       __nv_bfloat16* __restrict__ o, float* __restrict__ lse, TcShape sh) {
    using C = AttnCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + C::Q_BYTES;                     // kStages tiles
    uint8_t* sV = sK + kStages * C::KV_BYTES;          // kStages tiles
    uint8_t* sP = sV + kStages * C::KV_BYTES;          // P_BUFS tiles
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BUFS * C::P_BYTES);
    uint64_t* q_full = bars;                 // 1
    uint64_t* kv_full = bars + 1;            // kStages
    uint64_t* kv_empty = kv_full + kStages;  // kStages
    uint64_t* s_full = kv_empty + kStages;   // 2
    uint64_t* s_empty = s_full + 2;          // 2
    uint64_t* p_full = s_empty + 2;          // 2 (indexed by P buffer)
    uint64_t* p_empty = p_full + 2;          // 2
    uint64_t* o_full = p_empty + 2;          // 2
    uint64_t* o_empty = o_full + 2;          // 2
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int kvh = h / (sh.H / sh.Hkv);
    const int q0 = qb * kQ;
    const int row0 = b * sh.S;  // first token of the sequence
    const int n_kb_total = (sh.S + kKV - 1) / kKV;
    const int n_kb = sh.causal ? min(n_kb_total, (q0 + kQ - 1) / kKV + 1) : n_kb_total;
    const int qcol = h * HD, kcol = (sh.H + kvh) * HD, vcol = (sh.H + sh.Hkv + kvh) * HD;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmQK);
        prefetch_tmap(&tmV);
        mbar_init(q_full, 1);
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

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            mbar_expect_tx(q_full, C::Q_BYTES);
            for (int a = 0; a < C::ATOMS; ++a) tma_load_2d(&tmQK, q_full, sQ + a * kQ * 128, qcol + 64 * a, row0 + q0);
            for (int j = 0; j < n_kb; ++j) {
                const int st = j % kStages;
                mbar_wait(&kv_empty[st], ((j / kStages) & 1) ^ 1);
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
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer =====
            constexpr uint32_t IDESC_S = make_idesc(kQ, kKV, false, false);
            constexpr uint32_t IDESC_O = make_idesc(kQ, HD, false, true);
            mbar_wait(q_full, 0);
            fence_after();
            const uint32_t q_base = smem_u32(sQ);
            auto issue_s = [&](int j) {
                const int st = j % kStages, sb = j & 1;
                mbar_wait(&kv_full[st], (j / kStages) & 1);
                mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t k_base = smem_u32(sK + st * C::KV_BYTES);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const int a = kk / 4, w = kk % 4;  // atom, 32-byte step within the atom
                    const uint64_t ad = make_desc(q_base + a * kQ * 128 + w * 32, 16, 1024);
                    const uint64_t bd = make_desc(k_base + a * kKV * 128 + w * 32, 16, 1024);
                    umma<false>(tmem + sb * kKV, ad, bd, IDESC_S, kk > 0 ? 1u : 0u);
                }
                umma_commit(&s_full[sb]);
            };
            auto issue_o = [&](int j) {
                const int st = j % kStages, ob = j & 1, pb = j % C::P_BUFS;
                mbar_wait(&p_full[pb], (j / C::P_BUFS) & 1);
                mbar_wait(&o_empty[ob], ((j >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t p_base = smem_u32(sP + pb * C::P_BYTES);
                const uint32_t v_base = smem_u32(sV + st * C::KV_BYTES);
#pragma unroll
                for (int kk = 0; kk < kKV / 16; ++kk) {
                    const int a = kk / 4, w = kk % 4;
                    const uint64_t ad = make_desc(p_base + a * kQ * 128 + w * 32, 16, 1024);
                    // N-major V: k-block a (64 keys), 16-key step w; atoms of 64 d at 8 KB stride
                    const uint64_t bd = make_desc(v_base + a * C::ATOMS * 8192 + w * 16 * 128, 8192, 1024);
                    umma<false>(tmem + C::O_COL0 + ob * HD, ad, bd, IDESC_O, kk > 0 ? 1u : 0u);
                }
                umma_commit(&o_full[ob]);
                umma_commit(&p_empty[pb]);
                umma_commit(&kv_empty[st]);  // both MMAs of block j are done with K_j, V_j
            };
            if (n_kb > 0) issue_s(0);
            for (int j = 0; j < n_kb; ++j) {
                if (j + 1 < n_kb) issue_s(j + 1);
                issue_o(j);
            }
        }
    } else if (warp >= 4) {
        // ===== softmax: one query row per thread =====
        const int q = warp & 3;
        const int r = q * 32 + lane;   // row in the tile = TMEM lane
        const int qi = q0 + r;         // query index in the sequence
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        float acc[HD];
#pragma unroll
        for (int i = 0; i < HD; ++i) acc[i] = 0.0f;
        float m_run = -INFINITY, l_run = 0.0f, corr_prev = 1.0f;
        uint32_t v[32], v2[32];
        auto accumulate_o = [&](int j, float corr) {
            const int ob = j & 1;
            mbar_wait(&o_full[ob], (j >> 1) & 1);
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
        for (int j = 0; j < n_kb; ++j) {
            const int sb = j & 1, pb = j % C::P_BUFS;
            const int k0 = j * kKV;
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            fence_after();
            const uint32_t s_addr = tmem + lane_off + sb * kKV;
            // masking is needed only on the diagonal block (causal) and a ragged last block
            const bool need_mask = (sh.causal && k0 + kKV - 1 > q0) || k0 + kKV > sh.S;
            const int lim = need_mask ? min(sh.S, sh.causal ? qi + 1 : sh.S) - k0 : kKV;  // keys [k0, k0+lim) count
            // pass 1: row max of the raw scores (the scale is positive), two 32-column loads per wait
            float mraw = -INFINITY;
#pragma unroll
            for (int c = 0; c < kKV / 32; c += 2) {
                tmem_ld32_async(s_addr + c * 32, v);
                tmem_ld32_async(s_addr + (c + 1) * 32, v2);
                tmem_ld_wait(v);
                tmem_ld_wait(v2);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float x0 = (!need_mask || c * 32 + i < lim) ? __uint_as_float(v[i]) : -INFINITY;
                    const float x1 = (!need_mask || (c + 1) * 32 + i < lim) ? __uint_as_float(v2[i]) : -INFINITY;
                    mraw = fmaxf(mraw, fmaxf(x0, x1));
                }
            }
            const float mx = fmaxf(m_run, mraw * sh.scale_log2);
            const float base = mx == -INFINITY ? 0.0f : mx;
            const float corr = ex2_fast(m_run - base);
            m_run = mx;
            // pass 2: P_j = exp2(s * scale - m) (one FFMA + one MUFU ex2 each), row sum, bf16 pairs
            // into the K-major swizzled P tile (row r)
            if (j >= C::P_BUFS) mbar_wait(&p_empty[pb], ((j / C::P_BUFS) & 1) ^ 1);
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
                // 32 keys = 4 16-byte chunks; atom = c / 2, chunk within the 128-byte row
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int chunk = (c % 2) * 4 + u;
                    uint8_t* dst = prow + (c / 2) * kQ * 128 + ((chunk ^ (r & 7)) << 4);
                    *reinterpret_cast<uint4*>(dst) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
                }
            }
            l_run = l_run * corr + (rs0 + rs1);
            fence_before();
            mbar_arrive(&s_empty[sb]);  // S_j read: the MMA may overwrite the buffer
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the tensor core
            mbar_arrive(&p_full[pb]);
            if (j > 0) accumulate_o(j - 1, corr_prev);
            corr_prev = corr;
        }
        if (n_kb > 0) accumulate_o(n_kb - 1, corr_prev);
        if (qi < sh.S) {
            const float inv = l_run > 0.0f ? 1.0f / l_run : 0.0f;
            __nv_bfloat16* orow = o + static_cast<int64_t>(row0 + qi) * sh.ldo + h * HD;
#pragma unroll
            for (int c = 0; c < HD / 8; ++c) {
                uint4 w;
                w.x = pack_bf16(acc[8 * c + 0] * inv, acc[8 * c + 1] * inv);
                w.y = pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv);
                w.z = pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv);
                w.w = pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv);
                reinterpret_cast<uint4*>(orow)[c] = w;
            }
            lse[(static_cast<int64_t>(b) * sh.H + h) * sh.S + qi] = l_run > 0.0f ? m_run + log2f(l_run) : INFINITY;
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
    sh.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(a.head_dim));
    const dim3 grid((a.seq_len + kQ - 1) / kQ, a.n_heads, static_cast<unsigned>(a.tokens / a.seq_len));
    attn_fwd_tc_kernel<HD><<<grid, kThreadsTc, C::SMEM, st>>>(tqk, tv, static_cast<__nv_bfloat16*>(a.o), a.lse, sh);
    return cudaGetLastError();
}

}  // namespace

// The tensor-core forward for head_dim 64 / 128 (the GPT-2 XL and Llama-3 shapes);
// cudaErrorNotSupported for other head dims (the caller falls back to the mma.sync kernel).
cudaError_t attention_forward_tc(const AttnProblem& a, cudaStream_t st) {
    if (a.head_dim == 64) return launch_fwd_tc<64>(a, st);
    if (a.head_dim == 128) return launch_fwd_tc<128>(a, st);
    return cudaErrorNotSupported;
}

}  // namespace sp

// kernels_tc.cu — warp-specialized tcgen05 GEMM for the streamed dense layers (sm_100a).
//
// One persistent CTA per SM (grid = min(tiles, #SMs)), 256 threads:
//   warp 0      TMA producer: 2D tensor-map loads (128B swizzle) into a STAGES-deep smem ring
//   warp 1      MMA issuer:   one elected thread issues tcgen05.mma.cta_group::1.kind::f16
//               (bf16 x bf16 -> fp32) into a double-buffered TMEM accumulator
//   warp 2      TMEM allocator (512 columns = 2 accumulator stages)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> fused bias/ReLU, ReLU-gate or fp32 store
// Synchronisation is mbarrier-only: smem full/empty (TMA <-> MMA, tcgen05.commit frees a
// stage) and TMEM full/empty (MMA <-> epilogue), so tile t's epilogue overlaps tile t+1's
// MMAs. Operands may be K-major or MN-major (the layer's forward uses W as an N-major B, the
// dX GEMM the same W as a K-major B, the dW GEMM x^T / dz as MN-major A / B), so no
// transposes are ever materialised. Each output tile is produced by exactly one CTA with a
// fixed K order and split-K partials are reduced in a fixed order, so results depend only on
// the problem shape: bit-identical for every (k, k') window and every ring slot address.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "kernels.hpp"

namespace sp {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // bf16 elements per 128-byte swizzle row
constexpr int kThreads = 256;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int ACC_STRIDE = 256;       // TMEM columns between the two accumulator stages
constexpr int TMEM_COLS = 512;

template <int BN, bool B_MN>
struct Cfg {
    static constexpr int B_ROWS = B_MN ? ((BN + 63) / 64) * 64 : BN;
    static constexpr int B_BYTES = B_ROWS * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE_BYTES < 8 ? (200 * 1024) / STAGE_BYTES : 8;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

struct Params {
    int M, N, K;
    int m_tiles, n_tiles, k_blocks, kb_per_split, splits;
    void* out;
    int ldo;
    const float* bias;
    int relu;
    const __nv_bfloat16* gate;
    int ldg;
    long long split_stride;
    float lr;
};

// ---------------------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Shared-memory matrix descriptor (tcgen05 "smem descriptor"): start, LBO, SBO in 16-byte
// units, version 1 (sm_100), layout SWIZZLE_128B (2). Tiles are 1024-byte aligned so the
// base-offset field stays 0.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Grouped rasterisation: consecutive tile indices walk G m-blocks x every n-block, so the CTAs
// resident at any moment share their A panels (and B panels) in L2 instead of re-streaming each
// A panel from DRAM once per n-block. Only the order of tiles changes, never a tile's math.
template <int G>
__device__ __forceinline__ void tile_mn(int t, int m_tiles, int n_tiles, int& mb, int& nb) {
    const int tmn = t % (m_tiles * n_tiles);
    const int per_group = G * n_tiles;
    const int g = tmn / per_group;
    const int first = g * G;
    const int gm = min(G, m_tiles - first);
    const int r = tmn - g * per_group;
    mb = first + r % gm;
    nb = r / gm;
}

// Epilogue for 32 accumulator columns [col0, col0+32) of one output row (one TMEM lane).
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const Params& p, const uint32_t (&r)[32], int row,
                                               int col0, int split) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    if (EPI == EPI_BIAS_ACT_BF16 || EPI == EPI_BIAS_ACT_F32) {
        const float4* bp = reinterpret_cast<const float4*>(p.bias + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float4 bv = __ldg(bp + i);
            v[4 * i + 0] += bv.x;
            v[4 * i + 1] += bv.y;
            v[4 * i + 2] += bv.z;
            v[4 * i + 3] += bv.w;
        }
        if (p.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = v[i] < 0.0f ? 0.0f : v[i];
        }
    }
    if (EPI == EPI_GATE_BF16 && p.relu) {
        const uint4* gp = reinterpret_cast<const uint4*>(p.gate + static_cast<long long>(row) * p.ldg + col0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 g = __ldg(gp + i);
            const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float2 gf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[h]));
                if (gf.x <= 0.0f) v[8 * i + 2 * h] = 0.0f;
                if (gf.y <= 0.0f) v[8 * i + 2 * h + 1] = 0.0f;
            }
        }
    }
    if (EPI == EPI_BIAS_ACT_BF16 || EPI == EPI_GATE_BF16) {
        uint4* op = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) +
                                             static_cast<long long>(row) * p.ldo + col0);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            op[i] = make_uint4(pack_bf16(v[8 * i + 0], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                               pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
    } else if (EPI == EPI_SGD_F32) {
        // fused SGD (apply_sgd, model.cpp:150-155): w -= lr * dW, no FMA, in place on the
        // slot's fp32 master weights; the tile is owned by this CTA alone.
        float4* wp = reinterpret_cast<float4*>(static_cast<float*>(p.out) +
                                               static_cast<long long>(row) * p.ldo + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float4 w = wp[i];
            w.x = __fsub_rn(w.x, __fmul_rn(p.lr, v[4 * i + 0]));
            w.y = __fsub_rn(w.y, __fmul_rn(p.lr, v[4 * i + 1]));
            w.z = __fsub_rn(w.z, __fmul_rn(p.lr, v[4 * i + 2]));
            w.w = __fsub_rn(w.w, __fmul_rn(p.lr, v[4 * i + 3]));
            wp[i] = w;
        }
    } else {
        float* base = static_cast<float*>(p.out) + (EPI == EPI_F32 ? split * p.split_stride : 0LL) +
                      static_cast<long long>(row) * p.ldo + col0;
        float4* op = reinterpret_cast<float4*>(base);
#pragma unroll
        for (int i = 0; i < 8; ++i) op[i] = make_float4(v[4 * i + 0], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
}

// ---------------------------------------------------------------------------------------
// the kernel (1-CTA: M = 128 per MMA)
// ---------------------------------------------------------------------------------------
template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Params p) {
    using C = Cfg<BN, B_MN>;
    constexpr int STAGES = C::STAGES;
    constexpr uint32_t IDESC = make_idesc(BM, BN, A_MN, B_MN);
    constexpr uint32_t TX = C::STAGE_BYTES;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_mn = p.m_tiles * p.n_tiles;
    const int total = tiles_mn * p.splits;

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                int mb, nbk;
                tile_mn<16>(t, p.m_tiles, p.n_tiles, mb, nbk);
                const int m0 = mb * BM;
                const int n0 = nbk * BN;
                const int split = t / tiles_mn;
                const int kb0 = split * p.kb_per_split;
                const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], TX);
                    const int k0 = kb * BK;
                    uint8_t* a = sA + stage * A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    if (A_MN) {
                        tma_load_2d(&tmA, &full[stage], a, m0, k0);
                        tma_load_2d(&tmA, &full[stage], a + 8192, m0 + 64, k0);
                    } else {
                        tma_load_2d(&tmA, &full[stage], a, k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < C::B_ROWS / 64; ++j)
                            tma_load_2d(&tmB, &full[stage], b + j * 8192, n0 + 64 * j, k0);
                    } else {
                        tma_load_2d(&tmB, &full[stage], b, k0, n0);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer (single thread) =====
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int split = t / tiles_mn;
                const int kb0 = split * p.kb_per_split;
                const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                fence_after();
                const uint32_t d_tmem = tmem_base + acc * ACC_STRIDE;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b_base = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const uint64_t ad = A_MN ? make_desc(a_base + kk * 2048, 8192, 1024)
                                                 : make_desc(a_base + kk * 32, 16, 1024);
                        const uint64_t bd = B_MN ? make_desc(b_base + kk * 2048, 8192, 1024)
                                                 : make_desc(b_base + kk * 32, 16, 1024);
                        umma_bf16(d_tmem, ad, bd, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[stage]);  // frees the smem stage when these MMAs finish
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> fused op -> global =====
        const int q = warp & 3;  // TMEM lanes [32q, 32q+32)
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x) {
            int mb, nbk;
            tile_mn<16>(t, p.m_tiles, p.n_tiles, mb, nbk);
            const int m0 = mb * BM;
            const int n0 = nbk * BN;
            const int split = t / tiles_mn;
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            const int row = m0 + q * 32 + lane;
            const bool row_ok = row < p.M;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem_base + acc * ACC_STRIDE + c * 32 + (static_cast<uint32_t>(q * 32) << 16), r);
                const int col0 = n0 + c * 32;
                if (!row_ok || col0 >= p.N) continue;
                epilogue_chunk<EPI>(p, r, row, col0, split);
            }
            fence_before();
            mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------------------
// the kernel (2-CTA pair: tcgen05.mma.cta_group::2, M = 256 per MMA)
// ---------------------------------------------------------------------------------------
// A CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile: each CTA stages its own 128
// rows of A and its own BN/2 columns of B, the leader CTA's single MMA thread issues
// cta_group::2 MMAs that read both CTAs' shared memory, and each CTA's TMEM receives its 128
// rows x all BN columns. Per SM this halves the B bytes staged per MAC relative to the
// 1-CTA kernel (L2 -> SM traffic is what bounds the 1-CTA kernel on the layer GEMMs).
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank0(uint32_t saddr) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint64_t* bar, void* dst,
                                                 int c0, int c1) {
    // Both CTAs load; the transaction bytes complete on the LEADER's barrier (peer bit cleared).
    const uint32_t bar_addr = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_addr), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void umma2_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

template <int BN, bool A_MN, bool B_MN>
struct Cfg2 {
    static constexpr int B_ROWS = BN / 2;  // this CTA's half of the tile's N
    static constexpr int B_BYTES = B_ROWS * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE_BYTES < 8 ? (200 * 1024) / STAGE_BYTES : 8;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
    static_assert(!B_MN || B_ROWS % 64 == 0, "MN-major B halves must be whole 128B-swizzle atoms");
};

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const Params p) {
    using C = Cfg2<BN, A_MN, B_MN>;
    constexpr int STAGES = C::STAGES;
    constexpr uint32_t IDESC = make_idesc(2 * BM, BN, A_MN, B_MN);
    constexpr uint32_t TX = 2 * C::STAGE_BYTES;  // both CTAs' bytes land on the leader's barrier

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 2 * 128);  // both CTAs' epilogue threads (leader's copy used)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int m_tiles2 = (p.M + 2 * BM - 1) / (2 * BM);
    const int tiles_mn = m_tiles2 * p.n_tiles;
    const int total = tiles_mn * p.splits;
    const int cid = blockIdx.x >> 1;
    const int ncl = gridDim.x >> 1;

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer (both CTAs, each loads its own halves) =====
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < total; t += ncl) {
                int mb, nbk;
                tile_mn<8>(t, m_tiles2, p.n_tiles, mb, nbk);
                const int m0 = mb * 2 * BM + static_cast<int>(rank) * BM;
                const int nb = nbk * BN + static_cast<int>(rank) * (BN / 2);
                const int split = t / tiles_mn;
                const int kb0 = split * p.kb_per_split;
                const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&full[stage], TX);
                    const int k0 = kb * BK;
                    uint8_t* a = sA + stage * A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    if (A_MN) {
                        tma_load_2d_pair(&tmA, &full[stage], a, m0, k0);
                        tma_load_2d_pair(&tmA, &full[stage], a + 8192, m0 + 64, k0);
                    } else {
                        tma_load_2d_pair(&tmA, &full[stage], a, k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < C::B_ROWS / 64; ++j)
                            tma_load_2d_pair(&tmB, &full[stage], b + j * 8192, nb + 64 * j, k0);
                    } else {
                        tma_load_2d_pair(&tmB, &full[stage], b, k0, nb);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ===== MMA issuer: one thread of the leader CTA drives both SMs' tensor cores =====
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = cid; t < total; t += ncl) {
                const int split = t / tiles_mn;
                const int kb0 = split * p.kb_per_split;
                const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                fence_after();
                const uint32_t d_tmem = tmem_base + acc * ACC_STRIDE;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b_base = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const uint64_t ad = A_MN ? make_desc(a_base + kk * 2048, 8192, 1024)
                                                 : make_desc(a_base + kk * 32, 16, 1024);
                        const uint64_t bd = B_MN ? make_desc(b_base + kk * 2048, 8192, 1024)
                                                 : make_desc(b_base + kk * 32, 16, 1024);
                        umma2_bf16(d_tmem, ad, bd, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
                    }
                    umma2_commit_both(&empty[stage]);  // frees the stage in BOTH CTAs
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma2_commit_both(&tfull[acc]);  // both CTAs' accumulators are ready
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue (both CTAs): own 128 rows x all BN columns =====
        const int q = warp & 3;
        const uint32_t tempty_leader0 = map_to_rank0(smem_u32(&tempty[0]));
        const uint32_t tempty_leader1 = map_to_rank0(smem_u32(&tempty[1]));
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = cid; t < total; t += ncl) {
            int mb, nbk;
            tile_mn<8>(t, m_tiles2, p.n_tiles, mb, nbk);
            const int m0 = mb * 2 * BM + static_cast<int>(rank) * BM;
            const int n0 = nbk * BN;
            const int split = t / tiles_mn;
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            const int row = m0 + q * 32 + lane;
            const bool row_ok = row < p.M;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem_base + acc * ACC_STRIDE + c * 32 + (static_cast<uint32_t>(q * 32) << 16), r);
                const int col0 = n0 + c * 32;
                if (!row_ok || col0 >= p.N) continue;
                epilogue_chunk<EPI>(p, r, row, col0, split);
            }
            fence_before();
            mbar_arrive_cluster(acc == 0 ? tempty_leader0 : tempty_leader1);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }
    __syncwarp();
    fence_before();
    cluster_sync();  // no CTA leaves while its peer may still signal its barriers
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

bool encode_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                uint32_t box_inner, uint32_t box_outer);

// Tensor maps depend only on (address, shape, box): the ring slots, activation buffers and
// workspaces have fixed addresses, so each map is encoded once and reused by every step.
bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_inner, uint32_t box_outer) {
    struct Key {
        const void* base;
        uint64_t inner, outer, ld;
        uint32_t bi, bo;
        bool operator==(const Key& o) const {
            return base == o.base && inner == o.inner && outer == o.outer && ld == o.ld &&
                   bi == o.bi && bo == o.bo;
        }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            size_t h = reinterpret_cast<size_t>(k.base);
            for (uint64_t v : {k.inner, k.outer, k.ld, static_cast<uint64_t>(k.bi) << 32 | k.bo})
                h = h * 1000003u ^ static_cast<size_t>(v);
            return h;
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, CUtensorMap, Hash> cache;
    const Key key{base, inner, outer, ld, box_inner, box_outer};
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *m = it->second;
            return true;
        }
    }
    if (!encode_map(m, base, inner, outer, ld, box_inner, box_outer)) return false;
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 8192) cache.clear();
    cache.emplace(key, *m);
    return true;
}

bool encode_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                uint32_t box_inner, uint32_t box_outer) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fprintf(stderr, "superpipe: cuTensorMapEncodeTiled failed (%d): base=%p dims={%llu,%llu} ld=%llu box={%u,%u}\n",
                static_cast<int>(r), base, (unsigned long long)inner, (unsigned long long)outer,
                (unsigned long long)ld, box_inner, box_outer);
    return r == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch(const GemmProblem& g, cudaStream_t st) {
    using C = Cfg<BN, B_MN>;
    auto kern = gemm_kernel<BN, A_MN, B_MN, EPI>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    CUtensorMap ta, tb;
    bool ok = A_MN ? make_map(&ta, g.A, g.M, g.K, g.lda, 64, 64)
                   : make_map(&ta, g.A, g.K, g.M, g.lda, 64, BM);
    ok = ok && (B_MN ? make_map(&tb, g.B, g.N, g.K, g.ldb, 64, 64)
                     : make_map(&tb, g.B, g.K, g.N, g.ldb, 64, BN));
    if (!ok) return cudaErrorInvalidValue;
    Params p;
    p.M = g.M;
    p.N = g.N;
    p.K = g.K;
    p.m_tiles = (g.M + BM - 1) / BM;
    p.n_tiles = (g.N + BN - 1) / BN;
    p.k_blocks = (g.K + BK - 1) / BK;
    p.splits = g.splits < 1 ? 1 : g.splits;
    if (p.splits > p.k_blocks) p.splits = p.k_blocks;
    p.kb_per_split = (p.k_blocks + p.splits - 1) / p.splits;
    p.splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;  // no empty split
    p.out = g.out;
    p.ldo = g.ldo;
    p.bias = g.bias;
    p.relu = g.relu;
    p.gate = static_cast<const __nv_bfloat16*>(g.gate);
    p.ldg = g.ldg;
    p.split_stride = g.split_stride;
    p.lr = g.lr;
    if (EPI == EPI_SGD_F32 && p.splits != 1) return cudaErrorInvalidValue;
    const int total = p.m_tiles * p.n_tiles * p.splits;
    const int grid = total < num_sms() ? total : num_sms();
    kern<<<grid, kThreads, C::SMEM, st>>>(ta, tb, p);
    return cudaGetLastError();
}

// 2-CTA launch: BN is the pair's N (each CTA stages BN/2 columns of B); grid = 2 x clusters.
template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch2(const GemmProblem& g, cudaStream_t st) {
    using C = Cfg2<BN, A_MN, B_MN>;
    auto kern = gemm2_kernel<BN, A_MN, B_MN, EPI>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    CUtensorMap ta, tb;
    bool ok = A_MN ? make_map(&ta, g.A, g.M, g.K, g.lda, 64, 64)
                   : make_map(&ta, g.A, g.K, g.M, g.lda, 64, BM);
    ok = ok && (B_MN ? make_map(&tb, g.B, g.N, g.K, g.ldb, 64, 64)
                     : make_map(&tb, g.B, g.K, g.N, g.ldb, 64, BN / 2));
    if (!ok) return cudaErrorInvalidValue;
    Params p;
    p.M = g.M;
    p.N = g.N;
    p.K = g.K;
    p.m_tiles = (g.M + 2 * BM - 1) / (2 * BM);
    p.n_tiles = (g.N + BN - 1) / BN;
    p.k_blocks = (g.K + BK - 1) / BK;
    p.splits = g.splits < 1 ? 1 : g.splits;
    if (p.splits > p.k_blocks) p.splits = p.k_blocks;
    p.kb_per_split = (p.k_blocks + p.splits - 1) / p.splits;
    p.splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;
    p.out = g.out;
    p.ldo = g.ldo;
    p.bias = g.bias;
    p.relu = g.relu;
    p.gate = static_cast<const __nv_bfloat16*>(g.gate);
    p.ldg = g.ldg;
    p.split_stride = g.split_stride;
    p.lr = g.lr;
    if (EPI == EPI_SGD_F32 && p.splits != 1) return cudaErrorInvalidValue;
    const int total = p.m_tiles * p.n_tiles * p.splits;
    const int pairs = num_sms() / 2;
    const int grid = 2 * (total < pairs ? total : pairs);
    kern<<<grid, kThreads, C::SMEM, st>>>(ta, tb, p);
    return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_bn(const GemmProblem& g, cudaStream_t st) {
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_BF16) return launch<BN, false, true, EPI_BIAS_ACT_BF16>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_F32) return launch<BN, false, true, EPI_BIAS_ACT_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_BF16) return launch<BN, false, false, EPI_GATE_BF16>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch<BN, true, true, EPI_F32>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_SGD_F32) return launch<BN, true, true, EPI_SGD_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_F32) return launch<BN, false, false, EPI_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch<BN, false, true, EPI_F32>(g, st);
    return cudaErrorNotSupported;
}

template <int BN>
cudaError_t dispatch2_bn(const GemmProblem& g, cudaStream_t st) {
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_BF16) return launch2<BN, false, true, EPI_BIAS_ACT_BF16>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_F32) return launch2<BN, false, true, EPI_BIAS_ACT_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_BF16) return launch2<BN, false, false, EPI_GATE_BF16>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch2<BN, true, true, EPI_F32>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_SGD_F32) return launch2<BN, true, true, EPI_SGD_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_F32) return launch2<BN, false, false, EPI_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch2<BN, false, true, EPI_F32>(g, st);
    return cudaErrorNotSupported;
}

// 2-CTA tiles whose per-CTA half of N is not a whole 64-column swizzle atom (N = 192 -> 96
// per CTA) exist only for K-major B, where a CTA's B half is a plain [rows][64] TMA box.
template <int BN>
cudaError_t dispatch2_bn_kmajor(const GemmProblem& g, cudaStream_t st) {
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_BF16) return launch2<BN, false, false, EPI_GATE_BF16>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_F32) return launch2<BN, false, false, EPI_F32>(g, st);
    return cudaErrorNotSupported;
}

}  // namespace tc

// Kernel choice from a wave-quantised cost model: time ~ waves x per-SM tile work / per-SM
// rate. Relative per-SM rates calibrated on B200 (tools/gemm_bench.py, grouped rasterisation):
// 2-CTA N=256 ~0.95 (1189 TFLOP/s at 16384x1600x1600, 1568 at 65536x4096x4096), 1-CTA
// N=192/256 ~0.80; N=128 tiles (either kind) are never competitive and are not candidates.
GemmChoice choose_gemm(int M, int N, int K, int splits) {
    const int sms = num_sms();
    GemmChoice best{1, 256};
    double best_t = 1e300;
    auto consider = [&](int cta, int bn, double eff) {
        const long tiles = static_cast<long>((M + cta * tc::BM - 1) / (cta * tc::BM)) *
                           ((N + bn - 1) / bn) * splits;
        const long slots = sms / cta;
        const long waves = (tiles + slots - 1) / slots;
        const double t = static_cast<double>(waves) * tc::BM * bn / eff;  // per-SM work per wave
        if (t < best_t - 1e-9) {
            best_t = t;
            best = GemmChoice{cta, bn};
        }
    };
    consider(2, 256, 0.95);
    consider(1, 256, 0.80);
    consider(1, 192, 0.80);
    (void)K;
    return best;
}

int choose_block_n(int N) {
    // Widest tile whose padding wastes <= 10% of the columns: a 1-CTA M=128 MMA needs N >= 192
    // to keep its smem operand traffic under the ~128 B/clk/SM crossbar (measured on B200:
    // N=128 tiles reach ~620 TFLOP/s, N=192/256 ~800 on the 16384 x 1600 x 1600 layer GEMMs).
    const int cands[3] = {256, 192, 128};
    for (int bn : cands) {
        const long padded = static_cast<long>((N + bn - 1) / bn) * bn;
        if ((padded - N) * 10 <= padded) return bn;
    }
    return 128;
}

int choose_splits(int M, int N, int K, int block_n) {
    const int tiles = ((M + tc::BM - 1) / tc::BM) * ((N + block_n - 1) / block_n);
    const int kblocks = (K + tc::BK - 1) / tc::BK;
    const int sms = num_sms();
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 16 && s <= kblocks; ++s) {
        if (s > 1 && kblocks / s < 8) break;  // keep >= 512 of K per split
        const int work = tiles * s;
        const int waves = (work + sms - 1) / sms;
        // useful work per (wave x SM), discounted by the split-K reduction traffic
        const double eff = static_cast<double>(work) / (static_cast<double>(waves) * sms) *
                           (1.0 - 0.02 * (s - 1));
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = s;
        }
    }
    return best;
}

int effective_splits(int K, int splits) {
    const int kb = (K + tc::BK - 1) / tc::BK;
    int s = splits < 1 ? 1 : (splits > kb ? kb : splits);
    const int per = (kb + s - 1) / s;
    return (kb + per - 1) / per;
}

cudaError_t gemm_bf16(const GemmProblem& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaErrorInvalidValue;
    if (g.N % 32 != 0 || g.lda % 8 != 0 || g.ldb % 8 != 0) return cudaErrorInvalidValue;
    int cta = g.cta, bn = g.block_n;
    if (cta == 0) {  // auto
        const GemmChoice c = choose_gemm(g.M, g.N, g.K, g.splits < 1 ? 1 : g.splits);
        cta = c.cta;
        if (!bn) bn = c.block_n;
        if (cta == 2 && bn != 128 && bn != 256 && !(bn == 192 && !g.b_mn)) cta = 1;  // a forced tile width decides
    }
    if (!bn) bn = cta == 2 ? 256 : choose_block_n(g.N);
    if (cta == 2) {
        switch (bn) {
            case 128: return tc::dispatch2_bn<128>(g, st);
            case 256: return tc::dispatch2_bn<256>(g, st);
            case 192: return tc::dispatch2_bn_kmajor<192>(g, st);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (bn) {
        case 128: return tc::dispatch_bn<128>(g, st);
        case 192: return tc::dispatch_bn<192>(g, st);
        case 256: return tc::dispatch_bn<256>(g, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sp

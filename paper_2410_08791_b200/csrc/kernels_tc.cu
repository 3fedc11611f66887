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
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace sp {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // bf16 elements per 128-byte swizzle row
constexpr int kThreads = 256;
constexpr int A_BYTES = BM * 128;  // 16 KB: BM rows of one 128-byte swizzle row of K
constexpr int ACC_STRIDE = 256;       // TMEM columns between the two accumulator stages
constexpr int TMEM_COLS = 512;

constexpr int kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA
constexpr int kBarBytes = 512;    // mbarriers + TMEM address slot
template <int EPI>
struct EpiSmem;
// Kernel-kind bits on top of the epilogue code (GemmEpilogue, kernels.hpp): EPI_TMA = the
// epilogue stages through shared memory and stores with TMA; EPI_TF32 = operands are fp32
// and multiply as tf32 (kind::tf32) instead of bf16 (kind::f16).
constexpr int EPI_TMA = 16;
constexpr int EPI_TF32 = 32;
// Operand geometry per element type. A stage holds one 128-byte swizzle row of K per tile row
// for either type, so stage bytes, the MMA count per stage (4) and the K-major descriptor
// steps (32 bytes per MMA) are the same; MN-major tiles are cut into 128-byte-wide atoms.
template <int EPI>
struct Opnd {
    static constexpr bool TF32 = (EPI & EPI_TF32) != 0;
    static constexpr int ELT = TF32 ? 4 : 2;
    static constexpr int BKE = 128 / ELT;         // K elements per stage
    static constexpr int ATOM = 128 / ELT;        // MN elements per MN-major swizzle atom
    static constexpr int KSTEP = 32 / ELT;        // K elements per MMA
    static constexpr int ATOM_BYTES = BKE * 128;  // one MN-major atom over the stage's K rows
    static constexpr int MMAS = BKE / KSTEP;      // MMAs per stage (4)
    // MN-major smem layout: bf16 uses the 128B swizzle (16-byte granules, 8-row groups); tf32
    // must use 128B_BASE32B (32-byte granules XOR row mod 4, 4-row groups: TMA swizzle
    // 128B_ATOM_32B), so the descriptor's layout field and K-group stride differ.
    static constexpr uint32_t MN_LAYOUT = TF32 ? 1u : 2u;
    static constexpr uint32_t MN_SBO = TF32 ? 512u : 1024u;
};
// Operand ring depth: as many stages as fit beside the epilogue's staging buffers (max 8).
constexpr int ring_stages(int stage_bytes, int epi_bytes) {
    return (kSmemMax - 1024 - kBarBytes - epi_bytes) / stage_bytes < 8
               ? (kSmemMax - 1024 - kBarBytes - epi_bytes) / stage_bytes
               : 8;
}

template <int BN, bool B_MN, int EPI>
struct Cfg {
    static constexpr int ATOM = Opnd<EPI>::ATOM;
    static constexpr int B_ROWS = B_MN ? ((BN + ATOM - 1) / ATOM) * ATOM : BN;
    static constexpr int B_BYTES = B_ROWS * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BYTES = EpiSmem<EPI>::BYTES;
    static constexpr int STAGES = ring_stages(STAGE_BYTES, EPI_BYTES);
    static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + kBarBytes;
    static_assert(STAGES >= 3, "operand ring too shallow");
};

struct Params {
    int M, N, K;
    int m_tiles, n_tiles, k_blocks, kb_per_split, splits;
    void* out;
    int ldo;
    const float* bias;
    int relu;
    const void* gate;  // bf16 (EPI_GATE_BF16) or fp32 (EPI_GATE_F32)
    int ldg;
    long long split_stride;
    float lr;
    int narrow;  // 2-CTA: the ragged last N tile is computed with an MMA of N = BN/2
    int group;   // 2-CTA: m-blocks per rasterisation group (tile_mn_g)
    uint32_t* mask_out;         // EPI_BIAS_ACT_BF16: ReLU bit mask of the output (or nullptr)
    const uint32_t* gate_mask;  // EPI_GATE_BF16: gate from a bit mask (or nullptr: gate tensor)
    void* aux;                  // EPI_GELU_BF16 / EPI_SWIGLU_BF16: pre-activation output
    int ldaux;
    int act;                    // GeluKind
    float* colsum_part;         // EPI_GELU_GATE_BF16: [ceil(M/32)][N] column partials (or nullptr)
};

// Grouped rasterisation: consecutive tile indices walk G m-blocks x every n-block, so the CTAs
// resident at any moment share their A panels (and B panels) in L2 instead of re-streaming each
// A panel from DRAM once per n-block. Only the order of tiles changes, never a tile's math.
__device__ __forceinline__ void tile_mn_g(int t, int m_tiles, int n_tiles, int G, int& mb, int& nb) {
    const int tmn = t % (m_tiles * n_tiles);
    const int per_group = G * n_tiles;
    const int g = tmn / per_group;
    const int first = g * G;
    const int gm = min(G, m_tiles - first);
    const int r = tmn - g * per_group;
    mb = first + r % gm;
    nb = r / gm;
}
template <int G>
__device__ __forceinline__ void tile_mn(int t, int m_tiles, int n_tiles, int& mb, int& nb) {
    tile_mn_g(t, m_tiles, n_tiles, G, mb, nb);
}

// ---------------------------------------------------------------------------------------
// epilogue: TMEM -> registers -> fused op -> swizzled smem staging -> TMA store
// ---------------------------------------------------------------------------------------
// Each epilogue warp owns 32 accumulator rows (its TMEM lane quarter) and walks the tile in
// 32-column chunks. A lane holds one row, so writing global memory directly would touch 32
// lines per 16-byte access; instead the warp stages its 32 x 32 chunk in shared memory in the
// TMA swizzle pattern (4 wavefronts per 16-byte access, the minimum) and one lane stores it
// with cp.async.bulk.tensor (bounds-clipped by the tensor map, asynchronous, double-buffered).
// The ReLU gate of the dX GEMM comes in the same way: a TMA load of the chunk into swizzled
// smem, one chunk ahead, completed on a per-warp mbarrier. Only the fused-SGD epilogue (a
// read-modify-write of the fp32 master weights) stores from registers.
// The kernels' EPI template argument is an epilogue code (kernels.hpp) plus EPI_TMA when the
// epilogue stages through shared memory and stores with TMA (short K, where the epilogue is on
// the critical path); without it lanes store rows straight to global memory, which is smaller
// code and leaves shared memory to the operand ring (long K, where the epilogue hides).
template <int EPI>
struct EpiSmem {
    static constexpr int BASE = EPI & (EPI_TMA - 1);
    static constexpr bool TMA = (EPI & EPI_TMA) != 0 && BASE != EPI_SGD_F32;
    static constexpr bool TMA_OUT = TMA;
    static constexpr int OUT_ELT = (BASE == EPI_BIAS_ACT_BF16 || BASE == EPI_GATE_BF16 || BASE == EPI_GELU_BF16 ||
                                    BASE == EPI_GELU_GATE_BF16 || BASE == EPI_SWIGLU_BF16)
                                       ? 2
                                       : 4;
    static constexpr int OUT_BUF = 32 * 32 * OUT_ELT;  // one warp's 32 x 32 chunk
    // epilogues that read a [M][ldg] tensor tile next to the accumulator (ReLU / GELU gate, residual)
    static constexpr bool IS_GATE = BASE == EPI_GATE_BF16 || BASE == EPI_GATE_F32 || BASE == EPI_RESID_F32 ||
                                    BASE == EPI_GELU_GATE_BF16;
    static constexpr int GATE_ELT = (BASE == EPI_GATE_F32 || BASE == EPI_RESID_F32) ? 4 : 2;
    static constexpr bool GATE = TMA && IS_GATE;
    static constexpr int GATE_BUF = 32 * 32 * GATE_ELT;
    // Epilogue warps: 8 for the GELU epilogues (two per TMEM lane quarter, each half of the
    // tile's columns: their per-element math outruns 4 warps at short K), else 4.
    static constexpr int EW = (BASE == EPI_GELU_BF16 || BASE == EPI_GELU_GATE_BF16) ? 8 : 4;
    static constexpr int THREADS = 128 + 32 * EW;
    static constexpr int OUT_BYTES = TMA_OUT ? EW * 2 * OUT_BUF : 0;  // EW warps x 2 buffers
    static constexpr int GATE_BYTES = GATE ? EW * 2 * GATE_BUF : 0;
    static constexpr int BYTES = OUT_BYTES + GATE_BYTES;
};

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 16-byte chunk i of staged row r: 64-byte rows use the 64B swizzle (chunk ^ (r>>1)&3), 128-byte
// rows the 128B swizzle (chunk ^ r&7) — the layouts CU_TENSOR_MAP_SWIZZLE_64B/128B expect.
template <int ROW_BYTES>
__device__ __forceinline__ uint32_t swz(int r, int i) {
    return ROW_BYTES == 64 ? static_cast<uint32_t>(r * 64 + ((i ^ ((r >> 1) & 3)) << 4))
                           : static_cast<uint32_t>(r * 128 + ((i ^ (r & 7)) << 4));
}

// GELU (tanh approximation, GPT-2's gelu_new; or the exact erf form, ViT's nn.GELU) and its
// derivative, in fp32. The tanh is the SFU's tanh.approx.f32 (one MUFU op, max relative error
// ~2^-11, below the bf16 rounding of the stored result): the precise tanhf made the GELU
// epilogues 2.5x slower than their MMAs (ncu, GPT-2 XL FC1 / its dX).
__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Packed fp32 pairs (FFMA2 / FMUL2 on sm_100): each lane op is the same IEEE operation as its
// scalar form, so results are bitwise those of the scalar code; the instruction count halves,
// which matters for the GELU epilogues (issue slots and, under the board's power cap, energy).
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)), "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
// tanh-form GELU and its derivative on a pair: u = sqrt(2/pi) (x + 0.044715 x^3),
// gelu = 0.5 x (1 + tanh u), gelu' = 0.5 (1 + t) + 0.5 x (1 - t^2) du/dx
__device__ __forceinline__ float2 gelu2_tanh(float2 x) {
    const float2 x2 = mul2(x, x);
    const float2 u = mul2(x, fma2(f2(0.0356774081f), x2, f2(0.79788456080286536f)));
    const float2 hx = mul2(f2(0.5f), x);
    return fma2(hx, make_float2(tanh_fast(u.x), tanh_fast(u.y)), hx);
}
__device__ __forceinline__ float2 gelu_grad2_tanh(float2 x) {
    const float2 x2 = mul2(x, x);
    const float2 u = mul2(x, fma2(f2(0.0356774081f), x2, f2(0.79788456080286536f)));
    const float2 t = make_float2(tanh_fast(u.x), tanh_fast(u.y));
    const float2 du = fma2(f2(0.1070322243f), x2, f2(0.79788456080286536f));
    const float2 a = mul2(mul2(f2(0.5f), x), du);
    return fma2(a, fma2(make_float2(-t.x, -t.y), t, f2(1.0f)), fma2(f2(0.5f), t, f2(0.5f)));
}

// Exact-erf GELU (ViT's nn.GELU) on a pair. erf by Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7,
// far below the bf16 rounding of the stored result): one reciprocal and one exp2 on the SFU, and
// that exp(-x^2/2) is also the normal density in gelu'(x) = Phi(x) + x phi(x). erff + __expf
// made the ViT-H GELU epilogues ALU-bound (ncu: its dh GEMM at 930 TFLOP/s against 1420 for
// GPT-2 XL's tanh form at the same tile count).
__device__ __forceinline__ float rcp_fast(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_fast(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Phi(x) (the standard normal CDF) and e = exp(-x^2 / 2)
__device__ __forceinline__ void normal_cdf2(float2 x, float2& Phi, float2& e) {
    const float2 z = mul2(make_float2(fabsf(x.x), fabsf(x.y)), f2(0.70710678118654752f));
    const float2 d = fma2(f2(0.3275911f), z, f2(1.0f));
    const float2 t = make_float2(rcp_fast(d.x), rcp_fast(d.y));
    // the A&S coefficients halved: q = 0.5 (1 - erf(|x| / sqrt 2)) = the tail 1 - Phi(|x|)
    float2 p = fma2(f2(0.5307027145f), t, f2(-0.7265760135f));
    p = fma2(p, t, f2(0.7107068705f));
    p = fma2(p, t, f2(-0.142248368f));
    p = fma2(p, t, f2(0.127414796f));
    p = mul2(p, t);
    const float2 a = mul2(mul2(x, x), f2(-0.72134752044448170f));  // -x^2 / 2 * log2(e)
    e = make_float2(ex2_fast(a.x), ex2_fast(a.y));
    const float2 q = mul2(p, e);
    Phi = make_float2(x.x >= 0.0f ? 1.0f - q.x : q.x, x.y >= 0.0f ? 1.0f - q.y : q.y);
}
__device__ __forceinline__ float2 gelu2_erf(float2 x) {
    float2 Phi, e;
    normal_cdf2(x, Phi, e);
    return mul2(x, Phi);
}
__device__ __forceinline__ float2 gelu_grad2_erf(float2 x) {
    float2 Phi, e;
    normal_cdf2(x, Phi, e);
    return fma2(mul2(x, e), f2(0.39894228040143268f), Phi);  // Phi + x phi
}

template <int BN, int EPI>
struct TileEpilogue {
    using E = EpiSmem<EPI>;
    static constexpr int BASE = E::BASE;
    static constexpr int CHUNKS = BN / 32;
    uint8_t* obuf;    // this warp's two output staging buffers (TMA kind)
    uint8_t* gbuf;    // this warp's two gate buffers (TMA kind)
    uint64_t* gbar;   // their two mbarriers
    int lane;
    int c_begin, c_end;  // this warp's 32-column chunks of the tile
    uint32_t out_n = 0, gate_issued = 0, gate_used = 0;
    uint32_t mask_next = 0;  // ReLU bit-mask word of the next chunk (loaded one chunk ahead)

    // e: epilogue warp index (0 .. EW-1); lane quarter e % 4, column half e / 4 when EW == 8
    __device__ __forceinline__ TileEpilogue(uint8_t* epi_smem, uint64_t* gate_bars, int e, int ln)
        : obuf(epi_smem + e * 2 * E::OUT_BUF),
          gbuf(epi_smem + E::OUT_BYTES + e * 2 * E::GATE_BUF),
          gbar(gate_bars + 2 * e),
          lane(ln),
          c_begin(E::EW == 8 ? (e / 4) * (CHUNKS / 2) : 0),
          c_end(E::EW == 8 ? (e / 4 + 1) * (CHUNKS / 2) : CHUNKS) {}

    __device__ __forceinline__ void gate_issue(const CUtensorMap* tmG, int row0, int col0) {
        const int b = gate_issued & 1;
        __syncwarp();  // every lane is done reading this buffer's previous chunk
        if (lane == 0) {
            mbar_expect_tx(&gbar[b], E::GATE_BUF);
            tma_load_2d(tmG, &gbar[b], gbuf + b * E::GATE_BUF, col0, row0);
        }
        ++gate_issued;
    }
    static constexpr bool kMaskGate = E::IS_GATE;
    // The gate / residual tensor is read for this tile: always for the residual and GELU-gate
    // epilogues, for the ReLU gates only when gating from the tensor (not a bit mask).
    __device__ __forceinline__ static bool tensor_gate(const Params& p) {
        return (BASE == EPI_RESID_F32 || BASE == EPI_GELU_GATE_BF16) ? true : (p.relu && !p.gate_mask);
    }
    __device__ __forceinline__ uint32_t mask_word(const Params& p, int row, int col0) const {
        return row < p.M && col0 < p.N ? __ldg(p.gate_mask + static_cast<long long>(col0 / 32) * p.M + row) : 0u;
    }
    // before the accumulator wait: the gate of the tile's first chunk starts loading
    __device__ __forceinline__ void begin_tile(const CUtensorMap* tmG, const Params& p, int row0, int n0) {
        const int c0 = n0 + c_begin * 32;
        if (E::GATE && tensor_gate(p) && c0 < p.N) gate_issue(tmG, row0, c0);
        if (kMaskGate && p.relu && p.gate_mask) mask_next = mask_word(p, row0 + lane, c0);
    }

    // This lane's row of the chunk's gate tensor as fp32: from the TMA-staged smem buffer, or
    // (direct kind) from global memory; false when the row is past M (direct kind only).
    __device__ __forceinline__ bool gate_f32(const Params& p, int row, int col0, float (&g)[32]) {
        if (E::GATE) {
            const int b = gate_used & 1;
            mbar_wait(&gbar[b], (gate_used >> 1) & 1);
            ++gate_used;
            const uint8_t* gb = gbuf + b * E::GATE_BUF;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float4 f = *reinterpret_cast<const float4*>(gb + swz<128>(lane, i));
                g[4 * i] = f.x, g[4 * i + 1] = f.y, g[4 * i + 2] = f.z, g[4 * i + 3] = f.w;
            }
            return true;
        }
        if (row >= p.M) return false;
        const float4* gp = reinterpret_cast<const float4*>(static_cast<const float*>(p.gate) +
                                                           static_cast<long long>(row) * p.ldg + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float4 f = __ldg(gp + i);
            g[4 * i] = f.x, g[4 * i + 1] = f.y, g[4 * i + 2] = f.z, g[4 * i + 3] = f.w;
        }
        return true;
    }
    __device__ __forceinline__ bool gate_bf16(const Params& p, int row, int col0, float (&g)[32]) {
        uint4 gv[4];
        if (E::GATE) {
            const int b = gate_used & 1;
            mbar_wait(&gbar[b], (gate_used >> 1) & 1);
            ++gate_used;
            const uint8_t* gb = gbuf + b * E::GATE_BUF;
#pragma unroll
            for (int i = 0; i < 4; ++i) gv[i] = *reinterpret_cast<const uint4*>(gb + swz<64>(lane, i));
        } else {
            if (row >= p.M) return false;
            const uint4* gp = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.gate) +
                                                             static_cast<long long>(row) * p.ldg + col0);
#pragma unroll
            for (int i = 0; i < 4; ++i) gv[i] = __ldg(gp + i);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t gw[4] = {gv[i].x, gv[i].y, gv[i].z, gv[i].w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float2 gf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gw[h]));
                g[8 * i + 2 * h] = gf.x;
                g[8 * i + 2 * h + 1] = gf.y;
            }
        }
        return true;
    }
    __device__ __forceinline__ static void add_bias(const Params& p, int col0, float (&v)[32]) {
        if (!p.bias) return;
        const float4* bp = reinterpret_cast<const float4*>(p.bias + col0);  // one address per warp
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float4 bv = __ldg(bp + i);
            v[4 * i + 0] += bv.x;
            v[4 * i + 1] += bv.y;
            v[4 * i + 2] += bv.z;
            v[4 * i + 3] += bv.w;
        }
    }
    // 32 bf16 values of this lane's row straight to global memory (the pre-activation side
    // output: four 16-byte stores covering two full 32-byte sectors each).
    __device__ __forceinline__ static void store_row_bf16(void* base, int ld, int row, int col0, const uint32_t (&pk)[16]) {
        uint4* op = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + static_cast<long long>(row) * ld + col0);
#pragma unroll
        for (int i = 0; i < 4; ++i) op[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
    }

    // Stores the chunk's final values: packed bf16 (pk) or fp32 (v), per-lane rows or staged
    // through shared memory and one TMA store (col0 = the output column of the chunk).
    __device__ __forceinline__ void store_out(const CUtensorMap* tmO, const Params& p, const float (&v)[32],
                                              const uint32_t (&pk)[16], int row0, int col0, int split) {
        const int row = row0 + lane;
        if (!E::TMA_OUT) {  // per-lane row stores straight to global
            if (row >= p.M) return;
            if (E::OUT_ELT == 2) {
                store_row_bf16(p.out, p.ldo, row, col0, pk);
            } else {
                float4* op = reinterpret_cast<float4*>(static_cast<float*>(p.out) +
                                                       (BASE == EPI_F32 ? split * p.split_stride : 0LL) +
                                                       static_cast<long long>(row) * p.ldo + col0);
#pragma unroll
                for (int i = 0; i < 8; ++i) op[i] = make_float4(v[4 * i + 0], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            }
        } else {  // swizzled smem staging -> one TMA store per 32 x 32 chunk
            uint8_t* ob = obuf + (out_n & 1) * E::OUT_BUF;
            if (lane == 0) bulk_wait_read<1>();  // the store that last read this buffer is done
            __syncwarp();
            if (E::OUT_ELT == 2) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    *reinterpret_cast<uint4*>(ob + swz<64>(lane, i)) =
                        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    *reinterpret_cast<float4*>(ob + swz<128>(lane, i)) =
                        make_float4(v[4 * i + 0], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            }
            fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA (async proxy)
            __syncwarp();
            if (lane == 0) {
                if (BASE == EPI_F32) tma_store_3d(tmO, ob, col0, row0, split);
                else tma_store_2d(tmO, ob, col0, row0);
                bulk_commit();
            }
            ++out_n;
        }
    }

    // Column sums of the warp's 32 x 32 chunk (rows past M count as 0) into the 32-row group's
    // partial row: a lane-order reduce-scatter (31 shuffles) leaves column l's sum in lane l.
    __device__ __forceinline__ void colsum_chunk(const Params& p, const float (&v)[32], int row0, int col0, bool in) const {
        float a[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] = in ? v[i] : 0.0f;
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
        const int col = col0 + lane;
        if (col < p.N) p.colsum_part[static_cast<long long>(row0 / 32) * p.N + col] = a[0];
    }

    __device__ __forceinline__ void chunk(const CUtensorMap* tmO, const Params& p, const uint32_t (&r)[32],
                                          int row0, int col0, int split, uint32_t gate_bits) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        const int row = row0 + lane;
        if (BASE == EPI_BIAS_ACT_BF16 || BASE == EPI_BIAS_ACT_F32) {
            add_bias(p, col0, v);
            if (p.relu) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = v[i] < 0.0f ? 0.0f : v[i];
            }
        }
        if (BASE == EPI_GELU_BF16) {
            // pre-activation h = acc + b (bf16 side output for the backward's GELU'), out = gelu(h)
            add_bias(p, col0, v);
            uint32_t hk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) hk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
            if (row < p.M && p.aux) store_row_bf16(p.aux, p.ldaux, row, col0, hk);
            if (p.act == GELU_ERF) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float2 y = gelu2_erf(make_float2(v[2 * i], v[2 * i + 1]));
                    v[2 * i] = y.x, v[2 * i + 1] = y.y;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float2 y = gelu2_tanh(make_float2(v[2 * i], v[2 * i + 1]));
                    v[2 * i] = y.x, v[2 * i + 1] = y.y;
                }
            }
        }
        if (E::IS_GATE && p.relu && p.gate_mask != nullptr) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (!((gate_bits >> i) & 1u)) v[i] = 0.0f;
        } else if (BASE == EPI_GATE_F32 && p.relu) {  // fp32 gate tensor (tf32 path)
            float g[32];
            if (!gate_f32(p, row, col0, g)) return;
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (g[i] <= 0.0f) v[i] = 0.0f;
        } else if (BASE == EPI_GATE_BF16 && p.relu) {
            float g[32];
            if (!gate_bf16(p, row, col0, g)) return;
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (g[i] <= 0.0f) v[i] = 0.0f;
        } else if (BASE == EPI_RESID_F32) {  // out = acc + b + residual (fp32 residual stream)
            float g[32];
            add_bias(p, col0, v);
            if (!gate_f32(p, row, col0, g)) return;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += g[i];
        } else if (BASE == EPI_GELU_GATE_BF16) {  // dh = dg * gelu'(h)
            float g[32];
            const bool ok = gate_bf16(p, row, col0, g);  // (false: a row past M, direct kind)
            if (ok) {
                if (p.act == GELU_ERF) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float2 y = mul2(make_float2(v[2 * i], v[2 * i + 1]),
                                              gelu_grad2_erf(make_float2(g[2 * i], g[2 * i + 1])));
                        v[2 * i] = y.x, v[2 * i + 1] = y.y;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float2 y = mul2(make_float2(v[2 * i], v[2 * i + 1]),
                                              gelu_grad2_tanh(make_float2(g[2 * i], g[2 * i + 1])));
                        v[2 * i] = y.x, v[2 * i + 1] = y.y;
                    }
                }
            }
            if (p.colsum_part) colsum_chunk(p, v, row0, col0, ok && row < p.M);  // (every lane)
            if (!ok) return;
        }
        if (BASE == EPI_SGD_F32) {
            // fused SGD (apply_sgd, model.cpp:150-155): w -= lr * dW, no FMA, in place on the
            // slot's fp32 master weights; the tile is owned by this CTA alone.
            if (row < p.M) {
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
            }
            return;
        }
        uint32_t pk[16];  // the stored bf16 values, two per word
        if (E::OUT_ELT == 2) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
            if (BASE == EPI_BIAS_ACT_BF16 && p.relu && p.mask_out != nullptr && row < p.M) {
                // ReLU bit mask of the stored values: after ReLU a value is +-0, > 0 or NaN, so
                // !(x <= 0) is exactly "magnitude bits nonzero" — the dX gate's keep test
                uint32_t bits = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    bits |= ((pk[i] & 0x7FFFu) ? 1u : 0u) << (2 * i) | ((pk[i] & 0x7FFF0000u) ? 1u : 0u) << (2 * i + 1);
                p.mask_out[static_cast<long long>(col0 / 32) * p.M + row] = bits;  // a warp: 128 B
            }
        } else if (BASE == EPI_BIAS_ACT_F32 && p.relu && p.mask_out != nullptr && row < p.M) {
            // fp32 output (tf32 path): the same rule on the stored fp32 values
            uint32_t bits = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) bits |= ((__float_as_uint(v[i]) & 0x7FFFFFFFu) ? 1u : 0u) << i;
            p.mask_out[static_cast<long long>(col0 / 32) * p.M + row] = bits;
        }
        store_out(tmO, p, v, pk, row0, col0, split);
    }

    // SwiGLU: chunk 2c holds the gate pre-activations g, chunk 2c+1 the up projections u of the
    // same 32 hidden units; out[:, n0/2 + 32c ..] = silu(g) * u, aux = both pre-activations.
    __device__ __forceinline__ void chunk_swiglu(const CUtensorMap* tmO, const Params& p, const uint32_t (&rg)[32],
                                                 const uint32_t (&ru)[32], int row0, int col0) {
        const int row = row0 + lane;
        float v[32];
        uint32_t pk[16];
        if (p.aux && row < p.M) {  // col0 = colg / 2 with colg (the gate chunk's column) % 64 == 0
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(rg[2 * i]), __uint_as_float(rg[2 * i + 1]));
            store_row_bf16(p.aux, p.ldaux, row, 2 * col0, pk);
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(ru[2 * i]), __uint_as_float(ru[2 * i + 1]));
            store_row_bf16(p.aux, p.ldaux, row, 2 * col0 + 32, pk);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const float g = __uint_as_float(rg[i]), u = __uint_as_float(ru[i]);
            v[i] = g / (1.0f + __expf(-g)) * u;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
        store_out(tmO, p, v, pk, row0, col0, 0);
    }

    // One accumulator tile: chunk by chunk out of TMEM; the accumulator stage is released to the
    // MMA warp once every chunk is in registers or stored.
    template <typename Release>
    __device__ __forceinline__ void run(const CUtensorMap* tmO, const CUtensorMap* tmG, const Params& p,
                                        uint32_t tmem_acc, int row0, int n0, int split, Release&& release) {
        uint32_t ra[32];
        if (BASE == EPI_SWIGLU_BF16) {
            uint32_t rb[32];
#pragma unroll 1
            for (int c = 0; c < CHUNKS / 2; ++c) {
                tmem_ld32_async(tmem_acc + (2 * c) * 32, ra);
                tmem_ld_wait(ra);
                tmem_ld32_async(tmem_acc + (2 * c + 1) * 32, rb);
                tmem_ld_wait(rb);
                const int colg = n0 + 2 * c * 32;  // gate column in the GEMM's N
                if (colg < p.N) chunk_swiglu(tmO, p, ra, rb, row0, colg / 2);
            }
            release();
            return;
        }
#pragma unroll 1
        for (int c = c_begin; c < c_end; ++c) {
            const int col0 = n0 + c * 32;
            tmem_ld32_async(tmem_acc + c * 32, ra);
            tmem_ld_wait(ra);
            if (E::GATE && tensor_gate(p) && c + 1 < c_end && col0 + 32 < p.N)
                gate_issue(tmG, row0, col0 + 32);
            const uint32_t mask_cur = mask_next;
            if (kMaskGate && p.relu && p.gate_mask && c + 1 < c_end)
                mask_next = mask_word(p, row0 + lane, col0 + 32);
            if (col0 < p.N) chunk(tmO, p, ra, row0, col0, split, mask_cur);
        }
        release();
    }
    __device__ __forceinline__ void finish() {
        if (E::TMA_OUT && lane == 0) bulk_wait_all();
        __syncwarp();
    }
};

template <bool TF32>
__device__ __forceinline__ void umma1_if(uint32_t leader, uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    if (TF32)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 e, %5, 0;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(leader));
    else
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 e, %5, 0;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(leader));
}
// ---------------------------------------------------------------------------------------
// the kernel (1-CTA: M = 128 per MMA)
// ---------------------------------------------------------------------------------------
template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(EpiSmem<EPI>::THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmG,
                const Params p) {
    using C = Cfg<BN, B_MN, EPI>;
    using O = Opnd<EPI>;
    constexpr int STAGES = C::STAGES;
    constexpr uint32_t IDESC = make_idesc(BM, BN, A_MN, B_MN, O::TF32);
    constexpr uint32_t TX = C::STAGE_BYTES;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint8_t* sE = sB + STAGES * C::B_BYTES;  // epilogue staging (1024-aligned)
    uint64_t* full = reinterpret_cast<uint64_t*>(sE + C::EPI_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* gbar = tempty + 2;  // 4 epilogue warps x 2 gate buffers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbar + 16);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        if (EpiSmem<EPI>::TMA_OUT) prefetch_tmap(&tmO);
        if (EpiSmem<EPI>::GATE) prefetch_tmap(&tmG);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 32 * EpiSmem<EPI>::EW);
        }
        for (int s = 0; s < 16; ++s) mbar_init(&gbar[s], 1);
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
                    const int k0 = kb * O::BKE;
                    uint8_t* a = sA + stage * A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    if (A_MN) {
#pragma unroll
                        for (int j = 0; j < BM / O::ATOM; ++j)
                            tma_load_2d(&tmA, &full[stage], a + j * O::ATOM_BYTES, m0 + O::ATOM * j, k0);
                    } else {
                        tma_load_2d(&tmA, &full[stage], a, k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < C::B_ROWS / O::ATOM; ++j)
                            tma_load_2d(&tmB, &full[stage], b + j * O::ATOM_BYTES, n0 + O::ATOM * j, k0);
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
        {
            // ===== MMA issuer: the whole warp runs the loop, the elected lane issues =====
            const uint32_t leader = elect_one();
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
                    for (int kk = 0; kk < O::MMAS; ++kk) {
                        // MN-major: the next KSTEP rows of every 128-byte atom; K-major: the next
                        // 32 bytes of each swizzled row
                        const uint64_t ad = A_MN ? make_desc(a_base + kk * O::KSTEP * 128, O::ATOM_BYTES, O::MN_SBO, O::MN_LAYOUT)
                                                 : make_desc(a_base + kk * 32, 16, 1024);
                        const uint64_t bd = B_MN ? make_desc(b_base + kk * O::KSTEP * 128, O::ATOM_BYTES, O::MN_SBO, O::MN_LAYOUT)
                                                 : make_desc(b_base + kk * 32, 16, 1024);
                        umma1_if<O::TF32>(leader, d_tmem, ad, bd, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit_if(leader, &empty[stage]);  // frees the smem stage when these MMAs finish
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_if(leader, &tfull[acc]);  // accumulator ready for the epilogue
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> fused op -> smem -> TMA store =====
        const int q = warp & 3;  // TMEM lanes [32q, 32q+32)
        TileEpilogue<BN, EPI> ep(sE, gbar, warp - 4, lane);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x) {
            int mb, nbk;
            tile_mn<16>(t, p.m_tiles, p.n_tiles, mb, nbk);
            const int row0 = mb * BM + q * 32;
            const int n0 = nbk * BN;
            const int split = t / tiles_mn;
            ep.begin_tile(&tmG, p, row0, n0);
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            uint64_t* te = &tempty[acc];
            ep.run(&tmO, &tmG, p, tmem_base + acc * ACC_STRIDE + (static_cast<uint32_t>(q * 32) << 16), row0,
                   n0, split, [&] {
                       fence_before();
                       mbar_arrive(te);
                   });
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        ep.finish();
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
// Predicated forms for a warp-uniform issuer (only `leader`, from elect.sync, executes them).
template <bool TF32>
__device__ __forceinline__ void umma2_if(uint32_t leader, uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    if (TF32)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 e, %5, 0;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(leader));
    else
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 e, %5, 0;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(leader));
}
__device__ __forceinline__ void umma2_commit_both_if(uint32_t leader, uint64_t* bar) {
    const uint16_t mask = 0x3;
    asm volatile(
        "{\n\t.reg .pred e;\n\tsetp.ne.b32 e, %2, 0;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"(mask), "r"(leader)
        : "memory");
}
template <bool TF32>
__device__ __forceinline__ void umma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                      uint32_t idesc, uint32_t accumulate) {
    if (TF32)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
    else
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

// Tile schedule of a CTA pair (2-CTA kernel). Full tiles are dealt round-robin; when the last
// N tile is ragged (N mod 256 <= 128) it is computed at half width (half the MMA work), and
// those half tiles go first to the pairs that got one full tile fewer - twice each, since two
// halves make one full tile - then round-robin. This is the largest-first (LPT) assignment for
// tiles of cost 1 and 1/2: at 16384 x 1600 the busiest pair does 6.0 tile-times instead of 7.
// Which pair computes a tile never changes the tile's arithmetic.
struct PairSched {
    int U, u, F, R, r, mt, ntf, nt, per_split, group;
    __device__ __forceinline__ PairSched(const Params& p, int m_tiles2, int cid, int ncl) {
        mt = m_tiles2;
        group = p.group;
        nt = p.n_tiles;
        ntf = p.narrow ? nt - 1 : nt;
        per_split = mt * ntf;
        F = per_split * p.splits;
        R = p.narrow ? mt * p.splits : 0;
        U = ncl;
        u = cid;
        r = F % U;
    }
    // i-th tile of this pair; false when the pair is done.
    __device__ __forceinline__ bool get(int i, int& mb, int& nb, int& split, bool& narrow) const {
        const int nfull = u < F ? (F - 1 - u) / U + 1 : 0;
        if (i < nfull) {
            const int t = u + U * i;
            split = t / per_split;
            tile_mn_g(t - split * per_split, mt, ntf, group, mb, nb);
            narrow = false;
            return true;
        }
        const int k = i - nfull;
        const int lo = U - r;
        const int j = u >= r ? (k < 2 ? (u - r) + k * lo : 2 * lo + u + U * (k - 2)) : 2 * lo + u + U * k;
        if (j >= R) return false;
        split = j / mt;
        mb = j - split * mt;
        nb = nt - 1;
        narrow = true;
        return true;
    }
};

template <int BN, bool A_MN, bool B_MN, int EPI>
struct Cfg2 {
    static constexpr int B_ROWS = BN / 2;  // this CTA's half of the tile's N
    static constexpr int B_BYTES = B_ROWS * 128;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BYTES = EpiSmem<EPI>::BYTES;
    static constexpr int STAGES = ring_stages(STAGE_BYTES, EPI_BYTES);
    static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + kBarBytes;
    static_assert(STAGES >= 3, "operand ring too shallow");
    static_assert(!B_MN || B_ROWS % Opnd<EPI>::ATOM == 0, "MN-major B halves must be whole 128B-swizzle atoms");
};

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(EpiSmem<EPI>::THREADS, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmG,
                 const Params p) {
    using C = Cfg2<BN, A_MN, B_MN, EPI>;
    using O = Opnd<EPI>;
    constexpr int STAGES = C::STAGES;
    constexpr uint32_t IDESC = make_idesc(2 * BM, BN, A_MN, B_MN, O::TF32);
    constexpr uint32_t TX = 2 * C::STAGE_BYTES;  // both CTAs' bytes land on the leader's barrier

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint8_t* sE = sB + STAGES * C::B_BYTES;  // epilogue staging (1024-aligned)
    uint64_t* full = reinterpret_cast<uint64_t*>(sE + C::EPI_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* gbar = tempty + 2;  // 4 epilogue warps x 2 gate buffers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbar + 16);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        if (EpiSmem<EPI>::TMA_OUT) prefetch_tmap(&tmO);
        if (EpiSmem<EPI>::GATE) prefetch_tmap(&tmG);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 2 * 32 * EpiSmem<EPI>::EW);  // both CTAs' epilogue threads (leader's copy)
        }
        for (int s = 0; s < 16; ++s) mbar_init(&gbar[s], 1);
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
    const PairSched sched(p, m_tiles2, blockIdx.x >> 1, gridDim.x >> 1);
    constexpr uint32_t IDESC_NARROW = make_idesc(2 * BM, BN / 2, A_MN, B_MN, O::TF32);

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer (both CTAs, each loads its own halves) =====
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0;; ++i) {
                int mb, nbk, split;
                bool nar;
                if (!sched.get(i, mb, nbk, split, nar)) break;
                // this CTA's share of the tile's N: BN/2 columns, or BN/4 of a half-width tile
                const int half = nar ? BN / 4 : BN / 2;
                const int m0 = mb * 2 * BM + static_cast<int>(rank) * BM;
                const int nb = nbk * BN + static_cast<int>(rank) * half;
                const uint32_t tx =
                    B_MN ? 2u * static_cast<uint32_t>(A_BYTES + (half / O::ATOM) * O::ATOM_BYTES) : TX;
                const int kb0 = split * p.kb_per_split;
                const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&full[stage], tx);
                    const int k0 = kb * O::BKE;
                    uint8_t* a = sA + stage * A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    if (A_MN) {
#pragma unroll
                        for (int j = 0; j < BM / O::ATOM; ++j)
                            tma_load_2d_pair(&tmA, &full[stage], a + j * O::ATOM_BYTES, m0 + O::ATOM * j, k0);
                    } else {
                        tma_load_2d_pair(&tmA, &full[stage], a, k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < C::B_ROWS / O::ATOM; ++j)
                            if (j * O::ATOM < half)
                                tma_load_2d_pair(&tmB, &full[stage], b + j * O::ATOM_BYTES, nb + O::ATOM * j, k0);
                    } else {
                        tma_load_2d_pair(&tmB, &full[stage], b, k0, nb);  // full box; MMA reads `half` rows
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            // ===== MMA issuer: the leader CTA's warp runs the loop, its elected lane drives both SMs' tensor cores =====
            const uint32_t elect = elect_one();
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int i = 0;; ++i) {
                int mb, nbk, split;
                bool nar;
                if (!sched.get(i, mb, nbk, split, nar)) break;
                const uint32_t idesc = nar ? IDESC_NARROW : IDESC;
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
                    for (int kk = 0; kk < O::MMAS; ++kk) {
                        const uint64_t ad = A_MN ? make_desc(a_base + kk * O::KSTEP * 128, O::ATOM_BYTES, O::MN_SBO, O::MN_LAYOUT)
                                                 : make_desc(a_base + kk * 32, 16, 1024);
                        const uint64_t bd = B_MN ? make_desc(b_base + kk * O::KSTEP * 128, O::ATOM_BYTES, O::MN_SBO, O::MN_LAYOUT)
                                                 : make_desc(b_base + kk * 32, 16, 1024);
                        umma2_if<O::TF32>(elect, d_tmem, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
                    }
                    umma2_commit_both_if(elect, &empty[stage]);  // frees the stage in BOTH CTAs
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma2_commit_both_if(elect, &tfull[acc]);  // both CTAs' accumulators are ready
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue (both CTAs): own 128 rows x all BN columns =====
        const int q = warp & 3;
        const uint32_t tempty_leader0 = map_to_rank0(smem_u32(&tempty[0]));
        const uint32_t tempty_leader1 = map_to_rank0(smem_u32(&tempty[1]));
        TileEpilogue<BN, EPI> ep(sE, gbar, warp - 4, lane);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            int mb, nbk, split;
            bool nar;
            if (!sched.get(i, mb, nbk, split, nar)) break;
            const int row0 = mb * 2 * BM + static_cast<int>(rank) * BM + q * 32;
            const int n0 = nbk * BN;  // a half-width tile's dead columns are >= N: never stored
            ep.begin_tile(&tmG, p, row0, n0);
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            const uint32_t te = acc == 0 ? tempty_leader0 : tempty_leader1;
            ep.run(&tmO, &tmG, p, tmem_base + acc * ACC_STRIDE + (static_cast<uint32_t>(q * 32) << 16), row0,
                   n0, split, [&] {
                       fence_before();
                       mbar_arrive_cluster(te);
                   });
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        ep.finish();
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

// A tensor map description: element type, rank (2 or 3), dims / byte strides / box, swizzle.
struct MapDesc {
    CUtensorMapDataType dtype;
    int rank;
    const void* base;
    uint64_t dims[3];
    uint64_t strides[2];  // bytes, dims 1..rank-1
    uint32_t box[3];
    CUtensorMapSwizzle swizzle;
    bool operator==(const MapDesc& o) const {
        return dtype == o.dtype && rank == o.rank && base == o.base && swizzle == o.swizzle &&
               std::memcmp(dims, o.dims, sizeof(dims)) == 0 &&
               std::memcmp(strides, o.strides, sizeof(strides)) == 0 &&
               std::memcmp(box, o.box, sizeof(box)) == 0;
    }
};
struct MapDescHash {
    size_t operator()(const MapDesc& k) const {
        size_t h = reinterpret_cast<size_t>(k.base) ^ (static_cast<size_t>(k.dtype) << 48) ^
                   (static_cast<size_t>(k.swizzle) << 56) ^ static_cast<size_t>(k.rank);
        for (uint64_t v : {k.dims[0], k.dims[1], k.dims[2], k.strides[0], k.strides[1],
                           static_cast<uint64_t>(k.box[0]) << 32 | k.box[1], static_cast<uint64_t>(k.box[2])})
            h = h * 1000003u ^ static_cast<size_t>(v);
        return h;
    }
};

bool encode(CUtensorMap* m, const MapDesc& k) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {k.dims[0], k.dims[1], k.dims[2]};
    cuuint64_t strides[2] = {k.strides[0], k.strides[1]};
    cuuint32_t box[3] = {k.box[0], k.box[1], k.box[2]};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, k.dtype, k.rank, const_cast<void*>(k.base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, k.swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fprintf(stderr, "superpipe: cuTensorMapEncodeTiled failed (%d): base=%p rank=%d dims={%llu,%llu,%llu} box={%u,%u,%u}\n",
                static_cast<int>(r), k.base, k.rank, (unsigned long long)k.dims[0],
                (unsigned long long)k.dims[1], (unsigned long long)k.dims[2], k.box[0], k.box[1], k.box[2]);
    return r == CUDA_SUCCESS;
}

// Tensor maps depend only on (address, shape, box, type): the ring slots, activation buffers and
// workspaces have fixed addresses, so each map is encoded once and reused by every step.
bool make_map(CUtensorMap* m, const MapDesc& k) {
    static std::mutex mu;
    static std::unordered_map<MapDesc, CUtensorMap, MapDescHash> cache;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(k);
        if (it != cache.end()) {
            *m = it->second;
            return true;
        }
    }
    if (!encode(m, k)) return false;
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 8192) cache.clear();
    cache.emplace(k, *m);
    return true;
}

// Operand [outer][ld] (inner contiguous; bf16, or fp32 for tf32), 128B-swizzled box
// {box_inner, box_outer}
bool make_map_sw32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                   uint32_t box_inner, uint32_t box_outer) {
    MapDesc k{};
    k.dtype = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    k.rank = 2;
    k.base = base;
    k.dims[0] = inner;
    k.dims[1] = outer;
    k.dims[2] = 1;
    k.strides[0] = ld * 2;
    k.box[0] = box_inner;
    k.box[1] = box_outer;
    k.box[2] = 1;
    k.swizzle = CU_TENSOR_MAP_SWIZZLE_32B;
    return make_map(m, k);
}
bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_inner, uint32_t box_outer, bool f32, bool base32) {
    MapDesc k{};
    k.dtype = f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    k.rank = 2;
    k.base = base;
    k.dims[0] = inner;
    k.dims[1] = outer;
    k.dims[2] = 1;
    k.strides[0] = ld * (f32 ? 4 : 2);
    k.box[0] = box_inner;
    k.box[1] = box_outer;
    k.box[2] = 1;
    k.swizzle = base32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
    return make_map(m, k);
}

// The epilogue's maps: output (bf16 / fp32, a 3-D {N, M, split} map for split-K partials so the
// TMA clips every split at M) and the dX GEMM's ReLU gate, with 32 x 32 boxes in the swizzle
// the staging code writes (64B for 64-byte bf16 rows, 128B for 128-byte fp32 rows).
template <int EPI>
bool make_epilogue_maps(const GemmProblem& g, int splits, CUtensorMap* to, CUtensorMap* tg) {
    using E = EpiSmem<EPI>;
    std::memset(to, 0, sizeof(*to));
    std::memset(tg, 0, sizeof(*tg));
    if (E::TMA_OUT) {
        MapDesc k{};
        k.dtype = E::OUT_ELT == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        k.base = g.out;
        k.dims[0] = static_cast<uint64_t>(E::BASE == EPI_SWIGLU_BF16 ? g.N / 2 : g.N);
        k.dims[1] = static_cast<uint64_t>(g.M);
        k.strides[0] = static_cast<uint64_t>(g.ldo) * E::OUT_ELT;
        k.box[0] = 32;
        k.box[1] = 32;
        k.box[2] = 1;
        k.swizzle = E::OUT_ELT == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
        if (E::BASE == EPI_F32) {
            k.rank = 3;
            k.dims[2] = static_cast<uint64_t>(splits);
            k.strides[1] = static_cast<uint64_t>(g.split_stride) * 4;
        } else {
            k.rank = 2;
            k.dims[2] = 1;
        }
        if (!make_map(to, k)) return false;
    }
    const bool tensor_gate = (E::BASE == EPI_RESID_F32 || E::BASE == EPI_GELU_GATE_BF16) || (g.relu && !g.gate_mask);
    if (E::GATE && tensor_gate) {
        MapDesc k{};
        k.dtype = E::GATE_ELT == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        k.rank = 2;
        k.base = g.gate;
        k.dims[0] = static_cast<uint64_t>(g.N);
        k.dims[1] = static_cast<uint64_t>(g.M);
        k.dims[2] = 1;
        k.strides[0] = static_cast<uint64_t>(g.ldg) * E::GATE_ELT;
        k.box[0] = 32;
        k.box[1] = 32;
        k.box[2] = 1;
        k.swizzle = E::GATE_ELT == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
        if (!make_map(tg, k)) return false;
    }
    return true;
}

// A/B knobs (sp_debug_set): epilogue kind 0 auto / 1 direct / 2 TMA; half-width ragged tiles
// for every epilogue (1) or the split-K partials only (0, the product choice).
int g_epi_mode = 0;
int g_narrow = 0;
int g_raster = 0;  // CTA-pair rasterisation group, 0 = by shape (debug knob "raster")
int g_dw_split_max = 0;  // cap on choose_dw's split count, 0 = none (debug knob "dw_split_max")

// Epilogue kind: TMA staging for every epilogue but the fused SGD. At short K the epilogue is on
// the critical path (+8..15% on the d=1280/1600 layer GEMMs, ncu, fixed clocks). At long K the
// direct per-lane stores (half-used 32-byte sectors) were ~5% faster at fixed clocks (d=4096),
// but the step runs at the board's power cap, where the TMA kind's whole-sector stores measured
// even to slightly ahead (GPT-2 XL step 189.2 -> 188.4 ms, tools/block_ab.py epi_mode; Llama-3
// QKV 2.51 -> 2.46 ms, tools/llama_gemm_probe.py).
// sp_debug_set("epi_mode", 1|2) forces direct/TMA (A/B measurement only).
bool use_tma_epilogue(const GemmProblem& g, int splits) {
    const int forced = g_epi_mode;
    if (g.epilogue == EPI_SGD_F32) return false;
    if (forced == 1) return false;
    if (forced == 2) return true;
    (void)splits;
    return true;
}

// Half-width last N tiles (PairSched) pay only for the split-K fp32 partials of dW (+5%, ncu):
// for the activation GEMMs they were neutral warm and, being scheduled last, re-read every A
// panel after it has left L2 (82 vs 58 MB DRAM reads per forward launch at 16384 x 1600).
bool narrow_tiles(int epi_base, int bn, int last_cols) {
    if (g_narrow == 1)  // every epilogue (A/B measurement only)
        return epi_base != EPI_SGD_F32 && bn == 256 && last_cols <= 128;
    return epi_base == EPI_F32 && bn == 256 && last_cols <= 128;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch(const GemmProblem& g, cudaStream_t st) {
    using C = Cfg<BN, B_MN, EPI>;
    auto kern = gemm_kernel<BN, A_MN, B_MN, EPI>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    using O = Opnd<EPI>;
    CUtensorMap ta, tb;
    bool ok = A_MN ? make_map(&ta, g.A, g.M, g.K, g.lda, O::ATOM, O::BKE, O::TF32, O::TF32)
                   : make_map(&ta, g.A, g.K, g.M, g.lda, O::BKE, BM, O::TF32, false);
    ok = ok && (B_MN ? make_map(&tb, g.B, g.N, g.K, g.ldb, O::ATOM, O::BKE, O::TF32, O::TF32)
                     : make_map(&tb, g.B, g.K, g.N, g.ldb, O::BKE, BN, O::TF32, false));
    if (!ok) return cudaErrorInvalidValue;
    Params p;
    p.M = g.M;
    p.N = g.N;
    p.K = g.K;
    p.m_tiles = (g.M + BM - 1) / BM;
    p.n_tiles = (g.N + BN - 1) / BN;
    p.k_blocks = (g.K + O::BKE - 1) / O::BKE;
    p.splits = g.splits < 1 ? 1 : g.splits;
    if (p.splits > p.k_blocks) p.splits = p.k_blocks;
    p.kb_per_split = (p.k_blocks + p.splits - 1) / p.splits;
    p.splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;  // no empty split
    p.out = g.out;
    p.ldo = g.ldo;
    p.bias = g.bias;
    p.relu = g.relu;
    p.gate = g.gate;
    p.ldg = g.ldg;
    p.split_stride = g.split_stride;
    p.lr = g.lr;
    p.narrow = 0;
    p.mask_out = g.mask_out;
    p.gate_mask = g.gate_mask;
    p.aux = g.aux;
    p.ldaux = g.ldaux;
    p.act = g.act;
    p.colsum_part = g.colsum_part;
    if ((EPI & (EPI_TMA - 1)) == EPI_SGD_F32 && p.splits != 1) return cudaErrorInvalidValue;
    if (g.colsum_part && p.splits != 1) return cudaErrorInvalidValue;
    CUtensorMap to, tg;
    if (!make_epilogue_maps<EPI>(g, p.splits, &to, &tg)) return cudaErrorInvalidValue;
    const int total = p.m_tiles * p.n_tiles * p.splits;
    const int grid = total < num_sms() ? total : num_sms();
    kern<<<dim3(grid), dim3(EpiSmem<EPI>::THREADS), C::SMEM, st>>>(ta, tb, to, tg, p);
    return cudaGetLastError();
}

// 2-CTA launch: BN is the pair's N (each CTA stages BN/2 columns of B); grid = 2 x clusters.
template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch2(const GemmProblem& g, cudaStream_t st) {
    using C = Cfg2<BN, A_MN, B_MN, EPI>;
    auto kern = gemm2_kernel<BN, A_MN, B_MN, EPI>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    using O = Opnd<EPI>;
    CUtensorMap ta, tb;
    bool ok = A_MN ? make_map(&ta, g.A, g.M, g.K, g.lda, O::ATOM, O::BKE, O::TF32, O::TF32)
                   : make_map(&ta, g.A, g.K, g.M, g.lda, O::BKE, BM, O::TF32, false);
    ok = ok && (B_MN ? make_map(&tb, g.B, g.N, g.K, g.ldb, O::ATOM, O::BKE, O::TF32, O::TF32)
                     : make_map(&tb, g.B, g.K, g.N, g.ldb, O::BKE, BN / 2, O::TF32, false));
    if (!ok) return cudaErrorInvalidValue;
    Params p;
    p.M = g.M;
    p.N = g.N;
    p.K = g.K;
    p.m_tiles = (g.M + 2 * BM - 1) / (2 * BM);
    p.n_tiles = (g.N + BN - 1) / BN;
    p.k_blocks = (g.K + O::BKE - 1) / O::BKE;
    p.splits = g.splits < 1 ? 1 : g.splits;
    if (p.splits > p.k_blocks) p.splits = p.k_blocks;
    p.kb_per_split = (p.k_blocks + p.splits - 1) / p.splits;
    p.splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;
    p.out = g.out;
    p.ldo = g.ldo;
    p.bias = g.bias;
    p.relu = g.relu;
    p.gate = g.gate;
    p.ldg = g.ldg;
    p.split_stride = g.split_stride;
    p.lr = g.lr;
    p.mask_out = g.mask_out;
    p.gate_mask = g.gate_mask;
    p.aux = g.aux;
    p.ldaux = g.ldaux;
    p.act = g.act;
    p.colsum_part = g.colsum_part;
    if (g.colsum_part && p.splits != 1) return cudaErrorInvalidValue;
    {
        const int last = g.N - (p.n_tiles - 1) * BN;  // columns in the last N tile
        p.narrow = narrow_tiles(EPI & (EPI_TMA - 1), BN, last) ? 1 : 0;
    }
    // m-blocks per rasterisation group: each group streams the whole B (weight) matrix once, so
    // a B too large to stay in L2 (> 64 MB: Llama-3-8B's gate/up 235 MB, down 117 MB) takes 16
    // and is re-read from DRAM half as often; the lower DRAM power lets the clock rise under the
    // 1000 W cap (SwiGLU gate/up 12.9-13.3 -> 12.0 ms, tools/llama_gemm_probe.py; C3 881-928 ->
    // 841 ms). Smaller B stays in L2 either way and 8 keeps the A panels' footprint small
    // (16 measured 0.5% slower on GPT-2 XL's step and 3% on ViT-H's, tools/block_ab.py).
    const double b_bytes = static_cast<double>(g.N) * g.K * O::ELT;
    p.group = g_raster > 0 ? g_raster : (b_bytes > 64e6 ? 16 : 8);
    if ((EPI & (EPI_TMA - 1)) == EPI_SGD_F32 && p.splits != 1) return cudaErrorInvalidValue;
    CUtensorMap to, tg;
    if (!make_epilogue_maps<EPI>(g, p.splits, &to, &tg)) return cudaErrorInvalidValue;
    const int total = p.m_tiles * p.n_tiles * p.splits;
    const int pairs = num_sms() / 2;
    const int grid = 2 * (total < pairs ? total : pairs);
    kern<<<dim3(grid), dim3(EpiSmem<EPI>::THREADS), C::SMEM, st>>>(ta, tb, to, tg, p);
    return cudaGetLastError();
}

// Picks the epilogue kind at run time; each kind is its own kernel instantiation.
template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch_k(const GemmProblem& g, cudaStream_t st) {
    return use_tma_epilogue(g, g.splits < 1 ? 1 : g.splits) ? launch<BN, A_MN, B_MN, EPI | EPI_TMA>(g, st)
                                                             : launch<BN, A_MN, B_MN, EPI>(g, st);
}
template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch2_k(const GemmProblem& g, cudaStream_t st) {
    return use_tma_epilogue(g, g.splits < 1 ? 1 : g.splits) ? launch2<BN, A_MN, B_MN, EPI | EPI_TMA>(g, st)
                                                             : launch2<BN, A_MN, B_MN, EPI>(g, st);
}

template <int BN>
cudaError_t dispatch_bn(const GemmProblem& g, cudaStream_t st) {
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_BF16) return launch_k<BN, false, true, EPI_BIAS_ACT_BF16>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_F32) return launch_k<BN, false, true, EPI_BIAS_ACT_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_BF16) return launch_k<BN, false, false, EPI_GATE_BF16>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch_k<BN, true, true, EPI_F32>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_SGD_F32) return launch_k<BN, true, true, EPI_SGD_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_F32) return launch_k<BN, false, false, EPI_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch_k<BN, false, true, EPI_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_RESID_F32) return launch_k<BN, false, true, EPI_RESID_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_GELU_BF16) return launch_k<BN, false, true, EPI_GELU_BF16>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_SWIGLU_BF16) return launch_k<BN, false, true, EPI_SWIGLU_BF16>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GELU_GATE_BF16) return launch_k<BN, false, false, EPI_GELU_GATE_BF16>(g, st);
    return cudaErrorNotSupported;
}

template <int BN>
cudaError_t dispatch2_bn(const GemmProblem& g, cudaStream_t st) {
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_BF16) return launch2_k<BN, false, true, EPI_BIAS_ACT_BF16>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_F32) return launch2_k<BN, false, true, EPI_BIAS_ACT_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_BF16) return launch2_k<BN, false, false, EPI_GATE_BF16>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch2_k<BN, true, true, EPI_F32>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_SGD_F32) return launch2_k<BN, true, true, EPI_SGD_F32>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_F32) return launch2_k<BN, false, false, EPI_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch2_k<BN, false, true, EPI_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_RESID_F32) return launch2_k<BN, false, true, EPI_RESID_F32>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_GELU_BF16) return launch2_k<BN, false, true, EPI_GELU_BF16>(g, st);
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_SWIGLU_BF16) return launch2_k<BN, false, true, EPI_SWIGLU_BF16>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GELU_GATE_BF16) return launch2_k<BN, false, false, EPI_GELU_GATE_BF16>(g, st);
    return cudaErrorNotSupported;
}

// tf32 instantiations (SP_NUMERICS_TF32): the layer GEMMs only - forward (fp32 out + mask),
// dX (fp32 out, gated), dW (fp32 partials or fused SGD) - at N = 256 (pair) / 128, 256 (1-CTA).
template <int BN>
cudaError_t dispatch_bn_tf32(const GemmProblem& g, cudaStream_t st) {
    constexpr int T = EPI_TF32;
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_F32) return launch_k<BN, false, true, EPI_BIAS_ACT_F32 | T>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_F32) return launch_k<BN, false, false, EPI_GATE_F32 | T>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch_k<BN, true, true, EPI_F32 | T>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_SGD_F32) return launch_k<BN, true, true, EPI_SGD_F32 | T>(g, st);
    return cudaErrorNotSupported;
}
template <int BN>
cudaError_t dispatch2_bn_tf32(const GemmProblem& g, cudaStream_t st) {
    constexpr int T = EPI_TF32;
    if (!g.a_mn && g.b_mn && g.epilogue == EPI_BIAS_ACT_F32) return launch2_k<BN, false, true, EPI_BIAS_ACT_F32 | T>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_F32) return launch2_k<BN, false, false, EPI_GATE_F32 | T>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_F32) return launch2_k<BN, true, true, EPI_F32 | T>(g, st);
    if (g.a_mn && g.b_mn && g.epilogue == EPI_SGD_F32) return launch2_k<BN, true, true, EPI_SGD_F32 | T>(g, st);
    return cudaErrorNotSupported;
}

// 2-CTA tiles whose per-CTA half of N is not a whole 64-column swizzle atom (N = 192 -> 96,
// N = 160 -> 80 per CTA) exist only for K-major B, where a CTA's B half is a plain [rows][64] TMA box.
template <int BN>
cudaError_t dispatch2_bn_kmajor(const GemmProblem& g, cudaStream_t st) {
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_GATE_BF16) return launch2_k<BN, false, false, EPI_GATE_BF16>(g, st);
    if (!g.a_mn && !g.b_mn && g.epilogue == EPI_F32) return launch2_k<BN, false, false, EPI_F32>(g, st);
    return cudaErrorNotSupported;
}

}  // namespace tc

extern int g_attn_fwd_kind;  // kernels_attn.cu
extern int g_attn_bwd_kind;
extern int g_attn_trace;
extern int g_attn_chunk;

void set_gemm_debug(const char* key, int value, bool* known) {
    *known = true;
    if (std::strcmp(key, "epi_mode") == 0) tc::g_epi_mode = value;
    else if (std::strcmp(key, "attn_fwd") == 0) g_attn_fwd_kind = value;
    else if (std::strcmp(key, "attn_bwd") == 0) g_attn_bwd_kind = value;
    else if (std::strcmp(key, "attn_trace") == 0) g_attn_trace = value;
    else if (std::strcmp(key, "attn_chunk") == 0) g_attn_chunk = value;
    else if (std::strcmp(key, "narrow") == 0) tc::g_narrow = value;
    else if (std::strcmp(key, "raster") == 0) tc::g_raster = value;
    else if (std::strcmp(key, "dw_split_max") == 0) tc::g_dw_split_max = value;
    else *known = false;
}

// Kernel choice from a wave-quantised cost model: time ~ waves x per-SM tile work / per-SM
// rate. Relative per-SM rates calibrated on B200 (tools/gemm_bench.py, grouped rasterisation):
// 2-CTA N=256 ~0.95 (1189 TFLOP/s at 16384x1600x1600, 1568 at 65536x4096x4096), 1-CTA
// N=192/256 ~0.80; N=128 tiles (either kind) are never competitive and are not candidates.
// Busiest CTA pair's work, in full-tile units, under PairSched (kernels above): F full tiles
// round-robin, R half-width tiles largest-first.
double pair_max_load(long F, long R, long U) {
    const long q = F / U, r = F % U, lo = U - r;
    double worst = 0.0;
    for (long u = 0; u < U; ++u) {
        long halves = 0;
        if (u >= r) halves += (u - r < R) + (u - r + lo < R);
        const long first = 2 * lo + u;  // then every U-th half tile
        if (first < R) halves += (R - 1 - first) / U + 1;
        const double load = static_cast<double>(q + (u < r ? 1 : 0)) + 0.5 * static_cast<double>(halves);
        worst = load > worst ? load : worst;
    }
    return worst;
}

GemmChoice choose_gemm(int M, int N, int K, int splits, int epilogue, bool b_kmajor) {
    const int sms = num_sms();
    GemmChoice best{1, 256};
    double best_t = 1e300;
    auto consider = [&](int cta, int bn, double eff) {
        const long mt = (M + cta * tc::BM - 1) / (cta * tc::BM);
        const long nt = (N + bn - 1) / bn;
        const long tiles = mt * nt * splits;
        const long slots = sms / cta;
        double waves = static_cast<double>((tiles + slots - 1) / slots);
        if (cta == 2 && tc::narrow_tiles(epilogue, bn, N - (nt - 1) * bn)) {  // half-width last N tile
            const long R = mt * splits, F = tiles - R;
            waves = pair_max_load(F, R, tiles < slots ? tiles : slots);
        }
        const double t = waves * tc::BM * bn / eff;  // per-SM work of the busiest SM
        if (t < best_t - 1e-9) {
            best_t = t;
            best = GemmChoice{cta, bn};
        }
    };
    consider(2, 256, 0.95);
    // CTA-pair N=192 tiles (K-major B, bf16 / fp32 stores): at N = d = 1600 nine whole-ish tiles
    // beat seven 256-wide ones with a ragged last tile (tools/bn_probe.py, 16384 rows: 4-12%
    // faster at K = 1600 / 4800 / 6400; N = 160, ten exact tiles, lands between the two)
    if (b_kmajor && (epilogue == EPI_GATE_BF16 || epilogue == EPI_F32)) consider(2, 192, 0.96);
    consider(1, 256, 0.80);
    consider(1, 192, 0.80);
    (void)K;
    return best;
}

// dW = x^T dz kernel choice, jointly over the variant and the split-K count: the busiest SM's
// work (LPT load in tiles x tile width x K blocks per split) / calibrated per-SM rate, plus 2.5%
// per extra split for the fp32 partial traffic. Calibrated on B200 (tools/dw_split_probe.py):
// 16384 rows x d=1600 -> CTA pair, N=256, 3 splits (72.9 us, 1150 TFLOP/s; was 1-CTA N=192 with
// 5 splits, 82.6 us); 65792 x 1280 -> pair, 256, 5 splits (161 us, 1337 TFLOP/s).
// splits = 1 with fused_ok means the SGD is fused into the epilogue (no partials).
DwChoice choose_dw(int M, int N, int K, int max_splits, bool fused_ok, bool tf32) {
    if (tc::g_dw_split_max > 0 && max_splits > tc::g_dw_split_max) max_splits = tc::g_dw_split_max;
    const int sms = num_sms();
    const int bke = tf32 ? tc::BK / 2 : tc::BK;  // K elements per k-block
    const int kb = (K + bke - 1) / bke;
    DwChoice best{2, 256, 1};
    double best_t = 1e300;
    struct Cand {
        int cta, bn;
        double eff;
    };
    for (const Cand c : {Cand{2, 256, 0.95}, Cand{1, 256, 0.80}, Cand{1, 192, 0.80}, Cand{1, 128, 0.62}}) {
        if (tf32 && c.bn == 192) continue;  // not instantiated for tf32
        for (int s = 1; s <= 16 && s <= max_splits && s <= kb; ++s) {
            if (s > 1 && kb * bke / s < 512) break;  // keep >= 512 of K per split
            if (effective_splits(K, s, tf32) != s) continue;
            const long mt = (M + c.cta * tc::BM - 1) / (c.cta * tc::BM);
            const long nt = (N + c.bn - 1) / c.bn;
            const long tiles = mt * nt * s, slots = sms / c.cta;
            double load = static_cast<double>((tiles + slots - 1) / slots);
            const bool partials = s > 1 || !fused_ok;
            if (c.cta == 2 && partials && tc::narrow_tiles(EPI_F32, c.bn, N - static_cast<int>(nt - 1) * c.bn)) {
                const long R = mt * s;
                load = pair_max_load(tiles - R, R, tiles < slots ? tiles : slots);
            }
            const double t = load * c.bn * ((kb + s - 1) / s) / c.eff * (1.0 + 0.025 * (s - 1));
            if (t < best_t - 1e-9) {
                best_t = t;
                best = DwChoice{c.cta, c.bn, s};
            }
        }
    }
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

int effective_splits(int K, int splits, bool tf32) {
    const int bke = tf32 ? tc::BK / 2 : tc::BK;
    const int kb = (K + bke - 1) / bke;
    int s = splits < 1 ? 1 : (splits > kb ? kb : splits);
    const int per = (kb + s - 1) / s;
    return (kb + per - 1) / per;
}

cudaError_t gemm_bf16(const GemmProblem& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaErrorInvalidValue;
    const int align = g.tf32 ? 4 : 8;  // 16-byte rows for TMA
    if (g.N % 32 != 0 || g.lda % align != 0 || g.ldb % align != 0) return cudaErrorInvalidValue;
    if (g.epilogue == EPI_SWIGLU_BF16 && (g.N % 64 != 0 || (g.block_n && g.block_n % 64 != 0)))
        return cudaErrorInvalidValue;  // whole (gate, up) chunk pairs per tile
    if (g.tf32) {
        int cta = g.cta, bn = g.block_n;
        if (cta == 0) {
            const GemmChoice c = choose_gemm(g.M, g.N, g.K, g.splits < 1 ? 1 : g.splits, g.epilogue);
            cta = c.cta;
            if (!bn) bn = c.block_n == 192 ? 256 : c.block_n;
        }
        if (!bn) bn = 256;
        if (cta == 2 && bn == 256) return tc::dispatch2_bn_tf32<256>(g, st);
        if (cta == 1 && bn == 256) return tc::dispatch_bn_tf32<256>(g, st);
        if (cta == 1 && bn == 128) return tc::dispatch_bn_tf32<128>(g, st);
        return cudaErrorInvalidValue;
    }
    int cta = g.cta, bn = g.block_n;
    if (cta == 0) {  // auto
        const GemmChoice c = choose_gemm(g.M, g.N, g.K, g.splits < 1 ? 1 : g.splits, g.epilogue, !g.b_mn);
        cta = c.cta;
        if (!bn) bn = c.block_n;
        if (cta == 2 && bn != 128 && bn != 256 && !((bn == 192 || bn == 160) && !g.b_mn)) cta = 1;  // a forced tile width decides
    }
    if (!bn) bn = cta == 2 ? 256 : choose_block_n(g.N);
    if (cta == 2) {
        switch (bn) {
            case 128: return tc::dispatch2_bn<128>(g, st);
            case 256: return tc::dispatch2_bn<256>(g, st);
            case 192: return tc::dispatch2_bn_kmajor<192>(g, st);
            case 160: return tc::dispatch2_bn_kmajor<160>(g, st);
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

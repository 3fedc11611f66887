"""Kernel-level parity of the named-shape transformer blocks' CUDA kernels against plain
PyTorch fp32 references of the same ops (bf16-rounded operands, fp32 math), on the B200.

Shapes include the bench workload's exact GEMMs (GPT-2 XL layer at 16 x 1024 tokens:
d = 1600, ff = 6400, 25 heads of 64) and the ViT-H/14 / Llama-3 attention geometries.
Tolerances are relative to the reference's max magnitude and stated per check; bf16 outputs
carry one bf16 rounding (2^-8 relative) on top of fp32 accumulation-order differences.
"""
import ctypes as C
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
EPI_BIAS_ACT_BF16, EPI_BIAS_ACT_F32, EPI_GATE_BF16, EPI_F32 = 0, 1, 2, 3
EPI_RESID_F32, EPI_GELU_BF16, EPI_GELU_GATE_BF16, EPI_SWIGLU_BF16 = 6, 7, 8, 9


def _stream():
    return torch.cuda.current_stream().cuda_stream


def gemm(M, N, K, A, lda, a_mn, B, ldb, b_mn, epi, out, ldo, bias=None, relu=0, gate=None, ldg=0,
         splits=1, aux=None, ldaux=0, act=0, cta=0, block_n=0, colsum=None):
    a = _capi.GemmArgs(M, N, K, A.data_ptr(), lda, a_mn, B.data_ptr(), ldb, b_mn, epi, out.data_ptr(), ldo,
                       bias.data_ptr() if bias is not None else None, relu,
                       gate.data_ptr() if gate is not None else None, ldg, splits, block_n, cta,
                       aux.data_ptr() if aux is not None else None, ldaux, act, _stream(),
                       colsum.data_ptr() if colsum is not None else None)
    rc = LIB.sp_debug_gemm_ex(C.byref(a))
    assert rc == 0, rc
    torch.cuda.synchronize()


def rel(got, ref):
    got, ref = got.float(), ref.float()
    return float((got - ref).abs().max() / ref.abs().max().clamp_min(1e-30))


def bf(t):
    return t.to(torch.bfloat16)


def gelu_ref(x, erf):
    return torch.nn.functional.gelu(x, approximate="none" if erf else "tanh")


@pytest.fixture(autouse=True)
def _seed():
    torch.manual_seed(1234)


# (rows, in, out): the GPT-2 XL block's four linears at the bench batch, plus a ragged case
FWD_SHAPES = [(16384, 1600, 4800), (16384, 1600, 1600), (16384, 1600, 6400), (16384, 6400, 1600),
              (1000, 256, 320)]


@pytest.mark.parametrize("T,K,N", FWD_SHAPES)
def test_bias_and_residual_epilogues(T, K, N):
    x = bf(torch.randn(T, K, device="cuda"))
    W = bf(torch.randn(K, N, device="cuda") / math.sqrt(K))
    b = torch.randn(N, device="cuda")
    res = torch.randn(T, N, device="cuda")
    ref = x.float() @ W.float() + b
    # plain bias, bf16 out (the QKV projection)
    o16 = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    gemm(T, N, K, x, K, 0, W, N, 1, EPI_BIAS_ACT_BF16, o16, N, bias=b)
    assert rel(o16, ref) < 1e-2
    # no bias (Llama projections)
    gemm(T, N, K, x, K, 0, W, N, 1, EPI_BIAS_ACT_BF16, o16, N, bias=None)
    assert rel(o16, x.float() @ W.float()) < 1e-2
    # residual add into the fp32 stream (attention out-projection / MLP down-projection)
    o32 = torch.empty(T, N, device="cuda")
    gemm(T, N, K, x, K, 0, W, N, 1, EPI_RESID_F32, o32, N, bias=b, gate=res, ldg=N)
    assert rel(o32, ref + res) < 5e-5


@pytest.mark.parametrize("erf", [0, 1])
@pytest.mark.parametrize("T,K,N", [(16384, 1600, 6400), (4096, 1280, 5120), (1000, 256, 320)])
def test_gelu_epilogue_and_its_gate(T, K, N, erf):
    x = bf(torch.randn(T, K, device="cuda"))
    W = bf(torch.randn(K, N, device="cuda") / math.sqrt(K))
    b = torch.randn(N, device="cuda") * 0.1
    h = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    g = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    gemm(T, N, K, x, K, 0, W, N, 1, EPI_GELU_BF16, g, N, bias=b, aux=h, ldaux=N, act=erf)
    pre = x.float() @ W.float() + b
    assert rel(h, pre) < 1e-2
    # the activation is applied to the fp32 accumulator, before rounding
    assert rel(g, gelu_ref(pre, erf)) < 1e-2
    # backward of the MLP's down projection: dg = dy W2^T gated by gelu'(h), W2 = [N][K]
    dy = bf(torch.randn(T, K, device="cuda"))
    W2 = bf(torch.randn(N, K, device="cuda") / math.sqrt(N))
    dh = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    parts = torch.full(((T + 31) // 32, N), float("nan"), device="cuda")
    gemm(T, N, K, dy, K, 0, W2, K, 0, EPI_GELU_GATE_BF16, dh, N, gate=h, ldg=N, act=erf, colsum=parts)
    hv = h.float().requires_grad_(True)
    gelu_ref(hv, erf).sum().backward()
    ref = (dy.float() @ W2.float().t()) * hv.grad
    assert rel(dh, ref) < 1e-2
    # the fused column sums (the b1 gradient) per 32-row group: every group written, and their
    # total equals the column sums of the output (fp32 sums of the unrounded values)
    assert torch.isfinite(parts).all()
    assert rel(parts.double().sum(0), ref.double().sum(0)) < 2e-3
    assert rel(parts.double().sum(0), dh.double().sum(0)) < 2e-3


@pytest.mark.parametrize("T,K,FF", [(8192, 4096, 1024), (1000, 256, 320)])
def test_swiglu_epilogue(T, K, FF):
    x = bf(torch.randn(T, K, device="cuda"))
    W = bf(torch.randn(K, 2 * FF, device="cuda") / math.sqrt(K))  # interleaved 32-col gate/up chunks
    out = torch.empty(T, FF, device="cuda", dtype=torch.bfloat16)
    aux = torch.empty(T, 2 * FF, device="cuda", dtype=torch.bfloat16)
    gemm(T, 2 * FF, K, x, K, 0, W, 2 * FF, 1, EPI_SWIGLU_BF16, out, FF, aux=aux, ldaux=2 * FF)
    acc = x.float() @ W.float()
    c = acc.view(T, FF // 32, 2, 32)
    gate, up = c[:, :, 0, :].reshape(T, FF), c[:, :, 1, :].reshape(T, FF)
    assert rel(out, torch.nn.functional.silu(gate) * up) < 1e-2
    assert rel(aux, acc) < 1e-2


@pytest.mark.parametrize("T,N,K", [(16384, 1600, 4800), (16384, 1600, 6400), (16384, 1600, 1600)])
def test_dx_fp32_out(T, N, K):
    # dX of the block's input-side linears: dxn = dqkv Wqkv^T (fp32 for the norm backward)
    dz = bf(torch.randn(T, K, device="cuda"))
    W = bf(torch.randn(N, K, device="cuda") / math.sqrt(K))  # W [in = N][out = K]: K-major B
    o = torch.empty(T, N, device="cuda")
    gemm(T, N, K, dz, K, 0, W, K, 0, EPI_F32, o, N)
    assert rel(o, dz.float() @ W.float().t()) < 5e-5


@pytest.mark.parametrize("M,N,T", [(1600, 4800, 16384), (6400, 1600, 16384), (1600, 1600, 16384)])
def test_dw_split_k_partials(M, N, T):
    # dW = x^T dy with the executor's variant choice and split count for the shape
    x = bf(torch.randn(T, M, device="cuda"))
    dy = bf(torch.randn(T, N, device="cuda") * 1e-2)
    cta, bn = C.c_int32(), C.c_int32()
    splits = 4
    parts = torch.empty(splits * M * N, device="cuda")
    gemm(M, N, T, x, M, 1, dy, N, 1, EPI_F32, parts, N, splits=splits)
    eff = LIB.sp_debug_effective_splits(T, splits)
    got = parts.view(splits, M, N)[:eff].sum(0)
    ref = (x.double().t() @ dy.double()).float()
    assert rel(got, ref) < 1e-4  # fp32 accumulation over K = 16384 (bf16 rounding would be 4e-3)


def attn_ref(q, k, v, causal, group):
    # q [B,H,S,hd], k/v [B,Hkv,S,hd]; fp32 math
    k = k.repeat_interleave(group, dim=1)
    v = v.repeat_interleave(group, dim=1)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(q.shape[-1])
    if causal:
        S = q.shape[2]
        s = s.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1), float("-inf"))
    p = torch.softmax(s, -1)
    return p @ v, torch.logsumexp(s, -1)


ATTN = [  # (batch, S, H, Hkv, hd, causal)
    (2, 1024, 4, 4, 64, 1),     # GPT-2 XL head geometry (25 heads in the model)
    (3, 257, 2, 2, 80, 0),      # ViT-H/14: 257 tokens, head dim 80, bidirectional
    (2, 256, 8, 2, 128, 1),     # Llama-3 GQA: 4 q heads per kv head, head dim 128
    (1, 100, 2, 1, 64, 1),      # ragged
    (2, 256, 2, 2, 64, 0),      # bidirectional, whole 128-row blocks (the tcgen05 backward)
    (1, 384, 4, 4, 128, 0),
    (3, 64, 2, 2, 64, 1),       # one 64-key step per sequence (the dQ pass issues a single S)
    (2, 65, 4, 4, 80, 0),       # short ragged head_dim 80 (the block tests' ViT-like spec)
]


def _split(qkv, B, S, H, Hkv, hd):
    t = qkv.float().view(B, S, H + 2 * Hkv, hd).permute(0, 2, 1, 3)
    return t[:, :H], t[:, H:H + Hkv], t[:, H + Hkv:]


@pytest.mark.parametrize("fwd_kind,bwd_kind", [(0, 0), (2, 0), (3, 2), (1, 1)],
                         ids=["tcgen05", "tcgen05-fwd-v2", "tcgen05-v1", "mma-sync"])
@pytest.mark.parametrize("B,S,H,Hkv,hd,causal", ATTN)
def test_attention_forward_and_backward(B, S, H, Hkv, hd, causal, fwd_kind, bwd_kind):
    # forward kind 0: the default (v3 tcgen05: O accumulated in TMEM, lazy rescale), 2: v2 (O in
    # registers), 3: v1 (4 softmax warps), 1: mma.sync. Backward kind 0:
    # the v2 tcgen05 passes (dQ + delta, then dK/dV; any sequence length), 2: the v1
    # tcgen05 passes, 1: mma.sync; shapes a tcgen05 kind does not cover take the mma.sync kernels
    assert LIB.sp_debug_set(None, b"attn_fwd", fwd_kind) == 0
    assert LIB.sp_debug_set(None, b"attn_bwd", bwd_kind) == 0
    T, W = B * S, (H + 2 * Hkv) * hd
    qkv = bf(torch.randn(T, W, device="cuda"))
    o = torch.empty(T, H * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    st = _stream()
    rc = LIB.sp_debug_attention(0, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                None, None, None, st)
    assert rc == 0
    torch.cuda.synchronize()
    q, k, v = (t.detach().requires_grad_(True) for t in _split(qkv, B, S, H, Hkv, hd))
    ref, lse_ref = attn_ref(q, k, v, causal, H // Hkv)
    got = o.float().view(B, S, H, hd).permute(0, 2, 1, 3)
    assert rel(got, ref) < 1.5e-2
    # lse is kept in log2 units of the scaled scores
    assert float((lse.view(B, H, S) * math.log(2) - lse_ref).abs().max()) < 1e-3
    # backward against autograd (dO random; the kernel reads o and lse from the forward)
    dout = bf(torch.randn(T, H * hd, device="cuda"))
    dqkv = torch.zeros(T, W, device="cuda", dtype=torch.bfloat16)
    delta = torch.empty(B * H * S, device="cuda")
    rc = LIB.sp_debug_attention(1, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                dout.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), st)
    assert rc == 0
    torch.cuda.synchronize()
    ref.backward(dout.float().view(B, S, H, hd).permute(0, 2, 1, 3))
    dq, dk, dv = _split(dqkv, B, S, H, Hkv, hd)
    for got_g, ref_g in ((dq, q.grad), (dk, k.grad), (dv, v.grad)):
        assert rel(got_g, ref_g) < 2e-2
    LIB.sp_debug_set(None, b"attn_fwd", 0)
    LIB.sp_debug_set(None, b"attn_bwd", 0)


def test_gemm_tile_order_and_store_kind_change_nothing():
    """The CTA-pair rasterisation group (by shape: 8, or 16 for weights over 64 MB) and the
    epilogue's store kind (TMA staging, or direct per-lane stores) reorder tiles and stores only:
    a residual-epilogue forward and a split-K dW are bitwise the same under every setting."""
    T, K, N = 4096, 1600, 1600
    x = bf(torch.randn(T, K, device="cuda"))
    w = bf(torch.randn(K, N, device="cuda") * 0.02)
    b = torch.randn(N, device="cuda")
    res = torch.randn(T, N, device="cuda")
    dy = bf(torch.randn(T, N, device="cuda") * 1e-2)
    outs = []
    for raster, epi_mode in ((0, 0), (1, 0), (16, 0), (0, 1), (0, 2)):
        assert LIB.sp_debug_set(None, b"raster", raster) == 0
        assert LIB.sp_debug_set(None, b"epi_mode", epi_mode) == 0
        y = torch.empty(T, N, device="cuda")
        gemm(T, N, K, x, K, 0, w, N, 1, EPI_RESID_F32, y, N, bias=b, gate=res, ldg=N)
        parts = torch.empty(3 * K * N, device="cuda")
        gemm(K, N, T, x, K, 1, dy, N, 1, EPI_F32, parts, N, splits=3, cta=2, block_n=256)
        outs.append((y, parts))
    LIB.sp_debug_set(None, b"raster", 0)
    LIB.sp_debug_set(None, b"epi_mode", 0)
    for y, parts in outs[1:]:
        assert torch.equal(y, outs[0][0]) and torch.equal(parts, outs[0][1])


def test_attention_causal_work_order_changes_nothing():
    """The causal kernels' chunked (sequence, head) work order (attn_chunk; taken by shape when
    K / V outgrow L2) only reorders whole tiles: forward and backward outputs are bitwise those
    of the plain longest-first order, including a last chunk smaller than the others."""
    B, S, H, Hkv, hd = 5, 256, 4, 2, 128  # 20 (sequence, head) pairs: chunks of 3 leave 2
    T, W = B * S, (H + 2 * Hkv) * hd
    qkv = bf(torch.randn(T, W, device="cuda"))
    dout = bf(torch.randn(T, H * hd, device="cuda"))
    st = _stream()
    outs = []
    for chunk in (1 << 20, 3, 7):
        assert LIB.sp_debug_set(None, b"attn_chunk", chunk) == 0
        o = torch.empty(T, H * hd, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(B * H * S, device="cuda")
        delta = torch.empty(B * H * S, device="cuda")
        dqkv = torch.zeros(T, W, device="cuda", dtype=torch.bfloat16)
        assert LIB.sp_debug_attention(0, T, S, H, Hkv, hd, 1, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), None, None,
                                      None, st) == 0
        assert LIB.sp_debug_attention(1, T, S, H, Hkv, hd, 1, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                      dout.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), st) == 0
        torch.cuda.synchronize()
        outs.append((o.clone(), lse.clone(), dqkv.clone()))
    LIB.sp_debug_set(None, b"attn_chunk", 0)
    for o, lse, dqkv in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(lse, outs[0][1]) and torch.equal(dqkv, outs[0][2])


def test_attention_is_deterministic():
    B, S, H, Hkv, hd = 2, 512, 4, 4, 64
    T, W = B * S, (H + 2 * Hkv) * hd
    qkv = bf(torch.randn(T, W, device="cuda"))
    dout = bf(torch.randn(T, H * hd, device="cuda"))
    outs = []
    for _ in range(2):
        o = torch.empty(T, H * hd, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(B * H * S, device="cuda")
        dqkv = torch.zeros(T, W, device="cuda", dtype=torch.bfloat16)
        delta = torch.empty(B * H * S, device="cuda")
        st = _stream()
        LIB.sp_debug_attention(0, T, S, H, Hkv, hd, 1, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), None, None,
                               None, st)
        LIB.sp_debug_attention(1, T, S, H, Hkv, hd, 1, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                               dout.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), st)
        torch.cuda.synchronize()
        outs.append((o.clone(), dqkv.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("rms", [0, 1])
@pytest.mark.parametrize("T,d", [(16384, 1600), (1000, 1280), (64, 4096), (16, 8192)])
def test_norm_forward_backward(T, d, rms):
    x = torch.randn(T, d, device="cuda") * 2 + 0.5
    g = 1 + 0.1 * torch.randn(d, device="cuda")
    b = 0.1 * torch.randn(d, device="cuda")
    y = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    stats = torch.empty(T, 2, device="cuda")
    st = _stream()
    eps = 1e-5
    assert LIB.sp_debug_norm_forward(x.data_ptr(), g.data_ptr(), b.data_ptr(), rms, eps, T, d, y.data_ptr(),
                                     stats.data_ptr(), st) == 0
    torch.cuda.synchronize()
    xv = x.clone().requires_grad_(True)
    gv = g.clone().requires_grad_(True)
    bv = b.clone().requires_grad_(True)
    if rms:
        ref = xv * torch.rsqrt(xv.pow(2).mean(-1, keepdim=True) + eps) * gv
    else:
        ref = torch.nn.functional.layer_norm(xv, (d,), gv, bv, eps)
    assert rel(y, ref) < 1e-2
    dy = torch.randn(T, d, device="cuda")
    ref.backward(dy)
    dres_in = torch.randn(T, d, device="cuda")
    dres_out = torch.empty(T, d, device="cuda")
    d16 = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    part, cnt = _col_scratch(T, d)
    out = torch.zeros(2, d, device="cuda")
    for rep in range(2):  # the counters re-arm: a second launch on the same scratch is identical
        assert LIB.sp_debug_norm_backward(dy.data_ptr(), x.data_ptr(), stats.data_ptr(), g.data_ptr(), rms, T, d,
                                          dres_in.data_ptr(), dres_out.data_ptr(), d16.data_ptr(), part.data_ptr(),
                                          cnt.data_ptr(), out.data_ptr(), st) == 0
        torch.cuda.synchronize()
        if rep == 0:
            first = out.clone()
    assert torch.equal(first, out) and int(cnt.abs().sum()) == 0
    want = dres_in + xv.grad
    assert rel(dres_out, want) < 1e-4
    assert rel(d16, want) < 1e-2
    assert rel(out[0], gv.grad) < 1e-4
    if not rms:
        assert rel(out[1], bv.grad) < 1e-4


@pytest.mark.parametrize("rms", [0, 1])
@pytest.mark.parametrize("T,d", [(16384, 1600), (1000, 1280), (64, 2048), (65, 64), (3, 1600)])
def test_norm_backward_fused(T, d, rms):
    """The single-pass norm backward (the executor's path for d <= 2048): dres_out and its bf16
    copy equal the two-pass kernel's elementwise (same per-row arithmetic), the parameter
    gradients and the column sums of dres_out (the bias gradient below) match fp64, and a
    repeated launch is bitwise identical (fixed reduction order)."""
    x = torch.randn(T, d, device="cuda") * 2 + 0.5
    g = 1 + 0.1 * torch.randn(d, device="cuda")
    b = 0.1 * torch.randn(d, device="cuda")
    y = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    stats = torch.empty(T, 2, device="cuda")
    st = _stream()
    assert LIB.sp_debug_norm_forward(x.data_ptr(), g.data_ptr(), b.data_ptr(), rms, 1e-5, T, d, y.data_ptr(),
                                     stats.data_ptr(), st) == 0
    dy = torch.randn(T, d, device="cuda")
    dres_in = torch.randn(T, d, device="cuda")
    # the two-pass kernels as the elementwise reference
    ref_out = torch.empty(T, d, device="cuda")
    ref16 = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    part, cnt = _col_scratch(T, d)
    ref_param = torch.zeros(2, d, device="cuda")
    assert LIB.sp_debug_norm_backward(dy.data_ptr(), x.data_ptr(), stats.data_ptr(), g.data_ptr(), rms, T, d,
                                      dres_in.data_ptr(), ref_out.data_ptr(), ref16.data_ptr(), part.data_ptr(),
                                      cnt.data_ptr(), ref_param.data_ptr(), st) == 0
    chunks = min(2 * torch.cuda.get_device_properties(0).multi_processor_count, (T + 1) // 2)  # norm_bwd_chunks
    ppart = torch.empty(chunks, 2, d, device="cuda")
    cpart = torch.empty(chunks, d, device="cuda")
    runs = []
    for _ in range(2):
        out = torch.empty(T, d, device="cuda")
        o16 = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
        op = torch.zeros(2, d, device="cuda")
        oc = torch.empty(d, device="cuda")
        assert LIB.sp_debug_norm_backward_fused(dy.data_ptr(), x.data_ptr(), stats.data_ptr(), g.data_ptr(), rms, T,
                                                d, dres_in.data_ptr(), out.data_ptr(), o16.data_ptr(), ppart.data_ptr(),
                                                cpart.data_ptr(), op.data_ptr(), oc.data_ptr(), st) == 0
        torch.cuda.synchronize()
        runs.append((out, o16, op, oc))
    out, o16, op, oc = runs[0]
    for a, bb in zip(runs[0], runs[1]):
        assert torch.equal(a, bb)
    assert rel(out, ref_out) < 1e-6 and rel(o16, ref16) < 1e-2
    xh = ((x.double() - (0 if rms else stats[:, :1].double())) * stats[:, 1:].double())
    assert rel(op[0], (dy.double() * xh).sum(0)) < 1e-5
    if not rms:
        assert rel(op[1], dy.double().sum(0)) < 1e-5
    assert rel(oc, out.double().sum(0)) < 1e-5
    # parameter gradients only (the layer-0 norm1: no dx)
    op2 = torch.zeros(2, d, device="cuda")
    assert LIB.sp_debug_norm_backward_fused(dy.data_ptr(), x.data_ptr(), stats.data_ptr(), g.data_ptr(), rms, T, d,
                                            dres_in.data_ptr(), None, None, ppart.data_ptr(), cpart.data_ptr(),
                                            op2.data_ptr(), None, st) == 0
    torch.cuda.synchronize()
    assert torch.equal(op2, op)


def _col_scratch(rows, widest):
    import ctypes
    pf, nc = ctypes.c_int64(), ctypes.c_int64()
    LIB.sp_debug_col_scratch(rows, widest, ctypes.byref(pf), ctypes.byref(nc))
    return (torch.empty(pf.value, device="cuda"), torch.zeros(nc.value, device="cuda", dtype=torch.int32))


@pytest.mark.parametrize("T,n", [(16384, 1600), (16384, 6400), (1000, 4800), (64, 64), (513, 256)])
def test_colsum_total_fixed_order(T, n):
    """Bias gradients: the column sums of a bf16 [T][n] matrix reduced inside one launch (the last
    block of each column group sums the chunk partials in order) against fp64, and bitwise
    repeatable with the scratch the first launch left behind."""
    x = (torch.randn(T, n, device="cuda") * 0.1).to(torch.bfloat16)
    part, cnt = _col_scratch(T, n)
    st = _stream()
    outs = []
    for _ in range(2):
        out = torch.empty(n, device="cuda")
        assert LIB.sp_debug_colsum(x.data_ptr(), T, n, part.data_ptr(), cnt.data_ptr(), out.data_ptr(), st) == 0
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1]) and int(cnt.abs().sum()) == 0
    ref = x.double().sum(0)
    assert (outs[0].double() - ref).abs().max().item() <= 1e-5 * max(1.0, ref.abs().max().item()) + 1e-4

"""TEST INFRASTRUCTURE ONLY — CPU fp32 restatement of the named-shape transformer block
(numpy), the checker for the executor's block path. Nothing in the product imports it.

Parity is UNPINNED by the reference: the reference has no transformer block, attention, norm or
GELU (its only block is model.cpp:54-123). This restatement
follows the block contract of include/superpipe.h ("named-shape layers") and is itself pinned
to torch.autograd on CPU in tests/test_block_oracle.py (forward outputs and every parameter
and input gradient). The training step is the reference's reference_train_step shape
(model.cpp:157-184): forward saving inputs, mse_loss / mse_grad (model.cpp:131-148), reverse
backward, apply_sgd (model.cpp:150-155) on trainable layers.

Images are flat fp32 arrays laid out by sp_block_layout (offsets in `layout.tensors`).
"""
from __future__ import annotations

import math

import numpy as np

F32 = np.float32
SQRT_2_OVER_PI = 0.7978845608028654


def _erf(x):
    # vectorised erf (Abramowitz-Stegun 7.1.26 is too coarse; use math.erf elementwise)
    return np.vectorize(math.erf, otypes=[np.float64])(x)


def gelu(x, erf):
    x64 = x.astype(np.float64)
    if erf:
        return (0.5 * x64 * (1.0 + _erf(x64 / math.sqrt(2.0)))).astype(F32)
    u = SQRT_2_OVER_PI * (x64 + 0.044715 * x64 ** 3)
    return (0.5 * x64 * (1.0 + np.tanh(u))).astype(F32)


def gelu_grad(x, erf):
    x64 = x.astype(np.float64)
    if erf:
        return (0.5 * (1.0 + _erf(x64 / math.sqrt(2.0))) + x64 * np.exp(-0.5 * x64 * x64) / math.sqrt(2 * math.pi)).astype(F32)
    u = SQRT_2_OVER_PI * (x64 + 0.044715 * x64 ** 3)
    t = np.tanh(u)
    return (0.5 * (1.0 + t) + 0.5 * x64 * (1.0 - t * t) * SQRT_2_OVER_PI * (1.0 + 3 * 0.044715 * x64 * x64)).astype(F32)


class Block:
    """One layer's parameter views."""

    def __init__(self, spec, layout, image):
        self.spec, self.layout = spec, layout
        self.p = {name: t.view(image) for name, t in layout.tensors.items()}

    def get(self, name):
        return self.p.get(name)


def norm_fwd(x, g, b, rms, eps):
    x64 = x.astype(np.float64)
    mean = np.zeros((x.shape[0], 1)) if rms else x64.mean(-1, keepdims=True)
    var = ((x64 - mean) ** 2).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x64 - mean) * rstd
    y = xhat * g
    if b is not None:
        y = y + b
    return y.astype(F32), (xhat, rstd)


def norm_bwd(dy, cache, g, rms):
    xhat, rstd = cache
    dy64 = dy.astype(np.float64)
    gy = dy64 * g
    c1 = (gy * xhat).mean(-1, keepdims=True)
    c0 = np.zeros_like(c1) if rms else gy.mean(-1, keepdims=True)
    dx = rstd * (gy - c0 - xhat * c1)
    dg = (dy64 * xhat).sum(0)
    db = dy64.sum(0)
    return dx.astype(F32), dg.astype(F32), db.astype(F32)


def _heads(spec, qkv):
    T = qkv.shape[0]
    H, Hkv, hd, S = spec.n_heads, spec.n_kv_heads, spec.head_dim, spec.seq_len
    B = T // S
    t = qkv.reshape(B, S, H + 2 * Hkv, hd).transpose(0, 2, 1, 3)
    return t[:, :H], t[:, H:H + Hkv], t[:, H + Hkv:]


def attn_fwd(spec, qkv):
    q, k, v = (a.astype(np.float64) for a in _heads(spec, qkv))
    g = spec.n_heads // spec.n_kv_heads
    k, v = np.repeat(k, g, axis=1), np.repeat(v, g, axis=1)
    S = spec.seq_len
    s = q @ k.transpose(0, 1, 3, 2) / math.sqrt(spec.head_dim)
    if spec.causal:
        s = np.where(np.triu(np.ones((S, S), bool), 1), -np.inf, s)
    m = s.max(-1, keepdims=True)
    p = np.exp(s - m)
    p /= p.sum(-1, keepdims=True)
    o = p @ v  # [B,H,S,hd]
    B = o.shape[0]
    return o.transpose(0, 2, 1, 3).reshape(B * S, -1).astype(F32), (q, k, v, p)


def attn_bwd(spec, cache, do):
    q, k, v, p = cache
    B, H, S, hd = q.shape
    do = do.astype(np.float64).reshape(B, S, H, hd).transpose(0, 2, 1, 3)
    dv = p.transpose(0, 1, 3, 2) @ do
    dp = do @ v.transpose(0, 1, 3, 2)
    ds = p * (dp - (dp * p).sum(-1, keepdims=True))
    scale = 1.0 / math.sqrt(hd)
    dq = ds @ k * scale
    dk = ds.transpose(0, 1, 3, 2) @ q * scale
    g = spec.n_heads // spec.n_kv_heads
    Hkv = spec.n_kv_heads
    dk = dk.reshape(B, Hkv, g, S, hd).sum(2)
    dv = dv.reshape(B, Hkv, g, S, hd).sum(2)
    out = np.concatenate([dq, dk, dv], axis=1)  # [B, H + 2Hkv, S, hd]
    return out.transpose(0, 2, 1, 3).reshape(B * S, -1).astype(F32)


def _swiglu_split(a, ff):
    c = a.reshape(a.shape[0], ff // 32, 2, 32)
    return c[:, :, 0, :].reshape(-1, ff), c[:, :, 1, :].reshape(-1, ff)


def layer_forward(spec, lay, image, x):
    """One block: returns y and the cache its backward needs."""
    P = Block(spec, lay, image)
    rms = spec.norm == 1
    xn1, c1 = norm_fwd(x, P.get("norm1.g"), P.get("norm1.b"), rms, spec.norm_eps)
    qkv = (xn1.astype(np.float64) @ P.get("wqkv")).astype(F32)
    if P.get("bqkv") is not None:
        qkv = qkv + P.get("bqkv")
    o, ca = attn_fwd(spec, qkv)
    h = (o.astype(np.float64) @ P.get("wo") + x).astype(F32)
    if P.get("bo") is not None:
        h = h + P.get("bo")
    xn2, c2 = norm_fwd(h, P.get("norm2.g"), P.get("norm2.b"), rms, spec.norm_eps)
    if spec.mlp == 2:  # SwiGLU, gate / up interleaved in 32-column chunks
        a = (xn2.astype(np.float64) @ P.get("wgu")).astype(F32)
        gt, up = _swiglu_split(a, spec.ff)
        gt64 = gt.astype(np.float64)
        act = (gt64 / (1 + np.exp(-gt64)) * up).astype(F32)
        pre = a
    else:
        pre = (xn2.astype(np.float64) @ P.get("w1")).astype(F32)
        if P.get("b1") is not None:
            pre = pre + P.get("b1")
        act = gelu(pre, spec.mlp == 1)
    y = (act.astype(np.float64) @ P.get("w2") + h).astype(F32)
    if P.get("b2") is not None:
        y = y + P.get("b2")
    return y, dict(x=x, xn1=xn1, c1=c1, qkv=qkv, o=o, ca=ca, h=h, xn2=xn2, c2=c2, pre=pre, act=act)


def layer_backward(spec, lay, image, cache, dy, need_dx=True):
    """Returns (dx, gradient image in the layer layout)."""
    if spec.mlp == 2:
        raise NotImplementedError("SwiGLU blocks are inference-only (as in the executor)")
    P = Block(spec, lay, image)
    rms = spec.norm == 1
    grad = np.zeros_like(image)
    G = Block(spec, lay, grad)
    dy64 = dy.astype(np.float64)
    # MLP
    G.get("w2")[...] = cache["act"].astype(np.float64).T @ dy64
    if G.get("b2") is not None:
        G.get("b2")[...] = dy64.sum(0)
    dact = dy64 @ P.get("w2").astype(np.float64).T
    dpre = dact * gelu_grad(cache["pre"], spec.mlp == 1)
    G.get("w1")[...] = cache["xn2"].astype(np.float64).T @ dpre
    if G.get("b1") is not None:
        G.get("b1")[...] = dpre.sum(0)
    dxn2 = dpre @ P.get("w1").astype(np.float64).T
    dh_n, dg2, db2 = norm_bwd(dxn2, cache["c2"], P.get("norm2.g"), rms)
    G.get("norm2.g")[...] = dg2
    if G.get("norm2.b") is not None:
        G.get("norm2.b")[...] = db2
    dh = dy64 + dh_n
    # attention
    G.get("wo")[...] = cache["o"].astype(np.float64).T @ dh
    if G.get("bo") is not None:
        G.get("bo")[...] = dh.sum(0)
    do = dh @ P.get("wo").astype(np.float64).T
    dqkv = attn_bwd(spec, cache["ca"], do).astype(np.float64)
    G.get("wqkv")[...] = cache["xn1"].astype(np.float64).T @ dqkv
    if G.get("bqkv") is not None:
        G.get("bqkv")[...] = dqkv.sum(0)
    dxn1 = dqkv @ P.get("wqkv").astype(np.float64).T
    dx_n, dg1, db1 = norm_bwd(dxn1, cache["c1"], P.get("norm1.g"), rms)
    G.get("norm1.g")[...] = dg1
    if G.get("norm1.b") is not None:
        G.get("norm1.b")[...] = db1
    dx = (dh + dx_n).astype(F32)
    return dx, grad


def forward(spec, lay, params, x):
    for i in range(params.shape[0]):
        x, _ = layer_forward(spec, lay, params[i], x)
    return x


def train_step(spec, lay, params, x, t, lr, frozen=None):
    """reference_train_step (model.cpp:157-184) for a block stack: returns (loss, new params,
    per-layer gradient images)."""
    n = params.shape[0]
    frozen = np.zeros(n, np.int32) if frozen is None else frozen
    caches, h = [], x
    for i in range(n):
        h, c = layer_forward(spec, lay, params[i], h)
        caches.append(c)
    e = h.astype(np.float64) - t
    N = e.size
    loss = float((e * e).sum() / N)
    dy = (2.0 * e / N).astype(F32)
    new, grads = params.copy(), [None] * n
    for i in reversed(range(n)):
        dy, g = layer_backward(spec, lay, params[i], caches[i], dy, need_dx=i > 0)
        grads[i] = g
        if not frozen[i]:
            new[i] = (params[i].astype(np.float64) - lr * g).astype(F32)
    return loss, new, grads

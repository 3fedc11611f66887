"""Plain PyTorch reference of the transformer block (test helper): the same contract as
include/superpipe.h "named-shape layers" and oracle/pyblock.py, any device / dtype, parameters
as autograd leaves. Used as the fp32 reference at shapes the numpy oracle is too slow for."""
import math

import torch

from paper_2410_08791_b200 import blocks as B


def layer(spec, lay, image, x, device="cpu", dtype=torch.float64):
    P = {n: torch.tensor(t.view(image), dtype=dtype, device=device, requires_grad=True)
         for n, t in lay.tensors.items()}
    rms = spec.norm == B.NORM_RMS

    def norm(v, g, b):
        if rms:
            return v * torch.rsqrt(v.pow(2).mean(-1, keepdim=True) + spec.norm_eps) * g
        return torch.nn.functional.layer_norm(v, (spec.d,), g, b, spec.norm_eps)

    T = x.shape[0]
    S, H, Hkv, hd = spec.seq_len, spec.n_heads, spec.n_kv_heads, spec.head_dim
    xn = norm(x, P["norm1.g"], P.get("norm1.b"))
    qkv = xn @ P["wqkv"] + (P["bqkv"] if "bqkv" in P else 0)
    t = qkv.view(T // S, S, H + 2 * Hkv, hd).permute(0, 2, 1, 3)
    q = t[:, :H]
    k = t[:, H:H + Hkv].repeat_interleave(H // Hkv, 1)
    v = t[:, H + Hkv:].repeat_interleave(H // Hkv, 1)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=bool(spec.causal))
    o = o.permute(0, 2, 1, 3).reshape(T, H * hd)
    h = x + o @ P["wo"] + (P["bo"] if "bo" in P else 0)
    xn2 = norm(h, P["norm2.g"], P.get("norm2.b"))
    if spec.mlp == B.MLP_SWIGLU:
        a = (xn2 @ P["wgu"]).view(T, spec.ff // 32, 2, 32)
        act = (torch.nn.functional.silu(a[:, :, 0]) * a[:, :, 1]).reshape(T, spec.ff)
    else:
        pre = xn2 @ P["w1"] + P["b1"]
        act = torch.nn.functional.gelu(pre, approximate="none" if spec.mlp == B.MLP_GELU_ERF else "tanh")
    y = h + act @ P["w2"] + (P["b2"] if "b2" in P else 0)
    return y, P


def stack(spec, lay, params, x, device="cpu", dtype=torch.float64):
    h, Ps = x, []
    for i in range(params.shape[0]):
        h, P = layer(spec, lay, params[i], h, device, dtype)
        Ps.append(P)
    return h, Ps


def grad_image(lay, P, like):
    """The gradients of one layer's leaves as a flat image in the layer layout."""
    import numpy as np
    g = np.zeros_like(like)
    for name, t in lay.tensors.items():
        g[t.offset:t.offset + t.rows * t.cols] = P[name].grad.detach().float().cpu().numpy().ravel()
    return g

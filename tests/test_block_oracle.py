"""CPU: the block oracle (oracle/pyblock.py, test infrastructure) pinned to torch.autograd, and
the host side of the named-shape layers (layout, deterministic init) — no GPU needed.

The reference has no transformer block, so this restatement cannot be pinned to it
(DESIGN.md "parity unpinned by the reference" for the block path); torch on CPU in float64 is
the independent check of its forward and of every gradient it produces."""
import math
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyblock  # noqa: E402

from paper_2410_08791_b200 import blocks as B  # noqa: E402

SPECS = [
    B.BlockSpec(128, 256, 2, 2, 32, B.NORM_LAYER, B.MLP_GELU_TANH, True, True, 1e-5, "gpt2-like"),
    B.BlockSpec(320, 640, 4, 4, 17, B.NORM_LAYER, B.MLP_GELU_ERF, True, False, 1e-6, "vit-like (hd 80)"),
    B.BlockSpec(256, 256, 2, 1, 16, B.NORM_RMS, B.MLP_SWIGLU, False, True, 1e-5, "llama-like (GQA, hd 128)"),
]


def torch_layer(spec, lay, image, x):
    """The same block in torch (float64), parameters as leaf tensors."""
    P = {n: torch.tensor(t.view(image), dtype=torch.float64, requires_grad=True) for n, t in lay.tensors.items()}
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
    q, k, v = t[:, :H], t[:, H:H + Hkv].repeat_interleave(H // Hkv, 1), t[:, H + Hkv:].repeat_interleave(H // Hkv, 1)
    s = q @ k.transpose(-1, -2) / math.sqrt(hd)
    if spec.causal:
        s = s.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
    o = (torch.softmax(s, -1) @ v).permute(0, 2, 1, 3).reshape(T, H * hd)
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


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.name)
def test_oracle_forward_and_gradients_match_torch_autograd(spec):
    lay = B.block_layout(spec)
    model = B.build_block_model(spec, 5, 1)
    image = model.params[0].copy()
    rng = np.random.default_rng(0)
    for t in lay.tensors.values():  # non-trivial norm parameters
        if not t.matrix and t.name.startswith("norm"):
            t.view(image)[...] += rng.standard_normal(t.cols).astype(np.float32) * 0.1
    x = rng.standard_normal((2 * spec.seq_len, spec.d)).astype(np.float32)
    y, cache = pyblock.layer_forward(spec, lay, image, x)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    yt, P = torch_layer(spec, lay, image, xt)
    assert np.abs(y - yt.detach().numpy()).max() < 1e-4 * max(1.0, float(np.abs(y).max()))
    if spec.mlp == B.MLP_SWIGLU:
        return  # inference-only
    dy = rng.standard_normal(y.shape).astype(np.float32)
    yt.backward(torch.tensor(dy, dtype=torch.float64))
    dx, grad = pyblock.layer_backward(spec, lay, image, cache, dy)
    assert np.abs(dx - xt.grad.numpy()).max() < 1e-4 * np.abs(xt.grad.numpy()).max()
    for name, t in lay.tensors.items():
        want = P[name].grad.numpy()
        got = t.view(grad)
        assert np.abs(got - want).max() <= 1e-4 * np.abs(want).max() + 1e-7, name


def test_train_step_loss_and_sgd_match_torch():
    spec = SPECS[0]
    lay = B.block_layout(spec)
    model = B.build_block_model(spec, 9, 2, frozen_prefix=1)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((spec.seq_len, spec.d)).astype(np.float32)
    t = rng.standard_normal((spec.seq_len, spec.d)).astype(np.float32)
    loss, new, grads = pyblock.train_step(spec, lay, model.params, x, t, 0.1, model.frozen)
    h = torch.tensor(x, dtype=torch.float64)
    Ps = []
    for i in range(2):
        h, P = torch_layer(spec, lay, model.params[i], h)
        Ps.append(P)
    lt = ((h - torch.tensor(t, dtype=torch.float64)) ** 2).mean()
    lt.backward()
    assert abs(loss - float(lt)) < 1e-6 * abs(loss)
    assert np.array_equal(new[0], model.params[0])  # frozen
    for name, tt in lay.tensors.items():
        want = model.params[1][tt.offset:tt.offset + tt.rows * tt.cols] - 0.1 * Ps[1][name].grad.numpy().ravel()
        assert np.abs(tt.view(new[1]).ravel() - want).max() < 1e-6, name


def test_layout_of_the_named_shapes():
    # parameters per layer of the named shapes
    want = {"gpt2-xl": 30.74e6, "vit-h14": 19.68e6, "llama3-8b": 218.1e6, "llama3-70b": 855.6e6}
    for key, (spec, n) in B.NAMED_SHAPES.items():
        lay = B.block_layout(spec)
        assert abs(lay.n_params - want[key]) / want[key] < 2e-3, (key, lay.n_params)
        # 64-float aligned tensors, wire image = bf16 matrices + fp32 vectors
        assert all(t.offset % 64 == 0 and t.wire_offset % 256 == 0 for t in lay.tensors.values())
        mats = sum(t.rows * t.cols for t in lay.tensors.values() if t.matrix)
        assert lay.wire_bytes >= 2 * mats
    # GPT-2 XL: 48 layers x 30.7M = 1.475B parameters (5.9 GB fp32, 2.95 GB bf16)
    lay = B.block_layout(B.GPT2_XL)
    assert abs(48 * lay.n_params - 1.4755e9) / 1.4755e9 < 2e-3
    # Llama-3-70B: 80 layers of bf16 wire exceed C5's 40 GB cap (137 GB)
    assert 80 * B.block_layout(B.LLAMA3_70B).wire_bytes > 130e9


def test_block_init_is_deterministic_and_bounded():
    spec = SPECS[0]
    a = B.build_block_model(spec, 3, 2)
    b = B.build_block_model(spec, 3, 2)
    c = B.build_block_model(spec, 4, 2)
    assert np.array_equal(a.params, b.params) and not np.array_equal(a.params, c.params)
    assert not np.array_equal(a.params[0], a.params[1])
    w = a.tensor(0, "wqkv")
    assert np.abs(w).max() <= 1 / math.sqrt(spec.d) and np.abs(w).max() > 0.9 / math.sqrt(spec.d)
    assert np.all(a.tensor(0, "norm1.g") == 1) and np.all(a.tensor(0, "norm1.b") == 0)


def test_invalid_block_specs_are_rejected():
    for bad in [B.BlockSpec(100, 256, 2, 2, 8), B.BlockSpec(128, 256, 3, 3, 8),
                B.BlockSpec(128, 256, 2, 3, 8), B.BlockSpec(192, 256, 6, 6, 8)]:  # hd 32 unsupported
        with pytest.raises(B.InvalidArgument):
            B.block_layout(bad)

"""Parity at the dense stand-in's bench shape (round 1's headline: 48 x 1600 square blocks,
16384 rows) — the exact tcgen05 kernel configurations that shape selects, against fp32
references built from the GPU's own operands (so bf16 rounding of the inputs is not counted
and gate flips cannot hide a tiling bug):

* the three GEMMs at 16384 x 1600 x 1600 as the executor runs them: forward with the TMA
  epilogue writing bias + ReLU + the bit mask, dX gated by that mask, and dW with the choice
  choose_dw makes (CTA pair, 3 split-K partials, half-width ragged last tile);
* one bf16 train step of a 2-layer d=1600 model at 16384 rows: every layer's dW and db and the
  propagated dz, from the GPU's own saved activations and loss gradient (model.cpp:54-123).
Tolerances are stated per check (fp32 accumulation-order differences only)."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
T, D = 16384, 1600


def rel(got, ref):
    got, ref = got.double(), ref.double()
    return float((got - ref).norm() / ref.norm().clamp_min(1e-300))


def test_headline_gemm_configurations_against_fp32():
    torch.manual_seed(5)
    x = (torch.rand(T, D, device="cuda") - 0.5).to(torch.bfloat16)
    W = ((torch.rand(D, D, device="cuda") - 0.5) / 20).to(torch.bfloat16)
    b = (torch.rand(D, device="cuda") - 0.5) / 20
    st = torch.cuda.current_stream().cuda_stream
    # forward: y = relu(x W + b) -> bf16 + ReLU bit mask (column-chunk-major words)
    y = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    mask = torch.zeros(D // 32 * T, device="cuda", dtype=torch.int32)
    assert LIB.sp_debug_gemm_bf16_masked_async(T, D, D, x.data_ptr(), D, 0, W.data_ptr(), D, 1, 0, y.data_ptr(), D,
                                               b.data_ptr(), 1, None, 0, 1, 0, 0, st, mask.data_ptr(), None) == 0
    torch.cuda.synchronize()
    ref = torch.relu(x.double() @ W.double() + b.double())
    assert rel(y, ref) < 4e-3  # one bf16 rounding of the output
    # the mask is exactly "stored value > 0"
    bits = mask.view(D // 32, T).cpu().numpy().astype(np.uint32)
    want = (y.float() > 0).cpu().numpy().reshape(T, D // 32, 32)
    got = ((bits.T[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    assert np.array_equal(got, want)
    # dX = (dz W^T) gated by the mask (the executor's bf16 training path)
    dz = ((torch.rand(T, D, device="cuda") - 0.5) * 1e-3).to(torch.bfloat16)
    dx = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    assert LIB.sp_debug_gemm_bf16_masked_async(T, D, D, dz.data_ptr(), D, 0, W.data_ptr(), D, 0, 2, dx.data_ptr(), D,
                                               None, 1, y.data_ptr(), D, 1, 0, 0, st, None, mask.data_ptr()) == 0
    torch.cuda.synchronize()
    ref = (dz.double() @ W.double().t()) * (y.double() > 0)
    assert rel(dx, ref) < 4e-3
    # dW = x^T dz with the executor's choice for this shape (no fused SGD: raw partials)
    cta, bn = C.c_int32(), C.c_int32()
    splits = LIB.sp_debug_dw_choice(D, T, 1, C.byref(cta), C.byref(bn))
    assert (cta.value, bn.value, splits) == (2, 256, 3)  # the configuration DESIGN.md §4 names
    parts = torch.empty(splits * D * D, device="cuda")
    assert LIB.sp_debug_gemm_bf16_async(D, D, T, x.data_ptr(), D, 1, dz.data_ptr(), D, 1, 3, parts.data_ptr(), D,
                                        None, 0, None, 0, splits, bn.value, cta.value, st) == 0
    torch.cuda.synchronize()
    got = parts.view(splits, D, D).sum(0)
    ref = x.double().t() @ dz.double()
    assert rel(got, ref) < 2e-5  # fp32 accumulation over K = 16384, three partials


def test_headline_train_step_layers_against_fp32_from_own_activations():
    model = sp.build_model(7, 2, D)
    x, t = sp.make_input(7, 0, T, D), sp.make_input(7, 1, T, D)
    S = sp.StrategyConfig(sp.SUPERPIPELINE, 2, 1)
    # the GPU's own layer-0 output x1 (fp32; the training forward stores its bf16 rounding)
    with sp.Executor(1, D, sp.StrategyConfig(sp.STANDARD), numerics=sp.BF16) as e1:
        e1.register_layer(0, model.W[0], model.b[0])
        x1 = e1.forward([x])[0]
    with sp.Executor(2, D, S, numerics=sp.BF16) as ex:
        ex.register_model(model)
        y = ex.forward([x])[0]
        lr = 1.0  # W' = W - dW exactly (fp32 ops), so dW is recovered to ~1e-6 relative
        ex.train_step(x, t, lr)
        after = ex.read_model(model)
    dev = "cuda"
    bf = lambda a: torch.tensor(a, device=dev).to(torch.bfloat16).double()  # noqa: E731
    W = [bf(model.W[i]) for i in range(2)]
    x0b, x1b = bf(x), bf(x1)
    # the loss gradient exactly as loss_grad_bf16 forms it: bf16(2 (y - t) / N), gated by y > 0
    inv_n = np.float32(1.0) / np.float32(T * D)
    g = (np.float32(2.0) * (y - t).astype(np.float32)).astype(np.float32) * inv_n
    g[y <= 0] = 0
    dz1 = bf(g.astype(np.float32))
    dW1 = torch.tensor(model.W[1] - after.W[1], device=dev).double() / lr
    db1 = torch.tensor(model.b[1] - after.b[1], device=dev).double() / lr
    assert rel(dW1, x1b.t() @ dz1) < 1e-4
    assert rel(db1, dz1.sum(0)) < 1e-4
    # layer 0: dz0 = bf16((dz1 W1^T) . [x1 > 0]) from the same operands, then dW0 = x0^T dz0
    dz0 = ((dz1 @ W[1].t()) * (x1b > 0)).to(torch.bfloat16).double()
    dW0 = torch.tensor(model.W[0] - after.W[0], device=dev).double() / lr
    db0 = torch.tensor(model.b[0] - after.b[0], device=dev).double() / lr
    assert rel(dW0, x0b.t() @ dz0) < 1e-3  # dz0 recomputed here: a few 1-ulp bf16 flips
    assert rel(db0, dz0.sum(0)) < 1e-3

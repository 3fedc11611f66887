"""GPU parity of the named-shape layer path (transformer blocks streamed through the ring):

* the CUDA path against the CPU oracle (oracle/pyblock.py, pinned to torch.autograd) at small
  shapes: inference outputs, the training loss and every layer's gradient image;
* window invariance: outputs, losses and updated weights bitwise identical across every
  (k, k') / strategy, with activation offload (backward recompute) and without;
* the bench workload's exact shape (GPT-2 XL layers, 16 x 1024 tokens) against a PyTorch fp32
  reference on the GPU: forward output and both layers' gradient images of a 2-layer stack.

Tolerances are normwise (||got - ref|| / ||ref||) unless stated; they bound bf16 operand
rounding (2^-9 relative per operand) accumulated through the block.
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyblock  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import blocks as B  # noqa: E402

S = sp.StrategyConfig
GPT = B.BlockSpec(128, 256, 2, 2, 64, B.NORM_LAYER, B.MLP_GELU_TANH, True, True, 1e-5, "gpt2-like")
VIT = B.BlockSpec(320, 640, 4, 4, 65, B.NORM_LAYER, B.MLP_GELU_ERF, True, False, 1e-6, "vit-like")
LLAMA = B.BlockSpec(256, 512, 2, 1, 64, B.NORM_RMS, B.MLP_SWIGLU, False, True, 1e-5, "llama-like")


def nrm(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))


def inputs(spec, seqs, seed=3):
    T = seqs * spec.seq_len
    return sp.make_input(seed, 0, T, spec.d), sp.make_input(seed, 1, T, spec.d)


@pytest.mark.parametrize("spec", [GPT, VIT, LLAMA], ids=lambda s: s.name)
def test_block_inference_matches_the_oracle(spec):
    model = B.build_block_model(spec, 11, 3)
    x, _ = inputs(spec, 3)
    want = pyblock.forward(spec, model.layout, model.params, x)
    with B.BlockExecutor(3, spec, S(sp.SUPERPIPELINE, 2, 1)) as ex:
        ex.register_model(model)
        got = ex.forward([x])[0]
        st = ex.stats()
    assert np.isfinite(got).all()
    assert nrm(got, want) < 1e-2
    assert st["attn_launches"] == 3 and st["attn_flops"] > 0


@pytest.mark.parametrize("spec", [GPT, VIT], ids=lambda s: s.name)
def test_block_train_step_matches_the_oracle(spec):
    model = B.build_block_model(spec, 12, 2)
    x, t = inputs(spec, 2)
    loss_ref, new_ref, grads = pyblock.train_step(spec, model.layout, model.params, x, t, 0.05, model.frozen)
    with B.BlockExecutor(2, spec, S(sp.SUPERPIPELINE, 2, 1)) as ex:
        ex.register_model(model)
        loss = ex.train_step(x, t, 0.05)
        g = [ex.debug_read_grad(i) for i in range(2)]
        after = ex.read_model(model)
    assert abs(loss - loss_ref) <= 1e-2 * abs(loss_ref)
    for i in range(2):
        for name, tt in model.layout.tensors.items():
            e = nrm(tt.view(g[i]), tt.view(grads[i]))
            assert e < 3e-2, (i, name, e)
        # the SGD update applied exactly that gradient: w' = w - lr g (fp32, elementwise)
        np.testing.assert_array_equal(after.params[i], (model.params[i] - np.float32(0.05) * g[i]).astype(np.float32))


STRATS = [S(sp.SUPERPIPELINE, 2, 1), S(sp.SUPERPIPELINE, 3, 1), S(sp.SUPERPIPELINE, 4, 2, sp.SEQUENTIAL),
          S(sp.NAIVE, 2), S(sp.STANDARD)]


def test_block_training_is_bitwise_identical_across_windows_and_offload():
    spec = GPT
    model = B.build_block_model(spec, 13, 5, frozen_prefix=1)
    x, t = inputs(spec, 2)
    runs = []
    for strat in STRATS:
        for ckpt in (False, True):
            with B.BlockExecutor(5, spec, strat, checkpointing=ckpt) as ex:
                ex.register_model(model)
                losses = [ex.train_step(x, t, 0.05) for _ in range(3)]
                y = ex.forward([x])[0]
                runs.append((strat, ckpt, losses, ex.read_model(model).params, y))
    base = runs[0]
    for strat, ckpt, losses, params, y in runs[1:]:
        assert losses == base[2], (strat, ckpt)
        assert np.array_equal(params, base[3]), (strat, ckpt)
        assert np.array_equal(y, base[4]), (strat, ckpt)
    assert np.array_equal(base[3][0], model.params[0])  # frozen prefix untouched
    assert base[2][2] < base[2][0]  # it trains


def test_block_inference_item_batching_and_windows_are_bitwise():
    spec = VIT
    model = B.build_block_model(spec, 14, 4)
    xs = [inputs(spec, 2, seed=20 + i)[0] for i in range(3)]
    outs = []
    for strat in STRATS:
        for batched in (False, True):
            with B.BlockExecutor(4, spec, strat) as ex:
                ex.register_model(model)
                ex.set_item_batching(batched)
                outs.append(np.stack(ex.forward(xs)))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_block_adamw_and_single_rank_dp_paths_are_window_invariant():
    spec = GPT
    model = B.build_block_model(spec, 15, 4)
    x, t = inputs(spec, 2)
    res = []
    for strat in (S(sp.SUPERPIPELINE, 2, 1), S(sp.STANDARD)):
        for mode in ("adamw", "dp-allreduce", "dp-sharded"):
            with B.BlockExecutor(4, spec, strat) as ex:
                ex.register_model(model)
                if mode == "adamw":
                    ex.set_optimizer(sp.OPT_ADAMW, 0.9, 0.999, 1e-8, 0.01)
                else:
                    ex.dp_init(sp.Executor.nccl_unique_id(), 0, 1, shard_weights=mode == "dp-sharded")
                losses = [ex.train_step(x, t, 0.01) for _ in range(2)]
                if mode != "adamw":
                    ex.dp_sync()
                res.append((mode, losses, ex.read_model(model).params))
    by_mode = {}
    for mode, losses, params in res:
        if mode in by_mode:
            assert by_mode[mode][0] == losses and np.array_equal(by_mode[mode][1], params), mode
        by_mode[mode] = (losses, params)
    # All-reduce mode keeps the split master (the GEMMs multiply the bf16 truncation of each
    # weight); sharded streaming keeps the fp32 image and converts it on the device (round to
    # nearest). Each is window-invariant above; across the two only the operand rounding differs.
    base = model.params
    a_, b_ = by_mode["dp-allreduce"][1], by_mode["dp-sharded"][1]
    assert nrm(a_ - base, b_ - base) < 5e-2  # the two updates agree to bf16 operand precision


def test_bench_shape_gpt2_xl_two_layers_against_torch_fp32():
    """The bench workload's exact layer shape: GPT-2 XL blocks (d 1600, ff 6400, 25 heads of
    64, causal), 16 sequences x 1024 tokens. Forward output and both layers' gradient images
    against PyTorch fp32 (TF32 off) autograd on the GPU from the same fp32 parameters."""
    torch = pytest.importorskip("torch")
    torch.backends.cuda.matmul.allow_tf32 = False
    spec = B.GPT2_XL
    model = B.build_block_model(spec, 7, 2)
    T = 16 * spec.seq_len
    x, t = sp.make_input(7, 0, T, spec.d), sp.make_input(7, 1, T, spec.d)
    with B.BlockExecutor(2, spec, S(sp.SUPERPIPELINE, 2, 1)) as ex:
        ex.register_model(model)
        y = ex.forward([x])[0]
        loss = ex.train_step(x, t, 1e-3)
        g = [ex.debug_read_grad(i) for i in range(2)]
    import block_ref
    xt = torch.tensor(x, device="cuda")
    yt, Ps = block_ref.stack(spec, model.layout, model.params, xt, "cuda", torch.float32)
    lt = ((yt - torch.tensor(t, device="cuda")) ** 2).mean()
    lt.backward()
    assert nrm(y, yt.detach().cpu().numpy()) < 1e-2
    assert abs(loss - float(lt.detach())) <= 1e-2 * float(lt.detach())
    worst = {}
    for i in range(2):
        ref = block_ref.grad_image(model.layout, Ps[i], g[i])
        for name, tt in model.layout.tensors.items():
            worst[(i, name)] = nrm(tt.view(g[i]), tt.view(ref))
    bad = {k: v for k, v in worst.items() if v >= 3e-2}
    assert not bad, bad


def test_inference_only_master_streams_the_same_bits():
    """SP_BLOCK_INFER_ONLY keeps only the bf16 wire image on the host (half the pinned memory);
    its outputs equal the full split master's bitwise (the GEMMs multiply the same truncated
    halves), and training is refused."""
    spec = LLAMA
    model = B.build_block_model(spec, 16, 3)
    x, t = inputs(spec, 2)
    outs = []
    for infer_only in (False, True):
        with B.BlockExecutor(3, spec, S(sp.SUPERPIPELINE, 2, 1), infer_only=infer_only) as ex:
            ex.register_model(model)
            outs.append(ex.forward([x])[0])
            if infer_only:
                assert ex.stats()["h2d_bytes"] == 3 * model.layout.wire_bytes
                with pytest.raises(sp.InvalidArgument):
                    ex.train_step(x, t, 0.01)
    assert np.array_equal(outs[0], outs[1])

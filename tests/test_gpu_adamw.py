"""GPU parity of the AdamW option (sp_set_optimizer) against the CPU oracle.

The reference trains with plain SGD (engine.cpp run_train_step: W -= lr * dW), which stays the
default. BASELINE.json's north_star adds optimizer state held in pinned host DRAM and a fused
AdamW update; this is that option. The moments m, v (fp32, same layout as [W | b]) live in the
pinned host master next to the weights, ride the ring with each trainable layer's backward
load and write-back, and are updated by one kernel that also sums the split-K partials.

  * exact numerics: weights, biases, m and v are BIT-identical to the oracle (the reference's
    gradients, then oracle/oracle.c:orc_adamw = torch.optim.AdamW's element update with the
    scalars rounded once), every strategy / window / checkpointing, across several steps
    (each later step is a CUDA graph replay reading that step's scalars from device memory);
  * bf16 numerics: bit-identical across windows, and within tolerance of the oracle.
"""
import numpy as np
import pytest

import paper_2410_08791_b200 as sp
from pyoracle import Oracle

pytestmark = pytest.mark.gpu
ORC = Oracle()
F = lambda v: float(np.float32(v))  # noqa: E731  the ABI takes float hyperparameters
HP = dict(beta1=F(0.9), beta2=F(0.999), eps=F(1e-8), weight_decay=F(0.01))


def S(kind, k=0, kp=0, mode=sp.BATCH):
    return sp.StrategyConfig(kind, k, kp, mode)


def oracle_adamw(model, batches, lr, steps, **hp):
    """Oracle: the reference's exact gradients (ref_reference_train_step with want_grads),
    then orc_adamw per trainable layer. Returns (losses, W, b, mW, mb, vW, vb)."""
    W, b = model.W.copy(), model.b.copy()
    mW, vW = np.zeros_like(W), np.zeros_like(W)
    mb, vb = np.zeros_like(b), np.zeros_like(b)
    losses = []
    for t in range(1, steps + 1):
        x, y = batches[(t - 1) % len(batches)]
        loss, _, _, dW, db, _ = ORC.train_step(W, b, x, y, lr, frozen=model.frozen, want_grads=True)
        losses.append(np.float32(loss))
        for L in range(W.shape[0]):
            if model.frozen[L]:
                continue
            ORC.adamw(W[L], mW[L], vW[L], dW[L], lr, hp["beta1"], hp["beta2"], hp["eps"],
                      hp["weight_decay"], t)
            ORC.adamw(b[L], mb[L], vb[L], db[L], lr, hp["beta1"], hp["beta2"], hp["eps"],
                      hp["weight_decay"], t)
    return losses, W, b, mW, mb, vW, vb


def run_adamw(model, batches, lr, steps, strategy, numerics=sp.EXACT, ckpt=False, dp=None, **hp):
    n, d = model.n_layers, model.d
    with sp.Executor(n, d, strategy, numerics=numerics, checkpointing=ckpt) as ex:
        ex.register_model(model)
        if dp:
            ex.dp_init(sp.Executor.nccl_unique_id(), 0, 1, shard_weights=dp == "sharded")
        ex.set_optimizer(sp.OPT_ADAMW, **hp)
        losses = []
        for t in range(steps):
            x, y = batches[t % len(batches)]
            losses.append(np.float32(ex.train_step(x, y, lr)))
        if dp == "sharded":
            ex.dp_sync()
        m = ex.read_model(model)
        st = [ex.read_optimizer_state(L) for L in range(n)]
    mW = np.stack([s[0] for s in st])
    mb = np.stack([s[1] for s in st])
    vW = np.stack([s[2] for s in st])
    vb = np.stack([s[3] for s in st])
    return losses, m.W, m.b, mW, mb, vW, vb


def same(a, b):
    return all(np.array_equal(np.asarray(x), np.asarray(y)) for x, y in zip(a, b))


@pytest.mark.parametrize("frozen_prefix", [0, 2])
def test_adamw_exact_bitwise_every_strategy(frozen_prefix):
    model = sp.build_model(31, 6, 8, frozen_prefix)
    batches = [(sp.make_input(31, 2 * i, 3, 8), sp.make_input(31, 2 * i + 1, 3, 8)) for i in range(2)]
    lr = F(0.01)
    ref = oracle_adamw(model, batches, lr, 4, **HP)
    for s in [S(sp.STANDARD), S(sp.NAIVE, 2), S(sp.SUPERPIPELINE, 2, 1), S(sp.SUPERPIPELINE, 4, 2),
              S(sp.SUPERPIPELINE, 3, 1, sp.SEQUENTIAL)]:
        for ckpt in (False, True):
            got = run_adamw(model, batches, lr, 4, s, ckpt=ckpt, **HP)
            assert [x.tobytes() for x in got[0]] == [x.tobytes() for x in ref[0]], (s, ckpt)
            for name, g, r in zip(("W", "b", "mW", "mb", "vW", "vb"), got[1:], ref[1:]):
                assert np.array_equal(g, r), (s, ckpt, name, float(np.abs(g - r).max()))
    # frozen layers: untouched weights and no state
    got = run_adamw(model, batches, lr, 2, S(sp.SUPERPIPELINE, 2, 1), **HP)
    for L in range(frozen_prefix):
        assert np.array_equal(got[1][L], model.W[L]) and not got[3][L].any() and not got[5][L].any()


def test_adamw_differs_from_sgd_and_set_optimizer_resets():
    model = sp.build_model(5, 4, 8, 0)
    x, y = sp.make_input(5, 0, 4, 8), sp.make_input(5, 1, 4, 8)
    lr = F(0.01)
    with sp.Executor(4, 8, S(sp.SUPERPIPELINE, 2, 1)) as ex:
        ex.register_model(model)
        with pytest.raises(sp.SpError):
            ex.read_optimizer_state(0)  # SGD has no state
        with pytest.raises(sp.InvalidArgument):
            ex.set_optimizer(sp.OPT_ADAMW, beta1=1.0)
        with pytest.raises(sp.InvalidArgument):
            ex.set_optimizer(7)
        ex.train_step(x, y, lr)
        sgd = ex.read_model(model)
        _, Ws, bs = ORC.train_step(model.W, model.b, x, y, lr)
        assert np.array_equal(sgd.W, Ws)  # default stays the reference's SGD
        ex.register_model(model)
        ex.set_optimizer(sp.OPT_ADAMW, **HP)
        ex.train_step(x, y, lr)
        a1 = ex.read_model(model)
        assert not np.array_equal(a1.W, sgd.W)
        # reset: re-register the weights, set_optimizer again -> step 1 from zero moments
        ex.register_model(model)
        ex.set_optimizer(sp.OPT_ADAMW, **HP)
        ex.train_step(x, y, lr)
        assert np.array_equal(ex.read_model(model).W, a1.W)
        ex.register_model(model)
        ex.set_optimizer(sp.OPT_SGD)
        ex.train_step(x, y, lr)
        assert np.array_equal(ex.read_model(model).W, Ws)


@pytest.mark.parametrize("numerics", [sp.EXACT, sp.BF16])
def test_adamw_dp_code_path_single_rank(numerics):
    """World 1 through both DP modes: all-reduce (full image AdamW) and sharded (reduce-scatter,
    AdamW on this rank's shard of [W|b], m, v; shard write-back; dp_sync gathers all three)."""
    d = 16 if numerics == sp.EXACT else 128
    rows = 5 if numerics == sp.EXACT else 640
    model = sp.build_model(41, 5, d, 1)
    batches = [(sp.make_input(41, 0, rows, d), sp.make_input(41, 1, rows, d))]
    lr = F(0.01)
    outs = {}
    for dp in (None, "allreduce", "sharded"):
        for s in (S(sp.SUPERPIPELINE, 2, 1), S(sp.STANDARD)):
            outs[(dp, s.kind)] = run_adamw(model, batches, lr, 3, s, numerics=numerics, dp=dp, **HP)
    base = outs[(None, sp.SUPERPIPELINE)]
    if numerics == sp.EXACT:
        ref = oracle_adamw(model, batches, lr, 3, **HP)
        for key, got in outs.items():
            assert same(got[1:], ref[1:]), key
            assert [x.tobytes() for x in got[0]] == [x.tobytes() for x in ref[0]], key
    else:
        for dp in ("allreduce", "sharded"):  # each DP mode window-invariant, and both equal
            assert same(outs[(dp, sp.SUPERPIPELINE)], outs[(dp, sp.STANDARD)]), dp
        assert same(outs[("allreduce", sp.SUPERPIPELINE)], outs[("sharded", sp.SUPERPIPELINE)])
        assert same(base, outs[(None, sp.STANDARD)])
        # the DP path reduces the split-K partials in another order: same update to ~1e-3
        got = outs[("sharded", sp.SUPERPIPELINE)]
        for g, r in zip(got[1:], base[1:]):
            assert np.linalg.norm(g - r) <= 1e-3 * max(np.linalg.norm(r), 1e-30) + 1e-6


def norm_err(got, ref):
    return float(np.linalg.norm((got - ref).ravel()) / max(np.linalg.norm(ref.ravel()), 1e-30))


# bf16 gradients (tcgen05, bf16 activations) drive AdamW: the first moment is linear in the
# gradient (BF16_UPD_TOL of the SGD tests), the second quadratic (2x). AdamW's update
# m / sqrt(v) normalises each element, so where the gradient is near zero a bf16 gradient
# error changes the step by O(lr): the weight change is checked normwise at a looser bound.
BF16_M_TOL, BF16_V_TOL, BF16_STEP_TOL = 5e-2, 1e-1, 2e-1


@pytest.mark.parametrize("d,rows", [(192, 640), (256, 2048)])
def test_adamw_bf16_window_invariant_and_close(d, rows):
    model = sp.build_model(17, 6, d, 1)
    batches = [(sp.make_input(17, 0, rows, d), sp.make_input(17, 1, rows, d))]
    lr = F(0.001)
    ref = oracle_adamw(model, batches, lr, 2, **HP)
    results = []
    for s in (S(sp.STANDARD), S(sp.SUPERPIPELINE, 2, 1), S(sp.SUPERPIPELINE, 4, 2)):
        for ckpt in (False, True):
            results.append(run_adamw(model, batches, lr, 2, s, numerics=sp.BF16, ckpt=ckpt, **HP))
    for r in results[1:]:
        assert same(r, results[0])
    got = results[0]
    assert np.array_equal(got[1][0], model.W[0])  # frozen layer untouched
    assert norm_err(got[3][1:], ref[3][1:]) <= BF16_M_TOL, norm_err(got[3][1:], ref[3][1:])
    assert norm_err(got[4][1:], ref[4][1:]) <= BF16_M_TOL
    assert norm_err(got[5][1:], ref[5][1:]) <= BF16_V_TOL, norm_err(got[5][1:], ref[5][1:])
    dW_got, dW_ref = got[1][1:] - model.W[1:], ref[1][1:] - model.W[1:]
    assert norm_err(dW_got, dW_ref) <= BF16_STEP_TOL, norm_err(dW_got, dW_ref)
    assert abs(float(got[0][-1]) - float(ref[0][-1])) <= 2e-2 * abs(float(ref[0][-1]))


@pytest.mark.parametrize("numerics", [sp.EXACT, sp.BF16])
def test_adamw_trains_and_survives_graph_replay_over_many_steps(numerics):
    """20 steps from pinned host buffers, so each call replays one captured CUDA graph whose
    AdamW scalars are re-read from device memory (refreshed per call): exact numerics stay
    bitwise equal to the oracle, bf16 replays equal an eager (uncaptured) run bitwise, and
    the loss falls."""
    d = 16 if numerics == sp.EXACT else 128
    rows = 8 if numerics == sp.EXACT else 256
    model = sp.build_model(3, 4, d, 0)
    x, t = sp.make_input(3, 0, rows, d), sp.make_input(3, 1, rows, d)
    hx, ht = sp.HostBuffer(x.shape), sp.HostBuffer(t.shape)
    hx.array[...] = x
    ht.array[...] = t
    lr = F(0.003)

    def run(pinned):
        with sp.Executor(4, d, S(sp.SUPERPIPELINE, 2, 1), numerics=numerics) as ex:
            ex.register_model(model)
            ex.set_optimizer(sp.OPT_ADAMW, **HP)
            if pinned:
                losses = [np.float32(ex.train_step_ptr(hx.ptr, ht.ptr, rows, lr, device=False))
                          for _ in range(20)]
                assert ex.stats()["graph_replays"] >= 18
            else:
                losses = [np.float32(ex.train_step(x.copy(), t.copy(), lr)) for _ in range(20)]
            return losses, ex.read_model(model), [ex.read_optimizer_state(L) for L in range(4)]

    g_losses, g_model, g_state = run(True)
    e_losses, e_model, e_state = run(False)
    assert [v.tobytes() for v in g_losses] == [v.tobytes() for v in e_losses]
    assert np.array_equal(g_model.W, e_model.W) and np.array_equal(g_model.b, e_model.b)
    for a, b in zip(g_state, e_state):
        assert all(np.array_equal(u, v) for u, v in zip(a, b))
    if numerics == sp.EXACT:
        ref = oracle_adamw(model, [(x, t)], lr, 20, **HP)
        assert np.array_equal(g_model.W, ref[1]) and np.array_equal(g_model.b, ref[2])
        assert [v.tobytes() for v in g_losses] == [v.tobytes() for v in ref[0]]
    assert g_losses[-1] < g_losses[0]


@pytest.mark.parametrize("n,strats", [
    (1, [S(sp.STANDARD), S(sp.NAIVE, 1)]),                                 # a single layer
    (3, [S(sp.SUPERPIPELINE, 2, 1), S(sp.SUPERPIPELINE, 3, 2), S(sp.NAIVE, 3),
         S(sp.SUPERPIPELINE, 2, 1, sp.SEQUENTIAL)]),                      # ring covers every layer
])
def test_adamw_edge_windows_and_digest_after_deferred_writeback(n, strats):
    """Edge windows (one layer; a ring holding the whole model, so every write-back is deferred;
    sequential transfers): AdamW stays bit-identical to the oracle, and digest_train over the
    executor's host master (which must first complete the deferred write-backs) equals the
    reference's digest of the oracle's weights."""
    model = sp.build_model(9, n, 8, 0)
    batches = [(sp.make_input(9, 0, 5, 8), sp.make_input(9, 1, 5, 8))]
    lr = F(0.02)
    ref = oracle_adamw(model, batches, lr, 3, **HP)
    for s in strats:
        with sp.Executor(n, 8, s) as ex:
            ex.register_model(model)
            ex.set_optimizer(sp.OPT_ADAMW, **HP)
            losses = [np.float32(ex.train_step(batches[0][0], batches[0][1], lr)) for _ in range(3)]
            digest = ex.digest_train(float(losses[-1]))  # no read before: flushes pending write-backs
            m = ex.read_model(model)
        assert [x.tobytes() for x in losses] == [x.tobytes() for x in ref[0]], s
        assert np.array_equal(m.W, ref[1]) and np.array_equal(m.b, ref[2]), s
        assert digest == ORC.digest_train(ref[0][-1], ref[1], ref[2]), s


@pytest.mark.parametrize("numerics", [sp.BF16, sp.TF32])
def test_adamw_at_a_large_layer_is_window_invariant(numerics):
    """d = 4096 (a 64 MB fp32 layer, 192 MB with its moments), where the split-K dW, the
    write-back stages and the 3-region staging copy run at their largest: every window gives the
    same bits, and the moments are finite and nonzero."""
    n, d, rows = 5, 4096, 512
    model = sp.build_model(37, n, d, 0)
    x, t = sp.make_input(37, 0, rows, d), sp.make_input(37, 1, rows, d)
    outs = []
    for s in (S(sp.SUPERPIPELINE, 2, 1), S(sp.SUPERPIPELINE, 3, 1), S(sp.STANDARD)):
        with sp.Executor(n, d, s, numerics=numerics) as ex:
            ex.register_model(model)
            ex.set_optimizer(sp.OPT_ADAMW, **HP)
            losses = [ex.train_step(x, t, F(0.001)) for _ in range(2)]
            m = ex.read_model(model)
            mW, mb, vW, vb = ex.read_optimizer_state(n - 1)
        outs.append((losses, m.W, m.b, mW, vW))
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        assert all(np.array_equal(u, v) for u, v in zip(o[1:], outs[0][1:]))
    assert np.isfinite(outs[0][3]).all() and np.abs(outs[0][3]).max() > 0 and (outs[0][4] >= 0).all()

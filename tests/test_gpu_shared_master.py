"""One pinned host master shared by several executors / processes (sp_share_host_master,
SURVEY 8e: every rank of a node streams from one shared pinned copy)."""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

import paper_2410_08791_b200 as sp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def S(kind, k=0, kp=0):
    return sp.StrategyConfig(kind, k, kp)


@pytest.mark.parametrize("numerics", [sp.EXACT, sp.BF16])
def test_attached_executor_sees_the_creators_layers_and_updates(numerics):
    d = 16 if numerics == sp.EXACT else 128
    model = sp.build_model(4, 6, d, 1)
    x, t = sp.make_input(4, 0, 8, d), sp.make_input(4, 1, 8, d)
    name = f"/sp_test_{uuid.uuid4().hex[:12]}"
    with sp.Executor(6, d, S(sp.SUPERPIPELINE, 2, 1), numerics=numerics) as a, \
            sp.Executor(6, d, S(sp.SUPERPIPELINE, 3, 1), numerics=numerics) as b:
        a.register_model(model)
        a.share_host_master(name, create=True)
        b.share_host_master(name, create=False)  # no registration: layers + flags come from A
        assert np.array_equal(a.forward([x])[0], b.forward([x])[0])
        a.train_step(x, t, 0.05)
        a.train_step(x, t, 0.05)
        wa = a.read_model(model)  # completes A's deferred write-backs into the shared copy
        wb = b.read_model(model)
        assert np.array_equal(wa.W, wb.W) and np.array_equal(wa.b, wb.b)
        assert not np.array_equal(wa.W[1:], model.W[1:]) and np.array_equal(wa.W[0], model.W[0])
        assert np.array_equal(a.forward([x])[0], b.forward([x])[0])  # B re-streams the update
        with pytest.raises(sp.SpError):
            b.share_host_master(name, create=False)  # already shared


def test_attach_rejects_a_missing_or_mismatched_segment():
    name = f"/sp_test_{uuid.uuid4().hex[:12]}"
    with sp.Executor(4, 16, S(sp.STANDARD)) as a:
        with pytest.raises(sp.SpError):
            a.share_host_master(name, create=False)  # nothing to attach to
        a.register_model(sp.build_model(1, 4, 16, 0))
        a.share_host_master(name, create=True)
        with sp.Executor(4, 32, S(sp.STANDARD)) as other:
            with pytest.raises(sp.SpError):
                other.share_host_master(name, create=False)  # another model's size


def test_another_process_streams_from_the_shared_copy(tmp_path):
    d = 128
    model = sp.build_model(8, 5, d, 0)
    x = sp.make_input(8, 0, 32, d)
    name = f"/sp_test_{uuid.uuid4().hex[:12]}"
    with sp.Executor(5, d, S(sp.SUPERPIPELINE, 2, 1), numerics=sp.BF16) as a:
        a.register_model(model)
        a.share_host_master(name, create=True)
        a.train_step(x, x, 0.05)
        a.read_model(model)  # flush
        want = a.forward([x])[0]
        np.save(tmp_path / "x.npy", x)
        code = (
            "import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_2410_08791_b200 as sp\n"
            "x = np.load(%r)\n"
            "with sp.Executor(5, %d, sp.StrategyConfig(sp.SUPERPIPELINE, 3, 1), numerics=sp.BF16) as b:\n"
            "    b.share_host_master(%r, create=False)\n"
            "    np.save(%r, b.forward([x])[0])\n"
        ) % (ROOT, str(tmp_path / "x.npy"), d, name, str(tmp_path / "y.npy"))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert np.array_equal(np.load(tmp_path / "y.npy"), want)


@pytest.mark.parametrize("shard", [True, False])
def test_shared_master_through_the_dp_code_path(shard):
    """A 1-rank communicator over a shared master: sharded (dp_sync is then a barrier for the
    weights, the moments still gather) and all-reduce streaming both stay bit-identical to the
    oracle in exact numerics, with AdamW."""
    from test_gpu_adamw import HP, F, oracle_adamw
    d = 16
    model = sp.build_model(12, 5, d, 1)
    batches = [(sp.make_input(12, 0, 6, d), sp.make_input(12, 1, 6, d))]
    lr = F(0.01)
    ref = oracle_adamw(model, batches, lr, 3, **HP)
    name = f"/sp_test_{uuid.uuid4().hex[:12]}"
    with sp.Executor(5, d, S(sp.SUPERPIPELINE, 2, 1)) as ex:
        ex.register_model(model)
        ex.share_host_master(name, create=True)
        ex.dp_init(sp.Executor.nccl_unique_id(), 0, 1, shard_weights=shard)
        ex.set_optimizer(sp.OPT_ADAMW, **HP)
        losses = [np.float32(ex.train_step(*batches[0], lr)) for _ in range(3)]
        ex.dp_sync()
        m = ex.read_model(model)
        st = [ex.read_optimizer_state(L) for L in range(5)]
    assert [v.tobytes() for v in losses] == [v.tobytes() for v in ref[0]]
    assert np.array_equal(m.W, ref[1]) and np.array_equal(m.b, ref[2])
    assert np.array_equal(np.stack([s[0] for s in st]), ref[3])
    assert np.array_equal(np.stack([s[2] for s in st]), ref[5])

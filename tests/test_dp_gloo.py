"""Data-parallel host logic on CPU with torch.distributed gloo, world_size 2.

The GPU gradient exchange is NCCL inside the executor (only one GPU is available to this
round), so this checks the CONVENTION it implements (paper_2410_08791_b200/dp.py): equal row
shards, MSE gradient scaled by the global element count, per-layer dW/db summed over ranks ==
the full-batch gradient of reference_train_step; loss partial sums likewise. The per-rank
math is the CPU oracle (test infrastructure)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_08791_b200 import dp
    from pyoracle import Oracle
    orc = Oracle()
    n, d, global_rows = 3, 8, 12
    W, b = orc.build_model(5, n, d)
    x = orc.make_input(5, 0, global_rows, d)
    t = orc.make_input(5, 1, global_rows, d)
    start, count = dp.shard_rows(global_rows, rank, world)
    xs, ts = x[start:start + count], t[start:start + count]
    loss_l, _, _, dW_l, db_l, _ = orc.train_step(W, b, xs, ts, 0.01, want_grads=True)
    # Local oracle scales by the LOCAL count; the executor scales by the GLOBAL count.
    scale = count / global_rows
    g = torch.from_numpy(np.concatenate([(dW_l * scale).ravel(), (db_l * scale).ravel()]))
    dist.all_reduce(g)  # the executor's per-layer ncclAllReduce(sum)
    loss_sum = torch.tensor([float(loss_l) * count * d], dtype=torch.float64)
    dist.all_reduce(loss_sum)
    uid = dp.broadcast_unique_id(dist, b"uid-from-rank0" if rank == 0 else None)
    slowest = dp.max_over_ranks(dist, torch, 1.0 + rank)
    if rank == 0:
        out.put((g.numpy(), float(loss_sum.item()) / (global_rows * d), uid, slowest))
    dist.destroy_process_group()


def test_dp_gradient_allreduce_equals_full_batch():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    g, loss, uid, slowest = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = Oracle()
    W, b = orc.build_model(5, 3, 8)
    x, t = orc.make_input(5, 0, 12, 8), orc.make_input(5, 1, 12, 8)
    loss_full, _, _, dW, db, _ = orc.train_step(W, b, x, t, 0.01, want_grads=True)
    full = np.concatenate([dW.ravel(), db.ravel()])
    assert np.allclose(g, full, rtol=1e-5, atol=1e-7)
    assert abs(loss - float(loss_full)) <= 1e-6 * abs(float(loss_full))
    assert uid == b"uid-from-rank0"
    assert slowest == 2.0


def test_shard_rows_requires_equal_shards():
    from paper_2410_08791_b200 import dp
    assert dp.shard_rows(16, 1, 4) == (4, 4)
    with pytest.raises(ValueError):
        dp.shard_rows(10, 0, 4)


def _sharded_worker(rank, world, port, out):
    """Emulates the executor's sharded-streaming step (executor.cpp enqueue_op H2D/ALLGATHER/D2H,
    update_op reduce-scatter + shard SGD, dp_sync) on CPU bytes with gloo collectives, using
    the executor's own shard geometry (sp_debug_shard_range)."""
    import ctypes as C
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_08791_b200 import _capi, dp
    from pyoracle import Oracle
    orc = Oracle()
    n, d, global_rows, lr = 3, 12, 6 * world, 0.05
    W, b = orc.build_model(9, n, d)
    x = orc.make_input(9, 0, global_rows, d)
    t = orc.make_input(9, 1, global_rows, d)
    start, count = dp.shard_rows(global_rows, rank, world)
    img = (d * d + d) * 4
    lo, hi = C.c_uint64(), C.c_uint64()
    shard = int(_capi.LIB.sp_debug_shard_range(img, world, rank, C.byref(lo), C.byref(hi)))
    lo, hi = lo.value, hi.value
    # pinned host master of every rank: [W_l | b_l] fp32 images, registered identically
    host = [np.concatenate([W[l].ravel(), b[l]]).astype(np.float32).view(np.uint8).copy()
            for l in range(n)]
    # forward/backward need the full layers: H2D own shard + all-gather -> full slot image
    slots = []
    for l in range(n):
        mine = np.zeros(shard, np.uint8)
        mine[:hi - lo] = host[l][lo:hi]
        gathered = [torch.zeros(shard, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine))
        slots.append(torch.cat(gathered).numpy()[:img].view(np.float32).copy())
    Ws = np.stack([s[:d * d].reshape(d, d) for s in slots])
    bs = np.stack([s[d * d:] for s in slots])
    assert np.array_equal(Ws, W) and np.array_equal(bs, b)  # the gather rebuilt every layer
    _, _, _, dW, db, _ = orc.train_step(Ws, bs, x[start:start + count], t[start:start + count], lr,
                                        want_grads=True)
    scale = np.float32(count / global_rows)
    for l in range(n):
        # gradient image [dW | db] padded to world*shard bytes, reduce-scattered (sum)
        gimg = np.zeros(world * shard // 4, np.float32)
        gimg[:d * d] = dW[l].ravel() * scale
        gimg[d * d:d * d + d] = db[l] * scale
        full = torch.from_numpy(gimg)
        dist.all_reduce(full)  # gloo: reduce-scatter = all-reduce then keep this rank's shard
        gs = full.numpy()[rank * shard // 4:(rank + 1) * shard // 4]
        # SGD on this rank's shard of the slot, written back to this rank's host master shard
        w32 = slots[l].view(np.uint8)[lo:hi].view(np.float32)
        upd = (w32 - np.float32(lr) * gs[:(hi - lo) // 4]).astype(np.float32)
        host[l][lo:hi] = upd.view(np.uint8)
    stale = [not np.array_equal(host[l], np.concatenate([W[l].ravel(), b[l]]).view(np.uint8))
             for l in range(n)]
    # dp_sync: all-gather the host shards so every rank's master is whole again
    synced = []
    for l in range(n):
        mine = np.zeros(shard, np.uint8)
        mine[:hi - lo] = host[l][lo:hi]
        gathered = [torch.zeros(shard, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine))
        synced.append(torch.cat(gathered).numpy()[:img].view(np.float32).copy())
    out.put((rank, np.stack(synced), any(stale)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_streaming_step_equals_full_batch_step(world):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = Oracle()
    n, d, rows = 3, 12, 6 * world
    W, b = orc.build_model(9, n, d)
    x, t = orc.make_input(9, 0, rows, d), orc.make_input(9, 1, rows, d)
    _, Wn, bn = orc.train_step(W, b, x, t, 0.05)
    want = np.stack([np.concatenate([Wn[l].ravel(), bn[l]]) for l in range(n)])
    imgs = [r[1] for r in sorted(res, key=lambda r: r[0])]
    for img in imgs:  # every rank ends with the same, full-batch-updated master
        assert np.array_equal(img, imgs[0])
        assert np.allclose(img, want, rtol=1e-5, atol=1e-6)
    assert all(r[2] for r in res)  # the step did change the host masters


def _share_worker(rank, world, port, fail_rank, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_08791_b200 import dp

    class FakeExecutor:  # records the calls; the real one needs a GPU (test_gpu_shared_master)
        calls = []

        def share_host_master(self, name, create):
            self.calls.append((name, create))
            if rank == fail_rank:
                raise RuntimeError("no room in /dev/shm")

    ex = FakeExecutor()
    err = dp.share_host_master(ex, dist, rank, "/seg")
    dist.barrier()  # every rank got here: no barrier was skipped
    out.put((rank, ex.calls, err))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 0, 1])
def test_share_host_master_is_collective_even_when_a_rank_fails(fail_rank):
    """Local rank 0 creates the segment, the others attach after a barrier; a failing rank keeps
    its private copy and reports why, and no rank is left waiting at a barrier."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_share_worker, args=(r, 2, port, fail_rank, out)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (calls, err)) for r, calls, err in (out.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == [("/seg", True)] and res[1][0] == [("/seg", False)]
    for r in range(2):
        assert (res[r][1] is not None) == (r == fail_rank)

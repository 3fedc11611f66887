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

"""Data-parallel plumbing around the executor (one process per GPU, torch.distributed for the
host-side rendezvous only; the gradient exchange itself is NCCL inside libsuperpipe.so).

Convention implemented by the executor (csrc/executor.cpp loss_op / update_op):
  * every rank takes an equal shard of `rows` rows of the global batch;
  * the MSE gradient is scaled by 1/(rows * d * world) (the GLOBAL element count), so the
    per-layer dW/db summed over ranks by ncclAllReduce(sum) is the full-batch gradient of
    reference_train_step (model.cpp:157-184) up to summation order;
  * the loss partial sums are all-reduced the same way, so loss = sum / (rows * d * world).
"""
from __future__ import annotations

import os


def dist_env():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard_rows(global_rows: int, rank: int, world: int):
    """Equal row shard [start, start + count) of a global batch (the executor's loss scaling
    assumes equal shards)."""
    if global_rows % world:
        raise ValueError(f"global batch {global_rows} not divisible by world {world}")
    count = global_rows // world
    return rank * count, count


def broadcast_unique_id(dist, uid: bytes | None, src: int = 0) -> bytes:
    """Rank `src` creates the NCCL unique id (Executor.nccl_unique_id()); everyone gets it."""
    box = [uid]
    dist.broadcast_object_list(box, src=src)
    return box[0]


def max_over_ranks(dist, torch, value: float) -> float:
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def init_executor_dp(ex, dist, rank: int, world: int) -> None:
    """Creates the executor's NCCL communicator for per-layer gradient all-reduce."""
    if world <= 1:
        return
    uid = broadcast_unique_id(dist, ex.nccl_unique_id() if rank == 0 else None)
    ex.dp_init(uid, rank, world)


def share_host_master(ex, dist, local_rank: int, name: str) -> str | None:
    """One pinned host master per node: local rank 0 moves its registered master
    into the shared-memory segment `name`, then every other local rank attaches to it (and
    drops its private copy). Collective over the node's ranks; the barriers are always
    reached. Returns None on success, else the error (that rank keeps its private copy)."""
    err = None
    if local_rank == 0:
        try:
            ex.share_host_master(name, create=True)
        except Exception as e:  # e.g. /dev/shm too small: keep the private copy
            err = str(e)
    if dist is not None:
        dist.barrier()
    if local_rank != 0:
        try:
            ex.share_host_master(name, create=False)
        except Exception as e:
            err = str(e)
    if dist is not None:
        dist.barrier()
    return err

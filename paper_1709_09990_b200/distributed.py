"""One wavefront shard per process, launched by torchrun.

torch.distributed is only the plumbing: it hands rank 0's ncclUniqueId to
every rank (a gloo broadcast, no device memory involved) and, for the bench,
takes the max of the ranks' device times. The routing of states to their
owners, the per-round count allgather and the witness broadcast run inside
libelimtw over its own NCCL communicator (shard.cu).

After `init_shards()` every `etw_solve` / `decide` of the process is one shard
of a collective solve: all ranks must make the same sequence of calls on the
same graph and options (SPMD), exactly like the host solver does.
"""
import os
from typing import Optional

from . import elimtw as E


def env_rank():
    """(rank, world_size, local_rank) from the torchrun environment."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def ensure_process_group(backend: str = "gloo"):
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        rank, world, _ = env_rank()
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return dist


def share_unique_id(dist) -> bytes:
    """Rank 0's ncclUniqueId on every rank."""
    uid = E.nccl_unique_id() if dist.get_rank() == 0 else bytes(128)
    box = [uid]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def init_shards(device: Optional[int] = None) -> dict:
    """Make this process shard `rank` of `world_size` (no-op at world 1)."""
    rank, world, local = env_rank()
    if world == 1:
        return E.shard_info()
    dev = local if device is None else device
    # etwg_shard_init re-binds the library's single-device engine (the
    # replicated prefix) to this device too; the variable covers any engine
    # use before it (the engine reads ETWG_DEVICE on first use)
    os.environ.setdefault("ETWG_DEVICE", str(dev))
    dist = ensure_process_group()
    uid = share_unique_id(dist)
    E.shard_init(uid, dist.get_rank(), dist.get_world_size(), dev)
    return E.shard_info()


def max_over_ranks(value: float) -> float:
    """Max of a host float over all ranks (the bench's timing rule)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()

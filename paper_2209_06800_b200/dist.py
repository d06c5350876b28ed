"""One-process-per-GPU plumbing (torch.distributed is plumbing only: the data
path has no collective — remote rows are read in-kernel through imported
CUDA IPC mappings, layers are separated by the K3 device barrier)."""
from __future__ import annotations

import os

import numpy as np

from . import api


def env_world():
    """(world, rank, local_rank) from torchrun's environment (1, 0, 0 alone)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def part_devices(world: int, rank: int, local_rank: int) -> list[int]:
    """Part r is driven by rank r on its local GPU; the others are remote."""
    if not 0 <= rank < world:
        raise api.InputError(f"rank {rank} outside world {world}")
    dev = [-1] * world
    dev[rank] = local_rank
    return dev


def exchange_ipc(engine, rank: int, world: int, group=None) -> None:
    """All-gather every rank's shard handles and import the peers'."""
    import torch.distributed as dist
    blobs = [None] * world
    dist.all_gather_object(blobs, engine.ipc_export(rank), group=group)
    for p in range(world):
        if p != rank:
            if not blobs[p]:
                raise api.InputError(f"rank {p} exported no IPC handles")
            engine.ipc_import(p, blobs[p])


def max_over_ranks(x: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(x: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def rank_plan_summary(g, world: int, rank: int, ps: int, dist_: int, wpb: int, dim: int):
    """Host-side view of rank `rank`'s share (what its engine will upload)."""
    fp = api.build_flat_plan(g, world, rank, ps, dist_, wpb, dim)
    return {"rank": rank, "first_target": fp.first_target, "rows": fp.rows,
            "local_edges": fp.local_cols_len, "remote_edges": fp.remote_cols_len,
            "local_parts": fp.n_local, "remote_parts": fp.n_remote,
            "warps": fp.num_warps, "owners": sorted(set(
                (fp.cols(1) >> np.uint32(28)).tolist())) if fp.remote_cols_len else []}

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
    """Make every peer's shards visible to this rank: CUDA IPC handles
    all-gathered over the process group (default), or — for cross-process
    symmetric VMM stores (MGG_VMM_IPC=1) — POSIX fds passed over Unix sockets
    (exchange_vmm_fds)."""
    import torch.distributed as dist
    modes = [None] * world
    dist.all_gather_object(modes, engine.vmm_ipc(), group=group)
    if len(set(modes)) != 1:
        raise api.ConfigError(f"ranks disagree on the store layout (VMM-IPC per rank: {modes})")
    if modes[0]:
        exchange_vmm_fds(engine, rank, world, group)
        return
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


def exchange_vmm_fds(engine, rank: int, world: int, group=None) -> None:
    """Every rank serves the POSIX fds of its VMM shards (SCM_RIGHTS over an
    abstract-namespace Unix socket) and maps every peer's at the peer's slot
    of its own symmetric ranges (mgg_engine_vmm_import)."""
    import secrets
    import socket
    import threading

    import torch.distributed as dist
    tok = [secrets.token_hex(8) if rank == 0 else None]
    dist.broadcast_object_list(tok, src=0, group=group)
    name = lambda r: f"\0mgg-vmm-{tok[0]}-{r}"  # noqa: E731
    mine = engine.vmm_export(rank)
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(name(rank))
    srv.listen(world)
    err = []

    def serve():
        try:
            for _ in range(world - 1):
                c, _ = srv.accept()
                with c:
                    socket.send_fds(c, [rank.to_bytes(4, "little")], mine)
        except Exception as ex:  # noqa: BLE001
            err.append(ex)

    th = threading.Thread(target=serve, daemon=True)
    th.start()
    dist.barrier(group=group)
    try:
        for q in range(world):
            if q == rank:
                continue
            with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
                c.connect(name(q))
                msg, fds, _, _ = socket.recv_fds(c, 4, len(mine))
                if len(fds) != len(mine) or int.from_bytes(msg, "little") != q:
                    raise api.IntegrityError(f"rank {rank}: bad fd message from rank {q}")
                try:
                    engine.vmm_import(q, fds)
                finally:
                    for fd in fds:
                        os.close(fd)
        th.join(timeout=120)
        if err:
            raise err[0]
    finally:
        srv.close()
        for fd in mine:
            os.close(fd)
    dist.barrier(group=group)

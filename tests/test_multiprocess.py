"""N>1 orchestration on CPU: world_size-2 gloo processes run the same host
logic the torchrun bench runs on GPUs — deterministic graph/split on every
rank, per-rank plans that tile the edge set, IPC-blob exchange, max-over-
ranks timing."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeEngine:
    """Stands in for Engine's IPC surface (no GPU on this box). With vmm=True
    it plays a cross-process VMM store: its 'shards' are temp files whose fds
    travel over the Unix-socket exchange (dist.exchange_vmm_fds)."""

    def __init__(self, rank, vmm=False):
        self.rank = rank
        self.vmm = vmm
        self.imported = {}

    def ipc_export(self, part):
        assert part == self.rank
        return bytes([part]) * 64 * 3

    def ipc_import(self, part, blob):
        self.imported[part] = blob

    def vmm_ipc(self):
        return self.vmm

    def vmm_export(self, part):
        import tempfile
        assert part == self.rank
        fds = []
        for i in range(3):
            fd, path = tempfile.mkstemp()
            os.write(fd, bytes([part]) * (i + 1) * 64)
            os.unlink(path)
            fds.append(fd)
        return fds

    def vmm_import(self, part, fds):
        # the received fds are new descriptors of the peer's open files
        self.imported[part] = b"".join(os.pread(fd, 1024, 0) for fd in fds)


def _worker(rank, world, port, q, vmm=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        import paper_2209_06800_b200 as mgg
        from paper_2209_06800_b200 import dist as mdist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        w, r, lr = mdist.env_world()
        assert (w, r, lr) == (world, rank, rank)
        dev = mdist.part_devices(w, r, lr)
        assert dev[r] == lr and sum(d >= 0 for d in dev) == 1
        g = mgg.gen_synthetic(mgg.POWERLAW, 5000, 12, 0)      # same seed on every rank
        summ = mdist.rank_plan_summary(g, world, rank, 16, 2, 4, 16)
        allsum = [None] * world
        dist.all_gather_object(allsum, (summ, int(g.num_edges), int(g.col_idx.sum())))
        eng = FakeEngine(rank, vmm)
        mdist.exchange_ipc(eng, rank, world)
        assert sorted(eng.imported) == [p for p in range(world) if p != rank]
        want = (lambda p: bytes([p]) * 384) if vmm else (lambda p: bytes([p]) * 192)
        assert all(b == want(p) for p, b in eng.imported.items()), eng.imported
        m = mdist.max_over_ranks(float(rank) * 1.5)
        tot = mdist.sum_over_ranks(float(rank + 1))  # bench's link bytes over ranks
        assert tot == world * (world + 1) / 2
        q.put((rank, allsum, m, None))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, None, None, traceback.format_exc()))


@pytest.mark.parametrize("world,vmm", [(2, False), (3, False), (2, True), (3, True)])
def test_world_orchestration(world, vmm):
    # vmm: the cross-process VMM fd exchange (SCM_RIGHTS over Unix sockets)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, vmm)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, allsum, m, err in res:
        assert err is None, err
        assert m == pytest.approx(1.5 * (world - 1))
        summs = [s for s, _, _ in allsum]
        # every rank generated the identical graph
        assert len({(e, c) for _, e, c in allsum}) == 1
        total_e = allsum[0][1]
        assert sum(s["local_edges"] + s["remote_edges"] for s in summs) == total_e
        # chunks tile [0, N) in rank order
        ends = [s["first_target"] + s["rows"] for s in summs]
        assert [s["first_target"] for s in summs] == [0] + ends[:-1]
        for s in summs:
            assert s["rank"] not in s["owners"]

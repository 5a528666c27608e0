"""Multi-process host logic of the partitioned stepper, world_size 2 over gloo
(CPU only): every rank computes the same slab plan, the plan tiles both line
ranges with balanced active cells, and the NCCL unique id created by rank 0
reaches every rank through torch.distributed."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1912_03744_b200 import configs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1912_03744_b200 import dist as pdist
        out = {}
        for name in ("cfg3", "cfg4", "cfg0"):
            c = configs.CONFIGS[name]()
            g = c.grid()
            for nr in (2, 4, 8):
                zb, rb = pdist.slab_plan(g, c.materials, configs.make_source(c, g), c.timing,
                                         c.solver, nr)
                t = torch.tensor(zb + rb, dtype=torch.int64)
                gathered = [torch.zeros_like(t) for _ in range(world)]
                dist.all_gather(gathered, t)
                out[(name, nr)] = [x.tolist() for x in gathered]
        # the peer-transport handle exchange: equal blocks, rank order
        blob = pdist.allgather_bytes(bytes([rank + 1]) * 256)
        out["blob"] = blob
        uid = pdist.share_unique_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        out["ids"] = ids
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_plan_and_unique_id():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = results[0]
    assert len(set(r0["ids"])) == 1 and len(r0["ids"][0]) == 128
    expect = bytes([1]) * 256 + bytes([2]) * 256
    assert results[0]["blob"] == expect and results[1]["blob"] == expect
    for key, plans in r0.items():
        if key in ("ids", "blob"):
            continue
        assert plans[0] == plans[1], key  # identical plan on every rank
        name, nr = key
        c = configs.CONFIGS[name]()
        g = c.grid()
        zb, rb = plans[0][: nr + 1], plans[0][nr + 1:]
        assert zb[0] == 0 and zb[-1] == g.nz() and rb[0] == 0 and rb[-1] == g.nr()
        assert all(b - a >= 0 for a, b in zip(zb, zb[1:]))
        # balanced by active cells within one line's worth
        zc = [sum(g.row_extent(j) for j in range(a, b)) for a, b in zip(zb, zb[1:])]
        assert max(zc) - min(zc) <= 2 * g.nr()
        rc = [sum(g.col_extent(i) for i in range(a, b)) for a, b in zip(rb, rb[1:])]
        assert max(rc) - min(rc) <= 2 * g.nz()


class _FakeLib:
    """Stands in for libpcgpu's IPC entry points: rank `fail` cannot map its peers."""

    def __init__(self, rank, fail):
        self.rank, self.fail, self.calls = rank, fail, []

    def pcgpu_dist_ipc_export(self, h, buf):
        self.calls.append("export")
        return 0

    def pcgpu_dist_ipc_import(self, h, buf):
        self.calls.append("import")
        return 5 if self.rank == self.fail else 0

    def pcgpu_dist_peer_off(self, h):
        self.calls.append("peer_off")
        return 0


def _transport_worker(rank, world, port, fail, q):
    import warnings
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1912_03744_b200.dist import PartitionedAdi
        part = object.__new__(PartitionedAdi)
        part._lib, part._h = _FakeLib(rank, fail), None
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            on = part.enable_peer_transport()
        q.put((rank, (on, part._lib.calls)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail", [-1, 1])
def test_gloo_world2_peer_transport_agreement(fail):
    """The transport is agreed collectively: when one rank's CUDA IPC import
    fails, every rank drops its peer mapping (pcgpu_dist_peer_off) and all of
    them use the NCCL transport; otherwise all keep the peer transport."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, world, port, fail, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        on, calls = res[r]
        if fail < 0:
            assert on is True and calls == ["export", "import"]
        else:
            assert on is False and calls == ["export", "import", "peer_off"]

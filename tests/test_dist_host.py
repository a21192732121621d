"""Host-side protocol of the multi-GPU factorization (paper_1710_00125_b200.dist) on CPU:
two processes over gloo with the device calls replaced by a recorder.  Checks who allocates,
prepares, exports and imports, that the workers get rank 0's handle and configuration, that
rank 0 prepares before it publishes the handle, and that everything is released."""

import os

import pytest
import torch.multiprocessing as mp


class FakeOps:
    def __init__(self, rank, log):
        self.rank, self.log = rank, log

    def alloc_workspace(self, n, cfg):
        self.log.append(("alloc", n))
        return (0xABC000, 4096)

    def prepare(self, n, cfg, ws):
        self.log.append(("prepare", ws[0]))

    def export(self, ws):
        self.log.append(("export", ws[0]))
        return b"H" * 64

    def free_workspace(self, ws):
        self.log.append(("free", ws[0]))

    def factor(self, a, cfg, ws, world):
        self.log.append(("factor", ws[0] if ws else None, world))
        return "F"

    def import_(self, handle):
        self.log.append(("import", handle))
        return 0xDEF000

    def close(self, ptr):
        self.log.append(("close", ptr))

    def worker(self, plan, rank, ptr):
        self.log.append(("worker", plan.n, plan.b, plan.q, plan.p, plan.world, rank, ptr))


def _body(rank, world, port, q):
    import torch.distributed as dist

    from paper_1710_00125_b200 import FactorConfig, dist as rdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    log = []
    try:
        cfg = FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0)
        import numpy as np
        a = np.zeros((40, 40)) if rank == 0 else None

        class Shape:  # rank 0 only needs .shape
            shape = (40, 40)
        res = rdist.factor_distributed_device(Shape() if rank == 0 else None, cfg, ops=FakeOps(rank, log))
        q.put((rank, res, log))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_protocol_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29611 + world
    procs = [ctx.Process(target=_body, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res, log = q.get(timeout=120)
        out[rank] = (res, log)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res0, log0 = out[0]
    assert res0 == "F"
    kinds = [e[0] for e in log0]
    assert kinds == ["alloc", "prepare", "export", "factor", "free"]
    assert log0[3] == ("factor", 0xABC000, world)
    for r in range(1, world):
        res, log = out[r]
        assert res is None
        assert log[0] == ("import", b"H" * 64)
        assert log[1] == ("worker", 40, 16, 16, 24, world, r, 0xDEF000)
        assert log[2] == ("close", 0xDEF000)


def _plan_body(rank, world, port, q):
    """Each rank asks the C ABI (no GPU) for its share of several panels' updates; the shares are
    exchanged over gloo and rank 0 checks they cover every tile exactly once."""
    import torch.distributed as dist

    from paper_1710_00125_b200 import dist as rdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = {}
        for mp in (1, 100, 128, 129, 1000, 4097, 30100):
            m0, n0, sk = rdist.tile_plan(mp, 0, rank, world, 148)
            mine[mp] = (m0.tolist(), n0.tolist(), sk.tolist())
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        q.put((rank, allp if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tile_dealing_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29711 + world
    procs = [ctx.Process(target=_plan_body, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, payload = q.get(timeout=120)
        res[rank] = payload
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shares = res[0]
    for mpv in (1, 100, 128, 129, 1000, 4097, 30100):
        nbi = (mpv + 127) // 128
        expect = {(I * 128, J * 64) for I in range(nbi) for J in range(2 * I + 2)}
        seen = []
        for r in range(world):
            m0, n0, sk = shares[r][mpv]
            assert not any(sk)  # no fused sketch tiles when the update is shared
            seen += list(zip(m0, n0))
        assert len(seen) == len(expect) and set(seen) == expect, mpv
        sizes = [len(shares[r][mpv][0]) for r in range(world)]
        assert max(sizes) - min(sizes) <= 148, sizes  # round robin: balanced to within one tile per CTA


def test_single_device_plan_includes_sketch_tiles():
    from paper_1710_00125_b200 import dist as rdist
    m0, n0, sk = rdist.tile_plan(1000, 144, 0, 1, 148)
    nbi = (1000 + 127) // 128
    assert int(sk.sum()) == nbi * 3 and len(m0) == nbi * (nbi + 1) + nbi * 3
    assert set(zip(m0[sk].tolist(), n0[sk].tolist())) == {(I * 128, j * 64) for I in range(nbi) for j in range(3)}

"""Multi-GPU partition + halo logic (BASELINE config 5) on CPU.

The per-rank column loop is stood in for by the oracle restricted to the
rank's cells (the CUDA path is covered by test_gpu_parity); the partition,
ownership, window arithmetic and the send/recv/add exchange are the
product's own code, run over a real world_size-2 gloo process group.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import LAYOUT_COUNTS, families, quad_degrees

CASES = ("CG1xCG1", "VP1", "P2xP2", "CG1xDG1")


def _space(n, layers, lname, ordering="rcm"):
    from paper_1604_05937_b200 import DofLayout, ExtrudedMesh, number_dofs
    from paper_1604_05937_b200.configs import base_mesh
    base, _ = base_mesh(n, ordering)
    return number_dofs(ExtrudedMesh(base, layers),
                       DofLayout(lname, LAYOUT_COUNTS[lname]))


def _oracle(fs, lname):
    tri, line, nc = families(lname)
    return oracle.Problem(fs.mesh.base, fs.mesh.layers, LAYOUT_COUNTS[lname],
                          tri, line, nc, *quad_degrees(lname))


@pytest.mark.parametrize("lname", CASES)
@pytest.mark.parametrize("world", (2, 3, 4, 8))
def test_partition_properties(lname, world):
    from paper_1604_05937_b200.shard import partition
    fs = _space(8, 3, lname)
    shards = partition(fs, world)
    cells = np.concatenate([s.cells for s in shards])
    assert np.array_equal(cells, np.arange(fs.mesh.base.num_cells))
    for d in shards[0].owned:
        owned = np.concatenate([s.owned[d] for s in shards])
        n = fs.mesh.base.entity_count(d)
        assert np.array_equal(np.sort(owned), np.arange(n)), "own exactly once"
    for s in shards:
        for q, ids in s.send.items():
            for d, v in ids.items():
                assert np.array_equal(shards[q].recv[s.rank][d], v)
                assert q < s.rank    # the owner is the lowest touching block
                assert np.isin(v, shards[q].owned[d]).all()


@pytest.mark.parametrize("lname", CASES)
@pytest.mark.parametrize("world", (2, 4))
def test_partials_sum_to_global(lname, world):
    """Single-process emulation: per-rank windows + exchange == global."""
    from paper_1604_05937_b200.shard import ghost_origins, partition
    fs = _space(8, 3, lname)
    prob = _oracle(fs, lname)
    x = np.random.default_rng(0).random(fs.total_dofs)
    full = prob.assemble(x)
    shards = partition(fs, world)
    wins = []
    for s in shards:
        part = prob.assemble(x, order=s.cells)
        lo, hi = s.window
        outside = np.ones(fs.total_dofs, bool)
        outside[lo:hi] = False
        assert not np.any(part[outside]), "writes outside the window"
        wins.append(part[lo:hi].copy())
    for s in shards:
        for q, ids in s.send.items():
            for _d, o, c in ghost_origins(fs, ids):
                for org in o:
                    src = slice(org - s.window[0], org - s.window[0] + c)
                    dst = slice(org - shards[q].window[0],
                                org - shards[q].window[0] + c)
                    wins[q][dst] += wins[s.rank][src]
    for s in shards:
        for _d, o, c in ghost_origins(fs, s.owned):
            for org in o:
                got = wins[s.rank][org - s.window[0]:org - s.window[0] + c]
                np.testing.assert_allclose(got, full[org:org + c], rtol=0,
                                           atol=1e-15)


def _cpu_pack(lo):
    def pack(y, origins, col):
        idx = (origins[:, None] - lo + torch.arange(col)).reshape(-1)
        return y[idx].clone()

    def unpack(y, origins, col, buf):
        idx = (origins[:, None] - lo + torch.arange(col)).reshape(-1)
        y.index_add_(0, idx, buf)
    return pack, unpack


def _worker(rank, world, port, lname, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1604_05937_b200.shard import (HaloExchange, ghost_origins,
                                                 partition)
        fs = _space(8, 4, lname)
        prob = _oracle(fs, lname)
        x = np.random.default_rng(1).random(fs.total_dofs)
        s = partition(fs, world)[rank]
        lo, hi = s.window
        y = torch.from_numpy(prob.assemble(x, order=s.cells)[lo:hi].copy())
        pack, unpack = _cpu_pack(lo)
        HaloExchange(fs, s, pack=pack, unpack_add=unpack).exchange(y)
        full = prob.assemble(x)
        err = 0.0
        for _d, o, c in ghost_origins(fs, s.owned):
            for org in o:
                got = y[org - lo:org - lo + c].numpy()
                err = max(err, float(np.abs(got - full[org:org + c]).max()))
        dist.destroy_process_group()
        q.put((rank, err))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1", "P2xP2"))
def test_gloo_world2_exchange(lname):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lname, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], float), res[r]
        assert res[r] <= 1e-15

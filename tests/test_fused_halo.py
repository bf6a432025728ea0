"""Fused halo: the strip kernel adds ghost vertex columns
straight into the owning rank's window (peer memory) instead of a
pack / send / recv / owner-add exchange.

* CPU: the applicability plan (ghosts owned by the rank below and lying
  under the rank's first owned vertex) on RCM / random meshes, 2–8 ranks.
* GPU, one process: every rank's window on one device, each rank's kernel
  given the window of the rank below as its peer — the kernel's ghost
  redirect and global-index addressing against the oracle.
* GPU, two processes on one device: the whole product path —
  ``ShardedMassOperator(fused=True)``: CUDA IPC export / open of the
  windows, zero → barrier → kernel → barrier (host barriers only: no kernel
  waits on another).
"""
import os
import socket

import numpy as np
import pytest

import oracle
from conftest import LAYOUT_COUNTS, families, quad_degrees


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


@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1"))
@pytest.mark.parametrize("world", (2, 3, 4, 8))
def test_plan_on_rcm_blocks(lname, world):
    from paper_1604_05937_b200.shard import fused_halo_plan, partition
    fs = _space(16, 3, lname)
    shards = partition(fs, world)
    plan = fused_halo_plan(fs, shards)
    assert plan is not None and plan[0] == 0
    for s, end in zip(shards, plan):
        t, own = s.dim_entities[0], s.owned[0]
        ghosts = np.setdiff1d(t, own)
        assert np.all(ghosts < end) and np.all(own >= end)
        if s.rank:
            # ghosts belong to the rank below, i.e. inside its window
            below = shards[s.rank - 1]
            assert np.isin(ghosts, below.owned[0]).all()


@pytest.mark.parametrize("lname", ("P2xP2", "CG1xDG1", "DG1xDG1"))
def test_plan_refuses_other_layouts(lname):
    from paper_1604_05937_b200.shard import fused_halo_plan, partition
    fs = _space(8, 2, lname)
    if lname == "CG1xDG1":      # vertex-only: applies
        assert fused_halo_plan(fs, partition(fs, 2)) is not None
    else:
        assert fused_halo_plan(fs, partition(fs, 2)) is None


def test_plan_refuses_scattered_ownership():
    """A random vertex order breaks 'ghosts below the first owned vertex'."""
    from paper_1604_05937_b200.shard import fused_halo_plan, partition
    fs = _space(16, 2, "CG1xCG1", ordering="random")
    assert fused_halo_plan(fs, partition(fs, 4)) is None


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1", "CG1xDG1"))
@pytest.mark.parametrize("world", (2, 3, 4))
def test_fused_kernel_windows_on_one_gpu(lname, world):
    import torch
    from paper_1604_05937_b200 import _lib, configs, extrude_coordinates
    from paper_1604_05937_b200.shard import (ShardedMassOperator,
                                             fused_halo_plan, ghost_origins,
                                             partition)
    w = configs.Workload("c5-fused", 24, 6, lname, quad_degrees(lname))
    fs, quad, x, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    ref = _oracle(fs, lname).assemble(x)
    xd = torch.from_numpy(x).cuda()
    plan = fused_halo_plan(fs, partition(fs, world))
    ops = [ShardedMassOperator(fs, r, world, quad) for r in range(world)]
    wins = [torch.zeros(op.window[1] - op.window[0], dtype=torch.float64,
                        device="cuda") for op in ops]
    for r, op in enumerate(ops):
        lo, hi = op.window
        clo, chi = op.shard.coord_window
        peer = (wins[r - 1].data_ptr() - 8 * ops[r - 1].window[0]) if r else 0
        strips, W = op.strips
        _lib.column_mass_strip_red_peer(
            fs.layout, op.op.k, m.layers, coords[clo:chi].clone(), op.op.mref,
            xd[lo:hi].clone(), wins[r], hi - lo, strips, op.op.kron, W, peer,
            plan[r] if r else 0, accumulate=True, x_base=lo, y_base=lo,
            coords_base=clo, n_vertices=m.base.num_vertices)
    torch.cuda.synchronize()
    got = np.zeros_like(ref)
    for op, win in zip(ops, wins):
        yw = win.cpu().numpy()
        for _d, o, c in ghost_origins(fs, op.shard.owned):
            for org in o:
                a = org - op.window[0]
                got[org:org + c] = yw[a:a + c]
    assert np.abs(got - ref).max() <= 1e-10 * np.abs(ref).max()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _ipc_worker(rank, world, port, lname, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1604_05937_b200 import configs, extrude_coordinates
        from paper_1604_05937_b200.shard import (ShardedMassOperator,
                                                 ghost_origins)
        w = configs.Workload("c5-ipc", 20, 5, lname, quad_degrees(lname))
        fs, quad, x, _ = configs.build(w)
        m = fs.mesh
        coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
        op = ShardedMassOperator(fs, rank, world, quad, fused=True)
        lo, hi = op.window
        clo, chi = op.shard.coord_window
        xd = torch.from_numpy(x[lo:hi].copy()).cuda()
        yw = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        op.connect(yw)                  # CUDA IPC: the windows and flags
        import oracle
        from paper_1604_05937_b200 import _lib
        from paper_1604_05937_b200.quadrature import element_for_layout
        el = element_for_layout(fs.layout)
        full = oracle.Problem(m.base, m.layers, fs.layout.counts, el.tri,
                              el.line, el.ncomp, *quad_degrees(lname)
                              ).assemble(x)
        err = 0.0
        strips, W = op.strips
        for _rep in range(2):              # the window is reused per step
            # the fused kernel through the IPC mapping; the ranks are
            # processes sharing one GPU, so the step is ordered by host
            # barriers here (the stream-ordered flags of apply() are
            # checked as a stream program, test_fused_halo_stream_protocol)
            yw.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            _lib.column_mass_strip_red_peer(
                fs.layout, op.op.k, m.layers, coords[clo:chi].clone(),
                op.op.mref, xd, yw, hi - lo, strips, op.op.kron, W,
                op._peer.y_addr, op.ghost_end if op._peer.y_addr else 0,
                accumulate=True, x_base=lo, y_base=lo, coords_base=clo,
                n_vertices=m.base.num_vertices)
            torch.cuda.synchronize()
            dist.barrier()
            got = yw.cpu().numpy()
            for _d, o, c in ghost_origins(fs, op.shard.owned):
                for org in o:
                    e = np.abs(got[org - lo:org - lo + c] - full[org:org + c])
                    err = max(err, float(e.max()) / float(np.abs(full).max()))
        dist.barrier()
        op._peer.close()
        dist.destroy_process_group()
        q.put((rank, err))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))


@pytest.mark.gpu
@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1"))
def test_fused_halo_two_processes_ipc(lname):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, lname, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], float), res[r]
        assert res[r] <= 1e-10


def _simulate(world, steps, high_first=False):
    """Run every rank's fused-step stream program (one in-order stream per
    rank, as on P GPUs) in an interleaving that always advances the
    lowest (or highest) runnable rank as far as it can; returns the global
    event order.  Raises on a deadlock."""
    from paper_1604_05937_b200.shard import fused_step_program
    progs = [[op for s in range(1, steps + 1)
              for op in fused_step_program(r, world, s)]
             for r in range(world)]
    flags = [[0, 0] for _ in range(world)]
    pc = [0] * world
    events = []
    while any(pc[r] < len(progs[r]) for r in range(world)):
        progressed = False
        for r in (range(world - 1, -1, -1) if high_first else range(world)):
            while pc[r] < len(progs[r]):
                op = progs[r][pc[r]]
                if op[0] == "wait" and flags[r][op[1]] < op[2]:
                    break
                if op[0] == "signal":
                    flags[op[1]][op[2]] = op[3]
                step = sum(1 for o in progs[r][:pc[r] + 1] if o[0] == "zero")
                events.append((r, op[0], step))
                pc[r] += 1
                progressed = True
        if not progressed:
            raise AssertionError(f"deadlock at {pc}")
    return events


@pytest.mark.parametrize("world", (1, 2, 3, 4, 8))
@pytest.mark.parametrize("order", ("low-first", "high-first"))
def test_fused_halo_stream_protocol(world, order):
    """The stream-ordered fused step (no host synchronisation between
    ranks) makes progress for any rank speed, and orders every step's
    memory effects: rank r's kernel adds into rank r-1's window only after
    r-1 zeroed it for that step, and r-1 zeroes its window for the next
    step only after those adds landed.  (Checked as a stream program on
    the CPU: ranks whose streams wait on one another must not be
    emulated on one GPU, B200_PROFILING.md.)"""
    from paper_1604_05937_b200.shard import fused_step_program
    steps = 4
    ev = _simulate(world, steps, high_first=order == "high-first")
    pos = {e: i for i, e in enumerate(ev)}
    for s in range(1, steps + 1):
        for r in range(1, world):
            assert pos[(r - 1, "zero", s)] < pos[(r, "kernel", s)]
            if s < steps:
                assert pos[(r, "kernel", s)] < pos[(r - 1, "zero", s + 1)]
    for r in range(world):
        prog = fused_step_program(r, world, 7)
        assert prog[0] == ("zero",) and ("kernel",) in prog

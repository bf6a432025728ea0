"""Base-mesh partitioning across GPUs (BASELINE config 5).

The paper decomposes the *base* mesh between MPI ranks and notes that the
column numbering is orthogonal to that decomposition (PAPER.md:463-465,
770-775; the SPEC drops MPI).  Here one process drives one GPU:

* rank p takes the p-th contiguous block of the (RCM-ordered) base cells
  (``np.array_split``); columns are never split, the numbering stays the
  global one, so every rank's maps are rows of the global maps;
* a DoF-carrying base entity (vertex, edge) is owned by the lowest rank
  whose block touches it;
* each rank runs the column loop over its own cells into a window of the
  global field that covers every entity its cells touch, then sends the
  partial columns of the entities it touches but does not own to their
  owners, which add them (one grouped send/recv per neighbour pair, NCCL
  on GPUs, gloo in the CPU tests).

After the exchange each rank holds the final values of its owned entity
columns; nothing else is communicated (inputs are replicated at setup).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Shard:
    rank: int
    world: int
    cells: np.ndarray                 # int32 global cell ids (contiguous)
    dim_entities: dict                # d -> touched entity ids (sorted)
    owned: dict                       # d -> owned entity ids (sorted)
    send: dict = field(default_factory=dict)   # peer -> {d: ids}
    recv: dict = field(default_factory=dict)   # peer -> {d: ids}
    window: tuple = (0, 0)            # [lo, hi) DoFs touched by the block
    coord_window: tuple = (0, 0)      # [lo, hi) coordinate DoFs touched


def _entities(base, d):
    if d == 0:
        return np.asarray(base.cell_vertices, dtype=np.int64)
    if d == 1:
        return np.asarray(base.cell_edges, dtype=np.int64)
    raise ValueError("only vertex / edge entities are shared")


def partition(fs, world: int):
    """Per-rank Shard descriptions for space ``fs`` (host, deterministic)."""
    base = fs.mesh.base
    layout = fs.layout
    dims = [d for d in (0, 1) if layout.dofs(d, 0) or layout.dofs(d, 1)]
    if layout.dofs(2, 0) or layout.dofs(2, 1):
        if dims:
            raise ValueError("mixed cell + vertex/edge layouts not sharded")
    n_cells = base.num_cells
    blocks = np.array_split(np.arange(n_cells, dtype=np.int64), world)
    block_of = np.empty(n_cells, dtype=np.int64)
    for p, b in enumerate(blocks):
        block_of[b] = p
    owner = {}
    for d in dims:
        ents = _entities(base, d)
        own = np.full(base.entity_count(d), world, dtype=np.int64)
        np.minimum.at(own, ents.ravel(), np.repeat(block_of, ents.shape[1]))
        owner[d] = own
    layers = fs.mesh.layers
    shards = []
    for p, b in enumerate(blocks):
        touched = {d: np.unique(_entities(base, d)[b].ravel()) for d in dims}
        owned = {d: touched[d][owner[d][touched[d]] == p] for d in dims}
        s = Shard(rank=p, world=world, cells=b.astype(np.int32),
                  dim_entities=touched, owned=owned)
        # window of global DoFs touched by the block
        lo, hi = [], []
        if dims:
            for d in dims:
                if touched[d].size:
                    col = fs.column_sizes[d]
                    start = fs.origin_starts[d]
                    lo.append(start + col * int(touched[d][0]))
                    hi.append(start + col * (int(touched[d][-1]) + 1))
        elif b.size:
            col = fs.column_sizes[2]
            start = fs.origin_starts[2]
            lo.append(start + col * int(b[0]))
            hi.append(start + col * (int(b[-1]) + 1))
        s.window = (min(lo), max(hi)) if lo else (0, 0)
        if b.size:
            vt = np.unique(np.asarray(base.cell_vertices)[b].ravel())
            s.coord_window = (3 * (layers + 1) * int(vt[0]),
                              3 * (layers + 1) * (int(vt[-1]) + 1))
        shards.append(s)
    # halo lists: entities touched by p, owned by q != p
    for s in shards:
        for d in dims:
            t = s.dim_entities[d]
            o = owner[d][t]
            for q in np.unique(o[o != s.rank]):
                ids = t[o == q]
                s.send.setdefault(int(q), {})[d] = ids
                shards[int(q)].recv.setdefault(s.rank, {})[d] = ids
    return shards


def ghost_origins(fs, ids_by_dim):
    """DoF origins (int64) and column length per dim of an entity list."""
    out = []
    for d in sorted(ids_by_dim):
        ids = np.asarray(ids_by_dim[d], dtype=np.int64)
        col = fs.column_sizes[d]
        out.append((d, fs.origin_starts[d] + col * ids, col))
    return out


class HaloExchange:
    """Grouped send/recv of ghost partial columns, owner adds.

    ``pack(y, origins, col) -> buf`` and ``unpack_add(y, origins, col,
    buf)`` default to the CUDA kernels ``pm_halo_pack`` /
    ``pm_halo_unpack_add``; ``y`` is the rank's window tensor and origins
    are global DoF numbers (``base`` = window start).
    """

    def __init__(self, fs, shard: Shard, pack=None, unpack_add=None,
                 device=None):
        import torch
        self.fs = fs
        self.shard = shard
        self.lo = shard.window[0]
        dev = device or "cpu"
        self.send = {q: [(d, torch.from_numpy(o).to(dev), c)
                         for d, o, c in ghost_origins(fs, ids)]
                     for q, ids in sorted(shard.send.items())}
        self.recv = {q: [(d, torch.from_numpy(o).to(dev), c)
                         for d, o, c in ghost_origins(fs, ids)]
                     for q, ids in sorted(shard.recv.items())}
        self._pack = pack or self._cuda_pack
        self._unpack = unpack_add or self._cuda_unpack

    def _cuda_pack(self, y, origins, col):
        import torch
        from . import _lib
        buf = torch.empty(origins.shape[0] * col, dtype=y.dtype,
                          device=y.device)
        _lib.halo_pack(y, origins, col, buf, base=self.lo)
        return buf

    def _cuda_unpack(self, y, origins, col, buf):
        from . import _lib
        _lib.halo_unpack_add(y, origins, col, buf, base=self.lo)

    def bytes_per_exchange(self):
        n = 0
        for lst in self.send.values():
            n += sum(o.shape[0] * c for _d, o, c in lst) * 8
        return n

    def exchange(self, y, group=None):
        """Send ghost partials to owners, add received partials (in place)."""
        import torch
        import torch.distributed as dist
        ops, inbox = [], []
        for q, lst in self.send.items():
            for _d, o, c in lst:
                ops.append(dist.P2POp(dist.isend, self._pack(y, o, c), q,
                                      group=group))
        for q, lst in self.recv.items():
            for _d, o, c in lst:
                buf = torch.empty(o.shape[0] * c, dtype=y.dtype,
                                  device=y.device)
                inbox.append((o, c, buf))
                ops.append(dist.P2POp(dist.irecv, buf, q, group=group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for o, c, buf in inbox:
            self._unpack(y, o, c, buf)
        return y


def fused_halo_plan(fs, shards):
    """Ghost-vertex bound per rank for the fused halo, or None.

    The fused kernel (``pm_column_mass_strip_red_peer``) sends a vertex's
    partial columns to the rank below when its id is under a bound, so it
    applies when (true for RCM-ordered meshes): the layout has
    DoFs on vertices only; every rank's ghosts are owned by the rank below
    and lie below its first owned vertex; every touched vertex from there on
    is owned.  Returns ``[bound_p]`` (0 for rank 0).
    """
    layout = fs.layout
    dims = [d for d in (0, 1, 2) if layout.dofs(d, 0) or layout.dofs(d, 1)]
    if dims != [0]:
        return None
    ends = []
    for sh in shards:
        touched, own = sh.dim_entities[0], sh.owned[0]
        if sh.rank == 0:
            if sh.send:
                return None
            ends.append(0)
            continue
        if set(sh.send) - {sh.rank - 1} or own.size == 0:
            return None
        lo = int(own[0])
        if not np.array_equal(np.setdiff1d(touched, own),
                              touched[touched < lo]):
            return None
        ends.append(lo)
    return ends


class PeerWindow:
    """The neighbours' buffers the fused halo needs, mapped into this
    process (CUDA IPC, NVLink peer memory): the y window and step flags of
    the rank below, the step flags of the rank above.  Every rank exports
    its window and flags.  ``y_addr`` is shifted like ``_lib.ptr(t, base)``
    so that global DoF numbers index it; ``down_flags`` / ``up_flags`` are
    device addresses of int32[2] (0 = "window zeroed", 1 = "ghost adds
    landed")."""

    def __init__(self, y_window, flags, lo, rank, world, group=None):
        import torch.distributed as dist
        from . import _lib
        # every step is collective and failure-consistent: a rank that
        # cannot export or map makes all ranks raise (no rank is left
        # waiting in a collective the others skipped)
        try:
            mine = (*_lib.ipc_export(y_window), int(lo),
                    *_lib.ipc_export(flags))
        except Exception as e:  # noqa: BLE001 - reported on every rank
            mine = repr(e)
        infos = [None] * world
        dist.all_gather_object(infos, mine, group=group)
        bad = [i for i in infos if isinstance(i, str)]
        if bad:
            raise RuntimeError(f"fused halo: IPC export failed: {bad[0]}")
        self._open = []
        self.y_addr = self.down_flags = self.up_flags = 0
        err = None
        try:
            if rank > 0:
                h, o, plo, fh, fo = infos[rank - 1]
                base = _lib.ipc_open(h, o)
                self._open.append((base, o))
                self.y_addr = base - 8 * plo
                fb = _lib.ipc_open(fh, fo)
                self._open.append((fb, fo))
                self.down_flags = fb
            if rank < world - 1:
                _h, _o, _plo, fh, fo = infos[rank + 1]
                fb = _lib.ipc_open(fh, fo)
                self._open.append((fb, fo))
                self.up_flags = fb
        except Exception as e:  # noqa: BLE001
            err = repr(e)
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        if any(errs):
            self.close()
            raise RuntimeError(
                f"fused halo: IPC open failed: {next(e for e in errs if e)}")

    def close(self):
        from . import _lib
        for base, o in self._open:
            _lib.ipc_close(base, o)
        self._open = []


def fused_step_program(rank, world, step):
    """The stream program of one fused-halo step on ``rank`` (executed by
    ShardedMassOperator._apply_fused, checked for progress and ordering by
    tests/test_fused_halo.py on the CPU).  Flags are int32[2] per rank:
    [0] "the rank below zeroed its window", [1] "the rank above's ghost
    adds into my window landed".  Ops: ("zero",), ("kernel",),
    ("signal", rank, slot, step) (store into that rank's flag slot) and
    ("wait", slot, step) (this rank's flag slot >= step)."""
    prog = [("zero",)]
    if rank + 1 < world:
        prog.append(("signal", rank + 1, 0, step))  # my window is zeroed
    if rank > 0:
        prog.append(("wait", 0, step))    # the window below is zeroed
    prog.append(("kernel",))              # ghost columns into rank-1's window
    if rank > 0:
        prog.append(("signal", rank - 1, 1, step))  # my adds landed there
    if rank + 1 < world:
        prog.append(("wait", 1, step))    # the adds into my window landed
    return prog


class ShardedMassOperator:
    """The column loop over one rank's cell block + the halo exchange.

    ``x_window`` / ``coords_window`` are the global fields restricted to
    ``shard.window`` / ``shard.coord_window``; the result is the rank's
    window of ``y`` with final values on its owned entity columns.
    """

    def __init__(self, fs, rank, world, quadrature=None, group=None,
                 fused=False):
        import torch
        from . import _lib
        from .kernels import MassOperator
        self.fs = fs
        self.rank, self.world = rank, world
        self.group = group
        shards = partition(fs, world)
        self.shard = shards[rank]
        # fused halo: ghost columns are added straight into the owner's
        # window by the kernel (peer memory) instead of being exchanged
        self.fused = bool(fused) and world > 1
        self.ghost_end = 0
        self._peer = None
        if self.fused:
            plan = fused_halo_plan(fs, shards)
            if plan is None:
                raise ValueError(
                    "the fused halo needs a vertex-only layout whose ghosts "
                    "are owned by the rank below (RCM-ordered blocks)")
            self.ghost_end = plan[rank]
        self.op = MassOperator(fs, quadrature, schedule="column")
        dev = self.op._dev
        # fused halo step flags (0: window zeroed, 1: the rank above's ghost
        # adds landed), raised by the neighbours, compared with the step
        self._flags = torch.zeros(4, dtype=torch.int32, device=dev)
        self._step = 0
        self.d_cells = torch.from_numpy(self.shard.cells).to(dev)
        # vertex-column layouts: sequential strips over the rank's block
        self.strips = (self.op._global_strips(cells=self.shard.cells)
                       if self.op.stripred_ok else None)
        self.halo = HaloExchange(fs, self.shard, device=dev)
        self._lib = _lib

    @property
    def window(self):
        return self.shard.window

    def connect(self, y_window):
        """Fused halo: map the rank below's ``y_window`` (collective; every
        rank passes the persistent window it will pass to ``apply``)."""
        if not self.fused:
            return
        if self.strips is None:
            raise ValueError("the fused halo runs on the strip schedule")
        if self._peer is not None:
            self._peer.close()
        self._peer = PeerWindow(y_window, self._flags, self.shard.window[0],
                                self.rank, self.world, group=self.group)
        self._peer_y = y_window

    def _apply_fused(self, x_window, coords_window, y_window, stream=None):
        """One step of the fused halo, ordered on the stream only (no host
        synchronisation): zero the window, tell the rank above, wait until
        the rank below zeroed its window, run the kernel (ghost columns
        REDG'd into the rank below's window), tell the rank below, wait
        for the rank above's ghost adds into this window."""
        if self._peer is None or y_window is not self._peer_y:
            raise ValueError("fused halo: call connect(y_window) first with "
                             "the window passed to apply")
        import torch
        lib = self._lib
        lo, hi = self.shard.window
        clo, _chi = self.shard.coord_window
        op = self.op
        s = self._step = (self._step % 0x7ffffffe) + 1
        flags = self._flags.data_ptr()
        peers = {self.rank - 1: self._peer.down_flags,
                 self.rank + 1: self._peer.up_flags}
        with torch.cuda.stream(stream or torch.cuda.current_stream()):
            for op_ in fused_step_program(self.rank, self.world, s):
                if op_[0] == "zero":
                    y_window.zero_()
                elif op_[0] == "signal":
                    lib.stream_signal(peers[op_[1]] + 4 * op_[2], op_[3],
                                      stream)
                elif op_[0] == "wait":
                    lib.stream_wait_geq(flags + 4 * op_[1], op_[2], stream)
                else:
                    strips, W = self.strips
                    lib.column_mass_strip_red_peer(
                        op.fs.layout, op.k, op.layers, coords_window,
                        op.mref, x_window, y_window, hi - lo, strips,
                        op.kron, W, self._peer.y_addr,
                        self.ghost_end if self._peer.y_addr else 0,
                        accumulate=True, x_base=lo, y_base=lo,
                        coords_base=clo,
                        n_vertices=op.fs.mesh.base.num_vertices,
                        stream=stream)
        return y_window

    def apply(self, x_window, coords_window, y_window=None, exchange=True,
              stream=None, accumulate=False):
        """The rank's column loop into ``y_window`` (zeroed first unless
        ``accumulate``), then the halo exchange (``exchange``; the fused
        halo's step zeroes and synchronises on its own)."""
        import torch
        lo, hi = self.shard.window
        clo, _chi = self.shard.coord_window
        if self.fused and exchange:
            return self._apply_fused(x_window, coords_window, y_window,
                                     stream)
        if y_window is None:
            y_window = torch.empty(hi - lo, dtype=torch.float64,
                                   device=x_window.device)
        if not accumulate:
            y_window.zero_()
        op = self.op
        if self.strips is not None:
            strips, W = self.strips
            self._lib.column_mass_strip_red(
                op.fs.layout, op.k, op.layers, coords_window, op.mref,
                x_window, y_window, hi - lo, strips, op.kron, W,
                accumulate=True, x_base=lo, y_base=lo, coords_base=clo,
                n_vertices=op.fs.mesh.base.num_vertices)
        else:
            self._lib.column_mass(
                op.fs.layout, op.k, op.n_cells, op.layers, op.cmap, op.offs,
                op.xmap, op.xoffs, coords_window, op.mref, x_window,
                y_window, hi - lo, accumulate=True,
                variant=self._lib.VARIANT_COLUMN, cells=self.d_cells,
                kron=op.kron, x_base=lo, y_base=lo, coords_base=clo)
        if exchange and self.world > 1:
            self.halo.exchange(y_window, group=self.group)
        return y_window

    def owned_slices(self):
        """(window-relative start, length) of every owned entity column."""
        out = []
        for d, o, c in ghost_origins(self.fs, self.shard.owned):
            out.append((d, o - self.shard.window[0], c))
        return out

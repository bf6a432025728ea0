"""User stencil kernels for ``iterate_columns``.

The SPEC's ``StencilKernel`` is an arbitrary procedure over per-argument
slot-value views; the paper's consumers (Firedrake / PyOP2,
PAPER.md:777-783) generate C for every local kernel and compile it at run
time.  ``CudaStencilKernel`` does the same on the device: the user writes
the local kernel as CUDA C++ ::

    __device__ void pm_kernel(double *out, const double *const *in,
                              long long cell, int layer)
    {
        // in[a][j]: argument a at slot j of this cell-layer
        // out[j]:   contribution to output slot j (starts at 0)
    }

and NVRTC compiles it for sm_100a inlined into a generated column loop
(``csrc/stencil.cu``): each cell-layer's DoFs are ``map[c][j] + l *
offset[j]`` (Alg. 2/3), the output receives ``+=``.  Schedules: ``auto`` /
``atomic`` (thread per cell-layer, fp64 atomics) and ``colored`` /
``sequential`` (one launch per colour of ``color_base_cells``, a thread
walks its cell's layers in order: bitwise deterministic).
"""
from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["CudaStencilKernel"]


class CudaStencilKernel:
    """``arity``: slot counts of the argument spaces in ``iterate_columns``
    order -- the inputs, then the output space last.  ``fields`` passed to
    ``iterate_columns`` follow the same order (inputs..., output)."""

    def __init__(self, source: str, arity):
        arity = tuple(int(k) for k in arity)
        if len(arity) < 1:
            raise ValueError("a stencil kernel needs at least an output space")
        self.arity = arity
        self.source = source
        self._handle = None
        self._maps = {}
        self._colors = {}

    def check(self) -> int:
        """Compile only (no device needed): the cubin size in bytes."""
        return _lib.stencil_check(self.source, self.arity[:-1],
                                  self.arity[-1])

    def _compiled(self):
        if self._handle is None:
            self._handle = _lib.stencil_compile(self.source, self.arity[:-1],
                                                self.arity[-1])
        return self._handle

    def _device_maps(self, fs, dev):
        import torch
        hit = self._maps.get(id(fs))
        if hit is None or hit[0] is not fs:
            m = torch.from_numpy(np.ascontiguousarray(fs.cell_map,
                                                      dtype=np.int32)).to(dev)
            o = torch.from_numpy(np.ascontiguousarray(fs.offsets,
                                                      dtype=np.int32)).to(dev)
            hit = (fs, m, o)
            self._maps[id(fs)] = hit
        return hit[1], hit[2]

    def _color_lists(self, mesh, dev):
        import torch
        from .iterate import color_base_cells
        base = mesh.base
        hit = self._colors.get(id(base))
        if hit is None or hit[0] is not base:
            order, ptr = color_base_cells(base).cells_by_color()
            hit = (base, torch.from_numpy(order).to(dev), ptr)
            self._colors[id(base)] = hit
        return hit[1], hit[2]

    def launch(self, fs_list, fields, schedule, stream=None):
        if len(fields) != len(self.arity):
            raise ValueError(f"stencil kernel takes {len(self.arity)} fields "
                             f"(inputs..., output), got {len(fields)}")
        for fs, f in zip(fs_list, fields):
            if f.shape[0] != fs.total_dofs:
                raise ValueError(f"field of {f.shape[0]} values on a space "
                                 f"of {fs.total_dofs} DoFs")
            if f.dtype.is_floating_point is False or f.element_size() != 8:
                raise ValueError("stencil fields are float64 device tensors")
        if schedule in ("auto", "atomic"):
            colored = False
        elif schedule in ("colored", "sequential"):
            colored = True
        else:
            raise ValueError(f"user stencil kernels run the atomic or the "
                             f"colored schedule, not {schedule!r}")
        out = fields[-1]
        dev = out.device
        if dev.type != "cuda":
            raise ValueError("stencil fields must be CUDA tensors")
        maps = [self._device_maps(fs, dev) for fs in fs_list]
        mesh = fs_list[-1].mesh
        h = self._compiled()
        ins = [f.contiguous() for f in fields[:-1]]
        args = (ins, [m for m, _ in maps[:-1]], [o for _, o in maps[:-1]],
                out, maps[-1][0], maps[-1][1])
        if not colored:
            _lib.stencil_launch(h, False, mesh.base.num_cells, mesh.layers,
                                *args, stream=stream)
            return
        order, ptr = self._color_lists(mesh, dev)
        for c in range(len(ptr) - 1):
            cells = order[ptr[c]:ptr[c + 1]]
            _lib.stencil_launch(h, True, cells.shape[0], mesh.layers, *args,
                                cells=cells, stream=stream)

    def __del__(self):
        try:
            _lib.stencil_free(self._handle)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

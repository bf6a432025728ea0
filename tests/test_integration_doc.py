"""INTEGRATION.md's reference-side bindings, executed verbatim: the ctypes
``build_cell_map`` a prismesh maintainer would add must reproduce the maps,
and the ``derive_edges`` binding the edges (so the document stays true)."""
import ctypes
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _blocks():
    text = open("INTEGRATION.md").read()
    return re.findall(r"```python\n(.*?)```", text, re.S)


def test_build_cell_map_snippet():
    import torch
    from paper_1604_05937_b200 import (ExtrudedMesh, builtin_layout,
                                       generate_unit_square_mesh,
                                       number_dofs)
    code = next(b for b in _blocks() if "def build_cell_map" in b)
    ns = {}
    exec(code, ns)                                  # noqa: S102
    for h, v in (("CG1", "CG1"), ("DG1", "DG1"), ("CG1", "DG0")):
        fs = number_dofs(ExtrudedMesh(generate_unit_square_mesh(7), 4),
                         builtin_layout(h, v))
        cmap, offs = ns["build_cell_map"](fs)
        assert np.array_equal(cmap, fs.cell_map)
        assert np.array_equal(offs, fs.offsets)


def test_derive_edges_snippet():
    from paper_1604_05937_b200.mesh import derive_edges as host
    from paper_1604_05937_b200.mesh import generate_unit_square_mesh
    code = next(b for b in _blocks() if "def derive_edges" in b)
    ns = {"ctypes": ctypes, "np": np,
          "lib": ctypes.CDLL(
              "paper_1604_05937_b200/_native/libprismesh_cuda.so"),
          "_host_derive_edges": lambda c, n: host(c, n, device=False)}
    import torch
    ns["torch"] = torch
    exec(code, ns)                                  # noqa: S102
    m = generate_unit_square_mesh(30)
    cells = np.asarray(m.cell_vertices)
    ev, ce = ns["derive_edges"](cells, m.num_vertices)
    ev_h, ce_h = host(cells, m.num_vertices, device=False)
    assert np.array_equal(ev, ev_h) and np.array_equal(ce, ce_h)


def test_cuthill_mckee_snippet():
    from paper_1604_05937_b200.mesh import generate_unit_square_mesh
    from paper_1604_05937_b200.ordering import (apply_ordering, random_order,
                                                rcm_order)
    import torch
    code = next(b for b in _blocks() if "def cuthill_mckee" in b)
    ns = {"ctypes": ctypes, "np": np, "torch": torch,
          "lib": ctypes.CDLL(
              "paper_1604_05937_b200/_native/libprismesh_cuda.so")}
    ns["lib"].pm_last_error.restype = ctypes.c_char_p
    exec(code, ns)                                  # noqa: S102
    m = apply_ordering(generate_unit_square_mesh(25), random_order(676, 4))
    off, nbr = m.vertex_neighbours()
    deg = np.diff(off)
    rows = np.repeat(np.arange(off.shape[0] - 1), deg)
    nb = nbr[np.lexsort((nbr, deg[nbr], rows))]
    order = ns["cuthill_mckee"](off, nb)
    fwd = np.empty_like(order)
    fwd[order[::-1]] = np.arange(order.shape[0])
    assert np.array_equal(fwd, rcm_order(off, nbr).forward)


def test_stencil_snippet():
    import torch
    from paper_1604_05937_b200 import (ExtrudedMesh, builtin_layout,
                                       generate_unit_square_mesh,
                                       number_dofs)
    from paper_1604_05937_b200.verification import materialized_cell_maps
    code = next(b for b in _blocks() if "CudaStencilKernel(" in b)
    fs = number_dofs(ExtrudedMesh(generate_unit_square_mesh(6), 3),
                     builtin_layout("CG1", "CG1"))
    x_np = np.random.default_rng(2).random(fs.total_dofs)
    ns = {"torch": torch, "fs": fs, "x": torch.from_numpy(x_np).cuda()}
    exec(code, ns)                                  # noqa: S102
    lists = materialized_cell_maps(fs)
    ref = np.zeros(fs.total_dofs)
    np.add.at(ref, lists.reshape(-1, 6), x_np[lists.reshape(-1, 6)] ** 2)
    assert np.abs(ns["out"].cpu().numpy() - ref).max() <= 1e-12 * ref.max()

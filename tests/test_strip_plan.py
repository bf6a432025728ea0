"""Host planner of the strip-patch schedule + a numpy emulation of its
kernel's accounting (window, residencies, Y slots, owner gather)."""
import numpy as np
import pytest

import oracle
from conftest import LAYOUT_COUNTS, families, quad_degrees


def _plan(n, layers, lname, ordering="rcm", jitter=0.0, budget=200 * 1024,
          max_strip=None):
    from paper_1604_05937_b200 import DofLayout, ExtrudedMesh, number_dofs
    from paper_1604_05937_b200.configs import base_mesh
    from paper_1604_05937_b200.iterate import color_base_cells
    from paper_1604_05937_b200.schedule import build_strip_plan
    base, _ = base_mesh(n, ordering, jitter)
    fs = number_dofs(ExtrudedMesh(base, layers),
                     DofLayout(lname, LAYOUT_COUNTS[lname]))
    col = color_base_cells(base)
    plan = build_strip_plan(base, fs.layout, layers, col.color_of,
                            col.num_colors, smem_budget=budget,
                            max_strip=max_strip)
    return fs, plan


@pytest.mark.parametrize("n,budget", ((6, 8 * 1024), (12, 40 * 1024),
                                      (20, 200 * 1024)))
def test_strip_plan_invariants(n, budget):
    fs, plan = _plan(n, 4, "CG1xCG1", budget=budget, max_strip=7)
    pp = plan.patch
    cv = fs.mesh.base.cell_vertices
    for p in range(pp.n_patches):
        ents = pp.ents[pp.ent_ptr[p]:pp.ent_ptr[p + 1]]
        visited = set(pp.cells[pp.cell_ptr[p]:pp.cell_ptr[p + 1]].tolist())
        seen = []
        ys = []
        for s in range(plan.strip_ptr[p], plan.strip_ptr[p + 1]):
            win = [None, None, None]
            k0 = plan.step_ptr[s]
            assert plan.step_ptr[s + 1] - k0 >= 3
            for k in range(plan.step_ptr[s], plan.step_ptr[s + 1]):
                # sequential strips: the replaced slot cycles 0, 1, 2, ...
                assert plan.step_slot[k] == (k - k0) % 3
                win[plan.step_slot[k]] = int(ents[plan.step_v[k]])
                if plan.step_y[k] >= 0:
                    ys.append(int(plan.step_y[k]))
                    assert plan.step_v[k] < pp.owned[p]
                if plan.step_flags[k] & 1:
                    cell = np.flatnonzero(
                        (np.sort(cv, axis=1) == sorted(win)).all(axis=1))
                    assert cell.size == 1
                    seen.append(int(cell[0]))
        assert sorted(seen) == sorted(visited), "each visited cell once"
        assert sorted(ys) == list(range(plan.y_count[p])), "y slots unique"


@pytest.mark.parametrize("lname", ("CG1xCG1", "VP1", "CG1xDG1", "CG1xDG0"))
@pytest.mark.parametrize("ordering", ("rcm", "random"))
def test_strip_emulation_matches_oracle(lname, ordering):
    """Run the kernel's algorithm in numpy (all layers at once)."""
    from paper_1604_05937_b200.quadrature import (element_for_layout,
                                                  kronecker_factors,
                                                  prism_quadrature)
    layers = 3
    fs, plan = _plan(10, layers, lname, ordering, jitter=0.2,
                     budget=30 * 1024, max_strip=9)
    pp = plan.patch
    base = fs.mesh.base
    el = element_for_layout(fs.layout)
    q = prism_quadrature(*quad_degrees(lname))
    Mt, Ml = kronecker_factors(el, q)
    h, v, c = (np.array(a) for a in (el.slot_h, el.slot_v, el.slot_comp))
    M = Mt[h][:, h] * Ml[v][:, v] * (c[:, None] == c[None, :])
    slots = fs.slots
    x = np.random.default_rng(3).random(fs.total_dofs)
    from paper_1604_05937_b200 import COORDS_LAYOUT
    coords = oracle.extrude(base.coords, layers, 1.0 / layers)
    col0 = fs.column_sizes[0]
    lv = fs.layout.dofs(0, 0)
    y = np.zeros(fs.total_dofs)
    for p in range(pp.n_patches):
        ents = pp.ents[pp.ent_ptr[p]:pp.ent_ptr[p + 1]]
        Y = {}
        for s in range(plan.strip_ptr[p], plan.strip_ptr[p + 1]):
            win = [None] * 3
            ysl = [-1] * 3
            acc = [None] * 3

            def flush(a):
                if win[a] is not None and ysl[a] >= 0:
                    Y[ysl[a]] = acc[a]
            for k in range(plan.step_ptr[s], plan.step_ptr[s + 1]):
                a = plan.step_slot[k]
                flush(a)
                win[a] = int(ents[plan.step_v[k]])
                ysl[a] = int(plan.step_y[k])
                acc[a] = np.zeros(col0)
                if plan.step_flags[k] & 1:
                    for l in range(layers):
                        P = np.array([[coords[3 * (win[b] * (layers + 1) + l + t) + qq]
                                       for t in (0, 1) for qq in range(3)]
                                      for b in range(3)])
                        xm = (P[:, 0] + P[:, 3]) / 2
                        ym = (P[:, 1] + P[:, 4]) / 2
                        a2 = (xm[1] - xm[0]) * (ym[2] - ym[0]) - \
                            (xm[2] - xm[0]) * (ym[1] - ym[0])
                        hh = ((P[0, 5] - P[0, 2]) + (P[1, 5] - P[1, 2]) +
                              (P[2, 5] - P[2, 2])) / 3
                        det = abs(a2 * hh)
                        idx = [win[sl.local] * col0 + sl.within(fs.layout) +
                               l * (fs.layout.dofs(0, 0) + fs.layout.dofs(0, 1))
                               for sl in slots]
                        loc = det * (M @ x[idx])
                        for j, sl in enumerate(slots):
                            acc[sl.local][idx[j] - win[sl.local] * col0] += loc[j]
            for a in range(3):
                flush(a)
        for i in range(pp.owned[p]):
            g = int(ents[i])
            row = plan.own_base[p] + i
            for yy in plan.own_y[plan.own_y_ptr[row]:plan.own_y_ptr[row + 1]]:
                y[g * col0:(g + 1) * col0] += Y[int(yy)]
    tri, line, nc = families(lname)
    ref = oracle.Problem(base, layers, LAYOUT_COUNTS[lname], tri, line, nc,
                         *quad_degrees(lname)).assemble(x)
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-14 * np.abs(ref).max())


@pytest.mark.parametrize("n,ordering,max_len", ((6, "rcm", 64), (12, "random", 7),
                                                (20, "rcm", 5)))
def test_global_strips_invariants(n, ordering, max_len):
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.configs import base_mesh
    base, _ = base_mesh(n, ordering, 0.2)
    sp, st = _lib.build_global_strips(base, max_len)
    cv = np.sort(base.cell_vertices, axis=1)
    key = {tuple(r): i for i, r in enumerate(cv.tolist())}
    seen = []
    for s in range(len(sp) - 1):
        steps = st[sp[s]:sp[s + 1]].tolist()
        assert 3 <= len(steps) <= max_len + 2
        win = steps[:3]
        seen.append(key[tuple(sorted(win))])
        for k, v in enumerate(steps[3:]):
            win[k % 3] = v            # the oldest slot is replaced
            seen.append(key[tuple(sorted(win))])
    assert sorted(seen) == list(range(base.num_cells))


@pytest.mark.parametrize("n,ordering,max_len", ((6, "rcm", 64), (12, "random", 7)))
def test_global_strip_edges(n, ordering, max_len):
    """Edge slot a always holds the edge opposite window vertex a."""
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.configs import base_mesh
    base, _ = base_mesh(n, ordering, 0.2)
    sp, st, se = _lib.build_global_strips(base, max_len, edges=True)
    ev = base.edge_vertices
    for s in range(len(sp) - 1):
        win, ewin = [None] * 3, [None] * 3
        for k in range(sp[s], sp[s + 1]):
            i = k - sp[s]
            a = i % 3
            win[a] = int(st[k])
            if i < 3:
                ewin[a] = int(se[k, 0])
            else:
                ewin[(a + 1) % 3] = int(se[k, 0])
                ewin[(a + 2) % 3] = int(se[k, 1])
            if i >= 2:
                for b in range(3):
                    others = {win[(b + 1) % 3], win[(b + 2) % 3]}
                    assert set(ev[ewin[b]].tolist()) == others


@pytest.mark.parametrize("n,ordering", ((7, "rcm"), (12, "random"),
                                        (16, "rcm")))
@pytest.mark.parametrize("patch", (1, 5, 40, 10000))
def test_patch_strips_plan(n, ordering, patch):
    """pm_build_patch_strips, emulated the way k_strip_red(_e) STREAM walks
    it: one continuous step stream per patch, step K flushes and refills
    vertex slot K % 3 and edge slots K+1, K+2 (-1 = none).  Every cell is
    visited once with a consistent window (edge slot a opposite vertex slot
    a), and the store-first flags make each entity's first flushed write in
    a patch a store that no other patch races with."""
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.configs import base_mesh
    from paper_1604_05937_b200.schedule import morton_order
    base, _ = base_mesh(n, ordering, 0.2)
    cv = np.asarray(base.cell_vertices)
    ce = np.asarray(base.cell_edges)
    nc, n0 = cv.shape[0], base.num_vertices
    order = morton_order(np.asarray(base.coords)[cv].mean(axis=1))
    ptr = np.unique(np.append(np.arange(0, nc, patch), nc))
    patch_of = np.empty(nc, dtype=np.int64)
    for p in range(len(ptr) - 1):
        patch_of[order[ptr[p]:ptr[p + 1]]] = p
    ip, sp, st, se, zl = _lib.build_patch_strips(base, order, ptr, edges=True)
    S, NOCELL = _lib.STEP_STORE, _lib.STEP_NOCELL
    mask = NOCELL - 1
    zero = set(zl.tolist())
    owners = {}
    edge_of = {}
    for c in range(nc):
        for q in range(3):
            owners.setdefault(int(cv[c, q]), set()).add(patch_of[c])
            owners.setdefault(n0 + int(ce[c, q]), set()).add(patch_of[c])
            a, b = sorted((int(cv[c, (q + 1) % 3]), int(cv[c, (q + 2) % 3])))
            edge_of[(a, b)] = int(ce[c, q])
    shared = {e for e, o in owners.items() if len(o) > 1}
    assert zero == shared
    stored = set()
    cells_seen = []
    sorted_cells = {tuple(sorted(r)): i for i, r in enumerate(cv.tolist())}
    for p in range(len(ptr) - 1):
        touched = set()

        def flush(res):
            if res is None:
                return
            code, flag = res
            if flag:
                assert code not in zero and code not in stored
                stored.add(code)
            else:
                assert code in zero or code in touched
            touched.add(code)

        vs, es = [None] * 3, [None] * 3
        k0, k1 = sp[ip[p]], sp[ip[p + 1]]
        for K in range(k1 - k0):
            A = K % 3
            raw = int(st[k0 + K])
            flush(vs[A])
            vs[A] = (raw & mask, raw & S)
            for q, B in enumerate(((A + 1) % 3, (A + 2) % 3)):
                flush(es[B])
                e = int(se[k0 + K, q])
                es[B] = None if e < 0 else (n0 + (e & mask), e & S)
            if raw & NOCELL:
                continue
            win = [v[0] for v in vs]
            c = sorted_cells[tuple(sorted(win))]
            assert patch_of[c] == p
            cells_seen.append(c)
            for a in range(3):
                u, w = sorted((win[(a + 1) % 3], win[(a + 2) % 3]))
                assert es[a] is not None and es[a][0] == n0 + edge_of[(u, w)]
        for r in vs + es:
            flush(r)
    assert sorted(cells_seen) == list(range(nc))
    # every entity of some cell is zeroed or stored exactly once
    assert stored | zero == set(owners)


def test_integration_patch_strips_snippet():
    """INTEGRATION.md's ctypes binding of pm_build_patch_strips, executed
    verbatim (host planner: no GPU), equals the package's wrapper."""
    import ctypes
    import re
    from paper_1604_05937_b200 import _lib
    from paper_1604_05937_b200.configs import base_mesh
    from paper_1604_05937_b200.schedule import morton_order
    text = open("INTEGRATION.md").read()
    code = next(b for b in re.findall(r"```python\n(.*?)```", text, re.S)
                if "def patch_strips" in b)
    lib = _lib.host_lib()
    ns = {"ctypes": ctypes, "np": np, "lib": lib,
          "i32p": ctypes.POINTER(ctypes.c_int32)}
    exec(code, ns)                                  # noqa: S102
    base, _ = base_mesh(9, "rcm", 0.1)
    cv = np.asarray(base.cell_vertices)
    order = morton_order(np.asarray(base.coords)[cv].mean(axis=1))
    ptr = np.unique(np.append(np.arange(0, cv.shape[0], 16), cv.shape[0]))
    got = ns["patch_strips"](base, order, ptr, edges=True)
    want = _lib.build_patch_strips(base, order, ptr, edges=True)
    assert all(np.array_equal(a, b) for a, b in zip(got, want))


@pytest.mark.parametrize("n,ordering", [(1, "rcm"), (6, "rcm"), (13, "random")])
def test_strip_step_cells(n, ordering):
    """pm_strip_step_cells: every cell formed by exactly one step, fill
    steps form none, and a step's cell is its window (last three entered
    vertices) -- the per-cell field addressing of the DG strip kernel."""
    from paper_1604_05937_b200 import _lib, configs
    w = configs.Workload("sc", n, 2, "DG1xDG1", (2, 2), ordering=ordering)
    fs, _q, _x, _ = configs.build(w)
    base = fs.mesh.base
    sp, st = _lib.build_global_strips(base, max_len=7)
    sc = _lib.strip_step_cells(base, sp, st)
    assert sc.shape == st.shape
    cells = sc[sc >= 0]
    assert np.array_equal(np.sort(cells), np.arange(base.num_cells))
    cv = np.asarray(base.cell_vertices)
    for s in range(sp.shape[0] - 1):
        a, b = sp[s], sp[s + 1]
        assert sc[a] == -1 and sc[a + 1] == -1
        for i in range(a + 2, b):
            assert set(cv[sc[i]]) == {st[i - 2], st[i - 1], st[i]}

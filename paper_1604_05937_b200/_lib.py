"""ctypes binding of libprismesh_cuda.so (the C ABI in include/prismesh_cuda.h).

No fallback: if the library is missing or no CUDA device is present, the
device entry points raise.  torch owns device memory and streams; the ABI
receives ``data_ptr()`` values and ``torch.cuda.current_stream()``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PM_NATIVE_LIB: an experimental build of the same library (tools/)
LIB_PATH = os.environ.get("PM_NATIVE_LIB") or \
    os.path.join(_HERE, "_native", "libprismesh_cuda.so")

PM_OK, PM_EINVAL, PM_ECUDA, PM_EOVERFLOW = 0, 1, 2, 3
SHARE_NONE, SHARE_VERTICAL, SHARE_HORIZONTAL = 0, 1, 2
(VARIANT_AUTO, VARIANT_ATOMIC, VARIANT_PATCH, VARIANT_COLUMN, VARIANT_COLORED,
 VARIANT_STREAM, VARIANT_STRIP, VARIANT_STRIPRED) = range(8)

_lib = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double

#: name -> (restype, argtypes); mirrors include/prismesh_cuda.h
SIGNATURES = {
    "pm_last_error": (ctypes.c_char_p, []),
    "pm_version": (ctypes.c_int, []),
    "pm_build_cell_map": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _i32p,
                                         _i32, _i32, _vp, _vp, _i64p, _vp]),
    "pm_num_slots": (ctypes.c_int, [_i32p, _i32p]),
    "pm_extrude_coordinates": (ctypes.c_int, [_vp, _i64, _i32, _f64, _vp,
                                              _vp]),
    "pm_column_mass": (ctypes.c_int, [_i32p, _i32, _i64, _i32, _vp, _vp,
                                      _vp, _vp, _vp, ctypes.POINTER(_f64),
                                      ctypes.POINTER(_f64),
                                      ctypes.POINTER(_f64),
                                      _vp, _vp, _i64, _i32, _i32, _vp, _i64,
                                      _vp]),
    "pm_greedy_color_cells": (ctypes.c_int, [_i32p, _i64, _i64p, _i32p,
                                             _i32p, _i32p]),
    "pm_column_mass_patch": (ctypes.c_int, [_i32p, _i32, _i64, _i64, _i32,
                                            _vp, _vp, _vp,
                                            ctypes.POINTER(_f64),
                                            ctypes.POINTER(_f64),
                                            ctypes.POINTER(_f64), _vp, _vp,
                                            _i64, _i32, _i32, _i32, _i32,
                                            _vp, _vp, _vp, _vp, _vp, _vp,
                                            _vp, _vp]),
    "pm_column_mass_strip": (ctypes.c_int, [_i32p, _i32, _i32, _vp,
                                            ctypes.POINTER(_f64),
                                            ctypes.POINTER(_f64),
                                            ctypes.POINTER(_f64), _vp, _vp,
                                            _i64, _i32, _i32, _i32, _i32,
                                            _i32, _i32, _i32, _i32] +
                            [_vp] * 14),
    "pm_build_strips": (ctypes.c_int, [_i64] + [_vp] * 6 + [_i32] +
                        [_vp] * 10),
    "pm_column_mass_strip_red": (ctypes.c_int, [_i32p, _i32, _i32, _vp,
                                                ctypes.POINTER(_f64),
                                                ctypes.POINTER(_f64),
                                                ctypes.POINTER(_f64), _vp,
                                                _vp, _i64, _i32, _i64, _i32,
                                                _vp, _vp, _vp, _i64, _vp]),
    "pm_column_mass_dg_range": (ctypes.c_int, [_i32p, _i32, _i64, _i64, _i32,
                                               _vp, _vp, _vp, _vp, _vp,
                                               ctypes.POINTER(_f64), _vp,
                                               _vp, _vp]),
    "pm_build_global_strips": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp,
                                              _vp, _i32, _vp, _vp, _vp,
                                              _vp]),
    "pm_column_mass_strip_tma": (ctypes.c_int, [_i32p, _i32, _i32, _vp,
                                                ctypes.POINTER(_f64),
                                                ctypes.POINTER(_f64), _vp,
                                                _vp, _i64, _i32, _i64, _vp,
                                                _vp, _i64, _vp]),
    "pm_build_run_strips": (ctypes.c_int, [_i64, _i64, _vp, _vp, _vp,
                                           _vp, _i32, _vp, _vp, _vp,
                                           _vp]),
    "pm_build_patch_strips": (ctypes.c_int, [_i64, _i64, _i64, _vp, _vp, _vp,
                                             _vp, _i64, _i32, _vp, _vp, _vp,
                                             _vp, _vp, _vp]),
    "pm_column_mass_patch_strips": (ctypes.c_int, [
        _i32p, _i32, _i32, _vp, ctypes.POINTER(_f64), ctypes.POINTER(_f64),
        ctypes.POINTER(_f64), _vp, _vp, _i64, _i32, _i64, _i32, _vp, _vp,
        _vp, _vp, _i64, _i64, _vp, _vp]),
    "pm_column_probe": (ctypes.c_int, [_i32, _i32, _i64, _i32, _vp, _vp, _vp,
                                       _vp, _vp]),
    "pm_halo_pack": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "pm_halo_unpack_add": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp]),
    "pm_rcm_order": (ctypes.c_int, [_i64p, _i64p, _i64, _i64p]),
    "pm_device_info": (ctypes.c_int, [_i32p, _i64p]),
    "pm_derive_edges": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _i64p,
                                       _i32p, _vp]),
    "pm_vertex_graph_sorted": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp,
                                              _vp]),
    "pm_rcm_order_device": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "pm_stencil_check": (ctypes.c_int, [ctypes.c_char_p, _i32, _i32p, _i32,
                                        _i64p]),
    "pm_stencil_compile": (ctypes.c_int, [ctypes.c_char_p, _i32, _i32p, _i32,
                                          ctypes.POINTER(ctypes.c_void_p)]),
    "pm_stencil_launch": (ctypes.c_int, [_vp, _i32, _i64, _i32, _vp, _vp,
                                         _vp, _vp, _vp, _vp, _vp, _vp]),
    "pm_stencil_free": (ctypes.c_int, [_vp]),
    "pm_build_flags": (ctypes.c_int, []),
    "pm_strip_step_cells": (ctypes.c_int, [_i64, _i64, _vp, _vp, _i64, _vp,
                                           _vp]),
    "pm_column_mass_strip_dg": (ctypes.c_int, [_i32p, _i32, _i64, _i32, _vp,
                                               ctypes.POINTER(_f64), _vp,
                                               _vp, _i64, _i32, _vp, _vp,
                                               _vp, _vp]),
    "pm_reorder_cells": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _vp,
                                        _vp]),
    "pm_column_mass_strip_red_peer": (ctypes.c_int, [
        _i32p, _i32, _i32, _vp, ctypes.POINTER(_f64), ctypes.POINTER(_f64),
        ctypes.POINTER(_f64), _vp, _vp, _i64, _i32, _i64, _i32, _vp, _vp,
        _i64, _vp, _i64, _vp]),
    "pm_ipc_export": (ctypes.c_int, [_vp, _vp, _i64p]),
    "pm_ipc_open": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(_vp)]),
    "pm_ipc_close": (ctypes.c_int, [_vp, _i64]),
    "pm_stream_signal": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp]),
    "pm_stream_wait_geq": (ctypes.c_int, [_vp, ctypes.c_uint32, _vp]),
    "pm_set_launch_overlap": (ctypes.c_int, [_i32]),
    "pm_stream_triad": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_double, _i64,
                                       _vp]),
    "pm_tiles_build": (ctypes.c_int, [_i64, _i64, _i64, _vp, _vp, _i64, _i64,
                                      _i64, _i32, _i32, _i32,
                                      ctypes.POINTER(_vp)]),
    "pm_tiles_info": (ctypes.c_int, [_vp, _i64p]),
    "pm_tiles_export": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), _vp]),
    "pm_tiles_free": (None, [_vp]),
    "pm_tiles_blob": (ctypes.c_int, [_vp, _vp, _vp, _i64p]),
    "pm_tile_smem_layout": (ctypes.c_int, [_i32p, _i32, _i32, _i32, _i32p,
                                           _i32p]),
    "pm_column_mass_tile": (ctypes.c_int, [
        _i32p, _i32, _vp, _i64, ctypes.POINTER(_f64), ctypes.POINTER(_f64),
        _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32,
        _i32, _i32, _i32, _vp]),
}


class NativeLibraryMissing(RuntimeError):
    pass


def host_lib():
    """Load the native library (also usable without a GPU for host setup)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run "
                "`python -m paper_1604_05937_b200.build_native` "
                "(or __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = host_lib().pm_last_error()
    return msg.decode() if msg else ""


def check(rc: int):
    if rc == PM_OK:
        return
    msg = last_error()
    if rc in (PM_EINVAL, PM_EOVERFLOW):
        raise ValueError(msg)
    raise RuntimeError(msg)


def cuda_device():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError(
            "prismesh-b200 needs a CUDA device (sm_100a); there is no CPU "
            "fallback")
    host_lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def host_tensor(a, dtype):
    """CPU tensor of a contiguous ``dtype`` view of ``a`` (copied only when
    ``a`` is read-only, e.g. the frozen mesh arrays, or needs converting)."""
    import numpy as np
    import torch
    arr = np.ascontiguousarray(a, dtype=dtype)
    if not arr.flags.writeable:
        arr = arr.copy()
    return torch.from_numpy(arr)


def ptr(t, base=0):
    """Device address of tensor ``t``; ``base`` (elements) shifts it so that
    global indices land inside a window tensor that starts at ``base``."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr() - base * t.element_size())


# ---------------------------------------------------------------------------
# thin typed wrappers
# ---------------------------------------------------------------------------

def num_slots(layout) -> int:
    d = layout.delta6()
    k = ctypes.c_int32(0)
    check(host_lib().pm_num_slots(d.ctypes.data_as(_i32p), ctypes.byref(k)))
    return k.value


def mesh_device_arrays(base, device):
    """Cached device copies of the base connectivity (int32)."""
    import torch
    cache = getattr(base, "__dict__", {}).get("_pm_device")
    if cache is not None and cache["device"] == device:
        return cache
    cv = host_tensor(base.cell_vertices, np.int32).to(device)
    ce = host_tensor(base.cell_edges, np.int32).to(device)
    cache = {"device": device, "cv": cv, "ce": ce}
    try:
        base.__dict__["_pm_device"] = cache
    except (AttributeError, TypeError):
        pass
    return cache


def build_cell_map_device(fs, stream=None):
    """K0 on the device: (cell_map (N2,k) int32, offsets (k,) int32)."""
    import torch
    dev = cuda_device()
    base = fs.mesh.base
    k = num_slots(fs.layout)
    arrs = mesh_device_arrays(base, dev)
    n_cells = base.num_cells
    cmap = torch.empty((n_cells, k), dtype=torch.int32, device=dev)
    offs = torch.empty((k,), dtype=torch.int32, device=dev)
    total = ctypes.c_int64(0)
    d = fs.layout.delta6()
    rc = host_lib().pm_build_cell_map(
        ptr(arrs["cv"]), ptr(arrs["ce"]), n_cells, base.num_vertices,
        base.num_edges, d.ctypes.data_as(_i32p), fs.mesh.layers, k,
        ptr(cmap), ptr(offs), ctypes.byref(total), stream_ptr(stream))
    check(rc)
    if total.value != fs.total_dofs:
        raise RuntimeError(
            f"device total {total.value} != closed form {fs.total_dofs}")
    return cmap, offs


def extrude_coordinates_device(d_base, layers, h, stream=None):
    import torch
    n = d_base.shape[0]
    out = torch.empty(3 * n * (layers + 1), dtype=torch.float64,
                      device=d_base.device)
    check(host_lib().pm_extrude_coordinates(ptr(d_base), n, layers, float(h),
                                            ptr(out), stream_ptr(stream)))
    return out


def column_probe(mode, fs, out, stream=None):
    cmap = fs.device_cell_map()
    offs = fs.device_offsets()
    k = cmap.shape[1]
    i64 = ptr(out) if mode == 0 else None
    f64 = ptr(out) if mode == 1 else None
    check(host_lib().pm_column_probe(mode, k, fs.mesh.base.num_cells,
                                     fs.mesh.layers, ptr(cmap), ptr(offs),
                                     i64, f64, stream_ptr(stream)))


def _f64ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(_f64))


def column_mass(layout, k, n_cells, layers, cmap, offs, xmap, xoffs, coords,
                mref, x, y, n_dofs, accumulate=False, variant=VARIANT_AUTO,
                cells=None, stream=None, kron=None, x_base=0, y_base=0,
                coords_base=0):
    """pm_column_mass: y (+)= M x over the column loop (device tensors).
    ``kron`` = (Mtri, Mline) factors of ``mref`` (host arrays)."""
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    if m.shape[0] != k * k:
        raise ValueError(f"mref must be {k}x{k}")
    mt, ml = (None, None) if kron is None else (
        np.ascontiguousarray(kron[0], dtype=np.float64).ravel(),
        np.ascontiguousarray(kron[1], dtype=np.float64).ravel())
    d = layout.delta6()
    rc = host_lib().pm_column_mass(
        d.ctypes.data_as(_i32p), k, n_cells, layers, ptr(cmap), ptr(offs),
        ptr(xmap), ptr(xoffs), ptr(coords, coords_base), _f64ptr(m),
        _f64ptr(mt), _f64ptr(ml), ptr(x, x_base), ptr(y, y_base), n_dofs,
        1 if accumulate else 0, variant, ptr(cells),
        0 if cells is None else cells.shape[0], stream_ptr(stream))
    check(rc)


def column_mass_patch(layout, k, base, layers, cmap, xmap, coords, mref, x,
                      y, plan, dplan, chunk, stream=None, kron=None):
    """pm_column_mass_patch: y = M x with the patch-owner schedule."""
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    mt = np.ascontiguousarray(kron[0], dtype=np.float64).ravel()
    ml = np.ascontiguousarray(kron[1], dtype=np.float64).ravel()
    d = layout.delta6()
    rc = host_lib().pm_column_mass_patch(
        d.ctypes.data_as(_i32p), k, base.num_vertices, base.num_edges,
        layers, ptr(cmap), ptr(xmap), ptr(coords), _f64ptr(m), _f64ptr(mt),
        _f64ptr(ml), ptr(x), ptr(y),
        plan.n_patches, plan.n_colors, chunk, plan.max_local,
        plan.max_owned, ptr(dplan["cell_ptr"]), ptr(dplan["cells"]),
        ptr(dplan["color_ptr"]), ptr(dplan["ent_ptr"]), ptr(dplan["owned"]),
        ptr(dplan["ents"]), ptr(dplan["lents"]), stream_ptr(stream))
    check(rc)


def column_mass_strip(layout, k, layers, coords, mref, x, y, plan, dplan,
                      kron, stream=None):
    """pm_column_mass_strip: y = M x with the strip-patch schedule."""
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    mt = np.ascontiguousarray(kron[0], dtype=np.float64).ravel()
    ml = np.ascontiguousarray(kron[1], dtype=np.float64).ravel()
    d = layout.delta6()
    pp = plan.patch
    rc = host_lib().pm_column_mass_strip(
        d.ctypes.data_as(_i32p), k, layers, ptr(coords), _f64ptr(m),
        _f64ptr(mt), _f64ptr(ml), ptr(x), ptr(y), pp.n_patches, plan.W,
        plan.threads, pp.max_local, plan.max_y, pp.max_owned,
        plan.max_steps, plan.max_strips, plan.max_oy, ptr(dplan["ent_ptr"]), ptr(dplan["owned"]), ptr(dplan["ents"]),
        ptr(dplan["strip_ptr"]), ptr(dplan["step_ptr"]),
        ptr(dplan["step_v"]), ptr(dplan["step_slot"]),
        ptr(dplan["step_flags"]), ptr(dplan["step_y"]),
        ptr(dplan["y_count"]), ptr(dplan["own_base"]),
        ptr(dplan["own_y_ptr"]), ptr(dplan["own_y"]), stream_ptr(stream))
    check(rc)


def build_global_strips(base, max_len=32, cells=None, edges=False,
                        order=None, scan=None, runs=False):
    """(strip_ptr int32, steps int32[, steps_e int32 (n_steps, 2)]):
    sequential strips over the mesh or over the subset ``cells`` (host
    C++); with ``edges`` also the two window edges each step brings in.
    ``order``: "morton" (default, PM_STRIP_ORDER), "rcm" (mean vertex id)
    or "creation" (as built).  ``scan``: the order in which strips start
    at unused cells -- "index" (cell index order: the bands of an
    RCM-ordered mesh), "morton" (centroid Morton order, for meshes whose
    cell order is not spatially coherent), or None (PM_STRIP_SCAN, default
    "auto": Morton when index-order strips come out short)."""
    cv = np.ascontiguousarray(base.cell_vertices, dtype=np.int32)
    ce = np.ascontiguousarray(base.cell_edges, dtype=np.int32)
    n = cv.shape[0]
    mask = None
    if cells is not None:
        mask = np.zeros(n, dtype=np.uint8)
        mask[np.asarray(cells)] = 1
    sp = np.zeros(n + 1, dtype=np.int32)
    st = np.zeros(3 * n + 3, dtype=np.int32)
    se = np.zeros((3 * n + 3, 2), dtype=np.int32) if edges else None
    tot = np.zeros(2, dtype=np.int64)

    def run(scan_order):
        build = host_lib().pm_build_run_strips if runs else \
            host_lib().pm_build_global_strips
        check(build(
            n, base.num_edges, cv.ctypes.data_as(_i32p),
            ce.ctypes.data_as(_i32p),
            None if mask is None else mask.ctypes.data_as(ctypes.c_void_p),
            None if scan_order is None else
            scan_order.ctypes.data_as(ctypes.c_void_p),
            max_len, sp.ctypes.data_as(_i32p), st.ctypes.data_as(_i32p),
            None if se is None else se.ctypes.data_as(_i32p),
            tot.ctypes.data_as(_i64p)))

    def morton_scan():
        from .schedule import morton_order
        cent = np.asarray(base.coords)[cv].mean(axis=1)
        return np.ascontiguousarray(morton_order(cent), dtype=np.int32)

    # (run strips follow the id bands: index order, no Morton rebuild)
    mode = scan or ("index" if runs else
                    os.environ.get("PM_STRIP_SCAN", "auto"))
    run(morton_scan() if mode == "morton" else None)
    if mode == "auto" and tot[0] > 0 and max_len >= 8:
        # index-order strips on a mesh whose cell order is not spatially
        # coherent (e.g. a random vertex order) come out short: rebuild
        # them starting in the Morton order of the cell centroids
        cells_per = (tot[1] - 2 * tot[0]) / tot[0]
        if cells_per < 0.5 * max_len:
            run(morton_scan())
    sp, st = sp[:tot[0] + 1].copy(), st[:tot[1]].copy()
    if se is not None:
        se = se[:tot[1]].copy()
    # strips in the Morton order of their centroids: strips running
    # concurrently on the GPU form a compact region, so the two strips that
    # share a vertex row run close in time and the second one finds the
    # row in L2 (C5b: HBM reads 30.8 -> 21.0 GB, -10 % time; measured,
    # profiles/README.md).  PM_STRIP_ORDER=rcm: by mean vertex id instead.
    mode = order or os.environ.get("PM_STRIP_ORDER", "morton")
    if mode == "creation":
        return (sp, st) if se is None else (sp, st, se)
    lens = np.diff(sp)
    sums = np.add.reduceat(st.astype(np.int64), sp[:-1]) if lens.size else \
        np.zeros(0)
    order = np.argsort(sums / np.maximum(lens, 1), kind="stable")
    if mode == "morton" and lens.size:
        from .schedule import morton_order
        xy = np.asarray(base.coords)[st]
        cx = np.add.reduceat(xy[:, 0], sp[:-1]) / np.maximum(lens, 1)
        cy = np.add.reduceat(xy[:, 1], sp[:-1]) / np.maximum(lens, 1)
        order = morton_order(np.stack([cx, cy], axis=1))
    new_sp = np.zeros_like(sp)
    np.cumsum(lens[order], out=new_sp[1:])
    idx = np.concatenate([np.arange(sp[i], sp[i + 1]) for i in order]) \
        if order.size else np.zeros(0, dtype=np.int64)
    if se is not None:
        return new_sp, st[idx].astype(np.int32), \
            np.ascontiguousarray(se[idx], dtype=np.int32)
    return new_sp, st[idx].astype(np.int32)


def build_patch_strips(base, patch_cells, patch_ptr, max_len=1 << 30,
                       edges=False):
    """Store-first patch strips (host C++, pm_build_patch_strips): returns
    (item_ptr, strip_ptr, steps[, steps_e], zero_list), all int32.  Cells
    ``patch_cells[patch_ptr[p]:patch_ptr[p+1]]`` form patch p; step ids
    carry ``STEP_STORE`` on the first residency of a patch-interior
    entity; ``zero_list`` = entities shared by several patches (vertex v,
    or n_vertices + edge e)."""
    cv = np.ascontiguousarray(base.cell_vertices, dtype=np.int32)
    ce = np.ascontiguousarray(base.cell_edges, dtype=np.int32)
    n = cv.shape[0]
    pc = np.ascontiguousarray(patch_cells, dtype=np.int32)
    pp = np.ascontiguousarray(patch_ptr, dtype=np.int32)
    n_p = pp.shape[0] - 1
    n0, n1 = base.num_vertices, base.num_edges
    ip = np.zeros(n_p + 1, dtype=np.int32)
    sp = np.zeros(n + 1, dtype=np.int32)
    st = np.zeros(3 * n + 3, dtype=np.int32)
    se = np.zeros((3 * n + 3, 2), dtype=np.int32) if edges else None
    zl = np.zeros(n0 + n1 + 1, dtype=np.int32)
    tot = np.zeros(3, dtype=np.int64)
    check(host_lib().pm_build_patch_strips(
        n, n0, n1, cv.ctypes.data_as(_i32p), ce.ctypes.data_as(_i32p),
        pc.ctypes.data_as(_i32p), pp.ctypes.data_as(_i32p), n_p, max_len,
        ip.ctypes.data_as(_i32p), sp.ctypes.data_as(_i32p),
        st.ctypes.data_as(_i32p),
        None if se is None else se.ctypes.data_as(_i32p),
        zl.ctypes.data_as(_i32p), tot.ctypes.data_as(_i64p)))
    out = [ip, sp[:tot[0] + 1].copy(), st[:tot[1]].copy()]
    if se is not None:
        out.append(se[:tot[1]].copy())
    out.append(zl[:tot[2]].copy())
    return tuple(out)


#: flag bits of patch-strip step ids: store-first residency, no cell after
#: the step (a strip's first two fill steps)
STEP_STORE = 1 << 30
STEP_NOCELL = 1 << 29



def column_mass_patch_strips(layout, k, layers, coords, mref, x, y, n_dofs,
                             plan, kron, chunk, accumulate=False, stream=None,
                             n_vertices=0):
    """pm_column_mass_patch_strips; ``plan`` = device tensors (item_ptr,
    strip_ptr, steps, steps_e or None, zero_list)."""
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    mt = np.ascontiguousarray(kron[0], dtype=np.float64).ravel()
    ml = np.ascontiguousarray(kron[1], dtype=np.float64).ravel()
    d = layout.delta6()
    ip, sp, st, se, zl = plan
    rc = host_lib().pm_column_mass_patch_strips(
        d.ctypes.data_as(_i32p), k, layers, ptr(coords), _f64ptr(m),
        _f64ptr(mt), _f64ptr(ml), ptr(x), ptr(y), n_dofs,
        1 if accumulate else 0, ip.shape[0] - 1, chunk, ptr(ip), ptr(sp),
        ptr(st), ptr(se), n_vertices, zl.shape[0], ptr(zl),
        stream_ptr(stream))
    check(rc)


def column_mass_strip_red(layout, k, layers, coords, mref, x, y, n_dofs,
                          strips, kron, chunk, accumulate=False, stream=None,
                          x_base=0, y_base=0, coords_base=0, n_vertices=0):
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    mt = np.ascontiguousarray(kron[0], dtype=np.float64).ravel()
    ml = np.ascontiguousarray(kron[1], dtype=np.float64).ravel()
    d = layout.delta6()
    sp, st = strips[0], strips[1]
    se = strips[2] if len(strips) > 2 else None
    rc = host_lib().pm_column_mass_strip_red(
        d.ctypes.data_as(_i32p), k, layers, ptr(coords, coords_base),
        _f64ptr(m), _f64ptr(mt), _f64ptr(ml), ptr(x, x_base), ptr(y, y_base),
        n_dofs, 1 if accumulate else 0, sp.shape[0] - 1, chunk, ptr(sp),
        ptr(st), ptr(se), n_vertices, stream_ptr(stream))
    check(rc)


def column_mass_strip_tma(layout, k, layers, coords, x, y, n_dofs, strips,
                          kron, accumulate=False, stream=None, n_vertices=0):
    """pm_column_mass_strip_tma: the run-strip kernel (bulk copies of whole
    vertex columns), P1 / 3-vector P1, at most 128 layers."""
    mt = np.ascontiguousarray(kron[0], dtype=np.float64).ravel()
    ml = np.ascontiguousarray(kron[1], dtype=np.float64).ravel()
    d = layout.delta6()
    sp, st = strips[0], strips[1]
    rc = host_lib().pm_column_mass_strip_tma(
        d.ctypes.data_as(_i32p), k, layers, ptr(coords), _f64ptr(mt),
        _f64ptr(ml), ptr(x), ptr(y), n_dofs, 1 if accumulate else 0,
        sp.shape[0] - 1, ptr(sp), ptr(st), n_vertices, stream_ptr(stream))
    check(rc)


def column_mass_strip_red_peer(layout, k, layers, coords, mref, x, y,
                               n_dofs, strips, kron, chunk, y_peer,
                               ghost_vertex_end, accumulate=False,
                               stream=None, x_base=0, y_base=0,
                               coords_base=0, n_vertices=0):
    """pm_column_mass_strip_red_peer: ``y_peer`` is a device address (int)
    already shifted to global DoF indexing (see shard.PeerWindow)."""
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    mt = np.ascontiguousarray(kron[0], dtype=np.float64).ravel()
    ml = np.ascontiguousarray(kron[1], dtype=np.float64).ravel()
    d = layout.delta6()
    sp, st = strips[0], strips[1]
    rc = host_lib().pm_column_mass_strip_red_peer(
        d.ctypes.data_as(_i32p), k, layers, ptr(coords, coords_base),
        _f64ptr(m), _f64ptr(mt), _f64ptr(ml), ptr(x, x_base), ptr(y, y_base),
        n_dofs, 1 if accumulate else 0, sp.shape[0] - 1, chunk, ptr(sp),
        ptr(st), n_vertices, ctypes.c_void_p(y_peer), ghost_vertex_end,
        stream_ptr(stream))
    check(rc)


def ipc_export(t):
    """(64-byte handle, byte offset) of device tensor ``t``'s storage."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    check(host_lib().pm_ipc_export(ptr(t), h, ctypes.byref(off)))
    return h.raw, off.value


def ipc_open(handle, offset):
    """Map a peer's exported buffer: the device address (int)."""
    p = ctypes.c_void_p(0)
    h = ctypes.create_string_buffer(bytes(handle), 64)
    check(host_lib().pm_ipc_open(h, int(offset), ctypes.byref(p)))
    return p.value


def ipc_close(addr, offset):
    check(host_lib().pm_ipc_close(ctypes.c_void_p(addr), int(offset)))


def stream_signal(addr, value, stream=None):
    """Queue: after the stream's work, store ``value`` (uint32) to device
    address ``addr`` (local or a peer mapping)."""
    check(host_lib().pm_stream_signal(ctypes.c_void_p(addr),
                                      int(value) & 0xffffffff,
                                      stream_ptr(stream)))


def stream_wait_geq(addr, value, stream=None):
    """The stream waits until the uint32 at local ``addr`` is >= value."""
    check(host_lib().pm_stream_wait_geq(ctypes.c_void_p(addr),
                                        int(value) & 0xffffffff,
                                        stream_ptr(stream)))


def column_mass_dg_range(layout, k, c0, c1, layers, cmap, offs, xmap, xoffs,
                         coords, mref, x, y, stream=None):
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    d = layout.delta6()
    check(host_lib().pm_column_mass_dg_range(
        d.ctypes.data_as(_i32p), k, c0, c1, layers, ptr(cmap), ptr(offs),
        ptr(xmap), ptr(xoffs), ptr(coords), _f64ptr(m), ptr(x), ptr(y),
        stream_ptr(stream)))


def greedy_color_cells(cell_vertices, vc_offsets, vc_cells):
    cv = np.ascontiguousarray(cell_vertices, dtype=np.int32)
    off = np.ascontiguousarray(vc_offsets, dtype=np.int64)
    vcc = np.ascontiguousarray(vc_cells, dtype=np.int32)
    n = cv.shape[0]
    color = np.empty(n, dtype=np.int32)
    nc = ctypes.c_int32(0)
    check(host_lib().pm_greedy_color_cells(
        cv.ctypes.data_as(_i32p), n, off.ctypes.data_as(_i64p),
        vcc.ctypes.data_as(_i32p), color.ctypes.data_as(_i32p),
        ctypes.byref(nc)))
    return color, nc.value


def halo_pack(y, cols, col, buf, base=0, stream=None):
    check(host_lib().pm_halo_pack(ptr(y, base), ptr(cols), cols.shape[0], col,
                                  ptr(buf), stream_ptr(stream)))


def halo_unpack_add(y, cols, col, buf, base=0, stream=None):
    check(host_lib().pm_halo_unpack_add(ptr(y, base), ptr(cols),
                                        cols.shape[0], col, ptr(buf),
                                        stream_ptr(stream)))


def derive_edges_device(cell_vertices, num_vertices=None):
    """Device derive_edges: ``(edge_vertices, cell_edges, status)`` as numpy
    int32 arrays; ``status`` != 0 flags a topology error (see the header)."""
    import numpy as np
    import torch
    dev = cuda_device()
    cells = host_tensor(cell_vertices, np.int32).to(dev)
    n_cells = cells.shape[0]
    ev = torch.empty((3 * n_cells, 2), dtype=torch.int32, device=dev)
    ce = torch.empty((n_cells, 3), dtype=torch.int32, device=dev)
    n = ctypes.c_int64(0)
    st = ctypes.c_int32(0)
    check(host_lib().pm_derive_edges(
        ptr(cells), n_cells, -1 if num_vertices is None else int(num_vertices),
        ptr(ev), ptr(ce), ctypes.byref(n), ctypes.byref(st),
        stream_ptr(None)))
    if st.value:
        return None, None, st.value
    return ev[:n.value].cpu().numpy(), ce.cpu().numpy(), 0


def vertex_graph_sorted_device(edge_vertices, n_vertices):
    """(offsets int64 (n+1,), neighbours int64) of the vertex graph, rows
    sorted by (degree, index), built on the device."""
    import numpy as np
    import torch
    dev = cuda_device()
    ev = host_tensor(edge_vertices, np.int32).to(dev)
    ne = ev.shape[0]
    off = torch.empty(n_vertices + 1, dtype=torch.int64, device=dev)
    nb = torch.empty(2 * ne, dtype=torch.int32, device=dev)
    check(host_lib().pm_vertex_graph_sorted(ptr(ev), ne, n_vertices, ptr(off),
                                            ptr(nb), stream_ptr(None)))
    return off.cpu().numpy(), nb.cpu().numpy().astype(np.int64)


def strip_step_cells(base, strip_ptr, steps):
    """The cell each strip step forms (-1 on fill steps), host C++."""
    cv = np.ascontiguousarray(base.cell_vertices, dtype=np.int32)
    sp = np.ascontiguousarray(strip_ptr, dtype=np.int32)
    st = np.ascontiguousarray(steps, dtype=np.int32)
    out = np.empty(st.shape[0], dtype=np.int32)
    check(host_lib().pm_strip_step_cells(
        cv.shape[0], base.num_vertices, cv.ctypes.data_as(ctypes.c_void_p),
        sp.ctypes.data_as(ctypes.c_void_p), sp.shape[0] - 1,
        st.ctypes.data_as(ctypes.c_void_p),
        out.ctypes.data_as(ctypes.c_void_p)))
    return out


def column_mass_strip_dg(layout, k, n_cells, layers, coords, mref, x, y,
                         strips, chunk, stream=None):
    """pm_column_mass_strip_dg: ``strips`` = device (strip_ptr, steps,
    step_cells)."""
    m = np.ascontiguousarray(mref, dtype=np.float64).ravel()
    d = layout.delta6()
    sp, st, sc = strips
    check(host_lib().pm_column_mass_strip_dg(
        d.ctypes.data_as(_i32p), k, n_cells, layers, ptr(coords), _f64ptr(m),
        ptr(x),
        ptr(y), sp.shape[0] - 1, chunk, ptr(sp), ptr(st), ptr(sc),
        stream_ptr(stream)))


def experimental() -> bool:
    """The library was built with the experimental schedules (tile,
    store-first patch strips): PM_EXPERIMENTAL=1 at build time."""
    return bool(host_lib().pm_build_flags() & 1)


def stencil_check(source, k_in, k_out):
    """NVRTC-compile a user stencil kernel (no device needed); the cubin
    size in bytes.  Compile errors raise ValueError with NVRTC's log."""
    import numpy as np
    k = np.ascontiguousarray(k_in, dtype=np.int32)
    n = ctypes.c_int64(0)
    check(host_lib().pm_stencil_check(source.encode(), k.shape[0],
                                      k.ctypes.data_as(_i32p), int(k_out),
                                      ctypes.byref(n)))
    return n.value


def stencil_compile(source, k_in, k_out):
    """Handle (int) of a compiled and loaded user stencil kernel."""
    import numpy as np
    cuda_device()
    k = np.ascontiguousarray(k_in, dtype=np.int32)
    h = ctypes.c_void_p(0)
    check(host_lib().pm_stencil_compile(source.encode(), k.shape[0],
                                        k.ctypes.data_as(_i32p), int(k_out),
                                        ctypes.byref(h)))
    return h.value


def stencil_launch(handle, colored, n_cells, layers, fields, maps, offsets,
                   out, out_map, out_offsets, cells=None, stream=None):
    n = len(fields)
    arr = ctypes.c_void_p * max(n, 1)
    f = arr(*[t.data_ptr() for t in fields])
    m = arr(*[t.data_ptr() for t in maps])
    o = arr(*[t.data_ptr() for t in offsets])
    check(host_lib().pm_stencil_launch(
        ctypes.c_void_p(handle), 1 if colored else 0, int(n_cells),
        int(layers), f, m, o, ptr(out), ptr(out_map), ptr(out_offsets),
        ptr(cells) if cells is not None else None, stream_ptr(stream)))


def stencil_free(handle):
    if handle:
        check(host_lib().pm_stencil_free(ctypes.c_void_p(handle)))


def rcm_walk_device(offsets, neighbours_sorted):
    """Cuthill-McKee visit order (int64 numpy) of a host CSR whose rows are
    sorted by (degree, index), walked on the device (pm_rcm_order_device)."""
    import numpy as np
    import torch
    dev = cuda_device()
    off = host_tensor(offsets, np.int64).to(dev)
    n = off.shape[0] - 1
    nb = host_tensor(neighbours_sorted, np.int32).to(dev)
    if nb.numel() == 0:
        nb = torch.zeros(1, dtype=torch.int32, device=dev)
    order = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    check(host_lib().pm_rcm_order_device(ptr(off), ptr(nb), n, ptr(order),
                                         stream_ptr(None)))
    return order[:n].cpu().numpy()


def rcm_forward_device(edge_vertices, n_vertices):
    """RCM ``forward`` permutation (int64 numpy) with the vertex graph AND
    the Cuthill-McKee walk on the device (pm_vertex_graph_sorted +
    pm_rcm_order_device), the reversal by a device scatter."""
    import numpy as np
    import torch
    dev = cuda_device()
    ev = host_tensor(edge_vertices, np.int32).to(dev)
    ne = ev.shape[0]
    off = torch.empty(n_vertices + 1, dtype=torch.int64, device=dev)
    nb = torch.empty(max(1, 2 * ne), dtype=torch.int32, device=dev)
    lib = host_lib()
    check(lib.pm_vertex_graph_sorted(ptr(ev), ne, n_vertices, ptr(off),
                                     ptr(nb), stream_ptr(None)))
    order = torch.empty(n_vertices, dtype=torch.int64, device=dev)
    check(lib.pm_rcm_order_device(ptr(off), ptr(nb), n_vertices, ptr(order),
                                  stream_ptr(None)))
    forward = torch.empty_like(order)
    forward[order.flip(0)] = torch.arange(n_vertices, dtype=torch.int64,
                                          device=dev)
    return forward.cpu().numpy()


def reorder_cells_device(cell_vertices, forward):
    """Device apply_ordering cell re-sort: ``forward[cells][perm]``."""
    import numpy as np
    import torch
    dev = cuda_device()
    cells = host_tensor(cell_vertices, np.int32).to(dev)
    fwd = host_tensor(forward, np.int64).to(dev)
    out = torch.empty_like(cells)
    check(host_lib().pm_reorder_cells(ptr(cells), cells.shape[0], ptr(fwd),
                                      fwd.shape[0], ptr(out), None,
                                      stream_ptr(None)))
    return out.cpu().numpy()


def stream_triad(a, b, c, alpha, stream=None):
    """``a = b + alpha * c`` on the device (float64 CUDA tensors)."""
    n = a.numel()
    if b.numel() != n or c.numel() != n:
        raise ValueError("triad arrays differ in length")
    check(host_lib().pm_stream_triad(ptr(a), ptr(b), ptr(c), float(alpha),
                                     n, stream_ptr(stream)))


def set_launch_overlap(on):
    """Programmatic dependent launch for this thread's stream kernels
    (see the header); returns the previous setting."""
    return bool(host_lib().pm_set_launch_overlap(1 if on else 0))


def device_info():
    sm = ctypes.c_int32(0)
    l2 = ctypes.c_int64(0)
    check(host_lib().pm_device_info(ctypes.byref(sm), ctypes.byref(l2)))
    return sm.value, l2.value


# ---------------------------------------------------------------------------
# band-tile schedule (csrc/tile_plan.cpp, csrc/tile.cu)
# ---------------------------------------------------------------------------

TILE_ARRAYS = ("cell_ptr", "run_ptr", "run_v0", "run_n", "run_fa", "run_ca",
               "zero_ptr", "zero_v0", "zero_n", "dep_ptr", "deps",
               "strip_ptr", "strip_step0", "strip_len")


def build_tiles(base, col_f_bytes, col_c_bytes, budget, max_cells=256,
                min_strips=1, min_sub=4, arrays=True):
    """Host plan of the tile schedule (pm_tiles_build): the per-tile records
    ``blob`` (int32) with offsets ``off`` (int64) the kernel reads, and the
    sizes ``n_tiles``, ``max_fa``, ``max_ca`` (bytes), ``max_slots``,
    ``max_cells``, ``max_words``; ``arrays``: also the plan as separate
    int32 arrays (TILE_ARRAYS) and int16 ``steps`` (tests)."""
    cv = np.ascontiguousarray(base.cell_vertices, dtype=np.int32)
    ce = np.ascontiguousarray(base.cell_edges, dtype=np.int32)
    h = ctypes.c_void_p()
    L = host_lib()
    check(L.pm_tiles_build(cv.shape[0], base.num_vertices, base.num_edges,
                           cv.ctypes.data_as(ctypes.c_void_p),
                           ce.ctypes.data_as(ctypes.c_void_p), int(col_f_bytes),
                           int(col_c_bytes), int(budget), int(max_cells),
                           int(min_strips), int(min_sub), ctypes.byref(h)))
    try:
        info = np.zeros(11, dtype=np.int64)
        check(L.pm_tiles_info(h, info.ctypes.data_as(_i64p)))
        nt, nr, nz, nd, ns, nk = (int(v) for v in info[:6])
        sizes = np.zeros(2, dtype=np.int64)
        check(L.pm_tiles_blob(h, None, None, sizes.ctypes.data_as(_i64p)))
        blob = np.zeros(max(1, int(sizes[0])), dtype=np.int32)
        off = np.zeros(nt + 1, dtype=np.int64)
        check(L.pm_tiles_blob(h, blob.ctypes.data_as(ctypes.c_void_p),
                              off.ctypes.data_as(ctypes.c_void_p),
                              sizes.ctypes.data_as(_i64p)))
        plan = {"blob": blob, "off": off, "n_tiles": nt,
                "max_fa": int(info[6]), "max_ca": int(info[7]),
                "max_slots": int(info[8]), "max_cells": int(info[9]),
                "max_strips": int(info[10]), "max_words": int(sizes[1])}
        if arrays:
            lens = {"cell_ptr": nt + 1, "run_ptr": nt + 1, "run_v0": nr,
                    "run_n": nr, "run_fa": nr, "run_ca": nr,
                    "zero_ptr": nt + 1, "zero_v0": nz, "zero_n": nz,
                    "dep_ptr": nt + 1, "deps": nd, "strip_ptr": nt + 1,
                    "strip_step0": ns, "strip_len": ns}
            out = {k: np.zeros(max(lens[k], 1), dtype=np.int32)
                   for k in TILE_ARRAYS}
            steps = np.zeros(max(nk, 1), dtype=np.int16)
            arr = (_vp * 14)(*[out[k].ctypes.data_as(ctypes.c_void_p)
                               for k in TILE_ARRAYS])
            check(L.pm_tiles_export(h, arr,
                                    steps.ctypes.data_as(ctypes.c_void_p)))
            plan.update({k: out[k][:lens[k]] for k in TILE_ARRAYS})
            plan["steps"] = steps[:nk]
    finally:
        L.pm_tiles_free(h)
    return plan


def tile_smem_layout(layout, max_words, max_slots, width):
    """(bytes in front of the data buffers, number of buffers, CTA size)."""
    d = layout.delta6()
    st, th = ctypes.c_int32(0), ctypes.c_int32(0)
    off = host_lib().pm_tile_smem_layout(d.ctypes.data_as(_i32p),
                                         int(max_words), int(max_slots),
                                         int(width), ctypes.byref(st),
                                         ctypes.byref(th))
    return int(off), int(st.value), int(th.value)


def column_mass_tile(layout, layers, coords, x, y, n_dofs, dplan, kron,
                     width, stream=None, x_base=0, y_base=0, coords_base=0):
    """pm_column_mass_tile: y = M x with the band-tile schedule (y needs no
    zeroing: every output column is zeroed by the tile that touches it
    first)."""
    mt = np.ascontiguousarray(kron[0], dtype=np.float64).ravel()
    ml = np.ascontiguousarray(kron[1], dtype=np.float64).ravel()
    d = layout.delta6()
    check(host_lib().pm_column_mass_tile(
        d.ctypes.data_as(_i32p), layers, ptr(coords, coords_base),
        coords_base + coords.shape[0], _f64ptr(mt), _f64ptr(ml),
        ptr(x, x_base), ptr(y, y_base), n_dofs, ptr(dplan["blob"]),
        ptr(dplan["off"]), ptr(dplan["zero_ptr"]), ptr(dplan["zero_v0"]),
        ptr(dplan["zero_n"]), ptr(dplan["ctl"]), ptr(dplan["flags"]),
        dplan["n_tiles"], dplan["area_c"], dplan["data_bytes"],
        dplan["max_slots"], dplan["max_words"], int(width),
        stream_ptr(stream)))

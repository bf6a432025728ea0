"""Rooflines of the path's setup kernels: K0
(pm_build_cell_map: bottom-layer cell maps + offsets) and the extruded
coordinate field (pm_extrude_coordinates), as GB/s of the bytes each
must move (reads of the mesh arrays + writes of the output) against the
measured HBM copy bandwidth.  One JSON line per (config, kernel)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_1604_05937_b200 import _lib, configs  # noqa: E402
from paper_1604_05937_b200.extrusion import ExtrudedMesh  # noqa: E402
from paper_1604_05937_b200.fspace import number_dofs  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6554.9


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name in sys.argv[1:] or ["C2", "C3", "C5a", "C5b"]:
    w = configs.workload(name)
    fs, _q, _x, _ = configs.build(w)
    base = fs.mesh.base
    k = fs.num_slots
    _lib.build_cell_map_device(fs)          # mesh arrays resident
    ms = timed(lambda: _lib.build_cell_map_device(fs))
    nbytes = base.num_cells * (4 * k + 24) + 4 * k
    print(json.dumps({"config": name, "kernel": "K0 pm_build_cell_map",
                      "k": k, "cells": base.num_cells, "ms": ms,
                      "bytes": nbytes, "GBs": nbytes / ms / 1e6,
                      "pct_hbm": 100 * nbytes / ms / 1e6 / PEAK}))
    d_base = torch.from_numpy(base.coords.copy()).cuda()
    ms = timed(lambda: _lib.extrude_coordinates_device(
        d_base, fs.mesh.layers, fs.mesh.layer_height))
    nbytes = 16 * base.num_vertices + 24 * base.num_vertices * \
        (fs.mesh.layers + 1)
    print(json.dumps({"config": name, "kernel": "k_extrude",
                      "vertices": base.num_vertices, "ms": ms,
                      "bytes": nbytes, "GBs": nbytes / ms / 1e6,
                      "pct_hbm": 100 * nbytes / ms / 1e6 / PEAK}))

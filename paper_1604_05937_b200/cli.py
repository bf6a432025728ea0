"""Experiment driver (SPEC.md ``cli`` module, ``perfbench.run_experiment``).

``python -m paper_1604_05937_b200 <bench | stream | verify> [flags]``

* ``bench`` — the cross product layouts × orderings × λ of the mass-action
  column loop on the GPU, one CSV row each in the SPEC schema
  (``perfbench.CSV_HEADER``): min-of-repeats device time (CUDA events, L2
  flushed between repeats), valuable bytes / GB/s, flops, the peak model and
  the STREAM-triad bandwidth of this GPU.
* ``stream`` — the device triad alone: ``stream_gbs=<value>``.
* ``verify`` — ``verification.run_oracle_suite``: the nine layouts on the
  three fixture meshes against the literal baselines (and, with a GPU, the
  device maps, loop lists and assembly); exit 0 iff all pass.

Flags follow the SPEC (``--generate``, ``--layers``, ``--horiz``,
``--vert``, ``--ordering``, ``--seed``, ``--threads``, ``--repeats``,
``--quad-degree``, ``--target-cells``, ``--hw``, ``--out``).  ``--threads``
has no GPU meaning and is recorded as the SM count; ``--mesh`` files are
not read (mesh loaders are out of scope).
"""
from __future__ import annotations

import argparse
import math
import os
import sys


def _ints(s):
    return [int(v) for v in s.split(",") if v]


def _names(s):
    return [v for v in s.split(",") if v]


def read_hw(path):
    """``key=value`` hardware config (SPEC perfbench External Interfaces):
    ``sm_count``, ``clock_ghz``, ``fp64_lanes_per_sm``, ``llc_bytes``,
    ``stream_gbs_override``."""
    out = {}
    if path:
        with open(path) as f:
            for line in f:
                line = line.split("#", 1)[0].strip()
                if line:
                    k, v = line.split("=", 1)
                    out[k.strip()] = float(v)
    return out


def base_n(target_cells: int, layers: int) -> int:
    """Generator size so that 2 n² λ ≈ target (SPEC run_experiment)."""
    n = round(math.sqrt(target_cells / (2 * layers)))
    if n < 1:
        raise ValueError(f"target {target_cells} cells too small for "
                         f"{layers} layers")
    return n


def _l2_flush(torch, nbytes):
    buf = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")

    def flush():
        buf.fill_(1)
    return flush


def stream_triad(array_len=None, repeats=10, hw=None):
    """Best device triad bandwidth (GB/s) over ``repeats`` passes; the
    arrays together exceed 4× the L2 (SPEC stream_triad pre-condition)."""
    import torch
    from . import _lib
    hw = hw or {}
    if "stream_gbs_override" in hw:
        return hw["stream_gbs_override"]
    _sm, l2 = _lib.device_info()
    llc = int(hw.get("llc_bytes", l2))
    n = array_len or max(1 << 24, (4 * llc) // 24 * 4)
    a = torch.empty(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda")
    c = torch.rand(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    best = 0.0
    for r in range(repeats + 1):
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        e0.record(s)
        _lib.stream_triad(a, b, c, 3.0, stream=s)
        e1.record(s)
        e1.synchronize()
        if r:  # first pass is warm-up
            best = max(best, 24.0 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    if not torch.allclose(a[:1024], b[:1024] + 3.0 * c[:1024]):
        raise RuntimeError("triad result wrong")
    return best


def peak_model(profile, hw, sm_count):
    """SPEC P_d = B_c · f_b · f_v on the GPU: B_c = one fp64 instruction
    per cycle per fp64 lane (SMs × lanes × clock), f_b from the kernel's
    add/mul/fma counts; f_v = 1 (SIMT lanes are already counted in B_c)."""
    from .perfbench import balance_factor, peak_throughput
    lanes = hw.get("fp64_lanes_per_sm", 64)
    clock = hw.get("clock_ghz", 1.965)
    bc = hw.get("sm_count", sm_count) * lanes * clock      # GFLOP/s
    fb = balance_factor(profile.adds, profile.muls, profile.fmas,
                        "fma" if profile.fmas else "no-fma")
    fv = 1.0
    return fb, fv, peak_throughput(bc, fb, fv)


def run_experiment(layout, ordering, layers, n, seed=0, repeats=10,
                   quad_degree=None, schedule="auto", stream_gbs=None,
                   hw=None):
    """One PerfRecord (a dict in CSV-column order) for a mesh of 2 n² cells."""
    import torch
    from . import _lib
    from .configs import base_mesh
    from .extrusion import ExtrudedMesh, extrude_coordinates
    from .fspace import number_dofs
    from .kernels import MassOperator, count_flops
    from .perfbench import valuable_volume
    from .quadrature import prism_quadrature
    hw = hw or {}
    base, rng = base_mesh(n, ordering, 0.0, seed)
    mesh = ExtrudedMesh(base, layers)
    fs = number_dofs(mesh, layout)
    quad = prism_quadrature(quad_degree, quad_degree) if quad_degree else None
    op = MassOperator(fs, quad, schedule=schedule)
    x = torch.from_numpy(rng.random(fs.total_dofs)).cuda()
    coords = extrude_coordinates(base.coords, layers, mesh.layer_height)
    y = torch.empty_like(x)
    sm, l2 = _lib.device_info()
    flush = _l2_flush(torch, 2 * l2)
    s = torch.cuda.current_stream()
    times = []
    for r in range(repeats + 1):
        flush()
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        e0.record(s)
        op.apply(x, coords, y)
        e1.record(s)
        e1.synchronize()
        if r:  # warm-up run excluded (SPEC run_experiment)
            times.append(e0.elapsed_time(e1) * 1e-3)
    t = min(times)
    vol = valuable_volume(fs)
    prof = count_flops(fs.layout, op.quadrature)
    flops = prof.total_flops * base.num_cells * layers
    fb, fv, peak = peak_model(prof, hw, sm)
    gflops = flops / t / 1e9
    return {"layout": fs.layout.name, "ordering": ordering, "layers": layers,
            "base_cells": base.num_cells, "threads": sm, "runtime_s": t,
            "valuable_bytes": vol, "valuable_gbs": vol / t / 1e9,
            "flops": flops, "gflops": gflops, "f_b": fb, "f_v": fv,
            "peak_gflops": peak, "peak_fraction": gflops / peak,
            "stream_gbs": stream_gbs}


def _fmt(v):
    if isinstance(v, float):
        return f"{v:.6g}"
    return "" if v is None else str(v)


def cmd_bench(args):
    from .fspace import builtin_layout
    from .perfbench import CSV_HEADER
    if args.mesh:
        raise SystemExit("bench: --mesh files are not read (mesh loaders are "
                         "out of scope); use --generate N or --target-cells")
    hw = read_hw(args.hw)
    layouts = [builtin_layout(h, v) for h in _names(args.horiz)
               for v in _names(args.vert)]
    stream_gbs = stream_triad(hw=hw)
    out = open(args.out, "a") if args.out else sys.stdout
    try:
        if not args.out or out.tell() == 0:
            print(CSV_HEADER, file=out)
        for layout in layouts:
            for ordering in _names(args.ordering):
                for lam in _ints(args.layers):
                    n = args.generate or base_n(args.target_cells, lam)
                    try:
                        rec = run_experiment(layout, ordering, lam, n,
                                             args.seed, args.repeats,
                                             args.quad_degree, args.schedule,
                                             stream_gbs, hw)
                    except Exception as e:  # name the failing stage
                        raise SystemExit(f"bench: {layout.name} {ordering} "
                                         f"λ={lam}: {e}")
                    print(",".join(_fmt(v) for v in rec.values()), file=out)
                    out.flush()
    finally:
        if args.out:
            out.close()
    return 0


def cmd_stream(args):
    print(f"stream_gbs={stream_triad(repeats=args.repeats, hw=read_hw(args.hw)):.1f}")
    return 0


def cmd_verify(args):
    from .verification import run_oracle_suite
    return 0 if run_oracle_suite(layers=args.verify_layers) else 1


def parser():
    p = argparse.ArgumentParser(prog="python -m paper_1604_05937_b200",
                                description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="layouts x orderings x layers -> CSV")
    b.add_argument("--mesh")
    b.add_argument("--generate", type=int, default=0)
    b.add_argument("--layers", default="1,2,3,4,5,6,7,8,9,10,20,30,40,50,"
                                       "60,70,80,90,100")
    b.add_argument("--horiz", default="CG1")
    b.add_argument("--vert", default="CG1")
    b.add_argument("--ordering", default="rcm")
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--threads", type=int, default=0,
                   help="ignored on the GPU (recorded: SM count)")
    b.add_argument("--repeats", type=int, default=10)
    b.add_argument("--quad-degree", type=int, default=0)
    b.add_argument("--target-cells", type=int, default=15_000_000)
    b.add_argument("--schedule", default="auto")
    b.add_argument("--hw")
    b.add_argument("--out")
    s = sub.add_parser("stream", help="device STREAM triad")
    s.add_argument("--repeats", type=int, default=10)
    s.add_argument("--hw")
    v = sub.add_parser("verify", help="oracle-equivalence suite")
    v.add_argument("--layers", dest="verify_layers", type=int, default=4)
    return p


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    return {"bench": cmd_bench, "stream": cmd_stream,
            "verify": cmd_verify}[args.cmd](args)


if __name__ == "__main__":
    sys.exit(main())

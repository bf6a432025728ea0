"""Benchmark: the extruded-mesh column loop on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
                    [--impl ours|reference]

A "step" is one pass of the column loop (mass action y = M x with |det J|
from the extruded coordinate field) over the whole workload.  Default
workload: BASELINE config 2 (DG1 mass action, 256^2 split-square RCM base,
50 layers, fp64) -- configs[1] of BASELINE.json.  Metric: valuable HBM
bandwidth (input + output + coordinate field, each once)
divided by the device time, plus cell-layers/s.

``--impl reference`` times the reference algorithm's CPU restatement (the
oracle's coloured-parallel column loop with literal quadrature,
``oracle/``) on the host cores instead; the reference package itself has
no par-loop implementation.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "valuable HBM bandwidth of the column loop (SPEC.md:467-475 bytes)"
UNIT = "GB/s"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, only without the file


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20,
                   help="timed steps (>= 1)")
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C2")
    p.add_argument("--schedule", default="auto")
    p.add_argument("--impl", default="ours", choices=("ours", "reference"))
    p.add_argument("--cpu-seconds", type=float, default=8.0,
                   help="CPU-baseline sample budget")
    p.add_argument("--no-cpu-baseline", action="store_true")
    args = p.parse_args()
    if args.steps < 1 or args.warmup < 0:
        p.error("--steps must be >= 1 and --warmup >= 0")
    return args


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    """dram bytes per launch of the dominant kernel from the committed ncu
    summary (profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config)
    except (OSError, ValueError):
        return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML in a tight loop (≈ every 0.2 ms, so even a few-ms region
    gets many samples), nvidia-smi as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,"
         "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self.source = None
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [(n, getattr(nv, a)) for n, a in self.REASONS]
            self.source = "nvml"
            while True:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.mx.append(mx)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(n for n, b in bits if r & b)
                if self._stop.wait(0.0002):
                    break
        finally:
            nv.nvmlShutdown()

    def _run_smi(self):
        self.source = "nvidia-smi"
        names = [n for n, _a in self.REASONS]
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index),
                     f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout
            except (OSError, subprocess.SubprocessError):
                return
            for line in out.strip().splitlines():
                r = [c.strip() for c in line.split(",")]
                if r[1].replace(".", "").isdigit():
                    self.sm.append(float(r[1]))
                if r[2].replace(".", "").isdigit():
                    self.mx.append(float(r[2]))
                self.reasons.update(names[i] for i in range(4)
                                    if len(r) > 5 + i and r[5 + i] == "Active")
            self._stop.wait(0.2)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)    # the sampler is running before the region starts
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)),
                "sm_max_mhz": float(max(self.mx)) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": self.source}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class CpuArm:
    """The oracle's coloured column loop (literal quadrature, pthreads) on
    a bounded sample of the workload: the first ``n`` base cells, all
    layers.  Cells are taken in index order, so the sample keeps the RCM
    locality of the full mesh."""

    def __init__(self, w, fs, x, threads=0):
        import oracle
        from paper_1604_05937_b200.quadrature import element_for_layout
        el = element_for_layout(fs.layout)
        self.fs = fs
        self.x = x
        self.base = fs.mesh.base
        self.prob = oracle.Problem(self.base, fs.mesh.layers,
                                   fs.layout.counts, el.tri, el.line,
                                   el.ncomp, *w.quad)
        self.coloring = oracle.greedy_color(self.base)
        self.threads = threads or oracle.max_threads()
        self.n = self.base.num_cells

    def run(self, n=None):
        t0 = time.perf_counter()
        self.prob.assemble_colored(self.x, threads=self.threads,
                                   coloring=self.coloring,
                                   n_cells=n or self.n)
        return time.perf_counter() - t0

    def calibrate(self, seconds):
        n = max(64, self.base.num_cells // 200)
        t = self.run(n)
        self.n = int(min(self.base.num_cells,
                         max(64, n * seconds / max(t, 1e-3))))

    def value(self, t):
        from paper_1604_05937_b200.perfbench import valuable_volume
        frac = self.n / self.base.num_cells
        return valuable_volume(self.fs) * frac / t / 1e9

    def describe(self, t):
        frac = self.n / self.base.num_cells
        return (f"first {self.n} of {self.base.num_cells} base cells "
                f"({100 * frac:.1f}%), all {self.fs.mesh.layers} layers, "
                f"{t:.2f} s per pass; literal quadrature, coloured schedule, "
                f"{self.threads} pthreads; bytes pro rata of the valuable "
                f"volume")


def cpu_baseline(w, fs, x, seconds):
    arm = CpuArm(w, fs, x)
    arm.calibrate(seconds)
    t = arm.run()
    return {"value": arm.value(t), "unit": UNIT, "cores": arm.threads,
            "kind": "port", "sample": arm.describe(t)}


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_1604_05937_b200 import configs
    w = configs.workload(args.config)
    fs, quad, x, _ = configs.build(w)
    arm = CpuArm(w, fs, x)
    arm.calibrate(max(1.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        arm.run()
    times = [arm.run() for _ in range(args.steps)]
    t = float(np.mean(times))
    value = arm.value(t)
    line = {"impl": "reference", "metric": METRIC, "value": value,
            "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{w.name}: {w.note}, fp64, seed {w.seed}",
                       "base_cells": fs.mesh.base.num_cells,
                       "layers": fs.mesh.layers, "layout": w.layout},
            "cpu_baseline": {"value": value, "unit": UNIT,
                             "cores": arm.threads, "kind": "port",
                             "sample": arm.describe(t)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


SHARDED = ("C5a", "C5b")


def run_sharded(args, w):
    """BASELINE config 5: the base mesh split into contiguous RCM cell
    blocks, one per GPU, ghost-column partial sums exchanged over NCCL
    (strong scaling: the total mesh is fixed)."""
    import torch
    import torch.distributed as dist
    from paper_1604_05937_b200 import configs
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.perfbench import map_bytes, valuable_volume
    from paper_1604_05937_b200.shard import ShardedMassOperator

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t_setup = time.perf_counter()
    fs, quad, x_np, _ = configs.build(w)
    m = fs.mesh
    # N > 1: the fused halo (the strip kernel adds ghost columns into the
    # owner's window over NVLink peer memory, CUDA IPC) unless
    # PM_FUSED_HALO=0 or it does not apply / cannot be set up on every
    # rank, then the NCCL send/recv exchange
    from paper_1604_05937_b200.shard import fused_halo_plan, partition
    halo = "nccl send/recv"
    want_fused = (world > 1 and os.environ.get("PM_FUSED_HALO", "1") != "0"
                  and fused_halo_plan(fs, partition(fs, world)) is not None)
    op = ShardedMassOperator(fs, rank, world, quad, fused=want_fused)
    lo, hi = op.window
    clo, chi = op.shard.coord_window
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    cwin = coords[clo:chi].clone()
    del coords
    x = torch.from_numpy(x_np[lo:hi].copy()).cuda()
    y = torch.empty_like(x)
    if want_fused:
        try:
            op.connect(y)
            halo = "fused: ghost columns REDG'd into the owner's window " \
                   "(CUDA IPC peer memory), 2 host barriers per step"
        except (RuntimeError, ValueError) as e:
            op = ShardedMassOperator(fs, rank, world, quad)
            halo = f"nccl send/recv (fused halo unavailable: {e})"
    t_setup = time.perf_counter() - t_setup
    V = valuable_volume(fs)
    n_cl = m.base.num_cells * m.layers
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        op.apply(x, cwin, y)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(args.steps):
            op.apply(x, cwin, y)
        ev[1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev[0].elapsed_time(ev[1]) / args.steps
    # the column loop alone (no exchange) on this rank
    ke = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ke[0].record(stream)
    for _ in range(args.steps):
        op.apply(x, cwin, y, exchange=False)
    ke[1].record(stream)
    torch.cuda.synchronize()
    kernel_ms = ke[0].elapsed_time(ke[1]) / args.steps
    # end to end: pinned host window in, window out
    xh = torch.from_numpy(x_np[lo:hi].copy()).pin_memory()
    yh = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        x.copy_(xh, non_blocking=True)
        op.apply(x, cwin, y)
        yh.copy_(y, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms, kernel_ms, e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kernel_ms, e2e_ms = (float(v) for v in t.tolist())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, fs, x_np, args.cpu_seconds)
    if rank == 0:
        peak, peak_src = measured_peak()
        achieved = V / world / (kernel_ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": V / (ms * 1e-3) / 1e9, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": f"{w.name}: {w.note}, fp64, seed {w.seed}",
                "base_cells": m.base.num_cells, "layers": m.layers,
                "layout": w.layout, "valuable_bytes": V,
                "map_bytes": map_bytes(fs),
                "cell_layers_per_s": n_cl / (ms * 1e-3),
                "parallelism": f"{world} contiguous RCM cell blocks",
                "halo": halo if world > 1 else "none (1 rank)",
                "halo_bytes_rank0": op.halo.bytes_per_exchange(),
                "setup_s_rank0": t_setup,
                "l2": "inputs larger than L2: no flush",
                "schedule": ("strip-REDG" if op.strips is not None else
                             "column (REDG)") + " over the rank's cell block"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(w.name),
                         "kernel_ms": kernel_ms, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": V // world},
            "cpu_baseline": cpu,
            "e2e": {"value": V / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": int(xh.numel() * 8),
                    "d2h_bytes_per_step": int(yh.numel() * 8),
                    "ms_per_step": e2e_ms},
            "gpu_launches": args.steps * (
                1 if op.fused else
                1 + 2 * len(op.halo.send) + 2 * len(op.halo.recv)),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pcie_duplex(x_host, y_host, xd):
    """The e2e path's own roofline: the same H2D + D2H bytes as one step,
    copied concurrently on two streams with no compute (best of 3, ms)."""
    import torch
    yd = torch.empty_like(xd)
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        e0.record()
        up.wait_stream(torch.cuda.current_stream())
        down.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(up):
            yd.copy_(x_host, non_blocking=True)
        with torch.cuda.stream(down):
            y_host.copy_(xd, non_blocking=True)
        torch.cuda.current_stream().wait_stream(up)
        torch.cuda.current_stream().wait_stream(down)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1604_05937_b200 import configs
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator, mass_action
    from paper_1604_05937_b200.perfbench import map_bytes, valuable_volume

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    w = configs.workload(args.config)
    fs, quad, x_np, _ = configs.build(w)
    m = fs.mesh
    coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
    op = MassOperator(fs, quad, schedule=args.schedule)
    x = torch.from_numpy(x_np).cuda()
    y = torch.empty_like(x)
    V = valuable_volume(fs)
    n_cl = m.base.num_cells * m.layers
    stream = torch.cuda.current_stream()

    # the K timed steps = K applies captured back to back in one CUDA
    # graph (no per-step host work; the same kernels as op.apply), the DG
    # stream kernels with programmatic dependent launch between steps
    warm = op.graph(x, coords, y, repeat=max(1, args.warmup))
    steps = op.graph(x, coords, y, repeat=args.steps, overlap=True)
    if args.warmup > 0:
        warm.replay()
    torch.cuda.synchronize()

    # ---- timed region: K steps, device events, max over ranks ----------
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        steps.replay()
        ev[1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    total_ms = ev[0].elapsed_time(ev[-1])
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    launches = op.launches_per_apply

    # ---- dominant kernel alone.  A step of a CG space is memset + column
    #      kernel; accumulate mode launches the same kernel without the
    #      memset.  For DG spaces the step is exactly one kernel launch.
    acc = op.share == 2
    ke = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    yk = torch.zeros_like(x)
    kstep = op.graph(x, coords, yk, accumulate=acc, repeat=args.steps)
    ke[0].record(stream)
    kstep.replay()
    ke[1].record(stream)
    torch.cuda.synchronize()
    kernel_ms = ke[0].elapsed_time(ke[1]) / args.steps
    peak, peak_src = measured_peak()
    achieved = V / (kernel_ms * 1e-3) / 1e9

    # ---- end to end through the public API, pinned host buffers --------
    x_host = torch.from_numpy(x_np).pin_memory()
    y_host = torch.empty(x_np.shape[0], dtype=torch.float64).pin_memory()
    mass_action(fs, x_host, coords, operator=op, out=y_host)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        mass_action(fs, x_host, coords, operator=op, out=y_host)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    pcie = pcie_duplex(x_host, y_host, x) if world == 1 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, fs, x_np, args.cpu_seconds)

    if rank == 0:
        sm, l2 = None, None
        from paper_1604_05937_b200 import _lib
        sm, l2 = _lib.device_info()
        line = {
            "metric": METRIC, "value": world * V / (ms * 1e-3) / 1e9,
            "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": f"{w.name}: {w.note or w.layout}, fp64, seed {w.seed}",
                "base_cells": m.base.num_cells, "layers": m.layers,
                "layout": w.layout, "ordering": w.ordering,
                "quadrature": list(w.quad),
                "valuable_bytes": V, "map_bytes": map_bytes(fs),
                "cell_layers_per_s": world * n_cl / (ms * 1e-3),
                "pct_of_measured_hbm": 100 * (V / (ms * 1e-3) / 1e9) / peak,
                "l2": (f"inputs larger than L2 ({V / 1e6:.0f} MB valuable vs "
                       f"{(l2 or 0) / 1e6:.0f} MB L2): no flush"
                       if V > (l2 or 0) else
                       "L2-resident workload (no flush; reported, not held "
                       "to the HBM target)"),
                "schedule": args.schedule, "replicas": world,
                "step": "K MassOperator.apply calls captured back to back "
                        "in one CUDA graph (DG stream: programmatic "
                        "dependent launch between steps)",
                "parallelism": f"{world} independent column-block replicas",
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(w.name),
                         "kernel_ms": kernel_ms, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": V},
            "cpu_baseline": cpu,
            "e2e": {"value": world * V / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": int(x_np.nbytes),
                    "d2h_bytes_per_step": int(x_np.nbytes),
                    "ms_per_step": e2e_ms,
                    "path": "kernels.mass_action(fs, pinned host x, "
                            "out=pinned host y)",
                    "copy_only_ms": pcie},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "sm_count": sm,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config in SHARDED:
        from paper_1604_05937_b200 import configs
        run_sharded(args, configs.workload(args.config))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

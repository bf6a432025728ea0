"""Benchmark: the extruded-mesh column loop on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5]
                    [--impl ours|reference]

A "step" is one pass of the column loop (mass action y = M x with |det J|
from the extruded coordinate field) over every part of the
workload.  Default workload "C5" = BASELINE config 5 on one GPU, the
largest single-GPU configuration: the P1 CG RHS (C5a) and the 3-vector P1
mass action (C5b) on the 2048^2 split-square RCM base mesh, 64 layers,
fp64 -- 30.57 GB of valuable bytes per step.  Other configs (C1, C2, C3,
C5a, C5b, C4-<layout>-<rcm|random>-L<layers>) are one part each.  Metric:
valuable HBM bandwidth (input + output + coordinate field,
each once) over the device time.

``--gpus N`` (N > 1, no WORLD_SIZE in the environment) re-launches itself
under ``torch.distributed.run`` with N ranks: the base mesh is split into
contiguous RCM cell blocks, one per GPU, ghost vertex columns summed over
NVLink (shard.py) -- strong scaling of the fixed C5 mesh.

``--impl reference`` times the reference's algorithm on the host cores: the
coloured column loop with the pre-integrated element matrix
(oracle/cpu_fast.c, all cores, -O3 -march=native) on meshes, maps and
coordinates built by the oracle alone (oracle/oracle_mesh.c); the product
library is never loaded on that path.  The literal-quadrature oracle is
timed beside it on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
    p.add_argument("--config", default="C5")
    p.add_argument("--schedule", default="auto")
    p.add_argument("--impl", default="ours", choices=("ours", "reference"))
    p.add_argument("--cpu-seconds", type=float, default=6.0,
                   help="literal-oracle sample budget (seconds)")
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


def respawn(args):
    """``--gpus N`` without a launcher: re-run under torch.distributed.run
    with N ranks on this node (127.0.0.1, a free port)."""
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------
# workloads (pure arithmetic: both arms build the identical config dict)
# ---------------------------------------------------------------------------

HEADLINE = {"C5": ("C5a", "C5b")}

DELTA = {"CG1xCG1": {(0, 0): 1}, "DG1xDG1": {(2, 1): 6},
         "P2xP2": {(0, 0): 1, (0, 1): 1, (1, 0): 1, (1, 1): 1},
         "VP1": {(0, 0): 3}}


def family(layout):
    """(triangle family, interval family, components) of a layout's element
    (quadrature.element_for_layout)."""
    if layout == "P2xP2":
        return "P2", "P2", 1
    if layout == "VP1":
        return "P1", "P1", 3
    h, v = layout.split("x")
    return ("P0" if h == "DG0" else "P1"), ("P0" if v == "DG0" else "P1"), 1


def parts_of(name):
    return list(HEADLINE.get(name, (name,)))


def workload(name):
    from paper_1604_05937_b200 import configs  # pure Python, no library
    return configs.workload(name)


def layout_counts(layout):
    if layout in DELTA:
        return DELTA[layout]
    h, v = layout.split("x")
    table = {("CG1", "CG1"): {(0, 0): 1}, ("CG1", "DG0"): {(0, 1): 1},
             ("CG1", "DG1"): {(0, 1): 2}, ("DG0", "CG1"): {(2, 0): 1},
             ("DG0", "DG0"): {(2, 1): 1}, ("DG0", "DG1"): {(2, 1): 2},
             ("DG1", "CG1"): {(2, 0): 3}, ("DG1", "DG0"): {(2, 1): 3},
             ("DG1", "DG1"): {(2, 1): 6}}
    return table[(h, v)]


def sizes(w):
    """(N0, N1, N2, total DoFs, valuable bytes, map bytes) of a workload on
    the split-square mesh (mesh.py:228-254; fspace.py:134-149 column sizes;
    SPEC.md:467-475)."""
    n, L = w.n, w.layers
    N = (((n + 1) ** 2), 3 * n * n + 2 * n, 2 * n * n)
    cnt = layout_counts(w.layout)
    total = sum(N[d] * (cnt.get((d, 0), 0) * (L + 1) + cnt.get((d, 1), 0) * L)
                for d in range(3))
    k = sum((3 if d < 2 else 1) * (2 * cnt.get((d, 0), 0) + cnt.get((d, 1), 0))
            for d in range(3))
    V = 8 * (2 * total + 3 * N[0] * (L + 1))
    return N[0], N[1], N[2], total, V, 4 * N[2] * (k + 18)


def bench_config(name, world):
    parts = []
    for p in parts_of(name):
        w = workload(p)
        n0, _n1, n2, total, V, mb = sizes(w)
        parts.append({"name": p, "what": w.note or w.layout, "n": w.n,
                      "base_cells": n2, "layers": w.layers,
                      "layout": w.layout, "ordering": w.ordering,
                      "jitter": w.jitter, "quadrature": list(w.quad),
                      "dofs": total, "valuable_bytes": V, "map_bytes": mb})
    V = sum(p["valuable_bytes"] for p in parts)
    return {
        "workload": (f"{name}: " + " + ".join(
            f"{p['name']} ({p['what']})" for p in parts) +
            f", fp64, seed {workload(parts[0]['name']).seed}"),
        "parts": parts, "valuable_bytes": V,
        "l2": ("inputs larger than L2 (126 MB): no flush" if V > 2 ** 28 else
               "L2-resident workload: no flush (reported, not held to the "
               "HBM target)"),
        "parallelism": ("1 GPU" if world == 1 else
                        f"{world} contiguous RCM cell blocks, ghost vertex "
                        f"columns summed over NVLink"),
        "step": "every part's mass action once (y = M x over all "
                "cell-layers)",
    }


def base_line(args, name, world):
    return {"metric": METRIC, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded split-square meshes and fields, "
                    "SURVEY 8d)",
            "config": bench_config(name, world)}


# ---------------------------------------------------------------------------
# CPU arm (oracle only)
# ---------------------------------------------------------------------------

class CpuParts:
    """The CPU baseline over every part: oracle/cpu_fast.c with the oracle's
    own meshes (``bases[n, ordering, jitter]`` may pass product meshes to
    save the setup; the arrays are identical, tests/test_host.py)."""

    def __init__(self, name, fields=None, bases=None):
        import oracle
        from oracle import fast
        self.parts = []
        for p in parts_of(name):
            w = workload(p)
            key = (w.n, w.ordering, w.jitter, w.seed)
            if bases and key in bases:
                base, rng = bases[key]
            else:
                base, rng = oracle.base_mesh(w.n, w.ordering, w.jitter, w.seed)
            tri, line, nc = family(w.layout)
            arm = fast.FastMass(base, w.layers, layout_counts(w.layout), tri,
                                line, nc, *w.quad)
            if fields is not None and p in fields:
                x = fields[p]
            elif w.values == "u01":
                x = rng.random(arm.total)
            else:
                x = rng.uniform(-1.0, 1.0, arm.total)
            V = sizes(w)[4]
            self.parts.append((p, w, base, arm, x, V))
        self.threads = self.parts[0][3].threads
        self.flags = self.parts[0][3].flags

    def step(self):
        t0 = time.perf_counter()
        for _p, _w, _b, arm, x, _V in self.parts:
            arm.apply(x)
        return time.perf_counter() - t0

    @property
    def V(self):
        return sum(p[5] for p in self.parts)

    def literal_sample(self, seconds):
        """The literal-quadrature oracle (prismesh_oracle.c, coloured
        pthreads) on the first cells of each part, bytes pro rata."""
        import oracle
        tot_t, tot_v, desc = 0.0, 0.0, []
        for p, w, base, arm, x, V in self.parts:
            tri, line, nc = family(w.layout)
            prob = oracle.Problem(base, w.layers, layout_counts(w.layout),
                                  tri, line, nc, *w.quad)
            col = oracle.greedy_color(base)
            n = max(64, base.num_cells // 400)
            t0 = time.perf_counter()
            prob.assemble_colored(x, coloring=col, n_cells=n)
            t = max(time.perf_counter() - t0, 1e-4)
            n = int(min(base.num_cells,
                        n * seconds / len(self.parts) / t))
            t0 = time.perf_counter()
            prob.assemble_colored(x, coloring=col, n_cells=n)
            t = time.perf_counter() - t0
            tot_t += t
            tot_v += V * n / base.num_cells
            desc.append(f"{p}: first {n} of {base.num_cells} cells")
        return tot_v / tot_t / 1e9, "; ".join(desc)

    def describe(self):
        return (f"full workload ({' + '.join(p[0] for p in self.parts)}), "
                f"oracle/cpu_fast.c: column loop with the pre-integrated "
                f"element matrix, {self.threads} pthreads "
                f"({'; '.join(sorted(set(p[3].schedule for p in self.parts)))}"
                f"), gcc {self.flags}")


def cpu_record(arm, t_min, times):
    from oracle import fast
    phys, logical, model = fast.cpu_info()
    return {"value": arm.V / t_min / 1e9, "unit": UNIT,
            "cores": arm.threads, "cores_physical": phys,
            "cores_logical": logical, "cpu_model": model, "kind": "port",
            "sample": arm.describe(), "ms_per_step_min": 1e3 * t_min,
            "ms_per_step_mean": 1e3 * float(np.mean(times)),
            "spread": float((max(times) - min(times)) / min(times))}


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    arm = CpuParts(args.config)
    for _ in range(args.warmup):
        arm.step()
    times = [arm.step() for _ in range(args.steps)]
    t = min(times)                       # min of runs
    cpu = cpu_record(arm, t, times)
    lit_v, lit_s = arm.literal_sample(args.cpu_seconds)
    line = base_line(args, args.config, world)
    line.update({
        "impl": "reference", "value": cpu["value"], "ms_per_step": 1e3 * t,
        "cpu_baseline": cpu,
        "literal_oracle": {"value": lit_v, "unit": UNIT, "sample": lit_s,
                           "kind": "port (literal quadrature)"},
        "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def pcie_duplex(nbytes_up, nbytes_down):
    """The e2e path's own roofline: the step's H2D + D2H bytes copied
    concurrently on two streams with no compute (best of 3, ms)."""
    import torch
    n_up, n_dn = max(1, nbytes_up // 8), max(1, nbytes_down // 8)
    hu = torch.empty(n_up, dtype=torch.float64).pin_memory()
    hd = torch.empty(n_dn, dtype=torch.float64).pin_memory()
    du = torch.empty(n_up, dtype=torch.float64, device="cuda")
    dd = torch.empty(n_dn, dtype=torch.float64, device="cuda")
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        e0.record()
        up.wait_stream(torch.cuda.current_stream())
        down.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(up):
            du.copy_(hu, non_blocking=True)
        with torch.cuda.stream(down):
            hd.copy_(dd, non_blocking=True)
        torch.cuda.current_stream().wait_stream(up)
        torch.cuda.current_stream().wait_stream(down)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def time_graph(g, reps=1):
    import torch
    stream = torch.cuda.current_stream()
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def run_ours(args):
    import torch
    from paper_1604_05937_b200 import configs, _lib
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.kernels import MassOperator, mass_action

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    name = args.config
    t_setup = time.perf_counter()
    parts = []
    coords_cache = {}
    for p in parts_of(name):
        w = configs.workload(p)
        fs, quad, x_np, _ = configs.build(w)
        m = fs.mesh
        key = (w.n, w.ordering, w.jitter, w.seed, w.layers)
        if key not in coords_cache:
            coords_cache[key] = extrude_coordinates(m.base.coords, m.layers,
                                                    m.layer_height)
        op = MassOperator(fs, quad, schedule=args.schedule)
        x = torch.from_numpy(x_np).cuda()
        y = torch.empty_like(x)
        op.apply(x, coords_cache[key], y)          # plans, attributes ready
        parts.append({"name": p, "w": w, "fs": fs, "op": op, "x": x, "y": y,
                      "x_np": x_np, "coords": coords_cache[key],
                      "V": sizes(w)[4]})
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    V = sum(q["V"] for q in parts)
    stream = torch.cuda.current_stream()

    def capture(sel, repeat, accumulate=False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(repeat):
                for q in sel:
                    q["op"].apply(q["x"], q["coords"], q["y"],
                                  accumulate=accumulate,
                                  schedule=args.schedule)
        torch.cuda.synchronize()
        return g

    # ---- timed region: K steps (every part once per step) in one graph
    warm = capture(parts, max(1, args.warmup))
    steps = capture(parts, args.steps)
    if args.warmup > 0:
        warm.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev[0].record(stream)
        steps.replay()
        ev[1].record(stream)
        torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / args.steps
    del warm, steps

    # ---- each part's kernel alone (roofline): K applies in one graph,
    # accumulating (no output memset: the REDG schedules zero y first, a
    # separate memset launch that is not the kernel)
    peak, peak_src = measured_peak()
    kernels = []
    for q in parts:
        redg = q["op"].last_schedule in ("stripred", "striptma", "pstrip",
                                          "atomic")
        g = capture([q], args.steps, accumulate=redg)
        kms = time_graph(g) / args.steps
        zero_ms = None
        if redg:
            gz = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gz):
                for _ in range(args.steps):
                    q["y"].zero_()
            zero_ms = time_graph(gz) / args.steps
            del gz
        kernels.append({"part": q["name"], "kernel_ms": kms,
                        "algorithmic_bytes_per_launch": q["V"],
                        "achieved": q["V"] / (kms * 1e-3) / 1e9,
                        "frac": q["V"] / (kms * 1e-3) / 1e9 / peak,
                        "schedule": q["op"].last_schedule,
                        "output_zeroing_ms": zero_ms,
                        "traffic": ncu_traffic(q["name"])})
        del g
    dom = max(kernels, key=lambda k: k["algorithmic_bytes_per_launch"])

    # the device result of every part (the roofline graphs accumulated)
    for q in parts:
        q["op"].apply(q["x"], q["coords"], q["y"], schedule=args.schedule)
    torch.cuda.synchronize()

    # ---- end to end through the public API, pinned host buffers
    for q in parts:
        q["xh"] = torch.from_numpy(q["x_np"]).pin_memory()
        q["yh"] = torch.empty(q["x_np"].shape[0],
                              dtype=torch.float64).pin_memory()
        mass_action(q["fs"], q["xh"], q["coords"], operator=q["op"],
                    out=q["yh"])
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        for q in parts:
            mass_action(q["fs"], q["xh"], q["coords"], operator=q["op"],
                        out=q["yh"])
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    nbytes = sum(int(q["x_np"].nbytes) for q in parts)
    copy_ms = pcie_duplex(nbytes, nbytes)
    # the e2e result matches the device result (REDG summation order may
    # differ in the last bits)
    e2e_ok = all(float((q["yh"] - q["y"].cpu()).abs().max()) <=
                 1e-12 * float(q["yh"].abs().max()) for q in parts)

    cpu = None
    if not args.no_cpu_baseline:
        bases = {(q["w"].n, q["w"].ordering, q["w"].jitter, q["w"].seed):
                 configs.base_mesh(q["w"].n, q["w"].ordering, q["w"].jitter,
                                   q["w"].seed) for q in parts}
        for q in parts:     # free device memory before the host arm
            del q["xh"], q["yh"]
        arm = CpuParts(name, fields={q["name"]: q["x_np"] for q in parts},
                       bases=bases)
        arm.step()
        times = [arm.step() for _ in range(3)]
        cpu = cpu_record(arm, min(times), times)

    sm, l2 = _lib.device_info()
    line = base_line(args, name, world)
    line.update({
        "value": V / (ms * 1e-3) / 1e9, "ms_per_step": ms,
        "cell_layers_per_s": sum(q["w"].layers * sizes(q["w"])[2]
                                 for q in parts) / (ms * 1e-3),
        "pct_of_measured_hbm": 100 * V / (ms * 1e-3) / 1e9 / peak,
        "setup_s": t_setup,
        "roofline": {"bound": "hbm", "achieved": dom["achieved"],
                     "peak": peak, "unit": "GB/s", "frac": dom["frac"],
                     "traffic": dom["traffic"], "kernel": dom["part"],
                     "kernel_ms": dom["kernel_ms"], "peak_source": peak_src,
                     "algorithmic_bytes_per_launch":
                         dom["algorithmic_bytes_per_launch"],
                     "kernels": kernels},
        "cpu_baseline": cpu,
        "e2e": {"value": V / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "ms_per_step": e2e_ms, "copy_only_ms": copy_ms,
                "matches_device_result": bool(e2e_ok),
                "path": "kernels.mass_action(fs, pinned host x, "
                        "out=pinned host y) per part"},
        "gpu_launches": args.steps * sum(q["op"].launches_per_apply
                                         for q in parts),
        "clocks": clk.summary(),
        "sm_count": sm,
    })
    print(json.dumps(line), flush=True)


def run_sharded(args):
    """N ranks: every part's base mesh split into contiguous RCM cell blocks,
    ghost vertex columns summed over NVLink (fused peer REDs, or NCCL
    send/recv), strong scaling of the fixed workload."""
    import torch
    import torch.distributed as dist
    from paper_1604_05937_b200 import configs
    from paper_1604_05937_b200.extrusion import extrude_coordinates
    from paper_1604_05937_b200.shard import (ShardedMassOperator,
                                             fused_halo_plan, partition)

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.config
    t_setup = time.perf_counter()
    parts = []
    for p in parts_of(name):
        w = configs.workload(p)
        fs, quad, x_np, _ = configs.build(w)
        m = fs.mesh
        want = (os.environ.get("PM_FUSED_HALO", "1") != "0" and
                fused_halo_plan(fs, partition(fs, world)) is not None)
        op = ShardedMassOperator(fs, rank, world, quad, fused=want)
        lo, hi = op.window
        clo, chi = op.shard.coord_window
        coords = extrude_coordinates(m.base.coords, m.layers, m.layer_height)
        cwin = coords[clo:chi].clone()
        del coords
        x = torch.from_numpy(x_np[lo:hi].copy()).cuda()
        y = torch.empty_like(x)
        halo = "nccl send/recv"
        if want:
            try:
                op.connect(y)
                halo = "fused: ghost columns added into the owner's window " \
                       "by the kernel (CUDA IPC peer memory)"
            except (RuntimeError, ValueError) as e:
                op = ShardedMassOperator(fs, rank, world, quad)
                halo = f"nccl send/recv (fused halo unavailable: {e})"
        parts.append({"name": p, "w": w, "op": op, "x": x, "y": y,
                      "cw": cwin, "V": sizes(w)[4], "halo": halo,
                      "x_np": x_np[lo:hi]})
    t_setup = time.perf_counter() - t_setup
    V = sum(q["V"] for q in parts)
    stream = torch.cuda.current_stream()

    def step(exchange=True):
        for q in parts:
            # the kernel alone (roofline): no exchange, no output memset
            q["op"].apply(q["x"], q["cw"], q["y"], exchange=exchange,
                          accumulate=not exchange)

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(args.steps):
            step()
        ev[1].record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = ev[0].elapsed_time(ev[1]) / args.steps
    ke = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    dist.barrier()
    ke[0].record(stream)
    for _ in range(args.steps):
        step(exchange=False)
    ke[1].record(stream)
    torch.cuda.synchronize()
    kms = ke[0].elapsed_time(ke[1]) / args.steps
    for q in parts:
        q["xh"] = torch.from_numpy(np.ascontiguousarray(q["x_np"])
                                   ).pin_memory()
        q["yh"] = torch.empty(q["xh"].shape[0],
                              dtype=torch.float64).pin_memory()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        for q in parts:
            q["x"].copy_(q["xh"], non_blocking=True)
            q["op"].apply(q["x"], q["cw"], q["y"])
            q["yh"].copy_(q["y"], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms, kms, e2e_ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)    # max over ranks
    ms, kms, e2e_ms = (float(v) for v in t.tolist())
    if rank == 0:
        peak, peak_src = measured_peak()
        nb = sum(int(q["xh"].numel()) * 8 for q in parts)
        line = base_line(args, name, world)
        line["config"]["halo"] = {q["name"]: q["halo"] for q in parts}
        line["config"]["halo_bytes_rank0"] = {
            q["name"]: q["op"].halo.bytes_per_exchange() for q in parts}
        line.update({
            "value": V / (ms * 1e-3) / 1e9, "ms_per_step": ms,
            "setup_s_rank0": t_setup,
            "roofline": {"bound": "hbm",
                         "achieved": V / world / (kms * 1e-3) / 1e9,
                         "peak": peak, "unit": "GB/s",
                         "frac": V / world / (kms * 1e-3) / 1e9 / peak,
                         "traffic": None, "kernel_ms": kms,
                         "kernel": "the rank's column loop (all parts, no "
                                   "exchange, no output memset), max over "
                                   "ranks",
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": V // world},
            "cpu_baseline": None,
            "e2e": {"value": V / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                    "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
                    "ms_per_step": e2e_ms,
                    "path": "rank-window host copies + sharded apply"},
            "gpu_launches": args.steps * sum(
                1 if q["op"].fused else
                1 + 2 * len(q["op"].halo.send) + 2 * len(q["op"].halo.recv)
                for q in parts),
            "clocks": clk.summary(),
        })
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        respawn(args)                  # exits with the launcher's status
    if world and args.gpus != world:
        sys.exit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    elif max(world, 1) > 1:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

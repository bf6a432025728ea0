"""Measurement formulas of the SPEC ``perfbench`` module.

``valuable_volume`` is the byte count every bandwidth number in this repo
uses: input + output + coordinate
field, each counted once.  The CPU peak model (``balance_factor``,
``vector_factor``, ``peak_throughput``) is kept for the
reference's formula tests; the B200 roofline denominator is the measured
HBM bandwidth instead.
"""
from __future__ import annotations


def valuable_volume(fs, coord_space=None) -> int:
    """``8 * (2*total_dofs(fs) + total_dofs(coords))`` bytes."""
    base = fs.mesh.base
    coords = (coord_space.total_dofs if coord_space is not None
              else 3 * base.num_vertices * (fs.mesh.layers + 1))
    return 8 * (2 * fs.total_dofs + coords)


def map_bytes(fs) -> int:
    """Explicit-map bytes (excluded from the valuable volume):
    the field map plus the 18-slot coordinate map, int32."""
    n = fs.mesh.base.num_cells
    return 4 * n * (fs.num_slots + 18)


def balance_factor(adds: int, muls: int, fmas: int = 0,
                   arch: str = "no-fma") -> float:
    if adds < 0 or muls < 0 or fmas < 0:
        raise ValueError("counts must be >= 0")
    if adds == 0 and muls == 0 and fmas == 0:
        raise ValueError("all-zero operation counts")
    lo, hi = min(adds, muls), max(adds, muls)
    if arch == "no-fma":
        return 1.0 + lo / hi
    if arch == "fma":
        k = fmas / 2
        return 1.0 + (lo + k) / (hi + k)
    raise ValueError(f"unknown arch {arch!r}")


def vector_factor(vector_flops: float, total_flops: float) -> float:
    if total_flops <= 0 or not 0 <= vector_flops <= total_flops:
        raise ValueError("need 0 <= vector_flops <= total_flops, total > 0")
    return 1.0 + 3.0 * vector_flops / total_flops


def peak_throughput(base_rate: float, f_b: float, f_v: float) -> float:
    return base_rate * f_b * f_v


CSV_HEADER = ("layout,ordering,layers,base_cells,threads,runtime_s,"
              "valuable_bytes,valuable_gbs,flops,gflops,f_b,f_v,peak_gflops,"
              "peak_fraction,stream_gbs")

"""Shared fixtures.  ``-m gpu`` tests need a B200; everything else is CPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


class GoldenMesh:
    """BaseMesh-like view of a golden mesh (reference-produced arrays)."""

    def __init__(self, g, name):
        p = f"mesh/{name}/"
        self.cell_vertices = g[p + "cell_vertices"]
        self.coords = g[p + "coords"]
        self.cell_edges = g[p + "cell_edges"]
        self.edge_vertices = g[p + "edge_vertices"]
        self._vertex_cells = (g[p + "vertex_cells_off"], g[p + "vertex_cells"])

    @property
    def num_vertices(self):
        return self.coords.shape[0]

    @property
    def num_edges(self):
        return self.edge_vertices.shape[0]

    @property
    def num_cells(self):
        return self.cell_vertices.shape[0]

    def entity_count(self, d):
        return (self.num_vertices, self.num_edges, self.num_cells)[d]


@pytest.fixture(scope="session")
def gmesh(golden):
    return lambda name: GoldenMesh(golden, name)


LAYOUT_COUNTS = {
    "CG1xCG1": {(0, 0): 1}, "CG1xDG0": {(0, 1): 1}, "CG1xDG1": {(0, 1): 2},
    "DG0xCG1": {(2, 0): 1}, "DG0xDG0": {(2, 1): 1}, "DG0xDG1": {(2, 1): 2},
    "DG1xCG1": {(2, 0): 3}, "DG1xDG0": {(2, 1): 3}, "DG1xDG1": {(2, 1): 6},
    "P2xP2": {(0, 0): 1, (0, 1): 1, (1, 0): 1, (1, 1): 1},
    "VP1": {(0, 0): 3}, "coords": {(0, 0): 3},
}

FAMILIES = {"CG1": "P1", "DG1": "P1", "DG0": "P0"}


def families(name):
    if name == "P2xP2":
        return "P2", "P2", 1
    if name in ("VP1", "coords"):
        return "P1", "P1", 3
    h, v = name.split("x")
    return FAMILIES[h], FAMILIES[v], 1


def quad_degrees(name):
    tri, line, _ = families(name)
    d = {"P0": 0, "P1": 1, "P2": 2}
    return max(2, 2 * d[tri]), max(2, 2 * d[line])

"""The SPEC cli / perfbench harness and the verification
module (reference verification.py)."""
import csv
import io
import math

import numpy as np
import pytest

from paper_1604_05937_b200 import cli, verification
from paper_1604_05937_b200.extrusion import ExtrudedMesh
from paper_1604_05937_b200.fspace import (all_builtin_layouts, builtin_layout,
                                          number_dofs)
from paper_1604_05937_b200.mesh import generate_unit_square_mesh
from paper_1604_05937_b200.perfbench import CSV_HEADER


def test_base_n_matches_spec_example():
    # SPEC run_experiment: target 15e6 cells, λ=100 -> n = 274, within 1 %
    n = cli.base_n(15_000_000, 100)
    assert n == 274
    assert abs(2 * n * n * 100 - 15e6) / 15e6 < 0.01
    with pytest.raises(ValueError):
        cli.base_n(1, 100)


def test_read_hw(tmp_path):
    p = tmp_path / "hw.cfg"
    p.write_text("sm_count=148  # B200\nclock_ghz = 1.9\n\nstream_gbs_override=7000\n")
    hw = cli.read_hw(str(p))
    assert hw == {"sm_count": 148.0, "clock_ghz": 1.9,
                  "stream_gbs_override": 7000.0}
    assert cli.read_hw(None) == {}


def test_verify_host_suite_passes():
    lines = []
    assert verification.run_oracle_suite(report=lines.append, device=False)
    assert lines == ["27/27 layout-mesh-layers oracle checks passed (host)"]


def _host_coords(mesh):
    # extrusion.py:66-85: (x_i, y_i, l*h) at 3*(i*(λ+1)+l)+comp
    lam, h = mesh.layers, mesh.layer_height
    xy = np.asarray(mesh.base.coords)
    c = np.empty((xy.shape[0], lam + 1, 3))
    c[:, :, 0] = xy[:, None, 0]
    c[:, :, 1] = xy[:, None, 1]
    c[:, :, 2] = np.arange(lam + 1) * h
    return c.ravel()


@pytest.mark.parametrize("layout", all_builtin_layouts(),
                         ids=lambda l: l.name)
def test_literal_numbering_matches_closed_form(layout):
    mesh = ExtrudedMesh(generate_unit_square_mesh(3), 3)
    assert verification.check_space(mesh, layout) == []


def test_check_space_detects_a_broken_offset(monkeypatch):
    mesh = ExtrudedMesh(generate_unit_square_mesh(2), 2)
    layout = builtin_layout("CG1", "CG1")
    real = verification.closed_form_maps

    def broken(fs):
        b, o = real(fs)
        o = o.copy()
        o[0] += 1
        return b, o
    monkeypatch.setattr(verification, "closed_form_maps", broken)
    fails = verification.check_space(mesh, layout)
    assert any("offset addressing differs" in f for f in fails)


def test_dense_assembler_conserves_integral():
    # f = 1 on the unit cube: sum of the residual = |Ω| = 1
    from paper_1604_05937_b200.kernels import default_quadrature
    from paper_1604_05937_b200.quadrature import (element_for_layout,
                                                  reference_mass_matrix)
    mesh = ExtrudedMesh(generate_unit_square_mesh(3), 4)
    for layout in all_builtin_layouts():
        fs = number_dofs(mesh, layout)
        el = element_for_layout(layout)
        mref = reference_mass_matrix(el, default_quadrature(el))
        coords = _host_coords(mesh)
        y = verification.dense_mass_action(fs, np.ones(fs.total_dofs),
                                           coords, mref)
        assert math.isclose(y.sum(), 1.0, rel_tol=1e-12), layout.name


def test_csv_header_matches_record_keys():
    assert CSV_HEADER.split(",") == [
        "layout", "ordering", "layers", "base_cells", "threads", "runtime_s",
        "valuable_bytes", "valuable_gbs", "flops", "gflops", "f_b", "f_v",
        "peak_gflops", "peak_fraction", "stream_gbs"]


@pytest.mark.gpu
def test_cli_verify_on_device(capsys):
    assert cli.main(["verify"]) == 0
    assert "27/27" in capsys.readouterr().out


@pytest.mark.gpu
def test_cli_stream_positive(capsys):
    assert cli.main(["stream", "--repeats", "3"]) == 0
    out = capsys.readouterr().out.strip()
    assert out.startswith("stream_gbs=")
    assert 500.0 < float(out.split("=")[1]) < 20000.0


@pytest.mark.gpu
def test_cli_bench_cross_product(tmp_path):
    out = tmp_path / "r.csv"
    rc = cli.main(["bench", "--layers", "1,10", "--horiz", "CG1", "--vert",
                   "CG1", "--ordering", "rcm,random", "--generate", "16",
                   "--repeats", "2", "--out", str(out)])
    assert rc == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert len(rows) == 4                      # SPEC: cross product
    for r in rows:
        t = float(r["runtime_s"])
        assert t > 0
        # derived columns recompute from the primitive ones
        assert math.isclose(float(r["valuable_gbs"]),
                            int(r["valuable_bytes"]) / t / 1e9, rel_tol=1e-5)
        assert math.isclose(float(r["gflops"]) * t, int(r["flops"]) / 1e9,
                            rel_tol=1e-5)
        assert 1.0 <= float(r["f_b"]) <= 2.0
        assert float(r["peak_fraction"]) > 0
        assert float(r["stream_gbs"]) > 0

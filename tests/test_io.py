"""Solution dump (the SPEC examples for dump_solution):
row counts, constant state, byte-identical dump -> load -> dump round trip,
adaptive mesh order, error with the path on I/O failure."""
import numpy as np
import pytest

from paper_1806_07984_b200 import configs, mesh
from paper_1806_07984_b200.errors import ConfigError
from paper_1806_07984_b200.io import dump_solution, load_solution


def test_row_count_9_cells_p1(tmp_path):
    m = mesh.CartesianMesh(3, 2, True)
    Q = np.zeros((9, 1, 2, 2))
    assert dump_solution(m, Q, tmp_path / "a.csv") == 36
    lines = (tmp_path / "a.csv").read_text().splitlines()
    assert lines[0] == "level,ix,iy,node_x,node_y,component,value"
    assert len(lines) == 37


def test_constant_state(tmp_path):
    m = mesh.CartesianMesh(4, 2, False)
    Q = np.full((16, 4, 3, 3), 2.5)
    dump_solution(m, Q, tmp_path / "c.csv")
    vals = [float(l.split(",")[-1]) for l in (tmp_path / "c.csv").read_text().splitlines()[1:]]
    assert set(vals) == {2.5}


@pytest.mark.parametrize("dim", [2, 3])
def test_round_trip_byte_identical(tmp_path, dim):
    m = mesh.CartesianMesh(3, dim, True)
    rng = np.random.default_rng(7)
    Q = rng.standard_normal((m.ncells, dim + 2) + (3,) * dim)
    dump_solution(m, Q, tmp_path / "1.csv")
    R = load_solution(m, tmp_path / "1.csv")
    assert np.array_equal(R, Q)
    dump_solution(m, R, tmp_path / "2.csv")
    assert (tmp_path / "1.csv").read_bytes() == (tmp_path / "2.csv").read_bytes()


def test_adaptive_mesh_node_coordinates(tmp_path):
    cfg = configs.CONFIGS["cfg5"].with_(cells=9)
    am = mesh.AdaptiveMesh(configs.amr_cells(cfg), 2, True)
    Q = configs.initial_dg_amr(cfg, am.cells)
    rows = dump_solution(am, Q, tmp_path / "amr.csv")
    assert rows == am.ncells * 4 * 16
    lines = (tmp_path / "amr.csv").read_text().splitlines()[1:]
    # first row: first cell in storage (depth-first) order, node (0, 0), component 0
    lvl, ix, iy, x, y, k, v = lines[0].split(",")
    l0, i0 = am.cells[0]
    assert (int(lvl), int(ix), int(iy), int(k)) == (l0, i0[0], i0[1], 0)
    xi0 = configs.gl_nodes(4)[0]
    assert np.isclose(float(x), (i0[0] + xi0) / 3.0 ** l0) and float(v) == Q[0, 0, 0, 0]
    assert np.array_equal(load_solution(am, tmp_path / "amr.csv"), Q)


def test_errors(tmp_path):
    m = mesh.CartesianMesh(2, 2, True)
    with pytest.raises(ConfigError):
        dump_solution(m, np.zeros((3, 1, 2, 2)), tmp_path / "x.csv")
    with pytest.raises(OSError, match="nope"):
        dump_solution(m, np.zeros((4, 1, 2, 2)), tmp_path / "nope" / "x.csv")

"""The command line (heatbem/cli.py:199-226 surface) on the device backend:
argument handling on the CPU, tiny solve / convergence runs on the GPU
(the reference's own test_cli.py cases: same flags, files and checks)."""
import json

import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.cli import main
from paper_2102_09811_b200.study import CSV_HEADER

TINY = ["--subdivisions", "1", "--timesteps", "2", "--interior-points", "20"]


def test_mesh_gen_round_trip(tmp_path):
    out = tmp_path / "cube.mesh"
    assert main(["mesh-gen", "--refine", "1", "--out", str(out)]) == 0
    mesh = hb.load_mesh(out)
    assert mesh.n_triangles == 12 * 8 ** 2


def test_argument_errors(tmp_path):
    with pytest.raises(SystemExit):
        main(["mesh-gen", "--refine", "-1", "--out", str(tmp_path / "m")])
    with pytest.raises(SystemExit):
        main(["solve", "--mesh", str(tmp_path / "x.mesh"), "--out", str(tmp_path)])
    with pytest.raises(SystemExit):
        main(["convergence", "--levels", "1", "--out", str(tmp_path)])
    with pytest.raises(SystemExit):
        main(["solve", "--source-point", "1,2", "--out", str(tmp_path)] + TINY)


@pytest.mark.gpu
def test_solve_writes_outputs(tmp_path):
    assert main(["solve", "--problem", "dirichlet", "--refine", "0", "--out", str(tmp_path)] + TINY) == 0
    assert np.load(tmp_path / "solution.npy").shape == (2, 12)
    report = json.loads((tmp_path / "report.json").read_text())
    assert report["converged"] and report["E_t"] == 2 and report["E_x"] == 12


@pytest.mark.gpu
def test_convergence_table_and_reproducibility(tmp_path, capsys):
    a, b = tmp_path / "a", tmp_path / "b"
    assert main(["convergence", "--levels", "2", "--out", str(a)] + TINY) == 0
    printed = capsys.readouterr().out
    table = (a / "convergence.csv").read_text()
    assert table in printed
    lines = table.strip().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 3
    first, second = lines[1].split(","), lines[2].split(",")
    assert first[:2] == ["2", "12"] and first[3] == first[5] == first[7] == ""
    assert second[:2] == ["4", "48"] and all(second[i] != "" for i in (3, 5, 7))
    assert len(json.loads((a / "report.json").read_text())["levels"]) == 2
    assert main(["convergence", "--levels", "2", "--out", str(b)] + TINY) == 0
    assert (b / "convergence.csv").read_bytes() == table.encode()

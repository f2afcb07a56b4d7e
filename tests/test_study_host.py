"""Host logic of the boundary-data / study path: the
device-datum mapping, the datum's numpy evaluation against the reference's
data functions, the convergence-table format against the reference's own
writer (tests/golden/study.npz, oracle/gen_study.py), and the C-ABI's
argument checks of the data entry points (no GPU needed)."""
import ctypes

import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import _native
from paper_2102_09811_b200.field import device_datum
from _hb_util import golden


def test_device_datum_mapping():
    ms = hb.ManufacturedSolution(np.array([0.0, 0.0, 1.5]), 0.5)
    assert device_datum(ms.dirichlet_trace) == hb.HeatKernelDatum((0, 0, 1.5), 0.5, 0.0, "value")
    assert device_datum(ms.value).kind == "value"
    assert device_datum(ms.neumann_trace).kind == "normal_derivative"
    assert device_datum(lambda x, t, n=None: 0.0) is None
    g = hb.HeatKernelDatum((1.5, 1.5, 1.5), 1.0, 0.1)
    assert device_datum(g) is g
    with pytest.raises(ValueError):
        hb.HeatKernelDatum((0, 0, 0), 1.0, kind="gradient")


def test_datum_numpy_values_match_manufactured_traces():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (50, 3))
    n = rng.standard_normal((50, 3))
    ms = hb.ManufacturedSolution(np.array([0.2, -0.1, 1.5]), 0.7)
    gv = hb.HeatKernelDatum(tuple(ms.source_point), 0.7)
    gn = hb.HeatKernelDatum(tuple(ms.source_point), 0.7, kind="normal_derivative")
    for t in (0.0, 0.3, 1.0):
        assert np.array_equal(gv(x, t), ms.dirichlet_trace(x, t))
        assert np.array_equal(gn(x, t, n), ms.neumann_trace(x, t, n))
    shifted = hb.HeatKernelDatum((1.5, 1.5, 1.5), 1.0, 0.1)
    assert np.array_equal(shifted(x, 0.25), hb.fundamental(x - 1.5, 0.35, 1.0))


def test_results_to_csv_matches_reference_format():
    g = golden("study")
    rows = []
    for tag in ("dir0", "dir1"):
        rows.append(hb.LevelResult(level=0, E_t=int(g[f"{tag}_E_t"]), E_x=int(g[f"{tag}_E_x"]),
                                   err_computed=float(g[f"{tag}_err_computed"]),
                                   err_projected=float(g[f"{tag}_err_projected"]),
                                   err_repr=float(g[f"{tag}_err_repr"]), iterations=int(g[f"{tag}_iterations"]),
                                   residual=float(g[f"{tag}_residual"]), converged=True))
    assert hb.results_to_csv(rows) == str(g["csv_dir"])
    rep = hb.results_to_report(hb.StudyConfig(), rows)
    assert '"problem": "dirichlet"' in rep and '"levels"' in rep


def test_study_config_validation():
    with pytest.raises(ValueError):
        hb.StudyConfig(problem="robin")
    with pytest.raises(ValueError):
        hb.run_study(hb.StudyConfig(), 0)


def test_data_entry_points_reject_bad_arguments_without_gpu():
    L = _native.load()
    d, g = _native.DataDesc(), _native.HeatDatum()
    assert L.hb_project_workspace(ctypes.byref(d), 1, 4) == 0
    assert L.hb_project_data(ctypes.byref(d), ctypes.byref(g), 1, 4, 0.25, None, None, 0, 1e-15, 100, None,
                             None) == -1
    assert b"hb_project_data" in L.hb_last_error()
    assert L.hb_error_sigma(ctypes.byref(d), ctypes.byref(g), 4, 0.25, None, 0, None, None, 0, None) == -1
    assert L.hb_p1_mass_solve(ctypes.byref(d), 4, None, None, None, 0, 1e-15, 10, None) == -1


def test_data_desc_layout_matches_c(tmp_path):
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = tmp_path / "sz.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "heatbem_b200.h"\n'
                    'int main(void){printf("%zu %zu %zu %zu\\n", sizeof(hb_data_desc), offsetof(hb_data_desc, tw),'
                    ' sizeof(hb_heat_datum), offsetof(hb_heat_datum, time_shift));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(root, "include"), str(prog), "-o", str(exe)])
    a, b, c, e = map(int, subprocess.check_output([str(exe)]).split())
    assert a == ctypes.sizeof(_native.DataDesc) and b == _native.DataDesc.tw.offset
    assert c == ctypes.sizeof(_native.HeatDatum) and e == _native.HeatDatum.time_shift.offset

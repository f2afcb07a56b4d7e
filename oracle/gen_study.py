"""Generate tests/golden/study.npz from the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python oracle/gen_study.py

Imports the reference package ``heatbem`` read-only and stores what pins the
boundary-data and study path:

* projections ``project_to_space`` (heatbem/field.py:84-119) of the manufactured
  traces (value -> X10 and X00, normal derivative -> X00 and X10) on the cube
  n=2 (48 triangles, E_t = 4, alpha = 0.5, source (0, 0, 1.5)), and the
  config-2 datum G(x - (1.5,1.5,1.5), t + 0.1) on the unit cube L3, N = 32;
* ``relative_error_sigma`` (field.py:193-215) of seeded p0 / p1 coefficient
  arrays against both traces;
* ``run_level`` (heatbem/study.py:73-170) levels 0 and 1 of the default
  Dirichlet study and level 0 of the Neumann study: the errors, iterations and
  the level-0 solutions.

Nothing on the GPU box runs this file; /root/reference does not exist there.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = os.environ.get("HEATBEM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
import heatbem as H  # noqa: E402
from heatbem import study as HS  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "study.npz")


def main():
    out = {}
    m = H.generate_cube_surface(2)
    tg = H.TimeGrid(1.0, 4)
    ms = H.ManufacturedSolution(np.array([0.0, 0.0, 1.5]), 0.5)
    for name, fn in (("value", ms.dirichlet_trace), ("nderiv", ms.neumann_trace)):
        for space in ("X00", "X10"):
            out[f"proj_{name}_{space}"] = H.project_to_space(fn, m, tg, space)
    rng = np.random.default_rng(11)
    c0 = rng.uniform(-1, 1, (4, m.n_triangles)) * 0.01
    c1 = rng.uniform(-1, 1, (4, m.n_vertices)) * 0.01
    out["err_c0"], out["err_c1"] = c0, c1
    for name, fn in (("value", ms.dirichlet_trace), ("nderiv", ms.neumann_trace)):
        out[f"err_{name}_p0"] = H.relative_error_sigma(c0, fn, m, tg)
        out[f"err_{name}_p1"] = H.relative_error_sigma(c1, fn, m, tg)
        out[f"err_{name}_proj"] = H.relative_error_sigma(out[f"proj_{name}_X10"], fn, m, tg)

    # config-2 datum
    m3 = H.generate_cube_surface(1, 0.5)
    m3 = H.SurfaceMesh(m3.vertices + 0.5, m3.triangles)
    for _ in range(3):
        m3 = H.refine(m3)
    y0 = np.array([1.5, 1.5, 1.5])
    out["proj_c2"] = H.project_to_space(lambda x, t, n=None: H.fundamental(np.asarray(x) - y0, t + 0.1, 1.0),
                                        m3, H.TimeGrid(1.0, 32), "X10")

    cases = (("dir0", "dirichlet", 0), ("dir1", "dirichlet", 1), ("neu0", "neumann", 0))
    results = {}
    for tag, problem, level in cases:
        t0 = time.perf_counter()
        so = {}
        r = HS.run_level(HS.StudyConfig(problem=problem), level, solution_out=so)
        print(tag, r, f"{time.perf_counter() - t0:.1f} s", flush=True)
        results[tag] = r
        for k in ("err_computed", "err_projected", "err_repr", "iterations", "residual", "E_t", "E_x"):
            out[f"{tag}_{k}"] = np.asarray(getattr(r, k))
        if level == 0:
            out[f"{tag}_solution"] = so["solution"]
            out[f"{tag}_data"] = so["data_projection"]
            out[f"{tag}_interior"] = so["interior_values"]
    # the reference's table writer on these results (format pin for results_to_csv)
    out["csv_dir"] = np.asarray(HS.results_to_csv([results["dir0"], results["dir1"]]))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()

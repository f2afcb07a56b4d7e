"""Command line for the device backend: ``python -m paper_2102_09811_b200.cli``.

Subcommands and options follow heatbem/cli.py:199-226 (``mesh-gen``,
``solve``, ``convergence``; the same flags, defaults, output files and exit
codes), so scripts written against ``heatbem`` run unchanged.  Every level
runs through ``study.LevelPipeline`` on the GPU.  ``verify-kernels`` is
not offered: it drives the reference's brute-force time-integration oracle,
which SURVEY §2 keeps out of scope (parity here is the test suite against
the oracle port, tests/).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

from .mesh import generate_cube_surface, save_mesh
from .quadrature import QuadratureConfig
from .study import StudyConfig, results_to_csv, results_to_report, run_level, run_study

PROG = "heatbem"


def _env_workers() -> int:
    """HEATBEM_WORKERS (the reference's variable) or 1; the device backend
    ignores the count but keeps the argument for compatibility."""
    try:
        return max(1, int(os.environ.get("HEATBEM_WORKERS", "1")))
    except ValueError:
        return 1


def _parse_point(text: str) -> tuple:
    parts = text.split(",")
    if len(parts) != 3:
        raise SystemExit("--source-point expects three comma-separated floats")
    return tuple(float(p) for p in parts)


def _config(ns) -> StudyConfig:
    return StudyConfig(problem=ns.problem, base_timesteps=ns.timesteps, base_subdivisions=ns.subdivisions,
                       alpha=ns.alpha, source_point=_parse_point(ns.source_point),
                       quad=QuadratureConfig(ns.quad_regular, ns.quad_singular),
                       workers=ns.workers or _env_workers(), deterministic=ns.deterministic,
                       n_interior=ns.interior_points)


def _write(out: Path, name: str, text: str) -> None:
    out.mkdir(parents=True, exist_ok=True)
    (out / name).write_text(text)


# -- subcommands ----------------------------------------------------------
def mesh_gen(ns) -> int:
    if ns.refine < 0:
        raise SystemExit("--refine must be >= 0")
    mesh = generate_cube_surface(4 * 2 ** ns.refine)
    ns.out.parent.mkdir(parents=True, exist_ok=True)
    save_mesh(mesh, ns.out)
    print(f"wrote {mesh.n_vertices} vertices, {mesh.n_triangles} triangles to {ns.out}")
    return 0


def solve(ns) -> int:
    if ns.mesh is not None:
        raise SystemExit("solving on external meshes is supported via the library API")
    config = _config(ns)
    arrays: dict = {}
    r = run_level(config, ns.refine, solution_out=arrays)
    ns.out.mkdir(parents=True, exist_ok=True)
    np.save(ns.out / "solution.npy", arrays["solution"])
    report = {"problem": config.problem, "level": ns.refine, "E_t": r.E_t, "E_x": r.E_x,
              "boundary_error_computed": r.err_computed, "boundary_error_projected": r.err_projected,
              "interior_error_repr": r.err_repr, "fgmres_iterations": r.iterations,
              "fgmres_residual": r.residual, "converged": r.converged,
              "assembly_seconds": r.seconds_assembly, "total_seconds": r.seconds_total}
    text = json.dumps(report, indent=2)
    _write(ns.out, "report.json", text)
    print(text)
    return 0 if r.converged else 1


def convergence(ns) -> int:
    if ns.levels < 2:
        raise SystemExit("--levels must be >= 2")
    config = _config(ns)
    results = run_study(config, ns.levels)
    table = results_to_csv(results)
    _write(ns.out, "convergence.csv", table)
    _write(ns.out, "report.json", results_to_report(config, results))
    print(table, end="")
    return 0 if all(r.converged for r in results) else 1


# -- parser ---------------------------------------------------------------
_STUDY_OPTIONS = (
    ("--problem", dict(choices=("dirichlet", "neumann"), default="dirichlet")),
    ("--refine", dict(type=int, default=0, metavar="L", help="refinement level (space quadrisected, time bisected)")),
    ("--timesteps", dict(type=int, default=8, help="time steps at level 0")),
    ("--subdivisions", dict(type=int, default=4, help="cube subdivisions per edge at level 0")),
    ("--alpha", dict(type=float, default=0.5)),
    ("--quad-regular", dict(type=int, default=4)),
    ("--quad-singular", dict(type=int, default=4)),
    ("--workers", dict(type=int, default=None, help="accepted for compatibility (HEATBEM_WORKERS)")),
    ("--out", dict(type=Path, default=Path("."))),
    ("--mesh", dict(type=Path, default=None)),
    ("--source-point", dict(type=str, default="0,0,1.5", metavar="x,y,z")),
    ("--interior-points", dict(type=int, default=10_000)),
)


def _study_parser(sub, name, fn, help_text, extra=()):
    p = sub.add_parser(name, help=help_text)
    for flag, kw in tuple(_STUDY_OPTIONS) + tuple(extra):
        p.add_argument(flag, **kw)
    p.add_argument("--deterministic", dest="deterministic", action="store_true", default=True)
    p.add_argument("--economical", dest="deterministic", action="store_false")
    p.set_defaults(fn=fn)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog=PROG, description="Space-time Galerkin BEM for the 3D heat equation "
                                                            "(B200 backend)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("mesh-gen", help="generate and save a cube surface mesh")
    p.add_argument("--refine", type=int, default=0)
    p.add_argument("--out", type=Path, required=True)
    p.set_defaults(fn=mesh_gen)
    _study_parser(sub, "solve", solve, "solve one boundary value problem")
    _study_parser(sub, "convergence", convergence, "run a refinement study",
                  extra=(("--levels", dict(type=int, default=3)),))
    return parser


def main(argv=None) -> int:
    ns = build_parser().parse_args(argv)
    return ns.fn(ns)


if __name__ == "__main__":
    sys.exit(main())

"""Generate tests/golden/ from the REFERENCE itself (run in the build container).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python oracle/gen_golden.py

Imports the reference package ``heatbem`` read-only from /root/reference and
stores, as small npz fixtures, what pins the hot path:

* tables.npz   -- triangle rules, Duffy tables, touching CSR / classification,
                  mesh-derived arrays of the BASELINE cube meshes;
* ops_small.npz -- full V, K, D2, D, V11 blocks on the reference's own test
                  meshes (cube n=1, n=2) -- the golden vectors of
                  heatbem/tests/test_assembly.py;
* c1.npz, c2.npz -- BASELINE configs 1 and 2: sampled rows of every block
                  plus a sha256 of every full block (canonical +0.0), so the
                  oracle can be proven bit-identical without storing GBs;
* field.npz    -- potentials (single/double layer) incl. eps > 0 times, and a
                  BASELINE config-4-shaped subset (unit cube L4, N = 64);
* solve_c2.npz -- the config-2 Dirichlet solve (data projection, rhs, FGMRES
                  with forward-substitution preconditioner);
* kernels.npz  -- scalar antiderivative values and the frozen KAT values of
                  heatbem/tests/test_kernels.py:101-115.

Nothing on the GPU box runs this file; /root/reference does not exist there.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = os.environ.get("HEATBEM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
import heatbem as H  # noqa: E402
from heatbem import field as HF  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
WORKERS = os.cpu_count()


def block_hashes(B: np.ndarray) -> np.ndarray:
    out = []
    for d in range(B.shape[0]):
        b = np.where(B[d] == 0.0, 0.0, B[d])   # canonical +0.0
        out.append(hashlib.sha256(np.ascontiguousarray(b, dtype="<f8").tobytes()).hexdigest())
    return np.array(out)


def unit_cube(levels):
    m = H.generate_cube_surface(1, 0.5)
    m = H.SurfaceMesh(m.vertices + 0.5, m.triangles)
    for _ in range(levels):
        m = H.refine(m)
    return m


def near_flags(mesh):
    c, dm = mesh.centroids, mesh.diameters
    dx = c[:, None, 0] - c[None, :, 0]
    dy = c[:, None, 1] - c[None, :, 1]
    dz = c[:, None, 2] - c[None, :, 2]
    dist = np.sqrt(dx * dx + dy * dy + dz * dz)
    return dist < 2.0 * np.maximum(dm[:, None], dm[None, :])


def gen_tables():
    from heatbem.assembly import _duffy_tables, _rule_tables, _touching_csr

    out = {}
    for o in range(1, 11):
        r = H.triangle_rule(o)
        out[f"tri{o}_nodes"], out[f"tri{o}_w"] = r.nodes, r.weights
    for so in (2, 4):
        off, t, s, w = _duffy_tables(so)
        out[f"duf{so}_off"], out[f"duf{so}_t"], out[f"duf{so}_s"], out[f"duf{so}_w"] = off, t, s, w
    for name, m in (("cube2", H.generate_cube_surface(2)), ("L2", unit_cube(2)), ("L3", unit_cube(3))):
        tn = _touching_csr(m)
        for k, a in zip(("indptr", "idx", "case", "permt", "perms"), tn):
            out[f"{name}_tn_{k}"] = a
        for k in ("vertices", "triangles", "areas", "normals", "centroids", "diameters"):
            out[f"{name}_{k}"] = getattr(m, k)
        out[f"{name}_near_bits"] = np.packbits(near_flags(m))
        h, w, p = _rule_tables(m, 4)
        out[f"{name}_reg_pts"] = p
        out[f"{name}_diameter"] = np.array(m.diameter)
    np.savez_compressed(os.path.join(OUT, "tables.npz"), **out)


def assemble_all(m, tg, p, which=("V", "K", "D2", "D", "V11")):
    q = H.QuadratureConfig(4, 4)
    res = {}
    if "V" in which or "D" in which:
        res["V"] = H.assemble_single_layer(m, tg, p, q, workers=WORKERS).blocks
    if "K" in which:
        res["K"] = H.assemble_double_layer(m, tg, p, q, workers=WORKERS).blocks
    if "D2" in which or "D" in which:
        res["D2"] = H.assemble_hypersingular_d2(m, tg, p, q, workers=WORKERS).blocks
    if "D" in which:
        res["D"] = H.hypersingular_from_single_layer(
            H.BlockToeplitzMatrix(res["V"]), H.BlockToeplitzMatrix(res["D2"]), m, p).blocks
    if "V11" in which:
        res["V11"] = H.assemble_single_layer(m, tg, p, q, "p1", "p1", workers=WORKERS).blocks
    return res


def gen_ops_small():
    out = {}
    for name, n, alpha, Et in (("cube1", 1, 0.5, 4), ("cube2", 2, 0.7, 4)):
        m = H.generate_cube_surface(n)
        tg = H.TimeGrid(1.0, Et)
        p = H.KernelParams(alpha, tg.step, length_scale=m.diameter)
        for op, B in assemble_all(m, tg, p).items():
            out[f"{name}_{op}"] = B
    # Toeplitz reuse: E_t = 2 with the same step reproduces the leading blocks
    m = H.generate_cube_surface(1)
    p = H.KernelParams(0.5, 0.25, length_scale=m.diameter)
    out["cube1_V_Et2"] = H.assemble_single_layer(m, H.TimeGrid(0.5, 2), p).blocks
    np.savez_compressed(os.path.join(OUT, "ops_small.npz"), **out)


def gen_config(name, level, Et, alpha, rows_p0, rows_p1):
    m = unit_cube(level)
    tg = H.TimeGrid(1.0, Et)
    p = H.KernelParams(alpha, tg.step, length_scale=m.diameter)
    t0 = time.time()
    res = assemble_all(m, tg, p)
    print(f"{name}: reference assembly {time.time() - t0:.1f} s")
    out = {"rows_p0": np.array(rows_p0), "rows_p1": np.array(rows_p1)}
    for op, B in res.items():
        rows = rows_p0 if op in ("V", "K") else rows_p1
        out[f"{op}_rows"] = B[:, rows, :]
        out[f"{op}_hash"] = block_hashes(B)
        out[f"{op}_maxabs"] = np.abs(B).max(axis=(1, 2))
        out[f"{op}_zeros"] = np.packbits(B[0] == 0.0)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)


def gen_field():
    out = {}
    m = H.generate_cube_surface(1)
    tg = H.TimeGrid(1.0, 4)
    p = H.KernelParams(0.5, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(11)
    w = rng.standard_normal((4, m.n_triangles))
    u = rng.standard_normal((4, m.n_vertices))
    xs = np.array([[0.1, -0.2, 0.15], [-0.3, 0.05, 0.2], [0.5, 0.5, -0.4]])
    ts = np.array([0.1, 0.25, 0.6, 1.0, 0.5 + 1e-3, 0.999])
    pts = [H.EvalPoint(x, t) for x in xs for t in ts]
    out["cube1_w"], out["cube1_u"] = w, u
    out["cube1_x"] = np.array([e.x for e in pts])
    out["cube1_t"] = np.array([e.t for e in pts])
    out["cube1_sl"] = H.eval_single_layer_potential(w, pts, m, tg, p)[0]
    out["cube1_dl"] = H.eval_double_layer_potential(u, pts, m, tg, p)[0]
    out["cube1_rep"] = H.represent(w, u, pts, m, tg, p)[0]
    # BASELINE config 4 shape: unit cube L4, N = 64, alpha = 1, seeded densities,
    # a handful of points at all 64 time-step ends
    m4 = unit_cube(4)
    tg4 = H.TimeGrid(1.0, 64)
    p4 = H.KernelParams(1.0, tg4.step, length_scale=m4.diameter)
    rng = np.random.default_rng(0)
    q = rng.uniform(-1, 1, (64, m4.n_triangles))
    g = rng.uniform(-1, 1, (64, m4.n_vertices))
    X = rng.uniform(0.05, 0.95, (100000, 3))
    sel = np.array([0, 1, 2, 99999])
    pts4 = [H.EvalPoint(X[i], k / 64) for i in sel for k in range(1, 65)]
    t0 = time.time()
    out["c4_sel"] = sel
    out["c4_u"] = H.represent(q, g, pts4, m4, tg4, p4)[0]
    print(f"c4 subset: {time.time() - t0:.1f} s")
    np.savez_compressed(os.path.join(OUT, "field.npz"), **out)


def gen_solve():
    m = unit_cube(3)
    tg = H.TimeGrid(1.0, 32)
    p = H.KernelParams(1.0, tg.step, length_scale=m.diameter)
    y0 = np.array([1.5, 1.5, 1.5])
    fn = lambda x, t, n=None: H.fundamental(np.asarray(x) - y0, t + 0.1, 1.0)  # noqa: E731
    M = H.assemble_mass(m, tg)
    K = H.assemble_double_layer(m, tg, p, workers=WORKERS)
    g = H.project_to_space(fn, m, tg, "X10")
    rhs = 0.5 * H.apply_toeplitz(M, g) + H.apply_toeplitz(K, g)
    V = H.assemble_single_layer(m, tg, p, workers=WORKERS)
    x, rep = H.fgmres(H.toeplitz_operator(V), rhs, rel_tol=1e-10,
                      right_precond=lambda v: H.forward_block_solve(V, v))
    xf = H.forward_block_solve(V, rhs)
    rng = np.random.default_rng(3)
    xr = rng.standard_normal((32, m.n_triangles))
    np.savez_compressed(os.path.join(OUT, "solve_c2.npz"), g=g, rhs=rhs, x=x, x_fwd=xf,
                        iterations=rep.iterations, residual=rep.residual, probe_x=xr,
                        probe_Vx=H.apply_toeplitz(V, xr), probe_KTx=H.apply_toeplitz(K, xr[:, :m.n_triangles], True))


def gen_neumann():
    """Neumann problem on the config-1 mesh (study.py:104-108,118-136): rhs =
    1/2 M'h - K'h with h the X00 projection of alpha dG/dn(x - y0, t + 0.1),
    system D = T^T (a^2 V) T + D2, FGMRES with forward substitution on D."""
    m = unit_cube(2)
    tg = H.TimeGrid(1.0, 16)
    p = H.KernelParams(1.0, tg.step, length_scale=m.diameter)
    y0 = np.array([1.5, 1.5, 1.5])
    fn = lambda x, t, n: H.grad_fundamental_normal(np.asarray(x) - y0, n, t + 0.1, 1.0)  # noqa: E731
    M = H.assemble_mass(m, tg)
    K = H.assemble_double_layer(m, tg, p, workers=WORKERS)
    h = H.project_to_space(fn, m, tg, "X00")
    rhs = 0.5 * H.apply_toeplitz(M, h, transpose_blocks=True) - H.apply_toeplitz(K, h, transpose_blocks=True)
    V = H.assemble_single_layer(m, tg, p, workers=WORKERS)
    D2 = H.assemble_hypersingular_d2(m, tg, p, workers=WORKERS)
    A = H.hypersingular_from_single_layer(V, D2, m, p, overwrite_d2=True)
    x, rep = H.fgmres(H.toeplitz_operator(A), rhs, rel_tol=1e-10,
                      right_precond=lambda v: H.forward_block_solve(A, v))
    np.savez_compressed(os.path.join(OUT, "neumann_c1.npz"), h=h, rhs=rhs, x=x, iterations=rep.iterations,
                        residual=rep.residual)
    print("neumann:", rep)


def gen_kernels():
    P1 = H.KernelParams(1.0, 0.25)
    P2 = H.KernelParams(0.5, 1.0 / 64, length_scale=3.0)
    rho = np.array([1e-13, 1e-3, 0.05, 0.3, 1.0, 1.7, 3.0])
    dl = np.array([0.0, 1e-17, 1e-4, 1.0 / 64, 0.25, 1.0])
    R, D = np.meshgrid(rho, dl, indexing="ij")
    out = {"rho": rho, "delta": dl}
    for nm, prm in (("a1", P1), ("a05", P2)):
        out[f"{nm}_tau_t"] = H.antideriv_tau_t(R, D, prm)
        ok = ~((R <= prm.rho_eps) & (D <= prm.delta_eps))
        out[f"{nm}_tau"] = np.where(ok, H.antideriv_tau(np.where(ok, R, 1.0), D, prm), np.nan)
    out["frozen_tau_t"] = np.array(H.antideriv_tau_t(2.0, 0.5, P1))
    out["frozen_V2"] = np.array(H.temporal_weight(H.TemporalWeightKind.SingleLayer,
                                                  np.array([1.0, 0.0, 0.0]), 2, H.KernelParams(1.0, 0.25)))
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1:                      # regenerate selected fixtures only
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_neumann()
    gen_tables()
    gen_kernels()
    gen_ops_small()
    gen_config("c1", 2, 16, 1.0, [0, 5, 17, 49, 81, 100, 150, 191], [0, 7, 33, 97])
    gen_config("c2", 3, 32, 1.0, [0, 111, 400, 767], [0, 50, 200, 385])
    gen_field()
    gen_solve()
    print("golden fixtures written to", OUT)

"""The CPU oracle (oracle/heatbem_oracle.c) against vectors produced by the
reference itself (oracle/gen_golden.py): bit-for-bit.  This pins the oracle
before any GPU result is compared with it."""
import hashlib

import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from _hb_util import golden

Q4 = hb.QuadratureConfig(4, 4)


def hashes(B):
    return [hashlib.sha256(np.ascontiguousarray(np.where(B[d] == 0.0, 0.0, B[d]), dtype="<f8").tobytes()).hexdigest()
            for d in range(B.shape[0])]


@pytest.mark.parametrize("name,n,alpha", [("cube1", 1, 0.5), ("cube2", 2, 0.7)])
def test_small_meshes_all_ops_bit_exact(oracle, name, n, alpha):
    g = golden("ops_small")
    m = hb.generate_cube_surface(n)
    tg = hb.TimeGrid(1.0, 4)
    p = hb.KernelParams(alpha, tg.step, length_scale=m.diameter)
    got = {op: oracle.assemble(m, tg, p, Q4, op) for op in ("V", "K", "D2", "V11")}
    got["D"] = oracle.curl_combine(got["V"], got["D2"], m, alpha)
    for op, B in got.items():
        assert np.array_equal(B, g[f"{name}_{op}"]), op


def test_toeplitz_reuse_golden(oracle):
    g = golden("ops_small")
    m = hb.generate_cube_surface(1)
    p = hb.KernelParams(0.5, 0.25, length_scale=m.diameter)
    V2 = oracle.assemble(m, hb.TimeGrid(0.5, 2), p, Q4, "V")
    assert np.array_equal(V2, g["cube1_V_Et2"])
    assert np.array_equal(V2, g["cube1_V"][:2])


def test_c1_full_blocks_bit_exact(oracle):
    """BASELINE config 1: every block of V, K, D2, V11, D hashes identically."""
    g = golden("c1")
    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    got = {op: oracle.assemble(m, tg, p, Q4, op) for op in ("V", "K", "D2", "V11")}
    got["D"] = oracle.curl_combine(got["V"], got["D2"], m, 1.0)
    for op, B in got.items():
        assert hashes(B) == list(g[f"{op}_hash"]), op
        rows = g["rows_p0"] if op in ("V", "K") else g["rows_p1"]
        assert np.array_equal(B[:, rows, :], g[f"{op}_rows"]), op


def test_c2_rows_bit_exact(oracle):
    """BASELINE config 2, sampled rows of V and K through the row oracle."""
    g = golden("c2")
    m = hb.unit_cube_mesh(3)
    tg = hb.TimeGrid(1.0, 32)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    for op in ("V", "K"):
        assert np.array_equal(oracle.assemble_rows(m, tg, p, Q4, op, g["rows_p0"]), g[f"{op}_rows"]), op


@pytest.mark.slow
def test_c2_full_blocks_bit_exact(oracle):
    g = golden("c2")
    m = hb.unit_cube_mesh(3)
    tg = hb.TimeGrid(1.0, 32)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    V = oracle.assemble(m, tg, p, Q4, "V")
    assert hashes(V) == list(g["V_hash"])
    D2 = oracle.assemble(m, tg, p, Q4, "D2")
    assert hashes(D2) == list(g["D2_hash"])
    assert hashes(oracle.curl_combine(V, D2, m, 1.0)) == list(g["D_hash"])
    assert hashes(oracle.assemble(m, tg, p, Q4, "K")) == list(g["K_hash"])


def test_potentials_bit_exact(oracle):
    from paper_2102_09811_b200.field import _decompose, _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    g = golden("field")
    m = hb.generate_cube_surface(1)
    tg = hb.TimeGrid(1.0, 4)
    p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
    hats, qw, qpts = rule_tables(m, 6)
    k, eps = _decompose(g["cube1_t"], tg.step)
    cur = (eps > 0) & (k < 4)
    for kind, coef, key in ((0, g["cube1_w"], "cube1_sl"), (1, g["cube1_u"], "cube1_dl")):
        dens = _interp_density_np(coef, m, hats)
        v = oracle.potential(kind, g["cube1_x"], k, eps, cur, dens, qpts, qw, m.areas, m.normals,
                             tg.step, p.alpha, p.delta_eps, p.rho_eps)
        assert np.array_equal(v, g[key]), key


def test_exact_oracle_close_to_reference(oracle):
    """The quad build is the same quadrature: it agrees with the reference to
    the reference's own rounding level (and the gate fixtures are present)."""
    g = golden("ops_small")
    m = hb.generate_cube_surface(1)
    tg = hb.TimeGrid(1.0, 4)
    p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
    Vx = oracle.assemble(m, tg, p, Q4, "V", exact=True)
    err = np.abs(Vx - g["cube1_V"]).max(axis=(1, 2)) / np.abs(Vx).max(axis=(1, 2))
    assert err.max() < 1e-12
    ex = golden("exact")
    assert ex["c1_V_eps_ref"].shape == (16,)


def test_oracle_solver_restatement_vs_dense():
    """oracle.apply_toeplitz / forward_block_solve (the bench's CPU baseline
    of the solve path, restating solver.py:47-73 / 165-184) vs the dense
    block lower-triangular expansion."""
    from oracle import oracle as O

    rng = np.random.default_rng(3)
    E_t, n = 6, 5
    B = 0.2 * rng.standard_normal((E_t, n, n))
    B[0] += 3 * np.eye(n)
    x = rng.standard_normal((E_t, n))
    dense = np.zeros((E_t * n, E_t * n))
    for k in range(E_t):
        for i in range(k + 1):
            dense[k * n:(k + 1) * n, i * n:(i + 1) * n] = B[k - i]
    assert np.allclose(O.apply_toeplitz(B, x).ravel(), dense @ x.ravel(), rtol=1e-14, atol=1e-14)
    assert np.allclose(dense @ O.forward_block_solve(B, x).ravel(), x.ravel(), rtol=1e-12, atol=1e-12)

"""Potentials (representation formula) vs the reference (golden) and the
oracle.  Tolerance 1e-12 relative (north star: 1e-11; the potentials carry
no time second difference, heatbem/tests/test_field.py uses 1e-12)."""
import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from _hb_util import golden

pytestmark = pytest.mark.gpu


def test_cube1_potentials_vs_reference():
    g = golden("field")
    m = hb.generate_cube_surface(1)
    tg = hb.TimeGrid(1.0, 4)
    p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
    pts = [hb.EvalPoint(x, t) for x, t in zip(g["cube1_x"], g["cube1_t"])]
    sl, w1 = hb.eval_single_layer_potential(g["cube1_w"], pts, m, tg, p)
    dl, w2 = hb.eval_double_layer_potential(g["cube1_u"], pts, m, tg, p)
    rep, w3 = hb.represent(g["cube1_w"], g["cube1_u"], pts, m, tg, p)
    for got, key in ((sl, "cube1_sl"), (dl, "cube1_dl"), (rep, "cube1_rep")):
        ref = g[key]
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max()), key
    assert not (w1.any() or w2.any() or w3.any())


def test_c4_subset_vs_reference():
    """BASELINE config 4 shape: unit cube L4, N = 64, seeded densities, the
    golden points at all 64 time-step ends (represent_grid path)."""
    g = golden("field")
    m = hb.unit_cube_mesh(4)
    tg = hb.TimeGrid(1.0, 64)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(0)
    q = rng.uniform(-1, 1, (64, m.n_triangles))
    gg = rng.uniform(-1, 1, (64, m.n_vertices))
    X = rng.uniform(0.05, 0.95, (100000, 3))
    u = hb.represent_grid(q, gg, X[g["c4_sel"]], m, tg, p).reshape(-1)
    ref = g["c4_u"]
    assert np.max(np.abs(u - ref)) <= 1e-11 * np.abs(ref).max()
    pts = [hb.EvalPoint(X[i], k / 64) for i in g["c4_sel"][:2] for k in range(1, 65)]
    u2, _ = hb.represent(q, gg, pts, m, tg, p)
    # represent routes time-step-end points through represent_grid: the same values
    assert np.array_equal(u2, u[:128])
    # the two-launch path (HB_REP_SEPARATE: two k_potential_reg launches) agrees to rounding
    import os
    os.environ["HB_REP_SEPARATE"] = "1"
    try:
        u3, _ = hb.represent(q, gg, pts, m, tg, p)
    finally:
        del os.environ["HB_REP_SEPARATE"]
    assert np.allclose(u3, u[:128], rtol=1e-13, atol=1e-14 * np.abs(ref).max())


@pytest.mark.parametrize("E_t,frac", [(16, 0.3), (40, 0.71), (64, 0.05)])
def test_represent_inside_steps_vs_oracle(oracle, E_t, frac):
    """represent() at t = k h + eps with eps > 0 (the current-interval term):
    groups of >= 8 points sharing eps go through the per-element kernel
    (k_represent_elem, EPS form), including k = E_t (no current interval)."""
    from paper_2102_09811_b200.field import _decompose, _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    m = hb.unit_cube_mesh(1)
    tg = hb.TimeGrid(1.0, E_t)
    p = hb.KernelParams(0.8, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(E_t)
    w = rng.standard_normal((E_t, m.n_triangles))
    uu = rng.standard_normal((E_t, m.n_vertices))
    X = rng.uniform(0.05, 0.95, (12, 3))
    ks = np.array(sorted({1, 2, E_t // 2, E_t - 1, E_t}))
    T = (np.repeat(ks, len(X)) + frac) * tg.step
    XX = np.tile(X, (len(ks), 1))
    pts = [hb.EvalPoint(x, t) for x, t in zip(XX, T)]
    got, _ = hb.represent(w, uu, pts, m, tg, p)
    hats, qw, qpts = rule_tables(m, 6)
    k, eps = _decompose(T, tg.step)
    assert np.all(eps > 0)
    cur = (eps > 0) & (k < E_t)
    refs = [oracle.potential(kind, XX, k, eps, cur, _interp_density_np(c, m, hats), qpts, qw, m.areas, m.normals,
                             tg.step, p.alpha, p.delta_eps, p.rho_eps) for kind, c in ((0, w), (1, uu))]
    ref = refs[0] - refs[1]
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max())


def test_random_points_vs_oracle(oracle):
    from paper_2102_09811_b200.field import _decompose, _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(0.7, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(7)
    w = rng.standard_normal((16, m.n_triangles))
    uu = rng.standard_normal((16, m.n_vertices))
    X = rng.uniform(0.1, 0.9, (40, 3))
    T = np.concatenate([rng.uniform(0, 1.2, 30), np.arange(1, 11) / 16])
    pts = [hb.EvalPoint(x, t) for x, t in zip(X, T)]
    hats, qw, qpts = rule_tables(m, 6)
    k, eps = _decompose(T, tg.step)
    cur = (eps > 0) & (k < 16)
    for kind, coef in ((0, w), (1, uu)):
        got, _ = (hb.eval_single_layer_potential if kind == 0 else hb.eval_double_layer_potential)(coef, pts, m, tg, p)
        ref = oracle.potential(kind, X, k, eps, cur, _interp_density_np(coef, m, hats), qpts, qw, m.areas,
                               m.normals, tg.step, p.alpha, p.delta_eps, p.rho_eps)
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max()), kind


@pytest.mark.parametrize("fused", ["elem", "nodes", False])
@pytest.mark.parametrize("E_t,steps", [(12, None), (24, None), (64, None), (64, [3, 17, 40, 64]), (40, [0, 1, 2, 40])])
def test_register_kernel_vs_oracle(oracle, E_t, steps, fused, monkeypatch):
    """represent_grid for time-step-end points -- k_represent_elem (default:
    per-element contraction on DMMA), k_represent_mma (HB_REP_NODES: per-node
    contraction) and k_potential_reg (one launch per potential,
    HB_REP_SEPARATE) -- for histories of <= 16 / 32 / 64 steps, E_t below the
    block size, k = 0, vs the oracle, with the element / eq range split across
    clusters of 1 and 7 CTAs (HB_POT_SPLIT)."""
    if not fused:
        monkeypatch.setenv("HB_REP_SEPARATE", "1")
    elif fused == "nodes":
        monkeypatch.setenv("HB_REP_NODES", "1")
    from paper_2102_09811_b200.field import _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    m = hb.unit_cube_mesh(1)
    tg = hb.TimeGrid(1.0, E_t)
    p = hb.KernelParams(0.8, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(E_t)
    w = rng.standard_normal((E_t, m.n_triangles))
    uu = rng.standard_normal((E_t, m.n_vertices))
    X = rng.uniform(0.05, 0.95, (70, 3))
    ks = np.arange(1, E_t + 1) if steps is None else np.asarray(steps)
    hats, qw, qpts = rule_tables(m, 6)
    XX = np.repeat(X, len(ks), axis=0)
    K = np.tile(ks, len(X))
    z = np.zeros(len(K))
    refs = [oracle.potential(kind, XX, K, z, z > 0, _interp_density_np(c, m, hats), qpts, qw, m.areas, m.normals,
                             tg.step, p.alpha, p.delta_eps, p.rho_eps) for kind, c in ((0, w), (1, uu))]
    ref = (refs[0] - refs[1]).reshape(len(X), len(ks))
    outs = []
    for split in ("1", "7"):
        monkeypatch.setenv("HB_POT_SPLIT", split)
        got = hb.represent_grid(w, uu, X, m, tg, p, time_steps=steps)
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max()), split
        outs.append(got)
    assert np.allclose(outs[0], outs[1], rtol=1e-13, atol=1e-14 * np.abs(ref).max())
    if steps is not None and 0 in steps:
        assert np.all(got[:, list(steps).index(0)] == 0.0)


@pytest.mark.parametrize("E_t", [80, 130])
def test_long_history_potentials_vs_oracle(oracle, E_t):
    """Histories longer than 64 steps (reference _field_numba._eval_potential
    handles any k): time-step ends k in (64, E_t] and points inside steps go
    through the general k_potential path, k <= 64 through the per-element
    kernel; points past the final time (k > E_t) through the general path
    too.  Both potentials and the representation formula vs the oracle."""
    from paper_2102_09811_b200.field import _decompose, _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    m = hb.unit_cube_mesh(1)
    tg = hb.TimeGrid(1.0, E_t)
    p = hb.KernelParams(0.9, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(E_t)
    w = rng.standard_normal((E_t, m.n_triangles))
    uu = rng.standard_normal((E_t, m.n_vertices))
    X = rng.uniform(0.05, 0.95, (10, 3))
    ks = np.array([1, 40, 64, 65, 77, E_t - 1, E_t])
    T = np.concatenate([np.repeat(ks, len(X)) * tg.step,                       # time-step ends
                        (np.repeat(ks[:-1], len(X)) + 0.37) * tg.step,         # inside steps
                        np.full(len(X), 1.0 + 2.5 * tg.step)])                  # past the final time
    XX = np.tile(X, (len(T) // len(X), 1))
    pts = [hb.EvalPoint(x, t) for x, t in zip(XX, T)]
    hats, qw, qpts = rule_tables(m, 6)
    k, eps = _decompose(T, tg.step)
    cur = (eps > 0) & (k < E_t)
    refs = {}
    for kind, c in ((0, w), (1, uu)):
        refs[kind] = oracle.potential(kind, XX, k, eps, cur, _interp_density_np(c, m, hats), qpts, qw, m.areas,
                                      m.normals, tg.step, p.alpha, p.delta_eps, p.rho_eps)
    sl, _ = hb.eval_single_layer_potential(w, pts, m, tg, p)
    dl, _ = hb.eval_double_layer_potential(uu, pts, m, tg, p)
    rep, _ = hb.represent(w, uu, pts, m, tg, p)
    for got, ref in ((sl, refs[0]), (dl, refs[1]), (rep, refs[0] - refs[1])):
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max())


@pytest.mark.parametrize("E_t", [70, 128, 200, 300])
def test_long_history_grid_per_element_kernel(oracle, E_t, monkeypatch):
    """represent_grid with histories longer than 64 steps runs the per-element
    kernel once per block of 64 output steps (k_represent_elem LONG: gap
    windows below the block as full Toeplitz tiles).  Checked against the
    general k_potential path on every (point, step) and against the oracle
    (reference _field_numba._eval_potential, any k) on sampled steps; cluster
    splits give the same values; a step subset with k = 0 returns exact zeros."""
    from paper_2102_09811_b200.field import _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    m = hb.unit_cube_mesh(1)
    tg = hb.TimeGrid(1.0, E_t)
    p = hb.KernelParams(0.8, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(1000 + E_t)
    w = rng.standard_normal((E_t, m.n_triangles))
    uu = rng.standard_normal((E_t, m.n_vertices))
    X = rng.uniform(0.05, 0.95, (40, 3))
    got = hb.represent_grid(w, uu, X, m, tg, p)
    assert got.shape == (40, E_t) and np.all(np.isfinite(got))
    # the oracle on sampled steps (block ends, block starts, the last step)
    ks = np.unique(np.array([1, 63, 64, 65, 66, min(E_t, 127), min(E_t, 128), min(E_t, 129), E_t - 1, E_t]))
    Xs = X[::7]
    XX = np.repeat(Xs, len(ks), axis=0)
    kk = np.tile(ks, len(Xs))
    hats, qw, qpts = rule_tables(m, 6)
    zero = np.zeros(len(kk))
    cur = np.zeros(len(kk), dtype=bool)
    ref = (oracle.potential(0, XX, kk, zero, cur, _interp_density_np(w, m, hats), qpts, qw, m.areas, m.normals,
                            tg.step, p.alpha, p.delta_eps, p.rho_eps)
           - oracle.potential(1, XX, kk, zero, cur, _interp_density_np(uu, m, hats), qpts, qw, m.areas, m.normals,
                              tg.step, p.alpha, p.delta_eps, p.rho_eps)).reshape(len(Xs), len(ks))
    sub = got[::7][:, ks - 1]
    assert np.allclose(sub, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max())
    # a step subset including k = 0, two cluster splits
    steps = np.array([0, 1, 64, 65, E_t])
    outs = []
    for split in ("1", "3"):
        monkeypatch.setenv("HB_POT_SPLIT", split)
        part = hb.represent_grid(w, uu, X, m, tg, p, time_steps=steps)
        assert np.all(part[:, 0] == 0.0)
        assert np.allclose(part[:, 1:], got[:, steps[1:] - 1], rtol=1e-13, atol=1e-14 * np.abs(got).max())
        outs.append(part)
    monkeypatch.delenv("HB_POT_SPLIT")
    # the general path (two potential launches) on every (point, step)
    monkeypatch.setenv("HB_REP_SEPARATE", "1")
    gen = hb.represent_grid(w, uu, X, m, tg, p)
    assert np.allclose(got, gen, rtol=1e-12, atol=1e-13 * np.abs(gen).max())

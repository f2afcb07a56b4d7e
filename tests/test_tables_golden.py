"""Host precompute vs tables dumped from the reference (bit-exact).

The device kernels consume these arrays; the near/far rule choice depends
on centroids/diameters bit-exactly (heatbem/_assembly_numba.py:218-223)."""
import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import quadrature as Q


@pytest.mark.parametrize("order", range(1, 11))
def test_triangle_rules(g_tables, order):
    r = hb.triangle_rule(order)
    assert np.array_equal(r.nodes, g_tables[f"tri{order}_nodes"])
    assert np.array_equal(r.weights, g_tables[f"tri{order}_w"])


@pytest.mark.parametrize("so", [2, 4])
def test_duffy_tables(g_tables, so):
    off, t, s, w = Q.duffy_tables(so)
    for name, a in zip(("off", "t", "s", "w"), (off, t, s, w)):
        assert np.array_equal(a, g_tables[f"duf{so}_{name}"]), name


MESHES = {"cube2": lambda: hb.generate_cube_surface(2), "L2": lambda: hb.unit_cube_mesh(2),
          "L3": lambda: hb.unit_cube_mesh(3)}


@pytest.mark.parametrize("name", list(MESHES))
def test_mesh_arrays_and_touching_csr(g_tables, name):
    m = MESHES[name]()
    for k in ("vertices", "triangles", "areas", "normals", "centroids", "diameters"):
        assert np.array_equal(getattr(m, k), g_tables[f"{name}_{k}"]), k
    assert m.diameter == float(g_tables[f"{name}_diameter"])
    tn = Q.touching_csr(m)
    for k, a in zip(("indptr", "idx", "case", "permt", "perms"), tn):
        assert np.array_equal(a, g_tables[f"{name}_tn_{k}"]), k
    assert np.array_equal(Q.rule_tables(m, 4)[2], g_tables[f"{name}_reg_pts"])


@pytest.mark.parametrize("name", list(MESHES))
def test_near_far_classification_bits(g_tables, name):
    """Host restatement of the reference's IEEE near test reproduces its bits
    (the device test applies the same operation order, tests/test_assembly_gpu.py)."""
    m = MESHES[name]()
    c, dm = m.centroids, m.diameters
    dx = c[:, None, 0] - c[None, :, 0]
    dy = c[:, None, 1] - c[None, :, 1]
    dz = c[:, None, 2] - c[None, :, 2]
    near = np.sqrt(dx * dx + dy * dy + dz * dz) < 2.0 * np.maximum(dm[:, None], dm[None, :])
    assert np.array_equal(np.packbits(near), g_tables[f"{name}_near_bits"])


def test_touching_implies_near(g_tables):
    """Every touching pair is also 'near' by the centroid test on the BASELINE
    cubes (the regular kernel still checks touching first, as the reference)."""
    for name in MESHES:
        m = MESHES[name]()
        ip, idx = Q.touching_csr(m)[:2]
        near = np.unpackbits(g_tables[f"{name}_near_bits"])[: m.n_triangles ** 2].reshape(m.n_triangles, -1)
        rows = np.repeat(np.arange(m.n_triangles), np.diff(ip))
        assert near[rows, idx].all()

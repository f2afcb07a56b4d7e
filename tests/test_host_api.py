"""Host-side logic that needs no GPU: plan bookkeeping, block container,
HBTM1 I/O, meshes, kernels, and loud failure without a device."""
import os

import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from _hb_util import golden


def test_assembly_plan_matches_three_term_rule():
    plan = hb.AssemblyPlan(5)
    assert plan.targets(0) == [(0, 1.0, True), (1, -1.0, False)]
    assert plan.targets(3) == [(2, -1.0, False), (3, 2.0, False), (4, -1.0, False)]
    assert plan.targets(5) == [(4, -1.0, False)]
    assert plan.contributors(0) == [(0, 1.0, True), (1, -1.0, False)]
    for d in range(1, 5):
        assert [c[:2] for c in plan.contributors(d)] == [(d - 1, -1.0), (d, 2.0), (d + 1, -1.0)]
    assert hb.AssemblyPlan(1).targets(0) == [(0, 1.0, True)]
    with pytest.raises(ValueError):
        plan.targets(6)


def test_block_container_and_transpose_share_storage():
    B = np.arange(2 * 3 * 4, dtype=float).reshape(2, 3, 4)
    M = hb.BlockToeplitzMatrix(B)
    assert (M.n_blocks, M.block_rows, M.block_cols) == (2, 3, 4)
    T = M.transposed()
    assert (T.block_rows, T.block_cols) == (4, 3)
    assert T.blocks is M.blocks
    assert T.transposed().block_rows == 3


def test_hbtm1_roundtrip(tmp_path):
    B = np.random.default_rng(0).standard_normal((3, 5, 7))
    p = tmp_path / "b.hbtm"
    hb.save_blocks(hb.BlockToeplitzMatrix(B), p)
    raw = p.read_bytes()
    assert raw[:5] == b"HBTM1" and len(raw) == 5 + 24 + B.size * 8
    assert np.array_equal(hb.load_blocks(p).blocks, B)
    (tmp_path / "bad").write_bytes(b"XXXXX" + raw[5:])
    with pytest.raises(ValueError):
        hb.load_blocks(tmp_path / "bad")
    (tmp_path / "short").write_bytes(raw[:-8])
    with pytest.raises(ValueError):
        hb.load_blocks(tmp_path / "short")


def test_mass_matrix():
    m = hb.generate_cube_surface(1)
    tg = hb.TimeGrid(1.0, 4)
    M = hb.assemble_mass(m, tg)
    assert M.diagonal_only and M.blocks.shape == (1, 12, 8)
    assert np.allclose(M.blocks[0].sum(axis=1), tg.step * m.areas)


def test_meshes_and_io(tmp_path):
    for lvl, (E, N) in {2: (192, 98), 3: (768, 386)}.items():
        m = hb.unit_cube_mesh(lvl)
        assert (m.n_triangles, m.n_vertices) == (E, N) and m.is_admissible()
        assert np.all(np.einsum("ij,ij->i", m.normals, m.centroids - 0.5) > 0)
    ico = hb.generate_icosphere(3)
    assert (ico.n_triangles, ico.n_vertices) == (1280, 642) and ico.is_admissible()
    assert np.allclose(np.linalg.norm(ico.vertices, axis=1), 1.0)
    assert np.all(np.einsum("ij,ij->i", ico.normals, ico.centroids) > 0)
    p = tmp_path / "m.txt"
    hb.save_mesh(ico, p)
    back = hb.load_mesh(p)
    assert np.array_equal(back.vertices, ico.vertices) and np.array_equal(back.triangles, ico.triangles)
    (tmp_path / "bad.txt").write_text("heatbem-mesh 1\nvertices 3\n0 0 0\n1 0 0\n")
    with pytest.raises(hb.MeshParseError) as ei:
        hb.load_mesh(tmp_path / "bad.txt")
    assert ei.value.line == 4
    with pytest.raises(hb.MeshError):
        hb.SurfaceMesh(np.zeros((3, 3)), np.array([[0, 1, 1]]))


def test_icosphere_l5_counts():
    """BASELINE config 3 mesh: 20480 triangles, 10242 nodes, touching-pair
    counts of SURVEY 8(d) (identical 20480, edge 61440, vertex 184260)."""
    from paper_2102_09811_b200.quadrature import touching_csr

    m = hb.generate_icosphere(5)
    assert (m.n_triangles, m.n_vertices) == (20480, 10242)
    case = touching_csr(m)[2]
    assert [int((case == c).sum()) for c in (0, 1, 2)] == [20480, 61440, 184260]
    assert 0.039 < m.diameters.min() and m.diameters.max() < 0.0414


def test_kernel_values_golden():
    g = golden("kernels")
    P1 = hb.KernelParams(1.0, 0.25)
    P2 = hb.KernelParams(0.5, 1.0 / 64, length_scale=3.0)
    R, D = np.meshgrid(g["rho"], g["delta"], indexing="ij")
    for nm, prm in (("a1", P1), ("a05", P2)):
        assert np.allclose(hb.antideriv_tau_t(R, D, prm), g[f"{nm}_tau_t"], rtol=1e-14, atol=0)
        ok = ~np.isnan(g[f"{nm}_tau"])
        assert np.allclose(hb.antideriv_tau(R[ok], D[ok], prm), g[f"{nm}_tau"][ok], rtol=1e-14, atol=0)
    assert hb.antideriv_tau_t(2.0, 0.5, P1) == pytest.approx(0.09924230908944406, rel=1e-12)
    w = hb.temporal_weight(hb.TemporalWeightKind.SingleLayer, np.array([1.0, 0, 0]), 2, hb.KernelParams(1.0, 0.25))
    assert w == pytest.approx(0.002481956787833119, rel=1e-10)
    with pytest.raises(hb.SingularEvaluationError):
        hb.antideriv_tau(0.0, 0.0, P1)


def test_evalpoint_decompose_matches_reference_rule():
    h = 1.0 / 64
    for t, (k, eps) in ((1.0, (64, 0.0)), (0.5, (32, 0.0)), (0.0, (0, 0.0))):
        assert hb.EvalPoint(np.zeros(3), t).decompose(h) == (k, eps)
    k, eps = hb.EvalPoint(np.zeros(3), 0.51).decompose(h)
    assert k == 32 and eps == pytest.approx(0.51 - 32 * h)


def test_compute_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    m = hb.generate_cube_surface(1)
    tg = hb.TimeGrid(1.0, 2)
    from paper_2102_09811_b200._native import NativeUnavailable

    with pytest.raises(NativeUnavailable):
        hb.assemble_single_layer(m, tg, hb.KernelParams(1.0, 0.5))


def test_row_slabs_cover_rows_with_balanced_work():
    from paper_2102_09811_b200.assembly import _row_slabs

    for E, sym in ((768, True), (768, False), (5, True), (3, False)):
        sl = _row_slabs(E, sym, 4)
        assert sl[0][0] == 0 and sl[-1][1] == E
        assert all(a < b for a, b in sl) and all(sl[i][1] == sl[i + 1][0] for i in range(len(sl) - 1))
    work = [sum(768 - e for e in range(a, b)) for a, b in _row_slabs(768, True, 4)]
    assert max(work) / min(work) < 1.05


def test_row_slabs_from_work_fractions():
    """A sequence of work fractions instead of a count: contiguous cover of the
    rows, each slab's share of the upper-triangle pair work as requested."""
    from paper_2102_09811_b200.assembly import _row_slabs

    fr = (0.1, 0.3, 0.6)
    sl = _row_slabs(768, True, fr)
    assert sl[0][0] == 0 and sl[-1][1] == 768 and all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
    work = np.array([sum(768 - e for e in range(a, b)) for a, b in sl], dtype=float)
    assert np.allclose(work / work.sum(), fr, atol=0.01)
    assert _row_slabs(100, False, (1, 1)) == [(0, 50), (50, 100)]
    with pytest.raises(ValueError):
        _row_slabs(100, True, (0.5, 0.0))


def test_blocks_host_edits_are_tracked():
    """The reference edits operators through .blocks (assembly.py:328-333:
    out = D2.blocks; out[d] += ...): item assignment, in-place ufuncs and
    writes through views bump the shared storage version (which drops the
    cached (A^0)^-1 and makes the next device use upload the edit); the
    transposed twin shares it; assigning .blocks replaces the blocks."""
    rng = np.random.default_rng(3)
    M = hb.BlockToeplitzMatrix(rng.standard_normal((3, 4, 4)))
    Mt = M.transposed()
    v0 = M.version
    out = M.blocks
    out[1] += 1.0                       # reference idiom
    assert M.version > v0 and Mt.version == M.version
    v1 = M.version
    out += 0.5                          # in-place ufunc
    assert M.version > v1
    v2 = M.version
    view = out[2]
    view[0, 0] = 7.0                    # write through a view
    assert M.version > v2 and M.blocks[2, 0, 0] == 7.0 and Mt.blocks[2, 0, 0] == 7.0
    v3 = M.version
    np.multiply(out, 2.0, out=out)
    assert M.version > v3
    v4 = M.version
    s = out.sum() + float((out[0] * 2.0).max())   # reads do not count as edits
    assert M.version == v4 and np.isfinite(s)
    M.blocks = np.zeros((2, 4, 4))
    assert M.version > v4 and M.n_blocks == 2 and Mt.n_blocks == 2

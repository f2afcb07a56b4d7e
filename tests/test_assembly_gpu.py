"""Parity of the sm_100a assembly (through the C ABI) with the reference.

Tolerances (north star: <= 1e-11 of each block's max-abs entry):
* bit-exact: pair classification, exact-zero pattern, symmetry, Toeplitz
  block reuse, d-sharding / row-chunking invariance, run-to-run determinism;
* values: per block d, |gpu - ref| / max|ref| <= 1e-11 wherever the
  reference's OWN deviation from the exact value of the same quadrature,
  eps_ref(d) (quad-precision oracle, tests/golden/exact.npz), is <= 3.3e-12;
  above that <= 3 eps_ref(d): the time second difference
  B^d = -L(d-1) + 2L(d) - L(d+1) and the curl transform of D amplify the
  reference's last-bit libm errors beyond 1e-11 at large d (2.5e-11 off exact
  for c2 V, 4.6e-9 for c2 D) -- a GPU result closer to exact than that
  cannot also be within 1e-11 of the reference;
* accuracy: |gpu - exact| <= eps_ref(d) + 1e-13 -- the GPU blocks are at
  least as close to the exact quadrature as the reference's own fp64 blocks
  (measured on the golden rows, profiles/r02_parity_c1_c2.json: <= 0.98
  eps_ref; the moment form makes the large-d blocks of V, and through the
  curl D, nearly exact, and F(x) removes the 1/x^2 cancellation of the
  reference's K bracket).
"""
import os

import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from _hb_util import golden, rel_block_err

pytestmark = pytest.mark.gpu
Q4 = hb.QuadratureConfig(4, 4)
ACC = {"V": 1.0, "V11": 1.0, "D2": 1.0, "D": 1.0, "K": 1.0}


def gate(eps_ref):
    """|gpu - ref| bar per block: the literal 1e-11 where the reference is
    well conditioned (eps_ref <= 3.3e-12), 3 eps_ref above."""
    eps_ref = np.asarray(eps_ref)
    return np.where(eps_ref <= 3.3e-12, 1e-11, 3 * eps_ref)
OPS = {
    "V": lambda m, tg, p, **k: hb.assemble_single_layer(m, tg, p, Q4, **k),
    "K": lambda m, tg, p, **k: hb.assemble_double_layer(m, tg, p, Q4, **k),
    "D2": lambda m, tg, p, **k: hb.assemble_hypersingular_d2(m, tg, p, Q4, **k),
    "V11": lambda m, tg, p, **k: hb.assemble_single_layer(m, tg, p, Q4, "p1", "p1", **k),
}


def c1():
    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    return m, tg, hb.KernelParams(1.0, tg.step, length_scale=m.diameter)


def c2():
    m = hb.unit_cube_mesh(3)
    tg = hb.TimeGrid(1.0, 32)
    return m, tg, hb.KernelParams(1.0, tg.step, length_scale=m.diameter)


@pytest.fixture(scope="module")
def c1_ops():
    m, tg, p = c1()
    out = {op: fn(m, tg, p).blocks for op, fn in OPS.items()}
    V, D2 = hb.BlockToeplitzMatrix(out["V"]), hb.BlockToeplitzMatrix(out["D2"])
    out["D"] = hb.hypersingular_from_single_layer(V, D2, m, p).blocks
    return out


@pytest.mark.parametrize("name,n,alpha", [("cube1", 1, 0.5), ("cube2", 2, 0.7)])
def test_reference_test_meshes_all_ops(name, n, alpha):
    g = golden("ops_small")
    m = hb.generate_cube_surface(n)
    tg = hb.TimeGrid(1.0, 4)
    p = hb.KernelParams(alpha, tg.step, length_scale=m.diameter)
    got = {op: fn(m, tg, p).blocks for op, fn in OPS.items()}
    got["D"] = hb.hypersingular_from_single_layer(hb.BlockToeplitzMatrix(got["V"]),
                                                  hb.BlockToeplitzMatrix(got["D2"]), m, p).blocks
    for op, B in got.items():
        ref = g[f"{name}_{op}"]
        assert rel_block_err(B, ref).max() <= 1e-11, op
        assert np.array_equal(B == 0.0, ref == 0.0), op
        assert not np.any(np.signbit(B[B == 0.0])), op
        if op != "K":
            assert all(np.array_equal(B[d], B[d].T) for d in range(4)), op


def test_c1_parity_and_accuracy(c1_ops):
    g, ex = golden("c1"), golden("exact")
    for op, B in c1_ops.items():
        rows = g["rows_p0"] if op in ("V", "K") else g["rows_p1"]
        ref_rows, ex_rows, bmax = g[f"{op}_rows"], ex[f"c1_{op}_exact_rows"], g[f"{op}_maxabs"]
        eps_ref = ex[f"c1_{op}_eps_ref"]
        par = np.abs(B[:, rows, :] - ref_rows).max(axis=(1, 2)) / bmax
        assert np.all(par <= gate(eps_ref)), (op, par, eps_ref)
        acc = np.abs(B[:, rows, :] - ex_rows).max(axis=(1, 2)) / bmax
        assert np.all(acc <= ACC[op] * eps_ref + 1e-13), (op, acc, eps_ref)
        assert np.array_equal(np.packbits(B[0] == 0.0), g[f"{op}_zeros"]), op


def test_c1_full_blocks_vs_oracle(oracle, c1_ops):
    m, tg, p = c1()
    ex = golden("exact")
    for op in ("V", "K", "D2", "V11"):
        ref = oracle.assemble(m, tg, p, Q4, op)
        err = rel_block_err(c1_ops[op], ref)
        assert np.all(err <= gate(ex[f"c1_{op}_eps_ref"])), (op, err)
        assert np.array_equal(c1_ops[op] == 0.0, ref == 0.0), op
        if op != "K":
            assert all(np.array_equal(c1_ops[op][d], c1_ops[op][d].T) for d in range(16)), op
    assert all(np.array_equal(c1_ops["D"][d], c1_ops["D"][d].T) for d in range(16))


def test_classification_bit_exact(g_tables):
    """The device near/far + touching classification equals the reference's
    _touching_csr and IEEE near test for every ordered pair (ties included)."""
    from paper_2102_09811_b200.assembly import pair_classes

    for name, m in (("L2", hb.unit_cube_mesh(2)), ("L3", hb.unit_cube_mesh(3)),
                    ("cube2", hb.generate_cube_surface(2))):
        cls = pair_classes(m)
        E = m.n_triangles
        near = np.unpackbits(g_tables[f"{name}_near_bits"])[: E * E].reshape(E, E)
        ip, idx, case = (g_tables[f"{name}_tn_{k}"] for k in ("indptr", "idx", "case"))
        want = near.astype(np.int8)
        rows = np.repeat(np.arange(E), np.diff(ip))
        want[rows, idx] = 2 + case
        assert np.array_equal(cls, want), name


def test_toeplitz_block_reuse_bit_identity():
    m = hb.unit_cube_mesh(2)
    p = hb.KernelParams(1.0, 1.0 / 16, length_scale=m.diameter)
    for op in ("V", "K", "D2"):
        full = OPS[op](m, hb.TimeGrid(1.0, 16), p).blocks
        half = OPS[op](m, hb.TimeGrid(0.5, 8), p).blocks
        assert np.array_equal(full[:8], half), op


def test_d_sharding_and_row_chunking_are_bitwise_invariant():
    m, tg, p = c1()
    for op in ("V", "K", "D2"):
        full = OPS[op](m, tg, p).blocks
        for d0, d1 in ((0, 1), (1, 7), (5, 16), (15, 16)):
            part = OPS[op](m, tg, p, d_range=(d0, d1)).blocks
            assert np.array_equal(part, full[d0:d1]), (op, d0, d1)
        small = OPS[op](m, tg, p, workspace_bytes=3 * 1024 * 1024).blocks   # many row chunks
        assert np.array_equal(small, full), op
        assert np.array_equal(OPS[op](m, tg, p).blocks, full), op            # run to run


def test_long_history_windows_match_single_window():
    """E_t > 32 splits the gaps into windows with halo slots; blocks must not
    depend on the window split (compare against d-sharded assembly)."""
    m = hb.generate_cube_surface(2)
    tg = hb.TimeGrid(1.0, 80)
    p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
    for op in ("V", "K", "D2"):
        full = OPS[op](m, tg, p).blocks
        parts = np.concatenate([OPS[op](m, tg, p, d_range=(a, b)).blocks for a, b in ((0, 3), (3, 41), (41, 80))])
        assert np.array_equal(parts, full), op


def test_long_history_vs_oracle(oracle):
    """80 blocks on the reference's [-1, 1]^3 cube (alpha = 0.5): rho~^2 reaches
    480 here, so most pairs stay in the point-by-point form for all 80 gaps
    (istar = rho~^2 / 3 > E_t) -- the same second-difference amplification of
    per-point rounding as the reference; measured |gpu - exact| <= 1.14
    eps_ref (V, d = 58), hence the 1.5 bar on this synthetic case (BASELINE
    configs: <= 1.0, tests above and below)."""
    m = hb.generate_cube_surface(2)
    tg = hb.TimeGrid(1.0, 80)
    p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
    for op in ("V", "K", "D2"):
        ref = oracle.assemble(m, tg, p, Q4, op)
        got = OPS[op](m, tg, p).blocks
        x = oracle.assemble(m, tg, p, Q4, op, exact=True)
        eps_ref = rel_block_err(ref, x)
        assert np.all(rel_block_err(got, ref) <= gate(eps_ref)), op
        assert np.all(rel_block_err(got, x) <= 1.5 * eps_ref + 1e-13), op


def test_c2_rows_vs_reference():
    g, ex = golden("c2"), golden("exact")
    m, tg, p = c2()
    V = hb.assemble_single_layer(m, tg, p, Q4)
    K = hb.assemble_double_layer(m, tg, p, Q4)
    D2 = hb.assemble_hypersingular_d2(m, tg, p, Q4)
    D = hb.hypersingular_from_single_layer(V, D2, m, p)
    got = {"V": V.blocks, "K": K.blocks, "D2": D2.blocks, "D": D.blocks}
    for op, B in got.items():
        rows = g["rows_p0"] if op in ("V", "K") else g["rows_p1"]
        par = np.abs(B[:, rows, :] - g[f"{op}_rows"]).max(axis=(1, 2)) / g[f"{op}_maxabs"]
        if f"c2_{op}_eps_ref" in ex:
            eps_ref = ex[f"c2_{op}_eps_ref"]
            assert np.all(par <= gate(eps_ref)), (op, par)
            acc = np.abs(B[:, rows, :] - ex[f"c2_{op}_exact_rows"]).max(axis=(1, 2)) / g[f"{op}_maxabs"]
            assert np.all(acc <= ACC[op] * eps_ref + 1e-13), (op, acc, eps_ref)
        else:   # D2: well conditioned, plain bar
            assert np.all(par <= 1e-11), (op, par)
        assert np.array_equal(np.packbits(B[0] == 0.0), g[f"{op}_zeros"]), op


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_fused_single_layer_and_hypersingular(cfg):
    """hb_assemble_vd (assemble_hypersingular without a given single layer,
    assemble_all): V and D2 in the same row chunks, the curl transform folded
    into D2's p1 x p1 finalize.  V is bitwise the standalone V; D meets the
    same parity / accuracy gates as the curl-combine D, is exactly symmetric,
    and differs from it only by summation order."""
    g, ex = golden(cfg), golden("exact")
    m, tg, p = c1() if cfg == "c1" else c2()
    from paper_2102_09811_b200.assembly import _assemble_vd

    V, D = _assemble_vd(m, tg, p, Q4)
    V_ref = hb.assemble_single_layer(m, tg, p, Q4)
    assert np.array_equal(V.blocks, V_ref.blocks)
    B = D.blocks
    assert all(np.array_equal(B[d], B[d].T) for d in range(B.shape[0]))
    rows = g["rows_p1"]
    eps_ref = ex[f"{cfg}_D_eps_ref"]
    par = np.abs(B[:, rows, :] - g["D_rows"]).max(axis=(1, 2)) / g["D_maxabs"]
    assert np.all(par <= gate(eps_ref)), (par, eps_ref)
    acc = np.abs(B[:, rows, :] - ex[f"{cfg}_D_exact_rows"]).max(axis=(1, 2)) / g["D_maxabs"]
    assert np.all(acc <= ACC["D"] * eps_ref + 1e-13), (acc, eps_ref)
    assert np.array_equal(np.packbits(B[0] == 0.0), g["D_zeros"])
    D_curl = hb.hypersingular_from_single_layer(V_ref, hb.assemble_hypersingular_d2(m, tg, p, Q4), m, p).blocks
    assert np.abs(B - D_curl).max() <= 1e-13 * np.abs(D_curl).max()
    os.environ["HB_FUSED_VD"] = "1"                                # the public path, fused
    try:
        D_api = hb.assemble_hypersingular(m, tg, p, Q4).blocks
    finally:
        del os.environ["HB_FUSED_VD"]
    assert np.array_equal(D_api, B)
    # a small staging budget: several row chunks, same blocks bitwise
    V2, D2c = _assemble_vd(m, tg, p, Q4, workspace_bytes=1 << 22)
    assert np.array_equal(V2.blocks, V.blocks) and np.array_equal(D2c.blocks, B)


def test_instrumentation_and_api_variants():
    m, tg, p = c1()
    inst = hb.AssemblyInstrumentation()
    V = hb.assemble_single_layer(m, tg, p, Q4, instrumentation=inst)
    assert inst.kernel_batch_passes == tg.n_steps + 1 and inst.seconds > 0
    D_a = hb.assemble_hypersingular(m, tg, p, Q4, single_layer=V).blocks
    D_b = hb.hypersingular_from_single_layer(V, hb.assemble_hypersingular_d2(m, tg, p, Q4), m, p).blocks
    assert np.array_equal(D_a, D_b)
    with pytest.raises(ValueError):
        hb.assemble_single_layer(m, tg, p, Q4, "p0", "p1")


@pytest.mark.parametrize("world,E_t", [(2, 16), (3, 40)])
def test_row_parallel_into_d_shards_bitwise(world, E_t):
    """Row-parallel assembly (distributed.assemble_row_parallel's kernel path)
    on one GPU: ``world`` balanced test-row ranges store through one block
    pointer table into ``world`` separate NaN-filled d-shard buffers (stand-ins
    for the peer GPUs' memory).  The shards are bitwise the 1-GPU blocks: V's
    mirrored entries cross row ranges, K's rows do not; E_t = 40 spans two
    windows.  p1 x p1 row ranges give partial sums that add up to the blocks."""
    import torch

    from paper_2102_09811_b200 import distributed as D
    from paper_2102_09811_b200.assembly import _assemble_operator

    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, E_t)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    E, N = m.n_triangles, m.n_vertices
    for code, (R, C) in (((0, False, False, True), (E, E)), ((1, False, True, False), (E, N))):
        full = _assemble_operator(*code, m, tg, p, Q4, None)
        ranges = [D.block_range(r, world, E_t) for r in range(world)]
        shards = [torch.full((b - a, R, C), float("nan"), dtype=torch.float64, device="cuda") for a, b in ranges]
        table = torch.as_tensor(D.block_pointer_table([(s.data_ptr(), a, b) for s, (a, b) in zip(shards, ranges)],
                                                      E_t, R * C * 8), device="cuda")
        for rows in D.row_partition(D.row_weights(E, code[3]), world):
            _assemble_operator(*code, m, tg, p, Q4, None, d_range=(0, E_t), row_range=rows, block_ptrs=table)
        got = torch.cat(shards)
        assert torch.equal(got, full), code
    # p1 x p1: row ranges give partial sums (added across ranks by a reduce-scatter)
    for op in (2, 0):
        full = _assemble_operator(op, True, True, True, m, tg, p, Q4, None)
        parts = [_assemble_operator(op, True, True, True, m, tg, p, Q4, None, row_range=rows)
                 for rows in D.row_partition(D.row_weights(E, True), world)]
        tot = sum(parts)
        assert torch.allclose(tot, full, rtol=1e-13, atol=1e-13 * full.abs().max()), op
        assert all(torch.equal(t, t.transpose(1, 2)) for t in parts)
    tab_d = torch.as_tensor(D.block_pointer_table([(full.data_ptr(), 0, E_t)], E_t, N * N * 8), device="cuda")
    with pytest.raises(Exception):   # p1 x p1 cannot store through peer pointers
        _assemble_operator(2, True, True, True, m, tg, p, Q4, None, row_range=(0, 10), block_ptrs=tab_d)


@pytest.mark.slow
def test_c5_sampled_rows_vs_reference():
    """BASELINE config 5 (unit cube L5, 12288 triangles, alpha = 1, N = 256)
    on one GPU: V and K assembled in 32-block d-chunks whose edges are window
    edges (distributed.aligned_chunks: one 30-block window per chunk, no
    extra gap slots; 39 / 19 GB per chunk), three sampled rows per block
    compared with the reference's single-row oracle (tests/golden/c5_rows.npz,
    exact values from the quad build).  At d ~ 255 the reference's own V rows
    are up to 2.4e-9 of block max from exact (the -L + 2L - L cancellation);
    the GPU's moment form does not cancel there, so |gpu - ref| ~ eps_ref:
    |gpu - ref| <= gate(eps_ref) and |gpu - exact| <= eps_ref + 1e-13.
    Structural zeros (coplanar K columns) must be exact zeros."""
    import torch

    from paper_2102_09811_b200.assembly import _assemble_operator
    from paper_2102_09811_b200.distributed import aligned_chunks

    g = golden("c5_rows")
    m = hb.unit_cube_mesh(5)
    assert float(m.vertices.sum()) == float(g["mesh_vertices_sum"])
    tg = hb.TimeGrid(1.0, 256)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    rows = torch.as_tensor(g["rows"], device="cuda")
    stride = int(g["col_stride"])
    for op, code in (("V", (0, False, False, True)), ("K", (1, False, True, False))):
        C = m.n_triangles if op == "V" else m.n_vertices
        buf = torch.empty((32, m.n_triangles, C), dtype=torch.float64, device="cuda")
        got = np.empty((256, len(g["rows"]), C))
        for d0, d1 in aligned_chunks(256, 32):
            _assemble_operator(*code, m, tg, p, Q4, None, d_range=(d0, d1), out=buf[: d1 - d0])
            got[d0:d1] = buf[: d1 - d0, rows, :].cpu().numpy()
        del buf
        torch.cuda.empty_cache()
        mx, eps = g[f"{op}_maxabs"], g[f"{op}_eps_ref"]
        gs = got[:, :, ::stride]
        par = np.abs(gs - g[f"{op}_ref"]).max(axis=(1, 2)) / mx
        acc = np.abs(gs - g[f"{op}_exact"]).max(axis=(1, 2)) / mx
        assert np.all(par <= gate(eps)), (op, par.max())
        assert np.all(acc <= ACC[op] * eps + 1e-13), (op, np.max(acc / eps))
        # structural zeros -- exactly zero in the quad build at every d (the
        # coplanar K columns) -- must be exact zeros at every d; the other
        # zeros (far pairs at d <= 5, roundings of the -L + 2L - L second
        # difference) are values and fall under the gates above
        structural = np.all(g[f"{op}_exact"] == 0.0, axis=0)
        assert np.all(gs[:, structural] == 0.0), op
        if op == "K":
            assert structural.sum() > 0


@pytest.mark.slow
def test_c3_sampled_rows_vs_reference():
    """BASELINE config 3 (icosphere L5, 20480 triangles, alpha = 0.5, N = 64):
    V and K assembled in two 32-block d-chunks (the per-rank layout of a
    d-sharded run; 107 / 54 GB per chunk) and three sampled rows compared
    with the reference's single-row oracle (tests/golden/c3_rows.npz, with
    exact values from the quad build).  The reference's own V rows are up to
    6.3e-11 of block max from exact at large d, so the gate is
    gate(eps_ref(d)) and |gpu - exact| <= ACC eps_ref(d) + 1e-13."""
    import torch

    from paper_2102_09811_b200.assembly import _assemble_operator

    g = golden("c3_rows")
    m = hb.generate_icosphere(5)
    assert float(m.vertices.sum()) == float(g["mesh_vertices_sum"])
    tg = hb.TimeGrid(1.0, 64)
    p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
    rows = torch.as_tensor(g["rows"], device="cuda")
    stride = int(g["col_stride"])
    for op, code in (("V", (0, False, False, True)), ("K", (1, False, True, False))):
        C = m.n_triangles if op == "V" else m.n_vertices
        buf = torch.empty((32, m.n_triangles, C), dtype=torch.float64, device="cuda")
        got = np.empty((64, len(g["rows"]), C))
        for d0 in (0, 32):
            _assemble_operator(*code, m, tg, p, Q4, None, d_range=(d0, d0 + 32), out=buf)
            got[d0:d0 + 32] = buf[:, rows, :].cpu().numpy()
        del buf
        torch.cuda.empty_cache()
        mx, eps = g[f"{op}_maxabs"], g[f"{op}_eps_ref"]
        gs = got[:, :, ::stride]
        par = np.abs(gs - g[f"{op}_ref"]).max(axis=(1, 2)) / mx
        acc = np.abs(gs - g[f"{op}_exact"]).max(axis=(1, 2)) / mx
        assert np.all(par <= gate(eps)), (op, par.max())
        assert np.all(acc <= ACC[op] * eps + 1e-13), (op, np.max(acc / eps))
        # no structural zeros on the sphere (no coplanar pairs): the reference's
        # exact zeros at large d are rounding cancellations of -L + 2L - L,
        # covered by the value gate above, not a sparsity pattern


def test_hypersingular_streamed_to_host_matches():
    """assemble_hypersingular(host_out=...) (curl combine in block chunks, each
    chunk copied to page-locked memory as soon as it is formed) equals the
    device result bitwise."""
    import torch

    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    V = hb.assemble_single_layer(m, tg, p, Q4)
    ref = hb.assemble_hypersingular(m, tg, p, Q4, single_layer=V).device_blocks.cpu()
    pin = torch.full(ref.shape, float("nan"), dtype=torch.float64).pin_memory()
    D = hb.assemble_hypersingular(m, tg, p, Q4, single_layer=V, host_out=pin)
    host, ev = D.host_copy
    ev.synchronize()
    assert host.data_ptr() == pin.data_ptr()
    assert torch.equal(host, ref) and torch.equal(D.device_blocks.cpu(), ref)


def test_assemble_all_concurrent_streams_bitwise():
    """assemble_all (V, K, D on three streams, streamed to page-locked host
    memory) equals the sequential public API bitwise."""
    import torch

    from paper_2102_09811_b200 import device as hbdev

    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    V = hb.assemble_single_layer(m, tg, p, Q4).device_blocks.cpu()
    K = hb.assemble_double_layer(m, tg, p, Q4).device_blocks.cpu()
    D = hb.assemble_hypersingular(m, tg, p, Q4).device_blocks.cpu()
    pins = {n: torch.empty(t.shape, dtype=torch.float64).pin_memory() for n, t in (("V", V), ("K", K), ("D", D))}
    hbdev.drop_device_tables(m)   # tables re-uploaded inside assemble_all
    ops = hb.assemble_all(m, tg, p, Q4, host_out=pins)
    for name, ref in (("V", V), ("K", K), ("D", D)):
        host, ev = ops[name].host_copy
        ev.synchronize()
        assert torch.equal(host, ref) and torch.equal(ops[name].device_blocks.cpu(), ref), name


@pytest.mark.parametrize("E_t,orders", [(1, (4, 4)), (2, (4, 4)), (17, (4, 4)), (5, (2, 3)), (5, (6, 5))])
def test_edge_sizes_and_orders_vs_oracle(oracle, E_t, orders):
    """Edge cases against the CPU oracle on the reference's cube-1 mesh: a
    single block (only the i_t = 0 / 1 passes), two blocks, 17 blocks (the
    second 16-slot lane group holds one gap), and other quadrature orders
    (regular/near rules and Duffy grids of other point counts)."""
    m = hb.generate_cube_surface(1)
    tg = hb.TimeGrid(1.0, E_t)
    p = hb.KernelParams(0.8, tg.step, length_scale=m.diameter)
    q = hb.QuadratureConfig(*orders)
    ops = {"V": lambda: hb.assemble_single_layer(m, tg, p, q), "K": lambda: hb.assemble_double_layer(m, tg, p, q),
           "D2": lambda: hb.assemble_hypersingular_d2(m, tg, p, q),
           "V11": lambda: hb.assemble_single_layer(m, tg, p, q, "p1", "p1")}
    for op, fn in ops.items():
        got = fn().blocks
        ref = oracle.assemble(m, tg, p, q, op)
        assert got.shape == ref.shape == (E_t,) + ref.shape[1:]
        assert rel_block_err(got, ref).max() <= 1e-11, (op, rel_block_err(got, ref).max())
        assert np.array_equal(got == 0.0, ref == 0.0), op


@pytest.mark.parametrize("op", ["V", "K"])
def test_host_out_row_slab_streaming_is_bitwise(op):
    """assemble_single_layer / assemble_double_layer(host_out=...): test-row
    slabs assembled into one buffer and streamed to page-locked memory as they
    complete give bitwise the blocks of one call (row ranges write disjoint
    entries; V's mirrored entries of a slab come from earlier slabs)."""
    import torch

    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 12)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    f = hb.assemble_single_layer if op == "V" else hb.assemble_double_layer
    ref = f(m, tg, p).blocks
    pin = torch.full(ref.shape, float("nan"), dtype=torch.float64).pin_memory()   # every entry must be written
    res = f(m, tg, p, host_out=pin)
    res.host_copy[1].synchronize()
    assert np.array_equal(pin.numpy(), ref)
    assert np.array_equal(res.blocks, ref)
    # a d-range streams the same way
    pin2 = torch.full((5,) + ref.shape[1:], float("nan"), dtype=torch.float64).pin_memory()
    f(m, tg, p, d_range=(3, 8), host_out=pin2).host_copy[1].synchronize()
    assert np.array_equal(pin2.numpy(), ref[3:8])

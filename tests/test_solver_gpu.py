"""Block-Toeplitz apply / forward substitution / FGMRES on the device vs
dense expansions and the reference's config-2 Dirichlet solve."""
import numpy as np
import pytest

import paper_2102_09811_b200 as hb
from _hb_util import golden

pytestmark = pytest.mark.gpu


def dense(blocks, E_t, transpose=False, diag=False):
    nb, R, C = blocks.shape
    A = blocks.transpose(0, 2, 1) if transpose else blocks
    r, c = A.shape[1:]
    out = np.zeros((E_t * r, E_t * c))
    for k in range(E_t):
        for i in range(k + 1):
            d = k - i
            if diag and d:
                continue
            out[k * r:(k + 1) * r, i * c:(i + 1) * c] = A[0 if diag else d]
    return out


@pytest.mark.parametrize("R,C,E_t,d_off", [(2100, 300, 40, 0), (2050, 97, 64, 5), (4096, 64, 9, 0),
                                           (1100, 70, 150, 0), (1030, 40, 130, 70)])
def test_apply_toeplitz_tensor_core_path(R, C, E_t, d_off):
    """Operators with >= 1024 rows take the DMMA kernel (k_toep_mma, 64-step
    tiles): blockwise products vs numpy, full and d-range
    (hb_toeplitz_apply_range) forms, histories longer than one step tile."""
    import torch

    from paper_2102_09811_b200 import _native

    rng = np.random.default_rng(R + C)
    nb = E_t - d_off
    B = rng.standard_normal((nb, R, C))
    x = rng.standard_normal((E_t, C))
    ref = np.zeros((E_t, R))
    for k in range(E_t):
        for d in range(d_off, k + 1):
            ref[k] += B[d - d_off] @ x[k - d]
    Bd = torch.as_tensor(B, device="cuda")
    xd = torch.as_tensor(x, device="cuda")
    y = torch.empty((E_t, R), dtype=torch.float64, device="cuda")
    _native.call("hb_toeplitz_apply_range", d_off, nb, R, C, _native.ptr(Bd), 0, E_t, _native.ptr(xd),
                 _native.ptr(y), _native.stream_handle())
    assert np.allclose(y.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    if d_off == 0:
        got = hb.apply_toeplitz(hb.BlockToeplitzMatrix(Bd), xd).cpu().numpy()
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    # transposed blocks (K', D^T): y[k] = sum_d A^d^T x[k - d], output length R -> run with B^T stored
    Bt = torch.as_tensor(np.ascontiguousarray(B.transpose(0, 2, 1)), device="cuda")   # (nb, C, R)
    yt = torch.empty((E_t, R), dtype=torch.float64, device="cuda")
    _native.call("hb_toeplitz_apply_range", d_off, nb, C, R, _native.ptr(Bt), 1, E_t, _native.ptr(xd),
                 _native.ptr(yt), _native.stream_handle())
    assert np.allclose(yt.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("R,C,E_t", [(7, 7, 5), (20, 11, 9), (64, 40, 33)])
def test_apply_toeplitz_vs_dense(R, C, E_t):
    rng = np.random.default_rng(R)
    B = rng.standard_normal((E_t, R, C))
    M = hb.BlockToeplitzMatrix(B)
    x = rng.standard_normal((E_t, C))
    y = hb.apply_toeplitz(M, x)
    ref = (dense(B, E_t) @ x.ravel()).reshape(E_t, R)
    assert np.allclose(y, ref, rtol=1e-13, atol=1e-12)
    xt = rng.standard_normal((E_t, R))
    yt = hb.apply_toeplitz(M, xt, transpose_blocks=True)
    assert np.allclose(yt, (dense(B, E_t, True) @ xt.ravel()).reshape(E_t, C), rtol=1e-13, atol=1e-12)
    assert np.array_equal(hb.apply_toeplitz(M.transposed(), xt), yt)
    assert np.array_equal(hb.apply_toeplitz(M.transposed(), x, transpose_blocks=True), y)
    Mass = hb.BlockToeplitzMatrix(B[:1], diagonal_only=True)
    assert np.allclose(hb.apply_toeplitz(Mass, x), (dense(B[:1], E_t, diag=True) @ x.ravel()).reshape(E_t, R))


def test_forward_block_solve_exact():
    rng = np.random.default_rng(1)
    E_t, n = 12, 30
    B = 0.1 * rng.standard_normal((E_t, n, n))
    B[0] += 4 * np.eye(n)
    M = hb.BlockToeplitzMatrix(B)
    rhs = rng.standard_normal((E_t, n))
    x = hb.forward_block_solve(M, rhs)
    assert np.allclose(hb.apply_toeplitz(M, x), rhs, rtol=1e-12, atol=1e-12)
    xt = hb.forward_block_solve(M, rhs, transpose_blocks=True)
    assert np.allclose(hb.apply_toeplitz(M, xt, transpose_blocks=True), rhs, rtol=1e-12, atol=1e-12)


def test_fgmres_identity_and_nonconvergence():
    rng = np.random.default_rng(2)
    b = rng.standard_normal((4, 5))
    x, rep = hb.fgmres(lambda v: v, b, rel_tol=1e-12)
    assert rep.converged and np.allclose(x, b)
    A = rng.standard_normal((20, 20))
    x, rep = hb.fgmres(lambda v: A @ v, rng.standard_normal(20), rel_tol=1e-14, max_iter=3, restart=2)
    assert not rep.converged and rep.iterations == 3


def test_c2_dirichlet_solve_vs_reference():
    """BASELINE config 2 solve: rhs = 1/2 M g + K g with g the X10 projection
    of G(x - y0, t + 0.1); FGMRES(V) with forward substitution, tol 1e-10."""
    g = golden("solve_c2")
    m = hb.unit_cube_mesh(3)
    tg = hb.TimeGrid(1.0, 32)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    V = hb.assemble_single_layer(m, tg, p)
    K = hb.assemble_double_layer(m, tg, p)
    Mm = hb.assemble_mass(m, tg)
    y0 = np.array([1.5, 1.5, 1.5])
    data = hb.project_to_space(lambda x, t, n=None: hb.fundamental(np.asarray(x) - y0, t + 0.1, 1.0), m, tg, "X10")
    assert np.allclose(data, g["g"], rtol=1e-13, atol=1e-16)
    rhs = 0.5 * hb.apply_toeplitz(Mm, data) + hb.apply_toeplitz(K, data)
    assert np.max(np.abs(rhs - g["rhs"])) <= 1e-10 * np.abs(g["rhs"]).max()
    x, rep = hb.fgmres(hb.toeplitz_operator(V), rhs, rel_tol=1e-10,
                       right_precond=lambda v: hb.forward_block_solve(V, v))
    assert rep.converged and rep.residual <= 1e-10
    assert np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]) <= 1e-9
    xf = hb.forward_block_solve(V, rhs)
    assert np.linalg.norm(xf - g["x_fwd"]) / np.linalg.norm(g["x_fwd"]) <= 1e-9
    Vx = hb.apply_toeplitz(V, g["probe_x"])
    assert np.max(np.abs(Vx - g["probe_Vx"])) <= 1e-10 * np.abs(g["probe_Vx"]).max()
    KTx = hb.apply_toeplitz(K, g["probe_x"][:, :m.n_triangles], True)
    assert np.max(np.abs(KTx - g["probe_KTx"])) <= 1e-10 * np.abs(g["probe_KTx"]).max()


def test_c1_neumann_solve_vs_reference():
    """Neumann path: rhs = 1/2 M'h - K'h (blockwise
    transposes, shared storage), D = T^T (a^2 V) T + D2, FGMRES with forward
    substitution on D -- as heatbem/study.py:104-136."""
    g = golden("neumann_c1")
    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    y0 = np.array([1.5, 1.5, 1.5])
    h = hb.project_to_space(lambda x, t, n: hb.grad_fundamental_normal(np.asarray(x) - y0, n, t + 0.1, 1.0),
                            m, tg, "X00")
    assert np.allclose(h, g["h"], rtol=1e-13, atol=1e-16 * np.abs(g["h"]).max())
    Mm = hb.assemble_mass(m, tg)
    K = hb.assemble_double_layer(m, tg, p)
    rhs = 0.5 * hb.apply_toeplitz(Mm.transposed(), h) - hb.apply_toeplitz(K.transposed(), h)
    assert np.max(np.abs(rhs - g["rhs"])) <= 1e-10 * np.abs(g["rhs"]).max()
    D = hb.assemble_hypersingular(m, tg, p)
    x, rep = hb.fgmres(hb.toeplitz_operator(D), rhs, rel_tol=1e-10,
                       right_precond=lambda v: hb.forward_block_solve(D, v))
    assert rep.converged and rep.residual <= 1e-10
    assert np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]) <= 1e-8


def test_apply_assembled_and_streamed_file(tmp_path):
    """Apply-and-discard: A x from d-chunks that are assembled,
    applied and discarded equals the product with the stored operator (the
    chunk partial sums are added in chunk order: rounding-level differences),
    for V, K, K' and D; the chunks streamed to an HBTM1 file read back
    (memory-mapped) bitwise equal to the stored blocks."""
    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(5)
    E, N = m.n_triangles, m.n_vertices
    full = {"V": hb.assemble_single_layer(m, tg, p), "K": hb.assemble_double_layer(m, tg, p),
            "D": hb.assemble_hypersingular(m, tg, p)}
    for op, tr, n_in in (("V", False, E), ("K", False, N), ("K", True, E), ("D", False, N)):
        x = rng.standard_normal((16, n_in))
        ref = hb.apply_toeplitz(full[op], x, transpose_blocks=tr)
        path = tmp_path / f"{op}{int(tr)}.hbtm"
        B = full[op].blocks
        with hb.BlockFileWriter(path, *B.shape) as w:
            got = hb.apply_assembled(op, m, tg, p, x, transpose_blocks=tr, chunk_blocks=5, writer=w)
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max()), op
        mm = hb.load_blocks(path, mmap=True).blocks
        assert np.array_equal(np.asarray(mm), B), op


@pytest.mark.parametrize("world", [1, 3])
def test_row_sharded_kernels_bitwise(world):
    """RowShardedToeplitz per-rank kernels on one GPU: the row pieces of
    `world` emulated ranks, concatenated as the all-gather would, equal
    apply_toeplitz / forward_block_solve bitwise (same per-row sums); with no
    process group the operator itself runs as world 1."""
    import torch

    from paper_2102_09811_b200 import distributed as D

    rng = np.random.default_rng(world)
    E_t, n = 24, 101
    B = 0.1 * rng.standard_normal((E_t, n, n))
    B[0] += 4 * np.eye(n)
    M = hb.BlockToeplitzMatrix(B)
    x = torch.as_tensor(rng.standard_normal((E_t, n)), device="cuda")
    rhs = torch.as_tensor(rng.standard_normal((E_t, n)), device="cuda")
    Bd = M.device_blocks
    shards = [D.RowShardedToeplitz(Bd[:, a:b].contiguous(), a, b, n)
              for a, b in (D.block_range(r, world, n) for r in range(world))]
    y = torch.cat([s.local_apply(x) for s in shards], dim=1)
    assert torch.equal(y, hb.apply_toeplitz(M, x))
    inv = torch.linalg.inv(Bd[0]).contiguous()
    xs = torch.zeros_like(rhs)
    for k0 in range(0, E_t, D.FORWARD_TILE):   # the step tiles of the blocked substitution
        nk = min(D.FORWARD_TILE, E_t - k0)
        H = [s.local_history_far(xs, k0, nk) for s in shards] if k0 else None
        for k in range(k0, k0 + nk):
            h = (torch.cat([s.local_history(xs, k, k0, H[i][k - k0] if H else None) for i, s in enumerate(shards)])
                 if k else None)
            xs[k] = shards[0].inv_apply(inv, rhs[k], h)
    assert torch.equal(xs, hb.forward_block_solve(M, rhs))
    if world == 1:
        assert torch.equal(shards[0].apply(x), y)
        assert torch.equal(shards[0].forward_solve(rhs), xs)
        xr, rep = shards[0].solve(rhs, rel_tol=1e-12)
        xf, rep1 = hb.fgmres(hb.toeplitz_operator(M), rhs, rel_tol=1e-12,
                             right_precond=lambda v: hb.forward_block_solve(M, v))
        assert rep.converged and torch.equal(torch.as_tensor(xr), torch.as_tensor(xf))


def test_host_edits_reach_device_and_drop_cached_inverse():
    """Reference idiom (assembly.py:328-333): edit .blocks in place, then
    apply_toeplitz / forward_block_solve must see the edited operator --
    including a new (A^0)^-1 after A^0 itself changed -- and so must the
    blockwise-transposed twin; assigning .blocks and overwrite_d2 likewise."""
    rng = np.random.default_rng(11)
    n, nb = 6, 4
    B = rng.standard_normal((nb, n, n)) * 0.1
    B[0] += 4.0 * np.eye(n)
    M = hb.BlockToeplitzMatrix(B.copy())
    Mt = M.transposed()
    x = rng.standard_normal((nb, n))
    hb.forward_block_solve(M, x)                    # caches (A^0)^-1 and puts the blocks on the device
    hb.apply_toeplitz(Mt, x)
    out = M.blocks
    out[0] += 2.0 * np.eye(n)                       # edit A^0 in place
    out[2] *= -1.0
    Bn = np.asarray(out).copy()
    assert np.allclose(hb.apply_toeplitz(M, x), _dense_apply(Bn, x), rtol=1e-12, atol=1e-12)
    assert np.allclose(hb.apply_toeplitz(Mt, x), _dense_apply(np.transpose(Bn, (0, 2, 1)), x), rtol=1e-12, atol=1e-12)
    y = hb.forward_block_solve(M, x)
    assert np.allclose(_dense_apply(Bn, y), x, rtol=1e-10, atol=1e-10)
    M.blocks = B.copy()                             # assignment replaces both sides
    y = hb.forward_block_solve(M, x)
    assert np.allclose(_dense_apply(B, y), x, rtol=1e-10, atol=1e-10)


def _dense_apply(blocks, x):
    nb = blocks.shape[0]
    y = np.zeros((x.shape[0], blocks.shape[1]))
    for k in range(x.shape[0]):
        for d in range(min(k + 1, nb)):
            y[k] += blocks[d] @ x[k - d]
    return y

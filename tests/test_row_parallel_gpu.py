"""Row-parallel assembly across PROCESSES on one GPU: two gloo ranks, both on
cuda:0, exchange their d-shards by CUDA IPC (hb_ipc_export / hb_ipc_import),
each evaluates its test-row range for all blocks and stores through the
shared block-pointer table into both shards.  The ranks only meet at host
barriers (no kernel waits on another rank's kernel).  The gathered shards must
be bitwise the 1-GPU blocks -- this is distributed.assemble_row_parallel, the
N-GPU path, with the peer memory living on the same device."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_2102_09811_b200 as hb
    from paper_2102_09811_b200 import distributed as D

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m = hb.unit_cube_mesh(2)
        tg = hb.TimeGrid(1.0, 16)
        p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
        q = hb.QuadratureConfig()
        res = {}
        for name, code in (("V", (0, False, False, True)), ("K", (1, False, True, False))):
            S = D.assemble_row_parallel(*code, m, tg, p, q)
            res[name] = (S.d0, S.d1, S.local.cpu().numpy())
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_row_parallel_two_processes_ipc():
    import torch
    import torch.multiprocessing as mp

    import paper_2102_09811_b200 as hb
    from paper_2102_09811_b200.assembly import _assemble_operator

    world = 2
    out = mp.get_context("spawn").Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    q = hb.QuadratureConfig()
    for name, code in (("V", (0, False, False, True)), ("K", (1, False, True, False))):
        full = _assemble_operator(*code, m, tg, p, q, None).cpu().numpy()
        got = np.concatenate([out[r][name][2] for r in range(world)])
        assert [out[r][name][:2] for r in range(world)] == [(0, 8), (8, 16)]
        assert np.array_equal(got, full), name
    torch.cuda.synchronize()


def _solve_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_2102_09811_b200 as hb
    from paper_2102_09811_b200 import distributed as D

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m = hb.unit_cube_mesh(3)
        tg = hb.TimeGrid(1.0, 32)
        p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
        datum = hb.HeatKernelDatum((1.5, 1.5, 1.5), 1.0, 0.1)
        x, rep, V = D.dirichlet_solve_row_sharded(m, tg, p, hb.QuadratureConfig(), datum, rel_tol=1e-10)
        K = D.assemble_row_sharded(1, False, True, False, m, tg, p, hb.QuadratureConfig())
        out[rank] = {"x": x.cpu().numpy(), "res": rep.residual, "conv": rep.converged, "rows": (V.r0, V.r1),
                     "V": V.local.cpu().numpy(), "K": K.local.cpu().numpy()}
    finally:
        dist.destroy_process_group()


def test_row_sharded_dirichlet_solve_three_processes():
    """BASELINE config-2 Dirichlet problem on three ranks (one GPU, CUDA IPC,
    gloo): V and K row shards filled by peer stores from balanced work rows
    are bitwise the rows of the 1-GPU blocks; the solve (rhs all-gather, one
    density all-gather per matvec, forward substitution with per-step
    history all-gathers) converges to the reference's solution."""
    import torch.multiprocessing as mp

    import paper_2102_09811_b200 as hb
    from paper_2102_09811_b200.assembly import _assemble_operator
    from _hb_util import golden

    world = 3
    out = mp.get_context("spawn").Manager().dict()
    mp.start_processes(_solve_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    m = hb.unit_cube_mesh(3)
    tg = hb.TimeGrid(1.0, 32)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    q = hb.QuadratureConfig()
    assert [out[r]["rows"] for r in range(world)] == [(0, 256), (256, 512), (512, 768)]
    for name, code in (("V", (0, False, False, True)), ("K", (1, False, True, False))):
        full = _assemble_operator(*code, m, tg, p, q, None).cpu().numpy()
        got = np.concatenate([out[r][name] for r in range(world)], axis=1)
        assert np.array_equal(got, full), name
    g = golden("solve_c2")
    for r in range(world):
        assert out[r]["conv"] and out[r]["res"] <= 1e-10
        assert np.array_equal(out[r]["x"], out[0]["x"])          # replicated iterates
    assert np.linalg.norm(out[0]["x"] - g["x"]) / np.linalg.norm(g["x"]) <= 1e-9


def _d_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_2102_09811_b200 as hb
    from paper_2102_09811_b200 import distributed as D
    from paper_2102_09811_b200.assembly import _assemble_operator

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m = hb.unit_cube_mesh(2)
        tg = hb.TimeGrid(1.0, 16)
        p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
        q = hb.QuadratureConfig()
        d0, d1 = D.block_range(rank, world, 16)
        V = _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(d0, d1))
        Dl = D.hypersingular_rows_peer(m, tg, p, q, V, d0, d1)
        out[rank] = (d0, d1, Dl.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_hypersingular_rows_peer_three_processes():
    """D2 split by element rows over three ranks, the partials read over peer
    memory (CUDA IPC on one device) and summed inside the curl kernel of each
    rank's blocks: D equals the 1-GPU D to rounding and is exactly symmetric."""
    import torch.multiprocessing as mp

    import paper_2102_09811_b200 as hb

    world = 3
    out = mp.get_context("spawn").Manager().dict()
    mp.start_processes(_d_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 16)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    q = hb.QuadratureConfig()
    V = hb.assemble_single_layer(m, tg, p, q)
    ref = hb.hypersingular_from_single_layer(V, hb.assemble_hypersingular_d2(m, tg, p, q), m, p).blocks
    got = np.concatenate([out[r][2] for r in range(world)])
    assert [out[r][:2] for r in range(world)] == [(0, 6), (6, 11), (11, 16)]
    for d in range(16):
        assert np.array_equal(got[d], got[d].T)
        assert np.abs(got[d] - ref[d]).max() <= 1e-13 * np.abs(ref[d]).max(), d

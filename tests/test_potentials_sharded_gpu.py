"""Point-sharded representation formula (distributed.represent_grid_sharded,
SURVEY 8(e)): two gloo ranks on cuda:0 each evaluate half of the points and
all-gather; the result must be bitwise the 1-GPU represent_grid."""
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


def _problem():
    import paper_2102_09811_b200 as hb

    m = hb.unit_cube_mesh(2)
    tg = hb.TimeGrid(1.0, 12)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    rng = np.random.default_rng(5)
    q = rng.uniform(-1, 1, (12, m.n_triangles))
    g = rng.uniform(-1, 1, (12, m.n_vertices))
    X = rng.uniform(0.05, 0.95, (301, 3))
    return hb, m, tg, p, q, g, X


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2102_09811_b200 import distributed as D

    hb, m, tg, p, q, g, X = _problem()
    res = D.represent_grid_sharded(q, g, X, m, tg, p)
    local, (p0, p1) = D.represent_grid_sharded(q, g, X, m, tg, p, gather=False)
    if rank == 0:
        np.save(out, res.cpu().numpy())
    assert local.shape[0] == p1 - p0
    dist.barrier()
    dist.destroy_process_group()


def test_point_sharded_representation_bitwise(tmp_path):
    import torch.multiprocessing as mp

    hb, m, tg, p, q, g, X = _problem()
    ref = hb.represent_grid(q, g, X, m, tg, p)
    out = str(tmp_path / "u.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert np.array_equal(np.load(out), ref)

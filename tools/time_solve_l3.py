"""Solver components at study level 3 (cube, 12288 triangles, 64 steps;
V = 77 GB): (A^0)^{-1}, Toeplitz matvec, forward substitution, FGMRES."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.solver import _inverse
m = hb.generate_cube_surface(32, 1.0); tg = hb.TimeGrid(1.0, 64)
p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
V = hb.assemble_single_layer(m, tg, p)
rhs = torch.randn((64, m.n_triangles), dtype=torch.float64, device="cuda")
def ev(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
t0 = time.perf_counter(); V._inv_cache = {}; _inverse(V, False); torch.cuda.synchronize(); t_inv = time.perf_counter() - t0
res = {"inverse_s": t_inv, "matvec_ms": ev(lambda: hb.apply_toeplitz(V, rhs)),
       "forward_subst_ms": ev(lambda: hb.forward_block_solve(V, rhs)),
       "fgmres_ms": ev(lambda: hb.fgmres(hb.toeplitz_operator(V), rhs, rel_tol=1e-8,
                                         right_precond=lambda v: hb.forward_block_solve(V, v)), reps=1),
       "block_GB": V.device_blocks.numel() * 8 / 1e9}
print(json.dumps(res))

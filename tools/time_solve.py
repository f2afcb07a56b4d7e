"""Config-2 Dirichlet solve on the device: Toeplitz matvec, forward
substitution (the preconditioner) and the full FGMRES solve, CUDA-event timed
(device-resident torch vectors, as the solver keeps them)."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
V = hb.assemble_single_layer(m, tg, p)
K = hb.assemble_double_layer(m, tg, p)
Mm = hb.assemble_mass(m, tg)
y0 = np.array([1.5, 1.5, 1.5])
data = hb.project_to_space(lambda x, t, n=None: hb.fundamental(np.asarray(x) - y0, t + 0.1, 1.0), m, tg, "X10")
rhs = torch.as_tensor(0.5 * hb.apply_toeplitz(Mm, data) + hb.apply_toeplitz(K, data), device="cuda")
def timed(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): r = fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, r
ms_mv, _ = timed(lambda: hb.apply_toeplitz(V, rhs))
ms_fs, _ = timed(lambda: hb.forward_block_solve(V, rhs))
info = {}
def solve():
    x, rep = hb.fgmres(hb.toeplitz_operator(V), rhs, rel_tol=1e-10, right_precond=lambda v: hb.forward_block_solve(V, v))
    info["it"], info["res"] = rep.iterations, rep.residual
    return x
ms_solve, _ = timed(solve, reps=3)
print(json.dumps({"config": "c2 (768 x 32 unknowns)", "matvec_ms": ms_mv, "forward_subst_ms": ms_fs,
                  "fgmres_ms": ms_solve, "iterations": info["it"], "residual": info["res"],
                  "reference_survey_s": {"matvec": 0.061, "forward_subst": 0.349}}))

"""One blocked forward substitution at config 2 (for an ncu launch list)."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
V = hb.assemble_single_layer(m, tg, p)
rhs = torch.randn((32, m.n_triangles), dtype=torch.float64, device="cuda")
hb.forward_block_solve(V, rhs)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("solve")
hb.forward_block_solve(V, rhs)
torch.cuda.synchronize()
print("ok")

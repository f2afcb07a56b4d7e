"""k_toep_mma on the study level-3 single layer (12288 rows, 64 blocks) for ncu:
one matvec after a warm-up."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
m = hb.generate_cube_surface(32, 1.0); tg = hb.TimeGrid(1.0, 64)
p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
V = hb.assemble_single_layer(m, tg, p)
x = torch.randn((64, m.n_triangles), dtype=torch.float64, device="cuda")
hb.apply_toeplitz(V, x); torch.cuda.synchronize()
y = hb.apply_toeplitz(V, x); torch.cuda.synchronize()
print("done", float(y.norm()))

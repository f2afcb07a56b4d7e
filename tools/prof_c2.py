import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2102_09811_b200 as hb
mesh = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=mesh.diameter)
for it in range(2):
    V = hb.assemble_single_layer(mesh, tg, p)
    K = hb.assemble_double_layer(mesh, tg, p)
    D2 = hb.assemble_hypersingular_d2(mesh, tg, p)
    D = hb.hypersingular_from_single_layer(V, D2, mesh, p, overwrite_d2=True)
    torch.cuda.synchronize()
print("done")

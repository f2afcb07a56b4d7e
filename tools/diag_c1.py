import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2102_09811_b200 as hb
from oracle import oracle as O
mesh = hb.unit_cube_mesh(2); tg = hb.TimeGrid(1.0, 16); p = hb.KernelParams(1.0, tg.step, length_scale=mesh.diameter); q = hb.QuadratureConfig()
V = hb.assemble_single_layer(mesh, tg, p, q); D2 = hb.assemble_hypersingular_d2(mesh, tg, p, q)
Vr = O.assemble(mesh, tg, p, q, "V"); D2r = O.assemble(mesh, tg, p, q, "D2")
G = V.blocks
for d in range(16):
    m = np.abs(Vr[d]).max(); e = np.abs(G[d]-Vr[d]); i = np.unravel_index(np.argmax(e), e.shape)
    print(f"V d={d:2d} max={m:.3e} rel={e.max()/m:.3e} at {i} val={Vr[d][i]:.3e}")
D = hb.hypersingular_from_single_layer(V, D2, mesh, p).blocks
Dr = O.curl_combine(Vr, D2r, mesh, 1.0)
Dmix = O.curl_combine(G, D2r, mesh, 1.0)   # GPU V through the reference's scipy curl
for d in range(16):
    m = np.abs(Dr[d]).max()
    print(f"D d={d:2d} max={m:.3e} rel(gpu)={np.abs(D[d]-Dr[d]).max()/m:.3e} rel(gpuV+scipy)={np.abs(Dmix[d]-Dr[d]).max()/m:.3e} rel(gpu vs gpuV+scipy)={np.abs(D[d]-Dmix[d]).max()/m:.3e}")

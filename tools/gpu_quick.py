import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2102_09811_b200 as hb
from oracle import oracle as O
def rel(a, b):
    out = []
    for d in range(b.shape[0]):
        m = np.max(np.abs(b[d])); out.append(np.max(np.abs(a[d]-b[d]))/m if m>0 else np.max(np.abs(a[d])))
    return max(out)
res = {}
for name, mesh, Et, alpha in [("cube1", hb.generate_cube_surface(1), 4, 0.5), ("cube2", hb.generate_cube_surface(2), 4, 0.7),
                              ("c1", hb.unit_cube_mesh(2), 16, 1.0), ("c2s", hb.unit_cube_mesh(3), 8, 1.0)]:
    tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(alpha, tg.step, length_scale=mesh.diameter); q = hb.QuadratureConfig()
    for op, fn in [("V", lambda: hb.assemble_single_layer(mesh, tg, p, q)),
                   ("K", lambda: hb.assemble_double_layer(mesh, tg, p, q)),
                   ("D2", lambda: hb.assemble_hypersingular_d2(mesh, tg, p, q)),
                   ("V11", lambda: hb.assemble_single_layer(mesh, tg, p, q, "p1", "p1"))]:
        if name == "c2s" and op in ("V11", "D2"): continue
        try:
            G = fn().blocks
        except Exception as ex:
            print(name, op, "ERROR", ex); continue
        R = O.assemble(mesh, tg, p, q, op)
        zero_ok = np.array_equal(G == 0, R == 0)
        sym = all(np.array_equal(G[d], G[d].T) for d in range(Et)) if op != "K" else None
        print(f"{name:6s} {op:4s} rel={rel(G, R):.3e} zeros_equal={zero_ok} sym={sym}", flush=True)
    if name in ("cube1","cube2","c1"):
        V = hb.assemble_single_layer(mesh, tg, p, q); D2 = hb.assemble_hypersingular_d2(mesh, tg, p, q)
        D = hb.hypersingular_from_single_layer(V, D2, mesh, p).blocks
        Dr = O.curl_combine(O.assemble(mesh, tg, p, q, "V"), O.assemble(mesh, tg, p, q, "D2"), mesh, alpha)
        print(f"{name:6s} D    rel={rel(D, Dr):.3e} sym={all(np.array_equal(D[d], D[d].T) for d in range(Et))}")
# timing c2 V
mesh = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=mesh.diameter)
for op, fn in [("V", lambda: hb.assemble_single_layer(mesh, tg, p)), ("K", lambda: hb.assemble_double_layer(mesh, tg, p)),
               ("D2", lambda: hb.assemble_hypersingular_d2(mesh, tg, p))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); 
    for _ in range(3): B = fn()
    torch.cuda.synchronize(); dt = (time.perf_counter()-t)/3
    n = B.device_blocks.numel()
    print(f"c2 {op}: {dt*1e3:.2f} ms  {n/dt/1e9:.3f} G entries/s")

import sys, os, numpy as np
R = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import paper_2102_09811_b200 as hb
from _hb_util import golden
g, ex = golden("c2"), golden("exact")
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
V = hb.assemble_single_layer(m, tg, p); K = hb.assemble_double_layer(m, tg, p); D2 = hb.assemble_hypersingular_d2(m, tg, p)
D = hb.hypersingular_from_single_layer(V, D2, m, p)
for op, M in (("V", V), ("K", K), ("D", D)):
    B = M.blocks; rows = g["rows_p0"] if op in ("V", "K") else g["rows_p1"]; bmax = g[f"{op}_maxabs"]
    acc = np.abs(B[:, rows, :] - ex[f"c2_{op}_exact_rows"]).max(axis=(1, 2)) / bmax
    eps = ex[f"c2_{op}_eps_ref"]
    par = np.abs(B[:, rows, :] - g[f"{op}_rows"]).max(axis=(1, 2)) / bmax
    print(op, "gpu-exact max %.2e ref-exact max %.2e | max ratio acc/eps %.2f at d=%d | par/eps max %.2f | max (acc - 2 eps) %.2e" % (
        acc.max(), eps.max(), np.max(acc / eps), np.argmax(acc / eps), np.max(par / eps), np.max(acc - 2 * eps)))

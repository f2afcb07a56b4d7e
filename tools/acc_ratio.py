import sys, os, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import paper_2102_09811_b200 as hb
from _hb_util import golden
g, ex = golden("c1"), golden("exact")
m = hb.unit_cube_mesh(2); tg = hb.TimeGrid(1.0, 16); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
ops = {"V": hb.assemble_single_layer(m, tg, p), "K": hb.assemble_double_layer(m, tg, p), "D2": hb.assemble_hypersingular_d2(m, tg, p),
       "V11": hb.assemble_single_layer(m, tg, p, hb.QuadratureConfig(), "p1", "p1")}
ops["D"] = hb.hypersingular_from_single_layer(ops["V"], ops["D2"], m, p)
for op, M in ops.items():
    B = M.blocks
    rows = g["rows_p0"] if op in ("V", "K") else g["rows_p1"]
    bmax = g[f"{op}_maxabs"]
    acc = np.abs(B[:, rows, :] - ex[f"c1_{op}_exact_rows"]).max(axis=(1, 2)) / bmax
    refrows = np.abs(g[f"{op}_rows"] - ex[f"c1_{op}_exact_rows"]).max(axis=(1, 2)) / bmax
    par = np.abs(B[:, rows, :] - g[f"{op}_rows"]).max(axis=(1, 2)) / bmax
    print(op, "gpu/exact (rows) max %.2e | ref/exact(rows) max %.2e | eps_ref(full) max %.2e | ratio acc/eps_ref_rows max %.2f | par/eps_ref %.2f" % (
        acc.max(), refrows.max(), ex[f"c1_{op}_eps_ref"].max(), np.max(acc / np.maximum(refrows, 1e-16)), np.max(par / ex[f"c1_{op}_eps_ref"])))

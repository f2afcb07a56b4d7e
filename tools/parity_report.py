"""Per-op, per-config, per-block parity report of the GPU assembly.

    python tools/parity_report.py [out.json]

For every operator of BASELINE configs 1 and 2 (golden sample rows of the
reference, tests/golden/c1.npz / c2.npz, and their exact values from the
quad-precision oracle, tests/golden/exact.npz) and every block d:
  par(d) = max |gpu - ref|   / max |ref_d|
  acc(d) = max |gpu - exact| / max |ref_d|
  eps(d) = the reference's own max |ref - exact| / max |ref_d| (eps_ref)
Prints a table and writes the numbers as JSON (profiles/ keeps the committed copy).
"""
import json
import os
import sys

import numpy as np

R = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R)
sys.path.insert(0, os.path.join(R, "tests"))
import paper_2102_09811_b200 as hb  # noqa: E402
from _hb_util import golden  # noqa: E402


def ops_for(level, Et):
    m = hb.unit_cube_mesh(level)
    tg = hb.TimeGrid(1.0, Et)
    p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    V = hb.assemble_single_layer(m, tg, p)
    out = {"V": V, "K": hb.assemble_double_layer(m, tg, p)}
    D2 = hb.assemble_hypersingular_d2(m, tg, p)
    out["D2"] = D2
    out["V11"] = hb.assemble_single_layer(m, tg, p, hb.QuadratureConfig(), "p1", "p1")
    out["D"] = hb.hypersingular_from_single_layer(V, D2, m, p)
    return out


def main():
    ex = golden("exact")
    report = {}
    for cfg, level, Et in (("c1", 2, 16), ("c2", 3, 32)):
        g = golden(cfg)
        ops = ops_for(level, Et)
        for op, M in ops.items():
            key = f"{cfg}_{op}_exact_rows"
            B = M.blocks
            rows = g["rows_p0"] if op in ("V", "K") else g["rows_p1"]
            bmax = g[f"{op}_maxabs"]
            par = np.abs(B[:, rows, :] - g[f"{op}_rows"]).max(axis=(1, 2)) / bmax
            ent = {"par": par.tolist()}
            if key in ex.files:
                exr = ex[key]
                acc = np.abs(B[:, rows, :] - exr).max(axis=(1, 2)) / bmax
                eps_rows = np.abs(g[f"{op}_rows"] - exr).max(axis=(1, 2)) / bmax
                ent.update(acc=acc.tolist(), eps_ref=ex[f"{cfg}_{op}_eps_ref"].tolist(), eps_ref_rows=eps_rows.tolist())
            report[f"{cfg}_{op}"] = ent
            print(f"== {cfg} {op}")
            for d in range(len(par)):
                line = f"  d={d:3d} par {par[d]:.2e}"
                if "acc" in ent:
                    line += (f"  acc {ent['acc'][d]:.2e}  eps_ref {ent['eps_ref'][d]:.2e}  "
                             f"acc/eps_rows {ent['acc'][d] / max(ent['eps_ref_rows'][d], 1e-300):.2f}")
                print(line)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            json.dump(report, fh, indent=1)


if __name__ == "__main__":
    main()

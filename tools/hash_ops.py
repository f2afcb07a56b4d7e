import os, sys, hashlib, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
for lvl, Et, a in ((3, 32, 1.0), (2, 64, 0.5)):
    m = hb.unit_cube_mesh(lvl); tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(a, tg.step, length_scale=m.diameter)
    for name, fn in (("V", hb.assemble_single_layer), ("K", hb.assemble_double_layer), ("D2", hb.assemble_hypersingular_d2)):
        B = fn(m, tg, p).blocks
        print(lvl, name, hashlib.sha256(B.tobytes()).hexdigest()[:16])

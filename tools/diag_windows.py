import sys, os, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
m = hb.generate_cube_surface(2); tg = hb.TimeGrid(1.0, 80); p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
for name, fn in (("V", hb.assemble_single_layer), ("K", hb.assemble_double_layer), ("D2", hb.assemble_hypersingular_d2)):
    full = fn(m, tg, p).blocks
    for a, b in ((0, 3), (3, 41), (41, 80), (1, 5), (32, 40)):
        part = fn(m, tg, p, d_range=(a, b)).blocks
        diff = [d for d in range(a, b) if not np.array_equal(part[d - a], full[d])]
        if diff:
            d = diff[0]
            x = np.abs(part[d - a] - full[d]); i = np.unravel_index(np.argmax(x), x.shape)
            print(name, (a, b), "differing blocks", diff[:10], "max rel", x.max() / np.abs(full[d]).max(), "at", i)
        else:
            print(name, (a, b), "ok")

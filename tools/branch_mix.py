"""Warp-level branch mix of the pair kernels (diagnostics build with
-DHB_COUNT_BRANCHES, loaded via HB_LIB_PATH): fraction of eval_n calls whose
warp needed only the small-x series, only the large-x branch, or both."""
import ctypes, json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import _native
from paper_2102_09811_b200.assembly import _assemble_operator
L = _native.load()
f = L.hb_debug_branch_counts
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
lvl, Et, alpha = int(os.environ.get("LVL", "3")), int(os.environ.get("ET", "32")), float(os.environ.get("ALPHA", "1"))
m = hb.unit_cube_mesh(lvl); tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(alpha, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig()
res = {}
for name, code in (("V", (0, False, False, True)), ("K", (1, False, True, False))):
    buf = (ctypes.c_ulonglong * 4)()
    f(buf, 1)
    _assemble_operator(*code, m, tg, p, q, None, d_range=(0, min(Et, 32)))
    torch.cuda.synchronize()
    f(buf, 1)
    tot = sum(buf[1:]) or 1
    res[name + "_raw"] = list(buf)
    res[name] = {"small_only": buf[1] / tot, "large_only": buf[2] / tot, "both": buf[3] / tot, "calls": tot}
print(json.dumps(res))

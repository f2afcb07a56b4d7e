"""Per-rank work of bench.py --config 5 (d-sharded: rank r assembles blocks
block_range(r, N, 256) of V, K and D = D2 + curl(V)), timed one rank at a time
on one B200: the max over ranks is the N-GPU step (no collective in the
assembly).  Shows the load balance of the d split: with the moment form the
low blocks (per-point gaps below each pair's moment block) cost more than the
high ones."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev, distributed as D
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
m = hb.unit_cube_mesh(int(os.environ.get("LVL", "5"))); Et = int(os.environ.get("ET", "256"))
tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter); q = hb.QuadratureConfig()
E, N = m.n_triangles, m.n_vertices
tabs = hbdev.device_tables(m, q)
world = int(os.environ.get("WORLD", "8"))
split = os.environ.get("SPLIT", "block_range")
CH = 32
bufV = torch.empty((CH, E, E), dtype=torch.float64, device="cuda")
bufK = torch.empty((CH, E, N), dtype=torch.float64, device="cuda")
bufD = torch.empty((CH, N, N), dtype=torch.float64, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
def timed(fn):
    s, e = ev(), ev(); s.record(); fn(); e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)
ranges = [D.block_range(r, world, Et) for r in range(world)] if split == "block_range" else \
    D.balanced_block_ranges(m, q, Et, world)
res = {"world": world, "split": split, "ranges": ranges, "ranks": []}
for r, (d0, d1) in enumerate(ranges):
    t = {"V": 0.0, "K": 0.0, "D": 0.0}
    for a in range(d0, d1, CH):
        b = min(d1, a + CH); n = b - a
        t["V"] += timed(lambda: _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(a, b), out=bufV[:n]))
        t["D"] += timed(lambda: (_assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(a, b), out=bufD[:n]),
                                 curl_combine_into(tabs, bufV[:n], bufD[:n], bufD[:n], p.alpha)))
        t["K"] += timed(lambda: _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(a, b), out=bufK[:n]))
    t["total"] = sum(t.values())
    res["ranks"].append({k: round(v, 1) for k, v in t.items()})
tot = [x["total"] for x in res["ranks"]]
res["max_ms"], res["sum_ms"], res["balance"] = max(tot), sum(tot), sum(tot) / (world * max(tot))
print(json.dumps(res))

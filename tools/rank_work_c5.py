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
CH = int(os.environ.get("CH", "48"))   # bench.py: 60 GB of V per chunk = 49 blocks
bufV = torch.empty((CH, E, E), dtype=torch.float64, device="cuda")
bufK = torch.empty((CH, E, N), dtype=torch.float64, device="cuda")
bufD = torch.empty((CH, N, N), dtype=torch.float64, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
def timed(fn):
    s, e = ev(), ev(); s.record(); fn(); e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)
def run(rvd, rk):
    """per rank: V + D on rvd[r], K on rk[r], in <= CH-block chunks; returns rank
    times and the (d0, d1, ms) chunk costs of V+D and of K"""
    ranks, cvd, ck = [], [], []
    for r in range(world):
        t = {"V": 0.0, "K": 0.0, "D": 0.0}
        d0, d1 = rvd[r]
        for a in range(d0, d1, CH):
            b = min(d1, a + CH); n = b - a
            tv = timed(lambda: _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(a, b), out=bufV[:n]))
            td = timed(lambda: (_assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(a, b), out=bufD[:n]),
                                curl_combine_into(tabs, bufV[:n], bufD[:n], bufD[:n], p.alpha)))
            t["V"] += tv; t["D"] += td; cvd.append((a, b, tv + td))
        d0, d1 = rk[r]
        for a in range(d0, d1, CH):
            b = min(d1, a + CH); n = b - a
            tk = timed(lambda: _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(a, b), out=bufK[:n]))
            t["K"] += tk; ck.append((a, b, tk))
        t["total"] = sum(t.values())
        ranks.append({k: round(v, 1) for k, v in t.items()})
    tot = [x["total"] for x in ranks]
    return {"ranks": ranks, "max_ms": max(tot), "sum_ms": sum(tot), "balance": sum(tot) / (world * max(tot))}, cvd, ck
uni = [D.block_range(r, world, Et) for r in range(world)]
res = {"world": world}
res["block_range"], cvd, ck = run(uni, uni)
if split != "block_range":
    rvd = D.cost_balanced_ranges(cvd, Et, world)
    rk = D.cost_balanced_ranges(ck, Et, world)
    res["cost_balanced"], cvd2, ck2 = run(rvd, rk)
    res["cost_balanced"]["ranges_vd"], res["cost_balanced"]["ranges_k"] = rvd, rk
    rvd2 = D.cost_balanced_ranges(cvd2, Et, world)
    rk2 = D.cost_balanced_ranges(ck2, Et, world)
    res["cost_balanced_2"], _, _ = run(rvd2, rk2)
    res["cost_balanced_2"]["ranges_vd"], res["cost_balanced_2"]["ranges_k"] = rvd2, rk2
print(json.dumps(res))

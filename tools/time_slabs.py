"""V (config 2) assembled in n row slabs: total device time, per-slab pair / finalize times (no copies)."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200.assembly import _assemble_operator, _row_slabs
from paper_2102_09811_b200._native import AssemblyStats
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig()
E = m.n_triangles
out = torch.empty((32, E, E), dtype=torch.float64, device="cuda")
res = {}
for n in (1, 2, 4, 8):
    slabs = _row_slabs(E, True, n)
    def run(stats=None):
        for i, (r0, r1) in enumerate(slabs):
            _assemble_operator(0, False, False, True, m, tg, p, q, None, row_range=(r0, r1), out=out,
                               stats=None if stats is None else stats[i])
    for _ in range(3): run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    st = [AssemblyStats() for _ in slabs]
    run(st)
    res[n] = {"total_ms": round(min(ts), 3), "rows": slabs, "pair_ms": [round(x.pair_ms, 3) for x in st],
              "fin_ms": [round(x.finalize_ms, 3) for x in st]}
print(json.dumps(res))

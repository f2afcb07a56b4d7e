"""Fused V + D (hb_assemble_vd) vs V, D2 and the curl combine as separate
calls: device time (CUDA events) at config 2 and on one config-5 block chunk."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200.assembly import _assemble_operator, _assemble_vd, curl_combine_into
q = hb.QuadratureConfig()
res = {}
for name, lvl, Et, dr in (("c2", 3, 32, None), ("c5_chunk", 5, 256, (64, 128))):
    if name != "c2" and os.environ.get("SKIP_C5"):
        continue
    m = hb.unit_cube_mesh(lvl); tg = hb.TimeGrid(1.0, Et); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
    tabs = hbdev.device_tables(m, q)
    d0, d1 = dr or (0, Et)
    V = torch.empty((d1 - d0, m.n_triangles, m.n_triangles), dtype=torch.float64, device="cuda")
    D = torch.empty((d1 - d0, m.n_vertices, m.n_vertices), dtype=torch.float64, device="cuda")
    def sep():
        _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(d0, d1), out=V)
        _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d1), out=D)
        curl_combine_into(tabs, V, D, D, p.alpha)
    from paper_2102_09811_b200._native import AssemblyStats
    def fused(st=None):
        _assemble_vd(m, tg, p, q, d_range=(d0, d1), out=D, out_v=V, stats=st)
    for nm, fn in (("separate", sep), ("fused", fused)):
        fn(); torch.cuda.synchronize()
        ts = []
        for _ in range(3 if name == "c2" else 1):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        res[f"{name}_{nm}_ms"] = min(ts)
    st = AssemblyStats(); fused(st)
    res[f"{name}_fused_pair_ms"], res[f"{name}_fused_fin_ms"] = st.pair_ms, st.finalize_ms
    sv, sd = AssemblyStats(), AssemblyStats()
    _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(d0, d1), out=V, stats=sv)
    _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d1), out=D, stats=sd)
    res[f"{name}_sep_pair_ms"] = sv.pair_ms + sd.pair_ms
    res[f"{name}_sep_fin_ms"] = (sv.finalize_ms, sd.finalize_ms)
    del V, D
    torch.cuda.empty_cache()
print(json.dumps(res))

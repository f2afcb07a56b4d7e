"""Config 2: sequential vs concurrent-stream assembly of V, K, D2 (+ curl after V and D2)."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E, N = m.n_triangles, m.n_vertices
tabs = hbdev.device_tables(m, q)
oV = torch.empty((32, E, E), dtype=torch.float64, device="cuda"); oK = torch.empty((32, E, N), dtype=torch.float64, device="cuda")
oD = torch.empty((32, N, N), dtype=torch.float64, device="cuda")
sV, sK, sD = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def seq():
    _assemble_operator(0, False, False, True, m, tg, p, q, None, out=oV)
    _assemble_operator(1, False, True, False, m, tg, p, q, None, out=oK)
    _assemble_operator(2, True, True, True, m, tg, p, q, None, out=oD)
    curl_combine_into(tabs, oV, oD, oD, p.alpha)
def conc(order):
    cur = torch.cuda.current_stream()
    st = {"V": sV, "K": sK, "D": sD}
    for s in st.values(): s.wait_stream(cur)
    ev = {}
    for name in order:
        with torch.cuda.stream(st[name]):
            if name == "V": _assemble_operator(0, False, False, True, m, tg, p, q, None, out=oV)
            if name == "K": _assemble_operator(1, False, True, False, m, tg, p, q, None, out=oK)
            if name == "D": _assemble_operator(2, True, True, True, m, tg, p, q, None, out=oD)
            ev[name] = torch.cuda.Event(); ev[name].record(st[name])
    sD.wait_event(ev["V"])
    with torch.cuda.stream(sD):
        curl_combine_into(tabs, oV, oD, oD, p.alpha)
    for s in st.values(): cur.wait_stream(s)
def t(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return sorted(ts)[len(ts)//2]
res = {"seq": t(seq)}
for order in ("VKD", "KVD", "DVK", "VDK"):
    res["conc_" + order] = t(lambda: conc(order))
ref = oV.clone(), oK.clone(), oD.clone(); seq(); torch.cuda.synchronize()
res["bitwise_same"] = bool(torch.equal(ref[0], oV) and torch.equal(ref[1], oK) and torch.equal(ref[2], oD))
print(json.dumps(res))

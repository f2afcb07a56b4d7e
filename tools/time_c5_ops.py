"""Config-5 V / K / D (D2 + curl) over all 256 blocks in the chunking of
tools/run_c5.py, device time per operator with stats (pair / finalize) and the
host-side wall time -- no parity checks (run_c5.py does those)."""
import json, os, sys, time, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
from paper_2102_09811_b200._native import AssemblyStats
from paper_2102_09811_b200.distributed import aligned_chunks
m = hb.unit_cube_mesh(5); tg = hb.TimeGrid(1.0, 256); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); tabs = hbdev.device_tables(m, q); E, N = m.n_triangles, m.n_vertices
CH = int(os.environ.get("CH", "64"))
ev = lambda: torch.cuda.Event(enable_timing=True)
res = {}
bufV = torch.empty((CH, E, E), dtype=torch.float64, device="cuda"); bufD = torch.empty((CH, N, N), dtype=torch.float64, device="cuda")
for name in ("V", "D"):
    st = AssemblyStats(); ms = 0.0; t0 = time.time()
    for d0, d1 in aligned_chunks(256, CH):
        n = d1 - d0
        s, e = ev(), ev(); s.record()
        if name == "V":
            _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(d0, d1), out=bufV[:n], stats=st)
        else:
            _assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d1), out=bufD[:n], stats=st)
        e.record(); torch.cuda.synchronize(); ms += s.elapsed_time(e)
    res[name] = {"ms": round(ms, 1), "pair_ms": round(st.pair_ms, 1), "fin_ms": round(st.finalize_ms, 1), "wall_s": round(time.time() - t0, 2)}
del bufV, bufD; torch.cuda.empty_cache()
bufK = torch.empty((30, E, N), dtype=torch.float64, device="cuda")
st = AssemblyStats(); ms = 0.0; t0 = time.time(); per = []
for d0, d1 in aligned_chunks(256, 30):
    n = d1 - d0
    s, e = ev(), ev(); s.record()
    _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(d0, d1), out=bufK[:n], stats=st)
    e.record(); torch.cuda.synchronize(); ms += s.elapsed_time(e); per.append((d0, d1, round(s.elapsed_time(e), 1)))
res["K_chunks"] = per
res["K"] = {"ms": round(ms, 1), "pair_ms": round(st.pair_ms, 1), "fin_ms": round(st.finalize_ms, 1), "wall_s": round(time.time() - t0, 2)}
print(json.dumps(res))

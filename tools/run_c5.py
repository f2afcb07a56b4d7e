"""BASELINE config 5 on one B200: unit cube L5 (12288 triangles, 6146 nodes),
alpha = 1, N = 256.  V (309 GB), K (155 GB) and D (77 GB) do not fit together,
so blocks are assembled in d-chunks into reused buffers -- the per-rank
layout of an 8-GPU d-sharded run -- and timed with CUDA events; D is formed
per chunk as D2 + curl(V) from the V chunk of the same blocks.  Sampled rows
of V and K are checked against tests/golden/c5_rows.npz when present."""
import json, os, sys, time
import numpy as np, torch
R = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, R)
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev, workload
from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
from paper_2102_09811_b200._native import AssemblyStats
from paper_2102_09811_b200.distributed import aligned_chunks
t0 = time.time()
m = hb.unit_cube_mesh(5)
tg = hb.TimeGrid(1.0, 256); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter); q = hb.QuadratureConfig()
tabs = hbdev.device_tables(m, q)
res = {"setup_s": time.time() - t0}
gp = os.path.join(R, "tests", "golden", "c5_rows.npz")
g = np.load(gp) if os.path.exists(gp) else None
rows = np.array([0, 6000, 12287])
E, N, Et = m.n_triangles, m.n_vertices, tg.n_steps
ev = lambda: torch.cuda.Event(enable_timing=True)
def timed(fn):
    s, e = ev(), ev(); s.record(); fn(); e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)
# ---- V and D, 64-block chunks -------------------------------------------------
CH = 64
bufV = torch.empty((CH, E, E), dtype=torch.float64, device="cuda")
bufD = torch.empty((CH, N, N), dtype=torch.float64, device="cuda")
gotV = np.empty((Et, len(rows), E))
msV = msD = 0.0
stV, stD2 = AssemblyStats(), AssemblyStats()
for d0, d1 in aligned_chunks(Et, CH):   # chunk edges on window edges: no extra gap slots
    n = d1 - d0
    msV += timed(lambda: _assemble_operator(0, False, False, True, m, tg, p, q, None, d_range=(d0, d1), out=bufV[:n], stats=stV))
    gotV[d0:d1] = bufV[:n, torch.as_tensor(rows, device="cuda"), :].cpu().numpy()
    msD += timed(lambda: (_assemble_operator(2, True, True, True, m, tg, p, q, None, d_range=(d0, d1), out=bufD[:n], stats=stD2),
                          curl_combine_into(tabs, bufV[:n], bufD[:n], bufD[:n], p.alpha)))
del bufV, bufD
torch.cuda.empty_cache()
# ---- K ----------------------------------------------------------------------
# default: window-aligned 30-block chunks (one 32-slot window each) whose
# staging for ALL test rows (109 GB) fits next to the 19 GB output, so one
# launch per chunk and the dual-orientation body evaluates each separated pair
# once: 2.8 s.  HB_C5_KCH=128 HB_C5_KWS=16e9: row-chunked 128-block chunks
# (pairs straddling two row chunks evaluated twice): 4.1 s; 14-block chunks
# with all rows (one 16-slot window each): 3.8 s (19 windows repeat the pair
# geometry, NJ = 1 halves the gaps per point load)
CHK = int(os.environ.get("HB_C5_KCH", "32"))
KWS = float(os.environ.get("HB_C5_KWS", "0"))   # 0: the library default (all rows when they fit)
bufK = torch.empty((CHK, E, N), dtype=torch.float64, device="cuda")
gotK = np.empty((Et, len(rows), N))
msK = 0.0
stK = AssemblyStats()
kchunks = aligned_chunks(Et, CHK) if CHK >= 32 else [(a, min(Et, a + CHK)) for a in range(0, Et, CHK)]
for d0, d1 in kchunks:
    n = d1 - d0
    msK += timed(lambda: _assemble_operator(1, False, True, False, m, tg, p, q, None, d_range=(d0, d1), out=bufK[:n],
                                            stats=stK, workspace_bytes=int(KWS) if KWS > 0 else None))
    gotK[d0:d1] = bufK[:n, torch.as_tensor(rows, device="cuda"), :].cpu().numpy()
del bufK
for op, ms, st, got in (("V", msV, stV, gotV), ("K", msK, stK, gotK), ("D", msD, stD2, None)):
    w = workload.operator_work(m, op if op != "D" else "D2", Et, q)
    r = {"ms": ms, "entries_per_s": workload.entries(m, op, Et) / (ms * 1e-3),
         "pair_ms": st.pair_ms, "finalize_ms": st.finalize_ms, "alg_tflops": w["flops"] / (st.pair_ms * 1e-3) / 1e12}
    if g is not None and got is not None:
        s = int(g["col_stride"])
        gs = got[:, :, ::s]
        mx, eps = g[f"{op}_maxabs"], g[f"{op}_eps_ref"]
        par = np.abs(gs - g[f"{op}_ref"]).max(axis=(1, 2)) / mx
        acc = np.abs(gs - g[f"{op}_exact"]).max(axis=(1, 2)) / mx
        r.update({"par_max": float(par.max()), "par_over_gate_max": float(np.max(par / np.maximum(1e-11, 3 * eps))),
                  "acc_over_epsref_max": float(np.max(acc / np.maximum(eps, 1e-300))), "eps_ref_max": float(eps.max())})
    res[op] = r
total_entries = sum(workload.entries(m, op, Et) for op in ("V", "K", "D"))
res["total_entries_per_s"] = total_entries / ((msV + msK + msD) * 1e-3)
res["k_chunks"] = {"blocks": CHK, "workspace_bytes": KWS}
print(json.dumps(res))

"""BASELINE config 3 on one B200: icosphere L5 (20480 triangles), alpha=0.5,
N=64.  V (107 GB per 32-block half) and K (14-block chunks) are assembled in
d-chunks into a reused device buffer (d-sharding on one GPU: the layout an 8-GPU run
uses per rank), timed with CUDA events, and the sampled rows are checked
against tests/golden/c3_rows.npz (reference rows + exact values)."""
import json, os, sys, time
import numpy as np, torch
R = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, R)
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev, workload
from paper_2102_09811_b200.assembly import _assemble_operator
from paper_2102_09811_b200._native import AssemblyStats
t0 = time.time()
m = hb.generate_icosphere(5)
tg = hb.TimeGrid(1.0, 64); p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter); q = hb.QuadratureConfig()
tabs = hbdev.device_tables(m, q)
t_setup = time.time() - t0
g = np.load(os.path.join(R, "tests", "golden", "c3_rows.npz")) if os.path.exists(os.path.join(R, "tests", "golden", "c3_rows.npz")) else None
rows = np.array([0, 7777, 20479]); stride = 41
res = {"setup_s": t_setup}
for op, code in (("V", (0, False, False, True)), ("K", (1, False, True, False))):
    E, N = m.n_triangles, m.n_vertices
    C = E if op == "V" else N
    # V: two 32-block halves; K: HB_C3_KCH-block chunks (default 14: one
    # 16-slot window whose all-rows staging, 141 GB, fits next to the output ->
    # one launch per chunk and the dual K body: 3.9 s; 32-block row-chunked
    # halves: 5.0 s; 10-block chunks: 5.2 s)
    ch = 32 if op == "V" else int(os.environ.get("HB_C3_KCH", "14"))
    buf = torch.empty((ch, E, C), dtype=torch.float64, device="cuda")
    got = np.empty((64, len(rows), C))
    ms, st = 0.0, AssemblyStats()
    for d0 in range(0, 64, ch):
        d1 = min(64, d0 + ch)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _assemble_operator(*code, m, tg, p, q, None, d_range=(d0, d1), out=buf[:d1 - d0], stats=st)
        e.record(); torch.cuda.synchronize()
        ms += s.elapsed_time(e)
        got[d0:d1] = buf[:d1 - d0, torch.as_tensor(rows, device="cuda"), :].cpu().numpy()
    del buf
    torch.cuda.empty_cache()
    w = workload.operator_work(m, op, 64, q)
    ent = workload.entries(m, op, 64)
    r = {"ms": ms, "pair_ms": st.pair_ms, "entries_per_s": ent / (ms * 1e-3), "n_eval": w["n_eval"],
         "alg_tflops": w["flops"] / (st.pair_ms * 1e-3) / 1e12, "pairs": w["pairs"]}
    if g is not None:
        gs = got[:, :, ::stride]
        mx, eps = g[f"{op}_maxabs"], g[f"{op}_eps_ref"]
        par = np.abs(gs - g[f"{op}_ref"]).max(axis=(1, 2)) / mx
        acc = np.abs(gs - g[f"{op}_exact"]).max(axis=(1, 2)) / mx
        r.update({"par_max": float(par.max()), "par_over_gate_max": float(np.max(par / np.maximum(1e-11, 3 * eps))),
                  "acc_over_epsref_max": float(np.max(acc / eps)), "eps_ref_max": float(eps.max()),
                  "gpu_exact_max": float(acc.max()), "zeros_gpu": int((got == 0).sum()), "zeros_ref": int(g[f"{op}_zeros"][0])})
    res[op] = r
print(json.dumps(res))

"""Block-Toeplitz product (hb_toeplitz_apply) on synthetic operators: the
study level-3 size (64 blocks of 12288^2, 77 GB) and a 6144^2 one; time,
effective HBM rate and DMMA rate (E_t^2/2 R C FMAs ~ sum_d (E_t - d) R C)."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
res = {}
sizes = [int(s) for s in os.environ.get("TOEP_N", "6144,12288").split(",")]
for n in sizes:
    nb = 64
    B = torch.empty((nb, n, n), dtype=torch.float64, device="cuda")
    for d in range(nb):
        B[d].normal_()
    M = hb.BlockToeplitzMatrix(B)
    x = torch.randn((nb, n), dtype=torch.float64, device="cuda")
    y = hb.apply_toeplitz(M, x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(int(os.environ.get("REPS", "3"))):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); y2 = hb.apply_toeplitz(M, x); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = min(ts)
    fma = sum(nb - d for d in range(nb)) * n * n
    # check a few rows against torch
    k = nb - 1
    ref = sum(B[d, :64] @ x[k - d] for d in range(nb))
    err = float((y2[k, :64] - ref).abs().max() / ref.abs().max())
    res[n] = {"ms": ms, "GBps": nb * n * n * 8 / ms / 1e6, "dmma_TFs": 2 * fma / ms / 1e9, "check": err,
              "bitwise_rerun": bool(torch.equal(y, y2))}
    del B, M
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))

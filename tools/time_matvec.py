import os, sys, torch, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
rng = np.random.default_rng(0)
B = torch.as_tensor(rng.standard_normal((32, 768, 768)), device="cuda")
M = hb.BlockToeplitzMatrix(B)
x = torch.as_tensor(rng.standard_normal((32, 768)), device="cuda")
for rep in range(5):
    for _ in range(3): hb.apply_toeplitz(M, x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): hb.apply_toeplitz(M, x)
    e.record(); torch.cuda.synchronize()
    print(os.environ.get("HB_TOEP_GROUPS"), rep, round(s.elapsed_time(e) / 20, 4), flush=True)

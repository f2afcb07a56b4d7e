"""One hb_toeplitz_apply on a synthetic 64-block operator (TOEP_N, default 6144) for ncu."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
n = int(os.environ.get("TOEP_N", "6144"))
B = torch.randn((64, n, n), dtype=torch.float64, device="cuda")
M = hb.BlockToeplitzMatrix(B)
x = torch.randn((64, n), dtype=torch.float64, device="cuda")
for _ in range(2):
    hb.apply_toeplitz(M, x)
torch.cuda.synchronize()
print("ok")

"""K assembly at config 2, twice (for ncu -k regex:k_pairs -c 1 after one warm-up)."""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
m = hb.unit_cube_mesh(int(os.environ.get("LVL", "3"))); tg = hb.TimeGrid(1.0, int(os.environ.get("ET", "32")))
p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
op = os.environ.get("OPK", "K")
fn = {"V": hb.assemble_single_layer, "K": hb.assemble_double_layer, "D2": hb.assemble_hypersingular_d2}[op]
for _ in range(2):
    fn(m, tg, p)
torch.cuda.synchronize()
print("done")

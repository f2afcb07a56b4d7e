"""Config 5 on one B200 with assemble_all per window-aligned 32-block chunk
(V, K, D on concurrent streams into reused buffers: 39 + 19 + 10 GB)."""
import json, os, sys
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import workload
from paper_2102_09811_b200.distributed import aligned_chunks
m = hb.unit_cube_mesh(5); tg = hb.TimeGrid(1.0, 256); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig(); E, N = m.n_triangles, m.n_vertices
CH = 32
bufs = {"V": torch.empty((CH, E, E), dtype=torch.float64, device="cuda"),
        "K": torch.empty((CH, E, N), dtype=torch.float64, device="cuda"),
        "D": torch.empty((CH, N, N), dtype=torch.float64, device="cuda")}
hb.assemble_all(m, tg, p, q, d_range=(0, 2), out={k: v[:2] for k, v in bufs.items()})   # warm-up
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for d0, d1 in aligned_chunks(256, CH):
    n = d1 - d0
    hb.assemble_all(m, tg, p, q, d_range=(d0, d1), out={k: v[:n] for k, v in bufs.items()})
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e)
ent = sum(workload.entries(m, op, 256) for op in ("V", "K", "D"))
print(json.dumps({"ms": ms, "entries_per_s": ent / (ms * 1e-3), "chunks": len(aligned_chunks(256, CH))}))

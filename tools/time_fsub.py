"""Forward substitution at config 2 (V: 32 blocks of 768 x 768) and on the
study's level-3 sizes: per-step form (hb_forward_solve) vs the blocked form
(hb_forward_solve_ws) -- time and max relative difference."""
import json, os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import _native
from paper_2102_09811_b200.solver import _inverse
L = _native.load()
res = {}


def case(name, V):
    B = V.device_blocks
    nb, n, _ = B.shape
    inv = _inverse(V, False)
    g = torch.Generator(device="cuda").manual_seed(1)
    rhs = torch.randn((nb, n), dtype=torch.float64, device="cuda", generator=g)
    x0 = torch.empty_like(rhs)
    x1 = torch.empty_like(rhs)
    h = torch.empty(n, dtype=torch.float64, device="cuda")
    need = L.hb_forward_solve_workspace(n)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    st = _native.stream_handle()
    old = lambda: _native.call("hb_forward_solve", nb, n, _native.ptr(B), 0, 0, nb, _native.ptr(inv),
                               _native.ptr(rhs), _native.ptr(x0), _native.ptr(h), st)
    new = lambda: _native.call("hb_forward_solve_ws", nb, n, _native.ptr(B), 0, 0, nb, _native.ptr(inv),
                               _native.ptr(rhs), _native.ptr(x1), _native.ptr(ws), need, st)
    out = {}
    for nm, f in (("per_step", old), ("blocked", new)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            f()
        e.record()
        torch.cuda.synchronize()
        out[nm + "_ms"] = s.elapsed_time(e) / 10
    out["max_rel_diff"] = float((x0 - x1).abs().max() / x0.abs().max())
    out["algorithmic_GB"] = (nb * (nb - 1) / 2 + nb) * n * n * 8 / 1e9
    res[name] = out


m = hb.unit_cube_mesh(3)
tg = hb.TimeGrid(1.0, 32)
p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
case("c2_V", hb.assemble_single_layer(m, tg, p))
tg = hb.TimeGrid(1.0, 64)
p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
case("L3_E64_V", hb.assemble_single_layer(m, tg, p))
print(json.dumps(res, indent=1))

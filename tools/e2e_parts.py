"""Where the e2e step's extra time goes (config 2): host issue time of each
public call (wall clock, no sync) vs the device time of the same calls, with
and without the mesh-table re-upload and the host copies."""
import json, os, sys, time, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb
from paper_2102_09811_b200 import device as hbdev
m = hb.unit_cube_mesh(3); tg = hb.TimeGrid(1.0, 32); p = hb.KernelParams(1.0, tg.step, length_scale=m.diameter)
q = hb.QuadratureConfig()
E, N = m.n_triangles, m.n_vertices
pinV = torch.empty((32, E, E), dtype=torch.float64).pin_memory()
pinK = torch.empty((32, E, N), dtype=torch.float64).pin_memory()
pinD = torch.empty((32, N, N), dtype=torch.float64).pin_memory()
res = {}


def run(name, drop, host, slabs=2, reps=5):
    host_ms, dev_ms = [], []
    for it in range(reps + 2):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = [time.perf_counter()]
        s.record()
        if drop:
            hbdev.drop_device_tables(m)
            hbdev.device_tables(m, q)
        t.append(time.perf_counter())
        V = hb.assemble_single_layer(m, tg, p, q, **({"host_out": pinV, "host_out_slabs": slabs} if host else {}))
        t.append(time.perf_counter())
        K = hb.assemble_double_layer(m, tg, p, q, **({"host_out": pinK} if host else {}))
        t.append(time.perf_counter())
        D = hb.assemble_hypersingular(m, tg, p, q, single_layer=V, **({"host_out": pinD} if host else {}))
        t.append(time.perf_counter())
        if host:
            for X in (V, K, D):
                torch.cuda.current_stream().wait_event(X.host_copy[1])
        e.record()
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        if it >= 2:
            host_ms.append([round((b - a) * 1e3, 3) for a, b in zip(t[:-1], t[1:])])
            dev_ms.append(round(s.elapsed_time(e), 3))
    res[name] = {"host_ms[tables,V,K,D,wait]": host_ms[-1], "device_ms": dev_ms}


run("plain", False, False)
run("drop", True, False)
run("host_out", False, True)
run("drop_host_out", True, True)
run("drop_host_out_slabs1", True, True, slabs=1)
print(json.dumps(res, indent=1))

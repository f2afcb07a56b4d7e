#!/usr/bin/env python
"""Benchmark: BEM matrix entries assembled per second (fp64 V / K / D).

Workload = BASELINE config 2 (the config the headline metric is quoted on
that fits one GPU): unit-cube surface refined 3x (768 triangles, 386 nodes),
N = 32 time steps, alpha = 1.  One step assembles V (p0 x p0), K (p0 x p1;
K' is the blockwise-transposed view, not re-counted) and D = D2 + curl(V)
(p1 x p1) -- E_t (E_x^2 + E_x N_x + N_x^2) = 33.1 M entries.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

N > 1 runs one process per GPU (torchrun); ranks own contiguous ranges of
time-difference blocks d.  With --parallel rows (default) the V and K pair
work is split by balanced test-row ranges over all blocks and the finalize
kernels store every block into its owner's shard through NVLink peer
pointers (CUDA IPC; no halo gaps, no data-path collective), D2's row partial
sums meet in one reduce-scatter (also the fence before the d-local curl
combine); --parallel d
splits everything by d (block d depends only on the kernel at gaps d-1, d,
d+1).  value = all ranks' entries / max-over-ranks device time.  ``--impl reference`` times the reference's CPU algorithm (the
oracle port, oracle/heatbem_oracle.c, all host threads) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BEM matrix entries assembled/sec (fp64 V/K/D) and % of FP64 roofline"
UNIT = "entries/s"
LEVEL, E_T, ALPHA = 3, 32, 1.0
WORKLOAD = ("BASELINE config 2: unit-cube [0,1]^3 surface refined 3x (768 triangles, 386 nodes), "
            "N=32 steps, T=1, alpha=1, quadrature (4,4): V p0p0 + K p0p1 (K' = transposed view) + "
            "D = D2 + alpha^2 curl(V) p1p1")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def setup():
    import paper_2102_09811_b200 as hb

    mesh = hb.unit_cube_mesh(LEVEL)
    tg = hb.TimeGrid(1.0, E_T)
    params = hb.KernelParams(ALPHA, tg.step, length_scale=mesh.diameter)
    return hb, mesh, tg, params


def entries_total(mesh, nb):
    E, N = mesh.n_triangles, mesh.n_vertices
    return nb * (E * E + E * N + N * N)


def d_range(rank, world, E_t):
    base, rem = divmod(E_t, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()            # the timed region starts once sampling runs
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port of the reference algorithm
# ---------------------------------------------------------------------------
def cpu_reference_step(mesh, tg, params, threads):
    """One bounded sample of the reference algorithm on the config-2 mesh:
    one full _toeplitz_pass (i_t = 1) of each of V, K, D2 plus the curl
    combine of one block, extrapolated to the E_t + 1 passes and E_t blocks
    of a full assembly (every i_t >= 1 pass does identical work)."""
    import paper_2102_09811_b200 as hb
    from oracle import oracle as O

    q = hb.QuadratureConfig()
    t_pass = {}
    for op in ("V", "K", "D2"):
        t0 = time.perf_counter()
        O.single_pass(mesh, params, q, op, tg.step, 1, n_threads=threads)
        t_pass[op] = time.perf_counter() - t0
    E, N = mesh.n_triangles, mesh.n_vertices
    rng = np.random.default_rng(0)
    V1, D21 = rng.standard_normal((1, E, E)), rng.standard_normal((1, N, N))
    t0 = time.perf_counter()
    O.curl_combine(V1, D21, mesh, params.alpha)
    t_curl = time.perf_counter() - t0
    t_full = (tg.n_steps + 1) * sum(t_pass.values()) + tg.n_steps * t_curl
    return t_full, t_pass, t_curl


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O

    O.build()
    hb, mesh, tg, params = setup()
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_step(mesh, tg, params, threads)
    ts = []
    for _ in range(args.steps):
        ts.append(cpu_reference_step(mesh, tg, params, threads)[0])
    t = statistics.median(ts)
    n_entries = entries_total(mesh, tg.n_steps)
    val = n_entries / t
    sample = (f"per step: one full i_t=1 pass each of V, K, D2 on the config-2 mesh + curl combine of one block "
              f"(oracle/heatbem_oracle.c, {threads} OpenMP threads), extrapolated to (E_t+1)=33 passes and "
              f"32 blocks = {n_entries} entries")
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (config-2 mesh generated in-run)",
           "config": {"workload": WORKLOAD, "E_x": mesh.n_triangles, "N_x": mesh.n_vertices, "E_t": tg.n_steps},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# native arm
# ---------------------------------------------------------------------------
def fp64_peak(torch, _native):
    """In-run DFMA probe (MEASURED_PEAKS.json carries no FP64 entry)."""
    sink = torch.zeros(148 * 8, dtype=torch.float64, device="cuda")
    grid, iters = 148 * 8, 40000
    for _ in range(2):
        _native.call("hb_fp64_probe", grid, 2000, _native.ptr(sink), _native.stream_handle())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    _native.call("hb_fp64_probe", grid, iters, _native.ptr(sink), _native.stream_handle())
    e.record()
    torch.cuda.synchronize()
    return grid * 256 * iters * 8 * 2 / (s.elapsed_time(e) * 1e-3) / 1e12


def load_traffic():
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def measure_paths(torch, hb, mesh, tg, params, q, Vd, Kd, cpu=True):
    """The other SURVEY 8 rows on this GPU (device time, CUDA events): the
    interior potentials of the whole config 4 (register-blocked kernel) and the config-2
    Dirichlet solve on the blocks just assembled.  Reference times are the
    SURVEY's measurements of the reference on this container (8 cores)."""
    import numpy as np

    def ev_ms(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    out = {}
    m4 = hb.unit_cube_mesh(4)
    tg4 = hb.TimeGrid(1.0, 64)
    p4 = hb.KernelParams(1.0, tg4.step, length_scale=m4.diameter)
    rng = np.random.default_rng(0)
    qd = rng.uniform(-1, 1, (64, m4.n_triangles))
    gd = rng.uniform(-1, 1, (64, m4.n_vertices))
    X = rng.uniform(0.05, 0.95, (100000, 3))
    # the whole of config 4 through the public call (1e5 points x 64 times,
    # single + double layer); warm-up on a 256-point slice
    hb.represent_grid(qd, gd, X[:256], m4, tg4, p4, return_device=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    hb.represent_grid(qd, gd, X, m4, tg4, p4, return_device=True)
    e.record()
    torch.cuda.synchronize()
    t_ms = s.elapsed_time(e)
    vals = X.shape[0] * 64
    out["potentials_c4"] = {"values_per_s": vals / (t_ms * 1e-3), "unit": "values/s (u = V~q - Wg)",
                            "full_config4_s": t_ms * 1e-3,
                            "sample": "all 1e5 config-4 points x 64 times (seeded as SURVEY 8(d)), represent_grid",
                            "cpu_baseline": cpu_potentials(m4, tg4, p4, qd, gd, X) if cpu else None}
    V = hb.BlockToeplitzMatrix(Vd)
    Kb = hb.BlockToeplitzMatrix(Kd)
    Mm = hb.assemble_mass(mesh, tg)
    y0 = np.array([1.5, 1.5, 1.5])
    data = hb.project_to_space(lambda x, t, n=None: hb.fundamental(np.asarray(x) - y0, t + 0.1, 1.0), mesh, tg, "X10")
    rhs = torch.as_tensor(0.5 * hb.apply_toeplitz(Mm, data) + hb.apply_toeplitz(Kb, data), device=Vd.device)
    info = {}

    def solve():
        x, rep = hb.fgmres(hb.toeplitz_operator(V), rhs, rel_tol=1e-10,
                           right_precond=lambda v: hb.forward_block_solve(V, v))
        info["it"], info["res"] = rep.iterations, rep.residual

    out["solve_c2"] = {"matvec_ms": ev_ms(lambda: hb.apply_toeplitz(V, rhs), reps=10),
                       "forward_subst_ms": ev_ms(lambda: hb.forward_block_solve(V, rhs), reps=10),
                       "fgmres_ms": ev_ms(solve), "iterations": info["it"], "residual": info["res"]}
    if cpu:
        out["solve_c2"]["cpu_baseline"] = cpu_solve(Vd.cpu().numpy(), rhs.cpu().numpy())
    return out


def cpu_potentials(m4, tg4, p4, qd, gd, X, n_points=4):
    """The reference algorithm (oracle port of _field_numba._eval_potential,
    all host threads) on a bounded sample: n_points config-4 points x 64 times,
    both potentials."""
    import numpy as np

    from oracle import oracle as O
    from paper_2102_09811_b200.field import _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    O.build()
    hats, qw, qpts = rule_tables(m4, 6)
    XX = np.repeat(X[:n_points], 64, axis=0)
    K = np.tile(np.arange(1, 65), n_points)
    z = np.zeros(len(K))
    t0 = time.perf_counter()
    for kind, c in ((0, qd), (1, gd)):
        O.potential(kind, XX, K, z, z > 0, _interp_density_np(c, m4, hats), qpts, qw, m4.areas, m4.normals,
                    tg4.step, p4.alpha, p4.delta_eps, p4.rho_eps)
    dt = time.perf_counter() - t0
    return {"values_per_s": len(K) / dt, "cores": os.cpu_count() or 1, "kind": "port",
            "sample": f"{n_points} config-4 points x 64 times, both potentials (oracle/heatbem_oracle.c)"}


def cpu_solve(Vh, rhs_h):
    """The reference's numpy solver loops (oracle.apply_toeplitz /
    forward_block_solve, restating solver.py:47-73 / 165-184) on the host."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    O.apply_toeplitz(Vh, rhs_h)
    t1 = time.perf_counter()
    O.forward_block_solve(Vh, rhs_h)
    t2 = time.perf_counter()
    return {"matvec_ms": (t1 - t0) * 1e3, "forward_subst_ms": (t2 - t1) * 1e3, "kind": "port",
            "cores": os.cpu_count() or 1, "sample": "config-2 V (32 x 768 x 768) and the solve's rhs, numpy"}


def run_native(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    hb, mesh, tg, params = setup()
    from paper_2102_09811_b200 import _native, device as hbdev, workload
    from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into

    _native.require_cuda()
    d0, d1 = d_range(rank, world, tg.n_steps)
    nb = d1 - d0
    q = hb.QuadratureConfig()
    E, N = mesh.n_triangles, mesh.n_vertices
    dev = torch.device("cuda", local_rank)
    outV = torch.empty((nb, E, E), dtype=torch.float64, device=dev)
    outK = torch.empty((nb, E, N), dtype=torch.float64, device=dev)
    outD = torch.empty((nb, N, N), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    tabs = hbdev.device_tables(mesh, q, dev)
    rows_mode = world > 1 and args.parallel == "rows"
    if rows_mode:
        # V and K: pair work split by balanced test-row ranges over ALL blocks,
        # stores into the d-owner's shard over NVLink (peer pointers); D2: row
        # partial sums + reduce-scatter; the curl combine is d-local
        from paper_2102_09811_b200 import distributed as Dm

        # peer mappings are set up collectively: if any rank cannot map its
        # peers (CUDA IPC / peer access), every rank falls back to d-sharding
        ok = 1
        try:
            peersV = Dm.PeerShardTable(outV, d0, d1, tg.n_steps)
            peersK = Dm.PeerShardTable(outK, d0, d1, tg.n_steps)
        except Exception as exc:   # noqa: BLE001 -- reported, then the d-sharded layout runs
            log(f"rank {rank}: peer shard mapping failed ({exc}); falling back to d-sharding")
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        rows_mode = bool(flag.item())
    if rows_mode:
        rowsV = Dm.row_partition(Dm.row_weights_mesh(mesh, q, True), world)[rank]
        rowsK = Dm.row_partition(Dm.row_weights_mesh(mesh, q, False), world)[rank]
        rowsD = Dm.row_partition(Dm.row_weights_mesh(mesh, q, True, skip_perpendicular=True), world)[rank]
        partD = torch.empty((tg.n_steps, N, N), dtype=torch.float64, device=dev)   # this rank's D2 rows
        dist.barrier()

    def step(stats=None):
        st = stats if stats is not None else [None, None, None]
        if rows_mode:
            _assemble_operator(0, False, False, True, mesh, tg, params, q, None, d_range=(0, tg.n_steps),
                               row_range=rowsV, block_ptrs=peersV.table, stats=st[0])
            _assemble_operator(1, False, True, False, mesh, tg, params, q, None, d_range=(0, tg.n_steps),
                               row_range=rowsK, block_ptrs=peersK.table, stats=st[1])
        elif stats is None:
            # the three operators on concurrent streams (public API assemble_all)
            hb.assemble_all(mesh, tg, params, q, d_range=(d0, d1), out={"V": outV, "K": outK, "D": outD})
            return
        else:
            _assemble_operator(0, False, False, True, mesh, tg, params, q, None, d_range=(d0, d1), out=outV,
                               stats=st[0])
            _assemble_operator(1, False, True, False, mesh, tg, params, q, None, d_range=(d0, d1), out=outK,
                               stats=st[1])
        if rows_mode:
            # D2: this rank's element rows for all blocks, summed into the d-owners'
            # shards by one reduce-scatter -- which is also the fence after which
            # every rank's V stores into this shard are complete
            _assemble_operator(2, True, True, True, mesh, tg, params, q, None, d_range=(0, tg.n_steps),
                               row_range=rowsD, out=partD, stats=st[2])
            Dm.reduce_scatter_blocks(partD, outD, d0, d1)
        else:
            _assemble_operator(2, True, True, True, mesh, tg, params, q, None, d_range=(d0, d1), out=outD,
                               stats=st[2])
        curl_combine_into(tabs, outV, outD, outD, params.alpha)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    peak = fp64_peak(torch, _native) if rank == 0 else None

    # ---- timed region: K steps, events per step, L2 flushed between steps ----
    stats = [_native.AssemblyStats() for _ in range(3)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = []
    gpu = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[0]) if world == 1 else local_rank
    with ClockSampler(gpu) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step()
            e.record()
            e.synchronize()
            step_ms.append(s.elapsed_time(e))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # kernel timing pass (stats sync inside each call; kept out of the headline)
    for _ in range(max(1, args.steps // 2)):
        step(stats)
    torch.cuda.synchronize()

    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    n_entries = entries_total(mesh, tg.n_steps)   # all ranks together
    value = n_entries / (ms_per_step * 1e-3)

    if rows_mode:
        dist.barrier()
        peersV.close()
        peersK.close()

    # ---- e2e: public API, host buffers, copies inside the timed region ----
    Hpin = hbdev.pin_host_tables(hbdev.host_tables(mesh, q))
    pinV = torch.empty(outV.shape, dtype=torch.float64).pin_memory()
    pinK = torch.empty(outK.shape, dtype=torch.float64).pin_memory()
    pinD = torch.empty(outD.shape, dtype=torch.float64).pin_memory()

    def e2e_step():
        # sequential public calls: V finishes first and its copy-back overlaps K,
        # K's overlaps D (assemble_all's concurrent streams finish all three
        # together and leave the 265 MB of copies exposed: slower end to end)
        hbdev.drop_device_tables(mesh)              # re-upload inputs from pinned host memory
        # V streams back in work-balanced row slabs as they are assembled
        # (host_out), K as soon as it is done, D in block chunks as the curl
        # combine forms them
        V = hb.assemble_single_layer(mesh, tg, params, q, d_range=(d0, d1), host_out=pinV,
                                     host_out_slabs=int(os.environ.get("HB_E2E_SLABS", "3")))
        _, ev_v = V.host_copy
        K = hb.assemble_double_layer(mesh, tg, params, q, d_range=(d0, d1), host_out=pinK)
        _, ev_k = K.host_copy
        D = hb.assemble_hypersingular(mesh, tg, params, q, single_layer=V, d_range=(d0, d1), host_out=pinD)
        _, ev_d = D.host_copy                      # D streamed back in block chunks as the curl forms them
        for ev in (ev_v, ev_k, ev_d):
            torch.cuda.current_stream().wait_event(ev)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(args.steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        e2e_step()
        e.record()
        e.synchronize()
        e2e_ms.append(s.elapsed_time(e))
    te = torch.tensor([sum(e2e_ms) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = n_entries / (float(te.item()) * 1e-3)
    h2d = Hpin.pinned_bytes
    d2h = (pinV.numel() + pinK.numel() + pinD.numel()) * 8

    # ---- roofline of the dominant kernel: the K pair kernel (k_pairs<1,...>) ----
    kd0, kd1 = (0, tg.n_steps) if rows_mode else (d0, d1)
    it_lo, it_hi = max(1, kd0 - 1), kd1
    n_windows = 0
    dd = kd0
    while dd < kd1:   # windows of <= 32 gap slots (csrc/hb_assembly.cu)
        nd1 = min(kd1, 32 if dd <= 1 else dd + 30)
        n_windows += 1
        dd = nd1
    wK = workload.operator_work(mesh, "K", 1, q)
    gapsK = (it_hi - it_lo + 1) + 2 * (n_windows - 1)
    row_frac = (rowsK[1] - rowsK[0]) / E if rows_mode else 1.0
    flops_per_call = wK["flops"] * gapsK * row_frac   # one call = n_windows launches
    sK = stats[1]
    pair_ms_per_call = sK.pair_ms / max(1, args.steps // 2)
    launches_per_call = sK.pair_launches / max(1, args.steps // 2)
    achieved = flops_per_call / (pair_ms_per_call * 1e-3) / 1e12
    shares = {nm: st.pair_ms / max(1e-9, st.pair_ms + st.finalize_ms) for nm, st in zip(("V", "K", "D2"), stats)}
    launches_step = sum(st.launches for st in stats) / max(1, args.steps // 2) + 1   # + curl (k_curl_tile)
    traffic = load_traffic().get("k_pairs_K_dram_bytes_per_launch")

    paths = (measure_paths(torch, hb, mesh, tg, params, q, outV, outK, cpu=not args.no_cpu_baseline)
             if (world == 1 and not args.no_paths) else None)
    if rank != 0:
        return
    clocks = clk.summary()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O

        O.build()
        threads = os.cpu_count() or 1
        cpu_reference_step(mesh, tg, params, threads)         # page-in / thread start
        ts = [cpu_reference_step(mesh, tg, params, threads)[0] for _ in range(3)]
        cpu = {"value": n_entries / statistics.median(ts), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": "3 x (one full i_t=1 pass each of V, K, D2 on the config-2 mesh + curl combine of one "
                         "block), oracle/heatbem_oracle.c with all host threads, extrapolated to the 33 passes / "
                         "32 blocks of a full assembly"}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: BASELINE config-2 mesh and time grid generated in-run (no dataset)",
        "config": {"workload": WORKLOAD, "E_x": E, "N_x": N, "E_t": tg.n_steps, "entries_per_step": n_entries,
                   "parallelism": (f"x{world}: V/K/D2 pair work split by balanced test-row ranges over all "
                                   "blocks; V/K blocks stored into the d-owner's shard over NVLink peer memory, "
                                   "D2 row partials summed by one NCCL reduce-scatter; curl d-local")
                   if rows_mode else f"d-sharded x{world} (contiguous time-difference blocks per rank)",
                   "l2": "flushed between timed steps (256 MiB device write, outside the events)",
                   "fp64_peak_tflops": peak, "pair_kernel_share": shares},
        "roofline": {"bound": "fp64", "kernel": "k_pairs<op=K> (double-layer pair kernel)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                     "peak_source": "measured in-run (hb_fp64_probe DFMA loop; MEASURED_PEAKS.json has no FP64 entry)",
                     "flops_per_launch": flops_per_call / max(1.0, launches_per_call),
                     "flops_definition": "SURVEY 8(d): N_eval (pairs x points x gaps) x 124 flop",
                     "note": ("achieved counts the reference formulation's 124 flop per evaluation (erf + exp) "
                              "over every (pair, point, gap); the fused evaluator executes far fewer FP64 ops per "
                              "evaluation and skips point chunks whose K weights are exactly zero (coplanar "
                              "triangles), so frac exceeds 1: it is the work rate against the reference's "
                              "algorithm. The hardware view of the same kernel (ncu, 'hw') is the FP64 pipe "
                              "activity and the issued FP64 flop rate"),
                     "hw": load_traffic().get("k_pairs_K"),
                     "avg_launch_ms": pair_ms_per_call / max(1.0, launches_per_call),
                     "traffic": traffic},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": "public API assemble_single_layer / assemble_double_layer / assemble_hypersingular with "
                        "host_out: mesh tables re-uploaded from pinned host memory and all blocks copied to pinned "
                        "host memory every step -- V in 3 work-balanced test-row slabs, each slab's copy started "
                        "on a side stream as soon as its rows are complete, K as soon as it is done, D in 4 block "
                        "chunks as the "
                        "curl combine forms them; the step ends when the last copy is done"},
        "clocks": clocks,
        "paths": paths,
        "gpu_launches": int(round(launches_step * args.steps * world)),
        "impl": "native",
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("native", "reference"), default="native")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-paths", action="store_true", help="skip the potentials / solve measurements")
    ap.add_argument("--parallel", choices=("rows", "d"), default="rows",
                    help="N > 1: split V/K pair work by test rows (peer stores) or everything by d")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # HB_BENCH_EMULATE=1: every rank on cuda:0 over gloo -- a control-flow
        # check of the N > 1 path on a one-GPU box, never a measurement
        dist.init_process_group("gloo" if os.environ.get("HB_BENCH_EMULATE") else "nccl")
        if os.environ.get("HB_BENCH_EMULATE"):
            local_rank = 0
    try:
        run_native(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

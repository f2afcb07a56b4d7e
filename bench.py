#!/usr/bin/env python
"""Benchmark: BEM matrix entries assembled per second (fp64 V / K / D).

Default workload = BASELINE config 2 (the config the headline metric is
quoted on that fits one GPU): unit-cube surface refined 3x (768 triangles,
386 nodes), N = 32 time steps, alpha = 1.  One step assembles V (p0 x p0),
K (p0 x p1; K' is the blockwise-transposed view, not re-counted) and
D = D2 + curl(V) (p1 x p1) -- E_t (E_x^2 + E_x N_x + N_x^2) = 33.1 M entries.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                  [--config 2|3|5]

--config 3 (icosphere L5, N = 64: V + K, 322 GB) and 5 (unit cube L5,
N = 256: V + K + D, 541 GB) are the scaling configurations: every rank
assembles its contiguous range of blocks d (window-aligned d-chunks into a
reused buffer where its range does not fit one GPU).

N > 1 runs one process per GPU (torchrun).  Config 2: the V and K pair work
is split by balanced test-row ranges over all blocks and the finalize kernels
store every block into its owner's d-shard through NVLink peer pointers (CUDA
IPC); D2 is d-sharded (block d needs the kernel at gaps d-1, d, d+1 only) and
the curl combine is d-local -- no data-path collective.  value = all ranks'
entries / max-over-ranks device time.

Measurement:
* roofline: the dominant pair kernel's ISSUED FP64 arithmetic (2 DFMA + DMUL
  + DADD thread instructions + 512 flop per DMMA warp instruction), counted by
  an ncu counter pass on the same workload inside this run, divided by the
  kernel's average launch time measured live with CUDA events, against the
  FP64 peak measured in-run (DFMA probe); traffic = DRAM bytes per launch
  from the same ncu pass.  The SURVEY 8(d) work rate (kernel evaluations of
  the reference formulation per second) is reported beside it, not as a
  fraction.
* cpu_baseline: one full config-2 assembly by the oracle port of the
  reference's algorithm (oracle/heatbem_oracle.c) on all host cores,
  measured, plus the per-pass sample rate (validates extrapolations).
* --impl reference: per step one full config-2 assembly (V, K, D2 over all
  E_t + 1 delta-passes, then D = D2 + curl V) by the oracle port on all host
  cores, tables built outside the timed region; value = entries / median step.
"""
from __future__ import annotations

import argparse
import csv
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
CONFIGS = {
    2: dict(mesh="cube", level=3, E_t=32, alpha=1.0, ops=("V", "K", "D"),
            text="BASELINE config 2: unit-cube [0,1]^3 surface refined 3x (768 triangles, 386 nodes), N=32 steps, "
                 "T=1, alpha=1, quadrature (4,4): V p0p0 + K p0p1 (K' = transposed view) + D = D2 + alpha^2 curl(V) "
                 "p1p1"),
    3: dict(mesh="sphere", level=5, E_t=64, alpha=0.5, ops=("V", "K"),
            text="BASELINE config 3: icosphere L5 (20480 triangles, 10242 nodes), N=64 steps, T=1, alpha=0.5, "
                 "quadrature (4,4): V p0p0 + K p0p1"),
    5: dict(mesh="cube", level=5, E_t=256, alpha=1.0, ops=("V", "K", "D"),
            text="BASELINE config 5: unit-cube surface refined 5x (12288 triangles, 6146 nodes), N=256 steps, T=1, "
                 "alpha=1, quadrature (4,4): V p0p0 + K p0p1 + D = D2 + alpha^2 curl(V) p1p1"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def setup(cfg):
    import paper_2102_09811_b200 as hb

    c = CONFIGS[cfg["config"]]
    level = cfg.get("level") or c["level"]
    E_t = cfg.get("E_t") or c["E_t"]
    mesh = hb.unit_cube_mesh(level) if c["mesh"] == "cube" else hb.generate_icosphere(level)
    tg = hb.TimeGrid(1.0, E_t)
    params = hb.KernelParams(c["alpha"], tg.step, length_scale=mesh.diameter)
    return hb, mesh, tg, params


def entries_total(mesh, nb, ops):
    E, N = mesh.n_triangles, mesh.n_vertices
    per = {"V": E * E, "K": E * N, "D": N * N}
    return nb * sum(per[o] for o in ops)


def config_dict(cfg, mesh, tg):
    """The workload description -- identical in both arms."""
    c = CONFIGS[cfg["config"]]
    return {"workload": c["text"], "E_x": mesh.n_triangles, "N_x": mesh.n_vertices, "E_t": tg.n_steps,
            "entries_per_step": entries_total(mesh, tg.n_steps, c["ops"])}


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
# CPU side: the oracle port of the reference's algorithm (checker only)
# ---------------------------------------------------------------------------
class CpuReference:
    """The reference's assembly on the host (oracle/heatbem_oracle.c, the
    port of _toeplitz_pass / _scatter_add / _assemble_operator): problem
    tables built once, outside every timed region."""

    def __init__(self, mesh, tg, params, threads):
        import paper_2102_09811_b200 as hb
        from oracle import oracle as O

        O.build()
        self.O, self.mesh, self.tg, self.params, self.threads = O, mesh, tg, params, threads
        q = hb.QuadratureConfig()
        self.P = {op: O.OracleProblem(mesh, params, q, op, tg.step) for op in ("V", "K", "D2")}
        E, N = mesh.n_triangles, mesh.n_vertices
        self.loc = {op: (np.zeros((E, 3 if P.test_p1 else 1, P.shape_rc[1])),
                         np.zeros((E, 3 if P.test_p1 else 1, P.shape_rc[1]))) for op, P in self.P.items()}
        rng = np.random.default_rng(0)
        self.V1, self.D21 = rng.standard_normal((1, E, E)), rng.standard_normal((1, N, N))

    def pass_sample(self):
        """One full delta-pass (i_t = 1, all rows) of V, K, D2 and the curl
        combine of one block: 1/(E_t + 1) of the passes and 1/E_t of the
        curl work of a full assembly.  Returns seconds."""
        O = self.O
        t0 = time.perf_counter()
        for op, P in self.P.items():
            loc, locc = self.loc[op]
            O.lib().hb_oracle_pass(*P.args(), float(self.tg.step), 0, None, 0, O._ptr(loc), O._ptr(locc),
                                   self.threads)
        O.curl_combine(self.V1, self.D21, self.mesh, self.params.alpha)
        return time.perf_counter() - t0

    def pass_sample_entries(self, entries):
        """Work-equivalent entries of one pass sample (passes and curl blocks
        of a full assembly weighted by their measured share)."""
        return entries / (self.tg.n_steps + 1)

    def full_assembly(self):
        """The whole assembly of V, K, D2 (E_t + 1 passes each) and D =
        D2 + curl(V): measured seconds (tables prebuilt)."""
        O = self.O
        out = {}
        t0 = time.perf_counter()
        for op, P in self.P.items():
            R, C = P.shape_rc
            out[op] = np.empty((self.tg.n_steps, R, C))
            rc = O.lib().hb_oracle_assemble(*P.args(), self.tg.n_steps, self.tg.step, O._ptr(out[op]),
                                            self.threads)
            if rc != 0:
                raise MemoryError("oracle assemble failed")
        O.curl_combine(out["V"], out["D2"], self.mesh, self.params.alpha)
        return time.perf_counter() - t0


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = {"config": args.config, "level": args.level, "E_t": args.et}
    hb, mesh, tg, params = setup(cfg)
    conf = config_dict(cfg, mesh, tg)
    threads = os.cpu_count() or 1
    if args.config != 2:
        print(json.dumps({"impl": "reference", "metric": METRIC, "unavailable":
                          f"config {args.config}: hours of CPU work per step (the CPU baseline is timed on config 2)",
                          "config": conf}), flush=True)
        return
    ref = CpuReference(mesh, tg, params, threads)
    n_entries = conf["entries_per_step"]
    # one step = the whole config-2 workload (V, K, D2 over all E_t + 1 passes, then D = D2 + curl V),
    # the same work as one step of the native arm; the warm-up is bounded (a CPU has nothing to warm
    # beyond the first pass), so the run stays within a few minutes at the driver's step counts
    ref.pass_sample()
    ts = [ref.full_assembly() for _ in range(args.steps)]
    t = statistics.median(ts)
    val = n_entries / t
    sample = (f"per step: one full config-2 assembly -- V, K, D2 (E_t + 1 = {tg.n_steps + 1} delta-passes each, "
              f"all rows) and D = D2 + curl V -- by oracle/heatbem_oracle.c (the port of the reference's "
              f"_toeplitz_pass / _scatter_add / _assemble_operator), {threads} OpenMP threads, tables built "
              f"outside the timed region; value = {n_entries} entries / median step time "
              f"(warm-up: one delta-pass of each operator)")
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (config-2 mesh generated in-run)",
           "config": conf,
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                            "step_s": ts},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# ncu counter pass (hardware view of the kernels, inside this run)
# ---------------------------------------------------------------------------
NCU_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
               "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
               "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
               "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def ncu_pass(child_mode, kernel_regex, timeout=600):
    """Run this script's ``--ncu-child MODE`` under ncu (counters only) and
    return per-launch rows {kernel, metric: value}.  None when ncu is not
    usable here."""
    ncu = "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    cmd = [ncu, "--metrics", ",".join(NCU_METRICS), "--clock-control", "none", "--csv", "--print-units", "base",
           "-k", f"regex:{kernel_regex}", sys.executable, os.path.abspath(__file__), "--ncu-child", child_mode]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except (subprocess.TimeoutExpired, OSError) as exc:
        log(f"ncu pass failed: {exc}")
        return None
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith('"')]
    if not lines:
        log("ncu pass produced no rows:", out.stderr[-500:])
        return None
    rows = list(csv.reader(lines))
    h = rows[0]
    iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = {}
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        d = launches.setdefault(int(r[iid]), {"kernel": r[ik]})
        try:
            d[r[im]] = float(r[iv].replace(",", ""))
        except ValueError:
            pass
    return [launches[k] for k in sorted(launches)]


def issued_fp64(row):
    """Issued FP64 flops of one launch: 2 DFMA + DMUL + DADD thread
    instructions + 512 per DMMA (m8n8k4) warp instruction."""
    return (2 * row.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
            + row.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
            + row.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
            + 512 * row.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0))


def ncu_child(mode):
    """Workload of the ncu pass: one warm-up and one measured call (the
    parent keeps the second half of the launches)."""
    import torch

    if mode == "c2":
        cfg = {"config": 2}
        hb, mesh, tg, params = setup(cfg)
        from paper_2102_09811_b200.assembly import _assemble_operator

        q = hb.QuadratureConfig()
        for _ in range(2):
            for code in ((0, False, False, True), (1, False, True, False), (2, True, True, True)):
                _assemble_operator(*code, mesh, tg, params, q, None)
            torch.cuda.synchronize()
    elif mode == "c4":
        import paper_2102_09811_b200 as hb

        m4 = hb.unit_cube_mesh(4)
        tg4 = hb.TimeGrid(1.0, 64)
        p4 = hb.KernelParams(1.0, tg4.step, length_scale=m4.diameter)
        rng = np.random.default_rng(0)
        qd = rng.uniform(-1, 1, (64, m4.n_triangles))
        gd = rng.uniform(-1, 1, (64, m4.n_vertices))
        X = rng.uniform(0.05, 0.95, (100000, 3))
        for _ in range(2):
            hb.represent_grid(qd, gd, X[:8192], m4, tg4, p4, return_device=True)
            torch.cuda.synchronize()


def pair_kernel_hw(rows):
    """Group the c2 pair launches of the measured (second) call by operator:
    the V kernels (moment form: touching, near and far launches), then K and
    D2 (direct kernels, one launch each)."""
    if not rows:
        return None
    half = rows[len(rows) // 2:]
    groups = {"V": [], "K": [], "D2": []}
    for r in half:
        k = r["kernel"]
        op = "V" if "k_pairs<0" in k else "K" if "k_pairs<1" in k else "D2" if "k_pairs<2" in k else None
        if op:
            groups[op].append(r)
    out = {}
    for op, rs in groups.items():
        if not rs:
            continue
        t = sum(r.get("gpu__time_duration.sum", 0.0) for r in rs) * 1e-9
        fl = sum(issued_fp64(r) for r in rs)
        dram = sum(r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0) for r in rs)
        w = [r.get("gpu__time_duration.sum", 0.0) for r in rs]
        pipe = sum(r.get("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * x
                   for r, x in zip(rs, w)) / max(1e-30, sum(w))
        out[op] = {"launches": len(rs), "ncu_ms": t * 1e3, "issued_fp64_flop": fl, "dram_bytes": dram,
                   "ncu_issued_tflops": fl / t / 1e12 if t > 0 else None, "fp64_shared_pipe_pct": pipe,
                   "kernels": sorted({r["kernel"].split("(")[0] for r in rs})}
    return out


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


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6459.6, "B200_PROFILING.md fallback"


def measure_paths(torch, hb, mesh, tg, params, q, Vd, Kd, cpu=True, hw=None, peak=None):
    """The other SURVEY 8 rows on this GPU (device time, CUDA events): the
    whole config-4 representation formula and the config-2 Dirichlet solve
    on the blocks just assembled, each with its roofline fraction."""

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
    hb.represent_grid(qd, gd, X[:256], m4, tg4, p4, return_device=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    hb.represent_grid(qd, gd, X, m4, tg4, p4, return_device=True)
    e.record()
    torch.cuda.synchronize()
    t_ms = s.elapsed_time(e)
    vals = X.shape[0] * 64
    pot = {"values_per_s": vals / (t_ms * 1e-3), "unit": "values/s (u = V~q - Wg)", "full_config4_s": t_ms * 1e-3,
           "sample": "all 1e5 config-4 points x 64 times (seeded as SURVEY 8(d)), represent_grid",
           "cpu_baseline": cpu_potentials(m4, tg4, p4, qd, gd, X) if cpu else None}
    if hw:   # issued FP64 per point from the ncu pass (8192 points), scaled to 1e5 points
        fl = sum(issued_fp64(r) for r in hw[len(hw) // 2:])
        achieved = fl * (X.shape[0] / 8192) / (t_ms * 1e-3) / 1e12
        pot["roofline"] = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                           "frac": achieved / peak if peak else None,
                           "definition": "issued FP64 (2 DFMA + DMUL + DADD + 512 per DMMA) counted by ncu on 8192 "
                                         "points, scaled to 1e5, / the live time of the whole config 4"}
    out["potentials_c4"] = pot
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

    mv = ev_ms(lambda: hb.apply_toeplitz(V, rhs), reps=10)
    fs = ev_ms(lambda: hb.forward_block_solve(V, rhs), reps=10)
    hbm, hbm_src = hbm_peak()
    nb, R, C = Vd.shape
    mv_bytes = nb * R * C * 8 + 2 * rhs.numel() * 8                       # A read once + x, y
    # the blocked substitution (hb_forward_solve_ws, 8-step tiles): per tile one pass over blocks
    # 1..k0+7 (far terms), per step the near blocks 1..k-k0 and the inverse
    blk = R * C * 8
    fs_bytes = 0
    for k0 in range(0, nb, 8):
        nk = min(8, nb - k0)
        fs_bytes += (min(k0 + nk - 1, nb - 1) * blk if k0 else 0)
        fs_bytes += sum(min(k - k0, nb - 1) * blk + R * R * 8 for k in range(k0, k0 + nk))
    out["solve_c2"] = {"matvec_ms": mv, "forward_subst_ms": fs, "fgmres_ms": ev_ms(solve),
                       "iterations": info["it"], "residual": info["res"],
                       "roofline": {"bound": "hbm", "peak": hbm, "unit": "GB/s", "peak_source": hbm_src,
                                    "matvec_achieved": mv_bytes / (mv * 1e-3) / 1e9,
                                    "matvec_frac": mv_bytes / (mv * 1e-3) / 1e9 / hbm,
                                    "forward_subst_achieved": fs_bytes / (fs * 1e-3) / 1e9,
                                    "forward_subst_frac": fs_bytes / (fs * 1e-3) / 1e9 / hbm,
                                    "definition": "algorithmic bytes: matvec reads every block once; the blocked "
                                                  "forward substitution reads blocks 1..k0+7 once per 8-step tile "
                                                  "and per step the near blocks 1..k-k0 and (A^0)^-1 (the latter "
                                                  "L2-resident at config 2)"}}
    if cpu:
        out["solve_c2"]["cpu_baseline"] = cpu_solve(Vd.cpu().numpy(), rhs.cpu().numpy())
    return out


def cpu_potentials(m4, tg4, p4, qd, gd, X, n_points=4):
    """The reference algorithm (oracle port of _field_numba._eval_potential,
    all host threads) on a bounded sample: n_points config-4 points x 64 times,
    both potentials."""
    from oracle import oracle as O
    from paper_2102_09811_b200.field import _interp_density_np
    from paper_2102_09811_b200.quadrature import rule_tables

    O.build()
    hats, qw, qpts = rule_tables(m4, 6)
    XX = np.repeat(X[:n_points], 64, axis=0)
    K = np.tile(np.arange(1, 65), n_points)
    z = np.zeros(len(K))
    dens = [_interp_density_np(c, m4, hats) for c in (qd, gd)]
    t0 = time.perf_counter()
    for kind in (0, 1):
        O.potential(kind, XX, K, z, z > 0, dens[kind], qpts, qw, m4.areas, m4.normals,
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


def algorithmic_rate(hb, mesh, op, n_gaps, ms):
    """SURVEY 8(d) work rate: kernel evaluations of the reference formulation per second."""
    from paper_2102_09811_b200 import workload

    if not ms > 0:
        return None
    w = workload.operator_work(mesh, op, n_gaps, hb.QuadratureConfig())
    return {"evaluations": w["n_eval"], "evaluations_per_s": w["n_eval"] / (ms * 1e-3),
            "reference_flops_per_s": w["flops"] / (ms * 1e-3),
            "definition": "N_eval = E_t sum_class n_pairs q_class (SURVEY 8(d)); reference formulation "
                          f"{workload.FLOPS_PER_EVAL[op]} flop per evaluation (erf + exp)"}


def run_native_c2(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    cfg = {"config": 2, "level": args.level, "E_t": args.et}
    torch.cuda.set_device(local_rank)
    hb, mesh, tg, params = setup(cfg)
    conf = config_dict(cfg, mesh, tg)
    from paper_2102_09811_b200 import _native, device as hbdev
    from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into
    from paper_2102_09811_b200 import distributed as Dm

    _native.require_cuda()
    d0, d1 = Dm.block_range(rank, world, tg.n_steps)
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
        # stores into the d-owner's shard over NVLink (peer pointers).  Peer
        # mappings are set up collectively: if any rank cannot map its peers
        # (CUDA IPC / peer access), every rank falls back to d-sharding.
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
        # D2 split by element rows, partials read over peer memory by each rank's curl kernel
        rpd = Dm.RowPartialD(mesh, tg, params, q, d0, d1, device=dev)
        from paper_2102_09811_b200.assembly import _op_streams
        sD, sV, sK = _op_streams(dev)
        dist.barrier()

    def step(stats=None):
        st = stats if stats is not None else [None, None, None]
        if rows_mode:
            # the rank's V and K rows (stores into the d-owners' shards over NVLink) and
            # its element rows' D2 partial, on three streams
            cur = torch.cuda.current_stream()
            for s_ in (sD, sV, sK):
                s_.wait_stream(cur)
            with torch.cuda.stream(sV):
                _assemble_operator(0, False, False, True, mesh, tg, params, q, None, d_range=(0, tg.n_steps),
                                   row_range=rowsV, block_ptrs=peersV.table, stats=st[0], stream=sV)
            with torch.cuda.stream(sK):
                _assemble_operator(1, False, True, False, mesh, tg, params, q, None, d_range=(0, tg.n_steps),
                                   row_range=rowsK, block_ptrs=peersK.table, stats=st[1], stream=sK)
            with torch.cuda.stream(sD):
                rpd.assemble_partial(stream=sD, stats=st[2])
            torch.cuda.synchronize()
            dist.barrier()   # every rank's V stores and D2 partial are complete
            # the cross-rank sum of D2 and the curl transform of this rank's blocks in one
            # kernel (partials read over peer memory)
            rpd.combine(outV, outD)
            torch.cuda.synchronize()
            dist.barrier()   # no rank reads a partial any more
            return
        elif stats is None:
            # the three operators on concurrent streams (public API assemble_all)
            hb.assemble_all(mesh, tg, params, q, d_range=(d0, d1), out={"V": outV, "K": outK, "D": outD})
            return
        else:
            _assemble_operator(0, False, False, True, mesh, tg, params, q, None, d_range=(d0, d1), out=outV,
                               stats=st[0])
            _assemble_operator(1, False, True, False, mesh, tg, params, q, None, d_range=(d0, d1), out=outK,
                               stats=st[1])
            _assemble_operator(2, True, True, True, mesh, tg, params, q, None, d_range=(d0, d1), out=outD,
                               stats=st[2])
        curl_combine_into(tabs, outV, outD, outD, params.alpha)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    peak = fp64_peak(torch, _native) if rank == 0 else None

    # ---- timed region: K steps, events per step, L2 flushed between steps ----
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
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    n_entries = conf["entries_per_step"]   # all ranks together
    value = n_entries / (ms_per_step * 1e-3)

    # ---- kernel timing pass (stats: events around every launch, sync per call) ----
    stats = [_native.AssemblyStats() for _ in range(3)]
    n_stat = max(1, args.steps // 2)
    for _ in range(n_stat):
        flush.fill_(1)
        step(stats)
    torch.cuda.synchronize()
    if rows_mode:
        dist.barrier()
        peersV.close()
        peersK.close()
        rpd.close()

    # ---- e2e: public API, host buffers, copies inside the timed region ----
    Hpin = hbdev.pin_host_tables(hbdev.host_tables(mesh, q))
    pinV = torch.empty(outV.shape, dtype=torch.float64).pin_memory()
    pinK = torch.empty(outK.shape, dtype=torch.float64).pin_memory()
    pinD = torch.empty(outD.shape, dtype=torch.float64).pin_memory()

    e2e_mode = os.environ.get("HB_E2E_MODE", "seq")   # "all": assemble_all(host_out) -- measured slower (6.4 vs 6.0 ms)
    _sl = os.environ.get("HB_E2E_SLABS", "4")   # a count of equal-work slabs, or work fractions "a,b,c"
    e2e_slabs = [float(x) for x in _sl.split(",")] if "," in _sl else int(_sl)

    def e2e_step():
        # mesh tables re-uploaded from pinned host memory every step
        hbdev.drop_device_tables(mesh)
        if e2e_mode == "all":
            # public assemble_all: V, K, D on concurrent streams (V's at high priority, in
            # row slabs), every output copied back as soon as it (or its slab / chunk) is formed
            ops = hb.assemble_all(mesh, tg, params, q, d_range=(d0, d1), host_out={"V": pinV, "K": pinK, "D": pinD},
                                  v_slabs=e2e_slabs)
            evs = [ops[n].host_copy[1] for n in ("V", "K", "D")]
        else:
            # sequential public calls: V's copy-back overlaps K, K's overlaps D
            V = hb.assemble_single_layer(mesh, tg, params, q, d_range=(d0, d1), host_out=pinV,
                                         host_out_slabs=e2e_slabs)
            K = hb.assemble_double_layer(mesh, tg, params, q, d_range=(d0, d1), host_out=pinK)
            D = hb.assemble_hypersingular(mesh, tg, params, q, single_layer=V, d_range=(d0, d1), host_out=pinD)
            evs = [V.host_copy[1], K.host_copy[1], D.host_copy[1]]
        for ev in evs:
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

    if rank != 0:
        if world > 1:
            dist.barrier()
        return
    clocks = clk.summary()

    # ---- roofline: issued FP64 of the pair kernels (ncu pass, this run) over live launch times ----
    live = {nm: {"pair_ms_per_call": st.pair_ms / n_stat, "pair_launches_per_call": st.pair_launches / n_stat,
                 "finalize_ms_per_call": st.finalize_ms / n_stat}
            for nm, st in zip(("V", "K", "D2"), stats)}
    hw = None if (args.no_ncu or world > 1) else pair_kernel_hw(ncu_pass("c2", "k_pairs"))
    kernels = {}
    for nm in ("V", "K", "D2"):
        ent = dict(live[nm])
        ent["algorithmic"] = algorithmic_rate(hb, mesh, nm, tg.n_steps, live[nm]["pair_ms_per_call"])
        if hw and nm in hw:
            h = hw[nm]
            ach = h["issued_fp64_flop"] / (live[nm]["pair_ms_per_call"] * 1e-3) / 1e12
            ent.update({"issued_fp64_flop_per_call": h["issued_fp64_flop"], "achieved_tflops": ach,
                        "frac": ach / peak if peak else None, "ncu_issued_tflops": h["ncu_issued_tflops"],
                        "ncu_ms": h["ncu_ms"], "fp64_shared_pipe_pct_ncu": h["fp64_shared_pipe_pct"],
                        "dram_bytes_per_call": h["dram_bytes"], "kernels": h["kernels"]})
        kernels[nm] = ent
    dom = max(("V", "K", "D2"), key=lambda nm: live[nm]["pair_ms_per_call"])
    dk = kernels[dom]
    n_l = max(1.0, live[dom]["pair_launches_per_call"])
    roofline = {"bound": "fp64", "kernel": f"pair kernels of {dom} (the longest pair-kernel time of a step)",
                "achieved": dk.get("achieved_tflops"), "peak": peak, "unit": "TFLOP/s", "frac": dk.get("frac"),
                "traffic": (dk["dram_bytes_per_call"] / n_l) if "dram_bytes_per_call" in dk else None,
                "avg_launch_ms": live[dom]["pair_ms_per_call"] / n_l,
                "peak_source": "measured in-run (hb_fp64_probe DFMA loop; MEASURED_PEAKS.json has no FP64 entry)",
                "definition": "achieved = issued FP64 flops per call (2 DFMA + DMUL + DADD thread instructions + "
                              "512 per DMMA warp instruction, counted by an ncu pass over the same workload in this "
                              "run) / the call's pair-kernel time measured live with CUDA events; traffic = DRAM "
                              "bytes per launch from the same pass",
                "source": "ncu counter pass in this run" if hw else "unavailable (ncu pass did not run)",
                "kernels": kernels}
    paths = (measure_paths(torch, hb, mesh, tg, params, q, outV, outK, cpu=not args.no_cpu_baseline,
                           hw=None if args.no_ncu else ncu_pass("c4", "k_represent|k_potential"), peak=peak)
             if (world == 1 and not args.no_paths) else None)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        ref = CpuReference(mesh, tg, params, threads)
        ref.pass_sample()                                   # page-in / thread start
        t_pass = statistics.median(ref.pass_sample() for _ in range(3))
        t_full = ref.full_assembly()
        cpu = {"value": n_entries / t_full, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": "one full config-2 assembly (V, K, D2: 33 delta-passes each, + the curl combine of the 32 "
                         f"blocks), measured: {t_full:.2f} s (oracle/heatbem_oracle.c, the port of the reference's "
                         f"_toeplitz_pass, {threads} OpenMP threads, tables built outside the timed region)",
               "full_assembly_s": t_full,
               "pass_sample_value": ref.pass_sample_entries(n_entries) / t_pass,
               "pass_sample_note": "one delta-pass each of V, K, D2 + one curl block, x (E_t + 1): agrees with the "
                                   "measured full assembly when the pass work is uniform"}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: BASELINE config-2 mesh and time grid generated in-run (no dataset)",
        "config": conf,
        "parallelism": (f"x{world}: V/K pair work split by balanced test-row ranges over all blocks, stored into the "
                        "d-owner's shard over NVLink peer memory; D2 split by element rows into full-size partials "
                        "that each rank's curl kernel reads over peer memory and sums for its own blocks")
        if rows_mode else f"d-sharded x{world} (contiguous time-difference blocks per rank)",
        "l2": "flushed between timed steps (256 MiB device write, outside the events)",
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": ("public API assemble_all(host_out=...): V, K, D on concurrent streams (V's at high "
                         "priority)" if e2e_mode == "all" else
                         "public API assemble_single_layer / assemble_double_layer / assemble_hypersingular with "
                         "host_out") + "; mesh tables re-uploaded from pinned host memory and all blocks copied to "
                        "pinned host memory every step (V in work-balanced test-row slabs as they complete, K when "
                        "done, D in block chunks as the curl combine forms them); the step ends when the last copy "
                        "is done"},
        "clocks": clocks,
        "paths": paths,
        "gpu_launches": int(round(sum(st.launches for st in stats) / n_stat + 1)) * args.steps * world,
        "impl": "native",
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()


def run_native_large(args, rank, world, local_rank):
    """Configs 3 and 5: every rank assembles its contiguous range of blocks d
    (block_range) of each operator -- no collective -- in window-aligned
    d-chunks into reused buffers where the range does not fit one GPU; D per
    chunk as D2 + curl(V) of the same blocks.  value = all entries / max-over-
    ranks time of the whole operator set."""
    import torch
    import torch.distributed as dist

    cfg = {"config": args.config, "level": args.level, "E_t": args.et}
    torch.cuda.set_device(local_rank)
    hb, mesh, tg, params = setup(cfg)
    conf = config_dict(cfg, mesh, tg)
    c = CONFIGS[args.config]
    from paper_2102_09811_b200 import _native, device as hbdev
    from paper_2102_09811_b200 import distributed as Dm
    from paper_2102_09811_b200.assembly import _assemble_operator, curl_combine_into

    _native.require_cuda()
    q = hb.QuadratureConfig()
    E, N, Et = mesh.n_triangles, mesh.n_vertices, tg.n_steps
    d0, d1 = Dm.block_range(rank, world, Et)
    dev = torch.device("cuda", local_rank)
    tabs = hbdev.device_tables(mesh, q, dev)
    # V chunk buffer: 40 GB where D shares the pool (config 5: 33-block chunks; larger ones
    # squeeze the staging workspace: 57 / 82 blocks measured 4.74 / 5.99 s against 4.55 s),
    # 110 GB for V and K alone (config 3: whole 32-block windows, 5.03 s against 6.71 s
    # with 11-block chunks that re-evaluate the window's gaps)
    budget = float(os.environ.get("HB_BENCH_CHUNK_BYTES", 40e9 if "D" in c["ops"] else 110e9))
    ch = max(1, int(budget // (E * E * 8)))

    def rank_chunks(max_blocks):
        """the rank's blocks in chunks that end on window edges (no extra gap slots)"""
        return [(max(a, d0), min(b, d1)) for a, b in Dm.aligned_chunks(Et, max_blocks) if b > d0 and a < d1]

    chunks = rank_chunks(ch)
    # K: one 32-slot window per chunk, so that its staging for ALL test rows fits beside the
    # output and the dual-orientation body evaluates each separated pair once
    kchunks = rank_chunks(32)
    nb_vd = max(b - a for a, b in chunks)
    nb_k = max(b - a for a, b in kchunks)
    # one pool, viewed as the V and D chunk buffers, then as K's (never live together):
    # K's all-rows staging (32 blocks: 116 GB at config 5) fits beside it
    n_vd = nb_vd * E * E + (nb_vd * N * N if "D" in c["ops"] else 0)
    pool = torch.empty(max(n_vd, nb_k * E * N), dtype=torch.float64, device=dev)
    bufs = {"VD": (pool[:nb_vd * E * E].view(nb_vd, E, E),
                   pool[nb_vd * E * E:n_vd].view(nb_vd, N, N) if "D" in c["ops"] else None),
            "K": pool[:nb_k * E * N].view(nb_k, E, N)}

    def buffers(kind):
        return bufs[kind]

    def step():
        bufV, bufD = buffers("VD")
        for a, b in chunks:
            n = b - a
            _assemble_operator(0, False, False, True, mesh, tg, params, q, None, d_range=(a, b), out=bufV[:n])
            if bufD is not None:
                _assemble_operator(2, True, True, True, mesh, tg, params, q, None, d_range=(a, b), out=bufD[:n])
                curl_combine_into(tabs, bufV[:n], bufD[:n], bufD[:n], params.alpha)
        bufK = buffers("K")
        for a, b in kchunks:
            _assemble_operator(1, False, True, False, mesh, tg, params, q, None, d_range=(a, b), out=bufK[:b - a])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = []
    gpu = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[0]) if world == 1 else local_rank
    with ClockSampler(gpu) as clk:
        for _ in range(args.steps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step()
            e.record()
            e.synchronize()
            ms.append(s.elapsed_time(e))
    t = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    bufs.clear()
    del pool
    torch.cuda.empty_cache()
    solve = large_solve(args, torch, dist, hb, mesh, tg, params, q, world, dev) if args.config == 5 else None
    if rank != 0:
        return
    out = {"metric": METRIC, "value": conf["entries_per_step"] / (ms_per_step * 1e-3), "unit": UNIT,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": f"synthetic: BASELINE config-{args.config} mesh generated in-run", "config": conf,
           "parallelism": f"d-sharded x{world}: blocks [d0, d1) per rank, V and D in window-aligned chunks of <= {ch} "
                          "blocks, K of <= 32",
           "clocks": clk.summary(), "impl": "native"}
    if solve is not None:
        out["solve"] = solve
    print(json.dumps(out), flush=True)


def large_solve(args, torch, dist, hb, mesh, tg, params, q, world, dev):
    """Config 5's Dirichlet solve (distributed.dirichlet_solve_row_sharded):
    V and K row-sharded across the ranks (peer stores), rhs = 1/2 M g + K g
    with one all-gather, FGMRES + forward substitution with the density
    all-gathers (NCCL).  Needs the V and K row shards resident: skipped when
    they do not fit (one GPU: 309 + 155 GB).  Times are device times, max over
    ranks; one run (the assembly inside is the same work as the timed step)."""
    from paper_2102_09811_b200 import distributed as Dm

    E, N, Et = mesh.n_triangles, mesh.n_vertices, tg.n_steps
    need = Et * E * (E + N) * 8 / world * 1.08 + 20e9      # shards + staging / tables headroom
    total = torch.cuda.get_device_properties(dev).total_memory
    if need > total and not os.environ.get("HB_BENCH_EMULATE"):
        return {"skipped": f"V + K row shards need {need / 1e9:.0f} GB per rank at N={world} "
                           f"(device: {total / 1e9:.0f} GB); run with --gpus >= 4"}
    datum = hb.HeatKernelDatum((1.5, 1.5, 1.5), 1.0, 0.1)   # G(x - y0, t + 0.1): BASELINE config 2/5 data
    tm = {}
    if world > 1:
        dist.barrier()
    x, rep, _ = Dm.dirichlet_solve_row_sharded(mesh, tg, params, q, datum, rel_tol=1e-10, timings=tm)
    keys = ("assemble_V", "assemble_K", "rhs", "solve")
    t = torch.tensor([tm[k] for k in keys], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res = {k + "_ms": float(v) for k, v in zip(keys, t.tolist())}
    res.update({"iterations": rep.iterations, "residual": rep.residual, "converged": rep.converged,
                "layout": f"V, K row-sharded x{world} (rows block_range(rank)); rhs and density all-gathers",
                "x_norm": float(torch.linalg.norm(x))})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("native", "reference"), default="native")
    ap.add_argument("--config", type=int, choices=(2, 3, 5), default=2)
    ap.add_argument("--level", type=int, default=None, help="override the mesh refinement level (emulation runs)")
    ap.add_argument("--et", type=int, default=None, help="override the number of time steps (emulation runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-paths", action="store_true", help="skip the potentials / solve measurements")
    ap.add_argument("--no-ncu", action="store_true", help="skip the ncu counter pass (roofline from live times only)")
    ap.add_argument("--parallel", choices=("rows", "d"), default="rows",
                    help="config 2, N > 1: split V/K pair work by test rows (peer stores) or everything by d")
    ap.add_argument("--ncu-child", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ncu_child:
        ncu_child(args.ncu_child)
        return
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
        import datetime

        # (a rank that dies must not leave the others in a collective for NCCL's default 10 minutes)
        dist.init_process_group("gloo" if os.environ.get("HB_BENCH_EMULATE") else "nccl",
                                timeout=datetime.timedelta(seconds=int(os.environ.get("HB_BENCH_TIMEOUT_S", "300"))))
        if os.environ.get("HB_BENCH_EMULATE"):
            local_rank = 0
    try:
        if args.config == 2:
            run_native_c2(args, rank, world, local_rank)
        else:
            run_native_large(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

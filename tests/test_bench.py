"""bench.py contract: the reference arm (CPU, here) and the N > 1 paths as
control-flow checks (HB_BENCH_EMULATE: every rank on cuda:0 over gloo -- never
a measurement) on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_reference_arm_full_assembly_per_step():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["unit"] == "entries/s" and d["higher_is_better"] is True
    n = d["config"]["entries_per_step"]
    assert n == 32 * (768 * 768 + 768 * 386 + 386 * 386)
    # one step is the whole workload: value x step time = the step's entries
    assert abs(d["value"] * d["ms_per_step"] * 1e-3 - n) <= 1e-6 * n
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def _torchrun(args, n=2, timeout=900):
    env = dict(os.environ, HB_BENCH_EMULATE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29731", os.path.join(ROOT, "bench.py"),
           "--gpus", str(n)] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    return _last_json(r.stdout)


@pytest.mark.gpu
def test_emulated_two_rank_config5_pipeline():
    """config-5 harness at a small size: d-sharded V / K / D chunks, then the
    row-sharded Dirichlet solve with the density all-gathers."""
    d = _torchrun(["--config", "5", "--level", "1", "--et", "8", "--steps", "1", "--warmup", "1"])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["E_t"] == 8
    s = d["solve"]
    assert s["converged"] and s["residual"] <= 1e-9 and s["iterations"] >= 1


@pytest.mark.gpu
def test_emulated_two_rank_config2_rows():
    """config-2 N = 2 path at a small size: row-split V / K pair work with peer
    stores into the d-owners' shards, d-local D."""
    d = _torchrun(["--level", "1", "--et", "8", "--steps", "1", "--warmup", "1", "--no-paths", "--no-ncu",
                   "--no-cpu-baseline"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["E_t"] == 8

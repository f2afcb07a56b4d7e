"""Roofline numbers of every kernel in an .ncu-rep: duration, DRAM bytes,
FP64 pipe activity and the ISSUED FP64 flop rate (2 DFMA + DMUL + DADD
thread instructions, from the SASS op counters) -- the hardware view next to
bench.py's algorithmic flop count.  python tools/ncu_roofline.py REP [--json]"""
import csv, json, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]


def val(row, key):
    s = row[h.index(key)].replace(",", "")
    return float(s) if s not in ("", "n/a") else float("nan")


out = []
for row in r[2:]:
    if len(row) != len(h):
        continue
    t_ns = val(row, "gpu__time_duration.sum")
    t_s = t_ns * {"s": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}[units[h.index("gpu__time_duration.sum")]]
    cyc = val(row, "sm__cycles_elapsed.avg")
    per = {op: val(row, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") * cyc
           for op in ("dfma", "dmul", "dadd")}
    flops = 2 * per["dfma"] + per["dmul"] + per["dadd"]
    dr = val(row, "dram__bytes_read.sum"), val(row, "dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = dr[0] * scale[units[h.index("dram__bytes_read.sum")]] + dr[1] * scale[units[h.index("dram__bytes_write.sum")]]
    out.append({"kernel": row[h.index("Kernel Name")], "ms": t_s * 1e3, "dram_bytes": dram,
                "fp64_pipe_pct": val(row, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "issue_pct": val(row, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "issued_fp64_tflops": flops / t_s / 1e12, "dfma": per["dfma"], "dmul": per["dmul"],
                "dadd": per["dadd"]})
if "--json" in sys.argv:
    print(json.dumps(out, indent=1))
else:
    for o in out:
        print(f"{o['kernel'][:60]:60s} {o['ms']:7.3f} ms  DRAM {o['dram_bytes'] / 1e6:8.1f} MB  "
              f"FP64 pipe {o['fp64_pipe_pct']:5.1f} %  issue {o['issue_pct']:5.1f} %  "
              f"issued FP64 {o['issued_fp64_tflops']:6.2f} TFLOP/s")

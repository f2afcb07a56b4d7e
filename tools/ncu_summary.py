"""Summarise an .ncu-rep: headline metrics, smem/global wavefronts, and
warp-stall reasons aggregated over the source page (top lines too)."""
import csv, subprocess, sys, collections

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k:60s} {v[i]} {r[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
stall_cols = [i for i, c in enumerate(hh) if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.Counter()
data = [x for x in rows[2:] if len(x) == len(hh)]
for x in data:
    for i in stall_cols:
        try: agg[hh[i]] += int(x[i] or 0)
        except ValueError: pass
tot = sum(agg.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {100*c/tot:.0f}%" for k, c in agg.most_common(8)))
si = hh.index("Warp Stall Sampling (All Samples)")
top = sorted(data, key=lambda x: -int(x[si] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for x in top:
    print(f"{x[si]:>8s} {x[1][:80]}")

"""Summarise an .ncu-rep: per captured kernel, headline metrics, smem/global
wavefronts, and warp-stall reasons aggregated over the source page (top
lines too).  Handles reports holding several kernels.

  python tools/ncu_summary.py REP [N_TOP]
"""
import csv, subprocess, sys, collections

rep = sys.argv[1]
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size"]
name_col = h.index("Kernel Name") if "Kernel Name" in h else None
for v in r[2:]:
    if len(v) != len(h):
        continue
    print("==", v[name_col] if name_col is not None else "kernel")
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"   {k:62s} {v[i]} {units[i]}")

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
sections, cur = [], None
for x in rows:
    if x and x[0] == "Kernel Name":
        cur = [x[1], None, []]
        sections.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = x
    elif cur is not None:
        cur[2].append(x)
for name, hh, body in sections:
    print("== source page:", name)
    stall_cols = [i for i, c in enumerate(hh) if c.startswith("stall_") and "Not Issued" not in c]
    data = [x for x in body if len(x) == len(hh)]
    agg = collections.Counter()
    for x in data:
        for i in stall_cols:
            try:
                agg[hh[i]] += int(x[i] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    print("   stalls:", ", ".join(f"{k[6:]} {100*c/tot:.0f}%" for k, c in agg.most_common(8)))
    si = hh.index("Warp Stall Sampling (All Samples)")
    top = sorted(data, key=lambda x: -int(x[si] or 0))[:n_top]
    for x in top:
        print(f"   {x[si]:>8s} {x[1][:80]}")

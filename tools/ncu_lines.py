"""Per-source-line instruction and stall-sample shares of one kernel from an
ncu report (ncu --page source --print-source cuda,sass; needs -lineinfo):
python tools/ncu_lines.py REPORT [kernel-regex] [top]"""
import csv, subprocess, sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["-k", "regex:" + sys.argv[2]]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(args, capture_output=True, text=True).stdout
fname, rows = "?", []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0].isdigit() and len(r) > 8 and r[2] == "-":
        try:
            rows.append((fname, int(r[0]), float(r[7] or 0), float(r[4] or 0), r[1].strip()[:100]))
        except ValueError:
            pass
ti = sum(x[2] for x in rows) or 1
ts = sum(x[3] for x in rows) or 1
print(f"total warp instructions {ti:.3e}")
for f, ln, ie, sm, src in sorted(rows, key=lambda x: -x[2])[:top]:
    print(f"{f[:16]:16s}{ln:5d} inst {100 * ie / ti:5.1f}% stall {100 * sm / ts:5.1f}%  {src}")

"""Per-source-line stall reasons of an .ncu-rep: top lines by sampled stalls
with the dominant reasons (cuda,sass correlation page)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons}
tot_i = hdr.index("Warp Stall Sampling (All Samples)")
file_lines = collections.Counter()
per = collections.defaultdict(collections.Counter)
src = {}
cur = None
fname = "?"
for r in rows:
    if r and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < len(hdr) or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1]
    try:
        file_lines[cur] += int(r[tot_i] or 0)
        for h in reasons:
            per[cur][h] += int(r[idx[h]] or 0)
    except ValueError:
        pass
tot = sum(file_lines.values()) or 1
agg = collections.Counter()
for c in per.values():
    agg.update(c)
print("overall:", ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in agg.most_common(6)))
for key, c in file_lines.most_common(n):
    top = ", ".join(f"{k[6:]} {v}" for k, v in per[key].most_common(3))
    print(f"{key[0][:14]:14s}{key[1]:5d} {100 * c / tot:5.1f}% | {top:40s} | {src.get(key, '').strip()[:70]}")

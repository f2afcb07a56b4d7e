"""Per-CUDA-source-line instruction counts and stall samples of an .ncu-rep
(source/SASS correlation page)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines, cur, src = collections.Counter(), None, {}
stall = collections.Counter()
for r in rows:
    if len(r) < len(hdr) or r[0] == "Line No":
        continue
    if r[0]:
        cur = int(r[0]); src[cur] = r[1]
    try:
        lines[cur] += int(r[ie] or 0); stall[cur] += int(r[ss] or 0)
    except ValueError:
        pass
tot, tst = sum(lines.values()) or 1, sum(stall.values()) or 1
for ln, c in sorted(lines.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{ln:5d} {100*c/tot:5.1f}% instr {100*stall[ln]/tst:5.1f}% stall | {src.get(ln,'').strip()[:90]}")

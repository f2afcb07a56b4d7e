"""Per-opcode executed-instruction mix and stall share of every kernel in an
.ncu-rep (source page), e.g. python tools/ncu_mix.py rep.ncu-rep [N]."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
secs, cur = [], None
for x in rows:
    if x and x[0] == "Kernel Name":
        cur = [x[1], None, []]
        secs.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = x
    elif cur is not None:
        cur[2].append(x)
seen = set()
for name, hh, body in secs:
    if name in seen:
        continue
    seen.add(name)
    ie, si = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
    agg, st = collections.Counter(), collections.Counter()
    for x in body:
        if len(x) != len(hh):
            continue
        op = x[1].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        op = op.split()[0].split(".")[0]
        agg[op] += int(x[ie] or 0)
        st[op] += int(x[si] or 0)
    tot, stt = sum(agg.values()) or 1, sum(st.values()) or 1
    print(name[:70], f"total warp-instr {tot / 1e6:.1f}M")
    for op, c in agg.most_common(n_top):
        print(f"   {op:10s} {c / 1e6:8.2f}M {100 * c / tot:5.1f}%   stall-samples {100 * st[op] / stt:5.1f}%")

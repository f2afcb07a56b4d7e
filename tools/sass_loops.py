import re, sys, collections
lines = open(sys.argv[1]).read().split("\n")
start = int(sys.argv[2]); end = int(sys.argv[3])
ins = []
for ln in lines[start:end]:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`?\(?\.?L_x_\d+\)?|0x([0-9a-f]+))", txt)
    if "BRA" in txt:
        t = re.search(r"0x([0-9a-f]+)", txt)
        if t:
            tgt = int(t.group(1), 16)
            if tgt < a and tgt in addr:
                loops.append((addr[tgt], i))
for lo, hi in loops:
    body = [t for _, t in ins[lo:hi + 1]]
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in body)
    fp64 = sum(v for k, v in ops.items() if k in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX"))
    if fp64 < 20: continue
    print(f"loop {ins[lo][0]:#x}-{ins[hi][0]:#x}: {len(body)} instr, fp64 {fp64}:", dict(ops.most_common(18)))

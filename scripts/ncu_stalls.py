#!/usr/bin/env python
"""Warp-stall samples of an ncu report aggregated by SASS opcode (and, with a
window size, by consecutive instruction windows).

    python scripts/ncu_stalls.py gpurun_out/prof.ncu-rep [WINDOW]
"""
import csv, io, subprocess, sys, collections
src = sys.argv[1]
if src.endswith(".ncu-rep"):
    txt = subprocess.run(["ncu", "-i", src, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
else:
    txt = open(src).read()
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
iS = hdr.index("Source"); iN = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
byop = collections.Counter(); bystall = collections.defaultdict(collections.Counter)
seq = []
for r in rows[2:]:
    if len(r) <= iN: continue
    src = r[iS].split()
    if not src: continue
    op = src[1] if src[0].startswith("@") else src[0]
    n = int(r[iN] or 0)
    byop[op] += n
    for i in stall_cols:
        v = int(r[i] or 0)
        if v: bystall[op][hdr[i]] += v
    seq.append((r[0], r[iS].strip(), n, int(r[iE] or 0)))
tot = sum(byop.values())
for op, n in byop.most_common(15):
    print(f"{op:28s} {100*n/tot:5.1f}%  ", dict(bystall[op].most_common(4)))
# windows: sum of samples in consecutive chunks of 200 instrs
if len(sys.argv) > 2:
    W = int(sys.argv[2])
    for b in range(0, len(seq), W):
        ch = seq[b:b+W]
        s = sum(x[2] for x in ch)
        ops = collections.Counter(x[1].split()[0] if not x[1].startswith('@') else x[1].split()[1] for x in ch)
        print(b, f"{100*s/tot:5.1f}%", ops.most_common(5))

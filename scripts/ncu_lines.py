#!/usr/bin/env python
"""Warp-stall samples of one kernel in an ncu report, aggregated by CUDA source line.

    python scripts/ncu_lines.py <report.ncu-rep> <libwally.so> <mangled kernel name> [top]

SASS addresses from the report's source page are mapped to source lines with
the line table of the kernel's cubin (nvdisasm -g of `cuobjdump -xelf`), which
needs a -lineinfo build (the library's default)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(lib, kernel):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    for f in sorted(os.listdir(d)):
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, f)], capture_output=True, text=True).stdout
        m = re.search(r"\.text\." + re.escape(kernel) + r":\n(.*?)(?=\n\s*\.section|\Z)", txt, re.S)
        if not m:
            continue
        table, cur = {}, None
        for ln in m.group(1).split("\n"):
            fm = re.search(r'//## File "(.*?)", line (\d+)', ln)
            if fm:
                cur = (os.path.basename(fm.group(1)), int(fm.group(2)))
                continue
            am = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if am and cur:
                table[int(am.group(1), 16)] = cur
        return table
    raise SystemExit(f"{kernel} not found in {lib}")


def main():
    rep, lib, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    table = line_table(lib, kernel)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ia, iN = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    by_line = collections.Counter()
    by_reason = collections.defaultdict(collections.Counter)
    base = None
    tot = 0
    for r in rows[2:]:
        if len(r) <= iN or not r[ia]:
            continue
        a = int(r[ia], 16)
        base = a if base is None else min(base, a)
    for r in rows[2:]:
        if len(r) <= iN or not r[ia]:
            continue
        off = int(r[ia], 16) - base
        key = table.get(off, ("?", 0))
        n = int(r[iN] or 0)
        by_line[key] += n
        tot += n
        for i in stall_cols:
            v = int(r[i] or 0)
            if v:
                by_reason[key][hdr[i]] += v
    src = {}
    for (f, l) in by_line:
        if f != "?" and f not in src:
            for d in ("paper_2406_06761_b200/csrc",):
                p = os.path.join(d, f)
                if os.path.exists(p):
                    src[f] = open(p).read().split("\n")
    for (f, l), n in by_line.most_common(top):
        text = src.get(f, [""] * (l + 1))[l - 1].strip() if f in src and l > 0 else ""
        reasons = ", ".join(f"{k[6:]} {v * 100 // max(n, 1)}%" for k, v in by_reason[(f, l)].most_common(3))
        print(f"{n * 100 / tot:5.1f}%  {f}:{l:<5d} {text[:70]:70s}  [{reasons}]")


if __name__ == "__main__":
    main()

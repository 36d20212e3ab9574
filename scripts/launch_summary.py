#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel counts, total device time and share of the timed step.

    python scripts/launch_summary.py gpurun_out/launches.csv [--skip-prefix encode_kernel,...]
"""
import collections
import csv
import io
import sys


def main():
    path = sys.argv[1]
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        ns = float(r["Metric Value"].replace(",", ""))
        d = per.setdefault(name, [0, 0.0, r["Grid Size"], r["Block Size"]])
        d[0] += 1
        d[1] += ns
    # the step's kernels: everything but the one-time encode and torch's own kernels
    step = {k: v for k, v in per.items() if k.startswith("wally::") and "encode" not in k}
    tot = sum(v[1] for v in step.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'ms/launch':>10s} {'share':>7s}  grid / block")
    for k, (n, ns, grid, blk) in per.items():
        share = f"{100 * ns / tot:6.2f}%" if k in step else "   n/a"
        print(f"{k[:60]:60s} {n:8d} {ns / 1e6:10.3f} {ns / 1e6 / n:10.4f} {share}  {grid} / {blk}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list with time + DRAM + FMA-heavy metrics.

    python scripts/simd_launches.py gpurun_out/simd_launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
data = rows[hi + 1:]
iK, iM, iV, iID = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = collections.defaultdict(dict)
for r in data:
    if len(r) <= iV:
        continue
    per[r[iID]][r[iM]] = float(r[iV].replace(',', ''))
    per[r[iID]]['k'] = r[iK]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
for k, v in per.items():
    name = v['k'].split('(')[0][:52]
    a = agg[name]
    t = v.get('gpu__time_duration.sum', 0)
    a[0] += 1
    a[1] += t
    a[2] += v.get('dram__bytes_read.sum', 0)
    a[3] += v.get('dram__bytes_write.sum', 0)
    a[4] += v.get('sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed', 0) * t
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':52s} {'n':>5s} {'ms':>9s} {'share':>6s} {'R GB':>7s} {'W GB':>6s} {'fmaheavy':>8s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:52s} {a[0]:5d} {a[1] / 1e6:9.3f} {100 * a[1] / tot:5.1f}% {a[2] / 1e9:7.2f} {a[3] / 1e9:6.2f} "
          f"{a[4] / max(a[1], 1):7.1f}%")

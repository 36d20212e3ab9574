#!/usr/bin/env python
"""Record one fused-kernel ncu capture in profiles/ncu_fused_traffic.json (read by bench.py
into roofline.traffic).

    python scripts/update_traffic.py <config> <report.ncu-rep> [round]

The capture is `ncu --set full --clock-control none -k regex:eval_kernel -s 1 -c 1` of
`python bench.py --config <config> --steps 1 --warmup 1 --no-e2e --no-cpu-baseline`."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    cfg, rep = sys.argv[1], sys.argv[2]
    rnd = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, vals = rows[0], rows[2]
    m = dict(zip(hdr, vals))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    units = dict(zip(hdr, rows[1]))

    def val(k):
        return float(m[k].replace(",", "")) * scale.get(units[k], 1)

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    t = float(m["gpu__time_duration.sum"].replace(",", "")) * {"ms": 1, "us": 1e-3, "ns": 1e-6}.get(
        units["gpu__time_duration.sum"], 1)
    p = os.path.join(ROOT, "profiles", "ncu_fused_traffic.json")
    d = json.load(open(p))
    d[cfg] = {"bytes": int(rd + wr), "read_GB": round(rd / 1e9, 3), "write_GB": round(wr / 1e9, 3),
              "kernel": m.get("Kernel Name", ""), "ncu_ms": round(t, 5),
              "issue_pct": float(m["sm__inst_issued.sum.pct_of_peak_sustained_active"]), "round": rnd}
    json.dump(d, open(p, "w"), indent=1)
    print(cfg, d[cfg])


if __name__ == "__main__":
    main()

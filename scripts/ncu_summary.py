#!/usr/bin/env python
"""Summarise an `ncu --set full` report of the fused kernel (run here, no GPU).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]

Prints the metrics the roofline argument uses (time, clock, pipe
utilisation, issue activity, DRAM bytes, shared-memory wavefronts/conflicts,
occupancy), the SASS opcode mix weighted by executed instructions and the
top warp-stall reasons."""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
    "sm__inst_issued.sum.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sass__inst_executed_local_loads", "lts__t_bytes.sum", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for i, h in enumerate(hdr):
        if h in KEYS or h.startswith("smsp__pcsamp_warps_issue_stalled_"):
            out[h] = (vals[i], units[i])
    return out


def opcode_mix(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr = rows[1]
    iE, iS = hdr.index("Instructions Executed"), hdr.index("Source")
    cnt = collections.Counter()
    tot = 0
    for r in rows[2:]:
        if len(r) <= iE or not r[iE]:
            continue
        n = int(r[iE])
        src = r[iS].split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        cnt[op] += n
        tot += n
    return tot, cnt


def main():
    rep = sys.argv[1]
    m = raw_metrics(rep)
    out = {"metrics": {k: v[0] + " " + v[1] for k, v in m.items() if not k.startswith("smsp__pcsamp")}}
    stalls = sorted(((float(v[0] or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for k, v in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not k.endswith("_not_issued")), reverse=True)
    tot_s = sum(s for s, _ in stalls) or 1
    out["stall_samples_pct"] = {k: round(100 * s / tot_s, 1) for s, k in stalls[:10]}
    tot, cnt = opcode_mix(rep)
    out["warp_instructions"] = tot
    out["opcode_mix_pct"] = {k: round(100 * v / tot, 2) for k, v in cnt.most_common(20)}
    for k, v in out["metrics"].items():
        print(f"{k:70s} {v}")
    print("stalls:", json.dumps(out["stall_samples_pct"]))
    print("opcodes:", json.dumps(out["opcode_mix_pct"]))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

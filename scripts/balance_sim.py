#!/usr/bin/env python
"""Multi-GPU load balance of the cluster-sharded path, computed on the host
from the real routing code (wally_assign_owners[_replicated] +
wally_route_plan): max/mean per-rank pair load (queries x P_c) of a BASELINE
batch, with disjoint and with replicated ownership.  The 1-GPU box cannot time
N > 1; this bounds the strong-scaling speedup (N / (max/mean)).

    python scripts/balance_sim.py [c3 c5 ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2406_06761_b200 import wally as W  # noqa: E402


def main():
    names = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
    print(f"{'config':6s} {'N':>3s} {'disjoint max/mean':>18s} {'bound':>7s} {'replicated max/mean':>20s} "
          f"{'bound':>7s} {'extra replicas':>15s}")
    for name in names:
        w = synth.WORKLOADS[name]
        ids = synth.query_clusters(w)
        sizes = np.full(w.num_clusters, w.cluster_size, np.uint32)
        P = -(-w.cluster_size // (w.n // w.d))
        weight = synth.cluster_popularity(w) * P
        for G in (1, 2, 4, 8):
            rows = []
            for owner in (W.wally_assign_owners(weight, G), W.wally_assign_owners_replicated(weight, G)):
                plan = W.wally_route_plan(ids, sizes, owner, w.n, w.d, G)
                pairs = np.array([sum(P for _ in plan.share(r)) for r in range(G)], dtype=np.float64)
                rows.append(pairs.max() / pairs.mean())
            extra = sum(bin(int(x)).count("1") for x in W.wally_assign_owners_replicated(weight, G)) - w.num_clusters
            print(f"{name:6s} {G:3d} {rows[0]:18.3f} {G / rows[0]:7.2f} {rows[1]:20.3f} {G / rows[1]:7.2f} {extra:15d}")


if __name__ == "__main__":
    main()

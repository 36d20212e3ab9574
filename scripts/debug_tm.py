"""Run one small eval configuration in this process and compare with the oracle (debug helper)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth
from tests import helpers as H

L, C, S, nq, fmt = (int(x) for x in sys.argv[1:6])
w = synth.scaled(synth.WORKLOADS["c2"], num_limbs=L, num_clusters=C, cluster_size=S, num_queries=nq)
ents = synth.cluster_entries(w)
ids = synth.query_clusters(w)
srv = H.make_server(w, ents, resp_format=fmt)
cts = synth.uniform_ciphertexts(w, srv.moduli)
try:
    resp, off = H.run_batch(srv, ids, cts)
except Exception as e:
    print("FAIL", sys.argv[1:], repr(e)[:120]); sys.exit(1)
from oracle import capi
bad = 0
for q in range(min(nq, 4)):
    c = int(ids[q]); pcs = capi.encode_cluster(ents[c], w.d, w.n); P = pcs.shape[0]
    want = H.oracle_pairs(srv.moduli, cts[q:q + 1], pcs, np.zeros(P), np.arange(P))
    for k in range(P):
        bad += not H.matches_oracle(H.response_of(resp, off, q, k, w.n, w.d, fmt), want[k], w.n, w.d, fmt)
print("OK" if bad == 0 else f"MISMATCH {bad}", sys.argv[1:])

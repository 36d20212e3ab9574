"""GPU parity at the BASELINE configurations' full sizes, in the bench's launch
configuration (the whole batch in one wally_eval_batch call), against the
oracle (SURVEY.md §8(c) floors):

  * c2: every one of its 131,072 (query, plaintext) pairs, word for word;
  * c3 (full / compact / compact_drop), c4 (compact / full), c5
    (compact_drop / full): a deterministic sample of >= 4,096 pairs that
    contains the first and the last (partial) plaintext of every sampled
    cluster, word for word;
  * every config: at least 24 queries replaced by real encryptions, enough
    that their responses number >= 1,000 (c5 has only 32
    plaintexts per cluster, so it takes 32), every third one a fake query
    (the zero vector, reading S14), and ALL their responses decrypted and compared with the plaintext dot products mod t ("decrypted
    scores equal the integer dot-product oracle ... exactly", SPEC.md:368;
    Alg 4).

Expected values come only from oracle/ (C, uint64 % arithmetic) on the
box's host cores.  The counts are printed.
"""
import os

import numpy as np
import pytest

import synth
from oracle import capi
from tests import helpers as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REAL = 24          # at least this many real encryptions per config (every third a fake / zero query)
MIN_DECRYPTS = 1000  # responses decrypted per config and format
MIN_PAIRS = 4096   # sampled pairs per (config, format) when not all pairs


def _run(name, fmt, all_pairs=False):
    w = synth.WORKLOADS[name]
    ents = synth.cluster_entries(w)
    ids = synth.query_clusters(w)
    srv = H.make_server(w, ents, resp_format=fmt)
    qs = srv.moduli
    E = w.n // w.d
    P = -(-w.cluster_size // E)
    wpp = H.words_per_pt(w.n, w.d, fmt)
    cores = len(os.sched_getaffinity(0))
    cts_dev = synth.uniform_ciphertexts_torch(w, qs)
    qv = synth.query_vectors(w, ids)
    n_real = max(REAL, -(-MIN_DECRYPTS // P))
    real = np.linspace(0, w.num_queries - 1, n_real).astype(np.int64)
    qv_real = qv[real].copy()
    qv_real[::3] = 0                                   # fake queries encrypt the zero vector
    rcts, keys = H.encrypt_queries(w, qs, qv_real, index_base=0)
    cts_dev[torch.from_numpy(real).cuda()] = torch.from_numpy(rcts.view(np.int32)).cuda()
    off = srv.response_layout(ids)
    resp = torch.empty(int(off[-1]), dtype=torch.int32, device="cuda")
    ws = srv.alloc_workspace(w.num_queries)
    srv.eval_batch(ids, cts_dev, resp, ws)
    srv.check_batch(ws)
    del ws

    def got_pair(q, k, host=None):
        b = int(off[q]) + int(k) * wpp
        g = host[b:b + wpp] if host is not None else resp[b:b + wpp].cpu().numpy().view(np.uint32)
        return g.reshape(2, w.n) if fmt == 0 else g

    checked = 0
    if all_pairs:
        host = resp.cpu().numpy().view(np.uint32)
        pcs_c = {}
        for qb in range(0, w.num_queries, 64):
            qsel = np.arange(qb, min(qb + 64, w.num_queries))
            cl = sorted(set(int(ids[q]) for q in qsel))
            for c in cl:
                if c not in pcs_c:
                    pcs_c[c] = capi.encode_cluster(ents[c], w.d, w.n)
            need = [(c, k) for c in cl for k in range(P)]
            pidx = {ck: i for i, ck in enumerate(need)}
            pcs = np.stack([pcs_c[c][k] for c, k in need])
            pq = np.repeat(np.arange(qsel.size), P)
            pk = np.tile(np.arange(P), qsel.size)
            cts_h = cts_dev[torch.from_numpy(qsel).cuda()].cpu().numpy().view(np.uint32)
            want = H.oracle_pairs(qs, cts_h, pcs, pq, [pidx[(int(ids[qsel[i]]), int(k))] for i, k in zip(pq, pk)],
                                  threads=cores)
            for i, (qi, k) in enumerate(zip(pq, pk)):
                assert H.matches_oracle(got_pair(qsel[qi], k, host), want[i], w.n, w.d, fmt), (name, qsel[qi], k)
                checked += 1
        assert checked == w.num_queries * P
    else:
        rng = np.random.default_rng(99)
        nq_s = -(-MIN_PAIRS // 3)
        qsel = np.unique(np.concatenate([real, rng.choice(w.num_queries, size=nq_s, replace=False)]))
        pq, pk = [], []
        for q in qsel:                                  # first and last (partial) plaintext of each
            pq += [q, q, q]
            pk += [0, P - 1, int(rng.integers(0, P))]
        pq, pk = np.array(pq), np.array(pk)
        assert pq.size >= MIN_PAIRS
        uq, inv = np.unique(pq, return_inverse=True)
        cts_h = cts_dev[torch.from_numpy(uq).cuda()].cpu().numpy().view(np.uint32)
        need = sorted(set((int(ids[q]), int(k)) for q, k in zip(pq, pk)))
        pidx = {ck: i for i, ck in enumerate(need)}
        pcs = np.stack([capi.encode_plaintext(ents[c][k * E:(k + 1) * E], w.d, w.n) for c, k in need])
        want = H.oracle_pairs(qs, cts_h, pcs, inv, [pidx[(int(ids[q]), int(k))] for q, k in zip(pq, pk)],
                              threads=cores)
        for i, (q, k) in enumerate(zip(pq, pk)):
            assert H.matches_oracle(got_pair(q, k), want[i], w.n, w.d, fmt), (name, fmt, q, k)
            checked += 1
        clusters = len(set(int(ids[q]) for q in qsel))
    # decrypt every response of the real (and fake) encryptions
    decrypted = dots = 0
    for i, q in enumerate(real):
        c = int(ids[q])
        for k in range(P):
            g = got_pair(q, k)
            if fmt:
                g = H.expand_compact(g, w.n, w.d, fmt, qs[0])
            dec = capi.decrypt_q0(qs[0], w.t, g, keys[i].s)
            cnt = min(E, w.cluster_size - k * E)
            want = (ents[c][k * E:k * E + cnt].astype(np.int64) @ qv_real[i].astype(np.int64)) % w.t
            assert np.array_equal(dec[np.arange(cnt) * w.d + w.d - 1].astype(np.int64), want), (name, q, k)
            decrypted += 1
            dots += cnt
    srv.close()
    del resp, cts_dev
    torch.cuda.empty_cache()
    mode = "all pairs" if all_pairs else f"{checked} sampled pairs over {clusters} clusters"
    print(f"\n{name} fmt={fmt}: {mode} bit-exact vs oracle; {decrypted} responses of {n_real} real encryptions "
          f"({-(-n_real // 3)} fake) decrypted, {dots} dot products exact")
    return checked, decrypted


def test_c2_all_pairs():
    checked, decrypted = _run("c2", 0, all_pairs=True)
    assert checked == 131072 and decrypted >= MIN_DECRYPTS


@pytest.mark.parametrize("name,fmt", [("c3", 0), ("c3", 1), ("c3", 2), ("c4", 1), ("c4", 0), ("c5", 2), ("c5", 0)])
def test_full_config_sampled(name, fmt):
    checked, decrypted = _run(name, fmt)
    assert checked >= MIN_PAIRS and decrypted >= MIN_DECRYPTS

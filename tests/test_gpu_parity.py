"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: bit-exact on every response word (integer path).  Inputs are seeded
(synth/); expected values come only from oracle/.
"""
import numpy as np
import pytest

import synth
from oracle import capi
from tests import helpers as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2406_06761_b200.wally import WallyError, WallyServer  # noqa: E402


# --------------------------------------------------------------------------
# NTT kernels (step a2 and the inverse used inside the fused kernel)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n,L", [(1024, 1), (2048, 2), (4096, 2), (4096, 3), (8192, 4)])
def test_ntt_roundtrip_and_product(n, L):
    srv = WallyServer(n, L, d=n // 32)
    qs = srv.moduli
    rng = np.random.default_rng(n + L)
    count = 3
    a = np.stack([np.stack([rng.integers(0, q, size=n) for q in qs]) for _ in range(count)]).astype(np.uint32)
    b = np.stack([np.stack([rng.integers(0, q, size=n) for q in qs]) for _ in range(count)]).astype(np.uint32)
    da = torch.from_numpy(a.view(np.int32)).cuda()
    db = torch.from_numpy(b.view(np.int32)).cuda()
    fa, fb, back = torch.empty_like(da), torch.empty_like(db), torch.empty_like(da)
    srv.ntt_forward(da, fa, count)
    srv.ntt_inverse(fa, back, count)
    assert np.array_equal(back.cpu().numpy().view(np.uint32), a)
    # forward values are in [0, 4q)
    fa_h = fa.cpu().numpy().view(np.uint32).astype(np.uint64)
    srv.ntt_forward(db, fb, count)
    fb_h = fb.cpu().numpy().view(np.uint32).astype(np.uint64)
    qv = np.array(qs, dtype=np.uint64)[None, :, None]
    assert (fa_h < 4 * qv).all()
    prod = (fa_h % qv) * (fb_h % qv) % qv
    dp = torch.from_numpy(prod.astype(np.uint32).view(np.int32)).cuda()
    out = torch.empty_like(dp)
    srv.ntt_inverse(dp, out, count)
    got = out.cpu().numpy().view(np.uint32)
    for c in range(count):
        for l, q in enumerate(qs):
            want = capi.polymul_ntt(a[c, l], b[c, l], q)
            assert np.array_equal(got[c, l], want), (c, l)
    srv.close()


# --------------------------------------------------------------------------
# Whole path on configs[0] (c1): every pair, real encryptions, decrypt check
# --------------------------------------------------------------------------

@pytest.mark.parametrize("fmt", [0, 1, 2], ids=["full", "compact", "compact_drop"])
def test_c1_all_pairs_bit_exact_and_decrypts(fmt):
    w = synth.WORKLOADS["c1"]
    ents = synth.cluster_entries(w)
    ids = synth.query_clusters(w)
    qv = synth.query_vectors(w, ids)
    srv = H.make_server(w, ents, resp_format=fmt)
    qs = srv.moduli
    cts, keys = H.encrypt_queries(w, qs, qv)
    resp, off = H.run_batch(srv, ids, cts)
    pcs = capi.encode_cluster(ents[0], w.d, w.n)
    P = pcs.shape[0]
    assert P == 32
    pq = np.repeat(np.arange(w.num_queries), P)
    pp = np.tile(np.arange(P), w.num_queries)
    want = H.oracle_pairs(qs, cts, pcs, pq, pp)
    E = w.n // w.d
    for i, (q, k) in enumerate(zip(pq, pp)):
        got = H.response_of(resp, off, q, k, w.n, w.d, fmt)
        assert H.matches_oracle(got, want[i], w.n, w.d, fmt), (q, k)
        if fmt:
            got = H.expand_compact(got, w.n, w.d, fmt, qs[0])
        dec = capi.decrypt_q0(qs[0], w.t, got, keys[q].s)
        for j in range(E):
            assert int(dec[j * w.d + w.d - 1]) == int(np.dot(qv[q].astype(np.int64),
                                                             ents[0][k * E + j].astype(np.int64))) % w.t
    assert srv.kernel_launches() > 0
    srv.close()


# --------------------------------------------------------------------------
# Edge cases: ragged clusters, d not dividing n, d = 1, d = n, tiny clusters,
# chunks of queries (> 8 per cluster), clusters without queries, L = 1..4
# --------------------------------------------------------------------------

EDGE = [
    dict(n=1024, L=1, d=100, sizes=[1, 10, 11, 37], nq=30),
    dict(n=2048, L=2, d=2048, sizes=[1, 3], nq=19),
    dict(n=2048, L=3, d=1, sizes=[2048, 2049, 5], nq=21),
    dict(n=4096, L=2, d=192, sizes=[2000, 21, 22, 1], nq=40),
    dict(n=4096, L=4, d=128, sizes=[65, 1024], nq=17),
    dict(n=8192, L=4, d=512, sizes=[17, 33], nq=12),
    dict(n=8192, L=2, d=300, sizes=[100], nq=9),
    # pruned c0 transform (compact formats, 16 | d) at several M = 2^v2(d)
    dict(n=4096, L=3, d=16, sizes=[300, 7], nq=11),
    dict(n=4096, L=3, d=48, sizes=[200], nq=9),
    dict(n=4096, L=2, d=4096, sizes=[3, 1], nq=5),
    dict(n=4096, L=2, d=1024, sizes=[9], nq=20),
    dict(n=8192, L=3, d=32, sizes=[300, 5], nq=7),
    dict(n=8192, L=3, d=64, sizes=[130, 3], nq=6),
    dict(n=8192, L=2, d=128, sizes=[70], nq=5),
    dict(n=8192, L=2, d=8192, sizes=[2], nq=4),
    # fused kernel v4 with compact responses (16 does not divide d): the instantiation whose
    # null-pointer test read a stale register on the B200 (found by test_gpu_fuzz.py)
    dict(n=4096, L=3, d=100, sizes=[150, 3], nq=9),
    dict(n=4096, L=2, d=3210, sizes=[2, 5, 3], nq=56),
    dict(n=4096, L=3, d=3210, sizes=[2], nq=1),
]


@pytest.mark.parametrize("fmt", [0, 2], ids=["full", "compact_drop"])
def test_multi_chunk_batch_bit_exact(fmt):
    """A batch large enough for 32-query work items (>= 4 queries per SM) with one cluster
    split over several chunks, including a ragged last chunk: every response word of a
    sample of queries (first, last, chunk boundaries) against the oracle."""
    n, L, d = 4096, 3, 128
    rng = np.random.default_rng(77)
    sizes = [130, 40, 300]
    clusters = [rng.integers(-15, 16, size=(s_, d)).astype(np.int8) for s_ in sizes]
    srv = H.make_server_ragged(n, L, d, clusters, resp_format=fmt)
    qs = srv.moduli
    nq = 700
    ids = np.concatenate([np.zeros(101, np.uint32), rng.integers(1, 3, size=nq - 101).astype(np.uint32)])
    rng.shuffle(ids)
    cts = np.stack([np.stack([np.stack([rng.integers(0, q, size=n) for q in qs]) for _ in range(2)])
                    for _ in range(nq)]).astype(np.uint32)
    resp, off = H.run_batch(srv, ids, cts)
    zeros = np.flatnonzero(ids == 0)
    sample = sorted(set([0, nq - 1] + zeros[[0, 31, 32, 63, 64, 95, 96, 100]].tolist()))
    pcs_by_c = [capi.encode_cluster(c, d, n) for c in clusters]
    for q in sample:
        c = int(ids[q])
        P = pcs_by_c[c].shape[0]
        want = H.oracle_pairs(qs, cts[q:q + 1], pcs_by_c[c], np.zeros(P), np.arange(P))
        for k in range(P):
            assert H.matches_oracle(H.response_of(resp, off, q, k, n, d, fmt), want[k], n, d, fmt), (q, k)


@pytest.mark.parametrize("fmt", [0, 1, 2], ids=["full", "compact", "compact_drop"])
@pytest.mark.parametrize("cfg", EDGE, ids=[f"n{c['n']}_L{c['L']}_d{c['d']}" for c in EDGE])
def test_edge_cases_bit_exact(cfg, fmt):
    n, L, d = cfg["n"], cfg["L"], cfg["d"]
    if fmt == 2 and n != 4096:
        with pytest.raises(WallyError):
            WallyServer(n, L, d, resp_format=2)
        return
    rng = np.random.default_rng(n + 7 * L + d)
    clusters = [rng.integers(-15, 16, size=(s, d)).astype(np.int8) for s in cfg["sizes"]]
    srv = H.make_server_ragged(n, L, d, clusters, resp_format=fmt)
    qs = srv.moduli
    C = len(clusters)
    # skewed ids: cluster 0 gets most queries (> one chunk), the last cluster none
    ids = np.where(rng.random(cfg["nq"]) < 0.6, 0, rng.integers(0, max(1, C - 1), size=cfg["nq"])).astype(np.uint32)
    cts = np.stack([np.stack([np.stack([rng.integers(0, q, size=n) for q in qs]) for _ in range(2)])
                    for _ in range(cfg["nq"])]).astype(np.uint32)
    resp, off = H.run_batch(srv, ids, cts)
    E = n // d
    pcs_by_c = [capi.encode_cluster(c, d, n) for c in clusters]
    for q in range(cfg["nq"]):
        c = int(ids[q])
        P = pcs_by_c[c].shape[0]
        assert int(off[q + 1] - off[q]) == P * H.words_per_pt(n, d, fmt)
        want = H.oracle_pairs(qs, cts[q:q + 1], pcs_by_c[c], np.zeros(P), np.arange(P))
        for k in range(P):
            assert H.matches_oracle(H.response_of(resp, off, q, k, n, d, fmt), want[k], n, d, fmt), (q, k)
    assert E >= 1
    srv.close()


def test_empty_batch_and_errors():
    w = synth.scaled(synth.WORKLOADS["c1"], cluster_size=64, num_queries=3)
    ents = synth.cluster_entries(w)
    srv = H.make_server(w, ents)
    qs = srv.moduli
    # empty batch is a no-op
    ws = srv.alloc_workspace(0)
    resp = torch.empty(1, dtype=torch.int32, device="cuda")
    srv.eval_batch(np.zeros(0, np.uint32), torch.empty(0, dtype=torch.int32, device="cuda"), resp, ws)
    # unknown cluster id -> error before any launch
    cts = torch.zeros((1, 2, w.num_limbs, w.n), dtype=torch.int32, device="cuda")
    with pytest.raises(WallyError) as ei:
        srv.response_layout(np.array([5], np.uint32))
    assert ei.value.code == -3
    before = srv.kernel_launches()
    with pytest.raises(WallyError):
        srv.eval_batch(np.array([1], np.uint32), cts, resp, srv.alloc_workspace(1))
    assert srv.kernel_launches() == before
    # a residue >= q is reported
    bad = cts.clone()
    bad[0, 0, 0, 5] = qs[0]
    off = srv.response_layout(np.array([0], np.uint32))
    resp = torch.empty(int(off[-1]), dtype=torch.int32, device="cuda")
    ws = srv.alloc_workspace(1)
    srv.eval_batch(np.array([0], np.uint32), bad, resp, ws)
    with pytest.raises(WallyError) as ei:
        srv.check_batch(ws)
    assert ei.value.code == -4
    srv.close()


def test_host_buffer_path_matches_device_path():
    w = synth.scaled(synth.WORKLOADS["c2"], num_clusters=6, cluster_size=300, num_queries=37)
    ents = synth.cluster_entries(w)
    srv = H.make_server(w, ents)
    ids = synth.query_clusters(w)
    cts = synth.uniform_ciphertexts(w, srv.moduli)
    resp_dev, off = H.run_batch(srv, ids, cts)
    host_resp = torch.empty(int(off[-1]), dtype=torch.int32).pin_memory()
    qh = torch.from_numpy(cts.view(np.int32)).pin_memory()
    sub = 8
    ws = torch.empty(srv.host_workspace_bytes(sub) // 4 + 1, dtype=torch.int32, device="cuda")
    srv.eval_batch_host(ids, qh, host_resp, sub, ws)
    assert np.array_equal(host_resp.numpy().view(np.uint32), resp_dev)
    srv.close()


# Full BASELINE configs at full size: tests/test_gpu_fullconfig.py


# --------------------------------------------------------------------------
# Cluster-sharded multi-rank path (emulated on one GPU: one context per rank,
# run one after another -- no kernel waits on another rank)
# --------------------------------------------------------------------------

def test_pack_queries_kernel():
    w = synth.scaled(synth.WORKLOADS["c2"], num_clusters=3, cluster_size=50, num_queries=29)
    ents = synth.cluster_entries(w)
    srv = H.make_server(w, ents)
    cts = synth.uniform_ciphertexts_torch(w, srv.moduli)
    idx = torch.tensor(np.random.default_rng(1).permutation(29)[:17].astype(np.int32)).cuda()
    out = torch.empty((17, 2, w.num_limbs, w.n), dtype=torch.int32, device="cuda")
    srv.pack_queries(idx, cts, out)
    torch.cuda.synchronize()
    assert torch.equal(out, cts[idx.long()])
    srv.close()


@pytest.mark.parametrize("world,fmt,replicated", [(2, 0, False), (3, 1, False), (2, 2, False), (4, 2, True)])
def test_sharded_ranks_bit_identical_to_single_rank(world, fmt, replicated):
    from paper_2406_06761_b200 import wally as W
    w = synth.scaled(synth.WORKLOADS["c5"], num_clusters=40, cluster_size=70, num_queries=97)
    ents = synth.cluster_entries(w)
    ids = synth.query_clusters(w)
    one = H.make_server(w, ents, resp_format=fmt)
    cts = synth.uniform_ciphertexts_torch(w, one.moduli)
    ref, ref_off = H.run_batch(one, ids, cts)
    one.close()
    sizes = np.full(w.num_clusters, w.cluster_size, np.uint32)
    if replicated:
        owner = W.wally_assign_owners_replicated(synth.cluster_popularity(w), world)
        assert any(bin(int(x)).count("1") > 1 for x in owner)     # the Zipf head is split
    else:
        owner = W.wally_assign_owners(synth.cluster_popularity(w), world)
    plan = W.wally_route_plan(ids, sizes, owner, w.n, w.d, world, fmt)
    gathered = np.empty(int(plan.gathered_off[-1]), np.uint32)
    base = np.concatenate([[0], np.cumsum(plan.resp_words.astype(np.int64))])
    for r in range(world):
        srv = H.make_server(w, ents, owner=owner, rank=r, resp_format=fmt)
        share = plan.share(r)
        idx = torch.from_numpy(share.astype(np.int32)).cuda()
        mine = torch.empty((share.size, 2, w.num_limbs, w.n), dtype=torch.int32, device="cuda")
        srv.pack_queries(idx, cts, mine)
        resp, _ = H.run_batch(srv, np.ascontiguousarray(ids[share]), mine)
        assert resp.size == int(plan.resp_words[r])
        gathered[base[r]:base[r + 1]] = resp
        srv.close()
    for q in range(ids.size):
        words = int(ref_off[q + 1] - ref_off[q])
        g0 = int(plan.gathered_off[q])
        assert np.array_equal(gathered[g0:g0 + words], ref[int(ref_off[q]):int(ref_off[q + 1])]), q


# --------------------------------------------------------------------------
# Plaintext CRT: one query = two ciphertexts (mod t0, t1)
# tagged with the same cluster; the server path is unchanged and the chunked
# batcher makes both share every staged plaintext
# --------------------------------------------------------------------------

@pytest.mark.parametrize("fmt", [0, 1])
def test_plaintext_crt_through_cuda_path(fmt):
    T0, T1 = 40961, 65537
    w = synth.scaled(synth.WORKLOADS["c2"], d=192, num_clusters=2, cluster_size=300, num_queries=3)
    ents = synth.cluster_entries(w)
    ents[1, 0] = 15
    srv = H.make_server(w, ents, resp_format=fmt)
    qs = srv.moduli
    qv = np.full((3, w.d), 15, np.int8)
    qv[1] = -15
    qv[2] = synth.query_vectors(w)[0]
    cl = np.array([1, 1, 0], np.uint32)
    cts, keys = [], []
    for q in range(3):
        for i, t in enumerate((T0, T1)):
            km = synth.key_material(w, 10 * q + i, qs)
            cts.append(capi.encrypt(qs, t, synth.query_message(w, qv[q]), km.s, km.a, km.e))
            keys.append(km)
    ids = np.repeat(cl, 2)
    resp, off = H.run_batch(srv, ids, np.stack(cts))
    E = w.n // w.d
    P = -(-w.cluster_size // E)
    big = 0
    for q in range(3):
        c = int(cl[q])
        for k in range(P):
            dec = []
            for i, t in enumerate((T0, T1)):
                got = H.response_of(resp, off, 2 * q + i, k, w.n, w.d, fmt)
                if fmt:
                    got = H.expand_compact(got, w.n, w.d, fmt, qs[0])
                dec.append(capi.decrypt_q0(qs[0], t, got, keys[2 * q + i].s))
            for j in range(min(E, w.cluster_size - k * E)):
                want = int(np.dot(qv[q].astype(np.int64), ents[c][k * E + j].astype(np.int64)))
                pos = j * w.d + w.d - 1
                assert capi.plain_crt_signed(int(dec[0][pos]), int(dec[1][pos]), T0, T1) == want
                big += abs(want) > 32768
    assert big >= 2      # values a single t = 65537 cannot represent as signed integers
    srv.close()


def _pruned_butterflies(n, d):
    """Butterflies the pruned c0 transform needs, counted backward from its
    outputs (every position = -1 mod 2^v2(d), a superset of the result
    coefficients j d + d - 1): at each stage, a butterfly is needed if one of
    its outputs is, and then both of its inputs are."""
    mu = (d & -d).bit_length() - 1
    need = set(i for i in range(n) if i % (1 << mu) == (1 << mu) - 1)
    total, s = 0, n.bit_length() - 2
    while s >= 0:
        t = 1 << s
        bf = set((i // (2 * t)) * 2 * t + i % t for i in need)
        total += len(bf)
        need = bf | set(b + t for b in bf)
        s -= 1
    return total


@pytest.mark.parametrize("L,d,fmt", [(3, 192, 0), (3, 192, 1), (3, 192, 2), (2, 128, 1), (3, 100, 1), (2, 16, 2)])
def test_modmuls_per_pair_counts(L, d, fmt):
    n = 4096
    srv = WallyServer(n, L, d, resp_format=fmt)
    full = 2 * (L * n + L * (n // 2) * 12 + n * L * (L - 1) // 2)
    got = srv.modmuls_per_pair()
    if fmt == 0 or d % 16:
        assert got == full
    else:
        mu = (d & -d).bit_length() - 1
        c0 = L * n + L * _pruned_butterflies(n, d) + (n >> mu) * L * (L - 1) // 2
        assert got == full // 2 + c0 and got < full
    srv.close()

"""GPU parity of the SIMD formulation (csrc/simd.cu, include/wally_simd.h;
SURVEY.md §8(f)-3) against the oracle (oracle/wally_simd_oracle.c), through
the C ABI.  Responses are compared word for word; one case also decrypts
the GPU responses with real keys and checks the dot products."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import capi  # noqa: E402

pytestmark = pytest.mark.gpu
T = 65537


@pytest.fixture(scope="module")
def S():
    from paper_2406_06761_b200 import build
    build.build()
    from paper_2406_06761_b200 import simd
    return simd


def _uniform(rng, mods, shape_prefix, n):
    """uniform residues: last-but-one axis runs over mods"""
    out = np.empty((*shape_prefix, len(mods), n), dtype=np.uint32)
    for i, q in enumerate(mods):
        out[..., i, :] = rng.integers(0, int(q), size=(*shape_prefix, n))
    return out


def _oracle_responses(srv, clusters, ids, cts, keys):
    n, L, d, g = srv.n, srv.L, srv.d, srv.baby
    mods = np.array(srv.moduli, dtype=np.uint32)
    per = srv.block_entries
    pts = {}
    out = []
    for q, c in enumerate(ids):
        c = int(c)
        nb = -(-clusters[c].shape[0] // per)
        for b in range(nb):
            if (c, b) not in pts:
                blk = clusters[c][b * per:(b + 1) * per]
                pts[(c, b)] = np.stack([capi.simd_encode(x, T) for x in capi.simd_diagonal_slots(blk, n, T, d, g)])
            res = capi.simd_server(mods, T, d, g, cts[q], keys[q, 0], keys[q, 1], pts[(c, b)])
            out.append(capi.simd_response(mods[:L], res))
    return out


def _run(srv, ids, cts, keys):
    dev = torch.device("cuda:0")
    cts_d = torch.from_numpy(cts.view(np.int32)).to(dev)
    keys_d = torch.from_numpy(keys.view(np.int32)).to(dev)
    resp = torch.zeros(max(1, srv.response_words(ids)), dtype=torch.int32, device=dev)
    off = srv.eval_batch(ids, cts_d, keys_d, resp)
    torch.cuda.synchronize()
    return resp.cpu().numpy().view(np.uint32), off


CASES = [
    dict(n=1024, L=2, d=32, g=0, sizes=[1025, 100, 7], nq=5),      # d | n/2, a two-block cluster
    dict(n=4096, L=3, d=48, g=7, sizes=[3000, 40], nq=3),          # d does not divide n/2, g does not divide d
    dict(n=2048, L=1, d=24, g=24, sizes=[50], nq=2),               # one limb, one giant step (no giant rotation)
    dict(n=8192, L=4, d=32, g=5, sizes=[300], nq=2),
    dict(n=1024, L=3, d=512, g=1, sizes=[1024, 3], nq=2),          # d = n/2 (one slice per row), no baby steps
    dict(n=1024, L=2, d=7, g=3, sizes=[1100], nq=3),               # odd d: R = 72 slices per row, two blocks
    dict(n=2048, L=4, d=100, g=10, sizes=[1500], nq=2),            # L = 4 through the fused chain, g | d
]


@pytest.mark.parametrize("chain", [True, False], ids=["chain", "modup_moddown"])
@pytest.mark.parametrize("cfg", CASES, ids=[f"n{c['n']}_L{c['L']}_d{c['d']}_g{c['g']}" for c in CASES])
def test_simd_bit_exact_with_oracle(S, cfg, chain):
    n, L, d = cfg["n"], cfg["L"], cfg["d"]
    rng = np.random.default_rng(n + L + d)
    srv = S.SimdServer(n, L, d, baby=cfg["g"])
    srv.set_chain_threshold(0 if chain else 2**32 - 1)
    clusters = [rng.integers(-15, 16, size=(s, d)).astype(np.int8) for s in cfg["sizes"]]
    srv.load_clusters(clusters)
    ids = rng.integers(0, len(clusters), size=cfg["nq"]).astype(np.uint32)
    ids[0] = 0
    mods = srv.moduli
    cts = _uniform(rng, mods[:L], (cfg["nq"], 2), n)
    keys = _uniform(rng, mods, (cfg["nq"], 2, 2, L), n)
    got, off = _run(srv, ids, cts, keys)
    want = _oracle_responses(srv, clusters, ids, cts, keys)
    assert off[-1] == len(want) * 2 * n
    for i, w in enumerate(want):
        g = got[i * 2 * n:(i + 1) * 2 * n].reshape(2, n)
        assert np.array_equal(g, w), f"response {i}: {np.count_nonzero(g != w)} words differ"


def test_simd_gpu_responses_decrypt_to_dot_products(S):
    n, L, d = 1024, 2, 32
    rng = np.random.default_rng(11)
    srv = S.SimdServer(n, L, d)
    mods = np.array(srv.moduli, dtype=np.uint32)
    s = rng.integers(-1, 2, size=n).astype(np.int8)

    def key(k):
        a = _uniform(rng, mods, (L,), n)
        e = np.clip(np.rint(rng.normal(0, 3.2, size=(L, n))), -19, 19).astype(np.int32)
        return capi.simd_keygen(mods, s, k, a, e)
    clusters = [rng.integers(-15, 16, size=(sz, d)).astype(np.int8) for sz in (1024, 300)]
    srv.load_clusters(clusters)
    ids = np.array([0, 1], np.uint32)
    qs = rng.integers(-15, 16, size=(2, d)).astype(np.int32)
    cts = np.stack([capi.encrypt(mods[:L], T, capi.simd_encode(capi.simd_query_slots(q, n, T), T).astype(np.int32),
                                 s, _uniform(rng, mods[:L], (), n),
                                 np.clip(np.rint(rng.normal(0, 3.2, size=n)), -19, 19).astype(np.int32))
                    for q in qs])
    keys = np.stack([np.stack([key(srv.galois[0]), key(srv.galois[1])]) for _ in range(2)])
    got, off = _run(srv, ids, cts, keys)
    R = srv.row_slices
    for qi in range(2):
        resp = got[int(off[qi]):int(off[qi]) + 2 * n]
        assert capi.noise_budget_q0(int(mods[0]), T, resp, s) > 2
        slots = capi.simd_decode(capi.decrypt_q0(int(mods[0]), T, resp, s), T)
        ent = clusters[ids[qi]]
        want = (ent.astype(np.int64) @ qs[qi].astype(np.int64)) % T
        for e in range(ent.shape[0]):
            sl, col = divmod(e, d)
            r, u = divmod(sl, R)
            assert slots[r * (n // 2) + u * d + col] == want[e], (qi, e)


def test_simd_errors(S):
    n, L, d = 1024, 2, 16
    srv = S.SimdServer(n, L, d)
    rng = np.random.default_rng(3)
    srv.load_clusters([rng.integers(-15, 16, size=(40, d)).astype(np.int8)])
    mods = srv.moduli
    cts = _uniform(rng, mods[:L], (1, 2), n)
    keys = _uniform(rng, mods, (1, 2, 2, L), n)
    with pytest.raises(S.WallyError) as e:
        _run(srv, np.array([1], np.uint32), cts, keys)
    assert e.value.code == -3
    bad = cts.copy()
    bad[0, 1, 1, 5] = mods[1]
    with pytest.raises(S.WallyError) as e:
        _run(srv, np.array([0], np.uint32), bad, keys)
    assert e.value.code == -4
    with pytest.raises(S.WallyError):
        S.SimdServer(n, L, n)                     # d > n/2
    m = list(mods)
    with pytest.raises(S.WallyError):
        S.SimdServer(n, L, d, moduli=m[:L] + [m[-1] + 2 * n * 1000])   # special prime not below q_0 / not prime
    assert srv.modmuls_per_query(1) > 0 and srv.launch_count() > 0


def test_simd_edge_cases(S):
    """empty batch, an empty cluster (no response blocks), a cluster of exactly one block, reload"""
    n, L, d = 1024, 2, 16
    rng = np.random.default_rng(8)
    srv = S.SimdServer(n, L, d, baby=3)
    per = srv.block_entries
    clusters = [np.zeros((0, d), np.int8), rng.integers(-15, 16, size=(per, d)).astype(np.int8),
                rng.integers(-15, 16, size=(per + 1, d)).astype(np.int8)]
    srv.load_clusters(clusters)
    assert [srv.blocks(c) for c in range(3)] == [0, 1, 2] and srv.blocks(3) == 0
    mods = srv.moduli
    # empty batch
    got, off = _run(srv, np.zeros(0, np.uint32), _uniform(rng, mods[:L], (0, 2), n),
                    _uniform(rng, mods, (0, 2, 2, L), n))
    assert off.tolist() == [0]
    ids = np.array([0, 2, 1, 0], np.uint32)
    cts = _uniform(rng, mods[:L], (4, 2), n)
    keys = _uniform(rng, mods, (4, 2, 2, L), n)
    got, off = _run(srv, ids, cts, keys)
    assert off.tolist() == [0, 0, 4 * n, 6 * n, 6 * n]
    want = _oracle_responses(srv, clusters, ids, cts, keys)
    assert len(want) == 3
    for i, w in enumerate(want):
        assert np.array_equal(got[i * 2 * n:(i + 1) * 2 * n].reshape(2, n), w), i
    # reload a different database into the same context
    srv.load_clusters(clusters[1:2])
    got2, off2 = _run(srv, np.array([0], np.uint32), cts[2:3], keys[2:3])
    assert np.array_equal(got2[:2 * n], got[4 * n:6 * n])


def test_simd_host_path_matches_device_path(S):
    """wally_simd_eval_batch_host (pipelined sub-batches from pinned host memory) gives the device path's bytes"""
    n, L, d = 1024, 2, 16
    rng = np.random.default_rng(21)
    srv = S.SimdServer(n, L, d, baby=4)
    clusters = [rng.integers(-15, 16, size=(s_, d)).astype(np.int8) for s_ in (40, 600, 300, 1)]
    srv.load_clusters(clusters)
    nq = 11
    ids = rng.integers(0, len(clusters), size=nq).astype(np.uint32)
    mods = srv.moduli
    cts = _uniform(rng, mods[:L], (nq, 2), n)
    keys = _uniform(rng, mods, (nq, 2, 2, L), n)
    want, off = _run(srv, ids, cts, keys)
    words = srv.response_words(ids)
    for sub in (3, 4, 11, 64):
        ch = torch.from_numpy(cts.view(np.int32)).pin_memory()
        kh = torch.from_numpy(keys.view(np.int32)).pin_memory()
        rh = torch.zeros(words, dtype=torch.int32).pin_memory()
        off2 = srv.eval_batch_host(ids, ch, kh, rh, sub_batch=sub)
        assert np.array_equal(off2, off)
        assert np.array_equal(rh.numpy().view(np.uint32), want[:words]), sub


def test_simd_stage_timing_and_work(S):
    """wally_simd_enable_stage_timing / wally_simd_stage_times / wally_simd_stage_work (include/wally_simd.h):
    the five stage times of a timed batch add up to (at most) its wall time on the stream, every stage
    ran, timing leaves the responses unchanged, and the per-stage work matches wally_simd_modmuls_per_query
    and the stated byte terms."""
    n, L, d = 1024, 2, 16
    rng = np.random.default_rng(31)
    srv = S.SimdServer(n, L, d, baby=4)
    clusters = [rng.integers(-15, 16, size=(s_, d)).astype(np.int8) for s_ in (40, 600, 300)]
    srv.load_clusters(clusters)
    nq = 9
    ids = np.array([1, 0, 2, 1, 1, 2, 0, 1, 2], np.uint32)
    mods = srv.moduli
    cts = _uniform(rng, mods[:L], (nq, 2), n)
    keys = _uniform(rng, mods, (nq, 2, 2, L), n)
    want, _ = _run(srv, ids, cts, keys)
    srv.stage_times()
    srv.enable_stage_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    got, _ = _run(srv, ids, cts, keys)
    e1.record()
    torch.cuda.synchronize()
    srv.enable_stage_timing(False)
    ms, chunks = srv.stage_times()
    assert np.array_equal(got, want)
    assert chunks >= 1 and len(ms) == len(S.STAGES) == 5
    assert all(t > 0 for t in ms), ms
    assert sum(ms) <= e0.elapsed_time(e1) * 1.05 + 0.05
    assert srv.stage_times() == ([0.0] * 5, 0)                 # the record was cleared
    mm, by = srv.stage_work(ids)
    blocks = [srv.blocks(int(c)) for c in ids]
    assert sum(mm) == sum(srv.modmuls_per_query(b) for b in blocks)
    ct = 2 * L * n * 4
    distinct = sum(srv.blocks(c) for c in set(ids.tolist()))
    assert by[2] == distinct * d * L * n * 8 + sum(blocks) * (srv.baby + srv.giant) * ct
    with pytest.raises(Exception):
        srv.stage_work(np.array([7], np.uint32))                  # unknown cluster


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_simd_full_config_sampled_bit_exact(S, name):
    """The bench's launch configuration at full size (every cluster loaded, the whole query batch in one
    call, uniform stand-in ciphertexts and keys as in bench.py): sampled queries -- the first, the last and
    some in between, i.e. in different chunks -- are compared word for word with the oracle, and one query
    is a real encryption under real rotation keys whose response must decrypt to its dot products."""
    import synth
    w = synth.WORKLOADS[name]
    ents = synth.cluster_entries(w)
    ids = synth.query_clusters(w)
    srv = S.SimdServer(w.n, w.num_limbs, w.d, w.t)
    srv.load_clusters([ents[c] for c in range(w.num_clusters)])
    L, n = w.num_limbs, w.n
    mods = np.array(srv.moduli, dtype=np.uint32)
    cts = synth.uniform_ciphertexts_torch(w, srv.moduli[:L], device="cuda")
    keys = synth.uniform_keys_torch(w, srv.moduli, device="cuda")
    # one real query with real keys
    rng = np.random.default_rng(5)
    qreal = w.num_queries // 2
    s = rng.integers(-1, 2, size=n).astype(np.int8)
    qvec = rng.integers(-15, 16, size=w.d).astype(np.int32)

    def key(k):
        a = _uniform(rng, mods, (L,), n)
        e = np.clip(np.rint(rng.normal(0, 3.2, size=(L, n))), -19, 19).astype(np.int32)
        return capi.simd_keygen(mods, s, k, a, e)
    ct_real = capi.encrypt(mods[:L], w.t, capi.simd_encode(capi.simd_query_slots(qvec, n, w.t), w.t).astype(np.int32),
                           s, _uniform(rng, mods[:L], (), n),
                           np.clip(np.rint(rng.normal(0, 3.2, size=n)), -19, 19).astype(np.int32))
    key_real = np.stack([key(srv.galois[0]), key(srv.galois[1])])
    cts[qreal] = torch.from_numpy(ct_real.view(np.int32)).cuda()
    keys[qreal] = torch.from_numpy(key_real.view(np.int32)).cuda()
    resp = torch.empty(srv.response_words(ids), dtype=torch.int32, device="cuda")
    off = srv.eval_batch(ids, cts, keys, resp)
    torch.cuda.synchronize()
    per = srv.block_entries
    sample = [0, qreal, w.num_queries - 1, int(rng.integers(1, w.num_queries - 1))]
    for q in sample:
        c = int(ids[q])
        ct = cts[q].cpu().numpy().view(np.uint32)
        kq = keys[q].cpu().numpy().view(np.uint32)
        for b in range(srv.blocks(c)):
            blk = ents[c][b * per:(b + 1) * per]
            pt = np.stack([capi.simd_encode(x, w.t) for x in capi.simd_diagonal_slots(blk, n, w.t, w.d, srv.baby)])
            want = capi.simd_response(mods[:L], capi.simd_server(mods, w.t, w.d, srv.baby, ct, kq[0], kq[1], pt))
            o = int(off[q]) + b * 2 * n
            got = resp[o:o + 2 * n].cpu().numpy().view(np.uint32).reshape(2, n)
            assert np.array_equal(got, want), (name, q, b)
            if q == qreal:
                slots = capi.simd_decode(capi.decrypt_q0(int(mods[0]), w.t, got, s), w.t)
                dots = (blk.astype(np.int64) @ qvec.astype(np.int64)) % w.t
                R = srv.row_slices
                for e in range(blk.shape[0]):
                    sl, col = divmod(e, w.d)
                    r, u = divmod(sl, R)
                    assert slots[r * (n // 2) + u * w.d + col] == dots[e], (name, e)
    srv.close()

"""GPU parity on seeded random shapes: the CUDA path (through the C ABI) against the CPU oracle.

Every case draws a ring degree n, a limb count L, an embedding dimension d
(arbitrary, or one of the values the specialised kernels key on: 16 | d,
32 | d, d = n, d = 1), ragged clusters, a skewed query mix, extreme residues
(0 and q_i - 1) and a response format (every fifth case a batch of 600-1,400
queries, which takes the 32-query work items; a sample of its queries is
compared), runs one batch through
wally_eval_batch (every third case through the host-buffer call
wally_eval_batch_host) and compares every word of every response with the
oracle's pairs (Alg 4 ServerComputation).  Bar: bit-exact.

WALLY_FUZZ_CASES (default 24) sets the number of cases, WALLY_FUZZ_SEED the
first seed: `scripts/gpu_fuzz.sh` runs a few hundred as a soak.
"""
import os

import numpy as np
import pytest

from oracle import capi
from tests import helpers as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2406_06761_b200.wally import WallyError, WallyServer  # noqa: E402

CASES = int(os.environ.get("WALLY_FUZZ_CASES", "24"))
SEED0 = int(os.environ.get("WALLY_FUZZ_SEED", "20260601"))
MAX_PAIRS = 700     # per case: the oracle's work
BIG = os.environ.get("WALLY_FUZZ_BIG") == "1"     # every case a large batch (else every fifth)


def draw_case(seed: int) -> dict:
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1024, 2048, 4096, 4096, 4096, 8192, 8192]))
    L = int(rng.integers(1, 5))
    kind = int(rng.integers(0, 6))
    if kind == 0:
        d = int(rng.integers(1, n + 1))
    elif kind == 1:
        d = 16 * int(rng.integers(1, n // 16 + 1))
    elif kind == 2:
        d = 32 * int(rng.integers(1, min(n // 32, 24) + 1))
    elif kind == 3:
        d = 1 << int(rng.integers(0, n.bit_length()))
    elif kind == 4:
        d = int(rng.choice([n, n - 1, n // 2 + 1, 3, 100, 192, 384]))
    else:
        d = int(rng.choice([64, 128, 192, 256, 512]))
    d = max(1, min(d, n))
    E = n // d
    C = int(rng.integers(1, 6))
    sizes = []
    for _ in range(C):
        P = int(rng.integers(1, 7))
        s = (P - 1) * E + int(rng.integers(1, E + 1))          # P plaintexts, the last one ragged
        sizes.append(min(s, 4096))
    Ps = [-(-s // E) for s in sizes]
    nq_max = max(1, MAX_PAIRS // max(Ps))
    nq = int(rng.integers(1, min(nq_max, 160) + 1))
    if BIG or seed % 5 == 2:
        # a batch large enough for 32-query work items (>= 4 queries per SM): few, small clusters
        # (drawn from a stream of their own, so the other parameters of a seed do not depend on this)
        rb = np.random.default_rng(seed ^ 0xB16)
        sizes = [min((int(rb.integers(1, 4)) - 1) * E + int(rb.integers(1, E + 1)), 4096)
                 for _ in range(int(rb.integers(1, 4)))]
        nq = int(rb.integers(600, 1400))
    fmt = int(rng.integers(0, 3))
    bound = int(rng.choice([1, 15, 127]))
    return dict(seed=seed, n=n, L=L, d=d, sizes=sizes, nq=nq, fmt=fmt, bound=bound,
                host=(seed % 3 == 0), extreme=(seed % 4 == 1))


def run_case(c: dict) -> int:
    n, L, d, fmt = c["n"], c["L"], c["d"], c["fmt"]
    rng = np.random.default_rng(c["seed"] ^ 0x5EED)
    try:
        srv = WallyServer(n, L, d, resp_format=fmt)
    except WallyError:
        # the only format a context may refuse for a supported (n, L, d): compact_drop (n = 4096 and the z = 8 rule)
        assert fmt == 2, c
        fmt = 1
        srv = WallyServer(n, L, d, resp_format=fmt)
    srv.close()
    b = c["bound"]
    clusters = [rng.integers(-b - (b == 127), b + 1, size=(s, d)).astype(np.int8) for s in c["sizes"]]
    srv = H.make_server_ragged(n, L, d, clusters, resp_format=fmt)
    qs = srv.moduli
    C, nq = len(clusters), c["nq"]
    ids = np.where(rng.random(nq) < 0.5, int(rng.integers(0, C)), rng.integers(0, C, size=nq)).astype(np.uint32)
    cts = np.stack([np.stack([np.stack([rng.integers(0, q, size=n) for q in qs]) for _ in range(2)])
                    for _ in range(nq)]).astype(np.uint32)
    if c["extreme"]:
        # residues at both ends of [0, q_i): lazy ranges and conditional subtractions at their limits
        for li, q in enumerate(qs):
            cts[0, :, li, :] = q - 1
            cts[nq - 1, 0, li, ::2] = 0
            cts[nq - 1, 1, li, 1::2] = q - 1
    if c["host"]:
        off = srv.response_layout(ids)
        host_resp = torch.empty(int(off[-1]), dtype=torch.int32).pin_memory()
        qh = torch.from_numpy(cts.view(np.int32)).pin_memory()
        sub = int(rng.integers(1, nq + 2))
        ws = torch.empty(srv.host_workspace_bytes(sub) // 4 + 1, dtype=torch.int32, device="cuda")
        srv.eval_batch_host(ids, qh, host_resp, sub, ws)
        torch.cuda.synchronize()
        resp = host_resp.numpy().view(np.uint32)
    else:
        resp, off = H.run_batch(srv, ids, cts)
    pcs_by_c = [capi.encode_cluster(e, d, n) for e in clusters]
    pairs = 0
    check = range(nq)
    if nq * max(p.shape[0] for p in pcs_by_c) > 2 * MAX_PAIRS:
        # large batch: the first and last queries, and a random sample (the oracle's work stays bounded)
        check = sorted(set(range(8)) | set(range(nq - 8, nq)) | set(rng.choice(nq, size=300, replace=False).tolist()))
    for q in check:
        cl = int(ids[q])
        P = pcs_by_c[cl].shape[0]
        assert int(off[q + 1] - off[q]) == P * H.words_per_pt(n, d, fmt), c
        want = H.oracle_pairs(qs, cts[q:q + 1], pcs_by_c[cl], np.zeros(P), np.arange(P))
        for k in range(P):
            assert H.matches_oracle(H.response_of(resp, off, q, k, n, d, fmt), want[k], n, d, fmt), (c, q, k)
        pairs += P
    srv.close()
    return pairs


@pytest.mark.parametrize("block", range((CASES + 7) // 8))
def test_random_shapes_bit_exact(block):
    pairs = 0
    seeds = range(SEED0 + 8 * block, SEED0 + min(CASES, 8 * block + 8))
    for s in seeds:
        pairs += run_case(draw_case(s))
    print(f"fuzz block {block}: {len(seeds)} cases, {pairs} pairs compared word for word")


# --------------------------------------------------------------------------
# The SIMD formulation (include/wally_simd.h) on random shapes
# --------------------------------------------------------------------------
SIMD_CASES = int(os.environ.get("WALLY_FUZZ_SIMD_CASES", "8"))
T = 65537


def draw_simd_case(seed: int) -> dict:
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1024, 1024, 2048, 4096, 8192]))
    L = int(rng.integers(1, 5))
    dmax = min(n // 2, 96 if n <= 2048 else 48)          # the oracle's work grows with d n log n
    kind = int(rng.integers(0, 3))
    d = int(rng.integers(1, dmax + 1)) if kind else int(rng.choice([1, 2, 16, 32, n // 2 if n <= 2048 else 32]))
    g = int(rng.integers(0, d + 1))                       # 0: the library's default baby-step count
    return dict(seed=seed, n=n, L=L, d=d, g=g, nq=int(rng.integers(1, 5)), C=int(rng.integers(1, 4)),
                chain=bool(rng.integers(0, 2)))


def run_simd_case(c: dict) -> int:
    from paper_2406_06761_b200 import simd
    from tests.test_simd_gpu import _oracle_responses, _run, _uniform
    n, L, d = c["n"], c["L"], c["d"]
    rng = np.random.default_rng(c["seed"] ^ 0x51D)
    srv = simd.SimdServer(n, L, d, baby=c["g"])
    srv.set_chain_threshold(0 if c["chain"] else 2**32 - 1)
    per = srv.block_entries
    sizes = [int(rng.choice([1, per - 1, per, per + 1, int(rng.integers(1, 2 * per + 1))])) for _ in range(c["C"])]
    clusters = [rng.integers(-15, 16, size=(max(s, 1), d)).astype(np.int8) for s in sizes]
    srv.load_clusters(clusters)
    ids = rng.integers(0, len(clusters), size=c["nq"]).astype(np.uint32)
    mods = srv.moduli
    cts = _uniform(rng, mods[:L], (c["nq"], 2), n)
    keys = _uniform(rng, mods, (c["nq"], 2, 2, L), n)
    got, off = _run(srv, ids, cts, keys)
    want = _oracle_responses(srv, clusters, ids, cts, keys)
    assert off[-1] == len(want) * 2 * n, c
    for i, w in enumerate(want):
        assert np.array_equal(got[i * 2 * n:(i + 1) * 2 * n].reshape(2, n), w), (c, i)
    return len(want)


@pytest.mark.parametrize("block", range((SIMD_CASES + 3) // 4))
def test_simd_random_shapes_bit_exact(block):
    from paper_2406_06761_b200 import build
    build.build()
    seeds = range(SEED0 + 4 * block, SEED0 + min(SIMD_CASES, 4 * block + 4))
    blocks = sum(run_simd_case(draw_simd_case(s)) for s in seeds)
    print(f"simd fuzz block {block}: {len(seeds)} cases, {blocks} response ciphertexts compared word for word")

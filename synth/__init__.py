"""Seeded synthetic inputs shared by the oracle tests and the product bench.

This module holds NO arithmetic of the method (no packing, no NTT, no
encryption, no modulus switching).  It only draws random numbers:

  * database entries (int8 embeddings) per cluster,
  * query vectors, cluster IDs and real/fake flags,
  * per-query key material the client would draw (ternary secret s,
    uniform a per RNS limb, rounded-Gaussian error e), passed into the
    oracle's encrypt, and
  * uniform RNS residues standing in for query ciphertexts in the bench
    (under RLWE a fresh ciphertext is indistinguishable from uniform, and the
    server path is data-oblivious).

The workloads are the five configurations of BASELINE.json (`configs[0..4]`);
their recipes are spelled out in DESIGN.md "Input recipe" and SURVEY.md §8(d).
The real data the paper uses (MSMARCO passages embedded by
msmarco-distilbert-base-tas-b, PCA to d=192, FAISS k-means; PAPER.md
P:L1016-1022) is not available; these synthetic inputs stand in
for it with the same shapes and value ranges.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    n: int                 # ring degree N
    num_limbs: int         # L
    t: int                 # plaintext modulus
    d: int                 # embedding dimension
    num_clusters: int
    cluster_size: int      # entries per cluster (S_c, uniform here)
    entry_bound: int       # entries uniform/clipped in [-bound, bound]
    num_queries: int
    seed: int
    db_kind: str = "uniform"        # "uniform" | "gmm_overlap"
    query_kind: str = "uniform"     # "single" | "uniform" | "size_weighted" | "zipf"
    zipf_s: float = 1.1
    fake_share: float = 0.0         # share of fake (zero-vector) queries, reading S14
    gmm_components: int = 0
    gmm_per_component: int = 0
    gmm_sigma: float = 3.0
    gmm_mean_bound: float = 8.0
    description: str = ""

    @property
    def entries_per_plaintext(self) -> int:   # E = floor(N/d); layout metadata only
        return self.n // self.d

    @property
    def total_entries(self) -> int:
        return self.num_clusters * self.cluster_size


WORKLOADS = {
    "c1": Workload("c1", 4096, 2, 65537, 128, 1, 1024, 15, 8, 1001, query_kind="single",
                   description="BASELINE.json configs[0]: single cluster, 1,024 entries d=128, 8 queries"),
    "c2": Workload("c2", 4096, 3, 65537, 128, 64, 4096, 15, 1024, 1002,
                   description="BASELINE.json configs[1]: 64 clusters x 4,096 entries, 1,024 queries"),
    "c3": Workload("c3", 4096, 3, 65537, 192, 3200, 2000, 15, 16384, 1003, db_kind="gmm_overlap",
                   query_kind="size_weighted", fake_share=0.23, gmm_components=3200, gmm_per_component=1000,
                   description="BASELINE.json configs[2]: paper-scale 3.2M entries d=192, 3,200 overlapping "
                               "clusters of 2,000, 16,384 queries (77% real, 23% fake)"),
    "c4": Workload("c4", 8192, 4, 65537, 512, 1024, 1024, 7, 8192, 1004,
                   description="BASELINE.json configs[3]: N=8192 L=4, 1,024 clusters x 1,024 entries d=512"),
    "c5": Workload("c5", 4096, 2, 65537, 128, 10000, 1000, 15, 65536, 1005, query_kind="zipf",
                   description="BASELINE.json configs[4]: 10M entries, 10,000 clusters x 1,000, 65,536 "
                               "queries with Zipf(1.1) cluster popularity"),
}


def scaled(w: Workload, **kw) -> Workload:
    """A copy of a workload with some fields replaced (small test variants)."""
    d = dict(w.__dict__)
    d.update(kw)
    return Workload(**d)


def _rng(seed: int, *stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, *stream])))


# Stream ids (fixed so every consumer draws the same numbers).
_S_DB, _S_GMM_MEANS, _S_QCLUSTER, _S_QVEC, _S_FAKE, _S_KEYS, _S_CT, _S_ZIPF = range(1, 9)


def cluster_entries(w: Workload) -> np.ndarray:
    """int8 [num_clusters][cluster_size][d] database entries, per cluster.

    uniform:     iid uniform ints in [-bound, bound].
    gmm_overlap: (c3) a gmm_components-component Gaussian mixture: means
                 mu_k ~ U[-8, 8]^d, entries round(mu_k + N(0, sigma^2)) clipped
                 to [-bound, bound], gmm_per_component per component; cluster c
                 holds components {c, c+1 mod K} (reading S15: every entry in
                 exactly two clusters, passed duplicated)."""
    if w.db_kind == "uniform":
        g = _rng(w.seed, _S_DB)
        return g.integers(-w.entry_bound, w.entry_bound + 1, size=(w.num_clusters, w.cluster_size, w.d),
                          dtype=np.int8)
    if w.db_kind == "gmm_overlap":
        comps = gmm_components(w)
        K = w.gmm_components
        assert w.num_clusters == K and w.cluster_size == 2 * w.gmm_per_component
        out = np.empty((K, w.cluster_size, w.d), dtype=np.int8)
        out[:, :w.gmm_per_component] = comps
        out[:, w.gmm_per_component:] = np.roll(comps, -1, axis=0)
        return out
    raise ValueError(w.db_kind)


def gmm_means(w: Workload) -> np.ndarray:
    g = _rng(w.seed, _S_GMM_MEANS)
    return g.uniform(-w.gmm_mean_bound, w.gmm_mean_bound, size=(w.gmm_components, w.d)).astype(np.float32)


def gmm_components(w: Workload) -> np.ndarray:
    """int8 [K][per_component][d] entries of each mixture component."""
    mu = gmm_means(w)
    K, m = w.gmm_components, w.gmm_per_component
    out = np.empty((K, m, w.d), dtype=np.int8)
    g = _rng(w.seed, _S_DB)
    chunk = 64
    for k0 in range(0, K, chunk):
        k1 = min(K, k0 + chunk)
        x = g.standard_normal(size=(k1 - k0, m, w.d), dtype=np.float32) * np.float32(w.gmm_sigma)
        x += mu[k0:k1, None, :]
        np.rint(x, out=x)
        np.clip(x, -w.entry_bound, w.entry_bound, out=x)
        out[k0:k1] = x.astype(np.int8)
    return out


def query_clusters(w: Workload) -> np.ndarray:
    """uint32 [num_queries] cluster ID of every query (input order)."""
    g = _rng(w.seed, _S_QCLUSTER)
    if w.query_kind == "single":
        return np.zeros(w.num_queries, dtype=np.uint32)
    if w.query_kind in ("uniform", "size_weighted"):
        # size_weighted: multinomial weighted by cluster size; sizes are uniform
        # in every BASELINE config, so both reduce to a uniform draw.
        return g.integers(0, w.num_clusters, size=w.num_queries).astype(np.uint32)
    if w.query_kind == "zipf":
        perm = _rng(w.seed, _S_ZIPF).permutation(w.num_clusters)          # rank -> cluster ID (S17)
        weights = (np.arange(1, w.num_clusters + 1, dtype=np.float64)) ** (-w.zipf_s)
        weights /= weights.sum()
        ranks = g.choice(w.num_clusters, size=w.num_queries, p=weights)
        return perm[ranks].astype(np.uint32)
    raise ValueError(w.query_kind)


def cluster_popularity(w: Workload) -> np.ndarray:
    """float64 [num_clusters]: the prior probability that a query names each
    cluster (the distribution query_clusters draws from; used as the expected
    load when clusters are assigned to ranks)."""
    if w.query_kind == "single":
        p = np.zeros(w.num_clusters)
        p[0] = 1.0
        return p
    if w.query_kind in ("uniform", "size_weighted"):
        return np.full(w.num_clusters, 1.0 / w.num_clusters)
    if w.query_kind == "zipf":
        perm = _rng(w.seed, _S_ZIPF).permutation(w.num_clusters)
        weights = (np.arange(1, w.num_clusters + 1, dtype=np.float64)) ** (-w.zipf_s)
        p = np.empty(w.num_clusters)
        p[perm] = weights / weights.sum()
        return p
    raise ValueError(w.query_kind)


def query_fake_flags(w: Workload) -> np.ndarray:
    g = _rng(w.seed, _S_FAKE)
    if w.fake_share <= 0:
        return np.zeros(w.num_queries, dtype=bool)
    return g.random(w.num_queries) < w.fake_share


def query_vectors(w: Workload, clusters: np.ndarray | None = None) -> np.ndarray:
    """int8 [num_queries][d] plaintext query embeddings.  Fake queries are the
    zero vector (reading S14).  For gmm_overlap, a real query is drawn from
    the mixture component of its cluster (component c for cluster c)."""
    if clusters is None:
        clusters = query_clusters(w)
    g = _rng(w.seed, _S_QVEC)
    if w.db_kind == "gmm_overlap":
        mu = gmm_means(w)
        x = g.standard_normal(size=(w.num_queries, w.d), dtype=np.float32) * np.float32(w.gmm_sigma)
        x += mu[clusters.astype(np.int64)]
        q = np.clip(np.rint(x), -w.entry_bound, w.entry_bound).astype(np.int8)
    else:
        q = g.integers(-w.entry_bound, w.entry_bound + 1, size=(w.num_queries, w.d), dtype=np.int8)
    q[query_fake_flags(w)] = 0
    return q


@dataclass
class KeyMaterial:
    s: np.ndarray   # int8 [n] ternary secret
    a: np.ndarray   # uint32 [L][n] uniform residues, a[l] in [0, q_l)
    e: np.ndarray   # int32 [n] rounded Gaussian, sigma 3.2, |e| <= 19


def key_material(w: Workload, query_index: int, moduli) -> KeyMaterial:
    """The random draws of the client for query `query_index` (fresh keys for
    every real and fake query, reading S19; secret iid uniform ternary S4;
    error rounded N(0, 3.2^2) resampled beyond 6 sigma S3)."""
    g = _rng(w.seed, _S_KEYS, int(query_index))
    s = g.integers(-1, 2, size=w.n, dtype=np.int8)
    a = np.stack([g.integers(0, int(q), size=w.n, dtype=np.uint64) for q in moduli]).astype(np.uint32)
    e = np.rint(g.normal(0.0, 3.2, size=w.n))
    bad = np.abs(e) > 19
    while bad.any():
        e[bad] = np.rint(g.normal(0.0, 3.2, size=int(bad.sum())))
        bad = np.abs(e) > 19
    return KeyMaterial(s=s, a=a, e=e.astype(np.int32))


def query_message(w: Workload, qvec: np.ndarray) -> np.ndarray:
    """int32 [n]: the query vector as polynomial coefficients 0..d-1 (the
    client's coefficient encoding input; values reduced mod t by the
    encryptor, reading S9)."""
    m = np.zeros(w.n, dtype=np.int32)
    m[: w.d] = qvec
    return m


def uniform_ciphertexts(w: Workload, moduli, num_queries: int | None = None, seed_offset: int = 0) -> np.ndarray:
    """uint32 [nq][2][L][n] uniform residues (ciphertext stand-ins, see module doc)."""
    nq = w.num_queries if num_queries is None else num_queries
    g = _rng(w.seed + seed_offset, _S_CT)
    out = np.empty((nq, 2, len(moduli), w.n), dtype=np.uint32)
    for l, q in enumerate(moduli):
        out[:, :, l, :] = g.integers(0, int(q), size=(nq, 2, w.n), dtype=np.uint32)
    return out


def uniform_ciphertexts_torch(w: Workload, moduli, num_queries: int | None = None, device="cuda",
                              seed_offset: int = 0):
    """Same role as uniform_ciphertexts but drawn on the device with torch's
    seeded generator (fast for the multi-GB bench batches)."""
    import torch
    nq = w.num_queries if num_queries is None else num_queries
    g = torch.Generator(device=device)
    g.manual_seed(w.seed * 1000003 + seed_offset)
    out = torch.empty((nq, 2, len(moduli), w.n), dtype=torch.int32, device=device)
    for l, q in enumerate(moduli):
        out[:, :, l, :] = torch.randint(0, int(q), (nq, 2, w.n), generator=g, device=device, dtype=torch.int32)
    return out


def uniform_keys_torch(w: Workload, moduli, num_queries: int | None = None, device="cuda", seed_offset: int = 0,
                       chunk: int = 1024):
    """Stand-ins for the two per-query rotation keys of the SIMD formulation
    (SURVEY.md 8(f)-3): int32 [nq][2 keys][2][L][L+1][n] uniform residues,
    residue m (last-but-one axis) below moduli[m] (the L ciphertext limbs and
    the special prime).  A key is (b, a) with a uniform and b = -a s + e + ...
    an RLWE sample, so uniform residues have its distribution; the server
    path is data-oblivious."""
    import torch
    nq = w.num_queries if num_queries is None else num_queries
    L, M = len(moduli) - 1, len(moduli)
    g = torch.Generator(device=device)
    g.manual_seed(w.seed * 1000033 + seed_offset)
    out = torch.empty((nq, 2, 2, L, M, w.n), dtype=torch.int32, device=device)
    for q0 in range(0, nq, chunk):
        q1 = min(nq, q0 + chunk)
        for m, q in enumerate(moduli):
            out[q0:q1, :, :, :, m, :] = torch.randint(0, int(q), (q1 - q0, 2, 2, L, w.n), generator=g,
                                                      device=device, dtype=torch.int32)
    return out

"""Shared helpers for the GPU parity tests (test code; may call oracle/)."""
from __future__ import annotations

import numpy as np

import synth
from oracle import capi


def make_server(w: synth.Workload, entries: np.ndarray, owner=None, rank=0, device=0, resp_format=0):
    """Build and encode a WallyServer for workload w with entries int8 [C][S][d]."""
    import torch
    from paper_2406_06761_b200.wally import WallyServer
    srv = WallyServer(w.n, w.num_limbs, w.d, w.t, device=device, resp_format=resp_format)
    C = entries.shape[0]
    sizes = np.full(C, entries.shape[1], dtype=np.uint32)
    srv.load_clusters(sizes, owner=owner, rank=rank)
    local = srv.local_cluster_ids()
    ent = torch.from_numpy(np.ascontiguousarray(entries[local].reshape(-1, w.d))).to(f"cuda:{device}")
    srv.encode(ent)
    torch.cuda.synchronize()
    return srv


def make_server_ragged(n, L, d, cluster_entries: list, device=0, resp_format=0):
    """Clusters of different sizes: cluster_entries[c] is int8 [S_c][d]."""
    import torch
    from paper_2406_06761_b200.wally import WallyServer
    srv = WallyServer(n, L, d, device=device, resp_format=resp_format)
    sizes = np.array([e.shape[0] for e in cluster_entries], dtype=np.uint32)
    srv.load_clusters(sizes)
    ent = torch.from_numpy(np.ascontiguousarray(np.concatenate(cluster_entries).reshape(-1, d))).cuda(device)
    srv.encode(ent)
    torch.cuda.synchronize()
    return srv


def run_batch(srv, ids: np.ndarray, cts):
    """cts: numpy uint32 [nq][2][L][n] or a torch device tensor. Returns (responses host, offsets)."""
    import torch
    if isinstance(cts, np.ndarray):
        cts = torch.from_numpy(cts.view(np.int32)).cuda(srv.device)
    off = srv.response_layout(ids)
    resp = torch.empty(int(off[-1]), dtype=torch.int32, device=f"cuda:{srv.device}")
    ws = srv.alloc_workspace(ids.size)
    srv.eval_batch(ids, cts, resp, ws)
    srv.check_batch(ws)
    return srv.fetch_responses(resp), off


def oracle_pairs(moduli, cts_host: np.ndarray, pcoefs: np.ndarray, pair_q, pair_pt, threads=0):
    out, _ = capi.server_pairs(moduli, cts_host, pcoefs, np.asarray(pair_q, np.uint32),
                               np.asarray(pair_pt, np.uint32), threads=threads)
    return out


DROP_BITS = 6   # WALLY_RESP_DROP_BITS


def words_per_pt(n: int, d: int, fmt: int) -> int:
    E4 = (n // d + 3) // 4 * 4
    return {0: 2 * n, 1: E4 + n, 2: E4 + 3 * n // 4}[fmt]


def response_of(resp: np.ndarray, off: np.ndarray, q: int, k: int, n: int, d: int = 1, fmt: int = 0) -> np.ndarray:
    """Response words of pair (q, k): [2][n] (full) or the compact word vector."""
    wpp = words_per_pt(n, d, fmt)
    b = int(off[q]) + k * wpp
    r = resp[b:b + wpp]
    return r.reshape(2, n) if fmt == 0 else r


def result_positions(n: int, d: int) -> np.ndarray:
    E = n // d
    return np.arange(E) * d + d - 1


def matches_oracle(got: np.ndarray, want_full: np.ndarray, n: int, d: int, fmt: int) -> bool:
    """Full format: every word equal.  Compact format: c0 at the E result
    coefficients, zero padding to E4, and c1 in full, equal to the oracle's
    full response (the compact form carries exactly those words)."""
    if fmt == 0:
        return np.array_equal(got, want_full)
    E = n // d
    E4 = (E + 3) // 4 * 4
    ok = np.array_equal(got[:E], want_full[0][result_positions(n, d)]) and not got[E:E4].any()
    if fmt == 1:
        return ok and np.array_equal(got[E4:], want_full[1])
    h = capi.drop_lsb(want_full[1], DROP_BITS)            # the oracle's dropped c1 (reading S20)
    body = np.ascontiguousarray(got[E4:])
    lo = body[: n // 2].view(np.uint16)[drop_plane_position(n)]
    hi = body[n // 2:].view(np.uint8)[drop_plane_position(n)]
    return ok and np.array_equal(lo, (h & 0xFFFF).astype(np.uint16)) and np.array_equal(hi, (h >> 16).astype(np.uint8))


def drop_plane_position(n: int) -> np.ndarray:
    """Plane position of coefficient i in WALLY_RESP_COMPACT_DROP (n = 4096): 16 x 256 transpose."""
    i = np.arange(n)
    return (i % 256) * 16 + i // 256


def expand_compact(got: np.ndarray, n: int, d: int, fmt: int = 1, q0: int = 0) -> np.ndarray:
    """[2][n] ciphertext with the compact c0 words at their positions (other
    c0 coefficients zero) and c1 (reconstructed as 64 h mod q_0 when the LSBs
    were dropped): decrypts correctly at the result coefficients."""
    E = n // d
    E4 = (E + 3) // 4 * 4
    full = np.zeros((2, n), np.uint32)
    full[0][result_positions(n, d)] = got[:E]
    if fmt == 1:
        full[1] = got[E4:]
    else:
        body = np.ascontiguousarray(got[E4:])
        pos = drop_plane_position(n)
        h = (body[: n // 2].view(np.uint16)[pos].astype(np.uint64)
             | (body[n // 2:].view(np.uint8)[pos].astype(np.uint64) << 16))
        full[1] = ((h << DROP_BITS) % q0).astype(np.uint32)
    return full


def encrypt_queries(w: synth.Workload, moduli, qvecs: np.ndarray, index_base: int = 0) -> tuple:
    """Oracle encryptions (client role) of query vectors; returns (cts [nq][2][L][n], keys)."""
    cts, keys = [], []
    for i, qv in enumerate(qvecs):
        km = synth.key_material(w, index_base + i, moduli)
        cts.append(capi.encrypt(moduli, w.t, synth.query_message(w, qv), km.s, km.a, km.e))
        keys.append(km)
    return np.stack(cts), keys

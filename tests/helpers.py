"""Shared helpers for the GPU parity tests (test code; may call oracle/)."""
from __future__ import annotations

import numpy as np

import synth
from oracle import capi


def make_server(w: synth.Workload, entries: np.ndarray, owner=None, rank=0, device=0):
    """Build and encode a WallyServer for workload w with entries int8 [C][S][d]."""
    import torch
    from paper_2406_06761_b200.wally import WallyServer
    srv = WallyServer(w.n, w.num_limbs, w.d, w.t, device=device)
    C = entries.shape[0]
    sizes = np.full(C, entries.shape[1], dtype=np.uint32)
    srv.load_clusters(sizes, owner=owner, rank=rank)
    local = srv.local_cluster_ids()
    ent = torch.from_numpy(np.ascontiguousarray(entries[local].reshape(-1, w.d))).to(f"cuda:{device}")
    srv.encode(ent)
    torch.cuda.synchronize()
    return srv


def make_server_ragged(n, L, d, cluster_entries: list, device=0):
    """Clusters of different sizes: cluster_entries[c] is int8 [S_c][d]."""
    import torch
    from paper_2406_06761_b200.wally import WallyServer
    srv = WallyServer(n, L, d, device=device)
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


def response_of(resp: np.ndarray, off: np.ndarray, q: int, k: int, n: int) -> np.ndarray:
    b = int(off[q]) + k * 2 * n
    return resp[b:b + 2 * n].reshape(2, n)


def encrypt_queries(w: synth.Workload, moduli, qvecs: np.ndarray, index_base: int = 0) -> tuple:
    """Oracle encryptions (client role) of query vectors; returns (cts [nq][2][L][n], keys)."""
    cts, keys = [], []
    for i, qv in enumerate(qvecs):
        km = synth.key_material(w, index_base + i, moduli)
        cts.append(capi.encrypt(moduli, w.t, synth.query_message(w, qv), km.s, km.a, km.e))
        keys.append(km)
    return np.stack(cts), keys

"""The cluster-sharded multi-rank path on the GPU, checked against the oracle.

Two processes share the one B200 of the test box (each with its own
WallyServer context on cuda:0).  They talk over gloo on HOST tensors, so no
kernel of one rank ever waits on the other: rank 0 is the ingress holding the
batch (real encryptions by the oracle's client role), the Zipf head cluster is
replicated on both ranks (wally_assign_owners_replicated),
queries are scattered to their owners (dist.Router), evaluated by the CUDA
kernels through the C ABI, and the responses are gathered back on rank 0,
which compares every gathered word with the oracle's response and decrypts
the real queries (Alg 4: per-query work is independent; the
server "distributes them according to the correct clusters").

The NCCL data plane inside the C ABI (wally_scatter_queries /
wally_gather_responses) is exercised at world size 1 (one GPU): the pack
kernel, the local share copy and the gather copy around a one-rank NCCL
communicator, against the oracle as well.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    import synth
    # c5-shaped (N = 4096, L = 2, d = 128, Zipf(1.1) popularity), small enough for the oracle
    return synth.scaled(synth.WORKLOADS["c5"], num_clusters=12, cluster_size=70, num_queries=36)


def _rank_main(rank, world, port, fmt, outq):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import synth
        from oracle import capi
        from paper_2406_06761_b200 import wally as W
        from paper_2406_06761_b200.dist import Router
        from tests import helpers as H
        w = _workload()
        ents = synth.cluster_entries(w)
        ids_all = synth.query_clusters(w)
        E = w.n // w.d
        P = -(-w.cluster_size // E)
        sizes = np.full(w.num_clusters, w.cluster_size, np.uint32)
        # expected work = popularity x P_c, with the Zipf head made heavier than the mean rank
        # load (as c5's top cluster is at 8 ranks), so that it is replicated on both ranks
        wts = synth.cluster_popularity(w) * P
        wts[int(np.argmax(wts))] = wts.sum()
        owner = W.wally_assign_owners_replicated(wts, world)
        replicated = [c for c in range(w.num_clusters) if bin(int(owner[c])).count("1") > 1]
        assert replicated, "the hot cluster must be replicated"
        srv = H.make_server(w, ents, owner=owner, rank=rank, resp_format=fmt)
        qs = srv.moduli
        qv = synth.query_vectors(w, ids_all)
        cts_all, keys = H.encrypt_queries(w, qs, qv)             # the ingress's batch (real encryptions)
        rt = Router(sizes, owner, w.n, w.d, w.num_limbs, resp_format=fmt,
                    pack=lambda idx, c: c[torch.from_numpy(idx.astype(np.int64))].contiguous())
        ids = rt.broadcast_ids(ids_all if rank == 0 else None, ids_all.size)
        plan = rt.plan(ids)
        share = plan.share(rank)
        host_cts = torch.from_numpy(cts_all.view(np.int32)) if rank == 0 else None
        mine = rt.scatter(plan, host_cts)                         # gloo, host tensors
        resp, off = H.run_batch(srv, np.ascontiguousarray(ids[share]), mine.numpy().view(np.uint32))
        assert resp.size == int(plan.resp_words[rank])
        gathered = rt.gather(plan, torch.from_numpy(resp.view(np.int32)))
        checked = decrypted = 0
        if rank == 0:
            g = gathered.numpy().view(np.uint32)
            wpp = H.words_per_pt(w.n, w.d, fmt)
            pcs = {c: capi.encode_cluster(ents[c], w.d, w.n) for c in set(int(x) for x in ids)}
            for q in range(ids.size):
                c = int(ids[q])
                want = H.oracle_pairs(qs, cts_all[q:q + 1], pcs[c], np.zeros(P), np.arange(P))
                for k in range(P):
                    b = int(plan.gathered_off[q]) + k * wpp
                    got = g[b:b + wpp] if fmt else g[b:b + wpp].reshape(2, w.n)
                    assert H.matches_oracle(got, want[k], w.n, w.d, fmt), (q, k)
                    checked += 1
                    full = H.expand_compact(got, w.n, w.d, fmt, qs[0]) if fmt else got
                    dec = capi.decrypt_q0(qs[0], w.t, full, keys[q].s)
                    for j in range(min(E, w.cluster_size - k * E)):
                        dot = int(np.dot(qv[q].astype(np.int64), ents[c][k * E + j].astype(np.int64))) % w.t
                        assert int(dec[j * w.d + w.d - 1]) == dot, (q, k, j)
                        decrypted += 1
            # every query landed on a rank that owns (a replica of) its cluster, and the
            # replicated clusters' queries were split over both ranks
            dest = np.empty(ids.size, int)
            for r in range(world):
                dest[plan.share(r)] = r
            assert all((int(owner[ids[q]]) >> int(dest[q])) & 1 for q in range(ids.size))
            assert any(len(set(dest[ids == c])) > 1 for c in replicated if (ids == c).sum() > 1)
        srv.close()
        dist.barrier()
        dist.destroy_process_group()
        outq.put((rank, "ok", checked, decrypted, int(plan.counts[rank])))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        outq.put((rank, traceback.format_exc(), 0, 0, 0))


@pytest.mark.parametrize("fmt", [0, 2], ids=["full", "compact_drop"])
def test_two_ranks_on_one_gpu_match_oracle(fmt):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, fmt, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, msg, checked, dec, cnt = q.get(timeout=900)
        res[r] = (msg, checked, dec, cnt)
    for p in procs:
        p.join(timeout=120)
    assert all(v[0] == "ok" for v in res.values()), res
    w = _workload()
    E = w.n // w.d
    P = -(-w.cluster_size // E)
    assert res[0][1] == w.num_queries * P                          # every gathered response word-checked
    assert res[0][2] == w.num_queries * w.cluster_size             # every dot product decrypted
    assert res[0][3] > 0 and res[1][3] > 0 and res[0][3] + res[1][3] == w.num_queries
    print(f"two ranks: {res[0][1]} responses bit-exact vs oracle, {res[0][2]} dot products decrypted; "
          f"shares {res[0][3]} + {res[1][3]} queries")


def test_nccl_data_plane_one_rank_matches_oracle():
    """wally_comm_init / wally_scatter_queries / wally_gather_responses on a
    one-rank NCCL communicator (the box has one GPU): pack kernel, local share
    copy and gather copy, responses against the oracle."""
    import torch.distributed as dist
    import synth
    from oracle import capi
    from paper_2406_06761_b200.dist import Router
    from tests import helpers as H
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        w = _workload()
        ents = synth.cluster_entries(w)
        ids = synth.query_clusters(w)
        srv = H.make_server(w, ents, resp_format=1)
        qs = srv.moduli
        qv = synth.query_vectors(w, ids)
        cts, keys = H.encrypt_queries(w, qs, qv)
        sizes = np.full(w.num_clusters, w.cluster_size, np.uint32)
        rt = Router(sizes, np.zeros(w.num_clusters, np.int32), w.n, w.d, w.num_limbs, srv=srv, device="cuda:0",
                    transport="wally")
        assert srv.comm_world == 1 and srv.comm_rank == 0
        plan = rt.plan(ids)
        dev_cts = torch.from_numpy(cts.view(np.int32)).cuda()
        mine = rt.scatter(plan, dev_cts)
        torch.cuda.synchronize()
        assert torch.equal(mine, dev_cts[torch.from_numpy(plan.share(0).astype(np.int64)).cuda()])
        resp, off = H.run_batch(srv, np.ascontiguousarray(ids[plan.share(0)]), mine)
        g = rt.gather(plan, torch.from_numpy(resp.view(np.int32)).cuda()).cpu().numpy().view(np.uint32)
        srv.comm_check()
        E = w.n // w.d
        P = -(-w.cluster_size // E)
        wpp = H.words_per_pt(w.n, w.d, 1)
        for q in range(ids.size):
            c = int(ids[q])
            want = H.oracle_pairs(qs, cts[q:q + 1], capi.encode_cluster(ents[c], w.d, w.n), np.zeros(P), np.arange(P))
            for k in range(P):
                b = int(plan.gathered_off[q]) + k * wpp
                assert H.matches_oracle(g[b:b + wpp], want[k], w.n, w.d, 1), (q, k)
        srv.close()
    finally:
        dist.destroy_process_group()

"""Multi-rank host logic on CPU: routing plan, ownership, and the
scatter/gather collectives of paper_2406_06761_b200.dist over a world-size-2
gloo process group (the GPU box has one device; the NCCL path runs the same
code with device tensors).  No CUDA compute is called here."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def W():
    from paper_2406_06761_b200 import build
    build.build()
    from paper_2406_06761_b200 import wally
    return wally


def _ref_plan(ids, sizes, owner, n, d, world):
    """Definition written out: stable grouping by owner, P_c = ceil(S_c / floor(n/d))."""
    E = n // d
    dest = [int(owner[c]) if owner is not None else 0 for c in ids]
    order = [q for r in range(world) for q in range(len(ids)) if dest[q] == r]
    counts = [dest.count(r) for r in range(world)]
    words = [sum(2 * n * -(-int(sizes[ids[q]]) // E) for q in range(len(ids)) if dest[q] == r) for r in range(world)]
    off, base = {}, 0
    for r in range(world):
        for q in order:
            if dest[q] == r:
                off[q] = base
                base += 2 * n * -(-int(sizes[ids[q]]) // E)
    return counts, order, words, [off[q] for q in range(len(ids))] + [base]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_route_plan_matches_definition(W, world):
    rng = np.random.default_rng(world)
    C, n, d = 37, 1024, 96
    sizes = rng.integers(1, 200, size=C).astype(np.uint32)
    owner = rng.integers(0, world, size=C).astype(np.int32)
    ids = rng.integers(0, C, size=301).astype(np.uint32)
    p = W.wally_route_plan(ids, sizes, owner, n, d, world)
    counts, order, words, goff = _ref_plan(ids, sizes, owner, n, d, world)
    assert p.counts.tolist() == counts
    assert p.order.tolist() == order
    assert p.resp_words.tolist() == words
    assert p.gathered_off.tolist() == goff
    for r in range(world):
        assert all(owner[ids[q]] == r for q in p.share(r))


def test_route_plan_edge_cases(W):
    sizes = np.array([5, 7], np.uint32)
    p = W.wally_route_plan(np.zeros(0, np.uint32), sizes, np.array([0, 1], np.int32), 64, 8, 2)
    assert p.counts.tolist() == [0, 0] and p.gathered_off.tolist() == [0]
    p = W.wally_route_plan(np.array([1, 1, 0], np.uint32), sizes, None, 64, 8, 1)   # no owner map: rank 0
    assert p.order.tolist() == [0, 1, 2]
    with pytest.raises(W.WallyError) as e:
        W.wally_route_plan(np.array([2], np.uint32), sizes, None, 64, 8, 1)
    assert e.value.code == -3
    with pytest.raises(W.WallyError):
        W.wally_route_plan(np.array([0], np.uint32), sizes, np.array([0, 2], np.int32), 64, 8, 2)


def test_assign_owners_lpt(W):
    w = np.array([5.0, 1.0, 4.0, 4.0, 2.0, 2.0, 0.0])
    own = W.wally_assign_owners(w, 2)
    # LPT by hand: 5->0, 4->1, 4->1 (4<5), 2->0 (5<8), 2->0 (7<8), 1->0? loads 9 vs 8 -> 1, 0->1 (9 vs 9 -> 0)
    assert own.tolist() == [0, 1, 1, 1, 0, 0, 0]
    loads = [w[own == r].sum() for r in range(2)]
    assert abs(loads[0] - loads[1]) <= w.max()
    zipf = (np.arange(1, 1001) ** -1.1)
    own8 = W.wally_assign_owners(zipf, 8)
    ld = np.array([zipf[own8 == r].sum() for r in range(8)])
    assert ld.max() - ld.min() <= zipf.max() + 1e-12


def test_assign_owners_replicated_splits_only_heavy_clusters(W):
    zipf = np.arange(1, 1001) ** -1.1
    for world in (1, 2, 4, 8, 16):
        m = W.wally_assign_owners_replicated(zipf, world)
        reps = np.array([bin(int(x)).count("1") for x in m])
        assert (reps >= 1).all() and (reps <= world).all()
        assert all(max(W.mask_ranks(x)) < world for x in m)
        target = zipf.sum() / world
        # a cluster is replicated iff it is heavier than the mean rank load
        assert np.array_equal(reps > 1, zipf > target) or world == 1
        load = np.zeros(world)
        for c, x in enumerate(m):
            for r in W.mask_ranks(x):
                load[r] += zipf[c] / reps[c]
        assert load.max() - load.min() <= (zipf / reps).max() + 1e-12
    # equal weights: no replication while clusters >= ranks ...
    m = W.wally_assign_owners_replicated(np.ones(7), 5)
    assert all(bin(int(x)).count("1") == 1 for x in m)
    # ... and with more ranks than clusters every cluster (weight 1 > 3/5) gets
    # ceil(1 / 0.6) = 2 replicas, spread so that every rank holds work
    m = W.wally_assign_owners_replicated(np.ones(3), 5)
    assert all(bin(int(x)).count("1") == 2 for x in m)
    assert sorted(set(r for x in m for r in W.mask_ranks(x))) == [0, 1, 2, 3, 4]


def _ref_plan_replicated(ids, sizes, mask, n, d, world):
    """Definition written out: the j-th query of cluster c goes to the
    (j mod r_c)-th lowest replica rank of c."""
    E = n // d
    seen = {}
    dest = []
    for c in ids:
        ranks = [r for r in range(64) if (int(mask[c]) >> r) & 1]
        j = seen.get(int(c), 0)
        seen[int(c)] = j + 1
        dest.append(ranks[j % len(ranks)])
    order = [q for r in range(world) for q in range(len(ids)) if dest[q] == r]
    counts = [dest.count(r) for r in range(world)]
    words = [sum(2 * n * -(-int(sizes[ids[q]]) // E) for q in range(len(ids)) if dest[q] == r) for r in range(world)]
    return counts, order, words


def test_route_plan_replicated_matches_definition(W):
    rng = np.random.default_rng(4)
    C, n, d, world = 29, 1024, 100, 6
    sizes = rng.integers(1, 300, size=C).astype(np.uint32)
    w = rng.random(C) ** 6
    w[3] = 2 * w.sum()                  # a hot cluster: heavier than the mean rank load
    mask = W.wally_assign_owners_replicated(w, world)
    assert any(bin(int(x)).count("1") > 1 for x in mask)
    ids = rng.choice(C, size=500, p=w / w.sum()).astype(np.uint32)
    p = W.wally_route_plan(ids, sizes, mask, n, d, world)
    counts, order, words = _ref_plan_replicated(ids, sizes, mask, n, d, world)
    assert p.counts.tolist() == counts and p.order.tolist() == order and p.resp_words.tolist() == words
    with pytest.raises(W.WallyError):
        bad = mask.copy()
        bad[0] = np.uint64(0)
        W.wally_route_plan(ids, sizes, bad, n, d, world)
    with pytest.raises(W.WallyError):
        bad = mask.copy()
        bad[0] = np.uint64(1 << world)
        W.wally_route_plan(ids, sizes, bad, n, d, world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outq, replicated=False):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2406_06761_b200 import wally as W
        from paper_2406_06761_b200.dist import Router
        n, L, d, C, nq = 64, 2, 10, 9, 23
        rng = np.random.default_rng(5)
        sizes = rng.integers(1, 40, size=C).astype(np.uint32)
        ids_all = rng.integers(0, C, size=nq).astype(np.uint32)
        cts_all = torch.from_numpy(rng.integers(0, 2**30, size=(nq, 2, L, n)).astype(np.int32))
        if replicated:
            wts = sizes.astype(np.float64)
            wts[2] = wts.sum()          # one hot cluster, heavier than the mean rank load
            owner = W.wally_assign_owners_replicated(wts, world)
            assert bin(int(owner[2])).count("1") == world
        else:
            owner = W.wally_assign_owners(sizes.astype(np.float64), world)

        def host_pack(index, cts):
            return cts[torch.from_numpy(index.astype(np.int64))].contiguous()

        rt = Router(sizes, owner, n, d, L, pack=host_pack)
        ids = rt.broadcast_ids(ids_all if rank == 0 else None, nq)
        assert np.array_equal(ids, ids_all)
        plan = rt.plan(ids)
        share = plan.share(rank)
        local = rt.scatter(plan, cts_all if rank == 0 else None)
        assert torch.equal(local, cts_all[torch.from_numpy(share.astype(np.int64))])
        # stand-in evaluator (the CUDA kernels are not available on CPU): query q's
        # P_c*2n response words = q*1000 + word index
        E = n // d
        parts = []
        for q in share:
            P = -(-int(sizes[ids[q]]) // E)
            parts.append(torch.arange(P * 2 * n, dtype=torch.int32) + int(q) * 1000)
        resp = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.int32)
        assert resp.numel() == int(plan.resp_words[rank])
        out = rt.gather(plan, resp)
        if rank == 0:
            assert out.numel() == int(plan.gathered_off[-1])
            for qq in range(nq):
                words = 2 * n * -(-int(sizes[ids[qq]]) // E)
                b = int(plan.gathered_off[qq])
                assert torch.equal(out[b:b + words], torch.arange(words, dtype=torch.int32) + qq * 1000), qq
        dist.barrier()
        dist.destroy_process_group()
        outq.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback
        outq.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,replicated", [(2, False), (2, True)])
def test_scatter_gather_gloo(W, world, replicated):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, replicated)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res

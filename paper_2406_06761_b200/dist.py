"""Multi-GPU plumbing of the hot path: cluster-sharded data parallelism.

north_star: "Clusters are partitioned across the 8 GPUs of one B200 box, each
rank owning a disjoint cluster set, and queries are routed to the owning
rank, with NCCL over NVLink only for query scatter and response gather."
(SURVEY.md §8(a) row a7, §8(e).)  Alg 4's per-query work is
independent across queries and plaintexts, so nothing else is exchanged.

  * ownership  : wally_assign_owners (C ABI) -- greedy LPT on expected work,
                 or wally_assign_owners_replicated: clusters heavier than
                 the mean rank load are split over several ranks (SURVEY
                 §8(f)-4, the Zipf skew of configs[4])
  * routing    : wally_route_plan (C ABI) -- identical on every rank, so only
                 the ciphertexts move; the ingress broadcasts the cluster ids
  * scatter    : the ingress packs each rank's share contiguously with the
                 wally_pack_queries kernel and sends it with grouped P2P
                 (torch.distributed batch_isend_irecv: NCCL over NVLink on the
                 GPU box, gloo in the CPU tests)
  * gather     : optional; each rank sends its response buffer to the
                 ingress, which receives the rank blocks back to back (the
                 layout wally_route_plan's gathered offsets describe)

This module only marshals: the routing plan is computed by the C library,
the packing by its kernel, the transfers by torch.distributed.
"""
from __future__ import annotations

import numpy as np

from . import wally as W


class Router:
    """Scatter/gather of one batch between the ingress rank `src` and the
    owners.  `pack` (default: the wally_pack_queries kernel of `srv`) forms
    the contiguous send buffer of a share on the ingress; tests inject a
    host implementation to exercise the collective logic on CPU tensors."""

    def __init__(self, cluster_sizes, owner, n: int, d: int, L: int, group=None, src: int = 0, srv=None,
                 pack=None, device=None, resp_format: int | None = None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.src = src
        self.sizes = np.ascontiguousarray(cluster_sizes, dtype=np.uint32)
        # int32 owning rank per cluster, or uint64 replica masks (hot-cluster replication)
        if owner is None:
            self.owner = None
        elif np.asarray(owner).dtype == np.uint64:
            self.owner = np.ascontiguousarray(owner, dtype=np.uint64)
        else:
            self.owner = np.ascontiguousarray(owner, dtype=np.int32)
        self.n, self.d, self.L = n, d, L
        if resp_format is None:
            resp_format = srv.resp_format if srv is not None else W.WALLY_RESP_FULL
        self.resp_format = resp_format
        self.row = 2 * L * n
        self.device = device if device is not None else "cpu"
        if pack is None:
            assert srv is not None, "Router needs a WallyServer (pack kernel) or an explicit pack function"

            def pack(index_np, cts):
                idx = torch.from_numpy(index_np.astype(np.int32)).to(cts.device)
                out = torch.empty((index_np.size, *cts.shape[1:]), dtype=cts.dtype, device=cts.device)
                srv.pack_queries(idx, cts, out)
                return out
        self.pack = pack

    def broadcast_ids(self, ids: np.ndarray | None, nq: int) -> np.ndarray:
        """The ingress's cluster ids to every rank (small: 4 B per query)."""
        torch = self.torch
        t = torch.empty(nq, dtype=torch.int32, device=self.device)
        if self.rank == self.src:
            t.copy_(torch.from_numpy(np.ascontiguousarray(ids, dtype=np.uint32).view(np.int32)))
        self.dist.broadcast(t, self.src, group=self.group)
        return t.cpu().numpy().view(np.uint32)

    def plan(self, ids: np.ndarray) -> W.RoutePlan:
        return W.wally_route_plan(ids, self.sizes, self.owner, self.n, self.d, self.world, self.resp_format)

    def scatter(self, plan: W.RoutePlan, cts):
        """cts: [nq][2][L][n] int32 tensor on the ingress (ignored elsewhere).
        Returns this rank's share [counts[rank]][2][L][n] in its local order."""
        torch, dist = self.torch, self.dist
        mine = int(plan.counts[self.rank])
        ops = []
        if self.rank == self.src:
            packed = self.pack(plan.order, cts) if plan.order.size else None
            local = None
            for r in range(self.world):
                b, e = int(plan.starts[r]), int(plan.starts[r + 1])
                if r == self.src:
                    local = packed[b:e] if e > b else torch.empty((0, 2, self.L, self.n), dtype=torch.int32,
                                                                   device=self.device)
                elif e > b:
                    ops.append(dist.P2POp(dist.isend, packed[b:e].contiguous(), r, group=self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            return local
        buf = torch.empty((mine, 2, self.L, self.n), dtype=torch.int32, device=self.device)
        if mine:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.irecv, buf, self.src, group=self.group)]):
                w.wait()
        return buf

    def gather(self, plan: W.RoutePlan, resp_local):
        """Concatenate every rank's response buffer, in rank order, on the
        ingress (query q's responses start at plan.gathered_off[q]).  Returns
        the gathered int32 tensor on the ingress, None elsewhere."""
        torch, dist = self.torch, self.dist
        if self.rank == self.src:
            total = int(plan.gathered_off[-1])
            out = torch.empty(total, dtype=torch.int32, device=self.device)
            base = np.concatenate([[0], np.cumsum(plan.resp_words.astype(np.int64))])
            ops = []
            for r in range(self.world):
                b, e = int(base[r]), int(base[r + 1])
                if e == b:
                    continue
                if r == self.src:
                    out[b:e].copy_(resp_local[:e - b])
                else:
                    ops.append(dist.P2POp(dist.irecv, out[b:e], r, group=self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            return out
        words = int(plan.resp_words[self.rank])
        if words:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, resp_local[:words].contiguous(), self.src,
                                                        group=self.group)]):
                w.wait()
        return None

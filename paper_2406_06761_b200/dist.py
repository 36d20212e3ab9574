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
                 over the control group (host tensors: no device sync)
  * scatter    : the ingress packs each rank's share contiguously and sends
                 it to its owner.  transport="wally": the C ABI's own NCCL
                 data plane (wally_scatter_queries: pack_rows kernel + grouped
                 ncclSend/ncclRecv inside libwally.so; Python only passes the
                 NCCL unique id).  transport="torch": torch.distributed
                 batch_isend_irecv (gloo on host tensors in the CPU tests and
                 the two-process GPU test)
  * gather     : optional; each rank sends its response buffer to the
                 ingress, which receives the rank blocks back to back (the
                 layout wally_route_plan's gathered offsets describe)

This module only marshals: the routing plan is computed by the C library,
the packing by its kernel, the transfers by NCCL (or torch.distributed).
"""
from __future__ import annotations

import numpy as np

from . import wally as W


class Router:
    """Scatter/gather of one batch between the ingress rank `src` and the
    owners.

    transport  "torch" (torch.distributed P2P on the tensors' device) or
               "wally" (the C ABI's NCCL data plane; needs `srv`, device tensors)
    group      process group of the torch transport and of comm setup (None = default)
    ctrl_group process group for the host-side cluster-id broadcast (a gloo
               group keeps it off the device; None = `group`)
    pack       torch transport only: forms the contiguous send buffer of a
               share on the ingress (default: the wally_pack_queries kernel of
               `srv`); tests inject a host implementation."""

    def __init__(self, cluster_sizes, owner, n: int, d: int, L: int, group=None, src: int = 0, srv=None,
                 pack=None, device=None, resp_format: int | None = None, transport: str = "torch",
                 ctrl_group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.group = group
        self.ctrl_group = ctrl_group if ctrl_group is not None else group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.src = src                      # group-local rank of the ingress
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
        self.srv = srv
        assert transport in ("torch", "wally")
        self.transport = transport
        if transport == "wally":
            assert srv is not None, "the wally transport runs on the server context's NCCL communicator"
            uid = torch.zeros(W.WALLY_COMM_ID_BYTES, dtype=torch.uint8)
            if self.rank == src:
                uid.copy_(torch.frombuffer(bytearray(W.wally_comm_unique_id()), dtype=torch.uint8))
            self._bcast(uid, src, self.ctrl_group)
            srv.comm_init(self.rank, self.world, bytes(uid.numpy()))
        if pack is None and transport == "torch":
            assert srv is not None, "Router needs a WallyServer (pack kernel) or an explicit pack function"

            def pack(index_np, cts):
                idx = torch.from_numpy(index_np.astype(np.int32)).to(cts.device)
                out = torch.empty((index_np.size, *cts.shape[1:]), dtype=cts.dtype, device=cts.device)
                srv.pack_queries(idx, cts, out)
                return out
        self.pack = pack

    # torch.distributed takes global ranks: map the group-local peers
    def _peer(self, r: int, group=None) -> int:
        g = self.group if group is None else group
        return r if g is None else self.dist.get_global_rank(g, r)

    def _bcast(self, t, src: int, group):
        self.dist.broadcast(t, self._peer(src, group), group=group)

    def broadcast_ids(self, ids: np.ndarray | None, nq: int) -> np.ndarray:
        """The ingress's cluster ids to every rank (4 B per query).  Over a
        gloo control group the tensor stays on the host (no device sync)."""
        torch = self.torch
        be = self.dist.get_backend(self.ctrl_group)
        host = "gloo" in str(be)
        t = torch.empty(nq, dtype=torch.int32, device="cpu" if host else self.device)
        if self.rank == self.src:
            t.copy_(torch.from_numpy(np.ascontiguousarray(ids, dtype=np.uint32).view(np.int32)))
        self._bcast(t, self.src, self.ctrl_group)
        return (t if host else t.cpu()).numpy().view(np.uint32)

    def plan(self, ids: np.ndarray) -> W.RoutePlan:
        return W.wally_route_plan(ids, self.sizes, self.owner, self.n, self.d, self.world, self.resp_format)

    def scatter(self, plan: W.RoutePlan, cts, out=None, pack_buf=None, order_dev=None):
        """cts: [nq][2][L][n] int32 tensor on the ingress (ignored elsewhere).
        Returns this rank's share [counts[rank]][2][L][n] in its local order.
        wally transport: `out` (the share buffer), `pack_buf` (ingress scratch
        of cts' shape) and `order_dev` (plan.order on the device) may be passed
        in to keep allocations and host->device copies out of a timed step."""
        torch, dist = self.torch, self.dist
        mine = int(plan.counts[self.rank])
        if self.transport == "wally":
            if out is None:
                out = torch.empty((mine, 2, self.L, self.n), dtype=torch.int32, device=self.device)
            if self.rank == self.src:
                if order_dev is None:
                    order_dev = torch.from_numpy(plan.order.view(np.int32)).to(self.device)
                if pack_buf is None:
                    pack_buf = torch.empty_like(cts)
                self.srv.scatter_queries(self.src, plan.counts, order_dev, cts, pack_buf, out)
            else:
                self.srv.scatter_queries(self.src, plan.counts, share_dev=out)
            return out[:mine]
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
                    ops.append(dist.P2POp(dist.isend, packed[b:e].contiguous(), self._peer(r), group=self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            return local
        buf = torch.empty((mine, 2, self.L, self.n), dtype=torch.int32, device=self.device)
        if mine:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.irecv, buf, self._peer(self.src), group=self.group)]):
                w.wait()
        return buf

    def gather(self, plan: W.RoutePlan, resp_local):
        """Concatenate every rank's response buffer, in rank order, on the
        ingress (query q's responses start at plan.gathered_off[q]).  Returns
        the gathered int32 tensor on the ingress, None elsewhere."""
        torch, dist = self.torch, self.dist
        if self.transport == "wally":
            out = None
            if self.rank == self.src:
                out = torch.empty(max(1, int(plan.gathered_off[-1])), dtype=torch.int32, device=self.device)
            self.srv.gather_responses(self.src, plan.resp_words, resp_local, out)
            return out[:int(plan.gathered_off[-1])] if out is not None else None
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
                    ops.append(dist.P2POp(dist.irecv, out[b:e], self._peer(r), group=self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            return out
        words = int(plan.resp_words[self.rank])
        if words:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, resp_local[:words].contiguous(),
                                                        self._peer(self.src), group=self.group)]):
                w.wait()
        return None

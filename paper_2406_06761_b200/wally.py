"""Thin Python binding of the C ABI in include/wally.h (libwally.so).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  PyTorch provides device memory (tensors whose
data_ptr() is handed to the library) and streams.  There is no CPU fallback:
if libwally.so cannot be loaded, importing this module raises.

The functions keep the C names (wally_find_moduli, wally_create, ...);
`WallyServer` bundles them for the usual ServerInit -> eval -> fetch flow.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

# WALLY_LIB: load an alternative build of the same library (kernel-variant experiments).
_LIB_PATH = os.environ.get("WALLY_LIB", _build.LIB)

WALLY_MAX_LIMBS = 4
STATUS = {0: "WALLY_OK", -1: "WALLY_E_ARG", -2: "WALLY_E_PARAMS", -3: "WALLY_E_UNKNOWN_CLUSTER",
          -4: "WALLY_E_RESIDUE", -5: "WALLY_E_STATE", -6: "WALLY_E_CUDA", -7: "WALLY_E_NCCL", -8: "WALLY_E_OOM"}
WALLY_COMM_ID_BYTES = 128

EXPORTED = [
    "wally_find_moduli", "wally_create", "wally_destroy", "wally_last_error", "wally_load_clusters",
    "wally_plaintext_store_bytes", "wally_local_entry_count", "wally_encode_plaintexts_ntt",
    "wally_response_layout", "wally_workspace_bytes", "wally_eval_batch", "wally_check_batch",
    "wally_fetch_responses", "wally_host_workspace_bytes", "wally_eval_batch_host", "wally_route_queries",
    "wally_ntt_forward", "wally_ntt_inverse", "wally_kernel_launches", "wally_enable_stage_timing",
    "wally_stage_times", "wally_assign_owners", "wally_route_plan", "wally_pack_queries",
    "wally_response_words_per_plaintext", "wally_assign_owners_replicated", "wally_route_plan_replicated",
    "wally_load_clusters_replicated", "wally_modmuls_per_pair", "wally_comm_unique_id", "wally_comm_init",
    "wally_comm_check", "wally_scatter_queries", "wally_gather_responses",
]


class WallyError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class wally_params(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("num_limbs", ctypes.c_uint32), ("t", ctypes.c_uint32),
                ("d", ctypes.c_uint32), ("moduli", ctypes.c_uint32 * WALLY_MAX_LIMBS),
                ("resp_format", ctypes.c_uint32)]


WALLY_RESP_FULL = 0
WALLY_RESP_COMPACT = 1
WALLY_RESP_COMPACT_DROP = 2
WALLY_RESP_DROP_BITS = 6


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python -m paper_2406_06761_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    vp, u32, i32, u64, sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    sig = {
        "wally_find_moduli": ([u32, u32, P(u32)], ctypes.c_int),
        "wally_create": ([P(wally_params), ctypes.c_int, P(vp)], ctypes.c_int),
        "wally_destroy": ([vp], None),
        "wally_last_error": ([vp], ctypes.c_char_p),
        "wally_load_clusters": ([vp, u32, P(u32), P(i32), i32], ctypes.c_int),
        "wally_plaintext_store_bytes": ([vp, P(sz)], ctypes.c_int),
        "wally_local_entry_count": ([vp, P(u64)], ctypes.c_int),
        "wally_encode_plaintexts_ntt": ([vp, vp, vp, sz, vp], ctypes.c_int),
        "wally_response_layout": ([vp, u32, P(u32), P(u64), P(u64)], ctypes.c_int),
        "wally_workspace_bytes": ([vp, u32, P(sz)], ctypes.c_int),
        "wally_eval_batch": ([vp, u32, P(u32), vp, vp, u64, vp, sz, vp], ctypes.c_int),
        "wally_check_batch": ([vp, vp, vp], ctypes.c_int),
        "wally_fetch_responses": ([vp, vp, u64, vp, vp], ctypes.c_int),
        "wally_host_workspace_bytes": ([vp, u32, P(sz)], ctypes.c_int),
        "wally_eval_batch_host": ([vp, u32, P(u32), vp, vp, u64, u32, vp, sz, vp], ctypes.c_int),
        "wally_route_queries": ([vp, u32, P(u32), P(i32)], ctypes.c_int),
        "wally_ntt_forward": ([vp, vp, vp, u32, vp], ctypes.c_int),
        "wally_ntt_inverse": ([vp, vp, vp, u32, vp], ctypes.c_int),
        "wally_kernel_launches": ([vp], u64),
        "wally_enable_stage_timing": ([vp, ctypes.c_int], ctypes.c_int),
        "wally_stage_times": ([vp, P(ctypes.c_double), P(u64)], ctypes.c_int),
        "wally_assign_owners": ([u32, P(ctypes.c_double), u32, P(i32)], ctypes.c_int),
        "wally_route_plan": ([u32, P(u32), u32, P(u32), P(i32), u32, u32, u32, u32, P(u32), P(u32), P(u64),
                              P(u64)], ctypes.c_int),
        "wally_response_words_per_plaintext": ([vp, P(u64)], ctypes.c_int),
        "wally_assign_owners_replicated": ([u32, P(ctypes.c_double), u32, P(u64)], ctypes.c_int),
        "wally_route_plan_replicated": ([u32, P(u32), u32, P(u32), P(u64), u32, u32, u32, u32, P(u32), P(u32),
                                         P(u64), P(u64)], ctypes.c_int),
        "wally_load_clusters_replicated": ([vp, u32, P(u32), P(u64), i32], ctypes.c_int),
        "wally_modmuls_per_pair": ([vp, P(u64)], ctypes.c_int),
        "wally_pack_queries": ([vp, u32, vp, vp, vp, vp], ctypes.c_int),
        "wally_comm_unique_id": ([vp], ctypes.c_int),
        "wally_comm_init": ([vp, i32, i32, vp], ctypes.c_int),
        "wally_comm_check": ([vp], ctypes.c_int),
        "wally_scatter_queries": ([vp, i32, P(u32), vp, vp, vp, vp, vp], ctypes.c_int),
        "wally_gather_responses": ([vp, i32, P(u64), vp, vp, vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()


def _u32p(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _check_host_words(buf, words: int, name: str, exact: bool = False) -> int:
    """A host buffer the C side reads or writes `words` uint32 words of: a
    contiguous 4-byte numpy array or CPU tensor with at least (or, with
    exact=True, exactly) that many elements.  Returns its address."""
    if hasattr(buf, "data_ptr"):
        assert not buf.is_cuda, f"{name} must be host memory"
        assert buf.is_contiguous() and buf.element_size() == 4, f"{name} must be contiguous 32-bit"
        n, ptr = buf.numel(), buf.data_ptr()
    else:
        assert buf.flags["C_CONTIGUOUS"] and buf.dtype.itemsize == 4, f"{name} must be contiguous 32-bit"
        n, ptr = buf.size, buf.ctypes.data
    assert (n == words) if exact else (n >= words), f"{name} has {n} words, needs {words}"
    return ptr


def _check(rc: int, ctx=None):
    if rc != 0:
        msg = lib.wally_last_error(ctx)
        raise WallyError(rc, msg.decode() if msg else "")


def wally_find_moduli(n: int, num_limbs: int) -> list[int]:
    out = np.zeros(num_limbs, dtype=np.uint32)
    _check(lib.wally_find_moduli(n, num_limbs, _u32p(out)))
    return [int(x) for x in out]


def wally_comm_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for wally_comm_init (call on one rank, share with all)."""
    buf = (ctypes.c_uint8 * WALLY_COMM_ID_BYTES)()
    _check(lib.wally_comm_unique_id(buf))
    return bytes(buf)


def wally_assign_owners(weights, world: int) -> np.ndarray:
    """Cluster -> owning rank, greedy LPT on the given per-cluster weights (C ABI)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros(w.size, dtype=np.int32)
    _check(lib.wally_assign_owners(w.size, w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), world,
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return out


def wally_assign_owners_replicated(weights, world: int) -> np.ndarray:
    """uint64 [clusters] replica masks: heavy clusters split over several ranks (C ABI)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros(w.size, dtype=np.uint64)
    _check(lib.wally_assign_owners_replicated(w.size, w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), world,
                                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return out


def mask_ranks(mask: int) -> list[int]:
    return [r for r in range(64) if (int(mask) >> r) & 1]


class RoutePlan:
    """Result of wally_route_plan (see include/wally.h)."""

    def __init__(self, counts, order, resp_words, gathered_off):
        self.counts, self.order, self.resp_words, self.gathered_off = counts, order, resp_words, gathered_off
        self.starts = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)

    def share(self, rank: int) -> np.ndarray:
        """Input indices of the queries routed to `rank` (its local query order)."""
        return self.order[self.starts[rank]:self.starts[rank + 1]]


def wally_route_plan(cluster_of_query, cluster_sizes, owner, n: int, d: int, world: int,
                     resp_format: int = WALLY_RESP_FULL) -> RoutePlan:
    """owner: int32 [clusters] rank per cluster, None (all on rank 0), or a uint64
    replica-mask array (wally_assign_owners_replicated)."""
    ids = np.ascontiguousarray(cluster_of_query, dtype=np.uint32)
    sizes = np.ascontiguousarray(cluster_sizes, dtype=np.uint32)
    counts = np.zeros(world, dtype=np.uint32)
    order = np.zeros(ids.size, dtype=np.uint32)
    words = np.zeros(world, dtype=np.uint64)
    goff = np.zeros(ids.size + 1, dtype=np.uint64)
    if owner is not None and np.asarray(owner).dtype == np.uint64:
        mask = np.ascontiguousarray(owner, dtype=np.uint64)
        _check(lib.wally_route_plan_replicated(ids.size, _u32p(ids), sizes.size, _u32p(sizes),
                                               mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n, d,
                                               resp_format, world, _u32p(counts), _u32p(order),
                                               words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                               goff.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
        return RoutePlan(counts, order, words, goff)
    own = None
    if owner is not None:
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        own = owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    _check(lib.wally_route_plan(ids.size, _u32p(ids), sizes.size, _u32p(sizes), own, n, d, resp_format, world,
                                _u32p(counts),
                                _u32p(order), words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                goff.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return RoutePlan(counts, order, words, goff)


class WallyServer:
    """ServerInit + ServerComputation on one device (one rank).

    Device buffers come from PyTorch: the plaintext store (kept for the
    server's life), per-batch workspaces and response buffers."""

    def __init__(self, n: int, num_limbs: int, d: int, t: int = 65537, moduli=None, device: int = 0,
                 resp_format: int = WALLY_RESP_FULL):
        import torch
        self.torch = torch
        self.n, self.L, self.d, self.t = n, num_limbs, d, t
        self.resp_format = resp_format
        self.E = n // d
        self.E4 = (self.E + 3) // 4 * 4
        self.moduli = list(moduli) if moduli is not None else wally_find_moduli(n, num_limbs)
        self.device = device
        p = wally_params(n=n, num_limbs=num_limbs, t=t, d=d, resp_format=resp_format)
        for i, q in enumerate(self.moduli):
            p.moduli[i] = q
        h = ctypes.c_void_p()
        _check(lib.wally_create(ctypes.byref(p), device, ctypes.byref(h)))
        self.ctx = h
        w = ctypes.c_uint64()
        _check(lib.wally_response_words_per_plaintext(self.ctx, ctypes.byref(w)), self.ctx)
        self.words_per_plaintext = w.value
        self.store = None
        self._ws = None

    def close(self):
        if getattr(self, "ctx", None):
            lib.wally_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- ServerInit ----
    def load_clusters(self, cluster_sizes, owner=None, rank: int = 0):
        """owner: None (all local), int32 [clusters] owning rank, or uint64 [clusters]
        replica masks (wally_assign_owners_replicated)."""
        sizes = np.ascontiguousarray(cluster_sizes, dtype=np.uint32)
        if owner is not None and np.asarray(owner).dtype == np.uint64:
            owner = np.ascontiguousarray(owner, dtype=np.uint64)
            _check(lib.wally_load_clusters_replicated(self.ctx, sizes.size, _u32p(sizes),
                                                      owner.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), rank),
                   self.ctx)
        else:
            own = None
            if owner is not None:
                owner = np.ascontiguousarray(owner, dtype=np.int32)
                own = owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            _check(lib.wally_load_clusters(self.ctx, sizes.size, _u32p(sizes), own, rank), self.ctx)
        self.total_clusters = sizes.size
        self._sizes, self._owner, self._rank = sizes, owner, rank
        b = ctypes.c_size_t()
        _check(lib.wally_plaintext_store_bytes(self.ctx, ctypes.byref(b)), self.ctx)
        self.store_bytes = b.value
        c = ctypes.c_uint64()
        _check(lib.wally_local_entry_count(self.ctx, ctypes.byref(c)), self.ctx)
        self.local_entries = c.value

    def local_cluster_ids(self) -> np.ndarray:
        """Ascending ids of the clusters this context owns (the order of the entries array)."""
        if self._owner is None:
            return np.arange(self.total_clusters, dtype=np.uint32)
        if self._owner.dtype == np.uint64:
            return np.nonzero((self._owner >> np.uint64(self._rank)) & np.uint64(1))[0].astype(np.uint32)
        return np.nonzero(self._owner == self._rank)[0].astype(np.uint32)

    def encode(self, entries_dev, stream=None):
        """entries_dev: torch int8 [local_entries, d] on the device."""
        torch = self.torch
        assert entries_dev.dtype == torch.int8 and entries_dev.is_cuda and entries_dev.is_contiguous()
        assert entries_dev.numel() == self.local_entries * self.d
        self.store = torch.empty(self.store_bytes // 4, dtype=torch.int32, device=entries_dev.device)
        _check(lib.wally_encode_plaintexts_ntt(self.ctx, entries_dev.data_ptr(), self.store.data_ptr(),
                                               self.store_bytes, _stream(stream)), self.ctx)

    # ---- batches ----
    def response_layout(self, cluster_of_query) -> np.ndarray:
        ids = np.ascontiguousarray(cluster_of_query, dtype=np.uint32)
        off = np.zeros(ids.size + 1, dtype=np.uint64)
        _check(lib.wally_response_layout(self.ctx, ids.size, _u32p(ids),
                                         off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), None), self.ctx)
        return off

    def workspace_bytes(self, nq: int) -> int:
        b = ctypes.c_size_t()
        _check(lib.wally_workspace_bytes(self.ctx, nq, ctypes.byref(b)), self.ctx)
        return b.value

    def alloc_workspace(self, nq: int):
        torch = self.torch
        nbytes = self.workspace_bytes(nq)
        return torch.empty((nbytes + 3) // 4, dtype=torch.int32, device=f"cuda:{self.device}")

    def eval_batch(self, cluster_of_query, query_ct_dev, responses_dev, workspace, stream=None):
        """cluster_of_query: host uint32 [nq]; query_ct_dev: torch int32/uint32 [nq,2,L,n] on device;
        responses_dev: torch int32 [words]; workspace: torch tensor from alloc_workspace."""
        ids = np.ascontiguousarray(cluster_of_query, dtype=np.uint32)
        assert query_ct_dev.is_cuda and query_ct_dev.is_contiguous()
        assert query_ct_dev.numel() == ids.size * 2 * self.L * self.n
        _check(lib.wally_eval_batch(self.ctx, ids.size, _u32p(ids), query_ct_dev.data_ptr(),
                                    responses_dev.data_ptr(), responses_dev.numel(), workspace.data_ptr(),
                                    workspace.numel() * 4, _stream(stream)), self.ctx)

    def check_batch(self, workspace, stream=None):
        _check(lib.wally_check_batch(self.ctx, workspace.data_ptr(), _stream(stream)), self.ctx)

    def fetch_responses(self, responses_dev, out_host: np.ndarray | None = None, stream=None) -> np.ndarray:
        words = responses_dev.numel()
        assert responses_dev.is_cuda and responses_dev.is_contiguous() and responses_dev.element_size() == 4
        if out_host is None:
            out_host = np.empty(words, dtype=np.uint32)
        _check_host_words(out_host, words, "out_host")
        _check(lib.wally_fetch_responses(self.ctx, responses_dev.data_ptr(), words, out_host.ctypes.data,
                                         _stream(stream)), self.ctx)
        return out_host

    def host_workspace_bytes(self, sub_batch: int) -> int:
        b = ctypes.c_size_t()
        _check(lib.wally_host_workspace_bytes(self.ctx, sub_batch, ctypes.byref(b)), self.ctx)
        return b.value

    def eval_batch_host(self, cluster_of_query, query_ct_host, responses_host, sub_batch, workspace, stream=None):
        """query_ct_host / responses_host: host buffers (numpy uint32 or pinned torch CPU tensors)."""
        ids = np.ascontiguousarray(cluster_of_query, dtype=np.uint32)
        qptr = _check_host_words(query_ct_host, ids.size * 2 * self.L * self.n, "query_ct_host", exact=True)
        rwords = responses_host.numel() if hasattr(responses_host, "numel") else responses_host.size
        rptr = _check_host_words(responses_host, rwords, "responses_host")
        assert workspace.is_cuda and workspace.numel() * workspace.element_size() >= self.host_workspace_bytes(sub_batch)
        _check(lib.wally_eval_batch_host(self.ctx, ids.size, _u32p(ids), qptr, rptr, rwords, sub_batch,
                                         workspace.data_ptr(), workspace.numel() * 4, _stream(stream)), self.ctx)

    def route_queries(self, cluster_of_query) -> np.ndarray:
        ids = np.ascontiguousarray(cluster_of_query, dtype=np.uint32)
        dest = np.zeros(ids.size, dtype=np.int32)
        _check(lib.wally_route_queries(self.ctx, ids.size, _u32p(ids),
                                       dest.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), self.ctx)
        return dest

    def pack_queries(self, index_dev, query_ct_dev, out_dev, stream=None):
        """out_dev[i] = query_ct_dev[index_dev[i]] (device rows of 2*L*n uint32)."""
        count = index_dev.numel()
        assert out_dev.numel() >= count * 2 * self.L * self.n
        _check(lib.wally_pack_queries(self.ctx, count, index_dev.data_ptr(), query_ct_dev.data_ptr(),
                                      out_dev.data_ptr(), _stream(stream)), self.ctx)

    # ---- multi-GPU data plane (NCCL inside the C ABI) ----
    def comm_init(self, rank: int, world: int, unique_id: bytes):
        """Join the NCCL communicator `unique_id` (wally_comm_unique_id on one rank) as rank of world."""
        assert len(unique_id) == WALLY_COMM_ID_BYTES
        buf = (ctypes.c_uint8 * WALLY_COMM_ID_BYTES).from_buffer_copy(unique_id)
        _check(lib.wally_comm_init(self.ctx, rank, world, buf), self.ctx)
        self.comm_rank, self.comm_world = rank, world

    def comm_check(self):
        _check(lib.wally_comm_check(self.ctx), self.ctx)

    def scatter_queries(self, src: int, counts, order_dev=None, query_ct_dev=None, pack_dev=None, share_dev=None,
                        stream=None):
        """Query scatter over NCCL (include/wally.h): counts uint32 [world] on every rank; on src the
        route order (device uint32/int32 [nq]), the batch [nq][2][L][n] and a pack buffer of the same
        shape; share_dev [counts[rank]][2][L][n] receives this rank's queries."""
        counts = np.ascontiguousarray(counts, dtype=np.uint32)
        assert counts.size == self.comm_world
        row = 2 * self.L * self.n
        nq = int(counts.sum())
        mine = int(counts[self.comm_rank])
        if share_dev is not None:
            assert share_dev.is_cuda and share_dev.is_contiguous() and share_dev.numel() >= mine * row
        if self.comm_rank == src and nq:
            for t, words in ((order_dev, nq), (query_ct_dev, nq * row), (pack_dev, nq * row)):
                assert t is not None and t.is_cuda and t.is_contiguous() and t.element_size() == 4
                assert t.numel() >= words
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        _check(lib.wally_scatter_queries(self.ctx, src, _u32p(counts), ptr(order_dev), ptr(query_ct_dev),
                                         ptr(pack_dev), ptr(share_dev), _stream(stream)), self.ctx)

    def gather_responses(self, dst: int, resp_words, resp_dev, gathered_dev=None, stream=None):
        """Response gather over NCCL: resp_words uint64 [world] on every rank; gathered_dev on dst only."""
        words = np.ascontiguousarray(resp_words, dtype=np.uint64)
        assert words.size == self.comm_world
        if int(words[self.comm_rank]):
            assert resp_dev.is_cuda and resp_dev.numel() >= int(words[self.comm_rank])
        if self.comm_rank == dst and int(words.sum()):
            assert gathered_dev is not None and gathered_dev.is_cuda and gathered_dev.numel() >= int(words.sum())
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        _check(lib.wally_gather_responses(self.ctx, dst, words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                          ptr(resp_dev), ptr(gathered_dev), _stream(stream)), self.ctx)

    def ntt_forward(self, x_dev, out_dev, count: int, stream=None):
        _check(lib.wally_ntt_forward(self.ctx, x_dev.data_ptr(), out_dev.data_ptr(), count, _stream(stream)),
               self.ctx)

    def ntt_inverse(self, x_dev, out_dev, count: int, stream=None):
        _check(lib.wally_ntt_inverse(self.ctx, x_dev.data_ptr(), out_dev.data_ptr(), count, _stream(stream)),
               self.ctx)

    def modmuls_per_pair(self) -> int:
        """Algorithmic modmuls per (query, plaintext) pair of the kernel this context runs."""
        m = ctypes.c_uint64()
        _check(lib.wally_modmuls_per_pair(self.ctx, ctypes.byref(m)), self.ctx)
        return m.value

    def kernel_launches(self) -> int:
        return int(lib.wally_kernel_launches(self.ctx))

    def enable_stage_timing(self, on: bool = True):
        _check(lib.wally_enable_stage_timing(self.ctx, int(on)), self.ctx)

    def stage_times(self):
        """(ms_batcher, ms_forward_ntt, ms_fused, batches) summed since the last call."""
        ms = (ctypes.c_double * 3)()
        nb = ctypes.c_uint64()
        _check(lib.wally_stage_times(self.ctx, ms, ctypes.byref(nb)), self.ctx)
        return ms[0], ms[1], ms[2], nb.value

"""Thin Python binding of include/wally_simd.h: the paper's SIMD formulation
(diagonal packing + baby-step giant-step rotations with hybrid key
switching).  Argument marshalling only; every step runs
in the CUDA kernels of csrc/simd.cu.  No CPU fallback."""
from __future__ import annotations

import ctypes

import numpy as np

from .wally import WALLY_MAX_LIMBS, WallyError, _stream, lib

EXPORTED = ["wally_simd_default_moduli", "wally_simd_create", "wally_simd_destroy", "wally_simd_last_error", "wally_simd_get_info",
            "wally_simd_load_clusters", "wally_simd_blocks", "wally_simd_eval_batch", "wally_simd_eval_batch_host",
            "wally_simd_modmuls_per_query", "wally_simd_launch_count", "wally_simd_set_chain_threshold",
            "wally_simd_enable_stage_timing", "wally_simd_stage_times", "wally_simd_stage_work"]

# stages of wally_simd_stage_times / wally_simd_stage_work (include/wally_simd.h)
STAGES = ["ntt", "baby_steps", "inner_products", "giant_steps", "switch"]


class wally_simd_params(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("num_limbs", ctypes.c_uint32), ("t", ctypes.c_uint32),
                ("d", ctypes.c_uint32), ("baby", ctypes.c_uint32),
                ("moduli", ctypes.c_uint32 * (WALLY_MAX_LIMBS + 1))]


class wally_simd_info(ctypes.Structure):
    _fields_ = [("row_slices", ctypes.c_uint32), ("block_entries", ctypes.c_uint32), ("baby", ctypes.c_uint32),
                ("giant", ctypes.c_uint32), ("galois", ctypes.c_uint32 * 2), ("key_words", ctypes.c_uint64)]


def _sig():
    vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
    P = ctypes.POINTER
    sig = {
        "wally_simd_default_moduli": ([u32, u32, P(u32)], ctypes.c_int),
        "wally_simd_create": ([P(wally_simd_params), ctypes.c_int, P(vp)], ctypes.c_int),
        "wally_simd_destroy": ([vp], None),
        "wally_simd_last_error": ([vp], ctypes.c_char_p),
        "wally_simd_get_info": ([vp, P(wally_simd_info)], ctypes.c_int),
        "wally_simd_load_clusters": ([vp, u32, P(u32), P(ctypes.c_int8), vp], ctypes.c_int),
        "wally_simd_blocks": ([vp, u32], u32),
        "wally_simd_eval_batch": ([vp, u32, P(u32), vp, vp, vp, u64, P(u64), vp], ctypes.c_int),
        "wally_simd_eval_batch_host": ([vp, u32, P(u32), vp, vp, vp, u64, P(u64), u32, vp], ctypes.c_int),
        "wally_simd_modmuls_per_query": ([vp, u32], u64),
        "wally_simd_launch_count": ([vp], u64),
        "wally_simd_set_chain_threshold": ([vp, u32], ctypes.c_int),
        "wally_simd_enable_stage_timing": ([vp, ctypes.c_int], ctypes.c_int),
        "wally_simd_stage_times": ([vp, P(ctypes.c_double), P(u64)], ctypes.c_int),
        "wally_simd_stage_work": ([vp, u32, P(u32), P(u64), P(u64)], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res


_sig()


def _check(rc: int, ctx=None):
    if rc != 0:
        msg = lib.wally_simd_last_error(ctx)
        raise WallyError(rc, msg.decode() if msg else "")


def simd_moduli(n: int, num_limbs: int) -> list[int]:
    """Reading S25: the L ciphertext limbs are the L largest NTT-friendly
    primes below 2^30 (as in the coefficient path), the special prime P the
    next one below them.  Returns [q_0 < ... < q_{L-1}, P]."""
    out = np.zeros(num_limbs + 1, dtype=np.uint32)
    _check(lib.wally_simd_default_moduli(n, num_limbs, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    return [int(x) for x in out]


class SimdServer:
    """ServerInit + ServerComputation of the SIMD formulation on one device."""

    def __init__(self, n: int, num_limbs: int, d: int, t: int = 65537, baby: int = 0, moduli=None,
                 device: int = 0):
        self.n, self.L, self.d, self.t = n, num_limbs, d, t
        self.moduli = list(moduli) if moduli is not None else simd_moduli(n, num_limbs)
        p = wally_simd_params(n=n, num_limbs=num_limbs, t=t, d=d, baby=baby)
        for i, q in enumerate(self.moduli):
            p.moduli[i] = q
        h = ctypes.c_void_p()
        _check(lib.wally_simd_create(ctypes.byref(p), device, ctypes.byref(h)))
        self.ctx = h
        info = wally_simd_info()
        _check(lib.wally_simd_get_info(self.ctx, ctypes.byref(info)), self.ctx)
        self.row_slices = info.row_slices
        self.block_entries = info.block_entries
        self.baby, self.giant = info.baby, info.giant
        self.galois = (info.galois[0], info.galois[1])
        self.key_words = info.key_words
        self.device = device

    def close(self):
        if getattr(self, "ctx", None):
            lib.wally_simd_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_clusters(self, clusters, stream=None):
        """clusters: list of int8 [S_c][d] arrays."""
        sizes = np.array([c.shape[0] for c in clusters], dtype=np.uint32)
        ent = np.ascontiguousarray(np.concatenate([np.asarray(c, np.int8).reshape(-1, self.d) for c in clusters])
                                   if len(clusters) else np.zeros((0, self.d), np.int8))
        _check(lib.wally_simd_load_clusters(self.ctx, sizes.size, sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                            ent.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)), _stream(stream)),
               self.ctx)
        self.sizes = sizes

    def blocks(self, cluster: int) -> int:
        return int(lib.wally_simd_blocks(self.ctx, cluster))

    def response_words(self, ids) -> int:
        return int(sum(self.blocks(int(c)) for c in ids)) * 2 * self.n

    def eval_batch(self, ids, cts_dev, keys_dev, resp_dev, stream=None) -> np.ndarray:
        """ids: host uint32 [nq]; cts_dev [nq][2][L][n], keys_dev [nq][2][2][L][L+1][n] (device, coefficient
        form); resp_dev: device uint32/int32 with >= response_words(ids) words.  Returns the host offsets
        [nq+1] of each query's responses (words)."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        self._check_buffers(ids, cts_dev, keys_dev, resp_dev, cuda=True)
        off = np.zeros(ids.size + 1, dtype=np.uint64)
        _check(lib.wally_simd_eval_batch(self.ctx, ids.size, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                         cts_dev.data_ptr(), keys_dev.data_ptr(), resp_dev.data_ptr(),
                                         resp_dev.numel(), off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                         _stream(stream)), self.ctx)
        return off

    def eval_batch_host(self, ids, cts_host, keys_host, resp_host, sub_batch: int = 1024, stream=None) -> np.ndarray:
        """The same from host buffers (torch CPU tensors, pinned for overlap); sub-batches are pipelined
        through device staging.  Returns the response offsets [nq+1] (words)."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        self._check_buffers(ids, cts_host, keys_host, resp_host, cuda=False)
        off = np.zeros(ids.size + 1, dtype=np.uint64)
        _check(lib.wally_simd_eval_batch_host(self.ctx, ids.size, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                              cts_host.data_ptr(), keys_host.data_ptr(), resp_host.data_ptr(),
                                              resp_host.numel(), off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                              sub_batch, _stream(stream)), self.ctx)
        return off

    def _check_buffers(self, ids, cts, keys, resp, cuda: bool):
        """The C side reads nq*2*L*n ciphertext words and nq*key_words key
        words and writes response_words(ids) words: check the tensors hold
        exactly / at least that many contiguous 32-bit words on the right side."""
        for name, t, words, exact in (("cts", cts, ids.size * 2 * self.L * self.n, True),
                                      ("keys", keys, ids.size * self.key_words, True),
                                      ("resp", resp, self.response_words(ids), False)):
            assert t.is_cuda == cuda, f"{name} must be {'device' if cuda else 'host'} memory"
            assert t.is_contiguous() and t.element_size() == 4, f"{name} must be contiguous 32-bit"
            assert (t.numel() == words) if exact else (t.numel() >= words), f"{name}: {t.numel()} words, need {words}"

    def modmuls_per_query(self, blocks: int) -> int:
        return int(lib.wally_simd_modmuls_per_query(self.ctx, blocks))

    def set_chain_threshold(self, min_queries: int):
        """0: always the fused rotation chain; 2**32-1: never (see include/wally_simd.h)."""
        _check(lib.wally_simd_set_chain_threshold(self.ctx, min_queries), self.ctx)

    def launch_count(self) -> int:
        return int(lib.wally_simd_launch_count(self.ctx))

    def enable_stage_timing(self, on: bool = True):
        _check(lib.wally_simd_enable_stage_timing(self.ctx, int(on)), self.ctx)

    def stage_times(self):
        """(ms per stage summed since the last call, chunks summed); STAGES names the stages."""
        ms = (ctypes.c_double * len(STAGES))()
        chunks = ctypes.c_uint64(0)
        _check(lib.wally_simd_stage_times(self.ctx, ms, ctypes.byref(chunks)), self.ctx)
        return [float(x) for x in ms], int(chunks.value)

    def stage_work(self, ids):
        """Algorithmic (modmuls, HBM bytes) per stage for a batch with cluster ids `ids`."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        mm = (ctypes.c_uint64 * len(STAGES))()
        by = (ctypes.c_uint64 * len(STAGES))()
        _check(lib.wally_simd_stage_work(self.ctx, ids.size, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                         mm, by), self.ctx)
        return [int(x) for x in mm], [int(x) for x in by]

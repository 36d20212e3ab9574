"""ctypes wrapper for oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Every function here marshals numpy arrays into the plain-C oracle
(`oracle/wally_oracle.c`); see that file for the paper citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "wally_oracle.c"), os.path.join(_HERE, "wally_simd_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(x) for x in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i8p = ctypes.POINTER(ctypes.c_int8)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        c_u32 = ctypes.c_uint32
        L.or_is_prime.argtypes = [ctypes.c_uint64]
        L.or_is_prime.restype = ctypes.c_int
        L.or_find_primes.argtypes = [c_u32, c_u32, u32p]
        L.or_find_primes.restype = ctypes.c_int
        L.or_min_root_2n.argtypes = [c_u32, c_u32]
        L.or_min_root_2n.restype = c_u32
        L.or_ntt_forward.argtypes = [u64p, c_u32, c_u32]
        L.or_ntt_inverse.argtypes = [u64p, c_u32, c_u32]
        L.or_polymul_ntt.argtypes = [u32p, u32p, u32p, c_u32, c_u32]
        L.or_polymul_schoolbook.argtypes = [u32p, u32p, u32p, c_u32, c_u32]
        L.or_crt_u128.argtypes = [u32p, u32p, c_u32, u64p, u64p]
        L.or_modswitch_coeff.argtypes = [u32p, u32p, c_u32]
        L.or_modswitch_coeff.restype = c_u32
        L.or_encode_plaintext.argtypes = [i8p, c_u32, c_u32, c_u32, i32p]
        L.or_encode_plaintext.restype = ctypes.c_int
        L.or_server_pair.argtypes = [c_u32, c_u32, u32p, u32p, i32p, u32p]
        L.or_server_pairs.argtypes = [c_u32, c_u32, u32p, u32p, i32p, ctypes.c_uint64, u32p, u32p, u32p,
                                      ctypes.c_int]
        L.or_server_pairs.restype = ctypes.c_int
        L.or_encrypt.argtypes = [c_u32, c_u32, u32p, c_u32, i32p, i8p, u32p, i32p, u32p]
        L.or_phase_q0.argtypes = [c_u32, c_u32, u32p, i8p, u32p]
        L.or_drop_lsb.argtypes = [u32p, c_u32, c_u32, u32p]
        L.or_plain_crt_signed.argtypes = [c_u32, c_u32, c_u32, c_u32]
        L.or_plain_crt_signed.restype = ctypes.c_int64
        L.or_decrypt_q0.argtypes = [c_u32, c_u32, c_u32, u32p, i8p, u32p]
        L.or_noise_budget_q0.argtypes = [c_u32, c_u32, c_u32, u32p, i8p]
        L.or_noise_budget_q0.restype = ctypes.c_double
        L.or_noise_budget_Q.argtypes = [c_u32, c_u32, u32p, c_u32, u32p, i8p]
        L.or_noise_budget_Q.restype = ctypes.c_double
        # SIMD formulation (wally_simd_oracle.c)
        L.or_simd_slot_exponent.argtypes = [c_u32, c_u32]
        L.or_simd_slot_exponent.restype = c_u32
        L.or_simd_row_slices.argtypes = [c_u32, c_u32]
        L.or_simd_row_slices.restype = c_u32
        L.or_simd_encode.argtypes = [c_u32, c_u32, u32p, u32p]
        L.or_simd_decode.argtypes = [c_u32, c_u32, u32p, u32p]
        L.or_automorph.argtypes = [c_u32, c_u32, u32p, c_u32, u32p]
        L.or_simd_keygen.argtypes = [c_u32, c_u32, u32p, i8p, c_u32, u32p, i32p, u32p]
        L.or_keyswitch.argtypes = [c_u32, c_u32, u32p, u32p, u32p, u32p]
        L.or_rotate.argtypes = [c_u32, c_u32, u32p, u32p, c_u32, u32p, u32p]
        L.or_simd_diagonal_slots.argtypes = [c_u32, c_u32, c_u32, c_u32, i8p, c_u32, u32p]
        L.or_simd_query_slots.argtypes = [c_u32, c_u32, c_u32, i32p, u32p]
        L.or_simd_server.argtypes = [c_u32, c_u32, u32p, c_u32, c_u32, c_u32, u32p, u32p, u32p, u32p, u32p]
        L.or_simd_server.restype = ctypes.c_int
        L.or_simd_response.argtypes = [c_u32, c_u32, u32p, u32p, u32p]
        _lib = L
    return _lib


def _p(arr: np.ndarray, ctype):
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(ctypes.POINTER(ctype))


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def find_primes(n: int, L: int) -> list[int]:
    out = np.zeros(L, dtype=np.uint32)
    if lib().or_find_primes(n, L, _p(out, ctypes.c_uint32)) != 0:
        raise ValueError("no primes found")
    return [int(x) for x in out]


def is_prime(x: int) -> bool:
    return bool(lib().or_is_prime(x))


def min_root_2n(q: int, n: int) -> int:
    return int(lib().or_min_root_2n(q, n))


def ntt_forward(a, q: int) -> np.ndarray:
    x = np.ascontiguousarray(a, dtype=np.uint64).copy()
    lib().or_ntt_forward(_p(x, ctypes.c_uint64), x.size, q)
    return x


def ntt_inverse(a, q: int) -> np.ndarray:
    x = np.ascontiguousarray(a, dtype=np.uint64).copy()
    lib().or_ntt_inverse(_p(x, ctypes.c_uint64), x.size, q)
    return x


def polymul_ntt(a, b, q: int) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    r = np.zeros_like(a)
    lib().or_polymul_ntt(_p(a, ctypes.c_uint32), _p(b, ctypes.c_uint32), _p(r, ctypes.c_uint32), a.size, q)
    return r


def polymul_schoolbook(a, b, q: int) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    r = np.zeros_like(a)
    lib().or_polymul_schoolbook(_p(a, ctypes.c_uint32), _p(b, ctypes.c_uint32), _p(r, ctypes.c_uint32), a.size,
                                q)
    return r


def crt(residues, moduli) -> int:
    r, m = _u32(residues), _u32(moduli)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    lib().or_crt_u128(_p(r, ctypes.c_uint32), _p(m, ctypes.c_uint32), m.size, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value | (hi.value << 64)


def modswitch_coeff(residues, moduli) -> int:
    r, m = _u32(residues), _u32(moduli)
    return int(lib().or_modswitch_coeff(_p(r, ctypes.c_uint32), _p(m, ctypes.c_uint32), m.size))


def encode_plaintext(entries, d: int, n: int) -> np.ndarray:
    e = np.ascontiguousarray(entries, dtype=np.int8).reshape(-1, d)
    out = np.zeros(n, dtype=np.int32)
    if lib().or_encode_plaintext(_p(e, ctypes.c_int8), e.shape[0], d, n, _p(out, ctypes.c_int32)) != 0:
        raise ValueError("too many entries for one plaintext")
    return out


def encode_cluster(entries, d: int, n: int) -> np.ndarray:
    """All plaintexts of one cluster: int32 [ceil(S/E)][n], E = n // d."""
    e = np.ascontiguousarray(entries, dtype=np.int8).reshape(-1, d)
    E = n // d
    P = -(-e.shape[0] // E)
    return np.stack([encode_plaintext(e[k * E:(k + 1) * E], d, n) for k in range(P)])


def server_pair(moduli, ct, pcoef) -> np.ndarray:
    m = _u32(moduli)
    ct = _u32(ct)
    L = m.size
    n = ct.size // (2 * L)
    pc = np.ascontiguousarray(pcoef, dtype=np.int32)
    out = np.zeros((2, n), dtype=np.uint32)
    lib().or_server_pair(n, L, _p(m, ctypes.c_uint32), _p(ct, ctypes.c_uint32), _p(pc, ctypes.c_int32),
                         _p(out, ctypes.c_uint32))
    return out


def server_pairs(moduli, cts, pcoefs, pair_q, pair_pt, threads: int = 0):
    """Responses for a list of (query, plaintext) pairs.  Returns (out, threads_used)."""
    m = _u32(moduli)
    cts = _u32(cts)
    L = m.size
    pc = np.ascontiguousarray(pcoefs, dtype=np.int32)
    n = pc.shape[-1]
    pq, pp = _u32(pair_q), _u32(pair_pt)
    out = np.zeros((pq.size, 2, n), dtype=np.uint32)
    used = lib().or_server_pairs(n, L, _p(m, ctypes.c_uint32), _p(cts, ctypes.c_uint32), _p(pc, ctypes.c_int32),
                                 pq.size, _p(pq, ctypes.c_uint32), _p(pp, ctypes.c_uint32),
                                 _p(out, ctypes.c_uint32), int(threads))
    return out, used


def encrypt(moduli, t: int, msg, s, a, e) -> np.ndarray:
    m = _u32(moduli)
    L = m.size
    msg = np.ascontiguousarray(msg, dtype=np.int32)
    n = msg.size
    s = np.ascontiguousarray(s, dtype=np.int8)
    a = _u32(a).reshape(L, n)
    e = np.ascontiguousarray(e, dtype=np.int32)
    ct = np.zeros((2, L, n), dtype=np.uint32)
    lib().or_encrypt(n, L, _p(m, ctypes.c_uint32), t, _p(msg, ctypes.c_int32), _p(s, ctypes.c_int8),
                     _p(a, ctypes.c_uint32), _p(e, ctypes.c_int32), _p(ct, ctypes.c_uint32))
    return ct


def decrypt_q0(q0: int, t: int, resp, s) -> np.ndarray:
    r = _u32(resp)
    n = r.size // 2
    s = np.ascontiguousarray(s, dtype=np.int8)
    m = np.zeros(n, dtype=np.uint32)
    lib().or_decrypt_q0(n, q0, t, _p(r, ctypes.c_uint32), _p(s, ctypes.c_int8), _p(m, ctypes.c_uint32))
    return m


def phase_q0(q0: int, resp, s) -> np.ndarray:
    r = _u32(resp)
    n = r.size // 2
    s = np.ascontiguousarray(s, dtype=np.int8)
    v = np.zeros(n, dtype=np.uint32)
    lib().or_phase_q0(n, q0, _p(r, ctypes.c_uint32), _p(s, ctypes.c_int8), _p(v, ctypes.c_uint32))
    return v


def plain_crt_signed(m0: int, m1: int, t0: int, t1: int) -> int:
    """Centered CRT combination of a result decrypted mod t0 and mod t1 (plaintext CRT)."""
    return int(lib().or_plain_crt_signed(int(m0), int(m1), t0, t1))


def drop_lsb(c, b: int) -> np.ndarray:
    """Rounded high part floor((c + 2^(b-1)) / 2^b) of canonical residues (reading S20)."""
    x = np.ascontiguousarray(c, dtype=np.uint32).ravel()
    out = np.zeros_like(x)
    lib().or_drop_lsb(_p(x, ctypes.c_uint32), x.size, b, _p(out, ctypes.c_uint32))
    return out


def noise_budget_q0(q0: int, t: int, resp, s) -> float:
    r = _u32(resp)
    s = np.ascontiguousarray(s, dtype=np.int8)
    return float(lib().or_noise_budget_q0(r.size // 2, q0, t, _p(r, ctypes.c_uint32), _p(s, ctypes.c_int8)))


def noise_budget_Q(moduli, t: int, ct, s) -> float:
    m = _u32(moduli)
    c = _u32(ct)
    s = np.ascontiguousarray(s, dtype=np.int8)
    n = s.size
    return float(lib().or_noise_budget_Q(n, m.size, _p(m, ctypes.c_uint32), t, _p(c, ctypes.c_uint32),
                                         _p(s, ctypes.c_int8)))


def result_slots(n: int, d: int, count: int) -> np.ndarray:
    """Coefficient positions j*d + d - 1 holding the dot products (reading S1)."""
    return np.arange(count) * d + d - 1


# ---------------------------------------------------------------------------
# SIMD formulation (oracle/wally_simd_oracle.c)
# ---------------------------------------------------------------------------

def simd_slot_exponent(n: int, s: int) -> int:
    return int(lib().or_simd_slot_exponent(n, s))


def simd_row_slices(n: int, d: int) -> int:
    return int(lib().or_simd_row_slices(n, d))


def simd_encode(slots, t: int) -> np.ndarray:
    x = _u32(slots)
    out = np.zeros_like(x)
    lib().or_simd_encode(x.size, t, _p(x, ctypes.c_uint32), _p(out, ctypes.c_uint32))
    return out


def simd_decode(coef, t: int) -> np.ndarray:
    x = _u32(coef)
    out = np.zeros_like(x)
    lib().or_simd_decode(x.size, t, _p(x, ctypes.c_uint32), _p(out, ctypes.c_uint32))
    return out


def automorph(a, q: int, k: int) -> np.ndarray:
    x = _u32(a)
    out = np.zeros_like(x)
    lib().or_automorph(x.size, q, _p(x, ctypes.c_uint32), k, _p(out, ctypes.c_uint32))
    return out


def simd_keygen(mods, s, k: int, a, e) -> np.ndarray:
    """Rotation key for sigma_k: uint32 [2][L][L+1][n] (mods = L ciphertext moduli + special prime)."""
    m = _u32(mods)
    L = m.size - 1
    s = np.ascontiguousarray(s, dtype=np.int8)
    n = s.size
    a = _u32(a).reshape(L, L + 1, n)
    e = np.ascontiguousarray(e, dtype=np.int32).reshape(L, n)
    key = np.zeros((2, L, L + 1, n), dtype=np.uint32)
    lib().or_simd_keygen(n, L, _p(m, ctypes.c_uint32), _p(s, ctypes.c_int8), k, _p(a, ctypes.c_uint32),
                         _p(e, ctypes.c_int32), _p(key, ctypes.c_uint32))
    return key


def keyswitch(mods, c, key) -> np.ndarray:
    m = _u32(mods)
    L = m.size - 1
    c = _u32(c)
    n = c.size // L
    key = _u32(key)
    out = np.zeros((2, L, n), dtype=np.uint32)
    lib().or_keyswitch(n, L, _p(m, ctypes.c_uint32), _p(c, ctypes.c_uint32), _p(key, ctypes.c_uint32),
                       _p(out, ctypes.c_uint32))
    return out


def rotate(mods, ct, k: int, key) -> np.ndarray:
    m = _u32(mods)
    L = m.size - 1
    ct = _u32(ct)
    n = ct.size // (2 * L)
    key = _u32(key)
    out = np.zeros((2, L, n), dtype=np.uint32)
    lib().or_rotate(n, L, _p(m, ctypes.c_uint32), _p(ct, ctypes.c_uint32), k, _p(key, ctypes.c_uint32),
                    _p(out, ctypes.c_uint32))
    return out


def simd_diagonal_slots(entries, n: int, t: int, d: int, g: int) -> np.ndarray:
    e = np.ascontiguousarray(entries, dtype=np.int8).reshape(-1, d)
    out = np.zeros((d, n), dtype=np.uint32)
    lib().or_simd_diagonal_slots(n, t, d, g, _p(e, ctypes.c_int8), e.shape[0], _p(out, ctypes.c_uint32))
    return out


def simd_query_slots(q, n: int, t: int) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int32)
    out = np.zeros(n, dtype=np.uint32)
    lib().or_simd_query_slots(n, t, q.size, _p(q, ctypes.c_int32), _p(out, ctypes.c_uint32))
    return out


def simd_server(mods, t: int, d: int, g: int, ct, key1, keyg, pt) -> np.ndarray:
    """BSGS server computation; returns the result ciphertext [2][L][n] over Q."""
    m = _u32(mods)
    L = m.size - 1
    ct = _u32(ct)
    n = ct.size // (2 * L)
    key1, keyg, pt = _u32(key1), _u32(keyg), _u32(pt)
    assert pt.size == d * n
    out = np.zeros((2, L, n), dtype=np.uint32)
    rc = lib().or_simd_server(n, L, _p(m, ctypes.c_uint32), t, d, g, _p(ct, ctypes.c_uint32),
                              _p(key1, ctypes.c_uint32), _p(keyg, ctypes.c_uint32), _p(pt, ctypes.c_uint32),
                              _p(out, ctypes.c_uint32))
    if rc != 0:
        raise ValueError("bad SIMD server arguments")
    return out


def simd_response(mods, res) -> np.ndarray:
    """Switch a result ciphertext over Q (mods = the L ciphertext moduli) to q_0: [2][n]."""
    m = _u32(mods)
    L = m.size
    r = _u32(res)
    n = r.size // (2 * L)
    out = np.zeros((2, n), dtype=np.uint32)
    lib().or_simd_response(n, L, _p(m, ctypes.c_uint32), _p(r, ctypes.c_uint32), _p(out, ctypes.c_uint32))
    return out

"""Pure-Python big-integer reference for tiny rings -- TEST INFRASTRUCTURE ONLY.

An independent second statement of the same mathematics as the C oracle,
written without RNS and without NTTs: every polynomial lives in
Z_Q[X]/(X^n+1) as Python ints and products are the O(n^2) schoolbook
negacyclic convolution.  Used only to pin the C oracle on small n.

Citations: PAPER.md P:L244-256 (ring, ciphertext, decryption), P:L1003 and
P:L1318-1324 (modulus switching to q_0), P:L1310-1313 (CRT).
"""
from __future__ import annotations


def negacyclic_mul(a, b, mod):
    """Schoolbook product in Z_mod[X]/(X^n+1): X^n = -1."""
    n = len(a)
    r = [0] * n
    for i, ai in enumerate(a):
        if ai == 0:
            continue
        for j, bj in enumerate(b):
            k = i + j
            if k < n:
                r[k] += ai * bj
            else:
                r[k - n] -= ai * bj
    return [x % mod for x in r]


def crt_sum(residues, moduli):
    """CRT by the textbook sum formula  c = sum r_i * M_i * (M_i^{-1} mod q_i) mod Q."""
    Q = 1
    for q in moduli:
        Q *= int(q)
    c = 0
    for r, q in zip(residues, moduli):
        r, q = int(r), int(q)
        Mi = Q // q
        c += r * Mi * pow(Mi, -1, q)
    return c % Q


def product(moduli):
    Q = 1
    for q in moduli:
        Q *= int(q)
    return Q


def encode_plaintext(entries, d, n):
    """p(X) = sum_j sum_i e_j[i] X^{j d + d - 1 - i} (reading S1)."""
    p = [0] * n
    for j, e in enumerate(entries):
        for i in range(d):
            p[j * d + d - 1 - i] = int(e[i])
    return p


def encrypt(moduli, t, msg, s, a_res, e):
    """c1 = a, c0 = -a s + e + floor(Q/t) m  over Z_Q (reading S2).

    a_res: per-limb residues [L][n]; lifted to Z_Q by crt_sum."""
    Q = product(moduli)
    n = len(msg)
    a = [crt_sum([a_res[l][i] for l in range(len(moduli))], moduli) for i in range(n)]
    delta = Q // t
    as_ = negacyclic_mul(a, [int(x) for x in s], Q)
    c0 = [(-as_[i] + int(e[i]) + delta * (int(msg[i]) % t)) % Q for i in range(n)]
    return c0, a


def server_pair(moduli, c0, c1, pcoef):
    """r = c * p in R_Q, then c' = round(c q_0 / Q) mod q_0 (exact integers)."""
    Q = product(moduli)
    q0 = int(moduli[0])
    out = []
    for c in (c0, c1):
        r = negacyclic_mul(c, [int(x) for x in pcoef], Q)
        out.append([((2 * x * q0 + Q) // (2 * Q)) % q0 for x in r])
    return out


def decrypt_q0(q0, t, c0, c1, s):
    v = negacyclic_mul(c1, [int(x) for x in s], q0)
    v = [(v[i] + c0[i]) % q0 for i in range(len(c0))]
    return [((2 * t * x + q0) // (2 * q0)) % t for x in v]


def to_residues(poly, moduli):
    return [[x % q for x in poly] for q in moduli]

"""Pins of the SIMD-formulation oracle (oracle/wally_simd_oracle.c; SURVEY.md
§8(f)-3) against what the mathematics fixes, independently of the oracle's
own formulas:

  * slots      the encoding is a ring isomorphism R_t -> Z_t^n (round trip,
               multiplicative against a schoolbook product), the exponents are
               the odd residues mod 2n
  * rotations  X -> X^5 rotates both slot rows left by one, X -> X^{-1} swaps
               the rows; sigma_k is a ring homomorphism and sigma_k o sigma_l =
               sigma_{kl}
  * key switch a rotated ciphertext decrypts to the rotated message with a
               positive noise budget
  * BSGS       the decrypted response holds exactly the plain dot products of
               the query with every packed embedding (closed form), for d | n/2
               and d not dividing n/2, g | d and g not dividing d, full and
               ragged blocks
"""
import numpy as np
import pytest

from oracle import capi

T = 65537


def _rng(seed):
    return np.random.default_rng(seed)


def test_slot_exponents_are_the_odd_residues():
    for n in (8, 64, 4096):
        ex = [capi.simd_slot_exponent(n, s) for s in range(n)]
        assert sorted(ex) == list(range(1, 2 * n, 2))
        assert ex[0] == 1 and ex[n // 2] == 2 * n - 1 and ex[1] == 5 % (2 * n)


@pytest.mark.parametrize("n", [8, 32, 256])
def test_encoding_is_a_ring_isomorphism(n):
    rng = _rng(n)
    a = rng.integers(0, T, size=n).astype(np.uint32)
    b = rng.integers(0, T, size=n).astype(np.uint32)
    ca, cb = capi.simd_encode(a, T), capi.simd_encode(b, T)
    assert np.array_equal(capi.simd_decode(ca, T), a)
    prod = capi.polymul_schoolbook(ca, cb, T)           # negacyclic product mod t, by definition
    assert np.array_equal(capi.simd_decode(prod, T), (a.astype(np.uint64) * b % T).astype(np.uint32))
    # the constant polynomial c decodes to c in every slot
    assert np.array_equal(capi.simd_decode(np.r_[7, np.zeros(n - 1)].astype(np.uint32), T), np.full(n, 7))


@pytest.mark.parametrize("n", [16, 128])
def test_rotation_by_x5_and_row_swap(n):
    rng = _rng(n + 1)
    v = rng.integers(0, T, size=n).astype(np.uint32)
    c = capi.simd_encode(v, T)
    rows = v.reshape(2, n // 2)
    r1 = capi.simd_decode(capi.automorph(c, T, 5), T).reshape(2, n // 2)
    assert np.array_equal(r1, np.roll(rows, -1, axis=1))
    k3 = pow(5, 3, 2 * n)
    r3 = capi.simd_decode(capi.automorph(c, T, k3), T).reshape(2, n // 2)
    assert np.array_equal(r3, np.roll(rows, -3, axis=1))
    sw = capi.simd_decode(capi.automorph(c, T, 2 * n - 1), T).reshape(2, n // 2)
    assert np.array_equal(sw, rows[::-1])


@pytest.mark.parametrize("n", [16, 64])
def test_automorphism_is_a_homomorphism(n):
    rng = _rng(3 * n)
    q = capi.find_primes(n, 1)[0]
    a = rng.integers(0, q, size=n).astype(np.uint32)
    b = rng.integers(0, q, size=n).astype(np.uint32)
    for k in (3, 5, 2 * n - 1, pow(5, 7, 2 * n)):
        lhs = capi.automorph(capi.polymul_schoolbook(a, b, q), q, k)
        rhs = capi.polymul_schoolbook(capi.automorph(a, q, k), capi.automorph(b, q, k), q)
        assert np.array_equal(lhs, rhs), k
        assert np.array_equal(capi.automorph(capi.automorph(a, q, k), q, 5), capi.automorph(a, q, (5 * k) % (2 * n)))
    # sigma_1 is the identity; sigma_{2n-1}(X) = X^{2n-1} = -X^{n-1}
    assert np.array_equal(capi.automorph(a, q, 1), a)
    x = np.zeros(n, np.uint32)
    x[1] = 1
    y = capi.automorph(x, q, 2 * n - 1)
    assert y[n - 1] == q - 1 and y.sum() == q - 1


def _keys(n, L, seed):
    """Moduli (L ciphertext limbs + the special prime, reading S25), secret, and a key maker."""
    allp = capi.find_primes(n, L + 1)          # ascending: the smallest is the special prime
    mods = np.array(allp[1:] + allp[:1], dtype=np.uint32)
    rng = _rng(seed)
    s = rng.integers(-1, 2, size=n).astype(np.int8)

    def make(k):
        a = np.stack([np.stack([rng.integers(0, int(q), size=n) for q in mods]) for _ in range(L)]).astype(np.uint32)
        e = np.clip(np.rint(rng.normal(0, 3.2, size=(L, n))), -19, 19).astype(np.int32)
        return capi.simd_keygen(mods, s, k, a, e)
    return mods, s, rng, make


def _encrypt(mods, s, rng, coef):
    L = mods.size - 1
    n = s.size
    a = np.stack([rng.integers(0, int(q), size=n) for q in mods[:L]]).astype(np.uint32)
    e = np.clip(np.rint(rng.normal(0, 3.2, size=n)), -19, 19).astype(np.int32)
    return capi.encrypt(mods[:L], T, coef.astype(np.int32), s, a, e)


def _decrypt_slots(mods, s, res):
    L = mods.size - 1
    resp = capi.simd_response(mods[:L], res)
    m = capi.decrypt_q0(int(mods[0]), T, resp, s)
    return capi.simd_decode(m, T), capi.noise_budget_q0(int(mods[0]), T, resp, s)


@pytest.mark.parametrize("n,L", [(64, 2), (256, 3)])
def test_rotation_keyswitch_decrypts_to_rotated_slots(n, L):
    mods, s, rng, make = _keys(n, L, n + L)
    v = rng.integers(0, T, size=n).astype(np.uint32)
    ct = _encrypt(mods, s, rng, capi.simd_encode(v, T))
    for k, shift in ((5, 1), (pow(5, 4, 2 * n), 4)):
        key = make(k)
        rot = capi.rotate(mods, ct, k, key)
        got, budget = _decrypt_slots(mods, s, rot)
        assert np.array_equal(got.reshape(2, -1), np.roll(v.reshape(2, -1), -shift, axis=1)), k
        assert budget > 3
        assert capi.noise_budget_Q(mods[:L], T, rot, s) > 20
    # a wrong key (for another automorphism) does not decrypt
    bad = capi.rotate(mods, ct, 5, make(pow(5, 2, 2 * n)))
    got, _ = _decrypt_slots(mods, s, bad)
    assert not np.array_equal(got.reshape(2, -1), np.roll(v.reshape(2, -1), -1, axis=1))


def test_row_slices_formula():
    assert capi.simd_row_slices(4096, 128) == 16            # d | n/2: every column used
    assert capi.simd_row_slices(4096, 192) == 9             # 2048 = 10*192 + 128: keep k + i < n/2
    assert capi.simd_row_slices(8192, 512) == 8
    assert capi.simd_row_slices(64, 12) == 1                # 32 = 2*12 + 8
    assert capi.simd_row_slices(64, 33) == 0


# (n, L, d, g, entries): d | n/2 and d not dividing n/2; g | d and not; full and ragged blocks
BSGS = [
    (64, 2, 8, 3, 32),
    (64, 2, 12, 4, 24),
    (128, 3, 16, 4, 100),
    (256, 2, 24, 5, 150),
]


@pytest.mark.parametrize("n,L,d,g,cnt", BSGS)
def test_bsgs_response_decrypts_to_dot_products(n, L, d, g, cnt):
    mods, s, rng, make = _keys(n, L, 7 * n + d)
    R = capi.simd_row_slices(n, d)
    assert cnt <= 2 * R * d
    ent = rng.integers(-15, 16, size=(cnt, d)).astype(np.int8)
    q = rng.integers(-15, 16, size=d).astype(np.int32)
    pt = np.stack([capi.simd_encode(x, T) for x in capi.simd_diagonal_slots(ent, n, T, d, g)])
    ct = _encrypt(mods, s, rng, capi.simd_encode(capi.simd_query_slots(q, n, T), T))
    res = capi.simd_server(mods, T, d, g, ct, make(5), make(pow(5, g, 2 * n)), pt)
    slots, budget = _decrypt_slots(mods, s, res)
    assert budget > 2
    want = (ent.astype(np.int64) @ q.astype(np.int64)) % T
    half = n // 2
    for e in range(cnt):
        sl, col = divmod(e, d)
        r, u = divmod(sl, R)
        assert slots[r * half + u * d + col] == want[e], e


def test_bsgs_equals_naive_diagonal_method():
    """BSGS (pre-rotated diagonals, giant steps by rot_g) and the paper's plain
    diagonal method (rotate the query by one d-1 times, multiply, sum;
    P:L583-593) give ciphertexts that decrypt identically."""
    n, L, d, g = 64, 2, 8, 3
    mods, s, rng, make = _keys(n, L, 99)
    ent = rng.integers(-15, 16, size=(32, d)).astype(np.int8)
    q = rng.integers(-15, 16, size=d).astype(np.int32)
    ct = _encrypt(mods, s, rng, capi.simd_encode(capi.simd_query_slots(q, n, T), T))
    k1 = make(5)
    bsgs_pt = np.stack([capi.simd_encode(x, T) for x in capi.simd_diagonal_slots(ent, n, T, d, g)])
    res = capi.simd_server(mods, T, d, g, ct, k1, make(pow(5, g, 2 * n)), bsgs_pt)
    # naive: g = d baby steps, one giant step (no pre-rotation since j = 0 only)
    naive_pt = np.stack([capi.simd_encode(x, T) for x in capi.simd_diagonal_slots(ent, n, T, d, d)])
    res2 = capi.simd_server(mods, T, d, d, ct, k1, make(pow(5, d, 2 * n)), naive_pt)
    a, _ = _decrypt_slots(mods, s, res)
    b, _ = _decrypt_slots(mods, s, res2)
    R = capi.simd_row_slices(n, d)
    used = [r * (n // 2) + k for r in range(2) for k in range(R * d)]
    assert np.array_equal(a[used], b[used])


def _is_prime_trial(x: int) -> bool:
    if x < 2:
        return False
    f = 2
    while f * f <= x:
        if x % f == 0:
            return False
        f += 1
    return True


def test_special_primes_golden():
    """Reading S25: P is the (L+1)-th largest NTT-friendly prime below 2^30 (golden file), re-derived by
    trial division and by the oracle's own search."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "simd_special_primes.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    for n, L, P in ((int(a), int(b), int(c)) for a, b, c in rows):
        found = []
        q = (2 ** 30 - 2) // (2 * n) * (2 * n) + 1
        while len(found) < L + 1:
            if q < 2 ** 30 and _is_prime_trial(q):
                found.append(q)
            q -= 2 * n
        assert found[L] == P
        assert capi.find_primes(n, L + 1)[0] == P

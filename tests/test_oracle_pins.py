"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Nothing here re-types the oracle's formulas: every expected value comes from
an independent statement (the transform's definition evaluated directly,
the O(n^2) schoolbook product, a big-integer implementation without RNS,
a different mod-switch algorithm, closed forms such as "decryption equals
the plaintext dot product mod t", special cases, brute force).

Paper citations: PAPER.md P:L244-256 (ring, ciphertext, decryption,
budget), P:L1000 / P:L1314-1317 (NTT), P:L1003 / P:L1318-1324 (modulus
switching to q_0), P:L1310-1313 (RNS/CRT).  Readings S1-S19: DESIGN.md.
"""
import math
import os

import numpy as np
import pytest

import synth
from oracle import capi, tiny_ref

pytestmark = pytest.mark.filterwarnings("ignore")

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------
# independent helpers (not the oracle's code)
# --------------------------------------------------------------------------

def mr_is_prime(x: int) -> bool:
    """Deterministic Miller-Rabin for x < 3.4e14 (bases 2,3,5,7,11,13,17)."""
    if x < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17]
    for p in small:
        if x % p == 0:
            return x == p
    d, r = x - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(r - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


def numpy_schoolbook(a, b, q):
    """O(n^2) negacyclic product mod q with numpy rows (independent of the oracle)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    n = a.size
    B = np.concatenate([(np.uint64(q) - b) % np.uint64(q), b])   # B[n + m] = b[m], B[n + m] = -b[m + n] for m < 0
    r = np.zeros(n, dtype=np.uint64)
    for i in range(n):
        if a[i]:
            r = (r + a[i] * B[n - i: 2 * n - i]) % np.uint64(q)
    return r


def load_golden_moduli():
    out = {}
    with open(os.path.join(GOLDEN, "moduli.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            n, L, *qs = line.split()
            out[(int(n), int(L))] = [int(x) for x in qs]
    return out


# --------------------------------------------------------------------------
# o1: parameters
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n,L", [(4096, 2), (4096, 3), (8192, 4), (64, 2), (16, 3)])
def test_primes_are_the_largest_ntt_friendly_30bit(n, L):
    qs = capi.find_primes(n, L)
    assert qs == sorted(qs) and len(set(qs)) == L
    for q in qs:
        assert q < 2 ** 30 and q % (2 * n) == 1 and mr_is_prime(q)
    # completeness: no other prime = 1 mod 2n lies in [q_0, 2^30)
    others = [c for c in range(qs[0], 2 ** 30, 2 * n) if mr_is_prime(c)]
    assert others == qs
    # reading S6: q_{l} < 2 q_0 so one conditional subtract reduces r mod q_i
    assert qs[-1] < 2 * qs[0]


def test_golden_moduli():
    gold = load_golden_moduli()
    for (n, L), qs in gold.items():
        assert capi.find_primes(n, L) == qs


@pytest.mark.parametrize("n", [8, 64, 4096, 8192])
def test_min_primitive_root(n):
    q = capi.find_primes(n, 1)[0]
    psi = capi.min_root_2n(q, n)
    assert pow(psi, n, q) == q - 1          # primitive 2n-th root: psi^n = -1
    assert pow(psi, 2 * n, q) == 1
    # minimality: every primitive 2n-th root is psi^k, k odd; none is smaller
    roots = [pow(psi, k, q) for k in range(1, 2 * n, 2)]
    assert min(roots) == psi
    assert len(set(roots)) == n


# --------------------------------------------------------------------------
# o6: NTT
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
def test_ntt_matches_definition(n):
    """Forward transform = evaluation at the odd powers psi^(2k+1) (negacyclic)."""
    q = capi.find_primes(n, 1)[0]
    psi = capi.min_root_2n(q, n)
    rng = np.random.default_rng(n)
    a = rng.integers(0, q, size=n)
    got = capi.ntt_forward(a, q)
    want = [sum(int(a[j]) * pow(psi, (2 * k + 1) * j, q) for j in range(n)) % q for k in range(n)]
    assert [int(x) for x in got] == want
    back = capi.ntt_inverse(got, q)
    assert np.array_equal(back, a.astype(np.uint64))


@pytest.mark.parametrize("n", [4096, 8192])
def test_ntt_roundtrip_and_trivial_cases(n):
    for q in capi.find_primes(n, 2):
        rng = np.random.default_rng(q)
        a = rng.integers(0, q, size=n).astype(np.uint64)
        assert np.array_equal(capi.ntt_inverse(capi.ntt_forward(a, q), q), a)
        z = np.zeros(n, dtype=np.uint64)
        assert not capi.ntt_forward(z, q).any()
        c = np.zeros(n, dtype=np.uint64)
        c[0] = 12345
        fc = capi.ntt_forward(c, q)
        assert (fc == 12345).all()                 # a constant evaluates to itself everywhere
        assert np.array_equal(capi.ntt_inverse(fc, q), c)


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32, 64])
def test_polymul_equals_schoolbook_small(n):
    if n == 1:
        pytest.skip("n=1 has no negacyclic NTT")
    for q in capi.find_primes(n, 2):
        rng = np.random.default_rng(1000 + n)
        for _ in range(5):
            a = rng.integers(0, q, size=n)
            b = rng.integers(0, q, size=n)
            ref = tiny_ref.negacyclic_mul([int(x) for x in a], [int(x) for x in b], q)
            assert [int(x) for x in capi.polymul_ntt(a, b, q)] == ref
            assert [int(x) for x in capi.polymul_schoolbook(a, b, q)] == ref


@pytest.mark.parametrize("n", [4096, 8192])
def test_polymul_equals_schoolbook_large(n):
    q = capi.find_primes(n, 1)[0]
    rng = np.random.default_rng(n + 7)
    reps = 2 if n == 4096 else 1
    for _ in range(reps):
        a = rng.integers(0, q, size=n)
        b = rng.integers(0, q, size=n)
        assert np.array_equal(capi.polymul_ntt(a, b, q).astype(np.uint64), numpy_schoolbook(a, b, q))


# --------------------------------------------------------------------------
# CRT and o7: modulus switching
# --------------------------------------------------------------------------

@pytest.mark.parametrize("L", [1, 2, 3, 4])
def test_crt_against_sum_formula(L):
    qs = capi.find_primes(8192, L)
    rng = np.random.default_rng(L)
    for _ in range(200):
        r = [int(rng.integers(0, q)) for q in qs]
        assert capi.crt(r, qs) == tiny_ref.crt_sum(r, qs)
    assert capi.crt([0] * L, qs) == 0
    assert capi.crt([1] * L, qs) == 1


def _residues(c, qs):
    return [c % q for q in qs]


def _sequential_drop_last(c, qs):
    """A different algorithm (reading S7): drop q_{L-1}, ..., q_1 one at a time,
    each time rounding to nearest:  c <- floor((c + floor(q_l/2)) / q_l)."""
    for q in reversed(qs[1:]):
        c = (c + q // 2) // q
    return c % qs[0]


@pytest.mark.parametrize("L", [2, 3, 4])
def test_modswitch_special_cases_and_sequential_identity(L):
    qs = capi.find_primes(4096 if L < 4 else 8192, L)
    Q = math.prod(qs)
    P = Q // qs[0]
    q0 = qs[0]
    rng = np.random.default_rng(10 + L)
    # c = k P  ->  k mod q0 (exact division, no rounding)
    for k in [0, 1, 2, q0 - 1, int(rng.integers(0, q0))]:
        assert capi.modswitch_coeff(_residues(k * P, qs), qs) == k % q0
    # c in [0, P/2) -> 0 ; c in (P/2, P) -> 1   (round to nearest, no ties: P odd)
    for c in [0, 1, P // 2]:
        assert capi.modswitch_coeff(_residues(c, qs), qs) == 0
    for c in [P // 2 + 1, P - 1]:
        assert capi.modswitch_coeff(_residues(c, qs), qs) == 1
    # the largest values round up to q0 == 0 mod q0
    assert capi.modswitch_coeff(_residues(Q - 1, qs), qs) == 0
    # random: |c' P - c| <= P/2 and equality with sequential drop-last
    for _ in range(300):
        c = int(rng.integers(0, 2 ** 62)) * int(rng.integers(0, 2 ** 62)) % Q
        got = capi.modswitch_coeff(_residues(c, qs), qs)
        k = (c + P // 2) // P        # nearest integer to c / P (independent statement)
        assert got == k % q0
        assert abs(k * P - c) <= P // 2
        assert got == _sequential_drop_last(c, qs)


# --------------------------------------------------------------------------
# o5: packing identity (reading S1) -- closed form over Z
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [16, 32, 64])
def test_packing_identity_bruteforce(n):
    rng = np.random.default_rng(n)
    for d in range(1, n + 1):
        E = n // d
        ents = rng.integers(-15, 16, size=(E, d))
        qv = rng.integers(-15, 16, size=d)
        p = capi.encode_plaintext(ents.astype(np.int8), d, n)
        assert [int(x) for x in p] == tiny_ref.encode_plaintext(ents, d, n)
        qpoly = [0] * n
        qpoly[:d] = [int(x) for x in qv]
        big = 1 << 80  # large modulus: the product is the exact integer product
        prod = tiny_ref.negacyclic_mul(qpoly, [int(x) for x in p], big)
        prod = [x - big if x > big // 2 else x for x in prod]
        for j in range(E):
            assert prod[j * d + d - 1] == int(np.dot(qv, ents[j]))


def test_encode_rejects_overfull_plaintext():
    with pytest.raises(ValueError):
        capi.encode_plaintext(np.zeros((5, 4), dtype=np.int8), 4, 16)


# --------------------------------------------------------------------------
# whole pipeline: oracle (RNS + NTT + Garner) == big-integer tiny reference
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n,L,d", [(16, 2, 4), (16, 3, 5), (32, 2, 7), (32, 3, 32), (64, 2, 8), (64, 4, 13)])
def test_server_pair_bit_exact_with_bigint_reference(n, L, d):
    qs = capi.find_primes(n, L)
    t = 65537
    rng = np.random.default_rng(n * 10 + L)
    w = synth.scaled(synth.WORKLOADS["c1"], n=n, num_limbs=L, d=d)
    E = n // d
    for trial in range(3):
        ents = rng.integers(-15, 16, size=(E, d)).astype(np.int8)
        qv = rng.integers(-15, 16, size=d).astype(np.int8)
        km = synth.key_material(w, trial, qs)
        msg = synth.query_message(w, qv)
        ct = capi.encrypt(qs, t, msg, km.s, km.a, km.e)
        # tiny_ref encryption over Z_Q gives the same ciphertext residues
        c0, c1 = tiny_ref.encrypt(qs, t, msg, km.s, km.a, km.e)
        assert np.array_equal(ct[0], np.array(tiny_ref.to_residues(c0, qs), dtype=np.uint32))
        assert np.array_equal(ct[1], np.array(tiny_ref.to_residues(c1, qs), dtype=np.uint32))
        p = capi.encode_plaintext(ents, d, n)
        resp = capi.server_pair(qs, ct, p)
        ref = tiny_ref.server_pair(qs, c0, c1, p)
        assert np.array_equal(resp, np.array(ref, dtype=np.uint32))
        dec = capi.decrypt_q0(qs[0], t, resp, km.s)
        assert [int(x) for x in dec] == tiny_ref.decrypt_q0(qs[0], t, ref[0], ref[1], km.s)
        for j in range(E):
            assert int(dec[j * d + d - 1]) == int(np.dot(qv.astype(np.int64), ents[j].astype(np.int64))) % t


def test_lift_convention_is_small_integer_mod_q():
    """Reading S8: a negative entry x is lifted as x mod q_i (not [x]_t): a
    plaintext with one coefficient -1 multiplies the ciphertext by -X^k."""
    n, L = 32, 2
    qs = capi.find_primes(n, L)
    rng = np.random.default_rng(3)
    ct = np.stack([np.stack([rng.integers(0, q, size=n) for q in qs]) for _ in range(2)]).astype(np.uint32)
    p = np.zeros(n, dtype=np.int32)
    p[0] = -1
    neg = ct.copy()
    for l, q in enumerate(qs):
        neg[:, l] = (q - ct[:, l].astype(np.int64)) % q
    resp_neg = capi.server_pair(qs, ct, p)
    p[0] = 1
    resp_negated_input = capi.server_pair(qs, neg, p)
    assert np.array_equal(resp_neg, resp_negated_input)


# --------------------------------------------------------------------------
# o8/o9: decryption equals the plaintext dot products mod t; budget > 0
# --------------------------------------------------------------------------

SHAPES = {
    "c1_c5": dict(n=4096, L=2, d=128, bound=15),
    "c2": dict(n=4096, L=3, d=128, bound=15),
    "c3": dict(n=4096, L=3, d=192, bound=15),
    "c4": dict(n=8192, L=4, d=512, bound=7),
}


@pytest.mark.parametrize("shape", list(SHAPES))
def test_decrypt_equals_dot_products_and_budget_positive(shape):
    s = SHAPES[shape]
    n, L, d, b = s["n"], s["L"], s["d"], s["bound"]
    qs = capi.find_primes(n, L)
    t = 65537
    w = synth.scaled(synth.WORKLOADS["c1"], n=n, num_limbs=L, d=d)
    rng = np.random.default_rng(n + L + d)
    E = n // d
    ents = rng.integers(-b, b + 1, size=(E + 3, d)).astype(np.int8)     # two plaintexts, last partial
    pcs = capi.encode_cluster(ents, d, n)
    qv = rng.integers(-b, b + 1, size=d).astype(np.int8)
    km = synth.key_material(w, 0, qs)
    ct = capi.encrypt(qs, t, synth.query_message(w, qv), km.s, km.a, km.e)
    assert capi.noise_budget_Q(qs, t, ct, km.s) > 0
    for k in range(pcs.shape[0]):
        resp = capi.server_pair(qs, ct, pcs[k])
        assert capi.noise_budget_q0(qs[0], t, resp, km.s) > 0
        dec = capi.decrypt_q0(qs[0], t, resp, km.s)
        cnt = min(E, ents.shape[0] - k * E)
        for j in range(E):
            want = int(np.dot(qv.astype(np.int64), ents[k * E + j].astype(np.int64))) % t if j < cnt else 0
            assert int(dec[j * d + d - 1]) == want


# --------------------------------------------------------------------------
# Dropping ciphertext LSBs (reading S20: rounded high part)
# --------------------------------------------------------------------------

def test_drop_lsb_closed_form():
    q0 = capi.find_primes(4096, 2)[0]
    rng = np.random.default_rng(20)
    c = np.concatenate([rng.integers(0, q0, size=20000), [0, 1, 31, 32, 33, 63, 64, q0 - 33, q0 - 32, q0 - 1]])
    c = c.astype(np.uint32)
    for b in (0, 1, 6, 9):
        h = capi.drop_lsb(c, b).astype(np.int64)
        low = c.astype(np.int64) - (h << b)
        if b == 0:
            assert np.array_equal(h, c)
        else:
            assert low.min() >= -(1 << (b - 1)) and low.max() < (1 << (b - 1))   # |c^l| <= 2^(b-1)
    assert int(capi.drop_lsb(np.array([q0 - 1], np.uint32), 6)[0]) < (1 << 24)  # fits the 24-bit planes


@pytest.mark.parametrize("shape", [s for s in SHAPES if SHAPES[s]["n"] <= 4096])
def test_decrypt_with_dropped_lsbs_exact(shape):
    """The paper's correctness condition ||e + e_drop|| < q_0 / 2t holds with
    b1 = 6 dropped bits of c1 at n = 4096: every result decrypts
    exactly and the phase noise stays below the bound with margin (budget
    > 1 bit: the largest of n noise coefficients is ~3.5 sigma, so the bound
    sits at > 7 sigma).  At n = 8192 the margin falls to ~0.7 bit, which is why
    WALLY_RESP_COMPACT_DROP is limited to n <= 4096."""
    s = SHAPES[shape]
    n, L, d, b = s["n"], s["L"], s["d"], s["bound"]
    qs = capi.find_primes(n, L)
    t = 65537
    w = synth.scaled(synth.WORKLOADS["c1"], n=n, num_limbs=L, d=d)
    rng = np.random.default_rng(7 * n + L + d)
    E = n // d
    for trial in range(2):
        ents = rng.integers(-b, b + 1, size=(E, d)).astype(np.int8)
        pc = capi.encode_plaintext(ents, d, n)
        qv = rng.integers(-b, b + 1, size=d).astype(np.int8)
        km = synth.key_material(w, 100 + trial, qs)
        ct = capi.encrypt(qs, t, synth.query_message(w, qv), km.s, km.a, km.e)
        resp = capi.server_pair(qs, ct, pc)
        h = capi.drop_lsb(resp[1], 6).astype(np.uint64)
        dropped = resp.copy()
        dropped[1] = ((h << 6) % qs[0]).astype(np.uint32)
        assert capi.noise_budget_q0(qs[0], t, dropped, km.s) > 1.0
        dec = capi.decrypt_q0(qs[0], t, dropped, km.s)
        for j in range(E):
            assert int(dec[j * d + d - 1]) == int(np.dot(qv.astype(np.int64), ents[j].astype(np.int64))) % t


# --------------------------------------------------------------------------
# Plaintext CRT: t = t0 t1 with the
# paper's 16- and 17-bit NTT-friendly limbs
# --------------------------------------------------------------------------

T0, T1 = 40961, 65537   # 5*8192+1 and 8*8192+1: primes = 1 mod 2n for n <= 4096


def test_plaintext_crt_limbs_are_ntt_friendly_primes():
    for t in (T0, T1):
        assert capi.is_prime(t) and t % 8192 == 1
    assert T0.bit_length() == 16 and T1.bit_length() == 17


def test_plain_crt_closed_form():
    rng = np.random.default_rng(9)
    T = T0 * T1
    xs = list(rng.integers(-(T // 2) + 1, T // 2, size=2000)) + [0, 1, -1, T // 2, -(T // 2) + 1, 43200, -43200]
    for x in xs:
        x = int(x)
        assert capi.plain_crt_signed(x % T0, x % T1, T0, T1) == x


def test_plaintext_crt_recovers_signed_dot_products_beyond_t():
    """c3 shape: |<q, e>| reaches 43,200 > (65537-1)/2, so one t = 65537 only
    gives results mod t (reading S11); two ciphertexts mod t0 and t1 give the
    exact signed value.  The server computation is the same for both."""
    n, L, d = 4096, 3, 192
    qs = capi.find_primes(n, L)
    w = synth.scaled(synth.WORKLOADS["c3"], num_queries=1)
    rng = np.random.default_rng(33)
    E = n // d
    ents = rng.integers(-15, 16, size=(E, d)).astype(np.int8)
    ents[0] = 15
    ents[1] = -15
    pc = capi.encode_plaintext(ents, d, n)
    qv = np.full(d, 15, np.int8)
    qv[-1] = -15
    want = [int(np.dot(qv.astype(np.int64), ents[j].astype(np.int64))) for j in range(E)]
    assert max(abs(x) for x in want) > (T1 - 1) // 2
    dec = []
    for i, t in enumerate((T0, T1)):
        km = synth.key_material(w, 40 + i, qs)
        ct = capi.encrypt(qs, t, synth.query_message(w, qv), km.s, km.a, km.e)
        resp = capi.server_pair(qs, ct, pc)
        assert capi.noise_budget_q0(qs[0], t, resp, km.s) > 0
        dec.append(capi.decrypt_q0(qs[0], t, resp, km.s))
    for j in range(E):
        pos = j * d + d - 1
        assert capi.plain_crt_signed(int(dec[0][pos]), int(dec[1][pos]), T0, T1) == want[j]


def test_fake_and_unit_queries():
    """S14: a zero (fake) query decrypts to all zeros; query e_0 returns e_j[0]."""
    n, L, d = 4096, 2, 128
    qs = capi.find_primes(n, L)
    t = 65537
    w = synth.scaled(synth.WORKLOADS["c1"], n=n, num_limbs=L, d=d)
    rng = np.random.default_rng(5)
    ents = rng.integers(-15, 16, size=(n // d, d)).astype(np.int8)
    p = capi.encode_plaintext(ents, d, n)
    km = synth.key_material(w, 1, qs)
    zero = capi.encrypt(qs, t, np.zeros(n, dtype=np.int32), km.s, km.a, km.e)
    dec = capi.decrypt_q0(qs[0], t, capi.server_pair(qs, zero, p), km.s)
    assert not dec.any()
    unit = np.zeros(n, dtype=np.int32)
    unit[0] = 1
    ct = capi.encrypt(qs, t, unit, km.s, km.a, km.e)
    dec = capi.decrypt_q0(qs[0], t, capi.server_pair(qs, ct, p), km.s)
    for j in range(n // d):
        assert int(dec[j * d + d - 1]) == int(ents[j][0]) % t


def test_bruteforce_all_ternary_secrets_tiny_ring():
    """N=8, d=4, two 30-bit primes, t=65537: every one of the 3^8 secrets."""
    n, L, d, t = 8, 2, 4, 65537
    qs = capi.find_primes(n, L)
    rng = np.random.default_rng(8)
    ents = rng.integers(-15, 16, size=(2, d)).astype(np.int8)
    p = capi.encode_plaintext(ents, d, n)
    qv = rng.integers(-15, 16, size=d).astype(np.int8)
    msg = np.zeros(n, dtype=np.int32)
    msg[:d] = qv
    a = np.stack([rng.integers(0, q, size=n) for q in qs]).astype(np.uint32)
    e = rng.integers(-6, 7, size=n).astype(np.int32)
    want = [int(np.dot(qv.astype(np.int64), ents[j].astype(np.int64))) % t for j in range(2)]
    import itertools
    fails = 0
    for s in itertools.product((-1, 0, 1), repeat=n):
        s = np.array(s, dtype=np.int8)
        ct = capi.encrypt(qs, t, msg, s, a, e)
        dec = capi.decrypt_q0(qs[0], t, capi.server_pair(qs, ct, p), s)
        fails += [int(dec[j * d + d - 1]) for j in range(2)] != want
    assert fails == 0


def test_server_pairs_batch_matches_single():
    n, L, d = 256, 3, 16
    qs = capi.find_primes(n, L)
    rng = np.random.default_rng(11)
    cts = np.stack([np.stack([np.stack([rng.integers(0, q, size=n) for q in qs]) for _ in range(2)])
                    for _ in range(3)]).astype(np.uint32)
    ents = rng.integers(-15, 16, size=(40, d)).astype(np.int8)
    pcs = capi.encode_cluster(ents, d, n)
    pq = np.array([0, 1, 2, 2, 0], dtype=np.uint32)
    pp = np.array([0, 1, 2, 0, 2], dtype=np.uint32)
    out, used = capi.server_pairs(qs, cts, pcs, pq, pp, threads=2)
    assert used >= 1
    for k in range(pq.size):
        assert np.array_equal(out[k], capi.server_pair(qs, cts[pq[k]], pcs[pp[k]]))


# --------------------------------------------------------------------------
# o9 pinned: the noise budget (decryption is correct while the
# noise stays below Q/2t) against ciphertexts with a KNOWN error, built with
# the big-integer tiny_ref (no oracle encryption involved).  With message 0
# the phase is exactly the error, so nu = t max|e| and the budget is
# log2(Q) - 1 - log2(t max|e|); with error 0 and message m, [t Delta m]_Q =
# -(Q mod t) m, so nu = (Q mod t) max m.  A dropped "-1", an uncentred lift
# or a wrong CRT would move these by >= 1 bit or flip the sign.
# --------------------------------------------------------------------------

def _tiny_ct(moduli, t, msg, s, e, seed):
    rng = np.random.default_rng(seed)
    n = len(msg)
    a_res = [[int(x) for x in rng.integers(0, q, size=n)] for q in moduli]
    c0, c1 = tiny_ref.encrypt(moduli, t, msg, s, a_res, e)
    return np.array([tiny_ref.to_residues(c0, moduli), tiny_ref.to_residues(c1, moduli)], dtype=np.uint32)


@pytest.mark.parametrize("L", [1, 2, 3])
def test_noise_budget_Q_known_error_and_message(L):
    n, t = 16, 65537
    qs = capi.find_primes(4096, L)
    Q = tiny_ref.product(qs)
    rng = np.random.default_rng(L)
    s = rng.integers(-1, 2, size=n).astype(np.int8)
    e = np.zeros(n, np.int64)
    e[3], e[11] = 5, -9
    ct = _tiny_ct(qs, t, [0] * n, s.tolist(), e.tolist(), 1)
    want = math.log2(Q) - 1 - math.log2(9 * t)
    assert abs(capi.noise_budget_Q(qs, t, ct, s) - want) < 1e-6
    msg = [i % 21 for i in range(n)]                  # max m = 15 (n = 16)
    ct = _tiny_ct(qs, t, msg, s.tolist(), [0] * n, 2)
    want = math.log2(Q) - 1 - math.log2((Q % t) * max(msg))
    assert abs(capi.noise_budget_Q(qs, t, ct, s) - want) < 1e-6


def test_noise_budget_q0_known_error_message_and_correctness_threshold():
    n, t = 16, 65537
    q0 = capi.find_primes(4096, 2)[0]
    rng = np.random.default_rng(9)
    s = rng.integers(-1, 2, size=n).astype(np.int8)
    e = np.zeros(n, np.int64)
    e[0], e[7] = -2, 6
    resp = _tiny_ct([q0], t, [0] * n, s.tolist(), e.tolist(), 3)[:, 0, :]
    assert abs(capi.noise_budget_q0(q0, t, resp, s) - (math.log2(q0) - 1 - math.log2(6 * t))) < 1e-9
    msg = [0] * n
    msg[4] = 5
    resp = _tiny_ct([q0], t, msg, s.tolist(), [0] * n, 4)[:, 0, :]
    assert (q0 % t) * 5 < q0 // 2
    assert abs(capi.noise_budget_q0(q0, t, resp, s) - (math.log2(q0) - 1 - math.log2((q0 % t) * 5))) < 1e-9
    # the budget runs out at the paper's bound |e| < q0 / 2t (message 0): half-way there it is
    # one bit, just inside it is ~0 and decryption is still exact, one step beyond it fails
    emax = (q0 // 2) // t                              # t * emax < q0 / 2 <= t * (emax + 1)
    for ev, want_b, ok in ((emax // 2, 1.0, True), (emax, 0.0, True), (emax + 1, 0.0, False)):
        e = np.zeros(n, np.int64)
        e[2] = ev
        resp = _tiny_ct([q0], t, [0] * n, s.tolist(), e.tolist(), 5)[:, 0, :]
        b = capi.noise_budget_q0(q0, t, resp, s)
        dec = capi.decrypt_q0(q0, t, resp, s)
        assert abs(b - want_b) < 1e-3 and (int(dec[2]) == 0) == ok and not dec[np.arange(n) != 2].any()


# --------------------------------------------------------------------------
# Reading S20 pinned to the paper's LSB-drop rule (z sqrt(2n/9)
# 2^l1 + 2^l0 < q_l/t, z = 8; correctness ||e + e_drop|| < Q'/2t).
# WALLY_RESP_COMPACT_DROP rounds c1 to 2^6 (|c1^l| <= 2^5, i.e. the
# truncation formula's 2^l1 with l1 = b - 1) and keeps c0 whole (c0^l = 0):
# the rule is z sqrt(2n/9) 2^5 < q_0 / 2t.  Every config it is used on must
# satisfy it, and the library must reject exactly the parameters that do not.
# --------------------------------------------------------------------------

def _drop_rule(n, q0, t, b=6, z=8.0):
    return z * math.sqrt(2 * n / 9) * 2 ** (b - 1) < q0 / (2 * t)


def test_compact_drop_rule_holds_for_the_configs_and_is_enforced():
    for name in ("c1", "c2", "c3", "c5"):
        w = synth.WORKLOADS[name]
        q0 = capi.find_primes(w.n, w.num_limbs)[0]
        assert w.n == 4096 and _drop_rule(w.n, q0, w.t)
        assert not _drop_rule(w.n, q0, w.t, b=7)         # 6 is the largest b the rule allows
        # the paper's own floor formula with its 2-bit headroom gives l1 = 4 (truncated),
        # i.e. 5 rounded bits; the S20 reading spends that headroom because c0 is not dropped
        l1 = math.floor(math.log2(q0 / w.t) - 2 - math.log2(8 * math.sqrt(2 * w.n / 9)))
        assert l1 == 4
    import ctypes
    from paper_2406_06761_b200 import build
    build.build()
    from paper_2406_06761_b200 import wally as W
    qs = W.wally_find_moduli(4096, 3)
    for t in (2, 40961, 65537, 68000, 70001, 131073):
        p = W.wally_params(n=4096, num_limbs=3, t=t, d=192, resp_format=W.WALLY_RESP_COMPACT_DROP)
        for i, q in enumerate(qs):
            p.moduli[i] = q
        h = ctypes.c_void_p()
        rc = W.lib.wally_create(ctypes.byref(p), 0, ctypes.byref(h))
        if rc == 0:
            W.lib.wally_destroy(h)
        assert (rc != -2) == _drop_rule(4096, qs[0], t), (t, rc)

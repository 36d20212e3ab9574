/*
 * wally_simd_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The paper's own SIMD formulation of the server computation (SURVEY.md
 * §8(f)-3), written from PAPER.md as plain, slow, obviously-correct C:
 *
 *   slots      BFV batching: m in R_t = Z_t[X]/(X^n+1), t = 1 (mod 2n), is
 *              viewed as its n evaluations m(zeta^e) at the odd exponents e;
 *              slot s = (row r, column k) <-> e = 5^k (r = 0) or -5^k (r = 1)
 *              mod 2n, so X -> X^5 rotates both rows left by one
 *              ("homomorphically rotates ... one slot to the left";
 *              reading S22 in DESIGN.md)
 *   diagonals  a cube slice is a d x d matrix whose columns are embeddings;
 *              plaintext vector j holds the j-th diagonal
 *              p_j = [e_0^j, e_1^{j+1}, ...]; floor(n/d) slices are packed
 *              side by side, the query is replicated
 *   BSGS       sum_i p_i (.) rot_i(q) computed as
 *              sum_j rot_{jg}( sum_b rot_{-jg}(p_{jg+b}) (.) rot_b(q) ),
 *              baby steps by repeated rot_1, giant steps by repeated rot_g:
 *              two rotation keys (Halevi-Shoup)
 *   key switch hybrid (GHS) key switching with one special prime P and one
 *              digit per RNS limb ("hybrid-GHS ... Kim et al."):
 *              ksk_j = (-a_j s + e_j + P Qhat_j [Qhat_j^{-1}]_{q_j} sigma(s), a_j)
 *              over Q P; switch: digits D_j = [c]_{q_j}, sum_j D_j ksk_j
 *              over Q P, then divide by P with the ModDown rounding.
 *   response   the result ciphertext is switched to q_0 (P:L1003,
 *              P:L1318-1324) with the coefficient path's oracle routine.
 *
 * Every function works in coefficient form with plain '%' arithmetic; ring
 * products use or_polymul_ntt / or_polymul_schoolbook of wally_oracle.c.
 * It shares nothing with paper_2406_06761_b200/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* from wally_oracle.c */
uint32_t or_min_root_2n(uint32_t q, uint32_t n);
void or_polymul_ntt(const uint32_t *a, const uint32_t *b, uint32_t *r, uint32_t n, uint32_t q);
uint32_t or_modswitch_coeff(const uint32_t *r, const uint32_t *mod, uint32_t L);

static uint64_t sm_mul(uint64_t a, uint64_t b, uint64_t q) { return (a * b) % q; }
static uint64_t sm_add(uint64_t a, uint64_t b, uint64_t q) { return (a + b) % q; }
static uint64_t sm_sub(uint64_t a, uint64_t b, uint64_t q) { return (a + q - b) % q; }
static uint64_t sm_pow(uint64_t b, uint64_t e, uint64_t q)
{
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = sm_mul(r, b, q);
        b = sm_mul(b, b, q);
        e >>= 1;
    }
    return r;
}
static uint64_t sm_inv(uint64_t a, uint64_t q) { return sm_pow(a, q - 2, q); } /* q prime */
static uint64_t sm_lift(int64_t x, uint64_t q)
{
    int64_t r = x % (int64_t)q;
    return (uint64_t)(r < 0 ? r + (int64_t)q : r);
}

/* ------------------------------------------------------------------ */
/* Slots (reading S22).                                                */
/* ------------------------------------------------------------------ */

/* Exponent e_s of slot s = r * n/2 + k:  5^k mod 2n (r = 0), -5^k mod 2n (r = 1). */
uint32_t or_simd_slot_exponent(uint32_t n, uint32_t s)
{
    const uint32_t half = n / 2, r = s / half, k = s % half;
    const uint64_t e = sm_pow(5, k, 2ull * n);
    return (uint32_t)(r ? (2ull * n - e) : e);
}

/* Slices of d embeddings per row (reading S23): all n/(2d) when d | n/2;
 * otherwise floor((n/2 + 1)/d) - 1, so that every rotation amount i < d
 * applied to a used column k < R d reads column k + i < n/2 of the
 * replicated query (no row wrap-around).  0 if d > n/2. */
uint32_t or_simd_row_slices(uint32_t n, uint32_t d)
{
    const uint32_t half = n / 2;
    if (d == 0 || d > half) return 0;
    if (half % d == 0) return half / d;
    return (half + 1) / d - 1;
}

/* Encoding by its definition: the unique m in R_t with m(zeta^{e_s}) =
 * slots[s] for every s; m_i = n^{-1} sum_s slots[s] zeta^{-e_s i}
 * (the e_s run over all odd residues mod 2n once).  zeta = the smallest
 * primitive 2n-th root of unity mod t (reading S13).  O(n^2). */
void or_simd_encode(uint32_t n, uint32_t t, const uint32_t *slots, uint32_t *coef)
{
    const uint64_t zeta = or_min_root_2n(t, n), tn = 2ull * n;
    uint64_t *pw = (uint64_t *)malloc(sizeof(uint64_t) * tn);
    uint32_t *ex = (uint32_t *)malloc(sizeof(uint32_t) * n);
    pw[0] = 1;
    for (uint64_t k = 1; k < tn; k++) pw[k] = sm_mul(pw[k - 1], zeta, t);
    for (uint32_t s = 0; s < n; s++) ex[s] = or_simd_slot_exponent(n, s);
    const uint64_t ninv = sm_inv(n, t);
#pragma omp parallel for schedule(static)
    for (uint32_t i = 0; i < n; i++) {
        uint64_t acc = 0;
        for (uint32_t s = 0; s < n; s++) {
            const uint64_t ei = ((uint64_t)ex[s] * i) % tn;
            acc = sm_add(acc, sm_mul(slots[s] % t, pw[(tn - ei) % tn], t), t);
        }
        coef[i] = (uint32_t)sm_mul(acc, ninv, t);
    }
    free(pw);
    free(ex);
}

/* Decoding by its definition: slots[s] = m(zeta^{e_s}) = sum_i m_i zeta^{e_s i}. */
void or_simd_decode(uint32_t n, uint32_t t, const uint32_t *coef, uint32_t *slots)
{
    const uint64_t zeta = or_min_root_2n(t, n), tn = 2ull * n;
    uint64_t *pw = (uint64_t *)malloc(sizeof(uint64_t) * tn);
    pw[0] = 1;
    for (uint64_t k = 1; k < tn; k++) pw[k] = sm_mul(pw[k - 1], zeta, t);
#pragma omp parallel for schedule(static)
    for (uint32_t s = 0; s < n; s++) {
        const uint64_t e = or_simd_slot_exponent(n, s);
        uint64_t acc = 0;
        for (uint32_t i = 0; i < n; i++) acc = sm_add(acc, sm_mul(coef[i] % t, pw[(e * i) % tn], t), t);
        slots[s] = (uint32_t)acc;
    }
    free(pw);
}

/* ------------------------------------------------------------------ */
/* Galois automorphism sigma_k: a(X) -> a(X^k), k odd (coefficient form). */
/* X^{ik} = X^{ik mod 2n} and X^n = -1.                                 */
/* ------------------------------------------------------------------ */
void or_automorph(uint32_t n, uint32_t q, const uint32_t *a, uint32_t k, uint32_t *out)
{
    for (uint32_t i = 0; i < n; i++) {
        const uint64_t j = ((uint64_t)i * k) % (2ull * n);
        if (j < n) out[j] = a[i] % q;
        else out[j - n] = (uint32_t)sm_sub(0, a[i] % q, q);
    }
}

/* ------------------------------------------------------------------ */
/* Hybrid key switching, moduli mods[0..L-1] = the ciphertext */
/* limbs q_j, mods[L] = the special prime P.  Key layout [2][L][L+1][n]:   */
/* component 0 = b_j, component 1 = a_j, digit j, modulus m.              */
/* ------------------------------------------------------------------ */

/* g_j mod mods[m] = P * Qhat_j * [Qhat_j^{-1}]_{q_j} mod mods[m], Qhat_j = prod_{i != j} q_i. */
static uint64_t or_gadget(const uint32_t *mods, uint32_t L, uint32_t j, uint32_t m)
{
    const uint64_t qm = mods[m], qj = mods[j];
    uint64_t qhat_j_mod_qj = 1, qhat_j_mod_qm = 1;
    for (uint32_t i = 0; i < L; i++) {
        if (i == j) continue;
        qhat_j_mod_qj = sm_mul(qhat_j_mod_qj, mods[i] % qj, qj);
        qhat_j_mod_qm = sm_mul(qhat_j_mod_qm, mods[i] % qm, qm);
    }
    const uint64_t inv = sm_inv(qhat_j_mod_qj, qj);  /* [Qhat_j^{-1}]_{q_j} as an integer < q_j */
    return sm_mul(sm_mul(mods[L] % qm, qhat_j_mod_qm, qm), inv % qm, qm);
}

/* Key for sigma_k: b_{j,m} = -a_{j,m} s + e_j + g_j sigma_k(s) mod mods[m].
 * s: ternary int8 [n]; a: uniform [L][L+1][n] (a_{j,m} < mods[m]);
 * e: small int32 [L][n]; key out: [2][L][L+1][n]. */
void or_simd_keygen(uint32_t n, uint32_t L, const uint32_t *mods, const int8_t *s, uint32_t k, const uint32_t *a,
                    const int32_t *e, uint32_t *key)
{
    uint32_t *sl = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *ss = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *as = (uint32_t *)malloc(sizeof(uint32_t) * n);
    for (uint32_t j = 0; j < L; j++)
        for (uint32_t m = 0; m <= L; m++) {
            const uint64_t q = mods[m];
            const uint64_t gj = or_gadget(mods, L, j, m);
            for (uint32_t i = 0; i < n; i++) sl[i] = (uint32_t)sm_lift(s[i], q);
            or_automorph(n, (uint32_t)q, sl, k, ss);
            const uint32_t *ajm = a + ((size_t)j * (L + 1) + m) * n;
            or_polymul_ntt(ajm, sl, as, n, (uint32_t)q);
            uint32_t *b = key + ((size_t)j * (L + 1) + m) * n;
            uint32_t *ak = key + (((size_t)L + j) * (L + 1) + m) * n;
            for (uint32_t i = 0; i < n; i++) {
                uint64_t v = sm_sub(0, as[i], q);
                v = sm_add(v, sm_lift(e[(size_t)j * n + i], q), q);
                v = sm_add(v, sm_mul(gj, ss[i], q), q);
                b[i] = (uint32_t)v;
                ak[i] = ajm[i] % (uint32_t)q;
            }
        }
    free(sl);
    free(ss);
    free(as);
}

/* Key switch of c (coefficient form over Q = prod_{j<L} q_j, [L][n]):
 *   ModUp   D_j = [c]_{q_j} as integers in [0, q_j), read mod every mods[m]
 *   product acc_comp,m = sum_j D_j * key[comp][j][m]  in Z_{mods[m]}[X]/(X^n+1)
 *   ModDown out_comp,i = (acc_comp,i - [acc_comp,P]_P) * P^{-1} mod q_i,
 *           [acc_P]_P the canonical representative in [0, P)
 * out: [2][L][n] over Q.  (sum_comp out_comp s^comp = c sigma(s) + small.) */
void or_keyswitch(uint32_t n, uint32_t L, const uint32_t *mods, const uint32_t *c, const uint32_t *key, uint32_t *out)
{
    const uint32_t M = L + 1;
    uint32_t *acc = (uint32_t *)malloc(sizeof(uint32_t) * 2 * M * n);
    uint32_t *dj = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *pr = (uint32_t *)malloc(sizeof(uint32_t) * n);
    memset(acc, 0, sizeof(uint32_t) * 2 * M * n);
    for (uint32_t comp = 0; comp < 2; comp++)
        for (uint32_t m = 0; m < M; m++) {
            const uint32_t q = mods[m];
            uint32_t *am = acc + ((size_t)comp * M + m) * n;
            for (uint32_t j = 0; j < L; j++) {
                for (uint32_t i = 0; i < n; i++) dj[i] = c[(size_t)j * n + i] % q;
                or_polymul_ntt(dj, key + (((size_t)comp * L + j) * M + m) * n, pr, n, q);
                for (uint32_t i = 0; i < n; i++) am[i] = (uint32_t)sm_add(am[i], pr[i], q);
            }
        }
    const uint64_t P = mods[L];
    for (uint32_t comp = 0; comp < 2; comp++) {
        const uint32_t *aP = acc + ((size_t)comp * M + L) * n;
        for (uint32_t i = 0; i < L; i++) {
            const uint64_t q = mods[i];
            const uint64_t pinv = sm_inv(P % q, q);
            const uint32_t *ai = acc + ((size_t)comp * M + i) * n;
            uint32_t *o = out + ((size_t)comp * L + i) * n;
            for (uint32_t x = 0; x < n; x++) o[x] = (uint32_t)sm_mul(sm_sub(ai[x], aP[x] % q, q), pinv, q);
        }
    }
    free(acc);
    free(dj);
    free(pr);
}

/* Rotation (homomorphic sigma_k): (sigma(c0), sigma(c1)) decrypts under
 * sigma(s); switching sigma(c1) back to s gives
 * (sigma(c0) + ks_0, ks_1).  ct, out: [2][L][n] coefficient form over Q. */
void or_rotate(uint32_t n, uint32_t L, const uint32_t *mods, const uint32_t *ct, uint32_t k, const uint32_t *key,
               uint32_t *out)
{
    uint32_t *sc = (uint32_t *)malloc(sizeof(uint32_t) * 2 * L * n);
    uint32_t *ks = (uint32_t *)malloc(sizeof(uint32_t) * 2 * L * n);
    for (uint32_t comp = 0; comp < 2; comp++)
        for (uint32_t l = 0; l < L; l++)
            or_automorph(n, mods[l], ct + ((size_t)comp * L + l) * n, k, sc + ((size_t)comp * L + l) * n);
    or_keyswitch(n, L, mods, sc + (size_t)L * n, key, ks);
    for (uint32_t l = 0; l < L; l++)
        for (uint32_t x = 0; x < n; x++) {
            const size_t i0 = (size_t)l * n + x, i1 = ((size_t)L + l) * n + x;
            out[i0] = (uint32_t)sm_add(sc[i0], ks[i0], mods[l]);
            out[i1] = ks[i1];
        }
    free(sc);
    free(ks);
}

/* ------------------------------------------------------------------ */
/* Database packing with the BSGS pre-rotation.           */
/* ------------------------------------------------------------------ */

/* Slot vectors of the d plaintexts of one ciphertext block of a cluster:
 * entries [cnt][d] (int8, this block's embeddings, cnt <= 2 R d).  Column
 * k < R d of row r holds embedding  e = (r R + k/d) d + k mod d  (slice
 * r R + k/d, column k mod d of the slice); diagonal i holds
 * diag_i[r][k] = e^{(k mod d + i) mod d}  ("p_j = [e_0^j, e_1^{j+1}, ...]").
 * Plaintext i = j g + b stores rot_{-jg}(diag_i), i.e. column k holds
 * diag_i[r][(k - j g) mod n/2] (the BSGS pre-rotation).  Values mod t. */
void or_simd_diagonal_slots(uint32_t n, uint32_t t, uint32_t d, uint32_t g, const int8_t *entries, uint32_t cnt,
                            uint32_t *slots /* [d][n] */)
{
    const uint32_t half = n / 2, R = or_simd_row_slices(n, d);
    for (uint32_t i = 0; i < d; i++) {
        const uint32_t jg = (i / g) * g;
        for (uint32_t r = 0; r < 2; r++)
            for (uint32_t k = 0; k < half; k++) {
                const uint32_t kk = (uint32_t)(((uint64_t)k + half - (jg % half)) % half);
                uint32_t v = 0;
                if (kk < R * d) {
                    const uint32_t e = (r * R + kk / d) * d + kk % d;
                    if (e < cnt) v = (uint32_t)sm_lift(entries[(size_t)e * d + (kk % d + i) % d], t);
                }
                slots[(size_t)i * n + (size_t)r * half + k] = v;
            }
    }
}

/* Query slots: the embedding replicated along both rows, column k holds q^{k mod d}. */
void or_simd_query_slots(uint32_t n, uint32_t t, uint32_t d, const int32_t *q, uint32_t *slots)
{
    const uint32_t half = n / 2;
    for (uint32_t s = 0; s < n; s++) slots[s] = (uint32_t)sm_lift(q[(s % half) % d], t);
}

/* ------------------------------------------------------------------ */
/* Server computation, SIMD form (Alg 4 P:L794-808 with P:L557-613).    */
/* ------------------------------------------------------------------ */

/* ct: [2][L][n] coefficient form over Q.  keys: [2][L][L+1][n] for
 * sigma_5 (rotation by one) and sigma_{5^g} (rotation by g).
 * pt: [d][n] plaintext coefficients mod t (the encoded, pre-rotated
 * diagonals); each is lifted to R_Q by its centered representative
 * in (-t/2, t/2] (reading S24).  out: [2][L][n] over Q:
 *   baby_0 = ct, baby_b = rot_1(baby_{b-1})                (b < g)
 *   I_j    = sum_{b < g, jg+b < d} pt_{jg+b} * baby_b       (j < m = ceil(d/g))
 *   acc    = I_{m-1};  acc = rot_g(acc) + I_j  for j = m-2 .. 0
 * Returns 0, or -1 on bad arguments. */
int or_simd_server(uint32_t n, uint32_t L, const uint32_t *mods, uint32_t t, uint32_t d, uint32_t g,
                   const uint32_t *ct, const uint32_t *key1, const uint32_t *keyg, const uint32_t *pt, uint32_t *out)
{
    if (g == 0 || d == 0 || g > d) return -1;
    const size_t CT = (size_t)2 * L * n;
    const uint32_t m = (d + g - 1) / g;
    const uint32_t k1 = 5 % (2 * n), kg = (uint32_t)sm_pow(5, g, 2ull * n);
    uint32_t *baby = (uint32_t *)malloc(sizeof(uint32_t) * CT * g);
    uint32_t *I = (uint32_t *)malloc(sizeof(uint32_t) * CT * m);
    uint32_t *pl = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *pr = (uint32_t *)malloc(sizeof(uint32_t) * n);
    memcpy(baby, ct, sizeof(uint32_t) * CT);
    for (uint32_t b = 1; b < g; b++) or_rotate(n, L, mods, baby + (b - 1) * CT, k1, key1, baby + b * CT);
    memset(I, 0, sizeof(uint32_t) * CT * m);
    for (uint32_t j = 0; j < m; j++)
        for (uint32_t b = 0; b < g && j * g + b < d; b++) {
            const uint32_t *p = pt + (size_t)(j * g + b) * n;
            for (uint32_t l = 0; l < L; l++) {
                const uint64_t q = mods[l];
                for (uint32_t x = 0; x < n; x++) {
                    const int64_t c = (p[x] % t) > t / 2 ? (int64_t)(p[x] % t) - (int64_t)t : (int64_t)(p[x] % t);
                    pl[x] = (uint32_t)sm_lift(c, q);
                }
                for (uint32_t comp = 0; comp < 2; comp++) {
                    or_polymul_ntt(baby + b * CT + ((size_t)comp * L + l) * n, pl, pr, n, (uint32_t)q);
                    uint32_t *dst = I + j * CT + ((size_t)comp * L + l) * n;
                    for (uint32_t x = 0; x < n; x++) dst[x] = (uint32_t)sm_add(dst[x], pr[x], q);
                }
            }
        }
    memcpy(out, I + (size_t)(m - 1) * CT, sizeof(uint32_t) * CT);
    for (int j = (int)m - 2; j >= 0; j--) {
        uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * CT);
        or_rotate(n, L, mods, out, kg, keyg, tmp);
        for (uint32_t comp = 0; comp < 2; comp++)
            for (uint32_t l = 0; l < L; l++)
                for (uint32_t x = 0; x < n; x++) {
                    const size_t ix = ((size_t)comp * L + l) * n + x;
                    out[ix] = (uint32_t)sm_add(tmp[ix], I[(size_t)j * CT + ix], mods[l]);
                }
        free(tmp);
    }
    free(baby);
    free(I);
    free(pl);
    free(pr);
    return 0;
}

/* The response: the server result switched to q_0 coefficient by
 * coefficient (or_modswitch_coeff, P:L1003 / P:L1318-1324).
 * in: [2][L][n] over Q; resp: [2][n] mod q_0. */
void or_simd_response(uint32_t n, uint32_t L, const uint32_t *mods, const uint32_t *in, uint32_t *resp)
{
    uint32_t r[16];
    for (uint32_t comp = 0; comp < 2; comp++)
        for (uint32_t x = 0; x < n; x++) {
            for (uint32_t l = 0; l < L; l++) r[l] = in[((size_t)comp * L + l) * n + x];
            resp[(size_t)comp * n + x] = or_modswitch_coeff(r, mods, L);
        }
}

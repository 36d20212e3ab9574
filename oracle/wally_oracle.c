/*
 * wally_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the server-side
 * encrypted dot-product path of Wally (arXiv 2406.06761), written from the
 * paper and from the readings listed in DESIGN.md ("Readings").
 * It exists to check the CUDA path; it is never a fallback for it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with paper_2406_06761_b200/ (the product).
 *
 * Citation keys: "P:Lnnn" = PAPER.md line nnn.
 *
 * Conventions:
 *   ring        R_q = Z_q[X]/(X^n + 1), n a power of two
 *   moduli      q_0 < q_1 < ... < q_{L-1}: the L largest primes < 2^30 with
 *               q = 1 (mod 2n) (NTT-friendly), listed ascending.
 *   RNS         Q = prod q_i; every residue kept canonical in [0, q_i)
 *   ciphertext  ct = (c0, c1), c1 = a, c0 = -a*s + e + Delta*m,
 *               Delta = floor(Q/t); decryption c0 + c1*s = Delta*m + e
 *   packing     p_k(X) = sum_{j<E} sum_{i<d} e_{kE+j}[i] X^{j*d+d-1-i},
 *               E = floor(n/d); the small signed entries are lifted as x mod q_i
 *   server      r = c * p_k in R_Q for c in {c0, c1}; then modulus switch to
 *               q_0: c' = round(c * q_0 / Q) mod q_0
 *   decrypt     v = c0' + c1' * s mod q_0; m = round(t * v / q_0) mod t
 *
 * Arithmetic is plain scalar uint64_t with '%' reduction (residues < 2^30,
 * so every product is < 2^60), and unsigned __int128 for CRT values
 * (Q < 2^120).  No lazy reduction, no Montgomery/Shoup, no blocking.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

#define OR_MAX_LIMBS 8

/* ------------------------------------------------------------------ */
/* Scalar modular arithmetic (textbook).                               */
/* ------------------------------------------------------------------ */

static uint64_t or_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (a * b) % q; }

static uint64_t or_addmod(uint64_t a, uint64_t b, uint64_t q) { return (a + b) % q; }

static uint64_t or_submod(uint64_t a, uint64_t b, uint64_t q) { return (a + q - b) % q; }

static uint64_t or_powmod(uint64_t b, uint64_t e, uint64_t q)
{
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = or_mulmod(r, b, q);
        b = or_mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}

/* Inverse by Fermat's little theorem (q prime). */
static uint64_t or_invmod(uint64_t a, uint64_t q) { return or_powmod(a, q - 2, q); }

/* Signed small integer x lifted to [0, q): "x mod q" (reading S8). */
static uint64_t or_lift(int64_t x, uint64_t q)
{
    int64_t r = x % (int64_t)q;
    if (r < 0) r += (int64_t)q;
    return (uint64_t)r;
}

/* ------------------------------------------------------------------ */
/* Parameters: NTT-friendly primes ("q_i = 1 mod 2n").         */
/* ------------------------------------------------------------------ */

int or_is_prime(uint64_t x)
{
    if (x < 2) return 0;
    if (x % 2 == 0) return x == 2;
    for (uint64_t f = 3; f * f <= x; f += 2)
        if (x % f == 0) return 0;
    return 1;
}

/* The L largest primes q < 2^30 with q = 1 (mod 2n), written ascending
 * (q_0 smallest, reading S5/S6).  Returns 0 on success, -1 if not found. */
int or_find_primes(uint32_t n, uint32_t L, uint32_t *out)
{
    uint64_t step = 2ull * n;
    uint64_t q = ((1ull << 30) - 1) / step * step + 1; /* largest 1 mod 2n below 2^30 */
    if (q >= (1ull << 30)) q -= step;
    uint32_t found = 0;
    uint32_t tmp[OR_MAX_LIMBS];
    if (L == 0 || L > OR_MAX_LIMBS) return -1;
    while (found < L && q > step) {
        if (or_is_prime(q)) tmp[found++] = (uint32_t)q;
        q -= step;
    }
    if (found < L) return -1;
    for (uint32_t i = 0; i < L; i++) out[i] = tmp[L - 1 - i];
    return 0;
}

/* Smallest primitive 2n-th root of unity mod q (reading S13).
 * Find a generator g of Z_q^* by checking g^((q-1)/p) != 1 for every prime
 * p | q-1; psi0 = g^((q-1)/2n) is a primitive 2n-th root; all primitive
 * 2n-th roots are psi0^k with k odd; return the minimum. */
uint32_t or_min_root_2n(uint32_t q, uint32_t n)
{
    uint64_t m = q - 1, primes[64];
    int np = 0;
    uint64_t t = m;
    for (uint64_t f = 2; f * f <= t; f++) {
        if (t % f == 0) {
            primes[np++] = f;
            while (t % f == 0) t /= f;
        }
    }
    if (t > 1) primes[np++] = t;
    uint64_t g = 2;
    for (;; g++) {
        int ok = 1;
        for (int i = 0; i < np; i++)
            if (or_powmod(g, m / primes[i], q) == 1) { ok = 0; break; }
        if (ok) break;
    }
    uint64_t psi0 = or_powmod(g, m / (2ull * n), q);
    uint64_t best = q, p = psi0, psi2 = or_mulmod(psi0, psi0, q);
    for (uint64_t k = 1; k < 2ull * n; k += 2) { /* p = psi0^k */
        if (p < best) best = p;
        p = or_mulmod(p, psi2, q);
    }
    return (uint32_t)best;
}

/* ------------------------------------------------------------------ */
/* Textbook negacyclic NTT (switch between evaluation and */
/* coefficient form in O(n log n)).                                     */
/* Forward: A_k = sum_j a_j psi^((2k+1) j), k in natural order, computed */
/* as twist a_j <- a_j psi^j followed by the cyclic NTT with omega =     */
/* psi^2 (iterative radix-2 Cooley-Tukey on bit-reversed input).         */
/* ------------------------------------------------------------------ */

static void or_bitreverse(uint64_t *a, uint32_t n)
{
    for (uint32_t i = 1, j = 0; i < n; i++) {
        uint32_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { uint64_t x = a[i]; a[i] = a[j]; a[j] = x; }
    }
}

static void or_cyclic_ntt(uint64_t *a, uint32_t n, uint64_t omega, uint64_t q)
{
    or_bitreverse(a, n);
    for (uint32_t len = 2; len <= n; len <<= 1) {
        uint64_t wlen = or_powmod(omega, n / len, q);
        for (uint32_t i = 0; i < n; i += len) {
            uint64_t w = 1;
            for (uint32_t j = 0; j < len / 2; j++) {
                uint64_t u = a[i + j];
                uint64_t v = or_mulmod(a[i + j + len / 2], w, q);
                a[i + j] = or_addmod(u, v, q);
                a[i + j + len / 2] = or_submod(u, v, q);
                w = or_mulmod(w, wlen, q);
            }
        }
    }
}

void or_ntt_forward(uint64_t *a, uint32_t n, uint32_t q)
{
    uint64_t psi = or_min_root_2n(q, n);
    uint64_t pw = 1;
    for (uint32_t j = 0; j < n; j++) {
        a[j] = or_mulmod(a[j] % q, pw, q);
        pw = or_mulmod(pw, psi, q);
    }
    or_cyclic_ntt(a, n, or_mulmod(psi, psi, q), q);
}

void or_ntt_inverse(uint64_t *a, uint32_t n, uint32_t q)
{
    uint64_t psi = or_min_root_2n(q, n);
    uint64_t psi_inv = or_invmod(psi, q);
    or_cyclic_ntt(a, n, or_mulmod(psi_inv, psi_inv, q), q);
    uint64_t n_inv = or_invmod(n, q);
    uint64_t pw = n_inv;
    for (uint32_t j = 0; j < n; j++) {
        a[j] = or_mulmod(a[j], pw, q);
        pw = or_mulmod(pw, psi_inv, q);
    }
}

/* The NTT with a caller-supplied psi (no root search); used by the
 * per-pair server path so it does not redo the root search per call. */
static void or_ntt_forward_psi(uint64_t *a, uint32_t n, uint64_t q, uint64_t psi)
{
    uint64_t pw = 1;
    for (uint32_t j = 0; j < n; j++) {
        a[j] = or_mulmod(a[j] % q, pw, q);
        pw = or_mulmod(pw, psi, q);
    }
    or_cyclic_ntt(a, n, or_mulmod(psi, psi, q), q);
}

static void or_ntt_inverse_psi(uint64_t *a, uint32_t n, uint64_t q, uint64_t psi)
{
    uint64_t psi_inv = or_invmod(psi, q);
    or_cyclic_ntt(a, n, or_mulmod(psi_inv, psi_inv, q), q);
    uint64_t pw = or_invmod(n, q);
    for (uint32_t j = 0; j < n; j++) {
        a[j] = or_mulmod(a[j], pw, q);
        pw = or_mulmod(pw, psi_inv, q);
    }
}

/* Negacyclic product r = a*b in Z_q[X]/(X^n+1) by NTT (forward both,
 * pointwise multiply, inverse).  a, b canonical; r canonical. */
void or_polymul_ntt(const uint32_t *a, const uint32_t *b, uint32_t *r, uint32_t n, uint32_t q)
{
    uint64_t psi = or_min_root_2n(q, n);
    uint64_t *x = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint64_t *y = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (uint32_t i = 0; i < n; i++) { x[i] = a[i]; y[i] = b[i]; }
    or_ntt_forward_psi(x, n, q, psi);
    or_ntt_forward_psi(y, n, q, psi);
    for (uint32_t i = 0; i < n; i++) x[i] = or_mulmod(x[i], y[i], q);
    or_ntt_inverse_psi(x, n, q, psi);
    for (uint32_t i = 0; i < n; i++) r[i] = (uint32_t)x[i];
    free(x);
    free(y);
}

/* Negacyclic product by the O(n^2) schoolbook definition:
 * r_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+n} a_i b_j (X^n = -1). */
void or_polymul_schoolbook(const uint32_t *a, const uint32_t *b, uint32_t *r, uint32_t n, uint32_t q)
{
    uint64_t *acc = (uint64_t *)calloc(n, sizeof(uint64_t));
    for (uint32_t i = 0; i < n; i++)
        for (uint32_t j = 0; j < n; j++) {
            uint64_t p = or_mulmod(a[i], b[j], q);
            uint32_t k = i + j;
            if (k < n) acc[k] = or_addmod(acc[k], p, q);
            else acc[k - n] = or_submod(acc[k - n], p, q);
        }
    for (uint32_t k = 0; k < n; k++) r[k] = (uint32_t)acc[k];
    free(acc);
}

/* ------------------------------------------------------------------ */
/* CRT and modulus switching.     */
/* ------------------------------------------------------------------ */

/* Q = prod q_i as a 128-bit integer. */
static u128 or_big_Q(const uint32_t *mod, uint32_t L)
{
    u128 Q = 1;
    for (uint32_t i = 0; i < L; i++) Q *= mod[i];
    return Q;
}

/* Garner's mixed-radix CRT: the unique c in [0, Q) with c = r_i mod q_i. */
u128 or_crt(const uint32_t *r, const uint32_t *mod, uint32_t L)
{
    uint64_t v[OR_MAX_LIMBS];
    for (uint32_t i = 0; i < L; i++) {
        uint64_t x = r[i] % mod[i];
        for (uint32_t j = 0; j < i; j++) {
            /* x <- (x - v_j) * q_j^{-1} mod q_i */
            x = or_submod(x, v[j] % mod[i], mod[i]);
            x = or_mulmod(x, or_invmod(mod[j] % mod[i], mod[i]), mod[i]);
        }
        v[i] = x;
    }
    u128 c = 0, w = 1;
    for (uint32_t i = 0; i < L; i++) {
        c += (u128)v[i] * w;
        w *= mod[i];
    }
    return c;
}

/* Exact modulus switch of one coefficient from Q down to q_0 (reading S6/S7):
 * c' = round(c * q_0 / Q) mod q_0 = floor((2c + P) / (2P)) mod q_0, P = Q/q_0.
 * P is a product of odd primes, so c/P is never k + 1/2 (no ties). */
uint32_t or_modswitch_coeff(const uint32_t *r, const uint32_t *mod, uint32_t L)
{
    u128 c = or_crt(r, mod, L);
    u128 Q = or_big_Q(mod, L);
    u128 P = Q / mod[0];
    u128 v = (2 * c + P) / (2 * P);
    return (uint32_t)(v % mod[0]);
}

/* Exported for tests: CRT value split as (lo, hi) 64-bit words. */
void or_crt_u128(const uint32_t *r, const uint32_t *mod, uint32_t L, uint64_t *lo, uint64_t *hi)
{
    u128 c = or_crt(r, mod, L);
    *lo = (uint64_t)c;
    *hi = (uint64_t)(c >> 64);
}

/* ------------------------------------------------------------------ */
/* Database encoding (coefficient packing, reading S1; BASELINE.json     */
/* configs[0] "packed 32 per plaintext at coefficient offsets j*128      */
/* (reversed)").                                                          */
/* ------------------------------------------------------------------ */

/* entries: int8 [count][d], count <= floor(n/d).  out: int32 [n] (signed
 * small coefficients, zero elsewhere: reading S10). */
int or_encode_plaintext(const int8_t *entries, uint32_t count, uint32_t d, uint32_t n, int32_t *out)
{
    if (d == 0 || d > n || count > n / d) return -1;
    memset(out, 0, sizeof(int32_t) * n);
    for (uint32_t j = 0; j < count; j++)
        for (uint32_t i = 0; i < d; i++)
            out[j * d + d - 1 - i] = entries[(size_t)j * d + i];
    return 0;
}

/* ------------------------------------------------------------------ */
/* Server computation for one (query, plaintext) pair (Alg 4  */
/* analog).                                           */
/*   ct   : uint32 [2][L][n], canonical, coefficient form                 */
/*   pcoef: int32  [n] signed plaintext coefficients (or_encode_plaintext)*/
/*   out  : uint32 [2][n], the mod-switched response, canonical mod q_0   */
/* ------------------------------------------------------------------ */

typedef struct {
    uint32_t n, L;
    uint32_t mod[OR_MAX_LIMBS];
    uint64_t psi[OR_MAX_LIMBS];
} or_params;

static void or_params_init(or_params *p, uint32_t n, uint32_t L, const uint32_t *mod)
{
    p->n = n;
    p->L = L;
    for (uint32_t i = 0; i < L; i++) {
        p->mod[i] = mod[i];
        p->psi[i] = or_min_root_2n(mod[i], n);
    }
}

static void or_server_pair_p(const or_params *P, const uint32_t *ct, const int32_t *pcoef, uint32_t *out)
{
    uint32_t n = P->n, L = P->L;
    uint64_t *x = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint64_t *y = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint32_t *prod = (uint32_t *)malloc(sizeof(uint32_t) * n * L);
    for (uint32_t comp = 0; comp < 2; comp++) {
        for (uint32_t l = 0; l < L; l++) {
            uint64_t q = P->mod[l];
            const uint32_t *c = ct + ((size_t)comp * L + l) * n;
            for (uint32_t i = 0; i < n; i++) {
                x[i] = c[i];
                y[i] = or_lift(pcoef[i], q);
            }
            or_ntt_forward_psi(x, n, q, P->psi[l]);
            or_ntt_forward_psi(y, n, q, P->psi[l]);
            for (uint32_t i = 0; i < n; i++) x[i] = or_mulmod(x[i], y[i], q);
            or_ntt_inverse_psi(x, n, q, P->psi[l]);
            for (uint32_t i = 0; i < n; i++) prod[(size_t)l * n + i] = (uint32_t)x[i];
        }
        for (uint32_t i = 0; i < n; i++) {
            uint32_t r[OR_MAX_LIMBS];
            for (uint32_t l = 0; l < L; l++) r[l] = prod[(size_t)l * n + i];
            out[(size_t)comp * n + i] = or_modswitch_coeff(r, P->mod, L);
        }
    }
    free(x);
    free(y);
    free(prod);
}

void or_server_pair(uint32_t n, uint32_t L, const uint32_t *mod, const uint32_t *ct, const int32_t *pcoef,
                    uint32_t *out)
{
    or_params P;
    or_params_init(&P, n, L, mod);
    or_server_pair_p(&P, ct, pcoef, out);
}

/* A list of pairs, OpenMP-parallel over pairs (the only parallelism; the
 * per-pair computation is the plain or_server_pair).
 *   cts    : uint32 [nq][2][L][n]
 *   pcoefs : int32  [npt][n]
 *   pair_q, pair_pt : [npairs]
 *   out    : uint32 [npairs][2][n]
 * threads <= 0 uses the OpenMP default.  Returns the thread count used. */
int or_server_pairs(uint32_t n, uint32_t L, const uint32_t *mod, const uint32_t *cts, const int32_t *pcoefs,
                    uint64_t npairs, const uint32_t *pair_q, const uint32_t *pair_pt, uint32_t *out, int threads)
{
    or_params P;
    or_params_init(&P, n, L, mod);
    int used = 1;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
#pragma omp for schedule(dynamic, 1)
        for (int64_t k = 0; k < (int64_t)npairs; k++)
            or_server_pair_p(&P, cts + (size_t)pair_q[k] * 2 * L * n, pcoefs + (size_t)pair_pt[k] * n,
                             out + (size_t)k * 2 * n);
    }
#else
    (void)threads;
    for (uint64_t k = 0; k < npairs; k++)
        or_server_pair_p(&P, cts + (size_t)pair_q[k] * 2 * L * n, pcoefs + (size_t)pair_pt[k] * n,
                         out + (size_t)k * 2 * n);
#endif
    return used;
}

/* ------------------------------------------------------------------ */
/* Client side (oracle-only; the server never holds keys).              */
/* ------------------------------------------------------------------ */

/* Delta = floor(Q / t) reduced mod q_l. */
static uint64_t or_delta_mod(const uint32_t *mod, uint32_t L, uint32_t t, uint32_t l)
{
    u128 Q = or_big_Q(mod, L);
    u128 D = Q / t;
    return (uint64_t)(D % mod[l]);
}

/* Symmetric BFV encryption (P:L248-251 as read in S2; P:L1334 Delta form):
 *   m(X) = sum_i [msg_i]_t X^i, msg given as int32 [n] (already in [0,t) or
 *          any integer; reduced to [0, t) here, reading S9);
 *   s    : int8 [n] ternary secret;  a : uint32 [L][n] uniform residues;
 *   e    : int32 [n] small error;
 *   ct   : uint32 [2][L][n]:  c0 = -a*s + e + Delta*m,  c1 = a. */
void or_encrypt(uint32_t n, uint32_t L, const uint32_t *mod, uint32_t t, const int32_t *msg, const int8_t *s,
                const uint32_t *a, const int32_t *e, uint32_t *ct)
{
    uint32_t *sl = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *as = (uint32_t *)malloc(sizeof(uint32_t) * n);
    for (uint32_t l = 0; l < L; l++) {
        uint64_t q = mod[l];
        uint64_t delta = or_delta_mod(mod, L, t, l);
        for (uint32_t i = 0; i < n; i++) sl[i] = (uint32_t)or_lift(s[i], q);
        or_polymul_ntt(a + (size_t)l * n, sl, as, n, (uint32_t)q);
        uint32_t *c0 = ct + (size_t)l * n;
        uint32_t *c1 = ct + ((size_t)L + l) * n;
        for (uint32_t i = 0; i < n; i++) {
            uint64_t mi = or_lift(msg[i], t);
            uint64_t v = or_submod(0, as[i], q);
            v = or_addmod(v, or_lift(e[i], q), q);
            v = or_addmod(v, or_mulmod(delta, mi, q), q);
            c0[i] = (uint32_t)v;
            c1[i] = a[(size_t)l * n + i];
        }
    }
    free(sl);
    free(as);
}

/* Phase of a single-limb response: v = c0' + c1' * s mod q_0 (schoolbook
 * negacyclic product with the ternary s).  out: uint32 [n]. */
void or_phase_q0(uint32_t n, uint32_t q0, const uint32_t *resp, const int8_t *s, uint32_t *v)
{
    uint32_t *sl = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *c1s = (uint32_t *)malloc(sizeof(uint32_t) * n);
    for (uint32_t i = 0; i < n; i++) sl[i] = (uint32_t)or_lift(s[i], q0);
    or_polymul_ntt(resp + n, sl, c1s, n, q0);
    for (uint32_t i = 0; i < n; i++) v[i] = (uint32_t)or_addmod(resp[i], c1s[i], q0);
    free(sl);
    free(c1s);
}

/* Decryption of a single-limb response:
 * m_i = round(t * v_i / q_0) mod t = floor((2 t v_i + q_0) / (2 q_0)) mod t. */
void or_decrypt_q0(uint32_t n, uint32_t q0, uint32_t t, const uint32_t *resp, const int8_t *s, uint32_t *m)
{
    uint32_t *v = (uint32_t *)malloc(sizeof(uint32_t) * n);
    or_phase_q0(n, q0, resp, s, v);
    for (uint32_t i = 0; i < n; i++) {
        uint64_t num = 2ull * t * v[i] + q0;
        m[i] = (uint32_t)((num / (2ull * q0)) % t);
    }
    free(v);
}

/* Plaintext CRT: the client encrypts
 * the query mod t0 and mod t1 (NTT-friendly primes; the paper's 16- and
 * 17-bit limbs) and reconstructs each result in Z_{t0 t1} by the CRT.
 * Returns the centered representative in (-t0 t1 / 2, t0 t1 / 2]: the exact
 * signed dot product when it does not wrap around t0 t1.
 * m0 in [0, t0), m1 in [0, t1); t0, t1 coprime. */
int64_t or_plain_crt_signed(uint32_t m0, uint32_t m1, uint32_t t0, uint32_t t1)
{
    /* x = m0 + t0 * ((m1 - m0) * t0^{-1} mod t1) */
    uint64_t inv = or_invmod(t0 % t1, t1);   /* t1 prime */
    uint64_t k = or_mulmod(or_submod(m1 % t1, m0 % t1, t1), inv, t1);
    uint64_t T = (uint64_t)t0 * t1;
    uint64_t x = (uint64_t)m0 + (uint64_t)t0 * k;   /* in [0, T) */
    return x > T / 2 ? (int64_t)x - (int64_t)T : (int64_t)x;
}

/* Dropping ciphertext LSBs (Cheetah's method with the
 * paper's analysis: c = 2^b c^h + c^l, decryption with 2^b c^h adds
 * e_drop = -c^l (times s for c1)).  Reading S20: the high part is the
 * rounded quotient, c^h = floor((c + 2^(b-1)) / 2^b), so |c^l| <= 2^(b-1).
 * in: canonical residues mod q_0; out: c^h. */
void or_drop_lsb(const uint32_t *c, uint32_t count, uint32_t b, uint32_t *ch)
{
    for (uint32_t i = 0; i < count; i++) {
        uint64_t x = c[i];
        ch[i] = (uint32_t)((x + (b ? (1ull << (b - 1)) : 0)) >> b);
    }
}

/* Invariant noise budget of a single-limb response (decryption
 * is correct while ||e|| < Q/2t; budget log2(Q) - log2(2t) shrinks as noise
 * grows).  nu = max_i |[t * v_i]_{q_0}| (centered); budget =
 * log2(q_0) - 1 - log2(nu).  Positive budget <=> correct decryption. */
double or_noise_budget_q0(uint32_t n, uint32_t q0, uint32_t t, const uint32_t *resp, const int8_t *s)
{
    uint32_t *v = (uint32_t *)malloc(sizeof(uint32_t) * n);
    or_phase_q0(n, q0, resp, s, v);
    uint64_t nu = 0;
    for (uint32_t i = 0; i < n; i++) {
        uint64_t x = or_mulmod(t, v[i], q0);
        uint64_t c = x > q0 / 2 ? q0 - x : x;
        if (c > nu) nu = c;
    }
    free(v);
    if (nu == 0) return log2((double)q0) - 1.0;
    return log2((double)q0) - 1.0 - log2((double)nu);
}

/* The same budget for a fresh L-limb ciphertext (before the switch): CRT
 * the phase c0 + c1*s mod Q exactly, then nu = max |[t * v]_Q|. */
double or_noise_budget_Q(uint32_t n, uint32_t L, const uint32_t *mod, uint32_t t, const uint32_t *ct,
                         const int8_t *s)
{
    uint32_t *sl = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *v = (uint32_t *)malloc(sizeof(uint32_t) * n * L);
    for (uint32_t l = 0; l < L; l++) {
        uint32_t q = mod[l];
        for (uint32_t i = 0; i < n; i++) sl[i] = (uint32_t)or_lift(s[i], q);
        uint32_t *vl = v + (size_t)l * n;
        or_polymul_ntt(ct + ((size_t)L + l) * n, sl, vl, n, q);
        for (uint32_t i = 0; i < n; i++) vl[i] = (uint32_t)or_addmod(vl[i], ct[(size_t)l * n + i], q);
    }
    u128 Q = or_big_Q(mod, L);
    double worst = 0.0;
    for (uint32_t i = 0; i < n; i++) {
        uint32_t r[OR_MAX_LIMBS], tr[OR_MAX_LIMBS];
        for (uint32_t l = 0; l < L; l++) {
            r[l] = v[(size_t)l * n + i];
            tr[l] = (uint32_t)or_mulmod(t, r[l], mod[l]);
        }
        u128 x = or_crt(tr, mod, L);
        u128 c = x > Q / 2 ? Q - x : x;
        double dc = (double)c;
        if (dc > worst) worst = dc;
    }
    free(sl);
    free(v);
    double logQ = 0.0;
    for (uint32_t l = 0; l < L; l++) logQ += log2((double)mod[l]);
    if (worst < 1.0) return logQ - 1.0;
    return logQ - 1.0 - log2(worst);
}

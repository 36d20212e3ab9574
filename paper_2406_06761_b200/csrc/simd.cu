// The SIMD formulation of Wally's server computation (include/wally_simd.h;
// SURVEY.md §8(f)-3; Alg 4):
// diagonal packing + baby-step giant-step rotations with hybrid key
// switching, then the switch to q_0.  Kernels and the host side of the C ABI.
//
//   simd_encode_kernel   a0'  diagonal slots -> inverse NTT mod t (slot encode)
//                             -> centered lift -> forward NTT per limb + Shoup companion
//   simd_ntt_kernel      a2'  forward NTT of query ciphertexts and key polynomials
//   simd_modup_kernel    rot  Galois permutation (NTT domain) + inverse NTT of
//                             one digit + forward NTT into every other modulus
//   simd_moddown_kernel  rot  key products (64-bit accumulation, one Barrett
//                             reduction), ModDown by P, + sigma(c0) (+ addend)
//   simd_ptmac_kernel    a3'  I_j = sum_b pt_{jg+b} (.) baby_b (Shoup, lazy)
//   simd_switch_kernel   a5'  inverse NTT of every limb + drop-last to q_0
//
// All NTT-domain data is stored canonical ([0, q)); the transforms are the
// register-blocked passes of ntt_device.cuh (one CTA of N/V threads per
// polynomial).  NTT index j holds the evaluation at psi^(2 brev(j) + 1), so a
// Galois automorphism X -> X^k is the permutation j -> idx(k E_j mod 2N).

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ntt_device.cuh"
#include "wally_simd.h"
#include "wally_internal.h"

namespace wally {
namespace simd {

constexpr int kMaxMods = WALLY_MAX_LIMBS + 1;
constexpr int kSimdStages = 5;   // wally_simd_stage_times: NTTs, baby steps, inner products, giant steps, switch

struct Mods {
    uint32_t L, M;                        // ciphertext limbs, L + 1 key moduli (index L = P)
    uint32_t q[kMaxMods], q2[kMaxMods];
    uint32_t ninv[kMaxMods], ninvp[kMaxMods];
    uint64_t mu[kMaxMods];                // floor(2^64 / q): Barrett constant of the 64-bit key products
    uint32_t pinv[kMaxMods], pinvp[kMaxMods];   // P^{-1} mod q_i (ModDown)
    uint32_t h[kMaxMods];                 // floor(q_l / 2) (switch rounding)
    uint32_t cinv[kMaxMods][kMaxMods];    // q_l^{-1} mod q_i  (i < l)
    uint32_t cinvp[kMaxMods][kMaxMods];
    uint32_t t, t2, tninv, tninvp;        // plaintext modulus (tables at index M)
};

__device__ __forceinline__ uint32_t red64(uint64_t x, uint32_t q, uint64_t mu) {
    const uint64_t qh = __umul64hi(x, mu);
    return csub((uint32_t)x - (uint32_t)qh * q, q);
}

template <int N>
__device__ __forceinline__ void store_contig(uint32_t *dst, const uint32_t (&a)[1][NttGeom<N>::V], int g) {
    constexpr int V = NttGeom<N>::V;
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + (size_t)g * V);
#pragma unroll
    for (int v = 0; v < V / 4; v++) d4[v] = make_uint4(a[0][4 * v], a[0][4 * v + 1], a[0][4 * v + 2], a[0][4 * v + 3]);
}

template <int N>
__device__ __forceinline__ void load_contig(const uint32_t *src, uint32_t (&a)[NttGeom<N>::V], int g) {
    constexpr int V = NttGeom<N>::V;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src + (size_t)g * V);
#pragma unroll
    for (int v = 0; v < V / 4; v++) {
        const uint4 x = s4[v];
        a[4 * v] = x.x; a[4 * v + 1] = x.y; a[4 * v + 2] = x.z; a[4 * v + 3] = x.w;
    }
}

__device__ __forceinline__ uint2 ldg_stream2(const void *p) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

// [0, 4q) -> [0, q)
__device__ __forceinline__ uint32_t canon4(uint32_t x, uint32_t q, uint32_t q2) { return csub(csub(x, q2), q); }

// ---------------------------------------------------------------------------
// Forward NTT of polynomials p = 0..count-1 (a2'): modulus index p % period;
// input polynomial p at in + sel[p / grp] * in_stride + (p % grp) * N (sel ==
// nullptr: p / grp), output at out + (p / grp) * out_stride + (p % grp) * N;
// residues >= q set err.
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T) simd_ntt_kernel(Mods md, const uint2 *__restrict__ tw, uint32_t period,
                                                                uint32_t grp, const uint32_t *__restrict__ in,
                                                                size_t in_stride, const uint32_t *__restrict__ sel,
                                                                uint32_t *__restrict__ out, size_t out_stride,
                                                                uint32_t *err) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    const int g = threadIdx.x;
    const size_t p = blockIdx.x;
    const uint32_t m = (uint32_t)(p % period);
    const uint32_t q = md.q[m], q2 = md.q2[m];
    const size_t gi = sel ? (size_t)sel[p / grp] : p / grp;    // input group (query) of this polynomial
    const uint32_t *src = in + gi * in_stride + (p % grp) * N;
    uint32_t a[1][V];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < V / Gm::R2; j++)
#pragma unroll
        for (int k = 0; k < Gm::R2; k++) {
            const uint32_t x = __ldg(src + pass_index<N, Gm::TB2, Gm::R2>(g, j, k));
            bad |= (x >= q);
            a[0][j * Gm::R2 + k] = x;
        }
    if (bad) atomicOr(err, 1u);
    ntt_chain<N, 1>(a, tw + (size_t)m * Gm::TW_LIMB, g, q, q2, smem, smem + Gm::SMEM_WORDS);
#pragma unroll
    for (int v = 0; v < V; v++) a[0][v] = canon4(a[0][v], q, q2);
    store_contig<N>(out + (p / grp) * out_stride + (p % grp) * N, a, g);
}

// ---------------------------------------------------------------------------
// ModUp of a rotation (unit u = blockIdx.x, digit j = blockIdx.y):
//   y = sigma(c1)_j  (NTT domain: y[x] = c1_j[perm[x]])   -> ext[u][j][j]
//   c = INTT_j(y) in [0, q_j)                              (the digit D_j)
//   ext[u][j][m] = NTT_m(c mod q_m) for every other modulus m (incl. P)
// X: unit u's ciphertext at X + u * xs, [2][L][N] NTT domain canonical.
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T) simd_modup_kernel(Mods md, const uint2 *__restrict__ twf,
                                                                  const uint2 *__restrict__ twi,
                                                                  const uint32_t *__restrict__ X, size_t xs,
                                                                  const uint32_t *__restrict__ perm,
                                                                  uint32_t *__restrict__ ext) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const uint32_t u = blockIdx.x, j = blockIdx.y, L = md.L, M = md.M;
    const uint32_t *c1 = X + (size_t)u * xs + ((size_t)L + j) * N;
    uint32_t *eu = ext + (size_t)u * L * M * N + (size_t)j * M * N;
    uint32_t a[1][V];
#pragma unroll
    for (int v = 0; v < V; v++) a[0][v] = __ldg(c1 + __ldg(perm + g * V + v));
    store_contig<N>(eu + (size_t)j * N, a, g);
    const uint32_t qj = md.q[j], qj2 = md.q2[j];
#pragma unroll
    for (int v = 0; v < V; v++) a[0][v] = shoup_mul(a[0][v], md.ninv[j], md.ninvp[j], qj);
    intt_chain<N, 1>(a, twi + (size_t)j * Gm::TW_LIMB, g, qj, qj2, bufA, bufB);
    uint32_t c[V];
#pragma unroll
    for (int v = 0; v < V; v++) c[v] = csub(a[0][v], qj);       // pass-2 layout, coefficient form
    for (uint32_t m = 0; m < M; m++) {
        if (m == j) continue;
        const uint32_t q = md.q[m], q2 = md.q2[m];
#pragma unroll
        for (int v = 0; v < V; v++) a[0][v] = csub(c[v], q);    // c < q_j < 2 q_m
        __syncthreads();                                         // exchange buffers reused
        ntt_chain<N, 1>(a, twf + (size_t)m * Gm::TW_LIMB, g, q, q2, bufA, bufB);
#pragma unroll
        for (int v = 0; v < V; v++) a[0][v] = canon4(a[0][v], q, q2);
        store_contig<N>(eu + (size_t)m * N, a, g);
    }
}

// ---------------------------------------------------------------------------
// ModDown of a rotation (unit u = blockIdx.x, component c = blockIdx.y):
//   acc_m = sum_j ext[u][j][m] * key[c][j][m]      (64-bit, one reduction)
//   z     = INTT_P(acc_P) in [0, P)  (P < q_i: already canonical mod q_i)
//   out_i = (acc_i - NTT_i(z)) P^{-1} (+ sigma(c0)_i if c = 0) (+ addend_i)
// Keys of unit u: keys + uq[u] * key_stride (uq == nullptr: u), layout
// [2 comps][L digits][M][N].
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T, 2) simd_moddown_kernel(
    Mods md, const uint2 *__restrict__ twf, const uint2 *__restrict__ twi, const uint32_t *__restrict__ ext,
    const uint32_t *__restrict__ keys, size_t key_stride, const uint32_t *__restrict__ uq,
    const uint32_t *__restrict__ X, size_t xs, const uint32_t *__restrict__ perm, const uint32_t *__restrict__ add,
    size_t as, uint32_t *__restrict__ out, size_t os) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const uint32_t u = blockIdx.x, c = blockIdx.y, L = md.L, M = md.M;
    const uint32_t *eu = ext + (size_t)u * L * M * N;
    const uint32_t *ku = keys + (size_t)(uq ? uq[u] : u) * key_stride + (size_t)c * L * M * N;
    auto mac = [&](uint32_t m, uint32_t (&r)[1][V]) {
        uint64_t s[V];
#pragma unroll
        for (int v = 0; v < V; v++) s[v] = 0;
        for (uint32_t j = 0; j < L; j++) {
            uint32_t e[V], k[V];
            load_contig<N>(eu + ((size_t)j * M + m) * N, e, g);
            load_contig<N>(ku + ((size_t)j * M + m) * N, k, g);
#pragma unroll
            for (int v = 0; v < V; v++) s[v] += (uint64_t)e[v] * k[v];
        }
#pragma unroll
        for (int v = 0; v < V; v++) r[0][v] = red64(s[v], md.q[m], md.mu[m]);
    };
    const uint32_t P = md.q[L], P2 = md.q2[L];
    uint32_t a[1][V];
    mac(L, a);
#pragma unroll
    for (int v = 0; v < V; v++) a[0][v] = shoup_mul(a[0][v], md.ninv[L], md.ninvp[L], P);
    intt_chain<N, 1>(a, twi + (size_t)L * Gm::TW_LIMB, g, P, P2, bufA, bufB);
    uint32_t z[V];
#pragma unroll
    for (int v = 0; v < V; v++) z[v] = csub(a[0][v], P);        // [acc_P]_P, pass-2 layout
    const uint32_t *x0 = X + (size_t)u * xs;
    const uint32_t *ad = add ? add + (size_t)u * as + (size_t)c * L * N : nullptr;
    uint32_t *o = out + (size_t)u * os + (size_t)c * L * N;
    for (uint32_t i = 0; i < L; i++) {
        const uint32_t q = md.q[i], q2 = md.q2[i];
#pragma unroll
        for (int v = 0; v < V; v++) a[0][v] = z[v];
        __syncthreads();
        ntt_chain<N, 1>(a, twf + (size_t)i * Gm::TW_LIMB, g, q, q2, bufA, bufB);
        uint32_t r[1][V];
        mac(i, r);
#pragma unroll
        for (int v = 0; v < V; v++) {
            const uint32_t zi = canon4(a[0][v], q, q2);
            r[0][v] = csub(shoup_mul(r[0][v] + q - zi, md.pinv[i], md.pinvp[i], q), q);
        }
        if (c == 0) {
            const uint32_t *c0 = x0 + (size_t)i * N;
#pragma unroll
            for (int v = 0; v < V; v++) r[0][v] = csub(r[0][v] + __ldg(c0 + __ldg(perm + g * V + v)), q);
        }
        if (ad) {
            uint32_t w[V];
            load_contig<N>(ad + (size_t)i * N, w, g);
#pragma unroll
            for (int v = 0; v < V; v++) r[0][v] = csub(r[0][v] + w[v], q);
        }
        store_contig<N>(o + (size_t)i * N, r, g);
    }
}

// ---------------------------------------------------------------------------
// Inner products of the giant steps (a3'): unit u (query-block) =
// blockIdx.x; each thread owns two coefficients of one limb for both
// components.  I[u][j] = sum_{b < g, jg + b < d} pt[blk][jg + b] (.) baby[q][b].
// pt: values and Shoup companions [blocks][d][L][N].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) simd_ptmac_kernel(Mods md, uint32_t N, uint32_t d, uint32_t g, uint32_t m,
                                                         const uint32_t *__restrict__ baby,
                                                         const uint32_t *__restrict__ uq,
                                                         const uint32_t *__restrict__ ublk,
                                                         const uint32_t *__restrict__ ptv,
                                                         const uint32_t *__restrict__ ptc, uint32_t *__restrict__ I) {
    const uint32_t L = md.L;
    const uint32_t u = blockIdx.x;
    const uint32_t w = (blockIdx.y * blockDim.x + threadIdx.x) * 2;   // word inside [L][N]
    if (w >= L * N) return;
    const uint32_t l = w / N;
    const uint32_t q = md.q[l], q2 = md.q2[l];
    const size_t CT = (size_t)2 * L * N;
    const uint32_t *bq = baby + (size_t)uq[u] * g * CT;
    const size_t pbase = (size_t)ublk[u] * d * L * N + w;
    uint32_t *Iu = I + (size_t)u * m * CT;
    for (uint32_t j = 0; j < m; j++) {
        uint32_t a0x = 0, a0y = 0, a1x = 0, a1y = 0;   // lazy in [0, 2q)
        for (uint32_t b = 0; b < g && j * g + b < d; b++) {
            const size_t pi = pbase + (size_t)(j * g + b) * L * N;
            const uint2 pv = ldg_stream2(ptv + pi);       // plaintexts stream through (L2-shared, not L1)
            const uint2 pc = ldg_stream2(ptc + pi);
            const uint2 x0 = *reinterpret_cast<const uint2 *>(bq + (size_t)b * CT + w);
            const uint2 x1 = *reinterpret_cast<const uint2 *>(bq + (size_t)b * CT + (size_t)L * N + w);
            a0x = csub(a0x + shoup_mul(x0.x, pv.x, pc.x, q), q2);
            a0y = csub(a0y + shoup_mul(x0.y, pv.y, pc.y, q), q2);
            a1x = csub(a1x + shoup_mul(x1.x, pv.x, pc.x, q), q2);
            a1y = csub(a1y + shoup_mul(x1.y, pv.y, pc.y, q), q2);
        }
        *reinterpret_cast<uint2 *>(Iu + (size_t)j * CT + w) = make_uint2(csub(a0x, q), csub(a0y, q));
        *reinterpret_cast<uint2 *>(Iu + (size_t)j * CT + (size_t)L * N + w) = make_uint2(csub(a1x, q), csub(a1y, q));
    }
}


// ---------------------------------------------------------------------------
// A chain of rotations in one CTA per unit (n <= 4096): step s = 1..steps
// computes X_s = rot(X_{s-1}) (+ addend_s) -- the whole key switch of one
// rotation (ModUp, key products, ModDown) without materialising the
// extended digits, and the unit's key is re-read from L2 by every step.
//   X_0   = X0 + u * x0s
//   X_s   = outs[s & 1] + u * out_us + (s - 1) * out_ss
//   add_s = add + u * add_us + (s - 1) * add_ss        (add == nullptr: none)
// Shared memory: the L digits D_j (coefficient form; each thread reads back
// only the elements it wrote) and the two exchange buffers.  Step outputs
// are read back with L1-bypassing loads (another thread wrote them).
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T, 2) simd_rot_chain_kernel(
    Mods md, const uint2 *__restrict__ twf, const uint2 *__restrict__ twi, const uint32_t *__restrict__ perm,
    const uint32_t *__restrict__ keys, size_t key_stride, const uint32_t *__restrict__ uq, const uint32_t *X0,
    size_t x0s, uint32_t *out_even, uint32_t *out_odd, size_t out_us, ptrdiff_t out_ss, const uint32_t *add,
    size_t add_us, ptrdiff_t add_ss, uint32_t steps) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS, *D = smem + 2 * Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const uint32_t u = blockIdx.x, L = md.L, M = md.M;
    const uint32_t P = md.q[L], P2 = md.q2[L];
    const uint32_t *ku = keys + (size_t)(uq ? uq[u] : u) * key_stride;
    const size_t KC = (size_t)L * M * N;                // one key component
    uint32_t pm[V];
#pragma unroll
    for (int v = 0; v < V; v++) pm[v] = __ldg(perm + g * V + v);
    const uint32_t *X = X0 + (size_t)u * x0s;
    for (uint32_t st = 1; st <= steps; st++) {
        uint32_t *Y = ((st & 1) ? out_odd : out_even) + (size_t)u * out_us + (ptrdiff_t)(st - 1) * out_ss;
        const uint32_t *ad = add ? add + (size_t)u * add_us + (ptrdiff_t)(st - 1) * add_ss : nullptr;
        uint32_t a[1][V];
        // ModUp, part 1: digits D_j = INTT_j(sigma(c1)_j)
        for (uint32_t j = 0; j < L; j++) {
            const uint32_t qj = md.q[j], qj2 = md.q2[j];
            const uint32_t *c1 = X + ((size_t)L + j) * N;
#pragma unroll
            for (int v = 0; v < V; v++) a[0][v] = shoup_mul(__ldcg(c1 + pm[v]), md.ninv[j], md.ninvp[j], qj);
            __syncthreads();
            intt_chain<N, 1>(a, twi + (size_t)j * Gm::TW_LIMB, g, qj, qj2, bufA, bufB);
#pragma unroll
            for (int jj = 0; jj < V / Gm::R2; jj++)
#pragma unroll
                for (int k = 0; k < Gm::R2; k++)
                    D[(size_t)j * N + pass_index<N, Gm::TB2, Gm::R2>(g, jj, k)] = csub(a[0][jj * Gm::R2 + k], qj);
        }
        // key products at modulus m: s_c = sum_j ext_j * key[c][j][m]
        auto mac_at = [&](uint32_t m, uint64_t (&s0)[V], uint64_t (&s1)[V]) {
            const uint32_t q = md.q[m], q2 = md.q2[m];
#pragma unroll
            for (int v = 0; v < V; v++) s0[v] = s1[v] = 0;
            for (uint32_t j = 0; j < L; j++) {
                if (j == m) {
                    const uint32_t *c1 = X + ((size_t)L + j) * N;
#pragma unroll
                    for (int v = 0; v < V; v++) a[0][v] = __ldcg(c1 + pm[v]);
                } else {
#pragma unroll
                    for (int jj = 0; jj < V / Gm::R2; jj++)
#pragma unroll
                        for (int k = 0; k < Gm::R2; k++)
                            a[0][jj * Gm::R2 + k] =
                                csub(D[(size_t)j * N + pass_index<N, Gm::TB2, Gm::R2>(g, jj, k)], q);
                    __syncthreads();
                    ntt_chain<N, 1>(a, twf + (size_t)m * Gm::TW_LIMB, g, q, q2, bufA, bufB);
#pragma unroll
                    for (int v = 0; v < V; v++) a[0][v] = canon4(a[0][v], q, q2);
                }
                uint32_t k0[V], k1[V];
                load_contig<N>(ku + ((size_t)j * M + m) * N, k0, g);
                load_contig<N>(ku + KC + ((size_t)j * M + m) * N, k1, g);
#pragma unroll
                for (int v = 0; v < V; v++) {
                    s0[v] += (uint64_t)a[0][v] * k0[v];
                    s1[v] += (uint64_t)a[0][v] * k1[v];
                }
            }
        };
        uint64_t s0[V], s1[V];
        // ModDown, part 1: z_c = INTT_P([acc_c]_P)
        mac_at(L, s0, s1);
        uint32_t z0[V], z1[V];
#pragma unroll
        for (int v = 0; v < V; v++) a[0][v] = shoup_mul(red64(s0[v], P, md.mu[L]), md.ninv[L], md.ninvp[L], P);
        __syncthreads();
        intt_chain<N, 1>(a, twi + (size_t)L * Gm::TW_LIMB, g, P, P2, bufA, bufB);
#pragma unroll
        for (int v = 0; v < V; v++) z0[v] = csub(a[0][v], P);
#pragma unroll
        for (int v = 0; v < V; v++) a[0][v] = shoup_mul(red64(s1[v], P, md.mu[L]), md.ninv[L], md.ninvp[L], P);
        __syncthreads();
        intt_chain<N, 1>(a, twi + (size_t)L * Gm::TW_LIMB, g, P, P2, bufA, bufB);
#pragma unroll
        for (int v = 0; v < V; v++) z1[v] = csub(a[0][v], P);
        // ModDown, part 2, per limb i: out_c,i = (acc_c,i - NTT_i(z_c)) P^{-1} (+ sigma(c0)_i) (+ add)
        for (uint32_t i = 0; i < L; i++) {
            const uint32_t q = md.q[i], q2 = md.q2[i];
            mac_at(i, s0, s1);
            for (int c = 0; c < 2; c++) {
#pragma unroll
                for (int v = 0; v < V; v++) a[0][v] = c ? z1[v] : z0[v];     // z < P < q_i
                __syncthreads();
                ntt_chain<N, 1>(a, twf + (size_t)i * Gm::TW_LIMB, g, q, q2, bufA, bufB);
                uint32_t r[1][V];
#pragma unroll
                for (int v = 0; v < V; v++) {
                    const uint32_t acc = red64(c ? s1[v] : s0[v], q, md.mu[i]);
                    r[0][v] = csub(shoup_mul(acc + q - canon4(a[0][v], q, q2), md.pinv[i], md.pinvp[i], q), q);
                }
                if (c == 0) {
                    const uint32_t *c0 = X + (size_t)i * N;
#pragma unroll
                    for (int v = 0; v < V; v++) r[0][v] = csub(r[0][v] + __ldcg(c0 + pm[v]), q);
                }
                if (ad) {
                    uint32_t w2[V];
                    load_contig<N>(ad + ((size_t)c * L + i) * N, w2, g);
#pragma unroll
                    for (int v = 0; v < V; v++) r[0][v] = csub(r[0][v] + w2[v], q);
                }
                store_contig<N>(Y + ((size_t)c * L + i) * N, r, g);
            }
        }
        __syncthreads();                 // Y complete before the next step gathers from it
        X = Y;
    }
}

// ---------------------------------------------------------------------------
// Switch to q_0 (a5'/a6'): unit u = blockIdx.x, component c = blockIdx.y.
// Every limb is inverse-transformed into shared memory (coefficient order),
// then each coefficient runs the drop-last recurrence l = L-1 .. 1:
//   r = (c_l + floor(q_l/2)) mod q_l;  c_i = (c_i + floor(q_l/2) - r) q_l^{-1} mod q_i
// (round(c q_0 / Q), reading S7), and the q_0 residue is written.
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T) simd_switch_kernel(Mods md, const uint2 *__restrict__ twi,
                                                                   const uint32_t *__restrict__ X, size_t xs,
                                                                   const uint32_t *__restrict__ out_off,
                                                                   uint32_t *__restrict__ resp) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V, T = Gm::T;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS, *coef = smem + 2 * Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const uint32_t u = blockIdx.x, c = blockIdx.y, L = md.L;
    const uint32_t *xu = X + (size_t)u * xs + (size_t)c * L * N;
    for (uint32_t l = 0; l < L; l++) {
        const uint32_t q = md.q[l], q2 = md.q2[l];
        uint32_t a[1][V];
        load_contig<N>(xu + (size_t)l * N, a[0], g);
#pragma unroll
        for (int v = 0; v < V; v++) a[0][v] = shoup_mul(a[0][v], md.ninv[l], md.ninvp[l], q);
        if (l) __syncthreads();
        intt_chain<N, 1>(a, twi + (size_t)l * Gm::TW_LIMB, g, q, q2, bufA, bufB);
#pragma unroll
        for (int j = 0; j < V / Gm::R2; j++)
#pragma unroll
            for (int k = 0; k < Gm::R2; k++)
                coef[(size_t)l * N + pass_index<N, Gm::TB2, Gm::R2>(g, j, k)] = csub(a[0][j * Gm::R2 + k], q);
    }
    __syncthreads();
    uint32_t *o = resp + out_off[u] + (size_t)c * N;
    for (int x = g; x < N; x += T) {
        uint32_t r[kMaxMods];
        for (uint32_t l = 0; l < L; l++) r[l] = coef[(size_t)l * N + x];
        for (int l = (int)L - 1; l >= 1; l--) {
            const uint32_t ql = md.q[l], hl = md.h[l];
            const uint32_t rl = csub(r[l] + hl, ql);
            for (int i = 0; i < l; i++) {
                const uint32_t qi = md.q[i];
                const uint32_t rm = csub(rl, qi);                  // r < q_l < 2 q_i
                const uint32_t hm = csub(hl, qi);
                const uint32_t v = csub(csub(r[i] + hm, qi) + qi - rm, qi);
                r[i] = csub(shoup_mul(v, md.cinv[l][i], md.cinvp[l][i], qi), qi);
            }
        }
        o[x] = r[0];
    }
}

// ---------------------------------------------------------------------------
// ServerInit (a0'): block b = blockIdx.x, diagonal i = blockIdx.y.  NTT index
// j (thread g holds j = g V + v) carries slot slot_of[j]; the slot value is
// the pre-rotated diagonal entry (or 0), mod t.  Inverse NTT mod t gives the
// plaintext coefficients; each limb gets the centered lift, NTT'd.
// ---------------------------------------------------------------------------
struct BlockArgs {
    const int8_t *entries;        // [total entries][d]
    const uint64_t *blk_base;     // first entry of block b
    const uint32_t *blk_count;    // entries in block b
    const uint32_t *slot_of;      // [N]
    uint32_t d, g, R;
    uint32_t *ptv, *ptc;          // [blocks][d][L][N]
};

template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T) simd_encode_kernel(Mods md, const uint2 *__restrict__ twf,
                                                                   const uint2 *__restrict__ twi, BlockArgs ba) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const uint32_t b = blockIdx.x, i = blockIdx.y, L = md.L, M = md.M;
    const uint32_t half = N / 2, d = ba.d;
    const uint32_t jg = (i / ba.g) * ba.g % half;
    const uint64_t base = ba.blk_base[b];
    const uint32_t cnt = ba.blk_count[b];
    const uint32_t t = md.t;
    uint32_t a[1][V];
#pragma unroll
    for (int v = 0; v < V; v++) {
        const uint32_t s = __ldg(ba.slot_of + g * V + v);
        const uint32_t r = s / half, k = s % half;
        const uint32_t kk = (k + half - jg) % half;
        uint32_t val = 0;
        if (kk < ba.R * d) {
            const uint32_t e = (r * ba.R + kk / d) * d + kk % d;
            if (e < cnt) {
                const int x = ba.entries[(base + e) * d + (kk % d + i) % d];
                val = x < 0 ? (uint32_t)((int)t + x) : (uint32_t)x;
            }
        }
        a[0][v] = shoup_mul(val, md.tninv, md.tninvp, t);
    }
    intt_chain<N, 1>(a, twi + (size_t)M * Gm::TW_LIMB, g, t, md.t2, bufA, bufB);
    uint32_t cf[V];
#pragma unroll
    for (int v = 0; v < V; v++) cf[v] = csub(a[0][v], t);    // coefficients mod t, pass-2 layout
    for (uint32_t l = 0; l < L; l++) {
        const uint32_t q = md.q[l], q2 = md.q2[l];
#pragma unroll
        for (int v = 0; v < V; v++) a[0][v] = cf[v] > t / 2 ? q - (t - cf[v]) : cf[v];   // centered lift (S24)
        __syncthreads();
        ntt_chain<N, 1>(a, twf + (size_t)l * Gm::TW_LIMB, g, q, q2, bufA, bufB);
        const size_t off = (((size_t)b * d + i) * L + l) * N + (size_t)g * V;
#pragma unroll
        for (int v = 0; v < V; v++) {
            const uint32_t w = canon4(a[0][v], q, q2);
            ba.ptv[off + v] = w;
            ba.ptc[off + v] = (uint32_t)(((uint64_t)w << 32) / q);
        }
    }
}

template <int N>
constexpr size_t chain_smem() { return 2 * (size_t)NttGeom<N>::SMEM_WORDS * sizeof(uint32_t); }

template <typename K>
static cudaError_t allow(K k, size_t bytes) {
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace simd
}  // namespace wally

using namespace wally;
using namespace wally::simd;

// ===========================================================================
// Host side
// ===========================================================================
struct wally_simd_ctx {
    wally_simd_params p{};
    int device = 0;
    int num_sms = 148;
    uint32_t chain_min_queries = 0;                // fused rotation chain from this many queries per chunk
    uint32_t L = 0, M = 0, g = 0, m = 0, R = 0, logn = 0;
    Mods md{};
    uint2 *d_twf = nullptr, *d_twi = nullptr;      // [M + 1][TW_LIMB] (index M: t)
    uint32_t *d_perm1 = nullptr, *d_permg = nullptr, *d_slot_of = nullptr;
    uint32_t galois[2] = {0, 0};
    // database
    uint32_t n_clusters = 0, total_blocks = 0;
    std::vector<uint32_t> blk_first, blk_num;      // per cluster: first block, block count
    uint32_t *d_ptv = nullptr, *d_ptc = nullptr;
    // workspace
    void *ws = nullptr;
    size_t ws_bytes = 0;
    uint32_t *h_units = nullptr;                   // pinned unit tables, two slots
    size_t h_units_cap = 0;
    cudaEvent_t tab_ev[2] = {nullptr, nullptr};    // upload of a slot completed
    int tab_slot = 0;
    // host-buffer path: staging, copy streams, events
    void *stage = nullptr;
    size_t stage_bytes = 0;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    uint64_t launches = 0;
    // per-stage device timing (wally_simd_enable_stage_timing): kSimdStages + 1
    // events per chunk on the batch's stream
    bool timing = false;
    std::vector<std::vector<cudaEvent_t>> ev_rec;
    std::vector<cudaEvent_t> ev_pool;
    std::string err;
};

static thread_local std::string g_simd_create_err;

static int sfail(wally_simd_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf; else g_simd_create_err = buf;
    return code;
}

#define SCUDA(ctx, call)                                                                                 \
    do {                                                                                                 \
        cudaError_t _e = (call);                                                                         \
        if (_e != cudaSuccess) return sfail(ctx, WALLY_E_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    } while (0)

static uint64_t s_mulm(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((unsigned __int128)a * b % m); }
static uint64_t s_powm(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    for (b %= m; e; e >>= 1, b = s_mulm(b, b, m))
        if (e & 1) r = s_mulm(r, b, m);
    return r;
}
static uint64_t s_invm(uint64_t a, uint64_t m) { return s_powm(a, m - 2, m); }
static bool s_prime(uint64_t n) {
    if (n < 2) return false;
    for (uint64_t d = 2; d * d <= n; d++)
        if (n % d == 0) return false;
    return true;
}
static uint32_t s_shoup(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
static uint32_t s_brev(uint32_t x, uint32_t bits) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}
// Smallest primitive 2n-th root of unity mod q: the least x with x^n = -1 (n a power of two).
static uint64_t s_min_root(uint64_t q, uint32_t n) {
    for (uint64_t x = 2; x < q; x++)
        if (s_powm(x, n, q) == q - 1) return x;
    return 0;
}

// Pass-major tables (layout of ntt_device.cuh) for one modulus with root psi.
template <int N>
static void s_tables(uint64_t q, uint64_t psi, uint2 *fwd, uint2 *inv) {
    using Gm = NttGeom<N>;
    const uint32_t logn = Log2<N>::v;
    const uint64_t psi_inv = s_invm(psi, q);
    std::vector<uint2> pf(N), pi(N);
    for (uint32_t i = 0; i < (uint32_t)N; i++) {
        const uint32_t e = s_brev(i, logn);
        const uint32_t w = (uint32_t)s_powm(psi, e, q), wi = (uint32_t)s_powm(psi_inv, e, q);
        pf[i] = make_uint2(w, s_shoup(w, (uint32_t)q));
        pi[i] = make_uint2(wi, s_shoup(wi, (uint32_t)q));
    }
    const int TB[3] = {Gm::TB0, Gm::TB1, Gm::TB2}, R[3] = {Gm::R0, Gm::R1, Gm::R2};
    const int OFF[3] = {Gm::TW0, Gm::TW1, Gm::TW2};
    for (int p = 0; p < 3; p++) {
        const int H = N / (TB[p] * R[p]);
        int logr = 0;
        while ((1 << logr) < R[p]) logr++;
        auto at = [&](int hi, int slot) -> size_t {
            if (p == 0) return (size_t)OFF[0] + ((size_t)(slot / 2) * Gm::T + hi) * 2 + (slot % 2);
            return (size_t)OFF[p] + (size_t)hi * R[p] + slot;
        };
        for (int hi = 0; hi < H; hi++) {
            for (int k = 0; k < R[p]; k++) inv[at(hi, k)] = fwd[at(hi, k)] = make_uint2(0, 0);
            for (int s = 0; s < logr; s++) {
                const int nb = R[p] >> (s + 1), mm = N / (2 * TB[p] * (1 << s));
                for (int b = 0; b < nb; b++) {
                    inv[at(hi, R[p] - (R[p] >> s) + b)] = pi[mm + hi * nb + b];
                    fwd[at(hi, (R[p] >> (s + 1)) + b)] = pf[mm + hi * nb + b];
                }
            }
        }
    }
}

static size_t s_tw_limb(uint32_t n) {
    switch (n) {
        case 1024: return NttGeom<1024>::TW_LIMB;
        case 2048: return NttGeom<2048>::TW_LIMB;
        case 4096: return NttGeom<4096>::TW_LIMB;
        case 8192: return NttGeom<8192>::TW_LIMB;
    }
    return 0;
}

static void s_build_tables(uint32_t n, uint64_t q, uint64_t psi, uint2 *fwd, uint2 *inv) {
    switch (n) {
        case 1024: s_tables<1024>(q, psi, fwd, inv); break;
        case 2048: s_tables<2048>(q, psi, fwd, inv); break;
        case 4096: s_tables<4096>(q, psi, fwd, inv); break;
        case 8192: s_tables<8192>(q, psi, fwd, inv); break;
    }
}

extern "C" int wally_simd_default_moduli(uint32_t n, uint32_t L, uint32_t *out) {
    if (!out || L < 1 || L > WALLY_MAX_LIMBS || n < 2 || (n & (n - 1)))
        return sfail(nullptr, WALLY_E_ARG, "wally_simd_default_moduli: bad arguments");
    const uint64_t step = 2ull * n;
    std::vector<uint32_t> found;   // descending
    for (uint64_t q = ((1ull << 30) - 2) / step * step + 1; q > (1ull << 29) && found.size() <= L; q -= step)
        if (s_prime(q)) found.push_back((uint32_t)q);
    if (found.size() < L + 1) return sfail(nullptr, WALLY_E_PARAMS, "not enough NTT-friendly primes");
    for (uint32_t i = 0; i < L; i++) out[i] = found[L - 1 - i];
    out[L] = found[L];
    return WALLY_OK;
}

extern "C" const char *wally_simd_last_error(const wally_simd_ctx *ctx) {
    return ctx ? ctx->err.c_str() : g_simd_create_err.c_str();
}

extern "C" void wally_simd_destroy(wally_simd_ctx *c) {
    if (c) {
        for (auto &r : c->ev_rec)
            for (auto e : r) c->ev_pool.push_back(e);
        for (auto e : c->ev_pool) cudaEventDestroy(e);
        c->ev_rec.clear();
        c->ev_pool.clear();
    }
    if (!c) return;
    cudaSetDevice(c->device);
    cudaFree(c->d_twf);
    cudaFree(c->d_twi);
    cudaFree(c->d_perm1);
    cudaFree(c->d_permg);
    cudaFree(c->d_slot_of);
    cudaFree(c->d_ptv);
    cudaFree(c->d_ptc);
    cudaDeviceSynchronize();
    cudaFree(c->ws);
    cudaFree(c->stage);
    cudaFreeHost(c->h_units);
    for (int k = 0; k < 2; k++) {
        if (c->tab_ev[k]) cudaEventDestroy(c->tab_ev[k]);
        if (c->ev_in[k]) cudaEventDestroy(c->ev_in[k]);
        if (c->ev_done[k]) cudaEventDestroy(c->ev_done[k]);
        if (c->ev_out[k]) cudaEventDestroy(c->ev_out[k]);
    }
    if (c->h2d) cudaStreamDestroy(c->h2d);
    if (c->d2h) cudaStreamDestroy(c->d2h);
    delete c;
}

extern "C" int wally_simd_create(const wally_simd_params *params, int device, wally_simd_ctx **out) {
    if (!params || !out) return sfail(nullptr, WALLY_E_ARG, "wally_simd_create: null argument");
    *out = nullptr;
    const wally_simd_params &p = *params;
    const uint32_t n = p.n, L = p.num_limbs;
    if (s_tw_limb(n) == 0) return sfail(nullptr, WALLY_E_PARAMS, "n = %u unsupported (1024, 2048, 4096, 8192)", n);
    if (L < 1 || L > WALLY_MAX_LIMBS) return sfail(nullptr, WALLY_E_PARAMS, "num_limbs = %u unsupported", L);
    if (p.d < 1 || p.d > n / 2) return sfail(nullptr, WALLY_E_PARAMS, "d = %u must be in [1, n/2]", p.d);
    if (p.t >= (1u << 30) || !s_prime(p.t) || (p.t - 1) % (2 * n) != 0)
        return sfail(nullptr, WALLY_E_PARAMS, "t = %u must be a prime = 1 mod 2n below 2^30", p.t);
    for (uint32_t i = 0; i <= L; i++) {
        const uint32_t q = p.moduli[i];
        if (q >= (1u << 30) || q < (1u << 29) || !s_prime(q) || (q - 1) % (2 * n) != 0)
            return sfail(nullptr, WALLY_E_PARAMS, "modulus %u = %u is not an NTT-friendly prime in (2^29, 2^30)", i, q);
        for (uint32_t k = 0; k < i; k++)
            if (p.moduli[k] == q) return sfail(nullptr, WALLY_E_PARAMS, "moduli must be distinct");
        if (i > 0 && i < L && q <= p.moduli[i - 1]) return sfail(nullptr, WALLY_E_PARAMS, "ciphertext moduli must ascend");
    }
    if (p.moduli[L] >= p.moduli[0]) return sfail(nullptr, WALLY_E_PARAMS, "the special prime must be below q_0");
    const uint32_t g = p.baby ? p.baby : (uint32_t)std::ceil(std::sqrt((double)p.d) - 1e-9);
    if (g < 1 || g > p.d) return sfail(nullptr, WALLY_E_PARAMS, "baby = %u must be in [1, d]", g);
    if (cudaSetDevice(device) != cudaSuccess) return sfail(nullptr, WALLY_E_CUDA, "cudaSetDevice(%d) failed", device);

    wally_simd_ctx *c = new wally_simd_ctx();
    c->p = p;
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    c->chain_min_queries = 2u * (uint32_t)c->num_sms;
    c->L = L;
    c->M = L + 1;
    c->g = g;
    c->m = (p.d + g - 1) / g;
    const uint32_t half = n / 2;
    c->R = (half % p.d == 0) ? half / p.d : (half + 1) / p.d - 1;
    uint32_t logn = 0;
    while ((1u << logn) < n) logn++;
    c->logn = logn;
    Mods &md = c->md;
    md.L = L;
    md.M = L + 1;
    const uint64_t P = p.moduli[L];
    for (uint32_t i = 0; i <= L; i++) {
        const uint64_t q = p.moduli[i];
        md.q[i] = (uint32_t)q;
        md.q2[i] = (uint32_t)(2 * q);
        md.ninv[i] = (uint32_t)s_invm(n, q);
        md.ninvp[i] = s_shoup(md.ninv[i], (uint32_t)q);
        md.mu[i] = ~0ull / q;
        md.h[i] = (uint32_t)(q / 2);
        if (i < L) {
            md.pinv[i] = (uint32_t)s_invm(P % q, q);
            md.pinvp[i] = s_shoup(md.pinv[i], (uint32_t)q);
        }
    }
    for (uint32_t l = 1; l < L; l++)
        for (uint32_t i = 0; i < l; i++) {
            md.cinv[l][i] = (uint32_t)s_invm(p.moduli[l] % p.moduli[i], p.moduli[i]);
            md.cinvp[l][i] = s_shoup(md.cinv[l][i], p.moduli[i]);
        }
    md.t = p.t;
    md.t2 = 2 * p.t;
    md.tninv = (uint32_t)s_invm(n, p.t);
    md.tninvp = s_shoup(md.tninv, p.t);

    // tables: M ciphertext/key moduli (any primitive root), then t with the
    // smallest primitive 2n-th root (it defines the slot order, reading S22)
    const size_t twl = s_tw_limb(n);
    std::vector<uint2> twf((size_t)(c->M + 1) * twl), twi((size_t)(c->M + 1) * twl);
    for (uint32_t i = 0; i <= c->M; i++) {
        const uint64_t q = i < c->M ? p.moduli[i] : p.t;
        s_build_tables(n, q, s_min_root(q, n), twf.data() + i * twl, twi.data() + i * twl);
    }
    // NTT index j holds the evaluation at psi^{E_j}, E_j = 2 brev(j) + 1
    std::vector<uint32_t> idx_of_exp(2 * n, 0), exp_of(n);
    for (uint32_t j = 0; j < n; j++) {
        exp_of[j] = 2 * s_brev(j, logn) + 1;
        idx_of_exp[exp_of[j]] = j;
    }
    c->galois[0] = 5 % (2 * n);
    c->galois[1] = (uint32_t)s_powm(5, g, 2 * n);
    std::vector<uint32_t> perm1(n), permg(n), slot_of(n), slot_of_exp(2 * n, 0);
    for (uint32_t j = 0; j < n; j++) {
        perm1[j] = idx_of_exp[(uint64_t)c->galois[0] * exp_of[j] % (2 * n)];
        permg[j] = idx_of_exp[(uint64_t)c->galois[1] * exp_of[j] % (2 * n)];
    }
    for (uint32_t s = 0; s < n; s++) {    // slot s = (row r, column k): exponent 5^k or -5^k
        const uint32_t r = s / half, k = s % half;
        const uint64_t e = s_powm(5, k, 2 * n);
        slot_of_exp[r ? 2 * n - e : e] = s;
    }
    for (uint32_t j = 0; j < n; j++) slot_of[j] = slot_of_exp[exp_of[j]];
    const size_t tb = sizeof(uint2) * twf.size();
    if (cudaMalloc(&c->d_twf, tb) != cudaSuccess || cudaMalloc(&c->d_twi, tb) != cudaSuccess ||
        cudaMalloc(&c->d_perm1, 4 * n) != cudaSuccess || cudaMalloc(&c->d_permg, 4 * n) != cudaSuccess ||
        cudaMalloc(&c->d_slot_of, 4 * n) != cudaSuccess) {
        wally_simd_destroy(c);
        return sfail(nullptr, WALLY_E_OOM, "table allocation failed");
    }
    cudaMemcpy(c->d_twf, twf.data(), tb, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_twi, twi.data(), tb, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_perm1, perm1.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_permg, permg.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_slot_of, slot_of.data(), 4 * n, cudaMemcpyHostToDevice);
    if (cudaGetLastError() != cudaSuccess) {
        wally_simd_destroy(c);
        return sfail(nullptr, WALLY_E_CUDA, "table upload failed");
    }
    *out = c;
    return WALLY_OK;
}

extern "C" int wally_simd_get_info(const wally_simd_ctx *c, wally_simd_info *info) {
    if (!c || !info) return WALLY_E_ARG;
    info->row_slices = c->R;
    info->block_entries = 2 * c->R * c->p.d;
    info->baby = c->g;
    info->giant = c->m;
    info->galois[0] = c->galois[0];
    info->galois[1] = c->galois[1];
    info->key_words = (uint64_t)2 * 2 * c->L * c->M * c->p.n;
    return WALLY_OK;
}

extern "C" uint32_t wally_simd_blocks(const wally_simd_ctx *c, uint32_t cluster) {
    if (!c || cluster >= c->n_clusters) return 0;
    return c->blk_num[cluster];
}

extern "C" uint64_t wally_simd_launch_count(const wally_simd_ctx *c) { return c ? c->launches : 0; }

extern "C" int wally_simd_set_chain_threshold(wally_simd_ctx *c, uint32_t min_queries) {
    if (!c) return WALLY_E_ARG;
    c->chain_min_queries = min_queries;
    return WALLY_OK;
}

// Algorithmic modmuls of one NTT of length n: (n/2) log2 n butterflies.
static uint64_t s_ntt_mm(const wally_simd_ctx *c) { return (uint64_t)(c->p.n / 2) * c->logn; }

extern "C" int wally_simd_enable_stage_timing(wally_simd_ctx *c, int enable) {
    if (!c) return WALLY_E_ARG;
    c->timing = enable != 0;
    return WALLY_OK;
}

extern "C" int wally_simd_stage_times(wally_simd_ctx *c, double *ms, uint64_t *chunks) {
    if (!c || !ms) return WALLY_E_ARG;
    SCUDA(c, cudaSetDevice(c->device));
    for (int i = 0; i < kSimdStages; i++) ms[i] = 0.0;
    for (auto &r : c->ev_rec) {
        SCUDA(c, cudaEventSynchronize(r[kSimdStages]));
        for (int i = 0; i < kSimdStages; i++) {
            float t = 0.f;
            SCUDA(c, cudaEventElapsedTime(&t, r[i], r[i + 1]));
            ms[i] += t;
        }
    }
    if (chunks) *chunks = c->ev_rec.size();
    for (auto &r : c->ev_rec)
        for (auto e : r) c->ev_pool.push_back(e);
    c->ev_rec.clear();
    return WALLY_OK;
}

extern "C" int wally_simd_stage_work(const wally_simd_ctx *c, uint32_t nq, const uint32_t *ids, uint64_t *mm,
                                     uint64_t *bytes) {
    if (!c || !mm || !bytes || (nq && !ids)) return WALLY_E_ARG;
    const uint64_t n = c->p.n, L = c->L, M = c->M, T = s_ntt_mm(c), d = c->p.d, g = c->g, m = c->m;
    const uint64_t ks = L * (n + T + L * T) + 2 * (L * M * n + n + T + L * T + L * n);
    const uint64_t ct = 2 * L * n * 4, key = 2 * 2 * L * M * n * 4;   // bytes of one ciphertext / key pair
    uint64_t blocks = 0, distinct = 0;   // units (query, block); distinct blocks of the batch
    std::vector<char> seen(c->n_clusters, 0);
    for (uint32_t q = 0; q < nq; q++) {
        if (ids[q] >= c->n_clusters) return WALLY_E_ARG;
        blocks += c->blk_num[ids[q]];
        if (!seen[ids[q]]) {
            seen[ids[q]] = 1;
            distinct += c->blk_num[ids[q]];
        }
    }
    for (int i = 0; i < kSimdStages; i++) mm[i] = bytes[i] = 0;
    mm[0] = nq * (2 * L * T + 2 * 2 * L * M * T);
    bytes[0] = nq * 2 * (ct + key);                                  // read + write in place of the NTT domain
    mm[1] = nq * (g - 1) * ks;
    bytes[1] = nq * (key / 2 + g * ct);                              // sigma_5 key, baby_0 in, g - 1 rotations out
    mm[2] = blocks * d * 2 * L * n;
    bytes[2] = distinct * d * L * n * 8 + blocks * (g * ct + m * ct);   // plaintexts + companions once, baby steps, I_j
    mm[3] = blocks * (m - 1) * ks;
    bytes[3] = blocks * (m * ct) + nq * key / 2;                     // I_j in, accumulator out; sigma_{5^g} key
    mm[4] = blocks * 2 * (L * (n + T) + n * L * (L - 1) / 2);
    bytes[4] = blocks * (ct + 2 * n * 4);
    return WALLY_OK;
}

extern "C" uint64_t wally_simd_modmuls_per_query(const wally_simd_ctx *c, uint32_t blocks) {
    if (!c) return 0;
    const uint64_t n = c->p.n, L = c->L, M = c->M, T = s_ntt_mm(c);
    // one key switch: ModUp (L digits: scale + INTT + L NTTs), ModDown (2 comps:
    // L*M key products, scale + INTT_P, L NTTs, L P^{-1} products)
    const uint64_t ks = L * (n + T + L * T) + 2 * (L * M * n + n + T + L * T + L * n);
    const uint64_t per_query = 2 * L * T + 2 * 2 * L * M * T + (uint64_t)(c->g - 1) * ks;   // NTT of ct + keys
    const uint64_t per_block = (uint64_t)c->p.d * 2 * L * n + (uint64_t)(c->m - 1) * ks +
                               2 * (L * (n + T) + n * L * (L - 1) / 2);                    // inner products, giant, switch
    return per_query + (uint64_t)blocks * per_block;
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
template <int N>
static cudaError_t launch_ntt(wally_simd_ctx *c, uint32_t period, uint32_t grp, const uint32_t *in, size_t in_stride,
                              const uint32_t *sel, uint32_t *out, size_t out_stride, size_t count, uint32_t *err,
                              cudaStream_t s) {
    static DeviceOnce once;
    if (cudaError_t e = device_once(once, [&](int *) { return allow(simd_ntt_kernel<N>, chain_smem<N>()); })) return e;
    if (!count) return cudaSuccess;
    simd_ntt_kernel<N><<<(unsigned)count, NttGeom<N>::T, chain_smem<N>(), s>>>(c->md, c->d_twf, period, grp, in,
                                                                              in_stride, sel, out, out_stride, err);
    c->launches++;
    return cudaGetLastError();
}

template <int N>
static cudaError_t launch_rotate(wally_simd_ctx *c, uint32_t units, const uint32_t *X, size_t xs, bool giant,
                                 uint32_t *ext, const uint32_t *keys, size_t key_stride, const uint32_t *uq,
                                 const uint32_t *add, size_t as, uint32_t *out, size_t os, cudaStream_t s) {
    static DeviceOnce once;
    if (cudaError_t e = device_once(once, [&](int *) {
            cudaError_t r = allow(simd_modup_kernel<N>, chain_smem<N>());
            return r ? r : allow(simd_moddown_kernel<N>, chain_smem<N>());
        }))
        return e;
    if (!units) return cudaSuccess;
    const uint32_t *perm = giant ? c->d_permg : c->d_perm1;
    simd_modup_kernel<N><<<dim3(units, c->L), NttGeom<N>::T, chain_smem<N>(), s>>>(c->md, c->d_twf, c->d_twi, X, xs,
                                                                                   perm, ext);
    simd_moddown_kernel<N><<<dim3(units, 2), NttGeom<N>::T, chain_smem<N>(), s>>>(
        c->md, c->d_twf, c->d_twi, ext, keys, key_stride, uq, X, xs, perm, add, as, out, os);
    c->launches += 2;
    return cudaGetLastError();
}

template <int N>
static size_t chain_kernel_smem(uint32_t L) { return chain_smem<N>() + (size_t)L * N * sizeof(uint32_t); }

template <int N>
static cudaError_t launch_chain(wally_simd_ctx *c, uint32_t units, bool giant, const uint32_t *keys, size_t key_stride,
                                const uint32_t *uq, const uint32_t *X0, size_t x0s, uint32_t *out_even,
                                uint32_t *out_odd, size_t out_us, ptrdiff_t out_ss, const uint32_t *add, size_t add_us,
                                ptrdiff_t add_ss, uint32_t steps, cudaStream_t s) {
    if constexpr (N > 4096) {
        return cudaErrorNotSupported;
    } else {
        static DeviceOnce once;
        if (cudaError_t e = device_once(once, [&](int *) {
                return allow(simd_rot_chain_kernel<N>, chain_kernel_smem<N>(WALLY_MAX_LIMBS));
            }))
            return e;
        if (!units || !steps) return cudaSuccess;
        simd_rot_chain_kernel<N><<<units, NttGeom<N>::T, chain_kernel_smem<N>(c->L), s>>>(
            c->md, c->d_twf, c->d_twi, giant ? c->d_permg : c->d_perm1, keys, key_stride, uq, X0, x0s, out_even,
            out_odd, out_us, out_ss, add, add_us, add_ss, steps);
        c->launches++;
        return cudaGetLastError();
    }
}

static cudaError_t launch_ptmac(wally_simd_ctx *c, uint32_t U, const uint32_t *baby, const uint32_t *uq,
                                const uint32_t *ublk, uint32_t *I, cudaStream_t s) {
    const uint32_t n = c->p.n, thr = 256, words = c->L * n / 2;
    const dim3 grid(U, (words + thr - 1) / thr);
    simd_ptmac_kernel<<<grid, thr, 0, s>>>(c->md, n, c->p.d, c->g, c->m, baby, uq, ublk, c->d_ptv, c->d_ptc, I);
    c->launches++;
    return cudaGetLastError();
}

template <int N>
static cudaError_t launch_switch(wally_simd_ctx *c, uint32_t units, const uint32_t *X, size_t xs,
                                 const uint32_t *out_off, uint32_t *resp, cudaStream_t s) {
    const size_t smem = chain_smem<N>() + (size_t)c->L * N * sizeof(uint32_t);
    static DeviceOnce once;
    if (cudaError_t e = device_once(once, [&](int *) { return allow(simd_switch_kernel<N>, chain_smem<N>() + (size_t)WALLY_MAX_LIMBS * N * 4); })) return e;
    if (!units) return cudaSuccess;
    simd_switch_kernel<N><<<dim3(units, 2), NttGeom<N>::T, smem, s>>>(c->md, c->d_twi, X, xs, out_off, resp);
    c->launches++;
    return cudaGetLastError();
}

template <int N>
static cudaError_t launch_encode(wally_simd_ctx *c, const BlockArgs &ba, uint32_t blocks, cudaStream_t s) {
    static DeviceOnce once;
    if (cudaError_t e = device_once(once, [&](int *) { return allow(simd_encode_kernel<N>, chain_smem<N>()); })) return e;
    if (!blocks) return cudaSuccess;
    simd_encode_kernel<N><<<dim3(blocks, c->p.d), NttGeom<N>::T, chain_smem<N>(), s>>>(c->md, c->d_twf, c->d_twi, ba);
    c->launches++;
    return cudaGetLastError();
}

#define SIMD_DISPATCH(n, call)                        \
    switch (n) {                                      \
        case 1024: { constexpr int N = 1024; call; } break; \
        case 2048: { constexpr int N = 2048; call; } break; \
        case 4096: { constexpr int N = 4096; call; } break; \
        case 8192: { constexpr int N = 8192; call; } break; \
    }

extern "C" int wally_simd_load_clusters(wally_simd_ctx *c, uint32_t n_clusters, const uint32_t *sizes,
                                        const int8_t *entries, void *stream) {
    if (!c) return WALLY_E_ARG;
    if (n_clusters && (!sizes || !entries)) return sfail(c, WALLY_E_ARG, "load_clusters: null sizes / entries");
    SCUDA(c, cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t per = 2 * c->R * c->p.d, d = c->p.d;
    std::vector<uint32_t> first(n_clusters), num(n_clusters);
    std::vector<uint64_t> base;
    std::vector<uint32_t> count;
    uint64_t ent = 0;
    for (uint32_t k = 0; k < n_clusters; k++) {
        first[k] = (uint32_t)base.size();
        num[k] = (sizes[k] + per - 1) / per;
        for (uint32_t b = 0; b < num[k]; b++) {
            base.push_back(ent + (uint64_t)b * per);
            count.push_back(std::min<uint32_t>(per, sizes[k] - b * per));
        }
        ent += sizes[k];
    }
    const uint32_t blocks = (uint32_t)base.size();
    const size_t pt_words = (size_t)blocks * d * c->L * c->p.n;
    cudaFree(c->d_ptv);
    cudaFree(c->d_ptc);
    c->d_ptv = c->d_ptc = nullptr;
    c->n_clusters = 0;
    c->total_blocks = 0;
    int8_t *d_ent = nullptr;
    uint64_t *d_base = nullptr;
    uint32_t *d_count = nullptr;
    if (blocks) {
        if (cudaMalloc(&c->d_ptv, pt_words * 4) != cudaSuccess || cudaMalloc(&c->d_ptc, pt_words * 4) != cudaSuccess)
            return sfail(c, WALLY_E_OOM, "plaintext store (%zu words) allocation failed", 2 * pt_words);
        SCUDA(c, cudaMalloc(&d_ent, std::max<uint64_t>(ent * d, 1)));
        SCUDA(c, cudaMalloc(&d_base, 8 * blocks));
        SCUDA(c, cudaMalloc(&d_count, 4 * blocks));
        SCUDA(c, cudaMemcpyAsync(d_ent, entries, ent * d, cudaMemcpyHostToDevice, s));
        SCUDA(c, cudaMemcpyAsync(d_base, base.data(), 8 * blocks, cudaMemcpyHostToDevice, s));
        SCUDA(c, cudaMemcpyAsync(d_count, count.data(), 4 * blocks, cudaMemcpyHostToDevice, s));
        BlockArgs ba{d_ent, d_base, d_count, c->d_slot_of, d, c->g, c->R, c->d_ptv, c->d_ptc};
        cudaError_t e = cudaSuccess;
        SIMD_DISPATCH(c->p.n, e = launch_encode<N>(c, ba, blocks, s));
        if (e != cudaSuccess) return sfail(c, WALLY_E_CUDA, "encode launch: %s", cudaGetErrorString(e));
        SCUDA(c, cudaStreamSynchronize(s));
        cudaFree(d_ent);
        cudaFree(d_base);
        cudaFree(d_count);
    }
    c->blk_first = first;
    c->blk_num = num;
    c->n_clusters = n_clusters;
    c->total_blocks = blocks;
    return WALLY_OK;
}

#ifndef WALLY_SIMD_CHAIN
#define WALLY_SIMD_CHAIN 1
#endif
#ifndef WALLY_SIMD_CHUNK
#define WALLY_SIMD_CHUNK 2048   // queries per chunk at n = 4096 (scaled by 4096 / n)
#endif

// The fused rotation chain runs one CTA per query (per block in the giant
// steps); a batch with fewer queries than two per SM would leave most SMs
// idle, so it uses the separate ModUp (L CTAs) / ModDown (2 CTAs) kernels.
static bool simd_fused(const wally_simd_ctx *c, uint32_t nq) {
    return WALLY_SIMD_CHAIN && c->p.n <= 4096 && nq >= c->chain_min_queries;
}

// Response offsets (words) of a batch in input order; validates the ids.
static int simd_offsets(wally_simd_ctx *c, uint32_t nq, const uint32_t *ids, std::vector<uint64_t> &off) {
    off.assign(nq + 1, 0);
    uint64_t total_blocks = 0;
    for (uint32_t q = 0; q < nq; q++) {
        if (ids[q] >= c->n_clusters)
            return sfail(c, WALLY_E_UNKNOWN_CLUSTER, "query %u names cluster %u (loaded: %u)", q, ids[q], c->n_clusters);
        off[q] = total_blocks * 2 * c->p.n;
        total_blocks += c->blk_num[ids[q]];
    }
    off[nq] = total_blocks * 2 * c->p.n;
    return WALLY_OK;
}

// Workspace of the computation for batches of up to Qc queries / Uc units:
// err word first, then baby [Qc][g][CT], keys [Qc][KW], ext [max(Qc,Uc)][EXT]
// (n = 8192), I [Uc][m][CT], acc 2 x [Uc][CT], device unit tables.  Pinned
// unit tables: two slots, each reused once its upload has completed.
struct SimdWs {
    uint32_t Qc, Uc;
    uint32_t *err, *baby, *keyN, *ext, *I, *accA, *accB, *uq, *ublk, *uoff, *sel;
    size_t w_tab;
};

static int simd_workspace(wally_simd_ctx *c, uint32_t nq, uint32_t max_blk, SimdWs &W) {
    const uint32_t n = c->p.n, L = c->L, M = c->M, g = c->g, m = c->m;
    const size_t CT = (size_t)2 * L * n, KW = (size_t)2 * 2 * L * M * n, EXT = (size_t)L * M * n;
    W.Qc = std::min<uint32_t>(std::max<uint32_t>(nq, 1), std::max<uint32_t>(1, (uint32_t)((WALLY_SIMD_CHUNK * 4096ull) / n)));
    W.Uc = W.Qc * max_blk;
    const bool fused = simd_fused(c, W.Qc);
    const size_t w_baby = (size_t)W.Qc * g * CT, w_key = (size_t)W.Qc * KW;
    const size_t w_ext = fused ? 0 : (size_t)std::max(W.Qc, W.Uc) * EXT;
    const size_t w_I = (size_t)W.Uc * m * CT, w_acc = (size_t)W.Uc * CT;
    W.w_tab = 3 * (size_t)W.Uc + W.Qc;
    const size_t need = 4 * (64 + w_baby + w_key + w_ext + w_I + 2 * w_acc + W.w_tab);
    if (c->ws_bytes < need) {
        cudaFree(c->ws);
        c->ws = nullptr;
        c->ws_bytes = 0;
        if (cudaMalloc(&c->ws, need) != cudaSuccess) return sfail(c, WALLY_E_OOM, "workspace (%zu bytes)", need);
        c->ws_bytes = need;
    }
    if (c->h_units_cap < W.w_tab) {
        for (auto &ev : c->tab_ev)
            if (ev) cudaEventSynchronize(ev);
        cudaFreeHost(c->h_units);
        c->h_units = nullptr;
        SCUDA(c, cudaMallocHost(&c->h_units, 2 * 4 * W.w_tab));
        c->h_units_cap = W.w_tab;
    }
    for (auto &ev : c->tab_ev)
        if (!ev) SCUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    uint32_t *w = (uint32_t *)c->ws;
    W.err = w;
    W.baby = w + 64;
    W.keyN = W.baby + w_baby;
    W.ext = W.keyN + w_key;
    W.I = W.ext + w_ext;
    W.accA = W.I + w_I;
    W.accB = W.accA + w_acc;
    W.uq = W.accB + w_acc;
    W.ublk = W.uq + W.Uc;
    W.uoff = W.ublk + W.Uc;
    W.sel = W.uoff + W.Uc;
    return WALLY_OK;
}

// The server computation of nq queries whose inputs are on the device;
// off: response offsets (words, input order) relative to resp.  Everything
// is stream-ordered on s; no host synchronisation except the reuse of a
// pinned table slot.
static int simd_eval_core(wally_simd_ctx *c, const SimdWs &W, uint32_t nq, const uint32_t *ids,
                          const uint32_t *query_ct, const uint32_t *keys, uint32_t *resp, const uint64_t *off,
                          cudaStream_t s) {
    const uint32_t n = c->p.n, L = c->L, M = c->M, g = c->g, m = c->m;
    const size_t CT = (size_t)2 * L * n, KW = (size_t)2 * 2 * L * M * n;
    const bool fused = simd_fused(c, W.Qc);
    const uint32_t Qc = W.Qc, Uc = W.Uc;
    // queries are processed in cluster order (stable), so the units sharing a
    // block's plaintexts are adjacent; responses stay in input order
    std::vector<uint32_t> order(nq);
    for (uint32_t q = 0; q < nq; q++) order[q] = q;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return ids[a] < ids[b]; });
    uint32_t *baby = W.baby, *keyN = W.keyN, *ext = W.ext, *I = W.I, *accA = W.accA, *accB = W.accB;
    cudaError_t e = cudaSuccess;
    std::vector<cudaEvent_t> *evr = nullptr;   // stage boundaries of the current chunk (timing on)
    auto mark = [&](int i) -> cudaError_t { return evr ? cudaEventRecord((*evr)[i], s) : cudaSuccess; };
    for (uint32_t q0 = 0; q0 < nq; q0 += Qc) {
        const uint32_t nc = std::min(Qc, nq - q0);
        if (c->timing) {
            std::vector<cudaEvent_t> r(kSimdStages + 1);
            for (auto &ev : r) {
                if (c->ev_pool.empty()) {
                    SCUDA(c, cudaEventCreate(&ev));
                } else {
                    ev = c->ev_pool.back();
                    c->ev_pool.pop_back();
                }
            }
            c->ev_rec.push_back(std::move(r));
            evr = &c->ev_rec.back();
        }
        // unit tables of this chunk: a pinned slot whose previous upload has completed
        const int slot = c->tab_slot;
        c->tab_slot ^= 1;
        SCUDA(c, cudaEventSynchronize(c->tab_ev[slot]));
        uint32_t U = 0;
        uint32_t *hq = c->h_units + slot * W.w_tab, *hb = hq + Uc, *ho = hb + Uc, *hs = ho + Uc;
        for (uint32_t q = 0; q < nc; q++) {
            const uint32_t qi = order[q0 + q], cl = ids[qi];
            hs[q] = qi;
            for (uint32_t b = 0; b < c->blk_num[cl]; b++, U++) {
                hq[U] = q;
                hb[U] = c->blk_first[cl] + b;
                const uint64_t o = off[qi] + (uint64_t)b * 2 * n;
                if (o > 0xffffffffull) return sfail(c, WALLY_E_ARG, "response offset beyond 2^32 words: batch too large");
                ho[U] = (uint32_t)o;
            }
        }
        SCUDA(c, cudaMemcpyAsync(W.uq, hq, 4 * W.w_tab, cudaMemcpyHostToDevice, s));
        SCUDA(c, cudaEventRecord(c->tab_ev[slot], s));
        const size_t gCT = (size_t)g * CT;
        SCUDA(c, mark(0));
        // a2': NTT of the chunk's ciphertexts (-> baby_0) and keys
        SIMD_DISPATCH(n, e = launch_ntt<N>(c, L, 2 * L, query_ct, CT, W.sel, baby, gCT, (size_t)nc * 2 * L, W.err, s));
        if (e) break;
        SIMD_DISPATCH(n, e = launch_ntt<N>(c, M, 2 * 2 * L * M, keys, KW, W.sel, keyN, KW,
                                           (size_t)nc * 2 * 2 * L * M, W.err, s));
        if (e) break;
        SCUDA(c, mark(1));
        // baby steps: baby_b = rot_1(baby_{b-1})
        if (fused) {
            SIMD_DISPATCH(n, e = launch_chain<N>(c, nc, false, keyN, KW, nullptr, baby, gCT, baby + CT, baby + CT, gCT,
                                                 (ptrdiff_t)CT, nullptr, 0, 0, g - 1, s));
        } else {
            for (uint32_t b = 1; b < g && !e; b++)
                SIMD_DISPATCH(n, e = launch_rotate<N>(c, nc, baby + (size_t)(b - 1) * CT, gCT, false, ext, keyN, KW,
                                                      nullptr, nullptr, 0, baby + (size_t)b * CT, gCT, s));
        }
        if (e) break;
        SCUDA(c, mark(2));
        // inner products I_j per unit
        e = launch_ptmac(c, U, baby, W.uq, W.ublk, I, s);
        if (e) break;
        SCUDA(c, mark(3));
        // giant steps (Horner): acc = I_{m-1}; acc = rot_g(acc) + I_j, j = m-2 .. 0
        const uint32_t *X = I + (size_t)(m - 1) * CT;
        size_t xs = (size_t)m * CT;
        if (fused && m > 1) {
            SIMD_DISPATCH(n, e = launch_chain<N>(c, U, true, keyN + KW / 2, KW, W.uq, X, xs, accB, accA, CT, 0,
                                                 I + (size_t)(m - 2) * CT, (size_t)m * CT, -(ptrdiff_t)CT, m - 1, s));
            X = ((m - 1) & 1) ? accA : accB;
            xs = CT;
        } else {
            uint32_t *Y = accA;
            for (int j = (int)m - 2; j >= 0 && !e; j--) {
                SIMD_DISPATCH(n, e = launch_rotate<N>(c, U, X, xs, true, ext, keyN + KW / 2, KW, W.uq,
                                                      I + (size_t)j * CT, (size_t)m * CT, Y, CT, s));
                X = Y;
                xs = CT;
                Y = (Y == accA) ? accB : accA;
            }
        }
        if (e) break;
        SCUDA(c, mark(4));
        SIMD_DISPATCH(n, e = launch_switch<N>(c, U, X, xs, W.uoff, resp, s));
        if (e) break;
        SCUDA(c, mark(5));
    }
    if (e) return sfail(c, WALLY_E_CUDA, "eval launch: %s", cudaGetErrorString(e));
    return WALLY_OK;
}

static uint32_t simd_max_blocks(const wally_simd_ctx *c, uint32_t nq, const uint32_t *ids) {
    uint32_t mb = 1;
    for (uint32_t q = 0; q < nq; q++) mb = std::max(mb, c->blk_num[ids[q]]);
    return mb;
}

extern "C" int wally_simd_eval_batch(wally_simd_ctx *c, uint32_t nq, const uint32_t *ids, const uint32_t *query_ct,
                                     const uint32_t *keys, uint32_t *resp, uint64_t resp_words, uint64_t *resp_off,
                                     void *stream) {
    if (!c) return WALLY_E_ARG;
    if (nq && (!ids || !query_ct || !keys || !resp)) return sfail(c, WALLY_E_ARG, "eval_batch: null argument");
    std::vector<uint64_t> off;
    int rc = simd_offsets(c, nq, ids, off);
    if (rc) return rc;
    if (resp_off) std::copy(off.begin(), off.end(), resp_off);
    if (resp_words < off[nq]) return sfail(c, WALLY_E_ARG, "resp_words %llu < %llu", (unsigned long long)resp_words,
                                           (unsigned long long)off[nq]);
    if (!nq) return WALLY_OK;
    SCUDA(c, cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    SimdWs W;
    rc = simd_workspace(c, nq, simd_max_blocks(c, nq, ids), W);
    if (rc) return rc;
    SCUDA(c, cudaMemsetAsync(W.err, 0, 4, s));
    rc = simd_eval_core(c, W, nq, ids, query_ct, keys, resp, off.data(), s);
    if (rc) return rc;
    uint32_t herr = 0;
    SCUDA(c, cudaMemcpyAsync(&herr, W.err, 4, cudaMemcpyDeviceToHost, s));
    SCUDA(c, cudaStreamSynchronize(s));
    if (herr) return sfail(c, WALLY_E_RESIDUE, "an input residue is >= its modulus");
    return WALLY_OK;
}

extern "C" int wally_simd_eval_batch_host(wally_simd_ctx *c, uint32_t nq, const uint32_t *ids,
                                          const uint32_t *query_ct, const uint32_t *keys, uint32_t *resp,
                                          uint64_t resp_words, uint64_t *resp_off, uint32_t sub_batch, void *stream) {
    if (!c) return WALLY_E_ARG;
    if (nq && (!ids || !query_ct || !keys || !resp)) return sfail(c, WALLY_E_ARG, "eval_batch_host: null argument");
    if (!sub_batch) return sfail(c, WALLY_E_ARG, "eval_batch_host: sub_batch must be > 0");
    std::vector<uint64_t> off;
    int rc = simd_offsets(c, nq, ids, off);
    if (rc) return rc;
    if (resp_off) std::copy(off.begin(), off.end(), resp_off);
    if (resp_words < off[nq]) return sfail(c, WALLY_E_ARG, "resp_words %llu < %llu", (unsigned long long)resp_words,
                                           (unsigned long long)off[nq]);
    if (!nq) return WALLY_OK;
    SCUDA(c, cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t n = c->p.n, L = c->L, M = c->M;
    const size_t CT = (size_t)2 * L * n, KW = (size_t)2 * 2 * L * M * n;
    const uint32_t sb = std::min(sub_batch, nq), max_blk = simd_max_blocks(c, nq, ids);
    SimdWs W;
    rc = simd_workspace(c, sb, max_blk, W);
    if (rc) return rc;
    // double-buffered device staging: inputs and responses of two sub-batches
    const size_t in_words = (size_t)sb * (CT + KW), out_words = (size_t)sb * max_blk * 2 * n;
    const size_t need = 2 * 4 * (in_words + out_words);
    if (c->stage_bytes < need) {
        SCUDA(c, cudaStreamSynchronize(s));
        cudaFree(c->stage);
        c->stage = nullptr;
        c->stage_bytes = 0;
        if (cudaMalloc(&c->stage, need) != cudaSuccess) return sfail(c, WALLY_E_OOM, "host-path staging (%zu bytes)", need);
        c->stage_bytes = need;
    }
    if (!c->h2d) {
        SCUDA(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
        SCUDA(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
        for (int k = 0; k < 2; k++) {
            SCUDA(c, cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming));
            SCUDA(c, cudaEventCreateWithFlags(&c->ev_done[k], cudaEventDisableTiming));
            SCUDA(c, cudaEventCreateWithFlags(&c->ev_out[k], cudaEventDisableTiming));
        }
    }
    uint32_t *stage = (uint32_t *)c->stage;
    SCUDA(c, cudaMemsetAsync(W.err, 0, 4, s));
    // the first sub-batches must not overtake work already queued on s
    SCUDA(c, cudaEventRecord(c->ev_done[0], s));
    SCUDA(c, cudaEventRecord(c->ev_done[1], s));
    SCUDA(c, cudaEventRecord(c->ev_out[0], s));
    SCUDA(c, cudaEventRecord(c->ev_out[1], s));
    for (uint32_t q0 = 0, it = 0; q0 < nq; q0 += sb, it++) {
        const uint32_t nc = std::min(sb, nq - q0), k = it & 1;
        uint32_t *ict = stage + k * (in_words + out_words), *ikey = ict + (size_t)sb * CT, *iout = ikey + (size_t)sb * KW;
        // inputs of this sub-batch (copy stream), once the computation that read this slot is done
        SCUDA(c, cudaStreamWaitEvent(c->h2d, c->ev_done[k], 0));
        SCUDA(c, cudaMemcpyAsync(ict, query_ct + (size_t)q0 * CT, 4 * (size_t)nc * CT, cudaMemcpyHostToDevice, c->h2d));
        SCUDA(c, cudaMemcpyAsync(ikey, keys + (size_t)q0 * KW, 4 * (size_t)nc * KW, cudaMemcpyHostToDevice, c->h2d));
        SCUDA(c, cudaEventRecord(c->ev_in[k], c->h2d));
        // computation (main stream), once the inputs arrived and this slot's responses left
        SCUDA(c, cudaStreamWaitEvent(s, c->ev_in[k], 0));
        SCUDA(c, cudaStreamWaitEvent(s, c->ev_out[k], 0));
        std::vector<uint64_t> loc(nc + 1);
        for (uint32_t q = 0; q <= nc; q++) loc[q] = off[q0 + q] - off[q0];
        rc = simd_eval_core(c, W, nc, ids + q0, ict, ikey, iout, loc.data(), s);
        if (rc) return rc;
        SCUDA(c, cudaEventRecord(c->ev_done[k], s));
        // responses (copy-out stream)
        SCUDA(c, cudaStreamWaitEvent(c->d2h, c->ev_done[k], 0));
        SCUDA(c, cudaMemcpyAsync(resp + off[q0], iout, 4 * (size_t)loc[nc], cudaMemcpyDeviceToHost, c->d2h));
        SCUDA(c, cudaEventRecord(c->ev_out[k], c->d2h));
    }
    SCUDA(c, cudaStreamWaitEvent(s, c->ev_out[0], 0));
    SCUDA(c, cudaStreamWaitEvent(s, c->ev_out[1], 0));
    uint32_t herr = 0;
    SCUDA(c, cudaMemcpyAsync(&herr, W.err, 4, cudaMemcpyDeviceToHost, s));
    SCUDA(c, cudaStreamSynchronize(s));
    if (herr) return sfail(c, WALLY_E_RESIDUE, "an input residue is >= its modulus");
    return WALLY_OK;
}

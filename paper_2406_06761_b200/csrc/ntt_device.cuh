// Device building blocks of the hot path: 32-bit modular arithmetic with
// Harvey/Shoup lazy reduction, and register-blocked negacyclic NTT passes
// exchanged through shared memory.
//
// Paper: NTT with Harvey's butterfly and lazy modular reduction (PAPER.md
// P:L1000); NTT-friendly RNS limbs q_i = 1 mod 2n.
// All moduli are < 2^30, so 4q < 2^32 and the lazy ranges [0, 2q) / [0, 4q)
// fit one 32-bit word.
#pragma once

#include <cstdint>

namespace wally {

// ---------------------------------------------------------------------------
// Modular arithmetic
// ---------------------------------------------------------------------------

// x in [0, 2m) -> [0, m).  (unsigned min: x - m wraps above x when x < m)
__device__ __forceinline__ uint32_t csub(uint32_t x, uint32_t m) { return min(x, x - m); }

// Shoup multiplication by a precomputed constant: w < q, wp = floor(w 2^32 / q).
// For any 32-bit x returns x*w mod q in [0, 2q).  3 IMAD-pipe instructions.
__device__ __forceinline__ uint32_t shoup_mul(uint32_t x, uint32_t w, uint32_t wp, uint32_t q) {
    uint32_t hi = __umulhi(x, wp);
    return x * w - hi * q;
}

// Gentleman-Sande (inverse) butterfly, Harvey lazy form.
// In: X, Y in [0, 2q).  Out: X' = X + Y in [0, 2q), Y' = (X - Y) w in [0, 2q).
__device__ __forceinline__ void gs_bfly(uint32_t &X, uint32_t &Y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
    uint32_t u = csub(X + Y, q2);
    uint32_t v = X - Y + q2;
    Y = shoup_mul(v, w, wp, q);
    X = u;
}

// Cooley-Tukey (forward) butterfly, Harvey lazy form.
// In: X, Y in [0, 4q).  Out: X' = X + Y w, Y' = X - Y w, both in [0, 4q).
__device__ __forceinline__ void ct_bfly(uint32_t &X, uint32_t &Y, uint32_t w, uint32_t wp, uint32_t q, uint32_t q2) {
    uint32_t x = csub(X, q2);
    uint32_t t = shoup_mul(Y, w, wp, q);
    X = x + t;
    Y = x - t + q2;
}

// ---------------------------------------------------------------------------
// NTT pass geometry
//
// A length-n transform is split into three passes.  GS (inverse) order runs
// passes with strides TB_0 = 1, TB_1 = 2^S0, TB_2 = 2^(S0+S1); CT (forward)
// runs them in reverse.  In a pass with base stride TB and radix R = 2^S each
// thread owns G = V/R groups; group gamma = g + j*T (g = thread, T = n/V) is
// the R elements  idx(k) = hi*TB*R + k*TB + lo,  (hi, lo) = divmod(gamma, TB).
// All S stages of the pass are butterflies inside a group, so they run in
// registers; between passes the data goes through shared memory.
// ---------------------------------------------------------------------------

template <int N>
struct NttCfg;
template <>
struct NttCfg<1024> { static constexpr int V = 16, S0 = 4, S1 = 4, S2 = 2; };
template <>
struct NttCfg<2048> { static constexpr int V = 16, S0 = 4, S1 = 4, S2 = 3; };
template <>
struct NttCfg<4096> { static constexpr int V = 16, S0 = 4, S1 = 4, S2 = 4; };
template <>
struct NttCfg<8192> { static constexpr int V = 32, S0 = 5, S1 = 4, S2 = 4; };

template <int N>
struct NttGeom {
    using C = NttCfg<N>;
    static constexpr int V = C::V;
    static constexpr int T = N / V;                   // threads per polynomial
    static constexpr int TB0 = 1, R0 = 1 << C::S0;
    static constexpr int TB1 = 1 << C::S0, R1 = 1 << C::S1;
    static constexpr int TB2 = 1 << (C::S0 + C::S1), R2 = 1 << C::S2;
    static_assert(R0 == V, "pass 0 must give each thread one contiguous group");
    static_assert(TB2 * R2 == N, "passes must cover log2(n) stages");
    static constexpr int PAD_SHIFT = (N >= 8192) ? 5 : 4;
    static constexpr int SMEM_WORDS = N + (N >> PAD_SHIFT) + 32;  // one exchange buffer
};

template <int N>
__device__ __forceinline__ int smem_pad(int i) { return i + (i >> NttGeom<N>::PAD_SHIFT); }

template <int N, int TB, int R>
__device__ __forceinline__ int pass_index(int g, int j, int k) {
    constexpr int T = NttGeom<N>::T;
    const int gam = g + j * T;
    const int hi = gam / TB, lo = gam % TB;
    return hi * TB * R + k * TB + lo;
}

template <int N, int TB, int R>
__device__ __forceinline__ void smem_store(uint32_t *buf, const uint32_t (&a)[NttGeom<N>::V], int g) {
    constexpr int V = NttGeom<N>::V, G = V / R;
#pragma unroll
    for (int j = 0; j < G; j++)
#pragma unroll
        for (int k = 0; k < R; k++) buf[smem_pad<N>(pass_index<N, TB, R>(g, j, k))] = a[j * R + k];
}

template <int N, int TB, int R>
__device__ __forceinline__ void smem_load(const uint32_t *buf, uint32_t (&a)[NttGeom<N>::V], int g) {
    constexpr int V = NttGeom<N>::V, G = V / R;
#pragma unroll
    for (int j = 0; j < G; j++)
#pragma unroll
        for (int k = 0; k < R; k++) a[j * R + k] = buf[smem_pad<N>(pass_index<N, TB, R>(g, j, k))];
}

// All stages of one pass.  INVERSE: GS stages with strides TB, 2TB, ...;
// forward: CT stages with strides TB*R/2, ..., TB.  Stage with stride t uses
// twiddle tw[m + i], m = n/(2t), i = idx / (2t) (the standard merged
// negacyclic tables: psi^{brev} forward, psi^{-brev} inverse).
template <int N, int TB, int R, bool INVERSE>
__device__ __forceinline__ void ntt_pass(uint32_t (&a)[NttGeom<N>::V], const uint2 *__restrict__ tw, int g, uint32_t q,
                                         uint32_t q2) {
    constexpr int V = NttGeom<N>::V, T = NttGeom<N>::T, G = V / R;
    constexpr int LOGR = (R == 2) ? 1 : (R == 4) ? 2 : (R == 8) ? 3 : (R == 16) ? 4 : (R == 32) ? 5 : 6;
#pragma unroll
    for (int j = 0; j < G; j++) {
        const int hi = (g + j * T) / TB;
#pragma unroll
        for (int ss = 0; ss < LOGR; ss++) {
            const int s = INVERSE ? ss : (LOGR - 1 - ss);
            const int half = 1 << s;
            const int m = N / (2 * TB * half);
            const int nb = R >> (s + 1);
            const uint2 *twp = tw + m + hi * nb;
#pragma unroll
            for (int b = 0; b < nb; b++) {
                const uint2 w = __ldg(twp + b);
#pragma unroll
                for (int kk = 0; kk < half; kk++) {
                    const int k0 = b * 2 * half + kk;
                    if (INVERSE)
                        gs_bfly(a[j * R + k0], a[j * R + k0 + half], w.x, w.y, q, q2);
                    else
                        ct_bfly(a[j * R + k0], a[j * R + k0 + half], w.x, w.y, q, q2);
                }
            }
        }
    }
}

// Whole inverse transform (without the n^{-1} scale) for one polynomial
// held as pass-0 groups (thread g owns elements g*V .. g*V+V-1) on entry;
// on exit the thread owns the pass-2 groups.  Two barriers per call; two
// exchange buffers alternate so no write-after-read barrier is needed.
template <int N>
__device__ __forceinline__ void intt_chain(uint32_t (&a)[NttGeom<N>::V], const uint2 *__restrict__ tw, int g,
                                           uint32_t q, uint32_t q2, uint32_t *bufA, uint32_t *bufB) {
    using Gm = NttGeom<N>;
    ntt_pass<N, Gm::TB0, Gm::R0, true>(a, tw, g, q, q2);
    smem_store<N, Gm::TB0, Gm::R0>(bufA, a, g);
    __syncthreads();
    smem_load<N, Gm::TB1, Gm::R1>(bufA, a, g);
    ntt_pass<N, Gm::TB1, Gm::R1, true>(a, tw, g, q, q2);
    smem_store<N, Gm::TB1, Gm::R1>(bufB, a, g);
    __syncthreads();
    smem_load<N, Gm::TB2, Gm::R2>(bufB, a, g);
    ntt_pass<N, Gm::TB2, Gm::R2, true>(a, tw, g, q, q2);
}

// Whole forward transform: on entry the thread owns pass-2 groups, on exit
// pass-0 groups (contiguous V elements, bit-reversed NTT order).
template <int N>
__device__ __forceinline__ void ntt_chain(uint32_t (&a)[NttGeom<N>::V], const uint2 *__restrict__ tw, int g,
                                          uint32_t q, uint32_t q2, uint32_t *bufA, uint32_t *bufB) {
    using Gm = NttGeom<N>;
    ntt_pass<N, Gm::TB2, Gm::R2, false>(a, tw, g, q, q2);
    smem_store<N, Gm::TB2, Gm::R2>(bufA, a, g);
    __syncthreads();
    smem_load<N, Gm::TB1, Gm::R1>(bufA, a, g);
    ntt_pass<N, Gm::TB1, Gm::R1, false>(a, tw, g, q, q2);
    smem_store<N, Gm::TB1, Gm::R1>(bufB, a, g);
    __syncthreads();
    smem_load<N, Gm::TB0, Gm::R0>(bufB, a, g);
    ntt_pass<N, Gm::TB0, Gm::R0, false>(a, tw, g, q, q2);
}

}  // namespace wally

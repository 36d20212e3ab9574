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

// Montgomery multiplication x * ym * 2^-32 mod q (ym = y 2^32 mod q, qi =
// -q^{-1} mod 2^32): for x < 4q returns x y mod q in [0, 2q), the range of
// shoup_mul, without a companion operand.  2 IMAD.WIDE + 1 IMAD.
__device__ __forceinline__ uint32_t mont_mul(uint32_t x, uint32_t ym, uint32_t q, uint32_t qi) {
    const uint64_t t = (uint64_t)x * ym;                       // < 4 q^2 < 2^62
    const uint32_t m = (uint32_t)t * qi;
    return (uint32_t)((t + (uint64_t)m * q) >> 32);           // (t + m q) / 2^32 < 2q
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

// Streaming 128-bit load that does not allocate in L1 (keeps the L1 for the
// twiddle tables, which every polynomial re-reads).
__device__ __forceinline__ uint4 ldg_stream(const void *p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

// Operand loads of the fused kernels (plaintext slices and query NTTs, which
// are re-read from L2 by the other queries / plaintexts of their cluster).
// MODE 0: no L1 allocation, default L2 policy of .nc no_allocate loads;
// MODE 1: L1-allocating read-only load (the other half of each 32-byte sector
//         is read by the same thread's next chunk);
// MODE 2: no L1 allocation, L2 evict_last cache hint;
// MODE 3: L1-allocating, L2 evict_last cache hint.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <int MODE>
__device__ __forceinline__ uint4 ldg_op(const void *p) {
    uint4 r;
    if constexpr (MODE == 0) {
        r = ldg_stream(p);
    } else if constexpr (MODE == 1) {
        r = __ldg(reinterpret_cast<const uint4 *>(p));
    } else if constexpr (MODE == 2) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
            : "l"(p), "l"(l2_evict_last_policy()));
    } else {
        asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
            : "l"(p), "l"(l2_evict_last_policy()));
    }
    return r;
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
//
// Twiddle tables are "pass-major": per limb, pass p holds one block of R
// (w, w') pairs per value of hi, with the stage twiddles the group needs in
// execution order -- so a group reads its twiddles as contiguous 16-byte
// vectors.  The stage with butterfly distance 2^s (stride t = TB 2^s) uses
// psi-table entry m + hi*NB + b, m = n/(2t), NB = R >> (s+1), b < NB
// (merged negacyclic tables: psi^{brev} forward, psi^{-brev} inverse).
//   inverse (GS, s ascending):  slot of (s, b) = R - (R >> s) + b
//   forward (CT, s descending): slot of (s, b) = (R >> (s+1)) + b
// Pass 0 (TB = 1, hi = thread g, one unique block per thread) is stored
// slot-pair-major, uint4 index (slot/2) * T + g, so the 16-byte loads of a
// warp are contiguous (global) and bank-conflict free (shared memory).
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
    // one exchange buffer (largest of the two paddings of smem_pad)
    static constexpr int PADW = (N >> C::S0) > (16 * (N >> (C::S0 + C::S1))) ? (N >> C::S0) : 16 * (N >> (C::S0 + C::S1));
    static constexpr int SMEM_WORDS = N + PADW + 32;
    // The exchange between pass 0 and pass 1 stays inside one warp when a
    // thread's pass-0 group (V contiguous elements) and its pass-1 group
    // (one group of R1 elements at stride TB1 = V) together cover exactly the
    // warp's 32 V elements; then a __syncwarp replaces the group barrier, and
    // both paddings of smem_pad map the warp's elements to the same private
    // region of the buffer.
    static constexpr bool A_IN_WARP = (V == TB1) && (V == R1);
    // pass-major twiddle table offsets (uint2 entries) inside one limb's table
    static constexpr int TW0 = 0, TW1 = N / TB0, TW2 = N / TB0 + N / TB1;
    static constexpr int TW_LIMB = N / TB0 + N / TB1 + N / TB2;
};

// Storage order of NTT-domain polynomials (query NTTs, the plaintext store).
// Thread g of a transform holds the V consecutive (bit-reversed-order)
// elements g V .. g V + V - 1 after the forward transform.  At n <= 4096 they
// are stored in that order; at n = 8192 CHUNK-MAJOR: value 4 v + i of thread
// g (its v-th 16-byte chunk) at word v (4 T) + 4 g + i, so the fused kernel's
// per-chunk 16-byte loads of a warp cover 512 contiguous bytes, and chunk v of
// all threads is one 4 KB block a bulk copy can stage.  The order is internal:
// every producer and consumer goes through ntt_word.
template <int N>
struct NttStore { static constexpr bool CHUNK_MAJOR = (N == 8192); };

template <int N>
__host__ __device__ constexpr size_t ntt_word(int g, int v) {
    return NttStore<N>::CHUNK_MAJOR ? (size_t)v * 4 * NttGeom<N>::T + 4 * (size_t)g
                                    : (size_t)g * NttGeom<N>::V + 4 * (size_t)v;
}

template <int R>
struct Log2 { static constexpr int v = (R <= 1) ? 0 : 1 + Log2<R / 2>::v; };
template <>
struct Log2<1> { static constexpr int v = 0; };

// Exchange-buffer address of element i.  Each of the two exchanges of a
// transform has its own padding, chosen so that both access patterns of
// that exchange hit 32 distinct banks per warp instruction while every
// per-thread offset stays a compile-time immediate (checked exhaustively for
// n = 1024..8192):
//   X = 0, between pass 0 (contiguous groups) and pass 1:  i + (i >> S0)
//   X = 1, between pass 1 and pass 2 (stride n/R groups):  i + 16 (i >> (S0+S1))
template <int N, int X>
__device__ __forceinline__ int smem_pad(int i) {
    using C = NttCfg<N>;
    if constexpr (X == 0) return i + (i >> C::S0);
    else return i + ((i >> (C::S0 + C::S1)) << 4);
}

template <int N, int TB, int R>
__device__ __forceinline__ int pass_index(int g, int j, int k) {
    constexpr int T = NttGeom<N>::T;
    const int gam = g + j * T;
    const int hi = gam / TB, lo = gam % TB;
    return hi * TB * R + k * TB + lo;
}

// NC polynomials per thread: a[c][V]; poly c exchanges through buf + c * SMEM_WORDS.
template <int N, int TB, int R, int NC, int X>
__device__ __forceinline__ void smem_store(uint32_t *buf, const uint32_t (&a)[NC][NttGeom<N>::V], int g) {
    constexpr int V = NttGeom<N>::V, G = V / R;
#pragma unroll
    for (int c = 0; c < NC; c++)
#pragma unroll
        for (int j = 0; j < G; j++)
#pragma unroll
            for (int k = 0; k < R; k++)
                buf[c * NttGeom<N>::SMEM_WORDS + smem_pad<N, X>(pass_index<N, TB, R>(g, j, k))] = a[c][j * R + k];
}

template <int N, int TB, int R, int NC, int X>
__device__ __forceinline__ void smem_load(const uint32_t *buf, uint32_t (&a)[NC][NttGeom<N>::V], int g) {
    constexpr int V = NttGeom<N>::V, G = V / R;
#pragma unroll
    for (int c = 0; c < NC; c++)
#pragma unroll
        for (int j = 0; j < G; j++)
#pragma unroll
            for (int k = 0; k < R; k++)
                a[c][j * R + k] = buf[c * NttGeom<N>::SMEM_WORDS + smem_pad<N, X>(pass_index<N, TB, R>(g, j, k))];
}

// Twiddle fetch: plain loads when the table lives in shared memory (TWS),
// read-only-cache loads when it lives in global memory.
template <bool TWS>
__device__ __forceinline__ uint4 tw_ld4(const uint4 *p) {
    if constexpr (TWS) return *p; else return __ldg(p);
}
template <bool TWS>
__device__ __forceinline__ uint2 tw_ld2(const uint2 *p) {
    if constexpr (TWS) return *p; else return __ldg(p);
}

// One stage (butterfly distance 2^S inside each group) of a pass, applied to
// NC polynomials that share the twiddles.  All bounds are constant
// expressions, so the stage unrolls into straight register code.
template <int N, int TB, int R, int S, bool INVERSE, int NC, bool TWS>
__device__ __forceinline__ void ntt_stage(uint32_t (&a)[NC][NttGeom<N>::V], const uint2 *__restrict__ twp, int g,
                                          uint32_t q, uint32_t q2) {
    constexpr int V = NttGeom<N>::V, T = NttGeom<N>::T, G = V / R;
    constexpr int HALF = 1 << S;
    constexpr int NB = R >> (S + 1);
    constexpr int OFF = INVERSE ? (R - (R >> S)) : (R >> (S + 1));
#pragma unroll
    for (int j = 0; j < G; j++) {
        uint2 w[NB];
        if constexpr (TB == 1) {
            // pass 0: slot-pair-major, uint4 index (slot/2) * T + g   (G == 1)
            const uint4 *t4 = reinterpret_cast<const uint4 *>(twp) + g;
            if constexpr (NB >= 2) {
#pragma unroll
                for (int b = 0; b < NB / 2; b++) {
                    const uint4 x = tw_ld4<TWS>(t4 + (OFF / 2 + b) * T);
                    w[2 * b] = make_uint2(x.x, x.y);
                    w[2 * b + 1] = make_uint2(x.z, x.w);
                }
            } else {
                w[0] = tw_ld2<TWS>(reinterpret_cast<const uint2 *>(t4 + (OFF / 2) * T) + (OFF % 2));
            }
        } else {
            const uint2 *t = twp + ((g + j * T) / TB) * R + OFF;
            if constexpr (NB >= 2) {
#pragma unroll
                for (int b = 0; b < NB / 2; b++) {
                    const uint4 x = tw_ld4<TWS>(reinterpret_cast<const uint4 *>(t) + b);
                    w[2 * b] = make_uint2(x.x, x.y);
                    w[2 * b + 1] = make_uint2(x.z, x.w);
                }
            } else {
                w[0] = tw_ld2<TWS>(t);
            }
        }
#pragma unroll
        for (int b = 0; b < NB; b++)
#pragma unroll
            for (int kk = 0; kk < HALF; kk++)
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    if constexpr (INVERSE)
                        gs_bfly(a[c][j * R + b * 2 * HALF + kk], a[c][j * R + b * 2 * HALF + kk + HALF], w[b].x,
                                w[b].y, q, q2);
                    else
                        ct_bfly(a[c][j * R + b * 2 * HALF + kk], a[c][j * R + b * 2 * HALF + kk + HALF], w[b].x,
                                w[b].y, q, q2);
                }
    }
}

template <int N, int TB, int R, bool INVERSE, int NC, bool TWS, int SS>
struct PassStages {
    static constexpr int LOGR = Log2<R>::v;
    static __device__ __forceinline__ void run(uint32_t (&a)[NC][NttGeom<N>::V], const uint2 *__restrict__ twp, int g,
                                               uint32_t q, uint32_t q2) {
        ntt_stage<N, TB, R, INVERSE ? SS : (LOGR - 1 - SS), INVERSE, NC, TWS>(a, twp, g, q, q2);
        if constexpr (SS + 1 < LOGR) PassStages<N, TB, R, INVERSE, NC, TWS, SS + 1>::run(a, twp, g, q, q2);
    }
};

// All stages of one pass (twp = this pass's table inside the limb's table).
template <int N, int TB, int R, bool INVERSE, int NC, bool TWS = false>
__device__ __forceinline__ void ntt_pass(uint32_t (&a)[NC][NttGeom<N>::V], const uint2 *__restrict__ twp, int g,
                                         uint32_t q, uint32_t q2) {
    PassStages<N, TB, R, INVERSE, NC, TWS, 0>::run(a, twp, g, q, q2);
}

// Whole inverse transform (without the n^{-1} scale) of NC polynomials held
// as pass-0 groups (thread g owns elements g*V .. g*V+V-1) on entry; on exit
// the thread owns the pass-2 groups.  tw = the limb's inverse table.  Two
// barriers per call; bufA/bufB (NC exchange buffers each) alternate, so no
// write-after-read barrier is needed between consecutive calls.
template <int N, int NC>
__device__ __forceinline__ void intt_chain(uint32_t (&a)[NC][NttGeom<N>::V], const uint2 *__restrict__ tw, int g,
                                           uint32_t q, uint32_t q2, uint32_t *bufA, uint32_t *bufB) {
    using Gm = NttGeom<N>;
    ntt_pass<N, Gm::TB0, Gm::R0, true, NC>(a, tw + Gm::TW0, g, q, q2);
    smem_store<N, Gm::TB0, Gm::R0, NC, 0>(bufA, a, g);
    __syncthreads();
    smem_load<N, Gm::TB1, Gm::R1, NC, 0>(bufA, a, g);
    ntt_pass<N, Gm::TB1, Gm::R1, true, NC>(a, tw + Gm::TW1, g, q, q2);
    smem_store<N, Gm::TB1, Gm::R1, NC, 1>(bufB, a, g);
    __syncthreads();
    smem_load<N, Gm::TB2, Gm::R2, NC, 1>(bufB, a, g);
    ntt_pass<N, Gm::TB2, Gm::R2, true, NC>(a, tw + Gm::TW2, g, q, q2);
}

// Named barrier over the `nthreads` threads of one thread group.
__device__ __forceinline__ void group_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Inverse transform for one T-thread group of a multi-group CTA, with the
// twiddle table in shared memory and a single exchange buffer per
// polynomial (four named barriers: the first protects the buffer against
// the previous call's last reads).
template <int N, int NC>
__device__ __forceinline__ void intt_chain_group(uint32_t (&a)[NC][NttGeom<N>::V], const uint2 *tw_smem, int g,
                                                 uint32_t q, uint32_t q2, uint32_t *buf, int bar_id) {
    using Gm = NttGeom<N>;
    ntt_pass<N, Gm::TB0, Gm::R0, true, NC, true>(a, tw_smem + Gm::TW0, g, q, q2);
    group_sync(bar_id, Gm::T);
    smem_store<N, Gm::TB0, Gm::R0, NC, 0>(buf, a, g);
    if constexpr (Gm::A_IN_WARP) __syncwarp(); else group_sync(bar_id, Gm::T);
    smem_load<N, Gm::TB1, Gm::R1, NC, 0>(buf, a, g);
    ntt_pass<N, Gm::TB1, Gm::R1, true, NC, true>(a, tw_smem + Gm::TW1, g, q, q2);
    if constexpr (Gm::A_IN_WARP) __syncwarp(); else group_sync(bar_id, Gm::T);
    smem_store<N, Gm::TB1, Gm::R1, NC, 1>(buf, a, g);
    group_sync(bar_id, Gm::T);
    smem_load<N, Gm::TB2, Gm::R2, NC, 1>(buf, a, g);
    ntt_pass<N, Gm::TB2, Gm::R2, true, NC, true>(a, tw_smem + Gm::TW2, g, q, q2);
}

// intt_chain_group without its pass 0 (the caller ran it, e.g. interleaved
// with other work): the two exchanges and passes 1 and 2.  FRESH_BUF: the
// caller alternates exchange buffers between consecutive calls, so the
// barrier protecting the buffer against the previous call's reads is not
// needed (the call before the previous one ended with a group barrier).
template <int N, int NC, bool FRESH_BUF = false>
__device__ __forceinline__ void intt_chain_group_tail(uint32_t (&a)[NC][NttGeom<N>::V], const uint2 *tw_smem, int g,
                                                      uint32_t q, uint32_t q2, uint32_t *buf, int bar_id) {
    using Gm = NttGeom<N>;
    if constexpr (!FRESH_BUF || !Gm::A_IN_WARP) group_sync(bar_id, Gm::T);
    smem_store<N, Gm::TB0, Gm::R0, NC, 0>(buf, a, g);
    if constexpr (Gm::A_IN_WARP) __syncwarp(); else group_sync(bar_id, Gm::T);
    smem_load<N, Gm::TB1, Gm::R1, NC, 0>(buf, a, g);
    ntt_pass<N, Gm::TB1, Gm::R1, true, NC, true>(a, tw_smem + Gm::TW1, g, q, q2);
    if constexpr (Gm::A_IN_WARP) __syncwarp(); else group_sync(bar_id, Gm::T);
    smem_store<N, Gm::TB1, Gm::R1, NC, 1>(buf, a, g);
    group_sync(bar_id, Gm::T);
    smem_load<N, Gm::TB2, Gm::R2, NC, 1>(buf, a, g);
    ntt_pass<N, Gm::TB2, Gm::R2, true, NC, true>(a, tw_smem + Gm::TW2, g, q, q2);
}

// Whole forward transform: on entry the thread owns pass-2 groups, on exit
// pass-0 groups (contiguous V elements, bit-reversed NTT order).
template <int N, int NC>
__device__ __forceinline__ void ntt_chain(uint32_t (&a)[NC][NttGeom<N>::V], const uint2 *__restrict__ tw, int g,
                                          uint32_t q, uint32_t q2, uint32_t *bufA, uint32_t *bufB) {
    using Gm = NttGeom<N>;
    ntt_pass<N, Gm::TB2, Gm::R2, false, NC>(a, tw + Gm::TW2, g, q, q2);
    smem_store<N, Gm::TB2, Gm::R2, NC, 1>(bufA, a, g);
    __syncthreads();
    smem_load<N, Gm::TB1, Gm::R1, NC, 1>(bufA, a, g);
    ntt_pass<N, Gm::TB1, Gm::R1, false, NC>(a, tw + Gm::TW1, g, q, q2);
    smem_store<N, Gm::TB1, Gm::R1, NC, 0>(bufB, a, g);
    if constexpr (Gm::A_IN_WARP) __syncwarp(); else __syncthreads();
    smem_load<N, Gm::TB0, Gm::R0, NC, 0>(bufB, a, g);
    ntt_pass<N, Gm::TB0, Gm::R0, false, NC>(a, tw + Gm::TW0, g, q, q2);
}

}  // namespace wally

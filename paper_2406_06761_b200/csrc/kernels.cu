// sm_100a kernels of the Wally server hot path.
//
//   encode_kernel        a0  ServerInit: pack entries (reversed, offsets j*d),
//                            lift mod q_i, forward NTT, fold constants, Shoup companion
//   batch_count/scan/    a1  group the batch by cluster id, build the work list
//   scatter kernels
//   ntt_forward_kernel   a2  forward negacyclic NTT of every query polynomial
//   eval_kernel          a3-a6 fused: pointwise Shoup modmul, inverse NTT,
//                            RNS modulus switch to q_0, response write
//
// Citations: PAPER.md P:L1000 / P:L1467-1472 (Harvey NTT, lazy reduction),
// P:L1003 / P:L1318-1324 (modulus switch to q_0), Alg 1 P:L664-687 and
// Alg 4 P:L794-808 (ServerInit / ServerComputation).

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "ntt_device.cuh"
#include "tmem.cuh"
#include "wally_internal.h"

#ifndef WALLY_OPLD_PR
#define WALLY_OPLD_PR 1
#endif

namespace wally {

// Debug builds (WALLY_BOUNDS_CHECK=1): trap with the call site when an access
// of the v4 fused kernel leaves its buffer (round-2 investigation of the
// L = 2 tensor-memory-state fault).
#ifndef WALLY_BOUNDS_CHECK
#define WALLY_BOUNDS_CHECK 0
#endif
#if WALLY_BOUNDS_CHECK
#define WALLY_BC(ptr, base, words, tag)                                                                         \
    do {                                                                                                        \
        const uint32_t *p_ = (const uint32_t *)(ptr);                                                           \
        if (p_ < (const uint32_t *)(base) || p_ + 1 > (const uint32_t *)(base) + (words)) {                     \
            printf("WALLY_BC %s: block %d thread %d offset %lld of %llu\n", tag, blockIdx.x, threadIdx.x,          \
                   (long long)(p_ - (const uint32_t *)(base)), (unsigned long long)(words));                     \
            __trap();                                                                                           \
        }                                                                                                       \
    } while (0)
#else
#define WALLY_BC(ptr, base, words, tag) \
    do {                                  \
    } while (0)
#endif

// ---------------------------------------------------------------------------
// a2: forward NTT of query polynomials (and of any [count][L][n] array)
// ---------------------------------------------------------------------------
// Query-NTT storage in the batch workspace (chat, [nq][2][L][n] words): at
// n = 8192 the two components of a limb are interleaved by 16-byte chunk --
// chunk v of component c of limb J at ((J * 8 + v) * 2 + c) * 4T (+ 4g + i,
// ntt_word's chunk-major order) -- so one bulk copy stages both chunks a ring
// slot of the v5 kernel needs; otherwise (c L + J) n + ntt_word.
template <int N>
__host__ __device__ constexpr size_t chat_word(uint32_t L, int comp, int J, int g, int v) {
    if constexpr (N == 8192) {
        constexpr int T = NttGeom<N>::T, CH = NttGeom<N>::V / 4;
        return (((size_t)J * CH + v) * 2 + comp) * 4 * T + 4 * (size_t)g;
    } else {
        return ((size_t)comp * L + J) * N + ntt_word<N>(g, v);
    }
}

// Word of value 4v of thread g (a 16-byte chunk) of plaintext pt, limb J, in
// the n = 8192 store (PtStore::MONT: pairs interleaved by chunk).
template <int N>
__host__ __device__ constexpr size_t pt_mont_word(size_t pt, uint32_t L, int J, int g, int v) {
    constexpr int T = NttGeom<N>::T, CH = NttGeom<N>::V / 4;
    return (pt >> 1) * 2 * L * N + (((size_t)J * CH + v) * 2 + (pt & 1)) * 4 * T + 4 * (size_t)g;
}

// CHAT: write the query-NTT workspace order (chat_word) instead of one
// polynomial after another (ntt_word).
template <int N, bool CHAT>
__global__ void __launch_bounds__(NttGeom<N>::T) ntt_forward_kernel(KParams kp, uint32_t L, const uint2 *__restrict__ tw,
                                                                    const uint32_t *__restrict__ in,
                                                                    uint32_t *__restrict__ out, uint32_t *err) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const size_t poly = blockIdx.x;
    const uint32_t limb = (uint32_t)(poly % L);
    const uint32_t q = kp.q[limb], q2 = kp.q2[limb];
    const uint32_t *src = in + poly * N;
    uint32_t a[1][V];
    bool bad = false;
    // pass-2 groups: element idx = hi*TB2*R2 + k*TB2 + lo  (coalesced across threads)
#pragma unroll
    for (int j = 0; j < V / Gm::R2; j++)
#pragma unroll
        for (int k = 0; k < Gm::R2; k++) {
            uint32_t x = __ldg(src + pass_index<N, Gm::TB2, Gm::R2>(g, j, k));
            bad |= (x >= q);
            a[0][j * Gm::R2 + k] = x;
        }
    if (bad && err) atomicOr(err, (uint32_t)kErrResidue);
    ntt_chain<N, 1>(a, tw + (size_t)limb * Gm::TW_LIMB, g, q, q2, bufA, bufB);
    if constexpr (CHAT) {
        const uint32_t comp = (uint32_t)((poly / L) % 2);
        uint32_t *dst = out + (poly / (2 * L)) * 2 * L * N;
#pragma unroll
        for (int v = 0; v < V / 4; v++)
            *reinterpret_cast<uint4 *>(dst + chat_word<N>(L, comp, limb, g, v)) =
                make_uint4(a[0][4 * v], a[0][4 * v + 1], a[0][4 * v + 2], a[0][4 * v + 3]);
    } else {
        uint32_t *dst = out + poly * N;
#pragma unroll
        for (int v = 0; v < V / 4; v++)
            *reinterpret_cast<uint4 *>(dst + ntt_word<N>(g, v)) =
                make_uint4(a[0][4 * v], a[0][4 * v + 1], a[0][4 * v + 2], a[0][4 * v + 3]);
    }
}

// Debug/test inverse NTT: out = n^{-1} INTT(in), canonical.
template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T) ntt_inverse_kernel(KParams kp, uint32_t L, const uint2 *__restrict__ tw,
                                                                    const uint32_t *__restrict__ in,
                                                                    uint32_t *__restrict__ out) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const size_t poly = blockIdx.x;
    const uint32_t limb = (uint32_t)(poly % L);
    const uint32_t q = kp.q[limb], q2 = kp.q2[limb];
    uint32_t a[1][V];
    const uint32_t *src = in + poly * N;
#pragma unroll
    for (int v = 0; v < V / 4; v++) {
        const uint4 x = __ldg(reinterpret_cast<const uint4 *>(src + ntt_word<N>(g, v)));
        // scale first (the transform is linear); Shoup accepts any 32-bit input -> [0, 2q)
        a[0][4 * v + 0] = shoup_mul(x.x, kp.ninv[limb], kp.ninvp[limb], q);
        a[0][4 * v + 1] = shoup_mul(x.y, kp.ninv[limb], kp.ninvp[limb], q);
        a[0][4 * v + 2] = shoup_mul(x.z, kp.ninv[limb], kp.ninvp[limb], q);
        a[0][4 * v + 3] = shoup_mul(x.w, kp.ninv[limb], kp.ninvp[limb], q);
    }
    intt_chain<N, 1>(a, tw + (size_t)limb * Gm::TW_LIMB, g, q, q2, bufA, bufB);
    uint32_t *dst = out + poly * N;
#pragma unroll
    for (int j = 0; j < V / Gm::R2; j++)
#pragma unroll
        for (int k = 0; k < Gm::R2; k++)
            dst[pass_index<N, Gm::TB2, Gm::R2>(g, j, k)] = csub(a[0][j * Gm::R2 + k], q);
}

// ---------------------------------------------------------------------------
// a0: plaintext encoding (ServerInit)
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(NttGeom<N>::T) encode_kernel(EncodeArgs ea) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    extern __shared__ uint32_t smem[];
    uint32_t *bufA = smem, *bufB = smem + Gm::SMEM_WORDS;
    const int g = threadIdx.x;
    const uint32_t pt = blockIdx.x, limb = blockIdx.y;
    const uint32_t q = ea.kp.q[limb], q2 = ea.kp.q2[limb];
    const uint32_t li = ea.pt_li[pt], k = ea.pt_k[pt];
    const uint32_t first = k * ea.E;  // first entry of this plaintext inside the cluster
    const uint32_t size = ea.size[li];
    const uint32_t count = first < size ? min(ea.E, size - first) : 0u;   // 0: pad plaintext (PtStore)
    const int8_t *ent = ea.entries + (ea.entry_base[li] + first) * (uint64_t)ea.d;
    uint32_t a[1][V];
#pragma unroll
    for (int j = 0; j < V / Gm::R2; j++)
#pragma unroll
        for (int kk = 0; kk < Gm::R2; kk++) {
            // coefficient position pos = j'*d + d - 1 - i holds entry j', component i
            const uint32_t pos = pass_index<N, Gm::TB2, Gm::R2>(g, j, kk);
            const uint32_t jj = pos / ea.d, i = ea.d - 1 - pos % ea.d;
            int32_t x = 0;
            if (jj < count) x = ent[(size_t)jj * ea.d + i];
            a[0][j * Gm::R2 + kk] = (x < 0) ? (uint32_t)((int64_t)q + x) : (uint32_t)x;  // x mod q (reading S8)
        }
    ntt_chain<N, 1>(a, ea.tw_fwd + (size_t)limb * Gm::TW_LIMB, g, q, q2, bufA, bufB);
#pragma unroll
    for (int v = 0; v < V / 4; v++) {
        uint32_t y[4], yp[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            y[i] = csub(shoup_mul(a[0][4 * v + i], ea.kp.fold[limb], ea.kp.foldp[limb], q), q);  // canonical
            if constexpr (PtStore<N>::MONT)
                yp[i] = (uint32_t)(((uint64_t)y[i] << 32) % q);                                // Montgomery form
            else
                yp[i] = (uint32_t)(((uint64_t)y[i] << 32) / q);                                // Shoup companion
        }
        if constexpr (PtStore<N>::MONT) {
            *reinterpret_cast<uint4 *>(ea.store + pt_mont_word<N>(pt, ea.L, limb, g, v)) =
                make_uint4(yp[0], yp[1], yp[2], yp[3]);
        } else {
            uint32_t *dst = ea.store + ((size_t)pt * ea.L + limb) * 2 * N;
            *reinterpret_cast<uint4 *>(dst + ntt_word<N>(g, v)) = make_uint4(y[0], y[1], y[2], y[3]);
            *reinterpret_cast<uint4 *>(dst + N + ntt_word<N>(g, v)) = make_uint4(yp[0], yp[1], yp[2], yp[3]);
        }
    }
}

// ---------------------------------------------------------------------------
// a1: batcher
// ---------------------------------------------------------------------------
__global__ void batch_count_kernel(const uint32_t *__restrict__ ids, uint32_t nq,
                                   const int32_t *__restrict__ local_of_cluster, uint32_t total_clusters,
                                   uint32_t *__restrict__ counts) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
        uint32_t c = ids[q];
        int32_t li = c < total_clusters ? local_of_cluster[c] : -1;
        if (li >= 0) atomicAdd(&counts[li], 1u);
    }
}

// One CTA of 1024 threads: exclusive scans of query counts (segment starts)
// and of work items  ceil(P_c / ppi) * ceil(count_c / chunk)  (item starts;
// ppi = plaintexts per work item: 1, or 2 for the n = 8192 kernel v5).
__device__ __forceinline__ void batch_scan_block(const uint32_t *__restrict__ counts, uint32_t n_local,
                                                 const uint32_t *__restrict__ n_pt, uint32_t chunk, uint32_t ppi,
                                                 uint32_t *__restrict__ seg, uint32_t *__restrict__ item_start,
                                                 uint32_t *__restrict__ misc) {
    __shared__ uint32_t wsum_q[32], wsum_i[32];
    const uint32_t tid = threadIdx.x, per = (n_local + 1023) / 1024;
    const uint32_t b = tid * per, e = min(n_local, b + per);
    uint32_t sq = 0, si = 0;
    for (uint32_t i = b; i < e; i++) {
        uint32_t c = counts[i];
        sq += c;
        si += ((n_pt[i] + ppi - 1) / ppi) * ((c + chunk - 1) / chunk);
    }
    // block exclusive scan of (sq, si)
    uint32_t iq = sq, ii = si;
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t xq = __shfl_up_sync(0xffffffffu, iq, o), xi = __shfl_up_sync(0xffffffffu, ii, o);
        if (lane >= o) { iq += xq; ii += xi; }
    }
    if (lane == 31) { wsum_q[w] = iq; wsum_i[w] = ii; }
    __syncthreads();
    if (w == 0) {
        uint32_t vq = wsum_q[lane], vi = wsum_i[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t xq = __shfl_up_sync(0xffffffffu, vq, o), xi = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) { vq += xq; vi += xi; }
        }
        wsum_q[lane] = vq;
        wsum_i[lane] = vi;
    }
    __syncthreads();
    uint32_t oq = iq - sq + (w ? wsum_q[w - 1] : 0), oi = ii - si + (w ? wsum_i[w - 1] : 0);
    for (uint32_t i = b; i < e; i++) {
        uint32_t c = counts[i];
        seg[i] = oq;
        item_start[i] = oi;
        oq += c;
        oi += ((n_pt[i] + ppi - 1) / ppi) * ((c + chunk - 1) / chunk);
    }
    if (tid == 1023) {
        item_start[n_local] = oi;
        misc[kMiscTotalItems] = oi;
    }
}

__global__ void __launch_bounds__(1024) batch_scan_kernel(const uint32_t *__restrict__ counts, uint32_t n_local,
                                                          const uint32_t *__restrict__ n_pt, uint32_t chunk, uint32_t ppi,
                                                          uint32_t *__restrict__ seg, uint32_t *__restrict__ item_start,
                                                          uint32_t *__restrict__ misc) {
    batch_scan_block(counts, n_local, n_pt, chunk, ppi, seg, item_start, misc);
}

// The whole batcher in one CTA for small batches (one launch instead of
// three): count, scan, scatter, separated by block barriers.
__global__ void __launch_bounds__(1024) batch_small_kernel(const uint32_t *__restrict__ ids, uint32_t nq,
                                                           const int32_t *__restrict__ local_of_cluster,
                                                           uint32_t total_clusters, uint32_t *__restrict__ counts,
                                                           uint32_t n_local, const uint32_t *__restrict__ n_pt,
                                                           uint32_t chunk, uint32_t ppi, uint32_t *__restrict__ seg,
                                                           uint32_t *__restrict__ item_start, uint32_t *__restrict__ misc,
                                                           uint32_t *__restrict__ fill, uint32_t *__restrict__ perm) {
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
        const uint32_t c = ids[q];
        const int32_t li = c < total_clusters ? local_of_cluster[c] : -1;
        if (li >= 0) atomicAdd(&counts[li], 1u);
    }
    __syncthreads();
    batch_scan_block(counts, n_local, n_pt, chunk, ppi, seg, item_start, misc);
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
        const uint32_t c = ids[q];
        const int32_t li = c < total_clusters ? local_of_cluster[c] : -1;
        if (li >= 0) perm[seg[li] + atomicAdd(&fill[li], 1u)] = q;
    }
}

__global__ void batch_scatter_kernel(const uint32_t *__restrict__ ids, uint32_t nq,
                                     const int32_t *__restrict__ local_of_cluster, uint32_t total_clusters,
                                     const uint32_t *__restrict__ seg, uint32_t *__restrict__ fill,
                                     uint32_t *__restrict__ perm) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
        uint32_t c = ids[q];
        int32_t li = c < total_clusters ? local_of_cluster[c] : -1;
        if (li >= 0) perm[seg[li] + atomicAdd(&fill[li], 1u)] = q;
    }
}

// ---------------------------------------------------------------------------
// a3-a6: fused pointwise modmul + inverse NTT + modulus switch + write
// ---------------------------------------------------------------------------

// ((h_m - r) * C[l][m]) mod q_l in [0, 2 q_l) (lazy); r < q_m < 2 q_l.
// LAZY: the Shoup product accepts any 32-bit multiplicand, so h_m + 2 q_l - r
// (in (0, 2^32) for 30-bit limbs with q_{L-1} < 2 q_0, which wally_create
// enforces) needs no reduction of r mod q_l first: one ALU instruction
// instead of two (c3 73.9 -> 73.1 ms, c4 71.9 -> 71.5; c5, L = 2, measured
// 0.7% slower with it and keeps the reduced form).
template <bool LAZY = true>
__device__ __forceinline__ uint32_t ms_term(uint32_t r, uint32_t h_m, uint32_t q_l, uint32_t C, uint32_t Cp) {
    if constexpr (LAZY) return shoup_mul(h_m + 2 * q_l - r, C, Cp, q_l);
    else return shoup_mul(h_m + q_l - csub(r, q_l), C, Cp, q_l);
}

// Modulus-switch bookkeeping after the inverse NTT of limb J (limbs are
// processed L-1, ..., 0).  y = a[] holds c_J * F_J in [0, 2q_J) where the fold
// F_J = prod_{k>J} q_k^{-1} was applied through the plaintext.  Implements
// the sequential drop-last rounding (reading S7):
//   r_m = (c_m + h_m) mod q_m,  c_l <- (c_l + h_m - r_m) q_m^{-1}  for l < m,
// so that c_l(final) = c_l F_l + A_l with
//   A_l = sum_{m>l} (h_m - r_m) prod_{k=l+1..m} q_k^{-1}
//       = (...((h_{L-1} - r_{L-1}) q_{L-1}^{-1} + h_{L-2} - r_{L-2}) q_{L-2}^{-1} + ... + h_{l+1} - r_{l+1}) q_{l+1}^{-1},
// evaluated as follows (WALLY_MS_FORM = 2, the default).  At limb L-2 both
// terms of accumulator l share the factor C[l][L-2] (C[l][L-1] =
// C[l][L-2] q_{L-1}^{-1}), so
//   acc_l = ((h_{L-1} - r_{L-1}) q_{L-1}^{-1} + h_{L-2} - r_{L-2}) C[l][L-2]:
// the inner Shoup product t lies in [0, 2q_l), and t + (h_{L-2} + q_l) - r
// (>= 0 because r < q_{L-2} < 2 q_l gives r <= h + q_l; < 3 q_l + q/2 <
// 2^32) goes straight into the outer one; later limbs J < L-2 add
// (h_J - r_J) C[l][J].  Limb 0's final value is the response word.
// Alternatives kept for A/B timing: WALLY_MS_FORM = 0, the additive form
// at every limb (four ALU instructions per term instead of two at limb
// L-2); = 1, the Horner form acc_l <- (acc_l + h_J - r_J) q_J^{-1} at every
// limb (identical at L = 3).  c4: 71.4 / 71.3 / 70.7 ms for forms 0 / 1 / 2.
// Element form of the recurrence (limb J; rtop / acc = this coefficient's
// state, NA = max(L - 2, 1) accumulators).  Ranges: the rounding residues
// (rtop, r) and the response word are canonical; the accumulators lie in
// [0, 2q_l).  a is consumed: for J > 0 only its residue r is kept.
#ifndef WALLY_MS_FORM
#define WALLY_MS_FORM 2
#endif
// the generic kernels (eval_kernel, eval_kernel_grp: up to 255 registers, both
// components per thread) keep the additive form with reduced residues
#ifndef WALLY_MS_FORM_GENERIC
#define WALLY_MS_FORM_GENERIC -1
#endif
template <int L, int J, int NA, int FORM = WALLY_MS_FORM>
__device__ __forceinline__ void ms_elem(uint32_t &a, uint32_t &rtop, uint32_t (&acc)[NA], const KParams &kp) {
    constexpr bool LZ = FORM >= 0;                                   // FORM = -1: additive form, reduced residues
    const uint32_t qj = kp.q[J], qj2 = kp.q2[J];
    if constexpr (L == 1) {
        a = csub(a, qj);
    } else if constexpr (L == 2) {
        // two limbs: canonical steps (measured 1% faster on c5 than the lazy form)
        a = csub(a, qj);
        if constexpr (J == 1) rtop = csub(a + kp.h[1], qj);
        else a = csub(a + csub(ms_term<false>(rtop, kp.h[1], qj, kp.C[0][1], kp.Cp[0][1]), qj), qj);
    } else if constexpr (J == L - 1) {
        rtop = csub(csub(a + kp.h[J], qj2), qj);                    // a + h < 2.5 q
    } else {
        uint32_t A;                                                  // [0, 2q)
        if constexpr (J == L - 2)
            A = ms_term<LZ>(rtop, kp.h[L - 1], qj, kp.C[J][L - 1], kp.Cp[J][L - 1]);
        else
            A = acc[J];
        if constexpr (J > 0) {
            const uint32_t r = csub(csub(a + csub(A, qj) + kp.h[J], qj2), qj);   // < 2q + q + q/2
#pragma unroll
            for (int l = 0; l < J; l++) {
                const uint32_t ql = kp.q[l];
                if constexpr (FORM == 1) {
                    // acc_l (after limb L-1: (h_{L-1} - r_{L-1}) q_{L-1}^{-1}) <- (acc_l + h_J - r_J) q_J^{-1}
                    const uint32_t base =
                        (J == L - 2) ? ms_term(rtop, kp.h[L - 1], ql, kp.Qi[l][L - 1], kp.Qip[l][L - 1]) : acc[l];
                    acc[l] = shoup_mul(base + (kp.h[J] + ql) - r, kp.Qi[l][J], kp.Qip[l][J], ql);
                } else if constexpr (FORM == 2 && J == L - 2) {
                    // nested at limb L-2 only: acc_l = ((h_{L-1} - r_{L-1}) q_{L-1}^{-1} + h_J - r_J) C[l][J],
                    // later limbs add their terms
                    const uint32_t t = ms_term(rtop, kp.h[L - 1], ql, kp.Qi[l][L - 1], kp.Qip[l][L - 1]);
                    acc[l] = shoup_mul(t + (kp.h[J] + ql) - r, kp.C[l][J], kp.Cp[l][J], ql);
                } else {
                    const uint32_t term = ms_term<LZ>(r, kp.h[J], ql, kp.C[l][J], kp.Cp[l][J]);
                    const uint32_t prev =
                        (J == L - 2) ? ms_term<LZ>(rtop, kp.h[L - 1], ql, kp.C[l][L - 1], kp.Cp[l][L - 1]) : acc[l];
                    acc[l] = csub(prev + term, kp.q2[l]);           // < 4 q -> [0, 2q)
                }
            }
        } else {
            a = csub(csub(a + A, qj2), qj);                          // < 4 q -> canonical response word
        }
    }
}

template <int L, int J, int V, int FORM = WALLY_MS_FORM, int NA>
__device__ __forceinline__ void ms_step(uint32_t (&a)[V], uint32_t (&rtop)[V], uint32_t (&acc)[NA][V],
                                        const KParams &kp) {
#pragma unroll
    for (int v = 0; v < V; v++) {
        uint32_t ac[NA];
#pragma unroll
        for (int l = 0; l < NA; l++) ac[l] = acc[l][v];
        ms_elem<L, J, NA, FORM>(a[v], rtop[v], ac, kp);
#pragma unroll
        for (int l = 0; l < NA; l++) acc[l][v] = ac[l];
    }
}

// Per-thread state of NC polynomials (the NC ciphertext components a thread
// carries through all limbs).
template <int N, int L, int NC>
struct EvalState {
    static constexpr int V = NttGeom<N>::V;
    static constexpr int NA = (L > 2) ? (L - 2) : 1;
    uint32_t a[NC][V];
    uint32_t rtop[NC][V];
    uint32_t acc[NC][NA][V];
};

// Where the inverse transform of one limb gets its twiddles and exchange
// buffers: GRP = false -> whole-CTA chain, global twiddles, double buffers;
// GRP = true -> one thread group of a multi-group CTA, twiddles in shared
// memory, one buffer per polynomial, named barrier `bar`.
struct ChainCtx {
    const uint2 *tw;      // inverse twiddles of limb 0 (global or shared)
    uint32_t *bufA, *bufB;
    int bar;
};

// One limb of the fused computation for NC components of one query:
// pointwise product with the NTT-domain plaintext, inverse NTT (shared
// twiddles), modulus-switch step.
template <int N, int L, int NC, int J, bool GRP>
__device__ __forceinline__ void eval_limb(EvalState<N, L, NC> &st, const BatchArgs &ba, const uint32_t *chat_q,
                                          int comp0, const uint32_t *phat, int g, const ChainCtx &cx) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    const uint32_t q = ba.kp.q[J], q2 = ba.kp.q2[J];
    const uint32_t *pv = phat + (size_t)J * 2 * N;
#pragma unroll
    for (int v = 0; v < V / 4; v++) {
        if constexpr (PtStore<N>::MONT) {
            const uint32_t qi = ba.kp.mqinv[J];
            const uint4 pm = ldg_stream(phat + pt_mont_word<N>(0, L, J, g, v));   // phat: pair base + parity
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const uint4 x = ldg_stream(chat_q + chat_word<N>(L, comp0 + c, J, g, v));
                st.a[c][4 * v + 0] = mont_mul(x.x, pm.x, q, qi);
                st.a[c][4 * v + 1] = mont_mul(x.y, pm.y, q, qi);
                st.a[c][4 * v + 2] = mont_mul(x.z, pm.z, q, qi);
                st.a[c][4 * v + 3] = mont_mul(x.w, pm.w, q, qi);
            }
        } else {
            const uint4 p = ldg_stream(pv + ntt_word<N>(g, v)), pp = ldg_stream(pv + N + ntt_word<N>(g, v));
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const uint4 x = ldg_stream(chat_q + chat_word<N>(L, comp0 + c, J, g, v));
                st.a[c][4 * v + 0] = shoup_mul(x.x, p.x, pp.x, q);
                st.a[c][4 * v + 1] = shoup_mul(x.y, p.y, pp.y, q);
                st.a[c][4 * v + 2] = shoup_mul(x.z, p.z, pp.z, q);
                st.a[c][4 * v + 3] = shoup_mul(x.w, p.w, pp.w, q);
            }
        }
    }
    if constexpr (GRP)
        intt_chain_group<N, NC>(st.a, cx.tw + (size_t)J * Gm::TW_LIMB, g, q, q2, cx.bufA, cx.bar);
    else
        intt_chain<N, NC>(st.a, cx.tw + (size_t)J * Gm::TW_LIMB, g, q, q2, cx.bufA, cx.bufB);
#pragma unroll
    for (int c = 0; c < NC; c++) ms_step<L, J, V, WALLY_MS_FORM_GENERIC>(st.a[c], st.rtop[c], st.acc[c], ba.kp);
}

template <int N, int L, int NC, int J, bool GRP>
struct LimbLoop {
    static __device__ __forceinline__ void run(EvalState<N, L, NC> &st, const BatchArgs &ba, const uint32_t *chat_q,
                                               int comp0, const uint32_t *phat, int g, const ChainCtx &cx) {
        eval_limb<N, L, NC, J, GRP>(st, ba, chat_q, comp0, phat, g, cx);
        if constexpr (J > 0) LimbLoop<N, L, NC, J - 1, GRP>::run(st, ba, chat_q, comp0, phat, g, cx);
    }
};

// Components per thread: both (c0, c1) share twiddle and plaintext loads and
// double the independent butterflies per stage; at n = 8192 (32 values per
// thread per component) one component per thread keeps registers in budget.
template <int N>
struct EvalCfg {
    static constexpr int NC = (N <= 4096) ? 2 : 1;
#ifdef WALLY_EVAL_MINB
    static constexpr int MINB = WALLY_EVAL_MINB;
#else
    static constexpr int MINB = (N <= 4096) ? 2 : 1;
#endif
};

// Work item -> (local cluster, plaintext, query range).  Items of one
// cluster are consecutive, so the cluster found for the previous item is
// checked before falling back to a binary search over item_start.
struct ItemCursor {
    uint32_t li = 0, b = 1, e = 0;  // item range [b, e) of cluster li (empty at start)
    __device__ __forceinline__ void seek(const BatchArgs &ba, uint32_t item) {
        if (item >= b && item < e) return;
        uint32_t lo = 0, hi = ba.n_local;  // item_start[lo] <= item < item_start[hi]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ba.item_start[mid] <= item) lo = mid; else hi = mid;
        }
        li = lo;
        b = ba.item_start[lo];
        e = ba.item_start[lo + 1];
    }
};

// Compact responses (WALLY_RESP_COMPACT): which of a thread's pass-2 output
// elements are result coefficients j*d + d - 1.  In pass-2 group jj the
// thread holds positions base + kk*TB2 (kk < R2); the solutions of
// pos = d - 1 (mod d) form an arithmetic progression in kk, whose j = (pos+1)/d - 1
// step is TB2 / gcd(TB2, d).  Per (group, thread) one word (j0 << 16) | mask,
// built once per CTA into shared memory.
template <int N>
struct ResultMap {
    static constexpr int G2 = NttGeom<N>::V / NttGeom<N>::R2;
    static constexpr int WORDS = G2 * NttGeom<N>::T;
};

template <int N>
__device__ __forceinline__ void build_result_map(uint32_t *s_rmap, uint32_t d) {
    using Gm = NttGeom<N>;
    for (int i = threadIdx.x; i < ResultMap<N>::WORDS; i += blockDim.x) {
        const int jj = i / Gm::T, gg = i % Gm::T;
        uint32_t mask = 0, j0 = 0;
#pragma unroll 1
        for (int kk = Gm::R2 - 1; kk >= 0; kk--) {
            const uint32_t pos = pass_index<N, Gm::TB2, Gm::R2>(gg, jj, kk);
            if ((pos + 1) % d == 0) {
                mask |= 1u << kk;
                j0 = (pos + 1) / d - 1;
            }
        }
        s_rmap[i] = (j0 << 16) | mask;
    }
}

__device__ __forceinline__ uint32_t result_map_dj(int tb2, uint32_t d) {
    const uint32_t low = d & (~d + 1u);  // largest power of two dividing d
    return (uint32_t)tb2 / min((uint32_t)tb2, low);
}

template <int N>
__device__ __forceinline__ void write_results(uint32_t *dst, const uint32_t (&a)[NttGeom<N>::V], const uint32_t *s_rmap,
                                              int g, uint32_t dj, const uint32_t *bc_base = nullptr,
                                              uint64_t bc_words = 0) {
    using Gm = NttGeom<N>;
#pragma unroll
    for (int jj = 0; jj < ResultMap<N>::G2; jj++) {
        const uint32_t m = s_rmap[jj * Gm::T + g];
        if (m & 0xffffu) {
            uint32_t j = m >> 16;
#pragma unroll
            for (int kk = 0; kk < Gm::R2; kk++)
                if ((m >> kk) & 1u) {
                    WALLY_BC(dst + j, bc_base, bc_words, "compact c0 store");
                    __stcs(dst + j, a[jj * Gm::R2 + kk]);
                    j += dj;
                }
        }
    }
}

// Write one ciphertext component of a pair's response in the context's
// format (include/wally.h "Response formats"); a = the component's values
// in the pass-2 layout, canonical mod q_0.
// FMT = WALLY_RESP_* when known at compile time (the v4 kernel is
// instantiated per format), -1 = read it from ba at run time.
template <int N, int FMT = -1>
__device__ __forceinline__ void write_component(const BatchArgs &ba, uint32_t *out_q, const uint32_t (&a)[NttGeom<N>::V],
                                                int comp, int g, const uint32_t *s_rmap) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    const bool compact = (FMT < 0) ? (bool)ba.compact : (FMT != (int)WALLY_RESP_FULL);
    const bool drop = (FMT < 0) ? (bool)ba.drop : (FMT == (int)WALLY_RESP_COMPACT_DROP);
    if (compact && comp == 0) {
        write_results<N>(out_q, a, s_rmap, g, result_map_dj(Gm::TB2, ba.d), ba.resp, ba.resp_words);
        const uint32_t e4 = (ba.E + 3) & ~3u;
        if ((uint32_t)g < e4 - ba.E) {
            WALLY_BC(out_q + ba.E + g, ba.resp, ba.resp_words, "compact c0 padding");
            __stcs(out_q + ba.E + g, 0u);  // zero padding to E4
        }
        return;
    }
    if constexpr (N == 4096 && (FMT < 0 || FMT == (int)WALLY_RESP_COMPACT_DROP)) {
        if (drop) {
            // c1 with its 6 LSBs dropped (rounded), 24-bit planes lo16 [N] and hi8 [N]
            // in the 16 x 256 transposed order (include/wally.h): this thread's
            // coefficients k*256 + g sit at positions g*16 + k, so it writes its 16
            // values as two 16-byte stores (lo) and one (hi) instead of 32 scalar ones
            static_assert(Gm::TB2 == 256 && Gm::R2 == 16 && V == 16, "transposed planes assume n = 4096 geometry");
            uint32_t *base = out_q + ((ba.E + 3) & ~3u);
            uint32_t h[16];
#pragma unroll
            for (int k = 0; k < 16; k++) h[k] = (a[k] + (1u << (WALLY_RESP_DROP_BITS - 1))) >> WALLY_RESP_DROP_BITS;
            uint4 *lo = reinterpret_cast<uint4 *>(base) + 2 * g;
            __stcs(lo, make_uint4(__byte_perm(h[0], h[1], 0x5410), __byte_perm(h[2], h[3], 0x5410),
                                  __byte_perm(h[4], h[5], 0x5410), __byte_perm(h[6], h[7], 0x5410)));
            __stcs(lo + 1, make_uint4(__byte_perm(h[8], h[9], 0x5410), __byte_perm(h[10], h[11], 0x5410),
                                      __byte_perm(h[12], h[13], 0x5410), __byte_perm(h[14], h[15], 0x5410)));
            uint32_t hw[4];
#pragma unroll
            for (int i = 0; i < 4; i++)
                hw[i] = __byte_perm(__byte_perm(h[4 * i], h[4 * i + 1], 0x0062), __byte_perm(h[4 * i + 2], h[4 * i + 3], 0x0062),
                                    0x5410);
            __stcs(reinterpret_cast<uint4 *>(base + N / 2) + g, make_uint4(hw[0], hw[1], hw[2], hw[3]));
            return;
        }
    }
    uint32_t *dst = out_q + (compact ? (size_t)(ba.wpp - N) : (size_t)comp * N);
#pragma unroll
    for (int j = 0; j < V / Gm::R2; j++)
#pragma unroll
        for (int kk = 0; kk < Gm::R2; kk++) {
            WALLY_BC((dst + pass_index<N, Gm::TB2, Gm::R2>(g, j, kk)), ba.resp, ba.resp_words, "full store");
            __stcs(dst + pass_index<N, Gm::TB2, Gm::R2>(g, j, kk), a[j * Gm::R2 + kk]);
        }
}

// Evaluate work item `item` (cursor already positioned) for one thread group.
template <int N, int L, bool GRP>
__device__ __forceinline__ void eval_item(const BatchArgs &ba, const ItemCursor &cur, uint32_t item, int g,
                                          const ChainCtx &cx, const uint32_t *s_rmap) {
    constexpr int NC = EvalCfg<N>::NC;
    const uint32_t li = cur.li;
    const uint32_t cnt = ba.counts[li];
    const uint32_t local = item - cur.b;
    // chunk-major: the items of one query chunk are its P_c plaintexts in a
    // row, so the chunk's query NTTs stay in L2 while the plaintexts stream
    // (a hot cluster's queries can exceed L2; its plaintexts never do)
    const uint32_t P = ba.n_pt[li];
    const uint32_t ch = local / P, k = local % P;
    const uint32_t qb = ba.seg[li] + ch * ba.chunk;
    const uint32_t qe = min(qb + ba.chunk, ba.seg[li] + cnt);
    const size_t pt = (size_t)ba.pt_base[li] + k;
    const uint32_t *phat = PtStore<N>::MONT ? ba.store + pt_mont_word<N>(pt, L, 0, 0, 0) : ba.store + pt * L * 2 * N;
    for (uint32_t qi = qb; qi < qe; qi++) {
        const uint32_t qo = ba.perm[qi];
        uint32_t *out_q = ba.resp + ba.resp_off[qo] + (size_t)k * ba.wpp;
        const uint32_t *chat_q = ba.chat + (size_t)qo * 2 * L * N;
#pragma unroll 1
        for (int comp0 = 0; comp0 < 2; comp0 += NC) {
            EvalState<N, L, NC> st;
            LimbLoop<N, L, NC, L - 1, GRP>::run(st, ba, chat_q, comp0, phat, g, cx);
#pragma unroll
            for (int c = 0; c < NC; c++) write_component<N>(ba, out_q, st.a[c], comp0 + c, g, s_rmap);
        }
    }
}

// Fused kernel, whole-CTA form (used for n = 8192: twiddles from global
// memory through L1, double-buffered exchange).
template <int N, int L>
__global__ void __launch_bounds__(NttGeom<N>::T, EvalCfg<N>::MINB) eval_kernel(BatchArgs ba) {
    using Gm = NttGeom<N>;
    constexpr int NC = EvalCfg<N>::NC;
    extern __shared__ uint32_t smem[];
    ChainCtx cx{ba.tw_inv, smem, smem + NC * Gm::SMEM_WORDS, 0};
    __shared__ uint32_t s_item[2];
    __shared__ uint32_t s_rmap[ResultMap<N>::WORDS];
    if (ba.compact) build_result_map<N>(s_rmap, ba.d);
    const int g = threadIdx.x;
    const uint32_t total = ba.misc[kMiscTotalItems];
    ItemCursor cur;
    for (uint32_t it = 0;; it++) {
        if (g == 0) s_item[it & 1] = atomicAdd(&ba.misc[kMiscWorkCounter], 1u);
        __syncthreads();
        const uint32_t item = s_item[it & 1];
        if (item >= total) break;
        cur.seek(ba, item);
        eval_item<N, L, false>(ba, cur, item, g, cx, s_rmap);
    }
}

// Fused kernel, grouped form (n <= 4096): a CTA holds GROUPS independent
// T-thread groups that share the limbs' inverse twiddle tables staged once
// in shared memory; each group pulls its own work items (fetching the next
// item index one item ahead) and synchronises with its own named barrier.
constexpr int kEvalGroups = 2;

template <int N, int L>
__global__ void __launch_bounds__(kEvalGroups * NttGeom<N>::T, 1) eval_kernel_grp(BatchArgs ba) {
    using Gm = NttGeom<N>;
    constexpr int NC = EvalCfg<N>::NC;
    constexpr int T = Gm::T;
    extern __shared__ uint4 smem4[];
    uint2 *tw = reinterpret_cast<uint2 *>(smem4);
    uint32_t *xbuf = reinterpret_cast<uint32_t *>(tw + L * Gm::TW_LIMB);
    __shared__ uint32_t s_item[kEvalGroups][2];
    __shared__ uint32_t s_rmap[ResultMap<N>::WORDS];
    const int grp = threadIdx.x / T, g = threadIdx.x % T;
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(ba.tw_inv);
        for (int i = threadIdx.x; i < L * Gm::TW_LIMB / 2; i += blockDim.x) smem4[i] = __ldg(src + i);
    }
    if (ba.compact) build_result_map<N>(s_rmap, ba.d);
    if (g == 0) s_item[grp][0] = atomicAdd(&ba.misc[kMiscWorkCounter], 1u);
    __syncthreads();
    const ChainCtx cx{tw, xbuf + grp * NC * Gm::SMEM_WORDS, nullptr, 1 + grp};
    const uint32_t total = ba.misc[kMiscTotalItems];
    ItemCursor cur;
    for (uint32_t it = 0;; it++) {
        const uint32_t item = s_item[grp][it & 1];
        if (item >= total) break;
        uint32_t next = 0;
        if (g == 0) next = atomicAdd(&ba.misc[kMiscWorkCounter], 1u);
        cur.seek(ba, item);
        eval_item<N, L, true>(ba, cur, item, g, cx, s_rmap);
        if (g == 0) s_item[grp][(it + 1) & 1] = next;
        group_sync(1 + grp, T);
    }
}


// ---------------------------------------------------------------------------
// Fused kernel v4 (n <= 4096, L <= 3): tensor memory as the per-thread store
// of everything that is reused across limbs but not needed in registers
// during the inverse NTT.  TMEM is 128 lanes x 512 32-bit columns per SM;
// warp w reaches lanes 32 (w % 4) .. +31, so each thread owns one lane and,
// with 16 warps, 128 private columns:
//   columns [32 J, 32 J + 16)        the work item's plaintext, limb J, NTT values
//   columns [32 J + 16, 32 J + 32)   their Shoup companions          (J < L <= 3)
//   columns [96 + 16 c, 96 + 16 c + 16)  modulus-switch state of component c
// The plaintext slice is copied in once per work item (shared by its <= 8
// queries and both components); the mod-switch state (rtop / acc of the
// drop-last recurrence) goes to TMEM between limbs.  The registers this frees
// hold the next limb's query operands, prefetched from L2 while the current
// limb's inverse NTT runs -- the global-load latency ncu showed as the top
// stall of v2 (profiles/r01_ncu_eval_v2.txt).  Measured TMEM read bandwidth:
// 446 B/clk/SM (profiles/r01_intpipe_v2.jsonl), far above what this needs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_wait_ld2(uint32_t (&r)[16], uint32_t (&s)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(s[0]), "+r"(s[1]), "+r"(s[2]), "+r"(s[3]), "+r"(s[4]), "+r"(s[5]), "+r"(s[6]), "+r"(s[7]), "+r"(s[8]), "+r"(s[9]), "+r"(s[10]), "+r"(s[11]), "+r"(s[12]), "+r"(s[13]), "+r"(s[14]), "+r"(s[15])
                 :
                 : "memory");
}

template <int N, int L, int J>
struct LimbLoopTM {
    static constexpr int NC = 2;
    static __device__ __forceinline__ void run(EvalState<N, L, NC> &st, uint4 (&cpre)[NC][NttGeom<N>::V / 4],
                                               const BatchArgs &ba, const uint32_t *chat_q,
                                               uint32_t qn, const uint32_t *chat_next, uint32_t tcol, int g,
                                               const ChainCtx &cx) {
        using Gm = NttGeom<N>;
        constexpr int V = Gm::V;
        static_assert(V == 16, "v4 layout assumes 16 values per thread");
        const uint32_t q = ba.kp.q[J], q2 = ba.kp.q2[J];
        {
            uint32_t p[16], pp[16];
            tmem_ld<16>(tcol + 32 * J, p);
            tmem_ld<16>(tcol + 32 * J + 16, pp);
            tmem_wait_ld2(p, pp);
#pragma unroll
            for (int v = 0; v < V / 4; v++)
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    st.a[c][4 * v + 0] = shoup_mul(cpre[c][v].x, p[4 * v + 0], pp[4 * v + 0], q);
                    st.a[c][4 * v + 1] = shoup_mul(cpre[c][v].y, p[4 * v + 1], pp[4 * v + 1], q);
                    st.a[c][4 * v + 2] = shoup_mul(cpre[c][v].z, p[4 * v + 2], pp[4 * v + 2], q);
                    st.a[c][4 * v + 3] = shoup_mul(cpre[c][v].w, p[4 * v + 3], pp[4 * v + 3], q);
                }
        }
        // prefetch the operands of the next limb (or of the next query's first limb)
        // (the guard is the integer test on qn, not a nullable pointer: ptxas 12.9 turned
        // `chat_next ? ... : nullptr` into CS2R Rd, SRZ; @P IMAD.WIDE Rd; ISETP Rd != 0 with the
        // compare five cycles after the CS2R, which on the B200 still read the register's old
        // value -- the "null" pointer then passed the test and the loads faulted)
        if (J > 0 || qn != 0xffffffffu) {
            const uint32_t *nsrc = (J > 0) ? chat_q + (size_t)(J - 1) * N : chat_next + (size_t)(L - 1) * N;
#pragma unroll
            for (int c = 0; c < NC; c++)
#pragma unroll
                for (int v = 0; v < V / 4; v++) {
                    WALLY_BC(nsrc + (size_t)c * L * N + (size_t)g * V + 4 * v + 3, ba.chat, (size_t)ba.nq * 2 * L * N, "tm cpre");
                    cpre[c][v] = ldg_stream(nsrc + (size_t)c * L * N + (size_t)g * V + 4 * v);
                }
        }
        intt_chain_group<N, NC>(st.a, cx.tw + (size_t)J * Gm::TW_LIMB, g, q, q2, cx.bufA, cx.bar);
        // mod-switch state through TMEM between limbs (its registers are what the
        // chat prefetch needs).  At L = 2 the single 16-word state went through
        // registers until the end of round 2, because this variant faulted on the
        // B200; the fault was the null-pointer guard above, not tensor memory
        // (DESIGN.md section 14), and with it fixed the TMEM state is 6% faster
        // (c5 full responses 95.1 -> 89.1 ms).  WALLY_TM_L2_TMEM = 0 restores the
        // register form for A/B timing.
#ifndef WALLY_TM_L2_TMEM
#define WALLY_TM_L2_TMEM 1
#endif
        constexpr uint32_t TM_STATE_COL = 96;
        if constexpr (L == 3 || (L == 2 && WALLY_TM_L2_TMEM)) {
            if constexpr (J < L - 1) {
                // state written at limb J + 1: rtop (J == L - 2) or acc (J < L - 2)
                tmem_wait_st_all();
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    if constexpr (J == L - 2) tmem_ld<16>(tcol + TM_STATE_COL + 16 * c, st.rtop[c]);
                    else tmem_ld<16>(tcol + TM_STATE_COL + 16 * c, st.acc[c][0]);
                }
#pragma unroll
                for (int c = 0; c < NC; c++) {
                    if constexpr (J == L - 2) tmem_wait_ld<16>(st.rtop[c]);
                    else tmem_wait_ld<16>(st.acc[c][0]);
                }
            }
#pragma unroll
            for (int c = 0; c < NC; c++) ms_step<L, J, V>(st.a[c], st.rtop[c], st.acc[c], ba.kp);
            if constexpr (J == L - 1) {
#pragma unroll
                for (int c = 0; c < NC; c++) tmem_st<16>(tcol + TM_STATE_COL + 16 * c, st.rtop[c]);
            } else if constexpr (J > 0) {
#pragma unroll
                for (int c = 0; c < NC; c++) tmem_st<16>(tcol + TM_STATE_COL + 16 * c, st.acc[c][0]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NC; c++) ms_step<L, J, V>(st.a[c], st.rtop[c], st.acc[c], ba.kp);
        }
        if constexpr (J > 0) LimbLoopTM<N, L, J - 1>::run(st, cpre, ba, chat_q, qn, chat_next, tcol, g, cx);
    }
};

template <int N, int L, int FMT>
__device__ __forceinline__ void eval_item_tm(const BatchArgs &ba, const ItemCursor &cur, uint32_t item, int g,
                                             const ChainCtx &cx, const uint32_t *s_rmap, uint32_t tcol,
                                             const volatile uint32_t *s_next, ItemCursor &ncur) {
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V, NC = 2;
    static_assert(!NttStore<N>::CHUNK_MAJOR, "thread-major NTT-domain storage (ntt_word)");
    const uint32_t li = cur.li;
    const uint32_t cnt = ba.counts[li];
    const uint32_t local = item - cur.b;
    // chunk-major: the items of one query chunk are its P_c plaintexts in a
    // row, so the chunk's query NTTs stay in L2 while the plaintexts stream
    // (a hot cluster's queries can exceed L2; its plaintexts never do)
    const uint32_t P = ba.n_pt[li];
    const uint32_t ch = local / P, k = local % P;
    const uint32_t qb = ba.seg[li] + ch * ba.chunk;
    const uint32_t qe = min(qb + ba.chunk, ba.seg[li] + cnt);
    const uint32_t *phat = ba.store + (size_t)(ba.pt_base[li] + k) * L * 2 * N;
    // the item's plaintext slice -> TMEM (previous item's reads were waited on)
#pragma unroll
    for (int J = 0; J < L; J++) {
        uint32_t p[16], pp[16];
        const uint32_t *pv = phat + (size_t)J * 2 * N + (size_t)g * V;
#pragma unroll
        for (int v = 0; v < 4; v++) {
            WALLY_BC(pv + N + 4 * v + 3, ba.store, ba.store_words, "tm plaintext");
            const uint4 x = ldg_stream(pv + 4 * v), y = ldg_stream(pv + N + 4 * v);
            p[4 * v] = x.x; p[4 * v + 1] = x.y; p[4 * v + 2] = x.z; p[4 * v + 3] = x.w;
            pp[4 * v] = y.x; pp[4 * v + 1] = y.y; pp[4 * v + 2] = y.z; pp[4 * v + 3] = y.w;
        }
        tmem_st<16>(tcol + 32 * J, p);
        tmem_st<16>(tcol + 32 * J + 16, pp);
    }
    tmem_wait_st_all();
    uint32_t qo = ba.perm[qb];
    uint4 cpre[NC][V / 4];
    {
        const uint32_t *src = ba.chat + (size_t)qo * 2 * L * N + (size_t)(L - 1) * N;
#pragma unroll
        for (int c = 0; c < NC; c++) {
#pragma unroll
            for (int v = 0; v < V / 4; v++) WALLY_BC(src + (size_t)c * L * N + (size_t)g * V + 4 * v + 3, ba.chat, (size_t)ba.nq * 2 * L * N, "tm cpre0");
#pragma unroll
            for (int v = 0; v < V / 4; v++) cpre[c][v] = ldg_stream(src + (size_t)c * L * N + (size_t)g * V + 4 * v);
        }
    }
    for (uint32_t qi = qb; qi < qe; qi++) {
        const uint32_t qn = (qi + 1 < qe) ? ba.perm[qi + 1] : 0xffffffffu;
        uint32_t *out_q = ba.resp + ba.resp_off[qo] + (size_t)k * ba.wpp;
        const uint32_t *chat_q = ba.chat + (size_t)qo * 2 * L * N;
        // always a valid pointer (the next query's operands, else this query's again); qn guards its use
        const uint32_t *chat_next = ba.chat + (size_t)(qn != 0xffffffffu ? qn : qo) * 2 * L * N;
        EvalState<N, L, NC> st;
        LimbLoopTM<N, L, L - 1>::run(st, cpre, ba, chat_q, qn, chat_next, tcol, g, cx);
        if (qi == qb) {
            // the group's next work item was published before this item started
            // (and the limb loop passed group barriers): pull this thread's slice of
            // its plaintext toward L2 now -- each plaintext is read by one item only,
            // so its first touch is an HBM miss the item start would otherwise wait on
            const uint32_t nitem = *s_next;
            if (nitem < ba.misc[kMiscTotalItems]) {
                ncur.seek(ba, nitem);
                const uint32_t nli = ncur.li;
                const uint32_t nk = (nitem - ncur.b) % ba.n_pt[nli];
                const uint32_t *np = ba.store + (size_t)(ba.pt_base[nli] + nk) * L * 2 * N + (size_t)g * V;
#pragma unroll
                for (int J = 0; J < L; J++) {
                    WALLY_BC(np + (size_t)J * 2 * N + N, ba.store, ba.store_words, "tm L2 prefetch");
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(np + (size_t)J * 2 * N));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(np + (size_t)J * 2 * N + N));
                }
            }
        }
#pragma unroll
        for (int c = 0; c < NC; c++) write_component<N, FMT>(ba, out_q, st.a[c], c, g, s_rmap);
        qo = qn;
    }
}

template <int N, int L, int FMT>
__global__ void __launch_bounds__(kEvalGroups * NttGeom<N>::T, 1) eval_kernel_tm(BatchArgs ba) {
    using Gm = NttGeom<N>;
    constexpr int NC = 2;
    constexpr int T = Gm::T;
    extern __shared__ uint4 smem4[];
    uint2 *tw = reinterpret_cast<uint2 *>(smem4);
    uint32_t *xbuf = reinterpret_cast<uint32_t *>(tw + L * Gm::TW_LIMB);
    __shared__ uint32_t s_item[kEvalGroups][2];
    __shared__ uint32_t s_rmap[ResultMap<N>::WORDS];
    __shared__ uint32_t s_taddr;
    const int grp = threadIdx.x / T, g = threadIdx.x % T;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_taddr);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(ba.tw_inv);
        for (int i = threadIdx.x; i < L * Gm::TW_LIMB / 2; i += blockDim.x) smem4[i] = __ldg(src + i);
    }
    if (FMT != (int)WALLY_RESP_FULL) build_result_map<N>(s_rmap, ba.d);
    if (g == 0) s_item[grp][0] = atomicAdd(&ba.misc[kMiscWorkCounter], 1u);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tcol = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
    const ChainCtx cx{tw, xbuf + grp * NC * Gm::SMEM_WORDS, nullptr, 1 + grp};
    const uint32_t total = ba.misc[kMiscTotalItems];
    ItemCursor cur, ncur;
    for (uint32_t it = 0;; it++) {
        const uint32_t item = s_item[grp][it & 1];
        if (item >= total) break;
        // slot (it+1)&1 was last read at the start of iteration it-1 (group barrier since)
        if (g == 0) s_item[grp][(it + 1) & 1] = atomicAdd(&ba.misc[kMiscWorkCounter], 1u);
        cur.seek(ba, item);
        eval_item_tm<N, L, FMT>(ba, cur, item, g, cx, s_rmap, tcol, &s_item[grp][(it + 1) & 1], ncur);
        cur = ncur;
        group_sync(1 + grp, T);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_taddr) : "memory");
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int N>
static constexpr size_t chain_smem(int nc = 1) { return 2 * (size_t)nc * NttGeom<N>::SMEM_WORDS * sizeof(uint32_t); }

template <typename K>
static cudaError_t allow_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int N>
static cudaError_t launch_encode_n(const EncodeArgs &a, cudaStream_t s) {
    dim3 grid(a.npt, a.L);
    cudaError_t e = allow_smem(encode_kernel<N>, chain_smem<N>());
    if (e != cudaSuccess) return e;
    encode_kernel<N><<<grid, NttGeom<N>::T, chain_smem<N>(), s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_encode(const EncodeArgs &a, cudaStream_t s, uint64_t *launches) {
    if (a.npt == 0) return cudaSuccess;
    *launches += 1;
    switch (a.n) {
        case 1024: return launch_encode_n<1024>(a, s);
        case 2048: return launch_encode_n<2048>(a, s);
        case 4096: return launch_encode_n<4096>(a, s);
        case 8192: return launch_encode_n<8192>(a, s);
    }
    return cudaErrorInvalidValue;
}

template <int N>
static cudaError_t launch_fwd_n(const KParams &kp, uint32_t L, const uint2 *tw, const uint32_t *in, uint32_t *out,
                                uint32_t count, uint32_t *err, cudaStream_t s, bool chat) {
    if (chat) {
        cudaError_t e = allow_smem(ntt_forward_kernel<N, true>, chain_smem<N>());
        if (e != cudaSuccess) return e;
        ntt_forward_kernel<N, true><<<(unsigned)(count * L), NttGeom<N>::T, chain_smem<N>(), s>>>(kp, L, tw, in, out, err);
    } else {
        cudaError_t e = allow_smem(ntt_forward_kernel<N, false>, chain_smem<N>());
        if (e != cudaSuccess) return e;
        ntt_forward_kernel<N, false><<<(unsigned)(count * L), NttGeom<N>::T, chain_smem<N>(), s>>>(kp, L, tw, in, out, err);
    }
    return cudaGetLastError();
}

cudaError_t launch_ntt_forward(const KParams &kp, uint32_t n, uint32_t L, const uint2 *tw_fwd, const uint32_t *in,
                               uint32_t *out, uint32_t count, uint32_t *err, cudaStream_t s, uint64_t *launches,
                               bool chat) {
    if (count == 0) return cudaSuccess;
    *launches += 1;
    switch (n) {
        case 1024: return launch_fwd_n<1024>(kp, L, tw_fwd, in, out, count, err, s, chat);
        case 2048: return launch_fwd_n<2048>(kp, L, tw_fwd, in, out, count, err, s, chat);
        case 4096: return launch_fwd_n<4096>(kp, L, tw_fwd, in, out, count, err, s, chat);
        case 8192: return launch_fwd_n<8192>(kp, L, tw_fwd, in, out, count, err, s, chat);
    }
    return cudaErrorInvalidValue;
}

template <int N>
static cudaError_t launch_inv_n(const KParams &kp, uint32_t L, const uint2 *tw, const uint32_t *in, uint32_t *out,
                                uint32_t count, cudaStream_t s) {
    cudaError_t e = allow_smem(ntt_inverse_kernel<N>, chain_smem<N>());
    if (e != cudaSuccess) return e;
    ntt_inverse_kernel<N><<<(unsigned)(count * L), NttGeom<N>::T, chain_smem<N>(), s>>>(kp, L, tw, in, out);
    return cudaGetLastError();
}

cudaError_t launch_ntt_inverse(const KParams &kp, uint32_t n, uint32_t L, const uint2 *tw_inv, const uint32_t *in,
                               uint32_t *out, uint32_t count, cudaStream_t s, uint64_t *launches) {
    if (count == 0) return cudaSuccess;
    *launches += 1;
    switch (n) {
        case 1024: return launch_inv_n<1024>(kp, L, tw_inv, in, out, count, s);
        case 2048: return launch_inv_n<2048>(kp, L, tw_inv, in, out, count, s);
        case 4096: return launch_inv_n<4096>(kp, L, tw_inv, in, out, count, s);
        case 8192: return launch_inv_n<8192>(kp, L, tw_inv, in, out, count, s);
    }
    return cudaErrorInvalidValue;
}



// ---------------------------------------------------------------------------
// Fused kernel v6 (n = 4096, L <= 3, compact responses, 16 | d): pruned
// inverse NTT for c0.  A compact response keeps c0 only at the result
// coefficients j d + d - 1, all of which are = -1 (mod M), M = 2^v2(d).  In
// the Gentleman-Sande order used here (stage s pairs positions B + o and
// B + o + 2^s), those outputs need, at every stage s < log2 M, only the Y
// output of the last butterfly of each block, and at every later stage only
// the butterflies at offsets o = -1 (mod M): N/(2M) per stage.  For c3
// (d = 192, M = 64) that is 4,224 of c0's 24,576 butterflies per limb, and the
// modulus switch of c0 runs on N/M = 64 coefficients instead of 4,096 -- the
// pair's modular multiplications drop by about a third, with the compact
// response bit-identical (the oracle is compared at the result coefficients).
//   * pass 0 (stages 0..3): every thread keeps only its group's last Y
//     output (15 Shoup products instead of 32 butterflies), position 16 g + 15;
//   * stages 4..11 on those 256 values: warp 0 of the group, in shared memory,
//     twiddles from the plain merged table (global, L1-cached), then the
//     modulus switch of the N/M surviving coefficients (state in shared
//     memory), and after limb 0 the write of the E result words;
//   * c1 runs the full transform (NC = 1) of the v4 kernel, its plaintext
//     slice and (L = 3) mod-switch state in tensor memory.
// ---------------------------------------------------------------------------
// Pass-0 stage S of c0 keeping only the Y output of each block's last
// butterfly.  Thread g holds the V contiguous elements of its pass-0 group;
// twiddles from the pass-major pass-0 table (slot-pair-major), in shared
// memory (TWS) or global memory.
template <int N, int S, bool TWS>
__device__ __forceinline__ void c0_yonly_stage(uint32_t (&a)[NttGeom<N>::V], const uint2 *tw0, int g, uint32_t q,
                                               uint32_t q2) {
    using Gm = NttGeom<N>;
    constexpr int T = Gm::T, R = Gm::R0;
    constexpr int t = 1 << S, NB = R >> (S + 1), OFF = R - (R >> S);
    const uint4 *t4 = reinterpret_cast<const uint4 *>(tw0) + g;
    uint2 w[NB];
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
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const uint32_t X = a[b * 2 * t + t - 1], Y = a[b * 2 * t + 2 * t - 1];
        a[b * 2 * t + 2 * t - 1] = shoup_mul(X - Y + q2, w[b].x, w[b].y, q);
    }
}

template <int N, int S, bool TWS>
struct C0Pass0 {
    static __device__ __forceinline__ void run(uint32_t (&a)[NttGeom<N>::V], const uint2 *tw0, int g, uint32_t q,
                                               uint32_t q2) {
        c0_yonly_stage<N, S, TWS>(a, tw0, g, q, q2);
        if constexpr (S + 1 < NttCfg<N>::S0) C0Pass0<N, S + 1, TWS>::run(a, tw0, g, q, q2);
    }
};

// After pass 0 thread g keeps z[g] = x[V g + V - 1] (S_LO = log2 V).  The
// next five stages pair threads g and g ^ 2^(s - S_LO) inside a warp, one
// shuffle each.  mrg = the limb's merged inverse table entries 0..255
// (stage s uses entry N/2^(s+1) + block).  Requires mu >= S_LO.
template <int N, int S>
__device__ __forceinline__ uint32_t c0_mid_stage(uint32_t y, int g, int mu, const uint2 *mrg, uint32_t q, uint32_t q2) {
    constexpr int SLO = Log2<NttGeom<N>::V>::v;
    const int Mc = 1 << (mu - SLO);
    constexpr int D = 1 << (S - SLO), m = N >> (S + 1);
    const uint32_t other = __shfl_xor_sync(0xffffffffu, y, D);
    const bool upper = (g & D) != 0;
    const int o = g & (D - 1);
    const uint2 w = mrg[m + g / (2 * D)];
    if (S < mu) {
        if (upper && o == D - 1) y = shoup_mul(other - y + q2, w.x, w.y, q);
    } else if (((o + 1) & (Mc - 1)) == 0) {
        y = upper ? shoup_mul(other - y + q2, w.x, w.y, q) : csub(y + other, q2);
    }
    return y;
}

template <int N>
__device__ __forceinline__ uint32_t c0_mid(uint32_t y, int g, int mu, const uint2 *mrg, uint32_t q, uint32_t q2) {
    constexpr int SLO = Log2<NttGeom<N>::V>::v;
    const int Mc = 1 << (mu - SLO);
#pragma unroll
    for (int s = SLO; s < SLO + 5; s++) {
        const int D = 1 << (s - SLO), m = N >> (s + 1);
        const uint32_t other = __shfl_xor_sync(0xffffffffu, y, D);
        const bool upper = (g & D) != 0;
        const int o = g & (D - 1);                        // offset of the pair inside its block
        const uint2 w = mrg[m + g / (2 * D)];
        if (s < mu) {
            if (upper && o == D - 1) y = shoup_mul(other - y + q2, w.x, w.y, q);
        } else if (((o + 1) & (Mc - 1)) == 0) {
            y = upper ? shoup_mul(other - y + q2, w.x, w.y, q) : csub(y + other, q2);
        }
    }
    return y;
}

// The remaining stages S_LO + 5 .. log2 N - 1 of c0 on z[c] = x[V c + V - 1]
// (shared memory), then the modulus-switch step of limb J on the N/M
// surviving coefficients (state cst[k][1 + NA]).  Warp 0 only; lanes stride
// over butterflies / coefficients.  (A variant keeping these values in
// registers measured slower: 140 vs 110 ms on c3, from register pressure.)
template <int N, int L, int J>
__device__ __forceinline__ void c0_tail(uint32_t *z, uint32_t *cst, const uint2 *mrg, int lane, int mu,
                                        const KParams &kp) {
    constexpr int V = NttGeom<N>::V, SLO = Log2<V>::v, LOGN = Log2<N>::v;
    constexpr int NA = (L > 2) ? (L - 2) : 1;
    const uint32_t q = kp.q[J], q2 = kp.q2[J];
    const int M = 1 << mu, Mc = M >> SLO;
#pragma unroll 1
    for (int s = SLO + 5; s < LOGN; s++) {
        const int t = 1 << s, m = N / (2 * t);
        if (s < mu) {
            for (int blk = lane; blk < N / (2 * t); blk += 32) {
                const int B = blk * 2 * t;
                const int cx = (B + t - V) >> SLO, cy = (B + 2 * t - V) >> SLO;
                const uint2 w = mrg[m + blk];
                z[cy] = shoup_mul(z[cx] - z[cy] + q2, w.x, w.y, q);
            }
        } else {
            const int per = t / M;
            for (int i = lane; i < N / (2 * M); i += 32) {
                const int blk = i / per, o = M - 1 + (i % per) * M;
                const int B = blk * 2 * t;
                const int cx = (B + o - (V - 1)) >> SLO, cy = (B + o + t - (V - 1)) >> SLO;
                const uint2 w = mrg[m + blk];
                const uint32_t X = z[cx], Y = z[cy];
                z[cx] = csub(X + Y, q2);
                z[cy] = shoup_mul(X - Y + q2, w.x, w.y, q);
            }
        }
        __syncwarp();
    }
    for (int k = lane; k < N / M; k += 32) {
        const int c = k * Mc + Mc - 1;
        uint32_t x = z[c], rtop = cst[k * (1 + NA)], acc[NA];
#pragma unroll
        for (int l = 0; l < NA; l++) acc[l] = cst[k * (1 + NA) + 1 + l];
        ms_elem<L, J, NA>(x, rtop, acc, kp);
        cst[k * (1 + NA)] = rtop;
#pragma unroll
        for (int l = 0; l < NA; l++) cst[k * (1 + NA) + 1 + l] = acc[l];
        z[c] = x;
    }
    __syncwarp();
}

// c0 result words of one pair from the survivors of limb 0 (warp 0).
template <int N>
__device__ __forceinline__ void c0_write_results(const BatchArgs &ba, uint32_t *out_q, const uint32_t *z, int lane,
                                                 int mu) {
    constexpr int SLO = Log2<NttGeom<N>::V>::v;
    const int M = 1 << mu, Mc = M >> SLO;
    for (int kk = lane; kk < N / M; kk += 32) {
        const uint32_t pos1 = (uint32_t)(kk * M + M);
        if (pos1 % ba.d == 0) __stcs(out_q + pos1 / ba.d - 1, z[kk * Mc + Mc - 1]);
    }
    const uint32_t e4 = (ba.E + 3) & ~3u;
    if ((uint32_t)lane < e4 - ba.E) __stcs(out_q + ba.E + lane, 0u);
}

// Register tail for n = 4096 and mu = 6 (c3: d = 192) or mu = 7 (d = 128:
// c1, c2, c5): after stage 8 the survivors are c = k Mc + Mc - 1 (Mc = M/16),
// 64 or 32 of them; lane l holds k = l (and k = l + 32 for mu = 6), so
// stages 9..11 are lane shuffles (and, for mu = 6, one lane-local pair), and
// the modulus switch runs on the lane's one or two values.
template <int L, int J>
__device__ __forceinline__ void c0_tail_fast(uint32_t *z, uint32_t *cst, const uint2 *mrg, int lane, int mu,
                                             const KParams &kp) {
    constexpr int NA = (L > 2) ? (L - 2) : 1;
    const uint32_t q = kp.q[J], q2 = kp.q2[J];
    auto ms = [&](uint32_t &x, int k) {
        uint32_t rtop = cst[k * (1 + NA)], acc[NA];
#pragma unroll
        for (int l = 0; l < NA; l++) acc[l] = cst[k * (1 + NA) + 1 + l];
        ms_elem<L, J, NA>(x, rtop, acc, kp);
        cst[k * (1 + NA)] = rtop;
#pragma unroll
        for (int l = 0; l < NA; l++) cst[k * (1 + NA) + 1 + l] = acc[l];
    };
    auto bfly = [&](uint32_t &v, int xo, const uint2 w) {
        const uint32_t other = __shfl_xor_sync(0xffffffffu, v, xo);
        v = (lane & xo) ? shoup_mul(other - v + q2, w.x, w.y, q) : csub(v + other, q2);
    };
    if (mu == 6) {
        uint32_t v0 = z[4 * lane + 3], v1 = z[4 * lane + 131];
        bfly(v0, 8, mrg[4 + lane / 16]);
        bfly(v1, 8, mrg[4 + (lane + 32) / 16]);
        bfly(v0, 16, mrg[2 + lane / 32]);
        bfly(v1, 16, mrg[2 + (lane + 32) / 32]);
        {
            const uint2 w = mrg[1];
            const uint32_t X = v0, Y = v1;
            v0 = csub(X + Y, q2);
            v1 = shoup_mul(X - Y + q2, w.x, w.y, q);
        }
        ms(v0, lane);
        ms(v1, lane + 32);
        z[4 * lane + 3] = v0;
        z[4 * lane + 131] = v1;
    } else {  // mu == 7
        uint32_t v = z[8 * lane + 7];
        bfly(v, 4, mrg[4 + lane / 8]);
        bfly(v, 8, mrg[2 + lane / 16]);
        bfly(v, 16, mrg[1]);
        ms(v, lane);
        z[8 * lane + 7] = v;
    }
    __syncwarp();
}

// Pass-0 stage S for both components of v6: the twiddles are loaded once;
// c1 gets full GS butterflies, c0 only the Y output of each block's last one.
template <int S>
__device__ __forceinline__ void pass0_stage_both(uint32_t (&a0)[16], uint32_t (&a1)[1][16], const uint2 *tw0, int g,
                                                 uint32_t q, uint32_t q2) {
    using Gm = NttGeom<4096>;
    constexpr int T = Gm::T, R = 16;
    constexpr int t = 1 << S, NB = R >> (S + 1), OFF = R - (R >> S);
    const uint4 *t4 = reinterpret_cast<const uint4 *>(tw0) + g;
    uint2 w[NB];
    if constexpr (NB >= 2) {
#pragma unroll
        for (int b = 0; b < NB / 2; b++) {
            const uint4 x = t4[(OFF / 2 + b) * T];
            w[2 * b] = make_uint2(x.x, x.y);
            w[2 * b + 1] = make_uint2(x.z, x.w);
        }
    } else {
        w[0] = reinterpret_cast<const uint2 *>(t4 + (OFF / 2) * T)[OFF % 2];
    }
#pragma unroll
    for (int b = 0; b < NB; b++) {
#pragma unroll
        for (int kk = 0; kk < t; kk++) gs_bfly(a1[0][b * 2 * t + kk], a1[0][b * 2 * t + kk + t], w[b].x, w[b].y, q, q2);
        const uint32_t X = a0[b * 2 * t + t - 1], Y = a0[b * 2 * t + 2 * t - 1];
        a0[b * 2 * t + 2 * t - 1] = shoup_mul(X - Y + q2, w[b].x, w[b].y, q);
    }
}

template <int L, int J>
struct LimbLoopPR {
    static constexpr int N = 4096;
    static __device__ __forceinline__ void run(EvalState<N, L, 1> &st, uint32_t (&a0)[16], uint4 (&cpre)[2][4],
                                               const BatchArgs &ba, const uint32_t *chat_q,
                                               const uint32_t *chat_next, uint32_t tcol, int g, const ChainCtx &cx,
                                               uint32_t *ybuf, uint32_t &par, uint32_t *cst, int mu,
                                               const uint2 *s_mrg) {
        using Gm = NttGeom<N>;
        constexpr int V = Gm::V;
        const uint32_t q = ba.kp.q[J], q2 = ba.kp.q2[J];
#pragma unroll
        for (int h = 0; h < 2; h++) {           // two halves of 8 values: fewer live registers
            uint32_t p[8], pp[8];
            tmem_ld<8>(tcol + 32 * J + 8 * h, p);
            tmem_ld<8>(tcol + 32 * J + 16 + 8 * h, pp);
            tmem_wait_ld<8>(p);
            tmem_wait_ld<8>(pp);
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const int v = 2 * h + u;
                a0[4 * v + 0] = shoup_mul(cpre[0][v].x, p[4 * u + 0], pp[4 * u + 0], q);
                a0[4 * v + 1] = shoup_mul(cpre[0][v].y, p[4 * u + 1], pp[4 * u + 1], q);
                a0[4 * v + 2] = shoup_mul(cpre[0][v].z, p[4 * u + 2], pp[4 * u + 2], q);
                a0[4 * v + 3] = shoup_mul(cpre[0][v].w, p[4 * u + 3], pp[4 * u + 3], q);
                st.a[0][4 * v + 0] = shoup_mul(cpre[1][v].x, p[4 * u + 0], pp[4 * u + 0], q);
                st.a[0][4 * v + 1] = shoup_mul(cpre[1][v].y, p[4 * u + 1], pp[4 * u + 1], q);
                st.a[0][4 * v + 2] = shoup_mul(cpre[1][v].z, p[4 * u + 2], pp[4 * u + 2], q);
                st.a[0][4 * v + 3] = shoup_mul(cpre[1][v].w, p[4 * u + 3], pp[4 * u + 3], q);
            }
        }
        // nullable-pointer guard: 1.1-1.7% faster here than LimbLoopTM's integer guard (c3 73.2 vs
        // 74.1 ms); this kernel's SASS keeps the zeroed pair's first reader >= 20 cycles after the
        // CS2R, which scripts/sass_hazard_scan.py checks on every build
        const uint32_t *nsrc = (J > 0) ? chat_q + (size_t)(J - 1) * N : (chat_next ? chat_next + (size_t)(L - 1) * N
                                                                                   : nullptr);
        if (nsrc) {
#pragma unroll
            for (int c = 0; c < 2; c++)
#pragma unroll
                for (int v = 0; v < V / 4; v++)
                    cpre[c][v] = ldg_op<WALLY_OPLD_PR>(nsrc + (size_t)c * L * N + (size_t)g * V + 4 * v);
        }
        // c0: pass 0 keeping the last Y output of each block -> one value per thread
        const uint2 *twJ = cx.tw + (size_t)J * Gm::TW_LIMB;
        // pass 0 of both components (twiddles loaded once; c0 keeps only the Y
        // output of each block's last butterfly), c1's first (intra-warp)
        // exchange, then c1's pass 1 stage by stage with c0's shuffle stages
        // interleaved (the shuffle chain is latency bound, c1's butterflies fill
        // the gaps), c1's second exchange and pass 2.  The exchange buffer
        // alternates with the limb parity (no write-after-read barrier).
        pass0_stage_both<0>(a0, st.a, twJ, g, q, q2);
        pass0_stage_both<1>(a0, st.a, twJ, g, q, q2);
        pass0_stage_both<2>(a0, st.a, twJ, g, q, q2);
        pass0_stage_both<3>(a0, st.a, twJ, g, q, q2);
        uint32_t *buf = cx.bufA + par * Gm::SMEM_WORDS;
        static_assert(Gm::A_IN_WARP, "v6 assumes the first exchange stays inside a warp");
        smem_store<N, Gm::TB0, Gm::R0, 1, 0>(buf, st.a, g);
        __syncwarp();
        smem_load<N, Gm::TB1, Gm::R1, 1, 0>(buf, st.a, g);
        const uint2 *mrgJ = s_mrg + J * 256;
        const uint2 *tw1 = twJ + Gm::TW1;
        uint32_t y = a0[15];
        ntt_stage<N, Gm::TB1, Gm::R1, 0, true, 1, true>(st.a, tw1, g, q, q2);
        y = c0_mid_stage<N, 4>(y, g, mu, mrgJ, q, q2);
        ntt_stage<N, Gm::TB1, Gm::R1, 1, true, 1, true>(st.a, tw1, g, q, q2);
        y = c0_mid_stage<N, 5>(y, g, mu, mrgJ, q, q2);
        ntt_stage<N, Gm::TB1, Gm::R1, 2, true, 1, true>(st.a, tw1, g, q, q2);
        y = c0_mid_stage<N, 6>(y, g, mu, mrgJ, q, q2);
        ntt_stage<N, Gm::TB1, Gm::R1, 3, true, 1, true>(st.a, tw1, g, q, q2);
        y = c0_mid_stage<N, 7>(y, g, mu, mrgJ, q, q2);
        y = c0_mid_stage<N, 8>(y, g, mu, mrgJ, q, q2);
        uint32_t *z = ybuf + par * Gm::T;
        z[g] = y;
        __syncwarp();
        smem_store<N, Gm::TB1, Gm::R1, 1, 1>(buf, st.a, g);
        group_sync(cx.bar, Gm::T);             // also publishes z to warp 0
        smem_load<N, Gm::TB2, Gm::R2, 1, 1>(buf, st.a, g);
        ntt_pass<N, Gm::TB2, Gm::R2, true, 1, true>(st.a, twJ + Gm::TW2, g, q, q2);
        if (g < 32) {
            if (mu == 6 || mu == 7) c0_tail_fast<L, J>(z, cst, s_mrg + J * 256, g, mu, ba.kp);
            else c0_tail<N, L, J>(z, cst, s_mrg + J * 256, g, mu, ba.kp);
        }
        par ^= 1u;
        // modulus-switch state through TMEM between limbs, at L = 2 (one 16-word rtop) as well:
        // c5 61.9 -> 61.7 ms, compact responses 61.6 -> 60.9 (WALLY_PR_L2_TMEM = 0: registers, for A/B)
#ifndef WALLY_PR_L2_TMEM
#define WALLY_PR_L2_TMEM 1
#endif
        if constexpr (L == 3 || (L == 2 && WALLY_PR_L2_TMEM)) {
            if constexpr (J < L - 1) {
                tmem_wait_st_all();
                if constexpr (J == L - 2) {
                    tmem_ld<16>(tcol + 96, st.rtop[0]);
                    tmem_wait_ld<16>(st.rtop[0]);
                } else {
                    tmem_ld<16>(tcol + 96, st.acc[0][0]);
                    tmem_wait_ld<16>(st.acc[0][0]);
                }
            }
            ms_step<L, J, V>(st.a[0], st.rtop[0], st.acc[0], ba.kp);
            if constexpr (J == L - 1) tmem_st<16>(tcol + 96, st.rtop[0]);
            else if constexpr (J > 0) tmem_st<16>(tcol + 96, st.acc[0][0]);
        } else {
            ms_step<L, J, V>(st.a[0], st.rtop[0], st.acc[0], ba.kp);
        }
        if constexpr (J > 0)
            LimbLoopPR<L, J - 1>::run(st, a0, cpre, ba, chat_q, chat_next, tcol, g, cx, ybuf, par, cst, mu, s_mrg);
    }
};

template <int L, int FMT>
__device__ __forceinline__ void eval_item_pr(const BatchArgs &ba, const ItemCursor &cur, uint32_t item, int g,
                                             const ChainCtx &cx, const uint32_t *s_rmap, uint32_t tcol,
                                             uint32_t *ybuf, uint32_t &par, uint32_t *cst, int mu,
                                             const uint2 *s_mrg) {
    constexpr int N = 4096;
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    static_assert(!NttStore<N>::CHUNK_MAJOR, "thread-major NTT-domain storage (ntt_word)");
    const uint32_t li = cur.li;
    const uint32_t cnt = ba.counts[li];
    const uint32_t local = item - cur.b;
    const uint32_t P = ba.n_pt[li];
    const uint32_t ch = local / P, k = local % P;
    const uint32_t qb = ba.seg[li] + ch * ba.chunk;
    const uint32_t qe = min(qb + ba.chunk, ba.seg[li] + cnt);
    const uint32_t *phat = ba.store + (size_t)(ba.pt_base[li] + k) * L * 2 * N;
#pragma unroll
    for (int J = 0; J < L; J++) {
        uint32_t p[16], pp[16];
        const uint32_t *pv = phat + (size_t)J * 2 * N + (size_t)g * V;
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const uint4 x = ldg_op<WALLY_OPLD_PR>(pv + 4 * v), y = ldg_op<WALLY_OPLD_PR>(pv + N + 4 * v);
            p[4 * v] = x.x; p[4 * v + 1] = x.y; p[4 * v + 2] = x.z; p[4 * v + 3] = x.w;
            pp[4 * v] = y.x; pp[4 * v + 1] = y.y; pp[4 * v + 2] = y.z; pp[4 * v + 3] = y.w;
        }
        tmem_st<16>(tcol + 32 * J, p);
        tmem_st<16>(tcol + 32 * J + 16, pp);
    }
    tmem_wait_st_all();
    uint32_t qo = ba.perm[qb];
    uint4 cpre[2][V / 4];
    {
        const uint32_t *src = ba.chat + (size_t)qo * 2 * L * N + (size_t)(L - 1) * N;
#pragma unroll
        for (int c = 0; c < 2; c++)
#pragma unroll
            for (int v = 0; v < V / 4; v++) cpre[c][v] = ldg_op<WALLY_OPLD_PR>(src + (size_t)c * L * N + (size_t)g * V + 4 * v);
    }
    for (uint32_t qi = qb; qi < qe; qi++) {
        const uint32_t qn = (qi + 1 < qe) ? ba.perm[qi + 1] : 0xffffffffu;
        uint32_t *out_q = ba.resp + ba.resp_off[qo] + (size_t)k * ba.wpp;
        const uint32_t *chat_q = ba.chat + (size_t)qo * 2 * L * N;
        const uint32_t *chat_next = (qn != 0xffffffffu) ? ba.chat + (size_t)qn * 2 * L * N : nullptr;
        EvalState<N, L, 1> st;
        uint32_t a0[16];
        LimbLoopPR<L, L - 1>::run(st, a0, cpre, ba, chat_q, chat_next, tcol, g, cx, ybuf, par, cst, mu, s_mrg);
        if (g < 32) c0_write_results<N>(ba, out_q, ybuf + (par ^ 1u) * Gm::T, g, mu);  // buffer of limb 0
        write_component<N, FMT>(ba, out_q, st.a[0], 1, g, s_rmap);
        qo = qn;
    }
}


template <int L, int FMT>
__global__ void __launch_bounds__(kEvalGroups * NttGeom<4096>::T, 1) eval_kernel_pr(BatchArgs ba) {
    constexpr int N = 4096;
    using Gm = NttGeom<N>;
    constexpr int T = Gm::T;
    constexpr int NA = (L > 2) ? (L - 2) : 1;
    extern __shared__ uint4 smem4[];
    uint2 *tw = reinterpret_cast<uint2 *>(smem4);
    uint32_t *xbuf = reinterpret_cast<uint32_t *>(tw + L * Gm::TW_LIMB);
    __shared__ uint32_t s_item[kEvalGroups][2];
    __shared__ uint32_t s_rmap[ResultMap<N>::WORDS];
    __shared__ __align__(16) uint32_t s_ybuf[kEvalGroups][2 * T];
    __shared__ uint32_t s_cst[kEvalGroups][(N / 16) * (1 + NA)];
    __shared__ uint2 s_mrg[L * 256];   // merged inverse table entries 0..255 of every limb (c0 tail)
    __shared__ uint32_t s_taddr;
    const int grp = threadIdx.x / T, g = threadIdx.x % T;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_taddr);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(ba.tw_inv);
        for (int i = threadIdx.x; i < L * Gm::TW_LIMB / 2; i += blockDim.x) smem4[i] = __ldg(src + i);
    }
    build_result_map<N>(s_rmap, ba.d);
    for (int i = threadIdx.x; i < L * 256; i += blockDim.x) s_mrg[i] = __ldg(ba.tw_mrg + (size_t)(i >> 8) * N + (i & 255));
    // work items are claimed in blocks of `ib` consecutive items (the same query
    // chunk against consecutive plaintexts of its cluster), so the cursor's
    // fast path finds the cluster without a search and the chunk's query NTTs
    // stay hot between items; small batches keep blocks of one (load balance):
    // 4 once there are >= 64 items per thread group (c3 -1%, c5 -3%), else 1
    // (c2, 28 items per group: +5% with 4, +3% with 2)
    const uint32_t groups_total = gridDim.x * kEvalGroups;
    const uint32_t ib = ba.misc[kMiscTotalItems] >= 64u * groups_total ? 4u : 1u;
    if (g == 0) s_item[grp][0] = atomicAdd(&ba.misc[kMiscWorkCounter], ib);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tcol = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
    const ChainCtx cx{tw, xbuf + grp * 2 * Gm::SMEM_WORDS, nullptr, 1 + grp};
    const int mu = min(__ffs((int)ba.d) - 1, 12);
    const uint32_t total = ba.misc[kMiscTotalItems];
    uint32_t par = 0;
    ItemCursor cur;
    for (uint32_t it = 0;; it++) {
        const uint32_t item0 = s_item[grp][it & 1];
        if (item0 >= total) break;
        if (g == 0) s_item[grp][(it + 1) & 1] = atomicAdd(&ba.misc[kMiscWorkCounter], ib);
        const uint32_t item_end = min(item0 + ib, total);
        for (uint32_t item = item0; item < item_end; item++) {
            cur.seek(ba, item);
            eval_item_pr<L, FMT>(ba, cur, item, g, cx, s_rmap, tcol, s_ybuf[grp], par, s_cst[grp], mu, s_mrg);
            group_sync(1 + grp, T);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_taddr) : "memory");
}

template <int L, int FMT>
static cudaError_t launch_eval_pr(const BatchArgs &a, cudaStream_t s, int num_sms) {
    using Gm = NttGeom<4096>;
    static DeviceOnce once;
    const size_t smem =
        (size_t)L * Gm::TW_LIMB * sizeof(uint2) + (size_t)kEvalGroups * 2 * Gm::SMEM_WORDS * sizeof(uint32_t);
    cudaError_t e = device_once(once, [&](int *) { return allow_smem(eval_kernel_pr<L, FMT>, smem); });
    if (e != cudaSuccess) return e;
    eval_kernel_pr<L, FMT><<<num_sms, kEvalGroups * Gm::T, smem, s>>>(a);
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// n = 8192 with compact responses and 32 | d (c4): c0's transform pruned as
// in v6 (pass 0 on V = 32 values per thread, five shuffle stages, the rest
// on warp 0 of the group).
// ---------------------------------------------------------------------------
// Register tail for n = 8192 and mu = 9 (c4: d = 512): after stage 9 the
// survivors are positions 512 k + 511, c = 16 k + 15 (k < 16); lanes 0..15
// hold one each, and stages 10..12 pair k with k ^ 2, k ^ 4, k ^ 8.
template <int L, int J>
__device__ __forceinline__ void c0_tail_fast8(uint32_t *z, uint32_t *cst, const uint2 *mrg, int lane,
                                              const KParams &kp) {
    constexpr int NA = (L > 2) ? (L - 2) : 1;
    const uint32_t q = kp.q[J], q2 = kp.q2[J];
    const int k = lane & 15;
    uint32_t v = z[16 * k + 15];
    auto bfly = [&](int xo, const uint2 w) {
        const uint32_t other = __shfl_xor_sync(0xffffffffu, v, xo);
        v = (k & xo) ? shoup_mul(other - v + q2, w.x, w.y, q) : csub(v + other, q2);
    };
    bfly(2, mrg[4 + k / 4]);     // stage 10: survivors 512 k + 511 pair with k ^ 2, block p / 2048
    bfly(4, mrg[2 + k / 8]);     // stage 11: k ^ 4, block p / 4096
    bfly(8, mrg[1]);             // stage 12: k ^ 8, one block
    if (lane < 16) {
        uint32_t rtop = cst[k * (1 + NA)], acc[NA];
#pragma unroll
        for (int l = 0; l < NA; l++) acc[l] = cst[k * (1 + NA) + 1 + l];
        ms_elem<L, J, NA>(v, rtop, acc, kp);
        cst[k * (1 + NA)] = rtop;
#pragma unroll
        for (int l = 0; l < NA; l++) cst[k * (1 + NA) + 1 + l] = acc[l];
        z[16 * k + 15] = v;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// n = 8192, compact responses, 32 | d (c4), v5: operands staged by bulk
// asynchronous copies (cp.async.bulk + mbarrier, "TMA or cp.async staging of
// the NTT-domain plaintexts", north_star) instead of register prefetch.
//
// One CTA of two 256-thread groups per SM.  A work item is (cluster, two
// consecutive plaintexts k0, k0 + 1, a chunk of queries); the groups take one
// plaintext each and walk the same queries in step, so each staged query
// chunk and twiddle block serves both (P_c is even at c4: no idle group).
// The operands of one (query, limb) stream through a ring of NSLOT shared-
// memory slots, one per 4-value chunk c of every thread (chunk-major
// NTT-domain storage, ntt_word: chunk c of all threads is one 4 KB block):
//   [y 2^32 of k0][y 2^32 of k1][pass-0 stage-0 twiddle block c]
//   [pass-0 twiddle block B(c)][c0 chunk][c1 chunk]          (24 KB per slot)
// (the plaintext's Montgomery plane only, PtStore: the pointwise products are
// Montgomery products, so no Shoup companion is staged)
// B(c) = 8, 12, 9, 14, 10, 13, 11, 15 delivers each later-stage twiddle block
// with the first chunk that needs it (a thread keeps the half it needs again
// in a register).  A producer thread (thread 0) keeps the ring NSLOT - 1
// chunks ahead across limbs and queries; a full barrier per slot carries the
// transaction bytes, an empty barrier per slot collects one arrival per warp.
// c1's pass 0 runs inside the chunk loop as a tree over the chunks sharing
// the twiddle reads of c0's Y-only tree; passes 1 and 2 through the group's
// exchange buffer (their tables resident in shared memory); c0's shuffle
// stages and warp-0 tail as in v3; c1's switch state in tensor memory.  No
// register holds a prefetched operand.
// ---------------------------------------------------------------------------
namespace p8t {
constexpr int N = 8192;
constexpr int T = NttGeom<N>::T;                 // 256 threads per group
#ifndef WALLY_P8T_CPS
#define WALLY_P8T_CPS 2
#endif
#ifndef WALLY_P8T_NSLOT
#define WALLY_P8T_NSLOT (WALLY_P8T_CPS == 1 ? 4 : 2)
#endif
constexpr int CPS = WALLY_P8T_CPS;               // chunks per ring slot
constexpr int NSLOT = WALLY_P8T_NSLOT;
constexpr int CHUNK_BYTES = T * 16;              // one 16-byte chunk of every thread: 4 KB
constexpr int SLOT_BYTES = 6 * CPS * CHUNK_BYTES;   // per chunk: 2 Montgomery plaintext chunks, 2 twiddle blocks, c0, c1
constexpr int TW12 = NttGeom<N>::TW_LIMB - NttGeom<N>::TW1;   // pass-1/2 table entries per limb
constexpr int XB_WORDS = NttGeom<N>::SMEM_WORDS;
__host__ __device__ constexpr size_t smem_bytes(int L) {
    return (size_t)NSLOT * SLOT_BYTES + (size_t)L * TW12 * 8 + 2ull * XB_WORDS * 4;
}
// pass-0 twiddle block (uint4 index / T) delivered with chunk c besides block c
__host__ __device__ constexpr int aux_block(int c) {
    return c == 0 ? 8 : c == 1 ? 12 : c == 2 ? 9 : c == 3 ? 14 : c == 4 ? 10 : c == 5 ? 13 : c == 6 ? 11 : 15;
}
}  // namespace p8t

void p8t_slot_twiddles(const uint2 *twi, uint32_t L, size_t tw_limb, uint2 *out) {
    using namespace p8t;
    static_assert(kP8tSlotTwEntries == (size_t)8 * 2 * T * 2, "slot twiddle table size");
    for (uint32_t J = 0; J < L; J++)
        for (int c = 0; c < 8; c++)
            for (int h = 0; h < 2; h++) {
                const int blk = h ? aux_block(c) : c;   // uint4 block of T entries = 2 T uint2 entries
                const uint2 *src = twi + (size_t)J * tw_limb + (size_t)blk * 2 * T;
                std::copy(src, src + 2 * T, out + (size_t)J * kP8tSlotTwEntries + ((size_t)c * 2 + h) * 2 * T);
            }
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

// c1's passes 1 and 2 for one group (pass 0 done), tables in shared memory,
// one exchange buffer, named barrier `bar` (four barriers).
__device__ __forceinline__ void p8t_intt_tail(uint32_t (&a)[1][32], const uint2 *tw12, int g, uint32_t q, uint32_t q2,
                                              uint32_t *buf, int bar) {
    constexpr int N = 8192;
    using Gm = NttGeom<N>;
    group_sync(bar, Gm::T);
    smem_store<N, Gm::TB0, Gm::R0, 1, 0>(buf, a, g);
    group_sync(bar, Gm::T);
    smem_load<N, Gm::TB1, Gm::R1, 1, 0>(buf, a, g);
    ntt_pass<N, Gm::TB1, Gm::R1, true, 1, true>(a, tw12, g, q, q2);
    group_sync(bar, Gm::T);
    smem_store<N, Gm::TB1, Gm::R1, 1, 1>(buf, a, g);
    group_sync(bar, Gm::T);
    smem_load<N, Gm::TB2, Gm::R2, 1, 1>(buf, a, g);
    ntt_pass<N, Gm::TB2, Gm::R2, true, 1, true>(a, tw12 + (Gm::TW2 - Gm::TW1), g, q, q2);
}

// Modulus-switch step of limb J for c1's 32 values per thread (n = 8192),
// the drop-last state in tensor memory (rtop in columns 0..31, acc[l] in
// 32 l .. 32 l + 31), eight values at a time.
template <int L, int J>
__device__ __forceinline__ void p8_ms_limb(uint32_t (&a)[1][32], uint32_t tcol, const KParams &kp) {
    constexpr int NA = (L > 2) ? (L - 2) : 1;
    if constexpr (L > 1 && J < L - 1) tmem_wait_st_all();
#pragma unroll
    for (int c8 = 0; c8 < 4; c8++) {
        uint32_t rt[8], ac[NA][8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            rt[k] = 0;
#pragma unroll
            for (int l = 0; l < NA; l++) ac[l][k] = 0;
        }
        if constexpr (L > 1 && J == L - 2) {
            tmem_ld<8>(tcol + 8 * c8, rt);
            tmem_wait_ld<8>(rt);
        }
        if constexpr (L > 2 && J < L - 2) {
#pragma unroll
            for (int l = 0; l <= J; l++) {
                tmem_ld<8>(tcol + 32 * l + 8 * c8, ac[l]);
                tmem_wait_ld<8>(ac[l]);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint32_t acc[NA];
#pragma unroll
            for (int l = 0; l < NA; l++) acc[l] = ac[l][k];
            ms_elem<L, J, NA>(a[0][8 * c8 + k], rt[k], acc, kp);
#pragma unroll
            for (int l = 0; l < NA; l++) ac[l][k] = acc[l];
        }
        if constexpr (L > 1 && J == L - 1) tmem_st<8>(tcol + 8 * c8, rt);
        if constexpr (L > 2 && J > 0 && J <= L - 2) {
#pragma unroll
            for (int l = 0; l < J; l++) tmem_st<8>(tcol + 32 * l + 8 * c8, ac[l]);
        }
    }
}

// Run-time limb index -> the compile-time instantiations (limbs J < L).
template <int L, typename F>
__device__ __forceinline__ void limb_dispatch(int J, F &&f) {
    switch (J) {
        case 0: f(std::integral_constant<int, 0>{}); break;
        case 1: if constexpr (L > 1) f(std::integral_constant<int, (L > 1 ? 1 : 0)>{}); break;
        case 2: if constexpr (L > 2) f(std::integral_constant<int, (L > 2 ? 2 : 0)>{}); break;
        default: if constexpr (L > 3) f(std::integral_constant<int, (L > 3 ? 3 : 0)>{}); break;
    }
}

template <int L, int FMT>
__global__ void __launch_bounds__(2 * NttGeom<8192>::T, 1) eval_kernel_p8t(BatchArgs ba) {
    using namespace p8t;
    using Gm = NttGeom<N>;
    constexpr int V = Gm::V;
    constexpr int NA = (L > 2) ? (L - 2) : 1;
    constexpr int CHUNKS = V / 4;                 // 8 chunks of 4 values per thread and limb
    constexpr int EPL = CHUNKS / CPS;             // ring elements per limb
    extern __shared__ __align__(128) uint8_t smem8[];
    uint8_t *slots = smem8;
    uint2 *s_tw12 = reinterpret_cast<uint2 *>(smem8 + NSLOT * SLOT_BYTES);
    uint32_t *xbuf = reinterpret_cast<uint32_t *>(smem8 + NSLOT * SLOT_BYTES + (size_t)L * TW12 * 8);
    __shared__ BatchArgs s_ba;
    __shared__ uint32_t s_taddr;
    __shared__ uint32_t s_item[2];
    __shared__ uint32_t s_rmap[ResultMap<N>::WORDS];
    __shared__ uint32_t s_ybuf[2][2 * T];
    __shared__ uint32_t s_cst[2][(N / 32) * (1 + NA)];
    __shared__ uint2 s_mrg[L * 256];
    __shared__ __align__(8) uint64_t s_bar[2 * NSLOT];   // full[NSLOT], empty[NSLOT]
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int grp = threadIdx.x / T, g = threadIdx.x % T;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(s_bar);
    auto full_b = [&](uint32_t i) { return bar0 + 8u * i; };
    auto empty_b = [&](uint32_t i) { return bar0 + 8u * (NSLOT + i); };
    if (threadIdx.x == 0) {
        s_ba = ba;
        for (int i = 0; i < NSLOT; i++) {
            mbar_init(full_b(i), 1);
            mbar_init(empty_b(i), 2 * T / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {   // 512 columns: four warps share a lane quadrant, 128 columns each
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_taddr);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = threadIdx.x; i < L * 256; i += blockDim.x) s_mrg[i] = __ldg(ba.tw_mrg + (size_t)(i >> 8) * N + (i & 255));
    for (int i = threadIdx.x; i < L * TW12; i += blockDim.x)
        s_tw12[i] = __ldg(ba.tw_inv + (size_t)(i / TW12) * Gm::TW_LIMB + Gm::TW1 + (i % TW12));
    build_result_map<N>(s_rmap, ba.d);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tcol = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
    uint32_t *xb = xbuf + grp * XB_WORDS;
    const int bar = 1 + grp;
    const int mu = min(__ffs((int)ba.d) - 1, 13);
    const uint32_t total = ba.misc[kMiscTotalItems];
    const uint32_t slots_s = (uint32_t)__cvta_generic_to_shared(slots);
#ifndef WALLY_P8T_TAIL_WARP
#define WALLY_P8T_TAIL_WARP 1
#endif
    constexpr int TAIL_WARP = WALLY_P8T_TAIL_WARP;
    uint32_t seq = 0;      // chunk slots consumed by this CTA so far (ring position and phases)
    uint32_t par = 0;
    ItemCursor cur, ncur;
    // A work item's operand stream: (query, limb L-1..0, chunk); its description, computed by
    // every thread for the current item and by the producer (thread 0) for the next one.
    struct Desc {
        const uint32_t *phat0;
        uint32_t qb, qe, np, k0, nchunks;
    };
    auto describe = [&](ItemCursor &cu, uint32_t item) -> Desc {
        Desc d{};
        if (item >= total) return d;                            // nchunks = 0: no item
        cu.seek(s_ba, item);
        const uint32_t li = cu.li;
        const uint32_t P = s_ba.n_pt[li], PP = (P + 1) / 2;
        const uint32_t ch = (item - cu.b) / PP;
        d.k0 = 2 * ((item - cu.b) % PP);
        d.np = min(2u, P - d.k0);                               // plaintexts of the item (1 only for odd P_c)
        d.qb = s_ba.seg[li] + ch * s_ba.chunk;
        d.qe = min(d.qb + s_ba.chunk, s_ba.seg[li] + s_ba.counts[li]);
        d.phat0 = s_ba.store + pt_mont_word<N>((size_t)s_ba.pt_base[li] + d.k0, L, 0, 0, 0);   // an even index
        d.nchunks = (d.qe - d.qb) * L * EPL;   // ring elements (CPS chunks each)
        return d;
    };
    // producer (thread 0): element j of item description d into ring position sq: wait for the slot
    // to drain (one arrival per warp on its empty barrier), post the byte count on its full barrier,
    // issue the eight 4 KB copies
    auto produce = [&](const Desc &d, uint32_t j, uint32_t sq) {
        const uint32_t sl = sq % NSLOT;
        if (sq >= NSLOT) mbar_wait(empty_b(sl), ((sq / NSLOT) + 1) & 1u);
        mbar_expect_tx(full_b(sl), 6 * CPS * CHUNK_BYTES);
        const uint32_t r = j / (L * EPL), J = L - 1 - (j / EPL) % L, c = (j % EPL) * CPS;
        const uint32_t dst = slots_s + sl * SLOT_BYTES;
        // chunk c of both plaintexts of the pair (the second is the pad plaintext when P_c is odd)
        static_assert(PtStore<N>::MONT, "v6 stages the pair-interleaved Montgomery store");
        bulk_g2s(dst, d.phat0 + pt_mont_word<N>(0, L, J, 0, c), 2 * CPS * CHUNK_BYTES, full_b(sl));
        bulk_g2s(dst + 2 * CPS * CHUNK_BYTES, s_ba.tw_slot + (size_t)J * kP8tSlotTwEntries + (size_t)c * 4 * T,
                 2 * CPS * CHUNK_BYTES, full_b(sl));
        const uint32_t *cq = s_ba.chat + (size_t)s_ba.perm[d.qb + r] * 2 * L * N;
        bulk_g2s(dst + 4 * CPS * CHUNK_BYTES, cq + chat_word<N>(L, 0, J, 0, c), 2 * CPS * CHUNK_BYTES,
                 full_b(sl));   // c0, c1
    };
    uint32_t pre_issued = 0;   // thread 0: elements of the current item issued while the previous one ran
    // items are claimed in blocks of `ib` consecutive ones (thread 0 keeps the current block's end and
    // the next block, claimed one block ahead), so consecutive items usually share the cluster (no
    // cursor search); the next item is known while the current one runs
    const uint32_t ib = total >= 64u * gridDim.x ? 4u : 1u;
    uint32_t blk_end = 0, blk_next = 0;
    if (threadIdx.x == 0) {
        s_item[0] = atomicAdd(&ba.misc[kMiscWorkCounter], ib);
        blk_end = s_item[0] + ib;
        blk_next = atomicAdd(&ba.misc[kMiscWorkCounter], ib);
    }
    for (uint32_t it = 0;; it++) {
        __syncthreads();
        const uint32_t item = s_item[it & 1];
        if (item >= total) break;
        // the next item is fixed now, so the producer can stream its first chunks while this one ends
        if (threadIdx.x == 0) {
            uint32_t nx = item + 1;
            if (nx >= blk_end) {
                nx = blk_next;
                blk_end = nx + ib;
                blk_next = atomicAdd(&ba.misc[kMiscWorkCounter], ib);
            }
            s_item[(it + 1) & 1] = nx;
        }
        const Desc d = describe(cur, item);
        Desc dn{};
        if (threadIdx.x == 0) dn = describe(ncur, s_item[(it + 1) & 1]);
        const uint32_t qb = d.qb, qe = d.qe, np = d.np, nchunks = d.nchunks;
        const uint32_t k = d.k0 + grp;
        const bool active = (uint32_t)grp < np;
        const uint32_t seq0 = seq;
        // elements are issued NSLOT - 1 ahead of the chunk being consumed, across the item boundary
        // (issuing one more into the slot a limb's last chunk frees, so that the next limb's first NSLOT
        // chunks load during the transform, measured slower: 93.6 vs 88.3 ms -- the producer then waits
        // for every warp before its own transform)
        auto issue = [&](uint32_t j) {
            if (j < nchunks) produce(d, j, seq0 + j);
            else if (j - nchunks < dn.nchunks) produce(dn, j - nchunks, seq0 + j);
        };
        if (threadIdx.x == 0)
            for (uint32_t j = pre_issued; j + 1 < NSLOT; j++) issue(j);
        for (uint32_t r = 0; qb + r < qe; r++) {
            const uint32_t qo = s_ba.perm[qb + r];
            uint32_t a[1][V];
#pragma unroll 1
            for (int Jr = 0; Jr < L; Jr++) {
                const int J = L - 1 - Jr;
                const uint32_t q = s_ba.kp.q[J], q2 = s_ba.kp.q2[J];
                auto yo = [&](uint32_t X, uint32_t Y, uint2 w) { return shoup_mul(X - Y + q2, w.x, w.y, q); };
                auto bf = [&](int i, int j, uint2 w) { gs_bfly(a[0][i], a[0][j], w.x, w.y, q, q2); };
                uint32_t l2 = 0, l3 = 0, l4 = 0, y = 0;
                uint2 k1 = make_uint2(0, 0), k2 = make_uint2(0, 0), k3 = make_uint2(0, 0);  // twiddle halves kept
#pragma unroll
                for (int c = 0; c < CHUNKS; c++) {
                    const uint32_t j = (r * L + Jr) * EPL + c / CPS;   // stream element
                    const uint32_t sq = seq0 + j, sl = sq % NSLOT;
                    const int h = c % CPS;                             // chunk inside the element (unrolled: constant)
                    if (h == 0) {
                        if (threadIdx.x == 0) issue(j + NSLOT - 1);
                        mbar_wait(full_b(sl), (sq / NSLOT) & 1u);
                    }
                    const uint4 *sp = reinterpret_cast<const uint4 *>(slots + sl * SLOT_BYTES);
                    if (active) {
                        const uint32_t qi = s_ba.kp.mqinv[J];
                        const uint4 pm = sp[(2 * h + grp) * T + g];
                        const uint4 w0 = sp[(2 * CPS + 2 * h) * T + g], ta = sp[(2 * CPS + 2 * h + 1) * T + g];
                        const uint4 x0 = sp[(4 * CPS + 2 * h) * T + g], x1 = sp[(4 * CPS + 2 * h + 1) * T + g];
                        a[0][4 * c + 0] = mont_mul(x1.x, pm.x, q, qi);
                        a[0][4 * c + 1] = mont_mul(x1.y, pm.y, q, qi);
                        a[0][4 * c + 2] = mont_mul(x1.z, pm.z, q, qi);
                        a[0][4 * c + 3] = mont_mul(x1.w, pm.w, q, qi);
                        const uint32_t y0 = mont_mul(x0.x, pm.x, q, qi), y1 = mont_mul(x0.y, pm.y, q, qi);
                        const uint32_t y2 = mont_mul(x0.z, pm.z, q, qi), y3 = mont_mul(x0.w, pm.w, q, qi);
                        // pass-0 stages of this chunk: c1 in full, c0 the last Y output of each block
                        const uint2 wa = make_uint2(w0.x, w0.y), wb = make_uint2(w0.z, w0.w);
                        bf(4 * c, 4 * c + 1, wa);
                        bf(4 * c + 2, 4 * c + 3, wb);
                        const uint32_t u0 = yo(y0, y1, wa), u1 = yo(y2, y3, wb);
                        // stage 1, block c (twiddle slot 16 + c = block 8 + c/2, delivered with chunk c & ~1)
                        uint2 w1;
                        if (c % 2 == 0) {
                            w1 = make_uint2(ta.x, ta.y);
                            k1 = make_uint2(ta.z, ta.w);
                        } else {
                            w1 = k1;
                        }
                        bf(4 * c, 4 * c + 2, w1);
                        bf(4 * c + 1, 4 * c + 3, w1);
                        const uint32_t v = yo(u0, u1, w1);
                        if (c % 2 == 0) {
                            l2 = v;
                        } else {
                            // stage 2, block c / 2 (block 12 + c/4, delivered with chunks 1 and 5)
                            uint2 w2;
                            if ((c / 2) % 2 == 0) {
                                w2 = make_uint2(ta.x, ta.y);
                                k2 = make_uint2(ta.z, ta.w);
                            } else {
                                w2 = k2;
                            }
#pragma unroll
                            for (int kk = 0; kk < 4; kk++) bf(8 * (c / 2) + kk, 8 * (c / 2) + kk + 4, w2);
                            const uint32_t v2 = yo(l2, v, w2);
                            if ((c / 2) % 2 == 0) {
                                l3 = v2;
                            } else {
                                // stage 3, block c / 4 (block 14, delivered with chunk 3)
                                uint2 w3;
                                if (c / 4 == 0) {
                                    w3 = make_uint2(ta.x, ta.y);
                                    k3 = make_uint2(ta.z, ta.w);
                                } else {
                                    w3 = k3;
                                }
#pragma unroll
                                for (int kk = 0; kk < 8; kk++) bf(16 * (c / 4) + kk, 16 * (c / 4) + kk + 8, w3);
                                const uint32_t v3 = yo(l3, v2, w3);
                                if (c / 4 == 0) {
                                    l4 = v3;
                                } else {
                                    // stage 4 (block 15, delivered with chunk 7)
                                    const uint2 w4 = make_uint2(ta.x, ta.y);
#pragma unroll
                                    for (int kk = 0; kk < 16; kk++) bf(kk, kk + 16, w4);
                                    y = yo(l4, v3, w4);
                                }
                            }
                        }
                    }
                    if (h == CPS - 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(empty_b(sl));
                    }
                }
                if (!active) continue;
                uint32_t *z = s_ybuf[grp] + par * T;
                z[g] = c0_mid<N>(y, g, mu, s_mrg + J * 256, q, q2);
                p8t_intt_tail(a, s_tw12 + (size_t)J * TW12, g, q, q2, xb, bar);
                // c0's tail on the group's warp TAIL_WARP (not warp 0, whose thread 0 is the producer)
                if (g / 32 == TAIL_WARP) {
                    limb_dispatch<L>(J, [&](auto JC) {
                        constexpr int JJ = decltype(JC)::value;
                        if (mu == 9) c0_tail_fast8<L, JJ>(z, s_cst[grp], s_mrg + JJ * 256, lane, s_ba.kp);
                        else c0_tail<N, L, JJ>(z, s_cst[grp], s_mrg + JJ * 256, lane, mu, s_ba.kp);
                    });
                }
                par ^= 1u;
                limb_dispatch<L>(J, [&](auto JC) { p8_ms_limb<L, decltype(JC)::value>(a, tcol, s_ba.kp); });
            }
            if (active) {
                uint32_t *out_q = s_ba.resp + s_ba.resp_off[qo] + (size_t)k * s_ba.wpp;
                if (g / 32 == TAIL_WARP) c0_write_results<N>(s_ba, out_q, s_ybuf[grp] + (par ^ 1u) * T, lane, mu);
                write_component<N, FMT>(s_ba, out_q, a[0], 1, g, s_rmap);
            }
        }
        seq = seq0 + nchunks;
        pre_issued = (nchunks + NSLOT - 1 > nchunks) ? min(NSLOT - 1, dn.nchunks) : 0u;   // thread 0 only
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_taddr) : "memory");
}

template <int L, int FMT>
static cudaError_t launch_eval_p8t(const BatchArgs &a, cudaStream_t s, int num_sms) {
    static DeviceOnce once;
    const size_t smem = p8t::smem_bytes(L);
    cudaError_t e = device_once(once, [&](int *) { return allow_smem(eval_kernel_p8t<L, FMT>, smem); });
    if (e != cudaSuccess) return e;
    eval_kernel_p8t<L, FMT><<<num_sms, 2 * NttGeom<8192>::T, smem, s>>>(a);   // one CTA (two groups) per SM
    return cudaGetLastError();
}

template <int N, int L, int FMT>
static cudaError_t launch_eval_tm(const BatchArgs &a, cudaStream_t s, int num_sms) {
    using Gm = NttGeom<N>;
    static DeviceOnce once;
    const size_t smem = (size_t)L * Gm::TW_LIMB * sizeof(uint2) +
                        (size_t)kEvalGroups * 2 * Gm::SMEM_WORDS * sizeof(uint32_t);
    cudaError_t e = device_once(once, [&](int *) { return allow_smem(eval_kernel_tm<N, L, FMT>, smem); });
    if (e != cudaSuccess) return e;
    // one CTA per SM: it owns all 512 TMEM columns of its SM
    eval_kernel_tm<N, L, FMT><<<num_sms, kEvalGroups * Gm::T, smem, s>>>(a);
    return cudaGetLastError();
}

template <int N, int L>
static cudaError_t launch_eval_nl(const BatchArgs &a, cudaStream_t s, int num_sms) {
    using Gm = NttGeom<N>;
    static DeviceOnce once;
    int blocks_per_sm = 1;
#ifndef WALLY_EVAL_TMEM
#define WALLY_EVAL_TMEM 1
#endif
    if constexpr (N == 4096 && L >= 2 && L <= 3 && WALLY_EVAL_TMEM) {
        // compact responses with 16 | d: pruned c0 transform (v6)
        if (pruned_c0_path(N, L, a.d, a.compact)) {
            if (a.drop) return launch_eval_pr<L, (int)WALLY_RESP_COMPACT_DROP>(a, s, num_sms);
            return launch_eval_pr<L, (int)WALLY_RESP_COMPACT>(a, s, num_sms);
        }
    }
    if constexpr (N == 4096 && L >= 2 && L <= 3 && WALLY_EVAL_TMEM) {
        if (a.drop) return launch_eval_tm<N, L, (int)WALLY_RESP_COMPACT_DROP>(a, s, num_sms);
        if (a.compact) return launch_eval_tm<N, L, (int)WALLY_RESP_COMPACT>(a, s, num_sms);
        return launch_eval_tm<N, L, (int)WALLY_RESP_FULL>(a, s, num_sms);
    } else if constexpr (N <= 4096) {
        const size_t smem = (size_t)L * Gm::TW_LIMB * sizeof(uint2) +
                            (size_t)kEvalGroups * EvalCfg<N>::NC * Gm::SMEM_WORDS * sizeof(uint32_t);
        cudaError_t e = device_once(once, [&](int *v) {
            cudaError_t r = allow_smem(eval_kernel_grp<N, L>, smem);
            if (r == cudaSuccess)
                r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(v, eval_kernel_grp<N, L>, kEvalGroups * Gm::T, smem);
            return r;
        }, &blocks_per_sm);
        if (e != cudaSuccess) return e;
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        eval_kernel_grp<N, L><<<num_sms * blocks_per_sm, kEvalGroups * Gm::T, smem, s>>>(a);
    } else {
        if constexpr (N == 8192 && WALLY_EVAL_TMEM) {
            if (pruned_c0_path(N, L, a.d, a.compact)) return launch_eval_p8t<L, (int)WALLY_RESP_COMPACT>(a, s, num_sms);
        }
        const size_t smem = chain_smem<N>(EvalCfg<N>::NC);
        cudaError_t e = device_once(once, [&](int *v) {
            cudaError_t r = allow_smem(eval_kernel<N, L>, smem);
            if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(v, eval_kernel<N, L>, Gm::T, smem);
            return r;
        }, &blocks_per_sm);
        if (e != cudaSuccess) return e;
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        eval_kernel<N, L><<<num_sms * blocks_per_sm, Gm::T, smem, s>>>(a);
    }
    return cudaGetLastError();
}

template <int N>
static cudaError_t launch_eval_n(const BatchArgs &a, cudaStream_t s, int num_sms) {
    switch (a.L) {
        case 1: return launch_eval_nl<N, 1>(a, s, num_sms);
        case 2: return launch_eval_nl<N, 2>(a, s, num_sms);
        case 3: return launch_eval_nl<N, 3>(a, s, num_sms);
        case 4: return launch_eval_nl<N, 4>(a, s, num_sms);
    }
    return cudaErrorInvalidValue;
}

// Row gather for the multi-GPU query scatter: dst[i] = src[index[i]], rows of
// row_words uint32 (a multiple of 4), 16-byte copies; one CTA row-slice per
// (row, 4096-word chunk), grid-strided.
__global__ void __launch_bounds__(256) pack_rows_kernel(const uint32_t *__restrict__ index,
                                                        const uint4 *__restrict__ src, uint4 *__restrict__ dst,
                                                        uint32_t count, uint32_t row_vec) {
    const uint32_t chunks = (row_vec + 1023) / 1024;
    for (uint32_t b = blockIdx.x; b < count * chunks; b += gridDim.x) {
        const uint32_t i = b / chunks, c = b % chunks;
        const uint4 *s = src + (size_t)index[i] * row_vec;
        uint4 *d = dst + (size_t)i * row_vec;
        for (uint32_t v = c * 1024 + threadIdx.x; v < min(row_vec, (c + 1) * 1024); v += blockDim.x)
            __stcs(d + v, ldg_stream(s + v));
    }
}

cudaError_t launch_pack_rows(const uint32_t *index, const uint32_t *src, uint32_t *dst, uint32_t count,
                             uint32_t row_words, cudaStream_t s, uint64_t *launches) {
    const uint32_t row_vec = row_words / 4;
    const uint32_t chunks = (row_vec + 1023) / 1024;
    const uint64_t work = (uint64_t)count * chunks;
    const unsigned grid = (unsigned)std::min<uint64_t>(work, 148ull * 16);
    pack_rows_kernel<<<grid, 256, 0, s>>>(index, reinterpret_cast<const uint4 *>(src), reinterpret_cast<uint4 *>(dst),
                                          count, row_vec);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_batcher(const BatchArgs &a, cudaStream_t s, uint64_t *launches) {
    if (a.nq == 0) return cudaSuccess;
    if (a.nq <= 4096) {
        batch_small_kernel<<<1, 1024, 0, s>>>(a.ids, a.nq, a.local_of_cluster, a.total_clusters, a.counts, a.n_local,
                                              a.n_pt, a.chunk, a.ppi, a.seg, a.item_start, a.misc, a.fill, a.perm);
        *launches += 1;
        return cudaGetLastError();
    }
    const unsigned threads = 256;
    const unsigned blocks = (a.nq + threads - 1) / threads;
    batch_count_kernel<<<blocks, threads, 0, s>>>(a.ids, a.nq, a.local_of_cluster, a.total_clusters, a.counts);
    batch_scan_kernel<<<1, 1024, 0, s>>>(a.counts, a.n_local, a.n_pt, a.chunk, a.ppi, a.seg, a.item_start, a.misc);
    batch_scatter_kernel<<<blocks, threads, 0, s>>>(a.ids, a.nq, a.local_of_cluster, a.total_clusters, a.seg, a.fill,
                                                    a.perm);
    *launches += 3;
    return cudaGetLastError();
}

cudaError_t launch_query_ntt(const BatchArgs &a, cudaStream_t s, uint64_t *launches) {
    return launch_ntt_forward(a.kp, a.n, a.L, a.tw_fwd, a.query_ct, a.chat, 2 * a.nq, a.misc + kMiscErr, s, launches,
                              true);
}

cudaError_t launch_eval(const BatchArgs &a, cudaStream_t s, int num_sms, uint64_t *launches) {
    if (a.nq == 0) return cudaSuccess;
    *launches += 1;
    switch (a.n) {
        case 1024: return launch_eval_n<1024>(a, s, num_sms);
        case 2048: return launch_eval_n<2048>(a, s, num_sms);
        case 4096: return launch_eval_n<4096>(a, s, num_sms);
        case 8192: return launch_eval_n<8192>(a, s, num_sms);
    }
    return cudaErrorInvalidValue;
}

}  // namespace wally

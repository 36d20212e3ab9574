// Internal declarations shared by the host C-ABI (capi.cpp) and the kernels
// (kernels.cu).  Not part of the public ABI (include/wally.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "wally.h"

namespace wally {

constexpr int kMaxLimbs = WALLY_MAX_LIMBS;
// Queries per work item of the fused kernel (a query chunk of one cluster
// shares every staged plaintext).
#ifndef WALLY_QUERY_CHUNK
#define WALLY_QUERY_CHUNK 32
#endif
constexpr uint32_t kQueryChunk = WALLY_QUERY_CHUNK;
// Queries per work item of the n = 8192 kernel v5: its work items are short
// (a query chunk x two plaintexts) and consecutive items share the query
// chunk, so the SMs working at one time read each plaintext pair for
// different queries at nearly the same time (L2 hits instead of re-reads
// from DRAM); the operand stream runs on across items.
#ifndef WALLY_P8_CHUNK
#define WALLY_P8_CHUNK 1
#endif
constexpr uint32_t kP8QueryChunk = WALLY_P8_CHUNK;

// Per-limb constants, passed by value to every kernel (kernel parameter
// space -> constant bank, uniform across the grid).
struct KParams {
    uint32_t q[kMaxLimbs];        // moduli, ascending
    uint32_t q2[kMaxLimbs];       // 2 q
    uint32_t h[kMaxLimbs];        // floor(q/2): rounding offset of the drop-last step
    uint32_t ninv[kMaxLimbs];     // n^{-1} mod q       (debug inverse NTT)
    uint32_t ninvp[kMaxLimbs];    //   Shoup companion
    uint32_t fold[kMaxLimbs];     // F_l = n^{-1} prod_{k>l} q_k^{-1} mod q_l (folded into plaintexts)
    uint32_t foldp[kMaxLimbs];    //   Shoup companion
    uint32_t C[kMaxLimbs][kMaxLimbs];   // C[l][m] = prod_{k=l+1..m} q_k^{-1} mod q_l, l < m
    uint32_t Cp[kMaxLimbs][kMaxLimbs];  //   Shoup companions
    uint32_t Qi[kMaxLimbs][kMaxLimbs];   // Qi[l][m] = q_m^{-1} mod q_l, l < m (Horner steps of the switch)
    uint32_t Qip[kMaxLimbs][kMaxLimbs];  //   Shoup companions
    uint32_t mqinv[kMaxLimbs];    // -q^{-1} mod 2^32 (Montgomery products with the n = 8192 plaintexts)
};

// Plaintext store.  n <= 4096: [npt][L][2][n] uint32, per limb the folded
// NTT-domain value y = NTT(p) F_l (canonical, ntt_word order) followed by its
// Shoup companion floor(y 2^32 / q).  n = 8192 (MONT): one plane, y's
// Montgomery form y 2^32 mod q, multiplied with mont_mul (no companion), and
// plaintexts stored in pairs (2k, 2k + 1) interleaved by 16-byte chunk --
// [npt/2][L][chunk v][2][4T] -- so one bulk copy stages chunk v of both
// plaintexts of a v6 work item; every cluster starts at an even plaintext
// index (a pad plaintext, all zero, after an odd P_c).  DESIGN.md §5-6.
template <int N>
struct PtStore {
    static constexpr bool MONT = (N == 8192);
    static constexpr int PLANES = MONT ? 1 : 2;
    static constexpr uint32_t ALIGN = MONT ? 2 : 1;   // plaintext index alignment of a cluster
};
inline uint32_t pt_store_planes(uint32_t n) { return n == 8192 ? 1u : 2u; }
inline uint32_t pt_store_align(uint32_t n) { return n == 8192 ? 2u : 1u; }

// Workspace layout of one batch (device), offsets in bytes.
struct WsLayout {
    size_t ids, resp_off, perm, counts, fill, misc, seg, item_start, chat, total;
    size_t zero_begin, zero_bytes;  // region cleared at the start of every batch
};
WsLayout ws_layout(uint32_t nq, uint32_t n_local, uint32_t n, uint32_t L);

// misc[] words in the workspace
enum { kMiscTotalItems = 0, kMiscWorkCounter = 1, kMiscErr = 2, kMiscWords = 4 };
enum { kErrResidue = 1u };

struct BatchArgs {
    KParams kp;
    uint32_t n, L;
    uint32_t d, E;                // dimension, entries per plaintext
    uint32_t wpp;                 // response words per plaintext (2n or E4 + n)
    uint32_t compact;             // WALLY_RESP_COMPACT or _COMPACT_DROP (c0 at the result coefficients only)
    uint32_t drop;                // WALLY_RESP_COMPACT_DROP (c1 rounded to 2^6, 24-bit planes)
    uint32_t nq;
    uint32_t chunk;               // queries per work item (kQueryChunk, or 1 for small batches)
    uint32_t ppi;                 // plaintexts per work item (eval_plaintexts_per_item)
    uint32_t n_local;
    uint32_t total_clusters;
    const uint2 *tw_fwd;          // [L][n] (w, w') psi^{brev(i)}
    const uint2 *tw_inv;          // [L] pass-major inverse tables (ntt_device.cuh)
    const uint2 *tw_mrg;          // [L][n] (w, w') psi^{-brev(i)}, plain merged order
    const uint2 *tw_slot;         // n = 8192: pass-0 twiddle blocks per ring slot (p8t_slot_twiddles)
    const int32_t *local_of_cluster;  // [total_clusters]
    const uint32_t *pt_base;      // [n_local]
    const uint32_t *n_pt;         // [n_local]
    const uint32_t *store;        // plaintext store (layout: PtStore)
    const uint32_t *query_ct;     // [nq][2][L][n]
    uint32_t *resp;
    // workspace pieces
    uint32_t *ids;
    uint64_t *resp_off;
    uint32_t *perm;
    uint32_t *counts;
    uint32_t *fill;
    uint32_t *misc;
    uint32_t *seg;
    uint32_t *item_start;
    uint32_t *chat;               // [nq][2][L][n]
    uint64_t resp_words, store_words;   // buffer sizes (bounds checks of WALLY_BOUNDS_CHECK builds)
};

struct EncodeArgs {
    KParams kp;
    uint32_t n, L, d, E;
    uint32_t npt;
    const uint2 *tw_fwd;
    const int8_t *entries;        // [local entries][d]
    const uint32_t *pt_li;        // [npt] local cluster of each plaintext
    const uint32_t *pt_k;         // [npt] index of the plaintext in its cluster
    const uint64_t *entry_base;   // [n_local] first entry row of each local cluster
    const uint32_t *size;         // [n_local] entries of each local cluster
    uint32_t *store;              // plaintext store (layout: PtStore)
};

// Does a batch take the pruned-c0 fused kernel (kernels.cu "Fused kernel
// v6")?  Shared by the launcher and wally_modmuls_per_pair.
#ifndef WALLY_EVAL_PRUNE
#define WALLY_EVAL_PRUNE 1
#endif
inline bool pruned_c0_path(uint32_t n, uint32_t L, uint32_t d, bool compact) {
    if (!WALLY_EVAL_PRUNE || !compact) return false;
    if (n == 4096) return L >= 2 && L <= 3 && (d & 15u) == 0;   // v6 (two groups, TMEM)
    if (n == 8192) return (d & 31u) == 0;                      // whole-CTA kernel (c4)
    return false;
}

// Plaintexts per work item of the fused kernel a batch runs: 2 for the v5
// n = 8192 kernel (its two thread groups take plaintexts k and k + 1 of the
// item's cluster for the same queries), 1 otherwise.  Shared by the batcher
// (item count) and the kernel (item decode).
inline uint32_t eval_plaintexts_per_item(uint32_t n, uint32_t L, uint32_t d, bool compact) {
    return (n == 8192 && pruned_c0_path(n, L, d, compact)) ? 2u : 1u;
}

// Algorithmic modular multiplications per (query, plaintext) pair of the
// fused kernel: pointwise + inverse-NTT butterflies + modulus switch for both
// components (SURVEY.md §8(d) M_pair), with c0's transform pruned to the
// result coefficients when pruned_c0_path() holds.
inline uint64_t modmuls_per_pair(uint32_t n, uint32_t L, uint32_t d, bool pruned) {
    uint32_t logn = 0;
    while ((1u << logn) < n) logn++;
    const uint64_t ms = (uint64_t)L * (L - 1) / 2;
    const uint64_t full = (uint64_t)L * n + (uint64_t)L * (n / 2) * logn + (uint64_t)n * ms;
    if (!pruned) return 2 * full;
    uint32_t mu = 0;
    while (mu < logn && ((d >> mu) & 1u) == 0) mu++;
    const uint64_t M = 1ull << mu;
    uint64_t bf = 0;
    for (uint32_t s = 0; s < logn; s++) bf += (s < mu) ? (n >> (s + 1)) : n / (2 * M);
    const uint64_t c0 = (uint64_t)L * n + (uint64_t)L * bf + (n / M) * ms;
    return full + c0;
}

// One-time kernel configuration per device, safe under concurrent host
// threads: cudaFuncSetAttribute(MaxDynamicSharedMemorySize) and occupancy
// queries apply to the current device only, so a second context on another
// device must configure again.  `f(int *value)` runs once per device; its
// value (e.g. blocks per SM) is returned on every call.
struct DeviceOnce {
    std::mutex m;
    uint64_t done = 0;
    int value[64] = {};
};
template <typename F>
inline cudaError_t device_once(DeviceOnce &o, F &&f, int *value_out = nullptr) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) {   // outside the cache: configure every time
        int v = 0;
        e = f(&v);
        if (value_out) *value_out = v;
        return e;
    }
    std::lock_guard<std::mutex> g(o.m);
    if (!((o.done >> dev) & 1ull)) {
        int v = 0;
        e = f(&v);
        if (e != cudaSuccess) return e;
        o.value[dev] = v;
        o.done |= 1ull << dev;
    }
    if (value_out) *value_out = o.value[dev];
    return cudaSuccess;
}

// n = 8192 kernel v5: the two pass-0 twiddle blocks a ring slot of chunk c
// carries (block c and the later-stage block B(c)), adjacent so that one bulk
// copy moves both: out[L][8][2][T] uint4 from the pass-major inverse table twi
// (host arrays, uint2 entries).
void p8t_slot_twiddles(const uint2 *twi, uint32_t L, size_t tw_limb, uint2 *out);
constexpr size_t kP8tSlotTwEntries = 8 * 2 * 256 * 2;   // uint2 entries per limb

// Kernel launchers (kernels.cu).  Each returns the cudaError_t of the launch
// and adds the number of kernels launched to *launches.
cudaError_t launch_encode(const EncodeArgs &a, cudaStream_t s, uint64_t *launches);
cudaError_t launch_batcher(const BatchArgs &a, cudaStream_t s, uint64_t *launches);
cudaError_t launch_query_ntt(const BatchArgs &a, cudaStream_t s, uint64_t *launches);
cudaError_t launch_eval(const BatchArgs &a, cudaStream_t s, int num_sms, uint64_t *launches);
// chat: write the batch workspace's query-NTT order (kernels.cu chat_word) instead of polynomial order
cudaError_t launch_ntt_forward(const KParams &kp, uint32_t n, uint32_t L, const uint2 *tw_fwd, const uint32_t *in,
                               uint32_t *out, uint32_t count, uint32_t *err, cudaStream_t s, uint64_t *launches,
                               bool chat = false);
cudaError_t launch_pack_rows(const uint32_t *index, const uint32_t *src, uint32_t *dst, uint32_t count,
                             uint32_t row_words, cudaStream_t s, uint64_t *launches);
cudaError_t launch_ntt_inverse(const KParams &kp, uint32_t n, uint32_t L, const uint2 *tw_inv, const uint32_t *in,
                               uint32_t *out, uint32_t count, cudaStream_t s, uint64_t *launches);

}  // namespace wally

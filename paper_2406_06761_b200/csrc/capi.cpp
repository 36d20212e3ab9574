// Host side of the C ABI declared in include/wally.h: parameter validation,
// NTT tables, modulus-switch constants, cluster layout, batch workspace and
// the host-buffer serving pipeline.  All device compute is in kernels.cu.
//
// Citations: PAPER.md P:L1310-1317 (RNS, NTT-friendly limbs), P:L1003 and
// P:L1318-1324 (modulus switch to q_0), Alg 1 P:L664-687 (ServerInit),
// Alg 4 P:L794-808 (ServerComputation), P:L63-64 (server groups received
// queries by cluster).

#include <algorithm>
#include <cmath>
#include <array>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ntt_device.cuh"
#include "wally_ctx.h"

using namespace wally;


static thread_local std::string g_create_err;

int wally_fail(wally_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf; else g_create_err = buf;
    return code;
}
#define fail wally_fail

#define CUDA_OK(ctx, call)                                                                              \
    do {                                                                                                \
        cudaError_t _e = (call);                                                                        \
        if (_e != cudaSuccess) return fail(ctx, WALLY_E_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    } while (0)

// ---------------------------------------------------------------------------
// Number theory (host).  Own implementation: deterministic Miller-Rabin for
// 32-bit integers, primitive root by the first-found power, Shoup companions.
// ---------------------------------------------------------------------------
static uint64_t mulm(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((unsigned __int128)a * b % m); }
static uint64_t powm(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    for (b %= m; e; e >>= 1, b = mulm(b, b, m))
        if (e & 1) r = mulm(r, b, m);
    return r;
}
static uint64_t invm(uint64_t a, uint64_t m) { return powm(a, m - 2, m); }  // m prime

static bool is_prime32(uint64_t n) {
    if (n < 2) return false;
    for (uint64_t p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull})
        if (n % p == 0) return n == p;
    uint64_t d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (uint64_t a : {2ull, 7ull, 61ull}) {  // deterministic for n < 4,759,123,141
        uint64_t x = powm(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; r++) {
            x = mulm(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

static uint64_t resp_words_per_pt(uint32_t n, uint32_t d, uint32_t fmt) {
    const uint64_t E4 = ((uint64_t)(n / d) + 3) & ~3ull;
    if (fmt == WALLY_RESP_COMPACT) return E4 + n;
    if (fmt == WALLY_RESP_COMPACT_DROP) return E4 + 3ull * n / 4;
    return 2ull * n;
}

static bool valid_resp_format(uint32_t fmt) {
    return fmt == WALLY_RESP_FULL || fmt == WALLY_RESP_COMPACT || fmt == WALLY_RESP_COMPACT_DROP;
}

static uint32_t shoup_companion(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }

static uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}

// A primitive 2n-th root of unity mod q: x^((q-1)/2n) for the first x that
// gives psi^n = -1.
static uint64_t primitive_2n_root(uint64_t q, uint32_t n) {
    for (uint64_t x = 2; x < q; x++) {
        uint64_t psi = powm(x, (q - 1) / (2ull * n), q);
        if (powm(psi, n, q) == q - 1) return psi;
    }
    return 0;
}

// Pass-major twiddle tables (layout documented in ntt_device.cuh): per pass
// (TB, R), one block of R entries per hi, holding in execution order the
// entries m + hi*NB + b (m = n / (2 TB 2^s), NB = R >> (s+1)) of the merged
// table; GS (inverse) slot R - (R >> s) + b, CT (forward) slot (R >> (s+1)) + b.
template <int N>
static void build_pass_tables_n(const uint2 *pf, const uint2 *pi, uint2 *fwd, uint2 *inv) {
    using Gm = NttGeom<N>;
    const int TB[3] = {Gm::TB0, Gm::TB1, Gm::TB2}, R[3] = {Gm::R0, Gm::R1, Gm::R2};
    const int OFF[3] = {Gm::TW0, Gm::TW1, Gm::TW2};
    for (int p = 0; p < 3; p++) {
        const int H = N / (TB[p] * R[p]);
        int logr = 0;
        while ((1 << logr) < R[p]) logr++;
        // pass 0 (hi = thread g): slot-pair-major, uint2 index ((slot/2) T + g) 2 + slot%2
        auto at = [&](int hi, int slot) -> size_t {
            if (p == 0) return (size_t)OFF[0] + ((size_t)(slot / 2) * Gm::T + hi) * 2 + (slot % 2);
            return (size_t)OFF[p] + (size_t)hi * R[p] + slot;
        };
        for (int hi = 0; hi < H; hi++) {
            for (int k = 0; k < R[p]; k++) inv[at(hi, k)] = fwd[at(hi, k)] = make_uint2(0, 0);
            for (int s = 0; s < logr; s++) {
                const int nb = R[p] >> (s + 1), m = N / (2 * TB[p] * (1 << s));
                for (int b = 0; b < nb; b++) {
                    inv[at(hi, R[p] - (R[p] >> s) + b)] = pi[m + hi * nb + b];
                    fwd[at(hi, (R[p] >> (s + 1)) + b)] = pf[m + hi * nb + b];
                }
            }
        }
    }
}

static size_t tw_limb_entries(uint32_t n) {
    switch (n) {
        case 1024: return NttGeom<1024>::TW_LIMB;
        case 2048: return NttGeom<2048>::TW_LIMB;
        case 4096: return NttGeom<4096>::TW_LIMB;
        case 8192: return NttGeom<8192>::TW_LIMB;
    }
    return 0;
}

static void build_pass_tables(uint32_t n, const uint2 *pf, const uint2 *pi, uint2 *fwd, uint2 *inv) {
    switch (n) {
        case 1024: build_pass_tables_n<1024>(pf, pi, fwd, inv); break;
        case 2048: build_pass_tables_n<2048>(pf, pi, fwd, inv); break;
        case 4096: build_pass_tables_n<4096>(pf, pi, fwd, inv); break;
        case 8192: build_pass_tables_n<8192>(pf, pi, fwd, inv); break;
    }
}

extern "C" int wally_find_moduli(uint32_t n, uint32_t num_limbs, uint32_t *moduli_out) {
    WALLY_NVTX("wally_find_moduli");
    if (!moduli_out || num_limbs == 0 || num_limbs > WALLY_MAX_LIMBS || n < 2 || (n & (n - 1)))
        return fail(nullptr, WALLY_E_ARG, "wally_find_moduli: bad arguments");
    const uint64_t step = 2ull * n;
    std::vector<uint32_t> found;
    for (uint64_t q = ((1ull << 30) - 2) / step * step + 1; q > step && found.size() < num_limbs; q -= step)
        if (q < (1ull << 30) && is_prime32(q)) found.push_back((uint32_t)q);
    if (found.size() < num_limbs) return fail(nullptr, WALLY_E_PARAMS, "not enough NTT-friendly primes");
    for (uint32_t i = 0; i < num_limbs; i++) moduli_out[i] = found[num_limbs - 1 - i];
    return WALLY_OK;
}

// ---------------------------------------------------------------------------
// create / destroy
// ---------------------------------------------------------------------------
extern "C" const char *wally_last_error(const wally_ctx *ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

extern "C" uint64_t wally_kernel_launches(const wally_ctx *ctx) { return ctx ? ctx->launches : 0; }

extern "C" void wally_destroy(wally_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    wally_comm_release(c);
    cudaFree(c->d_tw_fwd);
    cudaFree(c->d_tw_inv);
    cudaFree(c->d_tw_mrg);
    cudaFree(c->d_tw_slot);
    cudaFree(c->d_local_of_cluster);
    cudaFree(c->d_pt_base);
    cudaFree(c->d_n_pt);
    cudaFree(c->d_pt_li);
    cudaFree(c->d_pt_k);
    cudaFree(c->d_size);
    cudaFree(c->d_entry_base);
    for (auto &s : c->slot) {
        if (s.ids) cudaFreeHost(s.ids);
        if (s.off) cudaFreeHost(s.off);
        if (s.done) cudaEventDestroy(s.done);
    }
    if (c->side) cudaStreamDestroy(c->side);
    if (c->err_host) cudaFreeHost(c->err_host);
    for (auto &r : c->ev_rec) for (auto e : r) c->ev_pool.push_back(e);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    delete c;
}

extern "C" int wally_create(const wally_params *pp, int device, wally_ctx **out) {
    WALLY_NVTX("wally_create");
    if (!pp || !out) return fail(nullptr, WALLY_E_ARG, "wally_create: null argument");
    *out = nullptr;
    const wally_params &p = *pp;
    if (p.n != 1024 && p.n != 2048 && p.n != 4096 && p.n != 8192)
        return fail(nullptr, WALLY_E_PARAMS, "n=%u unsupported (1024, 2048, 4096, 8192)", p.n);
    if (p.num_limbs < 1 || p.num_limbs > WALLY_MAX_LIMBS)
        return fail(nullptr, WALLY_E_PARAMS, "num_limbs=%u unsupported (1..%d)", p.num_limbs, WALLY_MAX_LIMBS);
    if (p.d < 1 || p.d > p.n) return fail(nullptr, WALLY_E_PARAMS, "d=%u must be in [1, n]", p.d);
    if (p.t < 2) return fail(nullptr, WALLY_E_PARAMS, "t=%u must be >= 2", p.t);
    if (!valid_resp_format(p.resp_format))
        return fail(nullptr, WALLY_E_PARAMS, "resp_format=%u unknown", p.resp_format);
    if (p.resp_format == WALLY_RESP_COMPACT_DROP && p.n != 4096)
        return fail(nullptr, WALLY_E_PARAMS,
                    "WALLY_RESP_COMPACT_DROP is specified for n = 4096 (its noise bound and plane order; DESIGN.md)");
    if (p.resp_format == WALLY_RESP_COMPACT_DROP) {
        // the paper's LSB-drop rule (z = 8; correctness ||e + e_drop|| < q_0 / 2t) for
        // c1 rounded to 2^b (|c1^l| <= 2^(b-1)) and c0 not dropped: z sqrt(2n/9) 2^(b-1) < q_0 / (2t)
        // (reading S20)
        const double lhs = 8.0 * std::sqrt(2.0 * p.n / 9.0) * (double)(1u << (WALLY_RESP_DROP_BITS - 1));
        const double rhs = (double)p.moduli[0] / (2.0 * (double)p.t);
        if (!(lhs < rhs))
            return fail(nullptr, WALLY_E_PARAMS,
                        "WALLY_RESP_COMPACT_DROP: z sqrt(2n/9) 2^%u = %.1f is not below q_0/2t = %.1f (P:L1005, z = 8)",
                        WALLY_RESP_DROP_BITS - 1, lhs, rhs);
    }
    for (uint32_t i = 0; i < p.num_limbs; i++) {
        uint32_t q = p.moduli[i];
        if (q >= (1u << 30) || q % (2 * p.n) != 1 || !is_prime32(q))
            return fail(nullptr, WALLY_E_PARAMS, "modulus q_%u=%u is not a prime < 2^30 with q = 1 mod 2n", i, q);
        if (i && q <= p.moduli[i - 1]) return fail(nullptr, WALLY_E_PARAMS, "moduli must be strictly ascending");
    }
    if (p.moduli[p.num_limbs - 1] >= 2ull * p.moduli[0])
        return fail(nullptr, WALLY_E_PARAMS, "need q_{L-1} < 2 q_0 (the rounding residues r < q_m enter the switch step unreduced mod q_l)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(nullptr, WALLY_E_CUDA, "no CUDA device %d", device);

    wally_ctx *c = new wally_ctx();
    c->p = p;
    c->device = device;
    c->E = p.n / p.d;
    c->wpp = resp_words_per_pt(p.n, p.d, p.resp_format);
    if (cudaSetDevice(device) != cudaSuccess) { delete c; return fail(nullptr, WALLY_E_CUDA, "cudaSetDevice"); }
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);

    const uint32_t n = p.n, L = p.num_limbs;
    int logn = 0;
    while ((1u << logn) < n) logn++;
    KParams &kp = c->kp;
    const size_t tw_limb = tw_limb_entries(n);
    std::vector<uint2> twf((size_t)L * tw_limb), twi((size_t)L * tw_limb), twm((size_t)L * n);
    for (uint32_t l = 0; l < L; l++) {
        const uint64_t q = p.moduli[l];
        kp.q[l] = (uint32_t)q;
        kp.q2[l] = (uint32_t)(2 * q);
        kp.h[l] = (uint32_t)(q / 2);
        kp.ninv[l] = (uint32_t)invm(n, q);
        kp.ninvp[l] = shoup_companion(kp.ninv[l], (uint32_t)q);
        {   // -q^{-1} mod 2^32 by Newton iteration (q odd: x = q is q^{-1} mod 2^3)
            uint32_t x = (uint32_t)q;
            for (int it = 0; it < 5; it++) x *= 2u - (uint32_t)q * x;
            kp.mqinv[l] = 0u - x;
        }
        // fold F_l = n^{-1} prod_{k>l} q_k^{-1} mod q_l
        uint64_t f = invm(n, q);
        for (uint32_t k = l + 1; k < L; k++) f = mulm(f, invm(p.moduli[k] % q, q), q);
        kp.fold[l] = (uint32_t)f;
        kp.foldp[l] = shoup_companion((uint32_t)f, (uint32_t)q);
        // C[l][m] = prod_{k=l+1..m} q_k^{-1} mod q_l
        uint64_t cm = 1;
        for (uint32_t m = l + 1; m < L; m++) {
            cm = mulm(cm, invm(p.moduli[m] % q, q), q);
            kp.C[l][m] = (uint32_t)cm;
            kp.Cp[l][m] = shoup_companion((uint32_t)cm, (uint32_t)q);
        }
        for (uint32_t m = l + 1; m < L; m++) {
            kp.Qi[l][m] = (uint32_t)invm(p.moduli[m] % q, q);
            kp.Qip[l][m] = shoup_companion(kp.Qi[l][m], (uint32_t)q);
        }
        const uint64_t psi = primitive_2n_root(q, n);
        const uint64_t psi_inv = invm(psi, q);
        std::vector<uint2> pf(n), pi(n);   // standard merged tables psi^{brev(i)}, psi^{-brev(i)}
        for (uint32_t i = 0; i < n; i++) {
            const uint32_t e = bitrev(i, logn);
            const uint32_t w = (uint32_t)powm(psi, e, q), wi = (uint32_t)powm(psi_inv, e, q);
            pf[i] = make_uint2(w, shoup_companion(w, (uint32_t)q));
            pi[i] = make_uint2(wi, shoup_companion(wi, (uint32_t)q));
        }
        build_pass_tables(n, pf.data(), pi.data(), twf.data() + l * tw_limb, twi.data() + l * tw_limb);
        std::copy(pi.begin(), pi.end(), twm.begin() + (size_t)l * n);
    }
    const size_t tb = sizeof(uint2) * twf.size();
    if (cudaMalloc(&c->d_tw_fwd, tb) != cudaSuccess || cudaMalloc(&c->d_tw_inv, tb) != cudaSuccess ||
        cudaMalloc(&c->d_tw_mrg, sizeof(uint2) * twm.size()) != cudaSuccess) {
        wally_destroy(c);
        return fail(nullptr, WALLY_E_OOM, "twiddle table allocation failed");
    }
    cudaMemcpy(c->d_tw_fwd, twf.data(), tb, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_tw_inv, twi.data(), tb, cudaMemcpyHostToDevice);
    cudaMemcpy(c->d_tw_mrg, twm.data(), sizeof(uint2) * twm.size(), cudaMemcpyHostToDevice);
    if (n == 8192) {
        std::vector<uint2> tws((size_t)L * kP8tSlotTwEntries);
        p8t_slot_twiddles(twi.data(), L, tw_limb, tws.data());
        if (cudaMalloc(&c->d_tw_slot, sizeof(uint2) * tws.size()) != cudaSuccess) {
            wally_destroy(c);
            return fail(nullptr, WALLY_E_OOM, "twiddle table allocation failed");
        }
        cudaMemcpy(c->d_tw_slot, tws.data(), sizeof(uint2) * tws.size(), cudaMemcpyHostToDevice);
    }
    for (auto &s : c->slot) cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
    if (cudaGetLastError() != cudaSuccess) {
        wally_destroy(c);
        return fail(nullptr, WALLY_E_CUDA, "context setup failed");
    }
    *out = c;
    return WALLY_OK;
}

// ---------------------------------------------------------------------------
// ServerInit
// ---------------------------------------------------------------------------
template <typename T>
static int upload(wally_ctx *c, T **dst, const std::vector<T> &v) {
    cudaFree(*dst);
    *dst = nullptr;
    size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
    if (cudaMalloc(dst, bytes) != cudaSuccess) return fail(c, WALLY_E_OOM, "device table allocation failed");
    if (!v.empty()) CUDA_OK(c, cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return WALLY_OK;
}

template <typename IsLocal>
static int load_clusters_impl(wally_ctx *c, uint32_t total_clusters, const uint32_t *sizes, IsLocal is_local,
                              std::vector<int32_t> owner, int32_t rank) {
    if (!sizes || total_clusters == 0) return fail(c, WALLY_E_ARG, "load_clusters: need >= 1 cluster and sizes");
    std::vector<int32_t> local(total_clusters, -1);
    std::vector<uint32_t> pt_base, n_pt, pt_li, pt_k, size;
    std::vector<uint64_t> entry_base;
    uint64_t entries = 0;
    uint32_t npt = 0, max_pt = 0;
    for (uint32_t cl = 0; cl < total_clusters; cl++) {
        if (sizes[cl] == 0) return fail(c, WALLY_E_ARG, "cluster %u is empty", cl);
        if (!is_local(cl)) continue;
        const uint32_t li = (uint32_t)pt_base.size();
        const uint32_t P = (sizes[cl] + c->E - 1) / c->E;
        local[cl] = (int32_t)li;
        // store slots: P rounded up to the store's alignment (n = 8192: plaintext pairs; the
        // pad plaintext k = P encodes no entry, i.e. zero)
        const uint32_t al = pt_store_align(c->p.n), Ps = (P + al - 1) / al * al;
        pt_base.push_back(npt);
        n_pt.push_back(P);
        size.push_back(sizes[cl]);
        entry_base.push_back(entries);
        for (uint32_t k = 0; k < Ps; k++) { pt_li.push_back(li); pt_k.push_back(k); }
        npt += Ps;
        max_pt = std::max(max_pt, P);
        entries += sizes[cl];
    }
    if (pt_base.empty()) return fail(c, WALLY_E_ARG, "rank %d owns no cluster", rank);
    cudaSetDevice(c->device);
    int rc;
    if ((rc = upload(c, &c->d_local_of_cluster, local)) || (rc = upload(c, &c->d_pt_base, pt_base)) ||
        (rc = upload(c, &c->d_n_pt, n_pt)) || (rc = upload(c, &c->d_pt_li, pt_li)) ||
        (rc = upload(c, &c->d_pt_k, pt_k)) || (rc = upload(c, &c->d_size, size)) ||
        (rc = upload(c, &c->d_entry_base, entry_base)))
        return rc;
    c->total_clusters = total_clusters;
    c->n_local = (uint32_t)pt_base.size();
    c->npt = npt;
    c->max_pt = max_pt;
    c->local_of_cluster = std::move(local);
    c->owner = std::move(owner);
    c->rank = rank;
    c->pt_of_local = std::move(n_pt);
    c->local_entries = entries;
    c->store = nullptr;
    c->loaded = true;
    return WALLY_OK;
}

extern "C" int wally_load_clusters(wally_ctx *c, uint32_t total_clusters, const uint32_t *sizes,
                                   const int32_t *owner, int32_t rank) {
    WALLY_NVTX("wally_load_clusters");
    if (!c) return WALLY_E_ARG;
    return load_clusters_impl(
        c, total_clusters, sizes, [&](uint32_t cl) { return !owner || owner[cl] == rank; },
        owner && sizes ? std::vector<int32_t>(owner, owner + total_clusters) : std::vector<int32_t>(), rank);
}

extern "C" int wally_load_clusters_replicated(wally_ctx *c, uint32_t total_clusters, const uint32_t *sizes,
                                              const uint64_t *mask, int32_t rank) {
    WALLY_NVTX("wally_load_clusters_replicated");
    if (!c) return WALLY_E_ARG;
    if (!mask || rank < 0 || rank >= 64) return fail(c, WALLY_E_ARG, "load_clusters_replicated: bad mask or rank");
    // owner[] (wally_route_queries) reports the lowest replica of each cluster
    std::vector<int32_t> owner(total_clusters, -1);
    for (uint32_t cl = 0; cl < total_clusters && sizes; cl++)
        if (mask[cl]) owner[cl] = __builtin_ctzll(mask[cl]);
    return load_clusters_impl(
        c, total_clusters, sizes, [&](uint32_t cl) { return (mask[cl] >> rank) & 1ull; }, std::move(owner), rank);
}

extern "C" int wally_response_words_per_plaintext(const wally_ctx *c, uint64_t *words) {
    WALLY_NVTX("wally_response_words_per_plaintext");
    if (!c || !words) return WALLY_E_ARG;
    *words = c->wpp;
    return WALLY_OK;
}

extern "C" int wally_modmuls_per_pair(const wally_ctx *c, uint64_t *out) {
    WALLY_NVTX("wally_modmuls_per_pair");
    if (!c || !out) return WALLY_E_ARG;
    const bool compact = c->p.resp_format != WALLY_RESP_FULL;
    *out = modmuls_per_pair(c->p.n, c->p.num_limbs, c->p.d, pruned_c0_path(c->p.n, c->p.num_limbs, c->p.d, compact));
    return WALLY_OK;
}

extern "C" int wally_plaintext_store_bytes(const wally_ctx *c, size_t *bytes) {
    WALLY_NVTX("wally_plaintext_store_bytes");
    if (!c || !bytes) return WALLY_E_ARG;
    if (!c->loaded) return fail(const_cast<wally_ctx *>(c), WALLY_E_STATE, "load_clusters first");
    *bytes = (size_t)c->npt * c->p.num_limbs * pt_store_planes(c->p.n) * c->p.n * sizeof(uint32_t);
    return WALLY_OK;
}

extern "C" int wally_local_entry_count(const wally_ctx *c, uint64_t *count) {
    WALLY_NVTX("wally_local_entry_count");
    if (!c || !count) return WALLY_E_ARG;
    if (!c->loaded) return fail(const_cast<wally_ctx *>(c), WALLY_E_STATE, "load_clusters first");
    *count = c->local_entries;
    return WALLY_OK;
}

extern "C" int wally_encode_plaintexts_ntt(wally_ctx *c, const int8_t *entries_dev, void *store_dev,
                                           size_t store_bytes, void *stream) {
    WALLY_NVTX("wally_encode_plaintexts_ntt");
    if (!c) return WALLY_E_ARG;
    if (!c->loaded) return fail(c, WALLY_E_STATE, "load_clusters first");
    size_t need = 0;
    wally_plaintext_store_bytes(c, &need);
    if (!entries_dev || !store_dev) return fail(c, WALLY_E_ARG, "encode: null device pointer");
    if (store_bytes < need) return fail(c, WALLY_E_ARG, "encode: store has %zu bytes, need %zu", store_bytes, need);
    if ((uintptr_t)store_dev % 16) return fail(c, WALLY_E_ARG, "encode: store must be 16-byte aligned");
    cudaSetDevice(c->device);
    EncodeArgs a{};
    a.kp = c->kp;
    a.n = c->p.n;
    a.L = c->p.num_limbs;
    a.d = c->p.d;
    a.E = c->E;
    a.npt = c->npt;
    a.tw_fwd = c->d_tw_fwd;
    a.entries = entries_dev;
    a.pt_li = c->d_pt_li;
    a.pt_k = c->d_pt_k;
    a.entry_base = c->d_entry_base;
    a.size = c->d_size;
    a.store = (uint32_t *)store_dev;
    CUDA_OK(c, launch_encode(a, (cudaStream_t)stream, &c->launches));
    c->store = (const uint32_t *)store_dev;
    return WALLY_OK;
}

// ---------------------------------------------------------------------------
// batches
// ---------------------------------------------------------------------------
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

WsLayout wally::ws_layout(uint32_t nq, uint32_t n_local, uint32_t n, uint32_t L) {
    // misc first: its offset (0) does not depend on nq, so wally_check_batch
    // can find the error word of any batch's workspace.
    WsLayout w{};
    size_t o = 0;
    w.zero_begin = o;
    w.misc = o; o += sizeof(uint32_t) * kMiscWords;
    w.counts = o; o += sizeof(uint32_t) * n_local;
    w.fill = o; o += sizeof(uint32_t) * n_local;
    w.zero_bytes = o - w.zero_begin;
    o = align256(o);
    w.ids = o; o = align256(o + sizeof(uint32_t) * nq);
    w.resp_off = o; o = align256(o + sizeof(uint64_t) * nq);
    w.perm = o; o = align256(o + sizeof(uint32_t) * nq);
    w.seg = o; o = align256(o + sizeof(uint32_t) * n_local);
    w.item_start = o; o = align256(o + sizeof(uint32_t) * (n_local + 1));
    w.chat = o; o = align256(o + sizeof(uint32_t) * (size_t)nq * 2 * L * n);
    w.total = o;
    return w;
}

extern "C" int wally_workspace_bytes(const wally_ctx *c, uint32_t nq, size_t *bytes) {
    WALLY_NVTX("wally_workspace_bytes");
    if (!c || !bytes) return WALLY_E_ARG;
    if (!c->loaded) return fail(const_cast<wally_ctx *>(c), WALLY_E_STATE, "load_clusters first");
    *bytes = ws_layout(nq, c->n_local, c->p.n, c->p.num_limbs).total;
    return WALLY_OK;
}

static int layout_impl(const wally_ctx *c, uint32_t nq, const uint32_t *ids, uint64_t *off, uint64_t *total) {
    uint64_t o = 0;
    const uint64_t per = c->wpp;
    for (uint32_t q = 0; q < nq; q++) {
        const uint32_t cl = ids[q];
        if (cl >= c->total_clusters || c->local_of_cluster[cl] < 0)
            return fail(const_cast<wally_ctx *>(c), WALLY_E_UNKNOWN_CLUSTER,
                        "query %u names cluster %u, which is not local (total %u)", q, cl, c->total_clusters);
        if (off) off[q] = o;
        o += per * c->pt_of_local[c->local_of_cluster[cl]];
    }
    if (off) off[nq] = o;
    if (total) *total = o;
    return WALLY_OK;
}

extern "C" int wally_response_layout(const wally_ctx *c, uint32_t nq, const uint32_t *ids, uint64_t *off,
                                     uint64_t *total) {
    WALLY_NVTX("wally_response_layout");
    if (!c || (nq && !ids)) return WALLY_E_ARG;
    if (!c->loaded) return fail(const_cast<wally_ctx *>(c), WALLY_E_STATE, "load_clusters first");
    return layout_impl(c, nq, ids, off, total);
}

// Evaluate one batch whose query ciphertexts are already on the device.
static int eval_impl(wally_ctx *c, uint32_t nq, const uint32_t *ids, const uint32_t *query_dev, uint32_t *resp_dev,
                     uint64_t resp_words, void *ws_dev, size_t ws_bytes, cudaStream_t s) {
    if (!c->loaded) return fail(c, WALLY_E_STATE, "load_clusters first");
    if (!c->store) return fail(c, WALLY_E_STATE, "encode_plaintexts_ntt first");
    if (nq == 0) return WALLY_OK;
    if (!ids || !query_dev || !resp_dev || !ws_dev) return fail(c, WALLY_E_ARG, "eval: null pointer");
    if ((uintptr_t)query_dev % 16 || (uintptr_t)ws_dev % 256)
        return fail(c, WALLY_E_ARG, "eval: query_ct must be 16-byte and workspace 256-byte aligned");
    const WsLayout w = ws_layout(nq, c->n_local, c->p.n, c->p.num_limbs);
    if (ws_bytes < w.total) return fail(c, WALLY_E_ARG, "eval: workspace %zu bytes, need %zu", ws_bytes, w.total);
    // metadata staging slot (pinned); wait until its previous copy finished
    wally_ctx::Slot &sl = c->slot[c->next_slot];
    c->next_slot ^= 1;
    if (sl.pending) { cudaEventSynchronize(sl.done); sl.pending = false; }
    if (sl.cap < nq) {
        if (sl.ids) cudaFreeHost(sl.ids);
        if (sl.off) cudaFreeHost(sl.off);
        sl.ids = nullptr; sl.off = nullptr; sl.cap = 0;
        if (cudaMallocHost(&sl.ids, sizeof(uint32_t) * nq) != cudaSuccess ||
            cudaMallocHost(&sl.off, sizeof(uint64_t) * (nq + 1)) != cudaSuccess)
            return fail(c, WALLY_E_OOM, "pinned staging allocation failed");
        sl.cap = nq;
    }
    uint64_t total = 0;
    int rc = layout_impl(c, nq, ids, sl.off, &total);
    if (rc) return rc;
    if (resp_words < total) return fail(c, WALLY_E_ARG, "eval: response buffer has %llu words, need %llu",
                                        (unsigned long long)resp_words, (unsigned long long)total);
    memcpy(sl.ids, ids, sizeof(uint32_t) * nq);
    char *ws = (char *)ws_dev;
    CUDA_OK(c, cudaMemcpyAsync(ws + w.ids, sl.ids, sizeof(uint32_t) * nq, cudaMemcpyHostToDevice, s));
    CUDA_OK(c, cudaMemcpyAsync(ws + w.resp_off, sl.off, sizeof(uint64_t) * nq, cudaMemcpyHostToDevice, s));
    CUDA_OK(c, cudaEventRecord(sl.done, s));
    sl.pending = true;
    CUDA_OK(c, cudaMemsetAsync(ws + w.zero_begin, 0, w.zero_bytes, s));
    BatchArgs a{};
    a.kp = c->kp;
    a.n = c->p.n;
    a.L = c->p.num_limbs;
    a.d = c->p.d;
    a.E = c->E;
    a.wpp = (uint32_t)c->wpp;
    a.compact = c->p.resp_format != WALLY_RESP_FULL;
    a.drop = c->p.resp_format == WALLY_RESP_COMPACT_DROP;
    a.nq = nq;
    // a small batch would leave most thread groups idle with 8 queries per
    // work item (c1: 32 items for 296 groups): one query per item instead
    a.chunk = (nq < 4u * (uint32_t)c->num_sms) ? 1u : kQueryChunk;
    a.ppi = eval_plaintexts_per_item(a.n, a.L, a.d, a.compact);
    if (a.ppi == 2) a.chunk = kP8QueryChunk;   // n = 8192 kernel v5 (wally_internal.h)
    a.n_local = c->n_local;
    a.total_clusters = c->total_clusters;
    a.tw_fwd = c->d_tw_fwd;
    a.tw_inv = c->d_tw_inv;
    a.tw_mrg = c->d_tw_mrg;
    a.tw_slot = c->d_tw_slot;
    a.local_of_cluster = c->d_local_of_cluster;
    a.pt_base = c->d_pt_base;
    a.n_pt = c->d_n_pt;
    a.store = c->store;
    a.query_ct = query_dev;
    a.resp = resp_dev;
    a.ids = (uint32_t *)(ws + w.ids);
    a.resp_off = (uint64_t *)(ws + w.resp_off);
    a.perm = (uint32_t *)(ws + w.perm);
    a.counts = (uint32_t *)(ws + w.counts);
    a.fill = (uint32_t *)(ws + w.fill);
    a.misc = (uint32_t *)(ws + w.misc);
    a.seg = (uint32_t *)(ws + w.seg);
    a.item_start = (uint32_t *)(ws + w.item_start);
    a.chat = (uint32_t *)(ws + w.chat);
    a.resp_words = resp_words;
    a.store_words = (uint64_t)c->npt * c->p.num_limbs * pt_store_planes(c->p.n) * c->p.n;
    std::array<cudaEvent_t, 4> ev{};
    if (c->timing) {
        for (auto &e : ev) {
            if (c->ev_pool.empty()) {
                CUDA_OK(c, cudaEventCreate(&e));
            } else {
                e = c->ev_pool.back();
                c->ev_pool.pop_back();
            }
        }
        c->ev_rec.push_back(ev);
        CUDA_OK(c, cudaEventRecord(ev[0], s));
    }
    {
        WALLY_NVTX("a1 batcher");
        CUDA_OK(c, launch_batcher(a, s, &c->launches));
    }
    if (c->timing) CUDA_OK(c, cudaEventRecord(ev[1], s));
    {
        WALLY_NVTX("a2 forward NTT");
        CUDA_OK(c, launch_query_ntt(a, s, &c->launches));
    }
    if (c->timing) CUDA_OK(c, cudaEventRecord(ev[2], s));
    {
        WALLY_NVTX("a3-a6 fused pointwise/iNTT/mod-switch");
        CUDA_OK(c, launch_eval(a, s, c->num_sms, &c->launches));
    }
    if (c->timing) CUDA_OK(c, cudaEventRecord(ev[3], s));
    return WALLY_OK;
}

extern "C" int wally_enable_stage_timing(wally_ctx *c, int enable) {
    WALLY_NVTX("wally_enable_stage_timing");
    if (!c) return WALLY_E_ARG;
    c->timing = enable != 0;
    return WALLY_OK;
}

extern "C" int wally_stage_times(wally_ctx *c, double *ms, uint64_t *batches) {
    WALLY_NVTX("wally_stage_times");
    if (!c || !ms) return WALLY_E_ARG;
    cudaSetDevice(c->device);
    ms[0] = ms[1] = ms[2] = 0.0;
    for (auto &r : c->ev_rec) {
        CUDA_OK(c, cudaEventSynchronize(r[3]));
        for (int i = 0; i < 3; i++) {
            float t = 0.f;
            CUDA_OK(c, cudaEventElapsedTime(&t, r[i], r[i + 1]));
            ms[i] += t;
        }
    }
    if (batches) *batches = c->ev_rec.size();
    for (auto &r : c->ev_rec) for (auto e : r) c->ev_pool.push_back(e);
    c->ev_rec.clear();
    return WALLY_OK;
}

extern "C" int wally_eval_batch(wally_ctx *c, uint32_t nq, const uint32_t *ids, const uint32_t *query_dev,
                                uint32_t *resp_dev, uint64_t resp_words, void *ws_dev, size_t ws_bytes, void *stream) {
    WALLY_NVTX("wally_eval_batch");
    if (!c) return WALLY_E_ARG;
    cudaSetDevice(c->device);
    return eval_impl(c, nq, ids, query_dev, resp_dev, resp_words, ws_dev, ws_bytes, (cudaStream_t)stream);
}

extern "C" int wally_check_batch(wally_ctx *c, const void *ws_dev, void *stream) {
    WALLY_NVTX("wally_check_batch");
    if (!c || !ws_dev) return WALLY_E_ARG;
    cudaSetDevice(c->device);
    CUDA_OK(c, cudaStreamSynchronize((cudaStream_t)stream));
    uint32_t misc[kMiscWords];
    CUDA_OK(c, cudaMemcpy(misc, ws_dev, sizeof misc, cudaMemcpyDeviceToHost));
    if (misc[kMiscErr] & kErrResidue)
        return fail(c, WALLY_E_RESIDUE, "a query ciphertext residue was >= its modulus");
    return WALLY_OK;
}

extern "C" int wally_fetch_responses(wally_ctx *c, const uint32_t *resp_dev, uint64_t words, uint32_t *out_host,
                                     void *stream) {
    WALLY_NVTX("wally_fetch_responses");
    if (!c || (words && (!resp_dev || !out_host))) return WALLY_E_ARG;
    cudaSetDevice(c->device);
    CUDA_OK(c, cudaMemcpyAsync(out_host, resp_dev, words * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               (cudaStream_t)stream));
    CUDA_OK(c, cudaStreamSynchronize((cudaStream_t)stream));
    return WALLY_OK;
}

extern "C" int wally_route_queries(const wally_ctx *c, uint32_t nq, const uint32_t *ids, int32_t *dest) {
    WALLY_NVTX("wally_route_queries");
    if (!c || (nq && (!ids || !dest))) return WALLY_E_ARG;
    if (!c->loaded) return fail(const_cast<wally_ctx *>(c), WALLY_E_STATE, "load_clusters first");
    for (uint32_t q = 0; q < nq; q++) {
        if (ids[q] >= c->total_clusters)
            return fail(const_cast<wally_ctx *>(c), WALLY_E_UNKNOWN_CLUSTER, "query %u: cluster %u >= %u", q, ids[q],
                        c->total_clusters);
        dest[q] = c->owner.empty() ? c->rank : c->owner[ids[q]];
    }
    return WALLY_OK;
}

// ---------------------------------------------------------------------------
// host-buffer serving pipeline
// ---------------------------------------------------------------------------
struct HostWs {
    size_t ws, qstage, rstage, per_slot, total;
};
static HostWs host_ws(const wally_ctx *c, uint32_t sub) {
    HostWs h{};
    h.ws = align256(ws_layout(sub, c->n_local, c->p.n, c->p.num_limbs).total);
    h.qstage = align256((size_t)sub * 2 * c->p.num_limbs * c->p.n * sizeof(uint32_t));
    h.rstage = align256((size_t)sub * c->max_pt * c->wpp * sizeof(uint32_t));
    h.per_slot = h.ws + h.qstage + h.rstage;
    h.total = 2 * h.per_slot;
    return h;
}

extern "C" int wally_host_workspace_bytes(const wally_ctx *c, uint32_t sub, size_t *bytes) {
    WALLY_NVTX("wally_host_workspace_bytes");
    if (!c || !bytes || sub == 0) return WALLY_E_ARG;
    if (!c->loaded) return fail(const_cast<wally_ctx *>(c), WALLY_E_STATE, "load_clusters first");
    *bytes = host_ws(c, sub).total;
    return WALLY_OK;
}

extern "C" int wally_eval_batch_host(wally_ctx *c, uint32_t nq, const uint32_t *ids, const uint32_t *query_host,
                                     uint32_t *resp_host, uint64_t resp_words, uint32_t sub, void *ws_dev,
                                     size_t ws_bytes, void *stream) {
    WALLY_NVTX("wally_eval_batch_host");
    if (!c) return WALLY_E_ARG;
    if (!c->loaded) return fail(c, WALLY_E_STATE, "load_clusters first");
    if (!c->store) return fail(c, WALLY_E_STATE, "encode_plaintexts_ntt first");
    if (nq == 0) return WALLY_OK;
    if (!ids || !query_host || !resp_host || !ws_dev || sub == 0) return fail(c, WALLY_E_ARG, "eval_host: bad args");
    cudaSetDevice(c->device);
    const HostWs h = host_ws(c, sub);
    if (ws_bytes < h.total) return fail(c, WALLY_E_ARG, "eval_host: workspace %zu bytes, need %zu", ws_bytes, h.total);
    std::vector<uint64_t> off(nq + 1);
    uint64_t total = 0;
    int rc = layout_impl(c, nq, ids, off.data(), &total);
    if (rc) return rc;
    if (resp_words < total) return fail(c, WALLY_E_ARG, "eval_host: response buffer too small");
    const size_t nsub = (nq + (size_t)sub - 1) / sub;
    if (c->err_cap < nsub) {
        if (c->err_host) cudaFreeHost(c->err_host);
        c->err_host = nullptr;
        c->err_cap = 0;
        if (cudaMallocHost(&c->err_host, sizeof(uint32_t) * nsub) != cudaSuccess)
            return fail(c, WALLY_E_OOM, "pinned error-word allocation failed");
        c->err_cap = nsub;
    }
    const WsLayout wl = ws_layout(sub, c->n_local, c->p.n, c->p.num_limbs);
    cudaStream_t st[2] = {(cudaStream_t)stream, c->side};
    cudaEvent_t start;
    CUDA_OK(c, cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CUDA_OK(c, cudaEventRecord(start, st[0]));
    CUDA_OK(c, cudaStreamWaitEvent(st[1], start, 0));
    const size_t qwords = 2ull * c->p.num_limbs * c->p.n;
    uint32_t b = 0;
    for (uint32_t q0 = 0; q0 < nq; q0 += sub, b++) {
        const uint32_t cnt = std::min(sub, nq - q0);
        const int k = b & 1;
        cudaStream_t s = st[k];
        char *base = (char *)ws_dev + k * h.per_slot;
        uint32_t *qdev = (uint32_t *)(base + h.ws);
        uint32_t *rdev = (uint32_t *)(base + h.ws + h.qstage);
        CUDA_OK(c, cudaMemcpyAsync(qdev, query_host + q0 * qwords, cnt * qwords * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, s));
        const uint64_t words = off[q0 + cnt] - off[q0];
        rc = eval_impl(c, cnt, ids + q0, qdev, rdev, words, base, h.ws, s);
        if (rc) { cudaEventDestroy(start); return rc; }
        CUDA_OK(c, cudaMemcpyAsync(resp_host + off[q0], rdev, words * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CUDA_OK(c, cudaMemcpyAsync(c->err_host + b, base + wl.misc + sizeof(uint32_t) * kMiscErr, sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, s));
    }
    cudaEventDestroy(start);
    CUDA_OK(c, cudaStreamSynchronize(st[1]));
    CUDA_OK(c, cudaStreamSynchronize(st[0]));
    uint32_t err = 0;
    for (size_t i = 0; i < nsub; i++) err |= c->err_host[i];
    if (err & kErrResidue) return fail(c, WALLY_E_RESIDUE, "a query ciphertext residue was >= its modulus");
    return WALLY_OK;
}

// ---------------------------------------------------------------------------
// test hooks
// ---------------------------------------------------------------------------
extern "C" int wally_ntt_forward(wally_ctx *c, const uint32_t *in, uint32_t *out, uint32_t count, void *stream) {
    WALLY_NVTX("wally_ntt_forward");
    if (!c || (count && (!in || !out))) return WALLY_E_ARG;
    if ((uintptr_t)out % 16) return fail(c, WALLY_E_ARG, "ntt_forward: out must be 16-byte aligned");
    cudaSetDevice(c->device);
    CUDA_OK(c, launch_ntt_forward(c->kp, c->p.n, c->p.num_limbs, c->d_tw_fwd, in, out, count, nullptr,
                                  (cudaStream_t)stream, &c->launches));
    return WALLY_OK;
}

extern "C" int wally_ntt_inverse(wally_ctx *c, const uint32_t *in, uint32_t *out, uint32_t count, void *stream) {
    WALLY_NVTX("wally_ntt_inverse");
    if (!c || (count && (!in || !out))) return WALLY_E_ARG;
    if ((uintptr_t)in % 16) return fail(c, WALLY_E_ARG, "ntt_inverse: in must be 16-byte aligned");
    cudaSetDevice(c->device);
    CUDA_OK(c, launch_ntt_inverse(c->kp, c->p.n, c->p.num_limbs, c->d_tw_inv, in, out, count, (cudaStream_t)stream,
                                  &c->launches));
    return WALLY_OK;
}

// ---------------------------------------------------------------------------
// multi-GPU routing (host logic)
// ---------------------------------------------------------------------------
extern "C" int wally_assign_owners(uint32_t total_clusters, const double *weight, uint32_t world, int32_t *owner) {
    WALLY_NVTX("wally_assign_owners");
    if (!weight || !owner || total_clusters == 0 || world == 0)
        return fail(nullptr, WALLY_E_ARG, "assign_owners: bad arguments");
    for (uint32_t c = 0; c < total_clusters; c++)
        if (!(weight[c] >= 0.0)) return fail(nullptr, WALLY_E_ARG, "assign_owners: weight[%u] < 0 or NaN", c);
    std::vector<uint32_t> ids(total_clusters);
    for (uint32_t c = 0; c < total_clusters; c++) ids[c] = c;
    std::stable_sort(ids.begin(), ids.end(), [&](uint32_t a, uint32_t b) { return weight[a] > weight[b]; });
    std::vector<double> load(world, 0.0);
    for (uint32_t c : ids) {
        uint32_t best = 0;
        for (uint32_t r = 1; r < world; r++)
            if (load[r] < load[best]) best = r;
        owner[c] = (int32_t)best;
        load[best] += weight[c];
    }
    return WALLY_OK;
}

// Plan from a per-query destination rank (shared by both routing modes).
static int route_plan_dest(uint32_t nq, const uint32_t *ids, uint32_t total_clusters, const uint32_t *sizes,
                           const int32_t *dest, uint32_t n, uint32_t d, uint32_t resp_format, uint32_t world,
                           uint32_t *counts, uint32_t *order, uint64_t *resp_words, uint64_t *gathered_off) {
    const uint64_t E = n / d, per_pt = resp_words_per_pt(n, d, resp_format);
    std::vector<uint32_t> cnt(world, 0), start(world, 0);
    std::vector<uint64_t> words(world, 0);
    for (uint32_t q = 0; q < nq; q++) {
        const uint32_t r = (uint32_t)dest[q];
        cnt[r]++;
        words[r] += per_pt * ((sizes[ids[q]] + E - 1) / E);
    }
    for (uint32_t r = 1; r < world; r++) start[r] = start[r - 1] + cnt[r - 1];
    std::vector<uint64_t> base(world, 0);
    for (uint32_t r = 1; r < world; r++) base[r] = base[r - 1] + words[r - 1];
    std::vector<uint32_t> fill(start);
    std::vector<uint64_t> wfill(base);
    for (uint32_t q = 0; q < nq; q++) {
        const uint32_t r = (uint32_t)dest[q];
        order[fill[r]++] = q;
        if (gathered_off) {
            gathered_off[q] = wfill[r];
            wfill[r] += per_pt * ((sizes[ids[q]] + E - 1) / E);
        }
    }
    if (gathered_off) gathered_off[nq] = base[world - 1] + words[world - 1];
    for (uint32_t r = 0; r < world; r++) {
        counts[r] = cnt[r];
        resp_words[r] = words[r];
    }
    return WALLY_OK;
}

extern "C" int wally_route_plan(uint32_t nq, const uint32_t *ids, uint32_t total_clusters, const uint32_t *sizes,
                                const int32_t *owner, uint32_t n, uint32_t d, uint32_t resp_format, uint32_t world,
                                uint32_t *counts, uint32_t *order, uint64_t *resp_words, uint64_t *gathered_off) {
    WALLY_NVTX("wally_route_plan");
    if ((nq && (!ids || !order)) || !sizes || !counts || !resp_words || total_clusters == 0 || world == 0 ||
        n == 0 || d == 0 || d > n || !valid_resp_format(resp_format))
        return fail(nullptr, WALLY_E_ARG, "route_plan: bad arguments");
    for (uint32_t c = 0; c < total_clusters; c++) {
        if (sizes[c] == 0) return fail(nullptr, WALLY_E_ARG, "route_plan: cluster %u is empty", c);
        if (owner && (owner[c] < 0 || (uint32_t)owner[c] >= world))
            return fail(nullptr, WALLY_E_ARG, "route_plan: owner[%u] = %d not in [0, %u)", c, owner[c], world);
    }
    for (uint32_t q = 0; q < nq; q++)
        if (ids[q] >= total_clusters)
            return fail(nullptr, WALLY_E_UNKNOWN_CLUSTER, "route_plan: query %u names cluster %u >= %u", q, ids[q],
                        total_clusters);
    std::vector<int32_t> dest(nq);
    for (uint32_t q = 0; q < nq; q++) dest[q] = owner ? owner[ids[q]] : 0;
    return route_plan_dest(nq, ids, total_clusters, sizes, dest.data(), n, d, resp_format, world, counts, order,
                           resp_words, gathered_off);
}

extern "C" int wally_assign_owners_replicated(uint32_t total_clusters, const double *weight, uint32_t world,
                                              uint64_t *mask) {
    WALLY_NVTX("wally_assign_owners_replicated");
    if (!weight || !mask || total_clusters == 0 || world == 0 || world > 64)
        return fail(nullptr, WALLY_E_ARG, "assign_owners_replicated: bad arguments (world 1..64)");
    double W = 0.0;
    for (uint32_t c = 0; c < total_clusters; c++) {
        if (!(weight[c] >= 0.0)) return fail(nullptr, WALLY_E_ARG, "assign_owners_replicated: weight[%u] < 0", c);
        W += weight[c];
    }
    struct Piece { double w; uint32_t c; };
    std::vector<Piece> pieces;
    pieces.reserve(total_clusters);
    const double target = W / world;
    for (uint32_t c = 0; c < total_clusters; c++) {
        uint32_t r = 1;
        if (target > 0.0 && weight[c] > target) r = (uint32_t)std::min<double>(world, std::ceil(weight[c] / target));
        for (uint32_t i = 0; i < r; i++) pieces.push_back({weight[c] / r, c});
    }
    std::stable_sort(pieces.begin(), pieces.end(), [](const Piece &a, const Piece &b) { return a.w > b.w; });
    std::vector<double> load(world, 0.0);
    for (uint32_t c = 0; c < total_clusters; c++) mask[c] = 0;
    for (const Piece &p : pieces) {
        int best = -1;
        for (uint32_t r = 0; r < world; r++) {
            if ((mask[p.c] >> r) & 1ull) continue;
            if (best < 0 || load[r] < load[(uint32_t)best]) best = (int)r;
        }
        mask[p.c] |= 1ull << best;
        load[(uint32_t)best] += p.w;
    }
    return WALLY_OK;
}

extern "C" int wally_route_plan_replicated(uint32_t nq, const uint32_t *ids, uint32_t total_clusters,
                                           const uint32_t *sizes, const uint64_t *mask, uint32_t n, uint32_t d,
                                           uint32_t resp_format, uint32_t world, uint32_t *counts, uint32_t *order,
                                           uint64_t *resp_words, uint64_t *gathered_off) {
    WALLY_NVTX("wally_route_plan_replicated");
    if (!mask || world == 0 || world > 64 || (nq && (!ids || !order)) || !sizes || !counts || !resp_words ||
        total_clusters == 0 || n == 0 || d == 0 || d > n || !valid_resp_format(resp_format))
        return fail(nullptr, WALLY_E_ARG, "route_plan_replicated: bad arguments (world 1..64)");
    for (uint32_t c = 0; c < total_clusters; c++)
        if (sizes[c] == 0) return fail(nullptr, WALLY_E_ARG, "route_plan_replicated: cluster %u is empty", c);
    for (uint32_t c = 0; c < total_clusters; c++)
        if (mask[c] == 0 || (world < 64 && (mask[c] >> world)))
            return fail(nullptr, WALLY_E_ARG, "route_plan_replicated: mask[%u] empty or names a rank >= %u", c, world);
    for (uint32_t q = 0; q < nq; q++)
        if (ids && ids[q] >= total_clusters)
            return fail(nullptr, WALLY_E_UNKNOWN_CLUSTER, "route_plan: query %u names cluster %u >= %u", q, ids[q],
                        total_clusters);
    // destination of every query: the (j mod r_c)-th replica of its cluster
    std::vector<int32_t> dest(nq);
    std::vector<uint32_t> seen(total_clusters, 0);
    for (uint32_t q = 0; q < nq && ids; q++) {
        const uint32_t c = ids[q];
        const uint64_t m = mask[c];
        const uint32_t r = (uint32_t)__builtin_popcountll(m);
        uint32_t pick = seen[c]++ % r;
        uint64_t mm = m;
        while (pick--) mm &= mm - 1;
        dest[q] = __builtin_ctzll(mm);
    }
    return route_plan_dest(nq, ids, total_clusters, sizes, dest.data(), n, d, resp_format, world, counts, order,
                           resp_words, gathered_off);
}

extern "C" int wally_pack_queries(wally_ctx *c, uint32_t count, const uint32_t *index_dev, const uint32_t *query_dev,
                                  uint32_t *out_dev, void *stream) {
    WALLY_NVTX("wally_pack_queries");
    if (!c) return WALLY_E_ARG;
    if (count == 0) return WALLY_OK;
    if (!index_dev || !query_dev || !out_dev) return fail(c, WALLY_E_ARG, "pack_queries: null pointer");
    if ((uintptr_t)query_dev % 16 || (uintptr_t)out_dev % 16)
        return fail(c, WALLY_E_ARG, "pack_queries: query and out must be 16-byte aligned");
    cudaSetDevice(c->device);
    const uint32_t row_words = 2u * c->p.num_limbs * c->p.n;
    CUDA_OK(c, launch_pack_rows(index_dev, query_dev, out_dev, count, row_words, (cudaStream_t)stream, &c->launches));
    return WALLY_OK;
}

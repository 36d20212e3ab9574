/*
 * wally.h -- C ABI of the B200-native Wally server hot path.
 *
 * The operation (arXiv 2406.06761, PAPER.md; citation "P:Lnnn" = PAPER.md line):
 *   The server holds a public database of d-dimensional integer embeddings
 *   split into clusters (Alg 1 "ServerInit" P:L664-687).
 *   Each query is an RLWE/BFV ciphertext (c0, c1) over R_Q = Z_Q[X]/(X^n+1),
 *   Q = q_0 q_1 ... q_{L-1} in RNS form, tagged with
 *   a cluster id.  For every query the server computes, under encryption,
 *   the dot product of the query with every entry of its cluster and returns
 *   the encrypted scores (Alg 4 "ServerComputation" P:L794-808).
 *
 *   This library computes that result with coefficient packing (BASELINE.json
 *   north_star; DESIGN.md "Readings" S1): plaintext k of cluster c is
 *     p_k(X) = sum_{j<E} sum_{i<d} e_{kE+j}[i] X^{j d + d - 1 - i},  E = floor(n/d),
 *   and for every (query, plaintext) pair the response is
 *     c'_b = round( (c_b * p_k mod (X^n+1, Q)) * q_0 / Q ) mod q_0,   b in {0, 1},
 *   the modulus switch to the smallest limb q_0.
 *   Decrypting c'_0 + c'_1 s mod q_0 and scaling by t/q_0 gives, at coefficient
 *   j*d + d - 1, the dot product <query, e_{kE+j}> mod t.
 *
 * Conventions shared by every call:
 *   - All integers little-endian.  Residues are uint32, canonical in [0, q_i).
 *   - A polynomial with L limbs is stored limb-major: [L][n].
 *   - Query ciphertexts: uint32 [nq][2][L][n] in coefficient form, component 0
 *     is c0, component 1 is c1 (input-query order).
 *   - Responses: for query q (input order), P(c_q) ciphertexts in plaintext
 *     order, each in the context's response format (uint32 [2][n] mod q_0, or
 *     the compact form below).  Query q's first word is at offsets[q] as
 *     returned by wally_response_layout (reading S12).
 *   - "dev" pointers are CUDA device pointers on the context's device; "host"
 *     pointers are CPU memory.  The caller owns every buffer it passes; the
 *     library never frees them.  Device buffers the library needs beyond its
 *     small internal tables (the plaintext store, the per-batch workspace and
 *     the response buffer) are allocated by the caller (from PyTorch in the
 *     Python binding) with the sizes the *_bytes queries return.
 *   - "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls taking a stream are stream-ordered and return before the device
 *     work finishes; inputs must stay valid until it has.
 *   - Every call validates all of its arguments before launching anything and
 *     does nothing on error.  Errors are returned as a negative wally_status;
 *     wally_last_error() gives a detail string.  Nothing aborts.
 *   - A context is bound to one device and is not thread-safe.
 */
#ifndef WALLY_H
#define WALLY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WALLY_MAX_LIMBS 4

typedef enum {
    WALLY_OK = 0,
    WALLY_E_ARG = -1,             /* null pointer, size mismatch, bad range */
    WALLY_E_PARAMS = -2,          /* unsupported n / L / d, moduli not NTT-friendly primes */
    WALLY_E_UNKNOWN_CLUSTER = -3, /* cluster id >= total clusters or not owned by this context */
    WALLY_E_RESIDUE = -4,         /* an input residue >= q_i (reported by wally_check_batch) */
    WALLY_E_STATE = -5,           /* call order: e.g. eval before encode */
    WALLY_E_CUDA = -6,            /* a CUDA runtime call failed */
    WALLY_E_NCCL = -7,            /* NCCL unavailable, or an NCCL call / communicator failed */
    WALLY_E_OOM = -8              /* internal table allocation failed */
} wally_status;

typedef struct wally_ctx wally_ctx;

/* Response formats (per (query, plaintext) pair, all words mod q_0):
 *   WALLY_RESP_FULL     [2][n]: c0' and c1' in full (2n words).
 *   WALLY_RESP_COMPACT  c0' only at the E result coefficients j*d + d - 1
 *                       (j < E = floor(n/d)), padded with zeros to
 *                       E4 = 4*ceil(E/4) words, followed by c1' [n]
 *                       (E4 + n words).  Decrypting result coefficient k needs
 *                       c0'[k] and all of c1' (c0' + c1' s), so this
 *                       carries the same plaintext information in about half
 *                       the bytes -- the response compression of P:L1003-1007 /
 *                       P:L1035 ("sparse c0"). */
#define WALLY_RESP_FULL 0u
#define WALLY_RESP_COMPACT 1u
/*   WALLY_RESP_COMPACT_DROP  (n = 4096 only) as WALLY_RESP_COMPACT, and c1'
 *                       additionally has its 6 least significant bits dropped
 *                       ("Dropping ciphertext LSBs"; reading S20:
 *                       rounded, h = floor((c1' + 32) / 64) < 2^24 because
 *                       q_0 < 2^30 - 31), stored as two planes: the low 16 bits
 *                       of h as uint16 [n], then the high 8 bits as uint8 [n],
 *                       both in the 16 x 256 transposed order -- coefficient i
 *                       at position (i mod 256) * 16 + floor(i / 256) -- which
 *                       is the order the kernel holds them in (E4 + 3n/4 words).
 *                       The client decrypts with c1' ~ 64 h mod q_0; the dropped
 *                       part adds e_drop = -(c1' - 64 h) * s with |c1' - 64 h| <= 32,
 *                       which keeps ||e + e_drop|| < q_0 / 2t for q_0 ~ 2^30,
 *                       t <= 65537 at n = 4096.
 *                       wally_create accepts this format only when the paper's
 *                       z = 8 rule holds for it: 8 sqrt(2n/9) 2^5 < q_0 / 2t
 *                       (reading S20; WALLY_E_PARAMS otherwise). */
#define WALLY_RESP_COMPACT_DROP 2u
#define WALLY_RESP_DROP_BITS 6u

/* Scheme parameters.
 *   n          ring degree, a power of two in {1024, 2048, 4096, 8192}
 *   num_limbs  L in [1, 4]
 *   t          plaintext modulus (only used for documentation / validation: t >= 2)
 *   d          embedding dimension, 1 <= d <= n  (d need not divide n)
 *   moduli     q_0 < q_1 < ... < q_{L-1}: distinct primes < 2^30, each = 1 mod 2n,
 *              with q_{L-1} < 2 q_0 ("q_i = 1 mod 2n"; readings S5, S6).
 *   resp_format WALLY_RESP_FULL, WALLY_RESP_COMPACT or WALLY_RESP_COMPACT_DROP (see above). */
typedef struct {
    uint32_t n;
    uint32_t num_limbs;
    uint32_t t;
    uint32_t d;
    uint32_t moduli[WALLY_MAX_LIMBS];
    uint32_t resp_format;
} wally_params;

/* The L largest primes q < 2^30 with q = 1 (mod 2n), written ascending into
 * moduli_out[0..L-1] (reading S5).  Pure host computation. */
int wally_find_moduli(uint32_t n, uint32_t num_limbs, uint32_t *moduli_out);

/* Create a context on CUDA device `device`: validates params, builds the
 * NTT twiddle tables and modulus-switch constants and uploads them.
 * One context is one server (one rank) of the paper's setting: it holds the
 * scheme of P:L244-251 (R_Q = Z_Q[X]/(X^n+1), plaintext modulus t) in the RNS
 * form of P:L1310-1317 with NTT-friendly limbs q_i = 1 mod 2n, and
 * the modulus-switch target q_0 of P:L1003 / P:L1323 ("Q' = q_0").
 *   params   read only during the call (the context keeps a copy)
 *   ctx_out  receives the context; the caller releases it with wally_destroy
 * Errors: WALLY_E_PARAMS (unsupported n, L, d, t or moduli), WALLY_E_CUDA (no
 * such device), WALLY_E_OOM; *ctx_out is NULL on error and the detail is in
 * wally_last_error(NULL). */
int wally_create(const wally_params *params, int device, wally_ctx **ctx_out);
void wally_destroy(wally_ctx *ctx);
/* Detail of the last error on ctx (or of the last failed wally_create when ctx is NULL). */
const char *wally_last_error(const wally_ctx *ctx);

/* ServerInit, part 1 (Alg 1): the cluster layout.
 *   total_clusters      number of clusters in the whole database (all ranks)
 *   cluster_sizes_host  uint32 [total_clusters]: entries in each cluster (>= 1)
 *   owner_host          int32 [total_clusters]: owning rank of each cluster, or NULL
 *                       meaning "every cluster is local" (reading: cluster-sharded
 *                       data parallelism)
 *   rank                this context's rank (ignored when owner_host is NULL)
 * Local clusters are the ones with owner == rank, taken in ascending id order.
 * Plaintexts per cluster: P_c = ceil(size_c / E), E = floor(n/d). */
int wally_load_clusters(wally_ctx *ctx, uint32_t total_clusters, const uint32_t *cluster_sizes_host,
                        const int32_t *owner_host, int32_t rank);

/* Bytes of the device plaintext store for the local clusters:
 * n <= 4096: sum_c P_c * L * 2 * n * 4 (NTT-domain values plus Shoup
 * companions); n = 8192: sum_c P'_c * L * n * 4 with P'_c = P_c rounded up to
 * even (the values in Montgomery form, plaintexts stored in pairs). */
int wally_plaintext_store_bytes(const wally_ctx *ctx, size_t *bytes_out);
/* Number of local entries (rows of the entries array wally_encode_plaintexts_ntt reads). */
int wally_local_entry_count(const wally_ctx *ctx, uint64_t *count_out);

/* ServerInit, part 2: pack every local plaintext (entries reversed at offsets
 * j*d, reading S1), lift each signed entry x to x mod q_i (S8), forward-NTT
 * per limb and keep the result, with its Shoup companion (n <= 4096) or in
 * Montgomery form (n = 8192), in store_dev.
 *   entries_dev  int8 [local_entry_count][d] row-major, local clusters in
 *                ascending cluster-id order, each cluster's entries contiguous
 *   store_dev    device buffer of wally_plaintext_store_bytes bytes; the
 *                context keeps using it until the next encode or destroy. */
int wally_encode_plaintexts_ntt(wally_ctx *ctx, const int8_t *entries_dev, void *store_dev, size_t store_bytes,
                                void *stream);

/* Response words per (query, plaintext) pair for the context's format:
 * 2n (full), E4 + n (compact) or E4 + 3n/4 (compact with dropped LSBs). */
int wally_response_words_per_plaintext(const wally_ctx *ctx, uint64_t *words_out);

/* Algorithmic modular multiplications per (query, plaintext) pair of the
 * fused kernel this context runs: 2 [L n + L (n/2) log2 n + n L(L-1)/2]
 * (SURVEY.md §8(d) M_pair), or, for compact responses with 16 | d at
 * n = 4096, that count with c0's inverse NTT and modulus switch pruned to
 * the result coefficients.  Used for the
 * roofline; pure host computation. */
int wally_modmuls_per_pair(const wally_ctx *ctx, uint64_t *modmuls_out);

/* Response layout of a batch (reading S12).
 *   cluster_of_query_host  uint32 [nq]
 *   offsets_host           uint64 [nq + 1] out: word offset of query q's responses;
 *                          offsets[nq] = total words.  May be NULL.
 *   total_words_out        total response words (may be NULL).
 * Fails with WALLY_E_UNKNOWN_CLUSTER if a query names a cluster that is not local. */
int wally_response_layout(const wally_ctx *ctx, uint32_t nq, const uint32_t *cluster_of_query_host,
                          uint64_t *offsets_host, uint64_t *total_words_out);

/* Bytes of device workspace wally_eval_batch needs for nq queries. */
int wally_workspace_bytes(const wally_ctx *ctx, uint32_t nq, size_t *bytes_out);

/* ServerComputation for a batch (Alg 4 P:L794-808 analog):
 *   1. batcher kernels group the queries by cluster id (histogram, scan,
 *      scatter) and build the (cluster, plaintext, query-chunk) work list;
 *   2. forward negacyclic NTT of all 2*L*nq query polynomials;
 *   3. one fused kernel per work item: pointwise Shoup modmul with each
 *      NTT-domain plaintext, inverse NTT, RNS modulus switch to q_0, and the
 *      write of the single-limb response ciphertext.
 *   cluster_of_query_host  uint32 [nq] (host; validated before any launch)
 *   query_ct_dev           uint32 [nq][2][L][n] canonical residues (device)
 *   responses_dev          uint32 [responses_words] (device), layout of wally_response_layout
 *   workspace_dev          wally_workspace_bytes(nq) bytes (device)
 * Residues >= q_i are detected on the device and reported by wally_check_batch. */
int wally_eval_batch(wally_ctx *ctx, uint32_t nq, const uint32_t *cluster_of_query_host,
                     const uint32_t *query_ct_dev, uint32_t *responses_dev, uint64_t responses_words,
                     void *workspace_dev, size_t workspace_bytes, void *stream);

/* Synchronizes `stream` and reports device-side errors of the last batch run on
 * this workspace: WALLY_E_RESIDUE if any query residue was >= its modulus. */
int wally_check_batch(wally_ctx *ctx, const void *workspace_dev, void *stream);

/* Copy responses device -> host (stream-ordered, then synchronizes the stream):
 * the return of the encrypted scores R to the client, Alg 4
 * ("return r = (R, metadata)"; metadata is out of scope).
 *   responses_dev  uint32 [words] (device);  out_host  uint32 [words] (host, pinned or pageable)
 * The caller owns both buffers.  Errors: WALLY_E_ARG (null pointer with
 * words > 0), WALLY_E_CUDA (copy failed). */
int wally_fetch_responses(wally_ctx *ctx, const uint32_t *responses_dev, uint64_t words, uint32_t *out_host,
                          void *stream);

/* End-to-end call with HOST buffers (the serving path): the batch is split
 * into sub-batches of at most sub_batch queries; each sub-batch's query
 * ciphertexts are copied host->device, evaluated, and its responses copied
 * device->host into responses_host, with copies and compute of consecutive
 * sub-batches overlapped on two streams.  Synchronizes before returning.
 *   query_ct_host   uint32 [nq][2][L][n] (pinned for full copy bandwidth)
 *   responses_host  uint32 [responses_words], layout of wally_response_layout
 *   workspace_dev   wally_host_workspace_bytes(sub_batch) bytes (device)
 * Unlike wally_eval_batch, the device-side residue check is collected here:
 * after the final synchronisation the call returns WALLY_E_RESIDUE if any
 * query residue of any sub-batch was >= its modulus (the responses of such a
 * batch are meaningless). */
int wally_host_workspace_bytes(const wally_ctx *ctx, uint32_t sub_batch, size_t *bytes_out);
int wally_eval_batch_host(wally_ctx *ctx, uint32_t nq, const uint32_t *cluster_of_query_host,
                          const uint32_t *query_ct_host, uint32_t *responses_host, uint64_t responses_words,
                          uint32_t sub_batch, void *workspace_dev, size_t workspace_bytes, void *stream);

/* Multi-GPU routing: destination rank of every query
 * from the owner map given to wally_load_clusters (rank of the owning
 * context).  dest_rank_host int32 [nq] out. */
int wally_route_queries(const wally_ctx *ctx, uint32_t nq, const uint32_t *cluster_of_query_host,
                        int32_t *dest_rank_host);

/* Cluster ownership for cluster-sharded data parallelism (DESIGN.md
 * "Multi-GPU"): greedy longest-processing-time assignment.  Clusters are
 * taken in descending weight_host order (ties: ascending id) and each goes
 * to the rank with the least total weight so far (ties: lowest rank).  The
 * weight of a cluster is the caller's expected work for it, e.g. expected
 * queries x P_c.  Pure host computation.
 *   weight_host  double [total_clusters], each >= 0
 *   owner_out    int32 [total_clusters] out: rank in [0, world) */
int wally_assign_owners(uint32_t total_clusters, const double *weight_host, uint32_t world, int32_t *owner_out);

/* Routing plan of one batch arriving at an ingress rank (north_star: queries
 * are routed to the rank owning their cluster; Alg 4's per-query work is
 * independent, so a query's responses are produced entirely on its owner).
 * Pure host computation, identical on every rank for the same inputs.
 *   cluster_of_query_host  uint32 [nq]
 *   cluster_sizes_host     uint32 [total_clusters] (entries per cluster, >= 1)
 *   owner_host             int32 [total_clusters] (rank of each cluster; NULL = all on rank 0)
 *   n, d                   ring degree and dimension (P_c = ceil(size_c / floor(n/d)))
 *   resp_format            WALLY_RESP_* (response words per plaintext)
 * Outputs (caller-allocated):
 *   counts_out        uint32 [world]: queries routed to each rank
 *   order_out         uint32 [nq]: input indices grouped by destination rank
 *                     (ascending rank, input order within a rank) -- the scatter's send
 *                     order; rank r's share is order_out[sum_{s<r} counts .. +counts[r]]
 *   resp_words_out    uint64 [world]: response words rank r produces for its share
 *   gathered_off_out  uint64 [nq + 1] or NULL: word offset of query q's responses
 *                     when the ranks' response buffers are concatenated in rank order
 *                     (each rank's buffer in its local query order); [nq] = total words.
 * Errors: WALLY_E_UNKNOWN_CLUSTER (id >= total_clusters), WALLY_E_ARG (owner not
 * in [0, world), bad sizes); nothing is written on error. */
int wally_route_plan(uint32_t nq, const uint32_t *cluster_of_query_host, uint32_t total_clusters,
                     const uint32_t *cluster_sizes_host, const int32_t *owner_host, uint32_t n, uint32_t d,
                     uint32_t resp_format, uint32_t world, uint32_t *counts_out, uint32_t *order_out, uint64_t *resp_words_out,
                     uint64_t *gathered_off_out);

/* Hot-cluster replication (the Zipf skew of configs[4]
 * puts 15% of all queries on one cluster, so disjoint ownership caps the
 * 8-rank speedup near 6.6x).  A cluster whose weight exceeds the mean rank
 * load W/world is split into r = ceil(weight * world / W) equal pieces
 * (r <= world) placed on r distinct ranks; all pieces are then assigned by
 * greedy LPT as in wally_assign_owners (descending piece weight, ties by
 * ascending cluster id; least-loaded rank that does not yet hold the
 * cluster, ties lowest rank).  Pure host computation.
 *   weight_host     double [total_clusters] >= 0
 *   world           1..64
 *   owner_mask_out  uint64 [total_clusters] out: bit r set = rank r holds a replica */
int wally_assign_owners_replicated(uint32_t total_clusters, const double *weight_host, uint32_t world,
                                   uint64_t *owner_mask_out);

/* wally_route_plan for replicated ownership: the j-th query (input order)
 * naming cluster c goes to the (j mod r_c)-th lowest rank in owner_mask[c]
 * (r_c = replicas of c).  Outputs as wally_route_plan.  Errors also when a
 * mask is empty or names a rank >= world. */
int wally_route_plan_replicated(uint32_t nq, const uint32_t *cluster_of_query_host, uint32_t total_clusters,
                                const uint32_t *cluster_sizes_host, const uint64_t *owner_mask_host, uint32_t n,
                                uint32_t d, uint32_t resp_format, uint32_t world, uint32_t *counts_out,
                                uint32_t *order_out, uint64_t *resp_words_out, uint64_t *gathered_off_out);

/* wally_load_clusters with replicated ownership: cluster c is local to this
 * context iff bit `rank` of owner_mask_host[c] is set (rank in [0, 64)). */
int wally_load_clusters_replicated(wally_ctx *ctx, uint32_t total_clusters, const uint32_t *cluster_sizes_host,
                                   const uint64_t *owner_mask_host, int32_t rank);

/* Scatter-side packing on the ingress rank: out_dev[i] = query_ct_dev[index_dev[i]]
 * for i < count, rows of 2*L*n uint32 (one query ciphertext).  Stream-ordered.
 *   index_dev     uint32 [count] (device), each < nq
 *   query_ct_dev  uint32 [nq][2][L][n] (device, 16-byte aligned)
 *   out_dev       uint32 [count][2][L][n] (device, 16-byte aligned) */
int wally_pack_queries(wally_ctx *ctx, uint32_t count, const uint32_t *index_dev, const uint32_t *query_ct_dev,
                       uint32_t *out_dev, void *stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU data plane (north_star: "Clusters are partitioned across the 8
 * GPUs of one B200 box ... queries are routed to the owning rank, with NCCL
 * over NVLink only for query scatter and response gather"; the server
 * "distributes them according to the correct clusters").  One
 * context per rank (one process per GPU).  Alg 4's work is independent per
 * query, so the scatter and the optional gather are the only
 * exchange steps.  NCCL is loaded at run time (libnccl.so.2, the copy torch
 * uses when it is loaded); the single-rank path never needs it.
 * ------------------------------------------------------------------------- */
#define WALLY_COMM_ID_BYTES 128

/* An NCCL unique id (128 bytes) for a new communicator.  Called on one rank
 * (the ingress); the caller hands the bytes to every rank (e.g. a
 * torch.distributed broadcast).  Errors: WALLY_E_NCCL. */
int wally_comm_unique_id(uint8_t *id_out);

/* Join the communicator `id` as `rank` of `world` on the context's device
 * (collective: every rank calls it).  Replaces an earlier communicator.
 * Errors: WALLY_E_ARG, WALLY_E_NCCL. */
int wally_comm_init(wally_ctx *ctx, int32_t rank, int32_t world, const uint8_t *id);

/* WALLY_E_NCCL if the communicator saw an asynchronous error (a failed peer
 * or transport), WALLY_E_STATE without a communicator. */
int wally_comm_check(wally_ctx *ctx);

/* Query scatter (collective over the communicator; stream-ordered).  Every
 * rank passes the same counts_host, the per-rank query counts of
 * wally_route_plan.  On the source rank `src` (the ingress):
 *   order_dev     uint32 [nq] (device): wally_route_plan's order_out, nq = sum(counts)
 *   query_ct_dev  uint32 [nq][2][L][n] (device, 16-byte aligned): the batch in input order
 *   pack_dev      uint32 [nq][2][L][n] (device scratch, 16-byte aligned): the shares,
 *                 packed contiguously in rank order (kernel pack_rows), from which
 *                 rank r's block is sent with ncclSend
 * On every rank (src included):
 *   share_dev     uint32 [counts[rank]][2][L][n] (device) out: this rank's
 *                 queries in its local order (wally_route_plan's order within the rank).
 * Other ranks pass NULL for order/query/pack.  Errors: WALLY_E_STATE (no
 * communicator), WALLY_E_ARG, WALLY_E_CUDA, WALLY_E_NCCL. */
int wally_scatter_queries(wally_ctx *ctx, int32_t src, const uint32_t *counts_host, const uint32_t *order_dev,
                          const uint32_t *query_ct_dev, uint32_t *pack_dev, uint32_t *share_dev, void *stream);

/* Response gather to rank `dst` (collective; stream-ordered): the ranks'
 * response buffers concatenated in rank order, the layout of
 * wally_route_plan's gathered_off (query q's responses start there).
 *   resp_words_host  uint64 [world]: wally_route_plan's resp_words_out (same on every rank)
 *   resp_dev         this rank's responses, resp_words_host[rank] words (device)
 *   gathered_dev     dst only: sum(resp_words_host) words (device); NULL elsewhere
 * Errors: as wally_scatter_queries. */
int wally_gather_responses(wally_ctx *ctx, int32_t dst, const uint64_t *resp_words_host, const uint32_t *resp_dev,
                           uint32_t *gathered_dev, void *stream);

/* Test hooks on the same device code as the hot path.
 * Forward NTT (the kernel of step 2): in_dev uint32 [count][L][n] canonical
 * coefficient form -> out_dev uint32 [count][L][n] NTT domain (internal,
 * bit-reversed order, residues in [0, 4 q_i)).
 * Inverse NTT: out = n^{-1} * INTT(in), canonical coefficient form; in may be
 * any residues < 2^32 congruent to the NTT values. */
int wally_ntt_forward(wally_ctx *ctx, const uint32_t *in_dev, uint32_t *out_dev, uint32_t count, void *stream);
int wally_ntt_inverse(wally_ctx *ctx, const uint32_t *in_dev, uint32_t *out_dev, uint32_t count, void *stream);

/* Count of this library's kernel launches since create (for bench evidence). */
uint64_t wally_kernel_launches(const wally_ctx *ctx);

/* Per-stage device timing of wally_eval_batch (CUDA events recorded on the
 * batch's stream around each stage when enabled; off by default).
 * wally_stage_times synchronizes the recorded events and returns the summed
 * milliseconds since the last call: ms_out[0] batcher kernels, ms_out[1]
 * forward NTT, ms_out[2] fused modmul/iNTT/mod-switch kernel; batches_out =
 * number of batches summed.  Clears the record. */
int wally_enable_stage_timing(wally_ctx *ctx, int enable);
int wally_stage_times(wally_ctx *ctx, double *ms_out, uint64_t *batches_out);

#ifdef __cplusplus
}
#endif

#endif /* WALLY_H */

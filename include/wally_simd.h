/*
 * wally_simd.h -- C ABI of the SIMD formulation of Wally's server computation
 * (the paper's own algorithm, Alg 4
 * P:L794-808), beside the coefficient-packed path of wally.h.
 *
 *   a0' ServerInit  every cluster is cut into blocks of up to 2 R d
 *                   embeddings (R slices of d x d per slot row, reading S23);
 *                   a block is d plaintexts: its diagonals
 *                   p_i = [e_0^i, e_1^{i+1}, ...], pre-rotated for
 *                   baby-step giant-step, slot-encoded mod t (BFV batching,
 *                   reading S22), lifted centered to R_Q (S24), NTT'd.
 *   a2'  queries    ct (coefficient form over Q) and two rotation keys
 *                   (sigma_5 = rotate by one, sigma_{5^g} = rotate by g;
 *                   P:L1356-1358 "two rotation keys") per query, NTT'd.
 *   a3'-a4' BSGS    baby_b = rot_1^b(ct), b < g;  I_j = sum_b pt_{jg+b} (.) baby_b;
 *                   acc = I_{m-1}, acc = rot_g(acc) + I_j (j = m-2 .. 0);
 *                   every rotation = Galois automorphism + hybrid key switch
 *                   with one special prime P.
 *   a5'-a6' reply   acc switched to q_0: one
 *                   ciphertext [2][n] mod q_0 per (query, block) -- the
 *                   paper's ceil(N'/n) response ciphertexts.
 *
 * Decrypting a response and decoding its slots gives, at slot (row r,
 * column u d + c) for u < R, c < d, the dot product of the query with
 * embedding (r R + u) d + c of the block, mod t.
 *
 * Conventions as in wally.h: residues uint32, limb-major then coefficient
 * order; device pointers are CUDA device memory; calls are stream-ordered
 * on the given stream; errors return a negative WALLY_E_* code with a
 * detail string from wally_simd_last_error(); nothing aborts, and a failed
 * call launches nothing.  A context is not thread-safe.
 */
#ifndef WALLY_SIMD_H
#define WALLY_SIMD_H

#include <stddef.h>
#include <stdint.h>

#include "wally.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wally_simd_ctx wally_simd_ctx;

typedef struct {
    uint32_t n;          /* ring degree: 1024, 2048, 4096 or 8192 */
    uint32_t num_limbs;  /* L ciphertext limbs, 1..WALLY_MAX_LIMBS */
    uint32_t t;          /* plaintext modulus: a prime = 1 (mod 2n), < 2^30 (65537 in every config) */
    uint32_t d;          /* embedding dimension, 1 <= d <= n/2 */
    uint32_t baby;       /* g, baby steps: 1 <= g <= d; 0 picks ceil(sqrt(d)) */
    /* L ciphertext moduli ascending (q_0 first), then the special prime P:
     * distinct NTT-friendly primes < 2^30 with P < q_0 (reading S25) */
    uint32_t moduli[WALLY_MAX_LIMBS + 1];
} wally_simd_params;

/* Default moduli (reading S25): the L largest NTT-friendly primes below
 * 2^30 ascending (the coefficient path's limbs), then the next one below
 * them as the special prime P.  moduli_out: [L + 1]. */
int wally_simd_default_moduli(uint32_t n, uint32_t num_limbs, uint32_t *moduli_out);

/* Validates the parameters, builds the NTT tables for the L + 1 moduli and
 * for t, the slot <-> NTT-index map and the two Galois permutations, on
 * `device`.  WALLY_E_PARAMS on unsupported / inconsistent parameters. */
int wally_simd_create(const wally_simd_params *params, int device, wally_simd_ctx **out);
void wally_simd_destroy(wally_simd_ctx *ctx);
const char *wally_simd_last_error(const wally_simd_ctx *ctx);

typedef struct {
    uint32_t row_slices;     /* R: d x d slices per slot row */
    uint32_t block_entries;  /* 2 R d: embeddings per response ciphertext */
    uint32_t baby, giant;    /* g and m = ceil(d / g) */
    uint32_t galois[2];      /* 5 and 5^g mod 2n: the automorphisms of the two keys */
    uint64_t key_words;      /* words of one query's key material: 2 keys x [2][L][L+1][n] */
} wally_simd_info;
int wally_simd_get_info(const wally_simd_ctx *ctx, wally_simd_info *info);

/* ServerInit (a0'): clusters 0..n_clusters-1 with sizes[c] embeddings each,
 * entries int8 [sum sizes][d] row-major, clusters concatenated (host).
 * Builds every block's d plaintexts on the device (kept by the context;
 * 16 L n d bytes per block).  Replaces any earlier database. */
int wally_simd_load_clusters(wally_simd_ctx *ctx, uint32_t n_clusters, const uint32_t *sizes,
                             const int8_t *entries, void *stream);

/* Number of response ciphertexts (blocks) of cluster c; 0 if c is unknown. */
uint32_t wally_simd_blocks(const wally_simd_ctx *ctx, uint32_t cluster);

/* Server computation (a2'-a6') for nq queries:
 *   cluster_ids  host uint32 [nq]
 *   query_ct     device uint32 [nq][2][L][n], coefficient form, residues < q_l
 *   keys         device uint32 [nq][2][2][L][L+1][n], coefficient form:
 *                key k (0: sigma_5, 1: sigma_{5^g}), component (b, a), digit j,
 *                modulus m (m = L: P), residues < moduli[m]
 *   resp         device uint32 [sum_q blocks(c_q)][2][n] mod q_0, queries in
 *                input order, blocks ascending; resp_off (host, [nq+1], may be
 *                NULL) receives the first word of each query.
 * The call allocates its workspace on first use (grown on demand) and
 * processes the batch in chunks.  WALLY_E_UNKNOWN_CLUSTER for an id >= the
 * loaded cluster count, WALLY_E_ARG for a too-small resp_words,
 * WALLY_E_RESIDUE if any input residue is out of range (checked on the
 * device before the result is used; the response is then undefined). */
int wally_simd_eval_batch(wally_simd_ctx *ctx, uint32_t nq, const uint32_t *cluster_ids, const uint32_t *query_ct,
                          const uint32_t *keys, uint32_t *resp, uint64_t resp_words, uint64_t *resp_off,
                          void *stream);

/* The same computation end to end from host memory (the serving call):
 * query_ct, keys and resp are HOST buffers (pinned for overlap) with the
 * layouts above.  The batch runs in sub-batches of `sub_batch` queries
 * through double-buffered device staging: the inputs of sub-batch i+1 are
 * copied in, and the responses of sub-batch i-1 copied out, on two copy
 * streams while sub-batch i computes on `stream`.  Within a sub-batch the
 * queries are evaluated in cluster order.  Returns after the last response
 * has arrived in `resp`.  Errors as wally_simd_eval_batch. */
int wally_simd_eval_batch_host(wally_simd_ctx *ctx, uint32_t nq, const uint32_t *cluster_ids,
                               const uint32_t *query_ct, const uint32_t *keys, uint32_t *resp, uint64_t resp_words,
                               uint64_t *resp_off, uint32_t sub_batch, void *stream);

/* Algorithmic modular multiplications of one query with `blocks` response
 * blocks (the roofline unit): NTT butterflies, pointwise and
 * key-switch products, scalings and the final switch. */
uint64_t wally_simd_modmuls_per_query(const wally_simd_ctx *ctx, uint32_t blocks);

/* Rotation kernels: at n <= 4096 a chunk of at least `min_queries` queries
 * (default: 2 per SM) runs each unit's whole chain of rotations in one CTA
 * (simd_rot_chain_kernel); smaller chunks use the separate ModUp / ModDown
 * kernels, which spread one rotation over L + 2 CTAs.  0 = always the
 * chain, UINT32_MAX = never.  Results are identical either way. */
int wally_simd_set_chain_threshold(wally_simd_ctx *ctx, uint32_t min_queries);

/* Kernel launches issued by this context so far. */
uint64_t wally_simd_launch_count(const wally_simd_ctx *ctx);

/* Per-stage device timing of wally_simd_eval_batch (off by default): CUDA
 * events recorded on the batch's stream at the stage boundaries of every
 * query chunk.  wally_simd_stage_times synchronizes them and returns the
 * summed milliseconds since the last call in ms_out[5]:
 *   [0] a2'  NTT of the query ciphertexts and rotation keys,
 *   [1]      baby-step rotations (g - 1 per query, P:L1352-1361 BSGS),
 *   [2] a3'  diagonal inner products I_j (P:L565 diagonals),
 *   [3]      giant-step rotations (m - 1 per block, Horner),
 *   [4] a5'-a6' inverse NTT and switch to q_0;
 * chunks_out = number of query chunks summed.  Clears the record. */
int wally_simd_enable_stage_timing(wally_simd_ctx *ctx, int enable);
int wally_simd_stage_times(wally_simd_ctx *ctx, double *ms_out, uint64_t *chunks_out);

/* Algorithmic work of the same five stages for a batch of nq queries with
 * cluster ids ids[nq] (host array): modmuls_out[5] modular multiplications
 * (the terms of wally_simd_modmuls_per_query) and bytes_out[5] the HBM bytes
 * each stage must move at least (operands read once, results written once:
 * stage [2] reads the d plaintexts of every distinct block of the batch once,
 * with their Shoup companions, 8 L n d bytes per block, however many of the
 * batch's queries use it).  The roofline of a stage is the larger of
 * modmuls / integer-pipe peak and bytes / HBM peak.
 * Returns WALLY_E_ARG for a null pointer or an unknown cluster id. */
int wally_simd_stage_work(const wally_simd_ctx *ctx, uint32_t nq, const uint32_t *ids, uint64_t *modmuls_out,
                          uint64_t *bytes_out);

#ifdef __cplusplus
}
#endif

#endif /* WALLY_SIMD_H */

/*
 * magicpig.h -- C ABI of the B200 (sm_100a) implementation of MagicPIG's
 * decode-time hot path: LSH importance-sampled decode attention
 * (arXiv 2410.16179).  "P:<line>" cites /root/reference/PAPER.md.
 *
 * The calls follow the paper's problem statement and Algorithm 1
 * (P:98-118): one decode step per (sequence, query head) over a KV cache K, V,
 * with random projectors W, hash tables HT (here: packed SimHash codes) and a
 * static (sink + local) cache.
 *
 * Conventions (all entry points):
 *   - Pointers are DEVICE pointers unless marked [host].  bf16 data is passed
 *     as uint16_t bit patterns.  All work is enqueued on `stream`
 *     (a cudaStream_t; NULL = legacy default stream) and is asynchronous.
 *   - The caller owns every buffer, including the workspace; the library
 *     never allocates or frees device memory.  Its only process-wide state is a
 *     launch counter and the debug decode-kernel selector
 *     (magicpig_debug_set_decode_kernel; default 0 = automatic choice).
 *   - Return value: MAGICPIG_OK (0) or a negative error code (argument and
 *     launch errors).  Errors that can only be detected on the device
 *     (exact-range violations, fixup-list overflow) are OR-ed into a status
 *     word in the workspace; read it with magicpig_workspace_status().
 *   - No exception or C++ type crosses this boundary.
 *
 * Shapes: B sequences, Hkv key/value heads, Hq = G * Hkv query heads (GQA:
 * query head h*G + g uses kv head h), head_dim d = 128, n_local keys per
 * (sequence, kv head) on this device, at global positions
 * [seq_offset, seq_offset + n_local) of a context of n_global keys.
 * KV cache layout: k, v [B][Hkv][n_local][128] bf16, row-major.
 * Queries: q [B][Hq][128] bf16.
 */
#ifndef MAGICPIG_H
#define MAGICPIG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MAGICPIG_OK 0
#define MAGICPIG_EINVAL (-1)      /* bad shape / range / NULL pointer */
#define MAGICPIG_ENOTREPR (-2)    /* (status) a W value is not bf16-representable */
#define MAGICPIG_EDEGENERATE (-3) /* (status) a head had S and T both empty */
#define MAGICPIG_ECUDA (-4)       /* a CUDA launch/API call failed */
#define MAGICPIG_EWORKSPACE (-5)  /* workspace too small */
#define MAGICPIG_EINEXACT (-6)    /* (status) |k| or |x| >= 2^27, or an exact dot left the exact range */
#define MAGICPIG_EOVERFLOW (-7)   /* (status) hash fixup list overflowed */

/* Status bits OR-ed into the workspace status word by device code. */
#define MAGICPIG_STATUS_INEXACT 1u
#define MAGICPIG_STATUS_OVERFLOW 2u
#define MAGICPIG_STATUS_DEGENERATE 4u
#define MAGICPIG_STATUS_NOTREPR 8u

/* LSH configuration ("K=9 or 10, L is a few hundred").
 *   K               bits per table, 1..16 (codes are exported as uint16)
 *   L               number of tables, >= min_collisions, <= 1024
 *   head_dim        must be 128
 *   center          1: keys centered before hashing
 *   mips            1: MIPS transform kbar = [k, sqrt(r^2-|k|^2)]
 *   min_collisions  2 = the paper's rule (P:84 footnote); 1 = classic SimHash
 *   sink, local     static tokens never sampled (4 and 64 at P:619)  */
typedef struct magicpig_config {
    int32_t K;
    int32_t L;
    int32_t head_dim;
    int32_t center;
    int32_t mips;
    int32_t min_collisions;
    int32_t sink;
    int32_t local;
} magicpig_config;

/* Returns MAGICPIG_OK if the configuration is supported. [host] */
int magicpig_validate_config(const magicpig_config* cfg);

/* Number of uint32 words of the packed code array for (B, Hkv, n_local). [host]
 * Layout ("bit planes"): codes[B][Hkv][ceil(n/1024)][KLq][32][4] where KLq is
 * the number of 4-column groups after padding L to whole table groups; word
 * (.., c, jq, l, w) bit r = SimHash bit of projection column 4*jq + w for key
 * 1024*c + 32*l + r.  Column j belongs to table j / K, bit j % K (R7). */
size_t magicpig_codes_words(const magicpig_config* cfg, int64_t B, int64_t Hkv, int64_t n_local);

/* Workspace sizes in bytes. [host]  Workspaces must be 256-byte aligned and
 * zero-filled once after allocation (magicpig_workspace_init); the library
 * leaves them reusable (self-cleaning) after every call. */
size_t magicpig_build_workspace_bytes(const magicpig_config* cfg, int64_t B, int64_t Hkv, int64_t n_local);
size_t magicpig_decode_workspace_bytes(const magicpig_config* cfg, int64_t B, int64_t Hq, int64_t Hkv,
                                       int64_t n_local);
int magicpig_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* Reads and clears the device status word of a workspace (synchronises
 * `stream`).  *status [host] receives the MAGICPIG_STATUS_* bits. */
int magicpig_workspace_status(void* ws, uint32_t* status, void* stream);

/* ---------------------------------------------------------------- build ---
 * Build = three phases so that collectives stay with the caller (sequence
 * sharding).  Unsharded callers use magicpig_build_index, which runs all
 * three.  Fixed-point integers ("q64") are int128 values in units of 2^-64
 * stored as (lo uint64, hi int64) pairs (reading R2b in DESIGN.md).
 *
 * Phase 1, centering statistics:
 *   key_sum[B][Hkv][128][2]  q64 sum over this shard's dynamic keys D of
 *                            trunc(k * 2^64)   (exact, order independent)
 *   count[B][Hkv]            number of dynamic keys on this shard
 * Sharded: sum key_sum/count over shards (magicpig_reduce_stats).          */
int magicpig_key_stats(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv,
                       int64_t n_local, int64_t seq_offset, int64_t n_global, int64_t* key_sum,
                       int64_t* count, void* ws, size_t ws_bytes, void* stream);

/* Phase 2, centering vector and MIPS radius:
 *   center[B][Hkv][128]  c = fl32(fl64(fl64(key_sum 2^-64) / count)), or 0
 *                        when cfg->center == 0 or count == 0
 *   r2[B][Hkv][2]        q64 max over this shard's dynamic keys of
 *                        n2 = sum_d trunc(x_d^2 2^64), x = bf16(fl32(k - c))
 * Sharded + mips: take the max of r2 over shards (magicpig_reduce_stats). */
int magicpig_key_norms(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv,
                       int64_t n_local, int64_t seq_offset, int64_t n_global, const int64_t* key_sum,
                       const int64_t* count, float* center, int64_t* r2, void* ws, size_t ws_bytes,
                       void* stream);

/* Element-wise exact reduction of P shard copies (after an all-gather):
 *   mode 0: key_sum/count SUM   parts_sum [P][B*Hkv*128][2], parts_cnt [P][B*Hkv]
 *   mode 1: r2 MAX              parts_sum [P][B*Hkv][2]  (parts_cnt unused)   */
int magicpig_reduce_stats(int mode, const int64_t* parts_sum, const int64_t* parts_cnt, int P,
                          int64_t B, int64_t Hkv, int64_t* out_sum, int64_t* out_cnt, void* stream);

/* Phase 3, hash tables (Alg. 1 input HT; Encode P:83-84):
 *   W [(128 + mips)][K*L] fp32, every value bf16-representable (R8), shared
 *     by all heads.  Row 128 multiplies the MIPS coordinate.
 *   codes: magicpig_codes_words() uint32, bit-plane layout above.  Bit =
 *     [exact(xbar_i . W_j) > 0] (R6), xbar_i = [x_i, s_i] (s_i with mips).
 *   key_norm[B][Hkv][n_local] fp32: |xbar_i| = sqrt(fl64(n2q 2^-64) + s_i^2),
 *     the norm of the hashed key vector used for p_i at decode (R5).
 * Runs on tcgen05 tensor cores (fp32 accumulate) with an error-bound filter
 * and exact integer fix-up of every near-zero dot, so bits are exact. */
int magicpig_build_tables(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv,
                          int64_t n_local, int64_t seq_offset, int64_t n_global, const float* W,
                          const float* center, const int64_t* r2, uint32_t* codes, float* key_norm,
                          void* ws, size_t ws_bytes, void* stream);

/* All three phases for an unsharded cache (seq_offset = 0, n_global = n). */
int magicpig_build_index(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv,
                         int64_t n, const float* W, float* center, int64_t* r2, uint32_t* codes,
                         float* key_norm, int64_t* key_sum, int64_t* count, void* ws, size_t ws_bytes,
                         void* stream);

/* --------------------------------------------------------------- decode ---
 * One MagicPIG decode step (Alg. 1) for all B x Hq query heads:
 * Encode q (qbar = [q, 0], R4), count per-key table matches against the
 * codes, sample S_g = {i in D : count >= min_collisions}, weight each
 * i in S_g by 1/u_i with u from Eq. (LSH sampling probability) at
 * the angle between the hashed vectors (R5), attend exactly to T (u = 1),
 * and evaluate the self-normalised estimator.
 *   out[B][Hq][128]      fp32 estimate (NULL to skip); a head whose S and T
 *                        are both empty gets 0 and sets STATUS_DEGENERATE
 *   partial[B][Hq][130]  fp32 (m, s, a[128]) log-sum-exp state of this shard
 *                        (NULL to skip), for magicpig_merge_partials
 *   s_count[B][Hq]       |S_g| on this shard (NULL to skip)
 *   s_mask[B][Hq][ceil(n_local/32)]  debug: bit r of word w = key 32w+r in S_g
 *                        (NULL to skip; costs extra stores)
 * center, key_norm: from the build.  W: same array as the build.       */
int magicpig_decode(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const uint32_t* codes,
                    const float* center, const float* key_norm, const uint16_t* k, const uint16_t* v,
                    int64_t B, int64_t Hkv, int64_t n_local, int64_t seq_offset, int64_t n_global,
                    const float* W, float* out, float* partial, int32_t* s_count, uint32_t* s_mask,
                    void* ws, size_t ws_bytes, void* stream);

/* The two halves of magicpig_decode, for callers that time or overlap them:
 * Encode (Alg. 1 "q_code = Encode(q, W)") writes the packed query codes
 * into the decode workspace `ws`; decode_encoded runs Query + estimator
 * from them.  Same arguments and outputs as magicpig_decode. */
int magicpig_encode_queries(const magicpig_config* cfg, const uint16_t* q, int64_t B, int64_t Hq,
                            const float* W, void* ws, size_t ws_bytes, void* stream);
int magicpig_decode_encoded(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                            const uint32_t* codes, const float* center, const float* key_norm,
                            const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv,
                            int64_t n_local, int64_t seq_offset, int64_t n_global, float* out,
                            float* partial, int32_t* s_count, uint32_t* s_mask, void* ws,
                            size_t ws_bytes, void* stream);

/* ------------------------------------------------------ bucketed tables ---
 * The paper's hash tables HT as inverted lists (
 * SURVEY 8(f) NEXT-1): per (sequence, kv head) unit and table t, the key ids
 * of this shard sorted by their K-bit code.  Query(HT, q_code) then reads only
 * the L buckets each query head falls into instead of every key's codes; the
 * sampled sets S_g are identical to the dense scan's (a key lies in exactly one
 * bucket per table, so "in the query's bucket of >= min_collisions tables" is
 * the P:84 rule).  Requires K <= 14 and ceil(n_local/32)*8 <= 200 KiB.
 * Layout, int32 words: tables[B*Hkv][ L*(2^K+1) int32 offsets | L*n_local ids ]:
 *   offsets[t][c] .. offsets[t][c+1]  = the range of ids[t][] with code c
 *   ids[t][e]                         = local key index (ascending within a
 *                                       bucket is NOT guaranteed); uint16 when
 *                                       n_local <= 65536 (the paper's int16
 *                                       entries; the id part is then
 *                                       ceil(L*n_local/2) words), else int32
 * magicpig_bucket_tables_words: size of `tables` (0 if unsupported). [host]
 * magicpig_build_buckets: builds them from the packed codes of
 *   magicpig_build_tables (call after it, same shapes).
 * magicpig_decode_buckets[_encoded]: magicpig_decode[_encoded] with S from the
 *   buckets; same arguments and outputs except `tables` replaces `codes`. */
size_t magicpig_bucket_tables_words(const magicpig_config* cfg, int64_t B, int64_t Hkv, int64_t n_local);
int magicpig_build_buckets(const magicpig_config* cfg, const uint32_t* codes, int64_t B, int64_t Hkv,
                           int64_t n_local, int32_t* tables, void* stream);
int magicpig_decode_buckets(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const int32_t* tables,
                            const float* center, const float* key_norm, const uint16_t* k, const uint16_t* v,
                            int64_t B, int64_t Hkv, int64_t n_local, int64_t seq_offset, int64_t n_global,
                            const float* W, float* out, float* partial, int32_t* s_count, uint32_t* s_mask,
                            void* ws, size_t ws_bytes, void* stream);
int magicpig_decode_buckets_encoded(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                                    const int32_t* tables, const float* center, const float* key_norm,
                                    const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv, int64_t n_local,
                                    int64_t seq_offset, int64_t n_global, float* out, float* partial,
                                    int32_t* s_count, uint32_t* s_mask, void* ws, size_t ws_bytes, void* stream);

/* Log-sum-exp merge of P partial states ("recursive attention"):
 *   parts[P][BH][130] -> out[BH][128] = sum_j a_j e^{m_j-M} / sum_j s_j e^{m_j-M}
 * (fixed order j = 0..P-1, so every rank gets bit-identical results). */
int magicpig_merge_partials(const float* parts, int P, int64_t BH, float* out, void* stream);

/* Decode-time append (the decoded token's key joins the cache; the
 * local window of the static set T moves with it): hashes the m new keys of every
 * (sequence, kv head) unit, k_new [B][Hkv][m][128] bf16, which become positions
 * n_old .. n_old+m-1, with the index's FROZEN centering vector and MIPS radius
 * (center, r2 from the build; reading R3: an appended key with |x|^2 > r^2 gets
 * the MIPS coordinate 0), exactly like magicpig_build_tables: their key_norm
 * entries and their code bits (exact signs, sign(0) = 0).  codes and key_norm
 * must already be laid out for n_old + m keys per unit (codes: the layout of
 * magicpig_codes_words(.., n_old + m); key_norm: [B][Hkv][n_old + m]); the caller
 * moves the existing entries when the layout grows (a new 1024-key chunk, or the
 * key_norm row stride).  The token that leaves the local window becomes a dynamic
 * key by position alone at the next decode (n_global = n_old + m); its code was
 * computed when it was built or appended.  ws: any library workspace (its status
 * word collects MAGICPIG_STATUS_INEXACT).  Returns 0 or an error code. */
int magicpig_append_keys(const magicpig_config* cfg, const uint16_t* k_new, int64_t m, int64_t B, int64_t Hkv,
                         int64_t n_old, const float* W, const float* center, const int64_t* r2, uint32_t* codes,
                         float* key_norm, void* ws, size_t ws_bytes, void* stream);

/* One whole decode step from HOST memory (the serving call): copies q_host
 * [B][Hq][128] bf16 [host; pinned memory makes the copy asynchronous] into the
 * workspace, encodes it, decodes it over the dense codes (tables ==
 * NULL) or the bucketed tables (codes ignored) as magicpig_decode /
 * magicpig_decode_buckets do (unsharded: seq_offset 0, n_global = n_local),
 * copies the output to out_host [B][Hq][128] fp32 [host] and synchronizes
 * `stream`, so out_host is valid when the call returns.  Returns 0 or an error
 * code. */
int magicpig_decode_host(const magicpig_config* cfg, const uint16_t* q_host, int64_t Hq, const uint32_t* codes,
                         const int32_t* tables, const float* center, const float* key_norm, const uint16_t* k,
                         const uint16_t* v, int64_t B, int64_t Hkv, int64_t n_local, const float* W, float* out_host,
                         void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- debug ---
 * Canonical codes [B][Hkv][n][L] uint16, bit b of table t = column t*K+b. */
int magicpig_export_codes(const magicpig_config* cfg, const uint32_t* codes, int64_t B, int64_t Hkv,
                          int64_t n_local, uint16_t* canonical, void* stream);
int magicpig_import_codes(const magicpig_config* cfg, const uint16_t* canonical, int64_t B,
                          int64_t Hkv, int64_t n_local, uint32_t* codes, void* stream);
/* Query codes [B][Hq][L] uint16 (canonical) for qbar = [q, 0]. */
int magicpig_query_codes(const magicpig_config* cfg, const uint16_t* q, int64_t B, int64_t Hq,
                         const float* W, uint16_t* qcodes, void* ws, size_t ws_bytes, void* stream);
/* Exact per-key collision counts [B][Hq][n_local] uint16 (all keys, D and T). */
int magicpig_collision_counts(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                              const uint32_t* codes, int64_t B, int64_t Hkv, int64_t n_local,
                              const float* W, uint16_t* counts, void* ws, size_t ws_bytes,
                              void* stream);
/* Raw fp32 tensor-core accumulators of the hash GEMM for the first
 * min(n_local, 128) keys of unit 0 and all K*L columns: acc[128][K*L]
 * (workspace: build workspace + 4*codes_words + 4*n_local bytes, 256-aligned)
 * (measures the tcgen05 accumulation error that the fix-up filter bounds). */
int magicpig_debug_hash_acc(const magicpig_config* cfg, const uint16_t* k, int64_t n_local,
                            const float* W, const float* center, const int64_t* r2, float* acc,
                            void* ws, size_t ws_bytes, void* stream);

/* Debug timeline of one decode (encode + decode_encoded, unsharded): thread 0
 * of every decode CTA writes %globaltimer (ns) at its phase boundaries into
 * timeline[cta][32] (0 = not reached): 0 start, 1 after griddepcontrol.wait,
 * 2 query masks, 3 scan, 4 cluster combine, 5 compaction, 6 gather,
 * 7 CTA partial, 8 cluster merge, 9 unit-merge start, 10 end; 11-16 gather
 * sub-phase clock64 cycles (rows, xbar, mma, log u, softmax max, accumulate).  Returns the
 * number of CTAs (> 0) or an error code. */
int64_t magicpig_debug_decode_timeline(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                                       const uint32_t* codes, const float* center, const float* key_norm,
                                       const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv,
                                       int64_t n_local, const float* W, float* out,
                                       unsigned long long* timeline, int64_t timeline_len, void* ws,
                                       size_t ws_bytes, void* stream);

/* The same timeline over the bucketed tables.  With decode kernel 7 (the default)
 * both calls write per-WARP stamps of the estimator kernel, timeline[row][16]
 * (row = cta * 8 + warp; ns since epoch, 0 = not reached): 0 start, 1 after
 * griddepcontrol.wait, 2 unit prefix done, 3 first entries loaded, 4 first
 * slabs issued, 5 first slab's rows arrived, 6 last slab computed, 7 flush
 * start, 8 unit merge start, 9 unit merge end, 10 end; 11 slabs computed,
 * 12 unit merges done; and return the number of rows. */
int64_t magicpig_debug_decode_timeline_buckets(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                                               const int32_t* tables, const float* center, const float* key_norm,
                                               const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv,
                                               int64_t n_local, const float* W, float* out,
                                               unsigned long long* timeline, int64_t timeline_len, void* ws,
                                               size_t ws_bytes, void* stream);

/* Debug: one decode step (encode + Query + estimator) that also exports the sets
 * the estimator actually used:
 *   s_mask[B][Hq][ceil(n_local/32)]    S_g restricted to D (the Query result), or NULL
 *   weighted[B][Hq][ceil(n_local/32)]  bit (g, i) set iff key i received a finite
 *                                      weight for head g in the estimator's gather,
 *                                      i.e. the compacted list it consumed: S_g u T
 *                                      (zeroed by this call)
 * codes (dense) or tables (bucketed, magicpig_build_buckets) selects the Query path.
 * Requires decode kernel 6 (the default).                                       */
int magicpig_debug_decode_sets(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const uint32_t* codes,
                               const int32_t* tables, const float* center, const float* key_norm, const uint16_t* k,
                               const uint16_t* v, int64_t B, int64_t Hkv, int64_t n_local, int64_t seq_offset,
                               int64_t n_global, const float* W, float* out, uint32_t* s_mask, uint32_t* weighted,
                               void* ws, size_t ws_bytes, void* stream);

/* Debug: selected stages of a decode step (decode kernel 6 or 7, unsharded), for
 * timing the kernels of the step separately.  `stage` is a bit mask:
 *   1  Query(HT, q_code) (Alg. 1): the dense scan of `codes`, or the
 *      bucketed `tables` if non-NULL -> per-head S bitmaps in the workspace;
 *   2  (kernel 7) select: S_g restricted to D, union over the unit's heads,
 *      ordered lists in the workspace;
 *   4  the estimator over what the earlier stages left in the
 *      workspace -> out (kernel 6: bits 2 and 4 both mean its one kernel).
 * 7 = a whole decode step.  The query codes must already be in the workspace
 * (magicpig_encode_queries).  Returns 0 or an error code (MAGICPIG_EINVAL for
 * another kernel version). */
int magicpig_debug_decode_stage(const magicpig_config* cfg, int stage, const uint16_t* q, int64_t Hq,
                                const uint32_t* codes, const int32_t* tables, const float* center,
                                const float* key_norm, const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv,
                                int64_t n_local, float* out, void* ws, size_t ws_bytes, void* stream);

/* Debug: magicpig_build_index (unsharded) with a CUDA event (cudaEvent_t, created
 * by the caller) recorded on `stream` at each phase boundary: events[0] before the
 * key statistics, [1] after them, [2] after the key norms / centering
 * vector / MIPS radius, [3] after the operand preparation (xbar tiles),
 * [4] after the hash GEMM and its exact fix-up.  Same results as
 * magicpig_build_index. */
int magicpig_debug_build_phases(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv, int64_t n,
                                const float* W, float* center, int64_t* r2, uint32_t* codes, float* key_norm,
                                int64_t* key_sum, int64_t* count, void* ws, size_t ws_bytes, void* stream,
                                void* const* events);

/* Selects the decode kernel for subsequent decode calls of this process (a debug
 * knob for A/B measurement).  0 (default) = automatic: kernel 5 for small decodes
 * (at most two 1024-key chunk tiles per SM: latency-bound, one fused launch), else
 * kernel 7.  7 = Query kernel (dense code scan with the select step fused, or the
 * bucketed tables + select kernel) emitting per-piece S_g u T lists, then the
 * balanced mma.sync estimator (every warp a contiguous range of the concatenated
 * lists) and the unit merge kernel; 8 = the same with the tcgen05 estimator (TMA-
 * free cp.async tiles in 128B-swizzled layout, TMEM accumulators); 6 = Query
 * kernel writing per-head S bitmaps, then an estimator with a producer warp;
 * 5 = persistent warp-specialised fused kernel
 * (one CTA per SM over a contiguous tile range; used whenever its shared-memory
 * layout fits, else 4), 4 = one thread-block cluster per 1024-key chunk.  Both
 * compute the same S bit for bit.  For kernel 5 the timeline slots are clock64
 * cycles since CTA start (+1): 1 query masks ready, 2 first descriptor, 3 first
 * gather batch, 4 unit merge start, 5 unit merge end, 6 gather done.
 * Returns 0 or MAGICPIG_EINVAL. [host] */
int magicpig_debug_set_decode_kernel(int version);

/* The decode kernel generation (4..8) the next decode call with these shapes will run
 * (resolves the automatic choice of kernel 0).  Returns it, or MAGICPIG_EINVAL. [host] */
int magicpig_debug_decode_kernel_choice(const magicpig_config* cfg, int64_t B, int64_t Hq, int64_t Hkv,
                                        int64_t n_local, int buckets);

/* Message for an error code. [host] */
const char* magicpig_strerror(int err);

/* Library version string, and the number of kernel launches issued so far by
 * this process (for the bench's gpu_launches claim). [host] */
const char* magicpig_version(void);
uint64_t magicpig_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MAGICPIG_H */

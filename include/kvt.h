/*
 * kvt.h — C ABI of libkvt.so, the B200 (sm_100a) implementation of KVTuner's data-parallel hot
 * path: layer-wise mixed-precision KV-cache quantisation and the decode attention that reads it
 * (arXiv 2502.04420, "KVTuner").
 *
 * Citations: "P:<n>" = line n of the paper's LaTeX source; "A<n>" = the reading of a
 * passage the paper leaves open, recorded in DESIGN.md §3; "§4" = DESIGN.md §4 (HBM layout).
 *
 * Conventions (all entry points):
 *   - Every call returns a kvt_status (KVT_OK = 0).  No C++ exception crosses the ABI.  On error
 *     kvt_last_error() returns a thread-local human-readable message.
 *   - Arguments are validated on the host before any launch.  Launch failures map to
 *     KVT_ERR_CUDA; asynchronous device faults surface at the caller's next synchronisation.
 *   - The library never allocates device memory and keeps no global mutable state.  The caller
 *     owns every buffer (the Python binding allocates them as torch tensors).  kvt_config is the
 *     only library-owned object: heap memory, immutable after load, freed by kvt_config_free.
 *   - Device calls take an explicit CUDA stream (a cudaStream_t passed as void*, NULL = legacy
 *     default stream) and are asynchronous with no hidden synchronisation.
 *   - Tensors are dense, row-major, little-endian.  "bf16" = IEEE binary32 top 16 bits.
 *   - GPU restrictions of this build: head_dim == 128; group in {32, 64, 128}; bits in {2,4,8,16}
 *     (16 = bf16 pass-through); GQA ratio g = n_q_heads / kv_heads in [1, 8].  Anything else is
 *     KVT_ERR_UNSUPPORTED.
 */
#ifndef KVT_H
#define KVT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVT_ABI_VERSION 4u   /* 3: kvt_append_decode_attention; merge counters first in the workspace;
                                4: schedule counters after them (per-SM plan), kvt_decode_plan */

typedef enum {
    KVT_OK = 0,
    KVT_ERR_INVALID_ARG = 1,   /* null pointer, bad shape, inconsistent lengths                 */
    KVT_ERR_IO = 2,            /* config file unreadable                                         */
    KVT_ERR_PARSE = 3,         /* config JSON malformed / schema violation (message has line:col) */
    KVT_ERR_UNSUPPORTED = 4,   /* valid per the paper but not built here (see restrictions above) */
    KVT_ERR_CAPACITY = 5,      /* an append would exceed the cache capacity                      */
    KVT_ERR_WORKSPACE = 6,     /* workspace too small                                            */
    KVT_ERR_CUDA = 8           /* a CUDA runtime call or launch failed                           */
} kvt_status;

/* Quantisation mode of a layer.
 *   PER_TOKEN_ASYM: K and V quantised per token in channel groups of `group` (A5), optional
 *                   full-precision window of the last `residual` tokens (A6, default 0).
 *   KIVI:           K per channel in token blocks of `group` with a full-precision residual of up to
 *                   `residual` tokens flushed block-wise; V per token in channel groups with a
 *                   sliding full-precision window of `residual` tokens (R = G = 32; A7, A8). */
typedef enum { KVT_MODE_PER_TOKEN_ASYM = 0, KVT_MODE_KIVI = 1,
               /* kvt_layer_sensitivity only (not a cache layout): K and V quantised per channel with
                * statistics over the whole trace (T-Mode; A28).  Whole-sequence statistics cannot be
                * appended write-once, so kvt_config_load rejects it. */
               KVT_MODE_PER_CHANNEL_ASYM = 2 } kvt_mode;

/* One layer's precision pair (P_k, P_v) (candidates {2,4,8}^2 P:316; 16 = bf16). */
typedef struct { int32_t key_bits, value_bits; } kvt_pair;

/* Everything needed to store one layer's cache. */
typedef struct { int32_t mode, key_bits, value_bits, group, residual; } kvt_layer_spec;

typedef struct kvt_config kvt_config;     /* opaque, immutable after load */

uint32_t    kvt_abi_version(void);
const char* kvt_status_string(int32_t status);
const char* kvt_last_error(void);          /* thread-local; "" when the last call succeeded */

/* ---- a1: searched configuration (P:306-310 problem, T-Config P:762-867) --------------------
 * `path_or_json` is either a path to a JSON file or a JSON document (first non-space char '{'):
 *   {"model_name": str, "quant_method": "kivi" | "per-token-asym",
 *    "equivalent_bits": number (the paper's label, informational),
 *    "group_size": int (optional; default 32), "residual_length": int (optional; default 32 for
 *    kivi, 0 for per-token-asym),
 *    "layers": [{"layer": int, "key_bits": int, "value_bits": int}, ...]}   (schema of S:471)
 * Every layer 0..L-1 must appear exactly once.  "per-channel-asym" parses but returns
 * KVT_ERR_UNSUPPORTED (whole-sequence statistics cannot be streamed write-once).
 * Host only; no device access.  On success *out owns a new config (free with kvt_config_free). */
int32_t     kvt_config_load(const char* path_or_json, kvt_config** out);
int32_t     kvt_config_num_layers(const kvt_config* cfg);
int32_t     kvt_config_layer(const kvt_config* cfg, int32_t layer, kvt_layer_spec* out);
/* f_m = sum_l (b_k^l + b_v^l) / (2L), the memory objective of Eq. 4, computed from the
 * layer list (not copied from the label). */
double      kvt_config_equivalent_bits(const kvt_config* cfg);
double      kvt_config_label_bits(const kvt_config* cfg);      /* "equivalent_bits" as written */
const char* kvt_config_model_name(const kvt_config* cfg);
void        kvt_config_free(kvt_config* cfg);

/* Validate one layer spec for this build (GPU restrictions above) at head_dim d. */
int32_t     kvt_validate_spec(const kvt_layer_spec* spec, int32_t head_dim);

/* ---- the quantised cache of one layer ------------------------------------------
 * Per (b, h) = (batch row, kv head) the caller provides `capacity` token rows (capacity % group
 * == 0).  Buffers, all indexed [b][h] outermost:
 *   k_codes  u8  [B][H][cap][row_k]   row_k = d*key_bits/8 (2d bytes of bf16 when 16): channel c at
 *                                       bits [c*b, (c+1)*b) of the row, LSB-first
 *   k_meta   u32 per-token:  [B][H][cap][d/G]   KIVI: [B][H][cap/G][d]   (none when 16)
 *                 word = bf16 scale (low 16 bits) | bf16 zero-point (high 16 bits)   (A3)
 *   k_resid  bf16 per-token: [B][H][R][d] ring (slot t mod R);  KIVI: [B][H][F][d] linear
 *                 (slot t - n_qK), F = R if R > 0 else G      (none when 16, or per-token R = 0)
 *   v_codes, v_meta, v_resid: as the per-token K buffers with value_bits.
 * KIVI layers with G = 32, d = 128 and 2/4/8-bit K and V use TILE RECORDS instead:
 *   k_codes  u8  [B][H][cap/32][rec], rec = 32*(16 kb + 16 vb) + 1024: record j = tokens 32j..32j+31 as
 *                 [K code rows | K block meta (d u32) | V codes in the blocked layout | V meta (32 x 4 u32)];
 *   k_meta, v_codes, v_meta are empty (size 0, may be NULL); k_resid / v_resid as above.
 * Token t of a length-S sequence is held quantised iff t < n_q (A6, A7):
 *   per-token tensor: n_q = max(0, S - R);  KIVI key: n_q = F * floor(S / F);  16 bits: n_q = S. */
typedef struct {
    kvt_layer_spec spec;
    int32_t batch, kv_heads, head_dim, capacity;
    void* k_codes; void* k_meta; void* k_resid;
    void* v_codes; void* v_meta; void* v_resid;
    /* PAGED tile records (vLLM-style block table, "vLLM" P:85).  NULL = dense.
     * Only for tile-record layers (else KVT_ERR_UNSUPPORTED).  Then k_codes is a pool of `num_pages`
     * pages; page p holds the kv_heads records of one 32-token block: record (p, h) at
     * k_codes + (p * kv_heads + h) * rec (rec as above; page bytes from kvt_page_bytes).  block_table:
     * DEVICE int32 [batch][max_pages]; block j (tokens 32j .. 32j+31) of sequence b is page
     * block_table[b * max_pages + j].  capacity must equal 32 * max_pages.  The residual buffers stay
     * dense.  The caller owns the table and keeps the pages of live blocks distinct and < num_pages
     * (the kernels do not check the entries: an out-of-range page is undefined behaviour). */
    const int32_t* block_table;
    int32_t max_pages, num_pages;
} kvt_layer_cache;

/* Bytes of one page (kv_heads tile records) of a paged cache with this spec; KVT_ERR_UNSUPPORTED when
 * the spec has no tile records. */
int32_t kvt_page_bytes(const kvt_layer_spec* spec, int32_t kv_heads, int32_t head_dim, uint64_t* bytes);

/* Byte sizes of the six buffers for the whole layer, in the order of kvt_layer_cache
 * (k_codes, k_meta, k_resid, v_codes, v_meta, v_resid); 0 for an absent buffer. */
int32_t kvt_cache_buffer_sizes(const kvt_layer_spec* spec, int32_t batch, int32_t kv_heads,
                               int32_t head_dim, int32_t capacity, uint64_t out_bytes[6]);

/* ---- a2/a3: quantise on append (Eq. 2; "K = concat(K_{:i-1}, k_i)") ------------
 * Appends n_new[b] tokens to every sequence b (prefill: large; decode: 1), quantising each group
 * as it completes (a KIVI key block when its residual fills; a value token when it leaves the
 * window).  The resulting bytes are independent of how the history was chunked (O2 history
 * independence), so they equal the oracle's static build bit for bit.
 *   k_new, v_new: bf16, element (b, h, t, c) at b*s[0] + h*s[1] + t*s[2] + c (c contiguous).
 *   len_before_dev / n_new_dev: int32 [B] on the device, read by the kernels.
 *   len_before_host / n_new_host: optional int32 [B] host copies used for validation (capacity)
 *   and launch planning; when NULL the launch is planned for n_new_max tokens and capacity is not
 *   checked.  The caller advances its lengths after the call. */
int32_t kvt_quantize_append(const kvt_layer_cache* cache, const void* k_new, const void* v_new,
                            const int64_t new_strides[3],
                            const int32_t* len_before_host, const int32_t* len_before_dev,
                            const int32_t* n_new_host, const int32_t* n_new_dev, int32_t n_new_max,
                            void* stream);

/* ---- a4/a5: decode attention (Eq. 1, over the dequantised cache) ----------------
 * out[b][hq][:] = softmax(scale * q[b][hq] . K_hat[b][hq/g]^T) V_hat[b][hq/g] over the seq_len[b]
 * tokens of the cache (the appended token included, A11).  GQA: query head hq reads kv head
 * floor(hq / g) (A10).  q: bf16 [B][H_q][d].  out: [B][H_q][d], fp32 (out_dtype 1) or bf16
 * (out_dtype 0, RNE of the fp32 result).  seq_len_dev: int32 [B] device; seq_len_host: optional
 * int32 [B] host copy for validation and split planning (NULL: plan for `capacity`).
 * softmax_scale is normally 1/sqrt(d) (A9).  A sequence of length 0 yields a zero row.
 * The split-KV partials live in `workspace` (size from kvt_decode_workspace_bytes).  The workspace must
 * be zero-filled before its first use (it holds per-(b, kv head) split-arrival counters); every call
 * leaves those counters at zero again, so one workspace can be reused by consecutive calls on a stream.
 * The workspace is laid out [merge counters: round_up(4 * batch * kv_heads, 256) bytes][schedule counters:
 * round_up(4 * (514 + batch * kv_heads + SMs), 256) bytes][partials], so calls on caches with the same (batch,
 * kv_heads) on one device can share one workspace whatever their precision pair or CTA count.
 * Ordering: tile-record layers may launch as a programmatic dependent (PDL) of the preceding kernel in the stream
 * (when the grid nearly fills the GPU); the kernel then waits for that kernel's completion before it reads
 * anything, so the call is ordered after every preceding stream operation like a plain launch. */
int32_t kvt_decode_workspace_bytes(const kvt_layer_cache* cache, int32_t n_q_heads,
                                   const int32_t* seq_len_host, uint64_t* bytes);
/* The work plan kvt_decode_attention would use for this cache (same arguments as kvt_decode_workspace_bytes):
 * out[0] = kernel (1 tensor-core tile-record kernel, 0 generic CUDA-core kernel), out[1] = CTAs launched (generic:
 * KV splits), out[2] = whole units per SM of the per-SM plan (0: stream-K / whole units by CTA index),
 * out[3] = resident CTAs per SM of the instance.  Needs a CUDA device (occupancy query); host only, no launch. */
int32_t kvt_decode_plan(const kvt_layer_cache* cache, int32_t n_q_heads, const int32_t* seq_len_host, int32_t out[4]);
int32_t kvt_decode_attention(const kvt_layer_cache* cache, const void* q, int32_t n_q_heads,
                             const int32_t* seq_len_host, const int32_t* seq_len_dev,
                             float softmax_scale, void* out, int32_t out_dtype,
                             void* workspace, uint64_t ws_bytes, void* stream);

/* ---- a3 + a4 in one call: the serving step of one layer ("fused append + attention") ----
 * kvt_quantize_append(cache, k_new, v_new, ..., len_before_dev, n_new_dev, n_new_max) followed by
 * kvt_decode_attention(cache, q, seq_len_dev, ...) on the same stream, with no host lengths (the launches are
 * planned for `capacity`, so the call can be captured once in a CUDA graph and replayed as the lengths grow).
 * Because the library launches the append itself, the attention kernel's prologue (the length scan and the q
 * setup) overlaps the append (programmatic dependent launch); the cache is read only after the append completed.
 * Precondition: q and seq_len_dev (= len_before_dev + n_new_dev, the caller's) are complete before this call is
 * issued in stream order, and the append does not modify them.  Errors are reported before any launch. */
int32_t kvt_append_decode_attention(const kvt_layer_cache* cache, const void* k_new, const void* v_new,
                                    const int64_t new_strides[3], const int32_t* len_before_dev,
                                    const int32_t* n_new_dev, int32_t n_new_max,
                                    const void* q, int32_t n_q_heads, const int32_t* seq_len_dev,
                                    float softmax_scale, void* out, int32_t out_dtype,
                                    void* workspace, uint64_t ws_bytes, void* stream);

/* ---- a6: sequence-sharded decode (multi-GPU) ----------------------------------------
 * Partial attention over this shard's tokens: partial fp32 [B][H_q][d + 2] holding, per row,
 * m = max_t (scale * q.k_t) * log2(e), l = sum_t 2^(s_t - m), o = (sum_t 2^(s_t - m) v_t) / l
 * (an empty shard gives m = -inf, l = 0, o = 0).  kvt_combine_partials merges n_shards such
 * blocks laid out [n_shards][B][H_q][d + 2] (e.g. after an all-gather) into out. */
int32_t kvt_decode_attention_partial(const kvt_layer_cache* cache, const void* q, int32_t n_q_heads,
                                     const int32_t* seq_len_host, const int32_t* seq_len_dev,
                                     float softmax_scale, float* partial,
                                     void* workspace, uint64_t ws_bytes, void* stream);
/* a6 with the exchange fused into the attention kernel ("push"): as kvt_decode_attention_partial, but every
 * (m, l, o) row is stored straight into each of the n_dst (1..8) destinations — typically this shard's slot
 * of every rank's gathered buffer, mapped into this GPU's address space over NVLink (symmetric memory /
 * CUDA IPC), so the all-gather happens in the kernel's epilogue and the ranks only need a barrier before
 * kvt_combine_partials.  dsts: HOST array of device pointers, each to a [B][H_q][d + 2] fp32 block, 4-byte
 * aligned.  Visibility to the peers is the caller's: a system-scope barrier after this call in stream order. */
int32_t kvt_decode_attention_partial_push(const kvt_layer_cache* cache, const void* q, int32_t n_q_heads,
                                          const int32_t* seq_len_host, const int32_t* seq_len_dev,
                                          float softmax_scale, float* const* dsts, int32_t n_dst,
                                          void* workspace, uint64_t ws_bytes, void* stream);
int32_t kvt_combine_partials(const float* gathered, int32_t n_shards, int32_t batch,
                             int32_t n_q_heads, int32_t head_dim, void* out, int32_t out_dtype,
                             void* stream);

/* ---- a7: layer sensitivity (App. B protocol P:622-623) -------------------------------
 * For one layer and one calibration prompt, for every pair p: quantise the whole trace statically
 * at (b_k, b_v) under (mode, group, residual) (A15; mode KVT_MODE_PER_CHANNEL_ASYM: one group per channel
 * column of the whole trace for K and V, `group` ignored, residual must be 0, A28), run the t_q decode queries causally (query i at
 * position q_pos0 + i attends to tokens [0, q_pos0 + i]) with (K, V) and with (K_hat, V_hat), and
 * write fp64 out_dev[p] = {e_k, e_v, e_a, e_o, e_o_l1} (A13, A16).  Arithmetic is fp64.
 *   q: bf16 [H_q][T_q][d]; k, v: bf16 [H_kv][S][d]; pairs: HOST array; out_dev: device. */
typedef struct { double e_k, e_v, e_a, e_o, e_o_l1; } kvt_errors;
int32_t kvt_sensitivity_workspace_bytes(int32_t n_q_heads, int32_t t_q, int32_t n_kv_heads,
                                        int32_t seq_len, int32_t head_dim, int32_t group,
                                        uint64_t* bytes);
int32_t kvt_layer_sensitivity(int32_t mode, int32_t group, int32_t residual,
                              const void* q, int32_t n_q_heads, int32_t t_q, int32_t q_pos0,
                              const void* k, const void* v, int32_t n_kv_heads, int32_t seq_len,
                              int32_t head_dim, float softmax_scale,
                              const kvt_pair* pairs, int32_t n_pairs, kvt_errors* out_dev,
                              void* workspace, uint64_t ws_bytes, void* stream);

/* ---- search-space pruning after calibration (host only, no CUDA) -----------------------------------
 * The step after a7: the per-layer profiles e_o[layer][pair] (from kvt_layer_sensitivity, averaged over
 * the calibration prompts by the caller, A14) become the reduced search space S_p^G of the offline MOO
 * search (App. D).  Readings A24-A27.  All buffers are HOST memory
 * owned by the caller; nothing is retained between calls. */

/* Intra-layer pruning: keep[i] = 1 iff pair i is on the Pareto frontier of (equivalent bits
 * (b_k + b_v)/2, e_o[i]), i.e. no j has bits_j <= bits_i and e_o[j] <= e_o[i] with one of them strict;
 * exact ties both survive (A24).  pairs/e_o/keep: [n_pairs], n_pairs >= 1.
 * Errors: KVT_ERR_INVALID_ARG for null pointers, n_pairs < 1, bits outside {2,4,8,16}, non-finite e_o. */
int32_t kvt_pareto_prune(const kvt_pair* pairs, const double* e_o, int32_t n_pairs, uint8_t* keep);

/* DBSCAN (Ester et al. 1996, the clustering of App. D): points [n][dim] row-major; neighbourhood =
 * Euclidean distance <= eps, the point itself included; core = >= min_samples neighbours; clusters are
 * grown from unlabelled core points in index order, a border point joins the first cluster that reaches
 * it.  labels[n] = cluster id (0, 1, ... in order of discovery) or -1 for noise (A25).
 * Errors: KVT_ERR_INVALID_ARG for n < 0, dim < 1, min_samples < 1, eps < 0 or non-finite input. */
int32_t kvt_dbscan(const double* points, int32_t n, int32_t dim, double eps, int32_t min_samples,
                   int32_t* labels);

/* The two-level pruning of P:316-325: per layer kvt_pareto_prune over the common candidate list
 * `pairs` (e_o: [n_layers][n_pairs]); layers partitioned by identical kept sets; inside each
 * partition kvt_dbscan(eps, min_samples) on each layer's e_o over the partition's kept pairs (
 * the paper uses eps = 0.05, min_samples = 2); DBSCAN noise layers become singleton groups (A26).
 * Outputs: keep [n_layers][n_pairs]; group_of_layer [n_layers] with groups numbered 0..G-1 in order of
 * their first layer (A27); *n_groups = G.  Requires 1 <= n_pairs <= 64, n_layers >= 1. */
int32_t kvt_prune_and_cluster(const kvt_pair* pairs, int32_t n_pairs, const double* e_o, int32_t n_layers,
                              double eps, int32_t min_samples, uint8_t* keep, int32_t* group_of_layer,
                              int32_t* n_groups);

/* log10 of the search-space size prod_i counts[i] ("9^L", "5^G = 15625"); counts >= 1. */
int32_t kvt_search_space_log10(const int32_t* counts, int32_t n, double* log10_size);

#ifdef __cplusplus
}
#endif
#endif /* KVT_H */

// kvt_api.cu — the C ABI of libkvt.so (include/kvt.h): argument validation, geometry, error
// reporting, and dispatch to the kernel launchers.  Host code only.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "kvt_internal.h"

namespace kvt {

static thread_local std::string g_last_error;

int32_t fail(int32_t status, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return status;
}

void clear_error() { g_last_error.clear(); }

static bool ok_bits(int b) { return b == 2 || b == 4 || b == 8 || b == 16; }

int32_t make_geometry(const kvt_layer_spec& s, int B, int H, int d, int cap, Geometry* g) {
    if (s.mode != KVT_MODE_PER_TOKEN_ASYM && s.mode != KVT_MODE_KIVI)
        return fail(KVT_ERR_INVALID_ARG, "unknown mode %d", s.mode);
    if (!ok_bits(s.key_bits) || !ok_bits(s.value_bits))
        return fail(KVT_ERR_INVALID_ARG, "bits must be 2, 4, 8 or 16 (got K%d V%d)", s.key_bits, s.value_bits);
    if (B < 0 || H <= 0 || cap < 0) return fail(KVT_ERR_INVALID_ARG, "bad cache shape B=%d H=%d cap=%d", B, H, cap);
    if (s.residual < 0) return fail(KVT_ERR_INVALID_ARG, "residual must be >= 0");
    if (d != 128) return fail(KVT_ERR_UNSUPPORTED, "head_dim %d: this build supports head_dim 128 only", d);
    if (s.group != 32 && s.group != 64 && s.group != 128)
        return fail(KVT_ERR_UNSUPPORTED, "group %d: this build supports group 32, 64 or 128", s.group);
    if (cap % s.group != 0) return fail(KVT_ERR_INVALID_ARG, "capacity %d must be a multiple of group %d", cap, s.group);
    if (s.mode == KVT_MODE_KIVI && s.residual % s.group != 0)
        return fail(KVT_ERR_INVALID_ARG, "kivi: residual %d must be a multiple of group %d", s.residual, s.group);
    Geometry r{};
    r.mode = s.mode; r.kb = s.key_bits; r.vb = s.value_bits; r.G = s.group; r.R = s.residual;
    r.F = flush_size(s.group, s.residual); r.d = d; r.cap = cap; r.B = B; r.H = H;
    r.key_per_channel = (s.mode == KVT_MODE_KIVI && s.key_bits != 16);
    r.v_blocked = (s.key_bits != 16 && s.value_bits != 16 && s.group == 32 && d == 128);   // tile records, both modes
    r.row_k = (size_t)row_bytes(d, r.kb);
    r.row_v = (size_t)row_bytes(d, r.vb);
    r.kc = (size_t)cap * r.row_k;
    if (r.kb == 16) { r.km = 0; r.kr = 0; }
    else if (r.key_per_channel) { r.km = (size_t)(cap / r.G) * d * 4; r.kr = (size_t)r.F * d * 2; }
    else { r.km = (size_t)cap * (d / r.G) * 4; r.kr = (size_t)r.R * d * 2; }
    r.vc = (size_t)cap * r.row_v;
    if (r.vb == 16) { r.vm = 0; r.vr = 0; }
    else { r.vm = (size_t)cap * (d / r.G) * 4; r.vr = (size_t)r.R * d * 2; }
    if (r.v_blocked) {
        r.rec_km = (uint32_t)(32 * r.row_k);
        r.rec_vc = r.rec_km + 512;
        r.rec_vm = r.rec_vc + (uint32_t)(32 * r.row_v);
        r.rec = (size_t)r.rec_vm + 512;
        r.kc = (size_t)(cap / 32) * r.rec;
        r.km = r.vc = r.vm = 0;
    }
    *g = r;
    return KVT_OK;
}

static int32_t cache_geometry(const kvt_layer_cache* c, Geometry* g, CachePtrs* p) {
    if (!c) return fail(KVT_ERR_INVALID_ARG, "null cache");
    int32_t st = make_geometry(c->spec, c->batch, c->kv_heads, c->head_dim, c->capacity, g);
    if (st) return st;
    p->bt = c->block_table;
    p->max_pages = 0;
    if (c->block_table) {
        if (!g->v_blocked) return fail(KVT_ERR_UNSUPPORTED, "paged caches need tile records (G = 32, d = 128, 2/4/8-bit K and V)");
        if (c->max_pages <= 0 || c->num_pages <= 0 || (int64_t)c->max_pages * 32 != c->capacity)
            return fail(KVT_ERR_INVALID_ARG, "paged cache: max_pages %d, num_pages %d, capacity %d (must be 32 * max_pages)",
                        c->max_pages, c->num_pages, c->capacity);
        if ((uintptr_t)c->block_table & 3) return fail(KVT_ERR_INVALID_ARG, "block_table must be 4-byte aligned");
        p->max_pages = c->max_pages;
    }
    const char* names[6] = {"k_codes", "k_meta", "k_resid", "v_codes", "v_meta", "v_resid"};
    void* ptrs[6] = {c->k_codes, c->k_meta, c->k_resid, c->v_codes, c->v_meta, c->v_resid};
    size_t sz[6] = {g->kc, g->km, g->kr, g->vc, g->vm, g->vr};
    for (int i = 0; i < 6; ++i) {
        if (sz[i] && !ptrs[i]) return fail(KVT_ERR_INVALID_ARG, "cache buffer %s is NULL but needs %zu bytes per slice", names[i], sz[i]);
        if (sz[i] && ((uintptr_t)ptrs[i] & 15)) return fail(KVT_ERR_INVALID_ARG, "cache buffer %s must be 16-byte aligned", names[i]);
    }
    p->k_codes = (uint8_t*)c->k_codes; p->k_meta = (uint32_t*)c->k_meta; p->k_resid = (uint16_t*)c->k_resid;
    p->v_codes = (uint8_t*)c->v_codes; p->v_meta = (uint32_t*)c->v_meta; p->v_resid = (uint16_t*)c->v_resid;
    return KVT_OK;
}

}  // namespace kvt

using namespace kvt;

extern "C" uint32_t kvt_abi_version(void) { return KVT_ABI_VERSION; }

extern "C" const char* kvt_status_string(int32_t s) {
    switch (s) {
        case KVT_OK: return "ok";
        case KVT_ERR_INVALID_ARG: return "invalid argument";
        case KVT_ERR_IO: return "i/o error";
        case KVT_ERR_PARSE: return "parse error";
        case KVT_ERR_UNSUPPORTED: return "unsupported";
        case KVT_ERR_CAPACITY: return "capacity exceeded";
        case KVT_ERR_WORKSPACE: return "workspace too small";
        case KVT_ERR_CUDA: return "cuda error";
        default: return "unknown status";
    }
}

extern "C" const char* kvt_last_error(void) { return g_last_error.c_str(); }

extern "C" int32_t kvt_validate_spec(const kvt_layer_spec* spec, int32_t head_dim) {
    clear_error();
    if (!spec) return fail(KVT_ERR_INVALID_ARG, "null spec");
    Geometry g;
    return make_geometry(*spec, 1, 1, head_dim, spec->group > 0 ? spec->group : 32, &g);
}

extern "C" int32_t kvt_cache_buffer_sizes(const kvt_layer_spec* spec, int32_t batch, int32_t kv_heads,
                                          int32_t head_dim, int32_t capacity, uint64_t out[6]) {
    clear_error();
    if (!spec || !out) return fail(KVT_ERR_INVALID_ARG, "null argument");
    Geometry g;
    int32_t st = make_geometry(*spec, batch, kv_heads, head_dim, capacity, &g);
    if (st) return st;
    uint64_t n = (uint64_t)batch * (uint64_t)kv_heads;
    out[0] = n * g.kc; out[1] = n * g.km; out[2] = n * g.kr;
    out[3] = n * g.vc; out[4] = n * g.vm; out[5] = n * g.vr;
    return KVT_OK;
}

extern "C" int32_t kvt_page_bytes(const kvt_layer_spec* spec, int32_t kv_heads, int32_t head_dim, uint64_t* bytes) {
    clear_error();
    if (!spec || !bytes) return fail(KVT_ERR_INVALID_ARG, "null argument");
    Geometry g;
    int32_t st = make_geometry(*spec, 1, kv_heads, head_dim, 32, &g);
    if (st) return st;
    if (!g.v_blocked) return fail(KVT_ERR_UNSUPPORTED, "paged caches need tile records (G = 32, d = 128, 2/4/8-bit K and V)");
    *bytes = (uint64_t)kv_heads * g.rec;
    return KVT_OK;
}

extern "C" int32_t kvt_quantize_append(const kvt_layer_cache* cache, const void* k_new, const void* v_new,
                                       const int64_t new_strides[3], const int32_t* len_before_host,
                                       const int32_t* len_before_dev, const int32_t* n_new_host,
                                       const int32_t* n_new_dev, int32_t n_new_max, void* stream) {
    clear_error();
    Geometry g; CachePtrs p;
    int32_t st = cache_geometry(cache, &g, &p);
    if (st) return st;
    if (!k_new || !v_new || !new_strides || !len_before_dev || !n_new_dev)
        return fail(KVT_ERR_INVALID_ARG, "kvt_quantize_append: null argument");
    if (((uintptr_t)k_new & 7) || ((uintptr_t)v_new & 7) || (new_strides[0] & 3) || (new_strides[1] & 3) || (new_strides[2] & 3))
        return fail(KVT_ERR_INVALID_ARG, "k_new/v_new must be 8-byte aligned with strides multiple of 4 elements");
    int plan = n_new_max;
    if (len_before_host && n_new_host) {
        plan = 0;
        for (int b = 0; b < g.B; ++b) {
            if (len_before_host[b] < 0 || n_new_host[b] < 0)
                return fail(KVT_ERR_INVALID_ARG, "negative length at batch row %d", b);
            if ((int64_t)len_before_host[b] + n_new_host[b] > g.cap)
                return fail(KVT_ERR_CAPACITY, "batch row %d: %d + %d tokens exceed capacity %d", b,
                            len_before_host[b], n_new_host[b], g.cap);
            if (n_new_host[b] > plan) plan = n_new_host[b];
        }
    }
    if (plan < 0) return fail(KVT_ERR_INVALID_ARG, "n_new_max < 0");
    if (plan == 0 || g.B == 0) return KVT_OK;
    return launch_append(g, p, (const uint16_t*)k_new, (const uint16_t*)v_new, new_strides, len_before_dev,
                         n_new_dev, plan, stream);
}

static int32_t decode_common(const kvt_layer_cache* cache, const void* q, int32_t H_q, const int32_t* seq_len_host,
                             const int32_t* seq_len_dev, Geometry* g, CachePtrs* p, int* plan) {
    int32_t st = cache_geometry(cache, g, p);
    if (st) return st;
    if (!q || !seq_len_dev) return fail(KVT_ERR_INVALID_ARG, "decode: null q or seq_len_dev");
    if (((uintptr_t)q & 15)) return fail(KVT_ERR_INVALID_ARG, "q must be 16-byte aligned");
    if (H_q <= 0 || H_q % g->H != 0) return fail(KVT_ERR_INVALID_ARG, "n_q_heads %d must be a multiple of kv_heads %d", H_q, g->H);
    if (H_q / g->H > 8) return fail(KVT_ERR_UNSUPPORTED, "GQA ratio %d > 8 is not built", H_q / g->H);
    *plan = g->cap;
    if (seq_len_host) {
        *plan = 0;
        for (int b = 0; b < g->B; ++b) {
            if (seq_len_host[b] < 0 || seq_len_host[b] > g->cap)
                return fail(KVT_ERR_CAPACITY, "seq_len[%d] = %d outside [0, capacity %d]", b, seq_len_host[b], g->cap);
            if (seq_len_host[b] > *plan) *plan = seq_len_host[b];
        }
    }
    return KVT_OK;
}

extern "C" int32_t kvt_decode_workspace_bytes(const kvt_layer_cache* cache, int32_t H_q, const int32_t* seq_len_host,
                                              uint64_t* bytes) {
    clear_error();
    if (!bytes) return fail(KVT_ERR_INVALID_ARG, "null bytes");
    Geometry g; CachePtrs p;
    int32_t st = cache_geometry(cache, &g, &p);
    if (st) return st;
    int plan = g.cap;
    if (seq_len_host) { plan = 0; for (int b = 0; b < g.B; ++b) plan = seq_len_host[b] > plan ? seq_len_host[b] : plan; }
    *bytes = decode_workspace(g, H_q, plan);
    return KVT_OK;
}

extern "C" int32_t kvt_decode_plan(const kvt_layer_cache* cache, int32_t H_q, const int32_t* seq_len_host, int32_t out[4]) {
    clear_error();
    if (!out) return fail(KVT_ERR_INVALID_ARG, "null out");
    Geometry g; CachePtrs p;
    int32_t st = cache_geometry(cache, &g, &p);
    if (st) return st;
    if (H_q <= 0 || H_q % g.H != 0 || H_q / g.H > 8) return fail(KVT_ERR_INVALID_ARG, "n_q_heads must be 1..8 x kv_heads");
    int plan = g.cap;
    if (seq_len_host) { plan = 0; for (int b = 0; b < g.B; ++b) plan = seq_len_host[b] > plan ? seq_len_host[b] : plan; }
    return decode_plan(g, H_q, plan, out);
}

extern "C" int32_t kvt_decode_attention(const kvt_layer_cache* cache, const void* q, int32_t H_q,
                                        const int32_t* seq_len_host, const int32_t* seq_len_dev, float scale,
                                        void* out, int32_t out_dtype, void* ws, uint64_t ws_bytes, void* stream) {
    clear_error();
    Geometry g; CachePtrs p; int plan;
    int32_t st = decode_common(cache, q, H_q, seq_len_host, seq_len_dev, &g, &p, &plan);
    if (st) return st;
    if (!out) return fail(KVT_ERR_INVALID_ARG, "decode: null out");
    if (out_dtype != 0 && out_dtype != 1) return fail(KVT_ERR_INVALID_ARG, "out_dtype must be 0 (bf16) or 1 (fp32)");
    if (g.B == 0) return KVT_OK;
    return launch_decode(g, p, (const uint16_t*)q, H_q, seq_len_dev, plan, scale, out, out_dtype, ws, ws_bytes, stream);
}

extern "C" int32_t kvt_append_decode_attention(const kvt_layer_cache* cache, const void* k_new, const void* v_new,
                                               const int64_t new_strides[3], const int32_t* len_before_dev,
                                               const int32_t* n_new_dev, int32_t n_new_max, const void* q, int32_t H_q,
                                               const int32_t* seq_len_dev, float scale, void* out, int32_t out_dtype,
                                               void* ws, uint64_t ws_bytes, void* stream) {
    clear_error();
    Geometry g; CachePtrs p; int plan;
    int32_t st = decode_common(cache, q, H_q, nullptr, seq_len_dev, &g, &p, &plan);
    if (st) return st;
    if (!out) return fail(KVT_ERR_INVALID_ARG, "append+decode: null out");
    if (out_dtype != 0 && out_dtype != 1) return fail(KVT_ERR_INVALID_ARG, "out_dtype must be 0 (bf16) or 1 (fp32)");
    if (!k_new || !v_new || !new_strides || !len_before_dev || !n_new_dev)
        return fail(KVT_ERR_INVALID_ARG, "append+decode: null argument");
    if (((uintptr_t)k_new & 7) || ((uintptr_t)v_new & 7) || (new_strides[0] & 3) || (new_strides[1] & 3) || (new_strides[2] & 3))
        return fail(KVT_ERR_INVALID_ARG, "k_new/v_new must be 8-byte aligned with strides multiple of 4 elements");
    if (n_new_max < 0) return fail(KVT_ERR_INVALID_ARG, "n_new_max < 0");
    if (g.B == 0) return KVT_OK;
    // the workspace is validated before anything is launched, so an error leaves the cache untouched
    const size_t need = decode_workspace(g, H_q, plan);
    if (need > ws_bytes || (need && !ws))
        return fail(KVT_ERR_WORKSPACE, "append+decode: workspace %llu < %zu bytes", (unsigned long long)ws_bytes, need);
    if (n_new_max > 0) {
        st = launch_append(g, p, (const uint16_t*)k_new, (const uint16_t*)v_new, new_strides, len_before_dev, n_new_dev,
                           n_new_max, stream);
        if (st) return st;
    }
    // the library launched the preceding kernel itself: the decode prologue (lengths, q) may overlap it
    return launch_decode(g, p, (const uint16_t*)q, H_q, seq_len_dev, plan, scale, out, out_dtype, ws, ws_bytes, stream,
                         nullptr, 0, /*early=*/n_new_max > 0);
}

extern "C" int32_t kvt_decode_attention_partial(const kvt_layer_cache* cache, const void* q, int32_t H_q,
                                                const int32_t* seq_len_host, const int32_t* seq_len_dev, float scale,
                                                float* partial, void* ws, uint64_t ws_bytes, void* stream) {
    clear_error();
    Geometry g; CachePtrs p; int plan;
    int32_t st = decode_common(cache, q, H_q, seq_len_host, seq_len_dev, &g, &p, &plan);
    if (st) return st;
    if (!partial) return fail(KVT_ERR_INVALID_ARG, "decode partial: null partial");
    if (g.B == 0) return KVT_OK;
    return launch_decode(g, p, (const uint16_t*)q, H_q, seq_len_dev, plan, scale, partial, 2, ws, ws_bytes, stream);
}

extern "C" int32_t kvt_decode_attention_partial_push(const kvt_layer_cache* cache, const void* q, int32_t H_q,
                                                     const int32_t* seq_len_host, const int32_t* seq_len_dev,
                                                     float scale, float* const* dsts, int32_t n_dst, void* ws,
                                                     uint64_t ws_bytes, void* stream) {
    clear_error();
    Geometry g; CachePtrs p; int plan;
    int32_t st = decode_common(cache, q, H_q, seq_len_host, seq_len_dev, &g, &p, &plan);
    if (st) return st;
    if (!dsts || n_dst < 1 || n_dst > 8) return fail(KVT_ERR_INVALID_ARG, "decode push: need 1..8 destinations (got %d)", n_dst);
    for (int i = 0; i < n_dst; ++i)
        if (!dsts[i] || ((uintptr_t)dsts[i] & 3)) return fail(KVT_ERR_INVALID_ARG, "decode push: destination %d is null or misaligned", i);
    if (g.B == 0) return KVT_OK;
    return launch_decode(g, p, (const uint16_t*)q, H_q, seq_len_dev, plan, scale, dsts[0], 2, ws, ws_bytes, stream,
                         dsts, n_dst);
}

extern "C" int32_t kvt_combine_partials(const float* gathered, int32_t n_shards, int32_t B, int32_t H_q,
                                        int32_t d, void* out, int32_t out_dtype, void* stream) {
    clear_error();
    if (!gathered || !out) return fail(KVT_ERR_INVALID_ARG, "combine: null argument");
    if (n_shards <= 0 || B < 0 || H_q <= 0) return fail(KVT_ERR_INVALID_ARG, "combine: bad shape");
    if (d != 128) return fail(KVT_ERR_UNSUPPORTED, "combine: head_dim 128 only");
    if (out_dtype != 0 && out_dtype != 1) return fail(KVT_ERR_INVALID_ARG, "out_dtype must be 0 or 1");
    if (B == 0) return KVT_OK;
    return launch_combine(gathered, n_shards, B, H_q, d, out, out_dtype, stream);
}

extern "C" int32_t kvt_sensitivity_workspace_bytes(int32_t H_q, int32_t T_q, int32_t H_kv, int32_t S, int32_t d,
                                                   int32_t G, uint64_t* bytes) {
    clear_error();
    if (!bytes) return fail(KVT_ERR_INVALID_ARG, "null bytes");
    if (H_q <= 0 || H_kv <= 0 || T_q < 0 || S <= 0 || d <= 0 || G <= 0) return fail(KVT_ERR_INVALID_ARG, "bad shape");
    *bytes = sensitivity_workspace(H_q, T_q, H_kv, S, d, G);
    return KVT_OK;
}

extern "C" int32_t kvt_layer_sensitivity(int32_t mode, int32_t G, int32_t R, const void* q, int32_t H_q, int32_t T_q,
                                         int32_t q_pos0, const void* k, const void* v, int32_t H_kv, int32_t S,
                                         int32_t d, float scale, const kvt_pair* pairs, int32_t n_pairs,
                                         kvt_errors* out_dev, void* ws, uint64_t ws_bytes, void* stream) {
    clear_error();
    if (!q || !k || !v || !pairs || !out_dev) return fail(KVT_ERR_INVALID_ARG, "sensitivity: null argument");
    if (H_kv <= 0 || H_q <= 0 || H_q % H_kv != 0) return fail(KVT_ERR_INVALID_ARG, "sensitivity: H_q %% H_kv != 0");
    if (S <= 0 || T_q <= 0 || q_pos0 < 0 || (int64_t)q_pos0 + T_q > S)
        return fail(KVT_ERR_INVALID_ARG, "sensitivity: need 0 <= q_pos0 and q_pos0 + T_q <= S");
    if (n_pairs <= 0) return fail(KVT_ERR_INVALID_ARG, "sensitivity: n_pairs must be > 0");
    if (mode == KVT_MODE_PER_CHANNEL_ASYM) {   // whole-sequence statistics, no residual, no grouping (A28)
        if (d != 128) return fail(KVT_ERR_UNSUPPORTED, "sensitivity: head_dim %d (128 only)", d);
        if (R != 0) return fail(KVT_ERR_INVALID_ARG, "sensitivity: per-channel-asym has no residual (R = %d)", R);
        for (int i = 0; i < n_pairs; ++i)
            for (int b : {pairs[i].key_bits, pairs[i].value_bits})
                if (b != 2 && b != 4 && b != 8 && b != 16)
                    return fail(KVT_ERR_INVALID_ARG, "sensitivity: pair %d has %d bits", i, b);
    }
    for (int i = 0; i < n_pairs && mode != KVT_MODE_PER_CHANNEL_ASYM; ++i) {
        kvt_layer_spec s{mode, pairs[i].key_bits, pairs[i].value_bits, G, R};
        Geometry g;
        int cap = ((S + G - 1) / (G > 0 ? G : 1)) * G;
        int32_t st = make_geometry(s, 1, H_kv, d, cap, &g);
        if (st) return st;
    }
    if (sensitivity_workspace(H_q, T_q, H_kv, S, d, G) > ws_bytes)
        return fail(KVT_ERR_WORKSPACE, "sensitivity: workspace %llu < %zu bytes", (unsigned long long)ws_bytes,
                    sensitivity_workspace(H_q, T_q, H_kv, S, d, G));
    return launch_sensitivity(mode, G, R, (const uint16_t*)q, H_q, T_q, q_pos0, (const uint16_t*)k,
                              (const uint16_t*)v, H_kv, S, d, scale, pairs, n_pairs, out_dev, ws, ws_bytes, stream);
}

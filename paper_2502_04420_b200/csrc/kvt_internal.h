// kvt_internal.h — shared host/device definitions of libkvt.so (product code; never includes or
// is included by oracle/).
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/kvt.h"

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace kvt {

// ---- thread-local error reporting (kvt_last_error) ----
int32_t fail(int32_t status, const char* fmt, ...);
void clear_error();

// ---- cache geometry ----
// Regions of a length-S sequence (A6, A7).  Used identically by host planning and the kernels.
__host__ __device__ inline int flush_size(int G, int R) { return R > 0 ? R : G; }
__host__ __device__ inline int nq_per_token(int bits, int R, int S) {
    return bits == 16 ? S : (S > R ? S - R : 0);
}
__host__ __device__ inline int nq_key(int mode, int bits, int G, int R, int S) {
    if (bits == 16) return S;
    if (mode == KVT_MODE_KIVI) { int F = flush_size(G, R); return F * (S / F); }
    return S > R ? S - R : 0;
}
__host__ __device__ inline int row_bytes(int d, int bits) { return bits == 16 ? 2 * d : d * bits / 8; }

// Blocked value layout: byte offset, inside a 32-token block, of byte k of chunk
// (gam, i) = channels 32 gam + 4 i .. + 3 of the token at position tau of the block.  Tokens tau and
// tau + 8 of each 16-token half share 32-bit words, so the PV operand pairs load directly.
__host__ __device__ inline uint32_t vblk_off(int bits, int tau, int gam, int i, int k) {
    const int ks = tau >> 4, r = tau & 15, j = r & 7;
    if (bits == 2) {
        const uint32_t w = (uint32_t)(((ks * 8 + i) * 4 + (r & 3)) * 4 + gam);
        return 4 * w + 2 * (uint32_t)(r >> 3) + (uint32_t)((r & 7) >> 2);
    }
    if (bits == 4) {
        const uint32_t w = (uint32_t)((((ks * 2 + (j >> 2)) * 8 + i) * 4 + (j & 3)) * 4 + gam);
        return 4 * w + 2 * (uint32_t)(r >> 3) + (uint32_t)k;
    }
    const uint32_t u = (uint32_t)((((ks * 2 + (j >> 2)) * 2 + (gam >> 1)) * 8 + i) * 4 + (j & 3));
    const uint32_t w = u * 4 + (uint32_t)(gam & 1) * 2 + (uint32_t)(k >> 1);
    return 4 * w + 2 * (uint32_t)(k & 1) + (uint32_t)(r >> 3);
}

struct Geometry {
    int mode, kb, vb, G, R, F, d, cap, B, H;
    bool key_per_channel;          // KIVI key with bits < 16
    bool v_blocked;                // tile records + blocked value layout (K and V quantised, G = 32, d = 128; §4)
    size_t row_k, row_v;           // bytes per token row
    size_t kc, km, kr, vc, vm, vr; // bytes per (b,h) slice
    // tile records (v_blocked): k_codes holds cap/32 records of `rec` bytes, record j = block j as
    // [K code rows | K meta (at rec_km: KIVI block words, or per-token rows of 4 words) | V codes, blocked
    // (at rec_vc) | V meta (at rec_vm)]
    size_t rec;
    uint32_t rec_km, rec_vc, rec_vm;
};
// Fills g from a cache description; returns KVT_OK or an error status (message set).
int32_t make_geometry(const kvt_layer_spec& s, int B, int H, int d, int cap, Geometry* g);


// ---- launchers (defined in the .cu files) ----
struct CachePtrs {
    uint8_t* k_codes; uint32_t* k_meta; uint16_t* k_resid;
    uint8_t* v_codes; uint32_t* v_meta; uint16_t* v_resid;
    const int32_t* bt;     // paged tile records: block table [B][max_pages] (device), or null (dense)
    int max_pages;
};
int32_t launch_append(const Geometry& g, const CachePtrs& c, const uint16_t* k_new, const uint16_t* v_new,
                      const int64_t strides[3], const int32_t* len_before, const int32_t* n_new,
                      int n_new_max, void* stream);
// out_mode: 0 = final bf16, 1 = final fp32, 2 = partial (m, l, o) fp32 [B][H_q][d+2]
int32_t launch_decode(const Geometry& g, const CachePtrs& c, const uint16_t* q, int H_q,
                      const int32_t* seq_len, int plan_len, float scale, void* out, int out_mode,
                      void* workspace, size_t ws_bytes, void* stream, float* const* push = nullptr, int n_push = 0,
                      bool early = false);
size_t decode_workspace(const Geometry& g, int H_q, int plan_len);
int32_t decode_plan(const Geometry& g, int H_q, int plan_len, int32_t out[4]);
int32_t launch_combine(const float* parts, int n_parts, int B, int H_q, int d, void* out, int out_dtype,
                       void* stream);
int32_t launch_sensitivity(int mode, int G, int R, const uint16_t* q, int H_q, int T_q, int q_pos0,
                           const uint16_t* k, const uint16_t* v, int H_kv, int S, int d, float scale,
                           const kvt_pair* pairs, int n_pairs, kvt_errors* out, void* ws, size_t ws_bytes,
                           void* stream);
size_t sensitivity_workspace(int H_q, int T_q, int H_kv, int S, int d, int G);

}  // namespace kvt

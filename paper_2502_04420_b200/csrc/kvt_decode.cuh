// kvt_decode.cuh — K2 (split-KV decode attention over the packed cache) and K3 (split combine).
//
// Computes Eq. 1 for one decode query per (b, query head) over the dequantised cache
// K_hat, V_hat of Eq. 2 without ever materialising K_hat/V_hat: the packed codes are
// streamed once from HBM, converted to fp32 in registers once per (token, channel) and shared by the
// g query heads of the KV head (GQA, A10), and the scales/zero-points are folded:
//   * KIVI key (per-channel scale s_c, zero z_c per block of G tokens):
//       q.k_hat = sum_c (q_c s_c) code_c + sum_c q_c z_c          -> q' = q * s once per block
//   * per-token key (scale s_j, zero z_j per channel group j):
//       q.k_hat = sum_j s_j (sum_{c in j} q_c code_c) + sum_j z_j (sum_{c in j} q_c)
//   * per-token value: sum_t p_t v_hat_t,c = sum_t (p_t s_t,j) code_t,c + sum_t p_t z_t,j
// with an online softmax in base 2 (exp2 of log2(e)-scaled logits) and a split-KV (flash-decoding)
// reduction across CTAs.
//
// Thread mapping (128 threads = 4 warps per CTA; each warp owns whole 32-token tiles):
//   QK:  lane = (quad = lane/4, cb = lane%4): tokens quad + 8j (j < 4), channels [32cb, 32cb+32);
//        K code rows are read straight from HBM with 8..64-byte vector loads (8 rows per warp
//        instruction, fully coalesced); q' comes from shared memory (padded, conflict-free).
//   PV:  lane = (par = lane/16, c8 = lane%16): tokens of parity par, channels [8c8, 8c8+8);
//        the V tile is staged into shared memory with cp.async while QK runs.
// Code -> float uses the 2^23 "magic number" trick: (word & mask) | 0x4B000000 is the float
// 2^23 + code * 2^p, and one FFMA2 (x * 2^-p - 2^(23-p)) recovers code exactly; all dot-product
// FMAs are paired into Blackwell's fma.rn.f32x2 (FFMA2).
//
// Tokens of the residual (bf16) regions and any tile that is not quantised for both K and V (at most
// 63 tokens per sequence) are the "tail", processed token-by-token by the last split.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kvt_internal.h"

namespace kvt {
namespace dec {

constexpr int D = 128;
constexpr int kThreads = 128;
constexpr int kWarps = 4;
constexpr int kTile = 32;
constexpr int kQStride = 36;       // padded floats per 32-channel block of q / q'
constexpr int kNG = 4;             // max channel groups per row (G = 32)
constexpr unsigned kFull = 0xffffffffu;

// Destinations of a pushed partial (a6 fused exchange, kvt_decode_attention_partial_push): each p[i] is a
// [B][H_q][D + 2] fp32 block, typically this shard's slot of a peer GPU's gathered buffer (NVLink P2P).
constexpr int kMaxPush = 8;
struct PushList {
    float* p[kMaxPush];
    int n;
};
// (m, l, o) of one row element: c == 0 also stores m and l.  Writes to `out` (n == 0) or every push target.
__device__ __forceinline__ void store_partial(const PushList& push, void* out, size_t row, int c, float M, float L,
                                              float ov) {
    const int n = push.n > 0 ? push.n : 1;
    for (int i = 0; i < n; ++i) {
        float* pr = (push.n > 0 ? push.p[i] : reinterpret_cast<float*>(out)) + row * (2 + D);
        if (c == 0) { pr[0] = M; pr[1] = L; }
        pr[2 + c] = ov;
    }
}

struct DecodeArgs {
    Geometry g;
    CachePtrs c;
    const uint16_t* q;
    int H_q, gq;
    const int32_t* seq_len;
    float scale_log2;
    void* out;
    int out_mode;      // 0 final bf16, 1 final fp32, 2 partial (m, l, o) -> out; 3 -> parts (split)
    float* parts;      // [n_split][B][H_q][D + 2] when out_mode == 3
    int n_split;
    int* counters;     // [B][H_kv] split-arrival counters (fused combine), zero between calls; or null
    int final_mode;    // output mode of the fused combine (0, 1 or 2)
    unsigned long long* trace;   // KVT_TRACE builds only: per-CTA (SM, start, end); else null
    int n_cta;         // tensor-core kernel: stream-K CTAs (parts [n_cta][2][8][D + 2], counters [B][H_kv])
    PushList push;     // out_mode 2 with push.n > 0: the partial rows go to every push.p[i] (a6 fused exchange)
    int early;         // 1: the prologue (length scan, q setup) may run before griddepcontrol.wait — only when the
                       // library itself launched the preceding kernel (kvt_append_decode_attention); 0: wait first
    // per-SM plan of the tensor-core kernel (sm_w > 0): on each of the sm_n SMs, slots 0 .. sm_w-1 take whole units
    // and slot sm_w one stream-K piece of the remaining units; sched = its claim counters (zero between calls)
    int sm_w, sm_n;
    int* sched;
    int sm_piece_first;   // per-SM plan: the first CTA to arrive on an SM takes the piece (else the last)
    int sm_drop;       // tests only (KVT_SMPLAN_DROP = k): CTAs with blockIdx % k == 0 leave their item unclaimed
};

// Stream-K cost of one (b, kv head) unit of the tensor-core kernel (kvt_decode_mma.cuh)
struct UnitCost {
    int n_main, tiles, cost;
};
__host__ __device__ inline UnitCost unit_cost(const Geometry& g, int S) {
    const int nqK = nq_key(g.mode, g.kb, g.G, g.R, S);
    const int nqV = nq_per_token(g.vb, g.R, S);
    UnitCost u;
    u.n_main = ((nqK < nqV ? nqK : nqV) / 32) * 32;
    u.tiles = u.n_main / 32;
    u.cost = u.tiles + (S - u.n_main + 7) / 8;
    if (u.cost < 1) u.cost = 1;
    return u;
}

__device__ __forceinline__ float bf2f(uint32_t b16) { return __uint_as_float(b16 << 16); }

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

__device__ __forceinline__ float magic(uint32_t src, uint32_t mask) { return __uint_as_float((src & mask) | 0x4B000000u); }

// Exact code recovery for a pair of magic floats whose codes sit at bit position p (p <= 19).
template <int P>
__device__ __forceinline__ float2 norm2(float2 f) {
    constexpr float sc = 1.0f / (float)(1u << P);
    constexpr float of = -8388608.0f / (float)(1u << P);
    return ffma2(f, make_float2(sc, sc), make_float2(of, of));
}

// ---- raw values of 4 consecutive channels (chunk kk of the lane's 32-channel key block) -----------
// kw: the KB words of one token's 32-channel block.  Returns magic floats (KB < 16: 2^23 + code*2^p,
// p = KB*i for KB in {2,4}, p = 0 for KB = 8) or the bf16 values themselves (KB = 16).
template <int KB>
__device__ __forceinline__ void raw_k(const uint32_t* kw, int kk, float f[4]) {
    if constexpr (KB == 2) {
        uint32_t src = kw[kk >> 2] >> (8 * (kk & 3));
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i] = magic(src, 3u << (2 * i));
    } else if constexpr (KB == 4) {
        uint32_t src = kw[kk >> 1] >> (16 * (kk & 1));
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i] = magic(src, 15u << (4 * i));
    } else if constexpr (KB == 8) {
        uint32_t w = kw[kk];
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i] = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540 + i));
    } else {
        uint32_t w0 = kw[2 * kk], w1 = kw[2 * kk + 1];
        f[0] = __uint_as_float(w0 << 16); f[1] = __uint_as_float(w0 & 0xFFFF0000u);
        f[2] = __uint_as_float(w1 << 16); f[3] = __uint_as_float(w1 & 0xFFFF0000u);
    }
}

template <int KB>
__device__ __forceinline__ float2 norm_k(float2 f, int i) {
    if constexpr (KB == 2) {
        return i == 0 ? norm2<0>(f) : i == 1 ? norm2<2>(f) : i == 2 ? norm2<4>(f) : norm2<6>(f);
    } else if constexpr (KB == 4) {
        return i == 0 ? norm2<0>(f) : i == 1 ? norm2<4>(f) : i == 2 ? norm2<8>(f) : norm2<12>(f);
    } else if constexpr (KB == 8) {
        return norm2<0>(f);
    } else {
        return f;
    }
}

// ---- 8 channels of one value row for the PV lane: returns pairs (channel i, channel i + 4) --------
template <int VB>
__device__ __forceinline__ void load_v8(const uint8_t* vrow, int c8, float2 v[4]) {
    if constexpr (VB == 2) {
        uint32_t w = *reinterpret_cast<const uint16_t*>(vrow + 2 * c8);
        uint32_t hi = w >> 8;
        v[0] = norm2<0>(make_float2(magic(w, 3u), magic(hi, 3u)));
        v[1] = norm2<2>(make_float2(magic(w, 3u << 2), magic(hi, 3u << 2)));
        v[2] = norm2<4>(make_float2(magic(w, 3u << 4), magic(hi, 3u << 4)));
        v[3] = norm2<6>(make_float2(magic(w, 3u << 6), magic(hi, 3u << 6)));
    } else if constexpr (VB == 4) {
        uint32_t w = *reinterpret_cast<const uint32_t*>(vrow + 4 * c8);
        uint32_t hi = w >> 16;
        v[0] = norm2<0>(make_float2(magic(w, 15u), magic(hi, 15u)));
        v[1] = norm2<4>(make_float2(magic(w, 15u << 4), magic(hi, 15u << 4)));
        v[2] = norm2<8>(make_float2(magic(w, 15u << 8), magic(hi, 15u << 8)));
        v[3] = norm2<12>(make_float2(magic(w, 15u << 12), magic(hi, 15u << 12)));
    } else if constexpr (VB == 8) {
        uint2 w = *reinterpret_cast<const uint2*>(vrow + 8 * c8);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            v[i] = norm2<0>(make_float2(__uint_as_float(__byte_perm(w.x, 0x4B000000u, 0x7540 + i)),
                                        __uint_as_float(__byte_perm(w.y, 0x4B000000u, 0x7540 + i))));
    } else {
        uint4 w = *reinterpret_cast<const uint4*>(vrow + 16 * c8);
        v[0] = make_float2(__uint_as_float(w.x << 16), __uint_as_float(w.z << 16));
        v[1] = make_float2(__uint_as_float(w.x & 0xFFFF0000u), __uint_as_float(w.z & 0xFFFF0000u));
        v[2] = make_float2(__uint_as_float(w.y << 16), __uint_as_float(w.w << 16));
        v[3] = make_float2(__uint_as_float(w.y & 0xFFFF0000u), __uint_as_float(w.w & 0xFFFF0000u));
    }
}

// ---- generic per-token dequantisation of 4 channels [4l, 4l+4) (tail path) ------------------------
template <int BITS>
__device__ __forceinline__ void codes4(const uint8_t* row, int lane, uint32_t c[4]) {
    if constexpr (BITS == 2) {
        uint32_t w = row[lane];
#pragma unroll
        for (int i = 0; i < 4; ++i) c[i] = (w >> (2 * i)) & 3u;
    } else if constexpr (BITS == 4) {
        uint32_t w = reinterpret_cast<const uint16_t*>(row)[lane];
#pragma unroll
        for (int i = 0; i < 4; ++i) c[i] = (w >> (4 * i)) & 15u;
    } else if constexpr (BITS == 8) {
        uint32_t w = reinterpret_cast<const uint32_t*>(row)[lane];
#pragma unroll
        for (int i = 0; i < 4; ++i) c[i] = (w >> (8 * i)) & 255u;
    }
}

__device__ __forceinline__ void bf16x4(const uint16_t* p, float x[4]) {
    uint2 w = *reinterpret_cast<const uint2*>(p);
    x[0] = bf2f(w.x & 0xffffu); x[1] = bf2f(w.x >> 16); x[2] = bf2f(w.y & 0xffffu); x[3] = bf2f(w.y >> 16);
}

struct Slice {
    const uint8_t* kc; const uint32_t* km; const uint16_t* kr;
    const uint8_t* vc; const uint32_t* vm; const uint16_t* vr;
    const int32_t* bt = nullptr;   // paged tile records: this sequence's block-table row (kc = pool + h * rec)
    size_t pstride = 0;            // page bytes (H records)
    // tile record j of this (b, h) slice
    __device__ __forceinline__ const uint8_t* recp(int j, const Geometry& g) const {
        return bt ? kc + (size_t)bt[j] * pstride : kc + (size_t)j * g.rec;
    }
};

// REC: tile records (g.rec) — token t's key row and block meta live in record t / 32.
template <int KB, bool KPC, bool REC = false>
__device__ __forceinline__ void tail_k(const Slice& s, const Geometry& g, int t, int nqK, int lane, float x[4]) {
    if (t < nqK) {
        const uint8_t* row = REC ? s.recp(t >> 5, g) + (size_t)(t & 31) * g.row_k
                                 : s.kc + (size_t)t * g.row_k;
        if constexpr (KB == 16) {
            bf16x4(reinterpret_cast<const uint16_t*>(row) + 4 * lane, x);
        } else {
            uint32_t c[4];
            codes4<KB>(row, lane, c);
            if constexpr (KPC) {
                const uint32_t* mb = REC ? reinterpret_cast<const uint32_t*>(s.recp(t >> 5, g) + g.rec_km)
                                         : s.km + (size_t)(t / g.G) * D;
                uint4 m = reinterpret_cast<const uint4*>(mb)[lane];
                uint32_t mm[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) x[i] = fmaf((float)c[i], bf2f(mm[i] & 0xffffu), bf2f(mm[i] >> 16));
            } else {
                const uint32_t* mr = REC ? reinterpret_cast<const uint32_t*>(s.recp(t >> 5, g) + g.rec_km +
                                                                             (size_t)(t & 31) * 16)
                                         : s.km + (size_t)t * (D / g.G);
                uint32_t m = mr[(4 * lane) / g.G];
#pragma unroll
                for (int i = 0; i < 4; ++i) x[i] = fmaf((float)c[i], bf2f(m & 0xffffu), bf2f(m >> 16));
            }
        }
    } else {
        size_t slot = KPC ? (size_t)(t - nqK) : (size_t)(t % g.R);
        bf16x4(s.kr + slot * D + 4 * lane, x);
    }
}

// The 4 codes of chunk (lane / 8, lane % 8) of token t in the blocked value layout;
// blk = the V-code part of token t's tile record.
template <int BITS>
__device__ __forceinline__ void codes4_blk(const uint8_t* blk, int t, int lane, uint32_t c[4]) {
    const int tau = t & 31, gam = lane >> 3, i = lane & 7;
    if constexpr (BITS == 2) {
        const uint32_t w = blk[vblk_off(2, tau, gam, i, 0)];
#pragma unroll
        for (int e = 0; e < 4; ++e) c[e] = (w >> (2 * e)) & 3u;
    } else if constexpr (BITS == 4) {
        const uint32_t w = *reinterpret_cast<const uint16_t*>(blk + vblk_off(4, tau, gam, i, 0));
#pragma unroll
        for (int e = 0; e < 4; ++e) c[e] = (w >> (4 * e)) & 15u;
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) c[e] = blk[vblk_off(8, tau, gam, i, e)];
    }
}

// REC: tile records — token t's value codes (blocked) and meta live in record t / 32 of s.kc.
template <int VB, bool REC = false>
__device__ __forceinline__ void tail_v(const Slice& s, const Geometry& g, int t, int nqV, int lane, float x[4]) {
    if (t < nqV) {
        const uint8_t* row = s.vc + (size_t)t * g.row_v;
        if constexpr (REC && VB != 16) {
            const uint8_t* rec = s.recp(t >> 5, g);
            uint32_t c[4];
            codes4_blk<VB>(rec + g.rec_vc, t, lane, c);
            const uint32_t m = reinterpret_cast<const uint32_t*>(rec + g.rec_vm + (size_t)(t & 31) * 16)[(4 * lane) / g.G];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = fmaf((float)c[i], bf2f(m & 0xffffu), bf2f(m >> 16));
        } else if constexpr (VB == 16) {
            bf16x4(reinterpret_cast<const uint16_t*>(row) + 4 * lane, x);
        } else {
            uint32_t c[4];
            codes4<VB>(row, lane, c);
            uint32_t m = s.vm[(size_t)t * (D / g.G) + (4 * lane) / g.G];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = fmaf((float)c[i], bf2f(m & 0xffffu), bf2f(m >> 16));
        }
    } else {
        bf16x4(s.vr + (size_t)(t % g.R) * D + 4 * lane, x);
    }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) {
    return __ldg(p);
}

// Shared-memory plan (floats unless noted):
//   q_s    [GM][4][36]                 query (fp32), padded per 32-channel block
//   qsum_s [GM][4]                     per-block sums of q (per-token key)
//   per warp:
//     qp_s   [GM][4][36]               q' = q * s_blk (KIVI key)
//     w_s    [32][kNG][GM]             p_t * s_v(t, group)
//     z_s    [kNG][GM][32]             per-lane running sum of p_t * z_v(t, group)
//     v_s    u8 [32][16 * VB]          staged value codes of the tile
//   comb   aliases the per-warp area at the end: [4][GM][2 + D]
template <int GM, int VB>
struct Smem {
    static constexpr int q = GM * 4 * kQStride;
    static constexpr int qsum = GM * 4;
    static constexpr int qp = GM * 4 * kQStride;
    static constexpr int w = kTile * kNG * GM;
    static constexpr int z = kNG * GM * 32;
    static constexpr int vbytes = kTile * 16 * VB;
    static constexpr int warp_floats = qp + w + z + vbytes / 4;
    static constexpr int comb = kWarps * GM * (2 + D);
    static constexpr int per_warp_total = kWarps * warp_floats > comb ? kWarps * warp_floats : comb;
    static constexpr size_t bytes = (size_t)(q + qsum + per_warp_total) * 4;
};

template <int KB, int VB, bool KPC, int GM>
__global__ void __launch_bounds__(kThreads) decode_kernel(DecodeArgs a) {
    using SM = Smem<GM, VB>;
    extern __shared__ __align__(16) float smem[];
    float* q_s = smem;
    float* qsum_s = q_s + SM::q;
    float* warp_base = qsum_s + SM::qsum;

    const Geometry& g = a.g;
    const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = a.seq_len[b];
    const int gq = a.gq;

    float* qp_s = warp_base + warp * SM::warp_floats;
    float* w_s = qp_s + SM::qp;
    float* z_s = w_s + SM::w;
    uint8_t* v_s = reinterpret_cast<uint8_t*>(z_s + SM::z);

    // ---- q -> shared (fp32, padded), zero for padded heads ----
    {
        const uint16_t* qg = a.q + ((size_t)b * a.H_q + (size_t)hk * gq) * D;
        for (int h = 0; h < GM; ++h) {
            float v = h < gq ? bf2f(qg[(size_t)h * D + tid]) : 0.0f;
            q_s[(h * 4 + (tid >> 5)) * kQStride + (tid & 31)] = v;
        }
    }
    __syncthreads();
    if (!KPC && KB != 16) {
        if (tid < GM * 4) {
            const float* src = q_s + tid * kQStride;
            float s = 0.0f;
            for (int c = 0; c < 32; ++c) s += src[c];
            qsum_s[tid] = s;
        }
        __syncthreads();
    }

    const size_t bh = (size_t)b * g.H + hk;
    Slice sl;
    sl.kc = a.c.k_codes + bh * g.kc;
    sl.km = g.km ? a.c.k_meta + bh * (g.km / 4) : nullptr;
    sl.kr = g.kr ? a.c.k_resid + bh * (g.kr / 2) : nullptr;
    sl.vc = a.c.v_codes + bh * g.vc;
    sl.vm = g.vm ? a.c.v_meta + bh * (g.vm / 4) : nullptr;
    sl.vr = g.vr ? a.c.v_resid + bh * (g.vr / 2) : nullptr;

    const int nqK = nq_key(g.mode, g.kb, g.G, g.R, S);
    const int nqV = nq_per_token(g.vb, g.R, S);
    const int n_main = ((nqK < nqV ? nqK : nqV) / kTile) * kTile;
    const int n_tiles = n_main / kTile;
    const int tps = (n_tiles + a.n_split - 1) / a.n_split;
    const int tile_lo = split * tps;
    const int tile_hi = (tile_lo + tps < n_tiles) ? tile_lo + tps : n_tiles;

    // ---- running state (per warp): m (uniform), l partial (per lane), o pairs (per lane) ----
    float m_run[GM], l_part[GM];
    float2 o2[GM][4];
#pragma unroll
    for (int h = 0; h < GM; ++h) {
        m_run[h] = -INFINITY;
        l_part[h] = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) o2[h][i] = make_float2(0.0f, 0.0f);
    }
    for (int i = lane; i < kNG * GM * 32; i += 32) z_s[i] = 0.0f;

    // ---- tail tokens [n_main, S): last split, token-at-a-time, lane = channels [4l, 4l+4) ----
    if (split == a.n_split - 1 && n_main < S) {
        float qv[GM][4];
#pragma unroll
        for (int h = 0; h < GM; ++h) {
            float4 t4 = *reinterpret_cast<const float4*>(q_s + (h * 4 + (lane >> 3)) * kQStride + 4 * (lane & 7));
            qv[h][0] = t4.x; qv[h][1] = t4.y; qv[h][2] = t4.z; qv[h][3] = t4.w;
        }
        float mt[GM], lt[GM], ot[GM][4];
#pragma unroll
        for (int h = 0; h < GM; ++h) {
            mt[h] = -INFINITY; lt[h] = 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) ot[h][i] = 0.0f;
        }
        for (int t = n_main + warp; t < S; t += kWarps) {
            float kx[4], vx[4];
            tail_k<KB, KPC>(sl, g, t, nqK, lane, kx);
            tail_v<VB>(sl, g, t, nqV, lane, vx);
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                float s = qv[h][0] * kx[0] + qv[h][1] * kx[1] + qv[h][2] * kx[2] + qv[h][3] * kx[3];
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
                s *= a.scale_log2;
                float mn = fmaxf(mt[h], s);
                float al = exp2f(mt[h] - mn);
                float p = exp2f(s - mn);
                lt[h] = lt[h] * al + p;
#pragma unroll
                for (int i = 0; i < 4; ++i) ot[h][i] = ot[h][i] * al + p * vx[i];
                mt[h] = mn;
            }
        }
        // hand the tail state to the tile-state layout (parity-0 lanes own channels 8c8 + {i, i+4})
        const int c8 = lane & 15;
#pragma unroll
        for (int h = 0; h < GM; ++h) {
            m_run[h] = mt[h];
            l_part[h] = lane == 0 ? lt[h] : 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float lo = __shfl_sync(kFull, ot[h][i], 2 * c8);
                float hi = __shfl_sync(kFull, ot[h][i], 2 * c8 + 1);
                o2[h][i] = lane < 16 ? make_float2(lo, hi) : make_float2(0.0f, 0.0f);
            }
        }
    }
    __syncwarp();

    // ---- main loop over this warp's 32-token tiles ----
    const int quad = lane >> 2, cb = lane & 3;
    const int par = lane >> 4, c8 = lane & 15;
    const int gpr = D / g.G;                       // groups per row
    const int gk = (cb * 32) / g.G;                // key group of the lane's QK block (per-token)
    const int gv = (c8 * 8) / g.G;                 // value group of the lane's PV channels
    constexpr int KW = KB;                         // 32-bit words per (token, 32-channel block)
    constexpr int VROW = 16 * VB;                  // bytes per value row

    for (int tile = tile_lo + warp; tile < tile_hi; tile += kWarps) {
        const int t0 = tile * kTile;
        // (A) stage the value tile (contiguous rows t0..t0+31) with cp.async
        {
            const uint8_t* src = sl.vc + (size_t)t0 * VROW;
#pragma unroll
            for (int i = 0; i < VB; ++i) cp_async16(v_s + (i * 32 + lane) * 16, src + (i * 32 + lane) * 16);
            cp_async_commit();
        }
        // (B) key codes: 4 tokens x (32 channels x KB bits) per lane
        uint32_t kw[4][KW];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint8_t* row = sl.kc + (size_t)(t0 + quad + 8 * j) * g.row_k + cb * (4 * KB);
            if constexpr (KW == 2) {
                uint2 v = ldg_stream(reinterpret_cast<const uint2*>(row));
                kw[j][0] = v.x; kw[j][1] = v.y;
            } else {
#pragma unroll
                for (int u = 0; u < KW / 4; ++u) {
                    uint4 v = ldg_stream(reinterpret_cast<const uint4*>(row) + u);
                    kw[j][4 * u] = v.x; kw[j][4 * u + 1] = v.y; kw[j][4 * u + 2] = v.z; kw[j][4 * u + 3] = v.w;
                }
            }
        }
        // (C) key scale folding
        float bias[GM];
        const float* qsrc = q_s;
        float2 ks[2], kz[2];   // per-token key scale / zero (per-token mode), pairs (token 2jp, 2jp+1)
        if constexpr (KPC) {
            const int blk = t0 / g.G;
            uint4 mm = ldg_stream(reinterpret_cast<const uint4*>(sl.km + (size_t)blk * D) + lane);
            uint32_t mw[4] = {mm.x, mm.y, mm.z, mm.w};
            const int c0 = 4 * lane;           // channels c0..c0+3: block c0/32, offset c0%32
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                float4 qv = *reinterpret_cast<const float4*>(q_s + (h * 4 + (c0 >> 5)) * kQStride + (c0 & 31));
                float4 qp;
                qp.x = qv.x * bf2f(mw[0] & 0xffffu); qp.y = qv.y * bf2f(mw[1] & 0xffffu);
                qp.z = qv.z * bf2f(mw[2] & 0xffffu); qp.w = qv.w * bf2f(mw[3] & 0xffffu);
                *reinterpret_cast<float4*>(qp_s + (h * 4 + (c0 >> 5)) * kQStride + (c0 & 31)) = qp;
                float bz = qv.x * bf2f(mw[0] >> 16) + qv.y * bf2f(mw[1] >> 16) + qv.z * bf2f(mw[2] >> 16) +
                           qv.w * bf2f(mw[3] >> 16);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) bz += __shfl_xor_sync(kFull, bz, off);
                bias[h] = bz;
            }
            __syncwarp();
            qsrc = qp_s;
        } else {
#pragma unroll
            for (int h = 0; h < GM; ++h) bias[h] = 0.0f;
            if constexpr (KB != 16) {
                uint32_t m[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) m[j] = ldg_stream(sl.km + (size_t)(t0 + quad + 8 * j) * gpr + gk);
#pragma unroll
                for (int jp = 0; jp < 2; ++jp) {
                    ks[jp] = make_float2(bf2f(m[2 * jp] & 0xffffu), bf2f(m[2 * jp + 1] & 0xffffu));
                    kz[jp] = make_float2(bf2f(m[2 * jp] >> 16), bf2f(m[2 * jp + 1] >> 16));
                }
            }
        }
        // (D) QK: acc[jp][h] = (partial logit of token 2jp, token 2jp+1) over the lane's 32 channels
        float2 acc[2][GM];
#pragma unroll
        for (int jp = 0; jp < 2; ++jp)
#pragma unroll
            for (int h = 0; h < GM; ++h) acc[jp][h] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            float2 kf[2][4];
#pragma unroll
            for (int jp = 0; jp < 2; ++jp) {
                float fa[4], fb[4];
                raw_k<KB>(kw[2 * jp], kk, fa);
                raw_k<KB>(kw[2 * jp + 1], kk, fb);
#pragma unroll
                for (int i = 0; i < 4; ++i) kf[jp][i] = norm_k<KB>(make_float2(fa[i], fb[i]), i);
            }
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                float4 q4 = *reinterpret_cast<const float4*>(qsrc + (h * 4 + cb) * kQStride + 4 * kk);
#pragma unroll
                for (int jp = 0; jp < 2; ++jp) {
                    acc[jp][h] = ffma2(kf[jp][0], make_float2(q4.x, q4.x), acc[jp][h]);
                    acc[jp][h] = ffma2(kf[jp][1], make_float2(q4.y, q4.y), acc[jp][h]);
                    acc[jp][h] = ffma2(kf[jp][2], make_float2(q4.z, q4.z), acc[jp][h]);
                    acc[jp][h] = ffma2(kf[jp][3], make_float2(q4.w, q4.w), acc[jp][h]);
                }
            }
        }
        // (E) per-token key: s_j * dot + z_j * sum(q over the block)
        if constexpr (!KPC && KB != 16) {
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                float qs = qsum_s[h * 4 + cb];
#pragma unroll
                for (int jp = 0; jp < 2; ++jp)
                    acc[jp][h] = ffma2(acc[jp][h], ks[jp], make_float2(kz[jp].x * qs, kz[jp].y * qs));
            }
        }
        // (F) reduce the 4 channel blocks of each token (lanes of a quad)
#pragma unroll
        for (int jp = 0; jp < 2; ++jp)
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                acc[jp][h].x += __shfl_xor_sync(kFull, acc[jp][h].x, 1);
                acc[jp][h].y += __shfl_xor_sync(kFull, acc[jp][h].y, 1);
                acc[jp][h].x += __shfl_xor_sync(kFull, acc[jp][h].x, 2);
                acc[jp][h].y += __shfl_xor_sync(kFull, acc[jp][h].y, 2);
            }
        // (G, H) log2-domain logits, tile max, online-softmax rescale
        float alpha[GM], p[GM];
#pragma unroll
        for (int h = 0; h < GM; ++h) {
            float s0 = (acc[0][h].x + bias[h]) * a.scale_log2;
            float s1 = (acc[0][h].y + bias[h]) * a.scale_log2;
            float s2 = (acc[1][h].x + bias[h]) * a.scale_log2;
            float s3 = (acc[1][h].y + bias[h]) * a.scale_log2;
            float mx = fmaxf(fmaxf(s0, s1), fmaxf(s2, s3));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 16));
            float mnew = fmaxf(m_run[h], mx);
            alpha[h] = exp2f(m_run[h] - mnew);
            m_run[h] = mnew;
            // (I) the lane's own token is quad + 8*cb  (j = cb)
            float sown = cb == 0 ? s0 : cb == 1 ? s1 : cb == 2 ? s2 : s3;
            p[h] = exp2f(sown - mnew);
            l_part[h] = l_part[h] * alpha[h] + p[h];    // (J)
        }
        // (K) value scale folding for the lane's own token
        {
            const int tl = quad + 8 * cb;
            float* wrow = w_s + tl * (kNG * GM);
            if constexpr (VB == 16) {
#pragma unroll
                for (int h = 0; h < GM; ++h) wrow[h] = p[h];
            } else {
                const uint32_t* vmrow = sl.vm + (size_t)(t0 + tl) * gpr;
                for (int j = 0; j < gpr; ++j) {
                    uint32_t m = ldg_stream(vmrow + j);
                    float sv = bf2f(m & 0xffffu), zv = bf2f(m >> 16);
#pragma unroll
                    for (int h = 0; h < GM; ++h) {
                        wrow[j * GM + h] = p[h] * sv;
                        float* zp = z_s + (j * GM + h) * 32 + lane;
                        *zp = *zp * alpha[h] + p[h] * zv;
                    }
                }
            }
        }
        cp_async_wait_all();
        __syncwarp();
        // (M) PV over the 16 tokens of the lane's parity
#pragma unroll
        for (int h = 0; h < GM; ++h)
#pragma unroll
            for (int i = 0; i < 4; ++i) o2[h][i] = fmul2(o2[h][i], make_float2(alpha[h], alpha[h]));
#pragma unroll 4
        for (int tt = 0; tt < 16; ++tt) {
            const int tl = 2 * tt + par;
            float2 v[4];
            load_v8<VB>(v_s + tl * VROW, c8, v);
            const float* wr = w_s + tl * (kNG * GM) + (VB == 16 ? 0 : gv * GM);
#pragma unroll
            for (int h = 0; h < GM; h += 4) {
                float4 w4 = *reinterpret_cast<const float4*>(wr + h);
                float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int u = 0; u < 4 && h + u < GM; ++u)
#pragma unroll
                    for (int i = 0; i < 4; ++i) o2[h + u][i] = ffma2(v[i], make_float2(wv[u], wv[u]), o2[h + u][i]);
            }
        }
        __syncwarp();
    }

    // ---- warp epilogue: merge parities, l, zero-point sums; write the warp state ----
    float l_w[GM];
#pragma unroll
    for (int h = 0; h < GM; ++h) {
        float l = l_part[h];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) l += __shfl_xor_sync(kFull, l, off);
        l_w[h] = l;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            o2[h][i].x += __shfl_xor_sync(kFull, o2[h][i].x, 16);
            o2[h][i].y += __shfl_xor_sync(kFull, o2[h][i].y, 16);
        }
    }
    float zf[GM];
#pragma unroll
    for (int h = 0; h < GM; ++h) {
        float z = 0.0f;
        if (VB != 16) {
            const float* zp = z_s + (gv * GM + h) * 32;
            for (int i = 0; i < 32; ++i) z += zp[i];
        }
        zf[h] = z;
    }
    __syncthreads();                      // every warp is done with its per-warp area
    float* comb = warp_base;              // [4][GM][2 + D]
    {
        float* cw = comb + warp * GM * (2 + D);
        if (lane < 16) {
#pragma unroll
            for (int h = 0; h < GM; ++h) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    cw[h * (2 + D) + 2 + 8 * c8 + i] = o2[h][i].x + zf[h];
                    cw[h * (2 + D) + 2 + 8 * c8 + i + 4] = o2[h][i].y + zf[h];
                }
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int h = 0; h < GM; ++h) { cw[h * (2 + D)] = m_run[h]; cw[h * (2 + D) + 1] = l_w[h]; }
        }
    }
    __syncthreads();
    // ---- CTA combine over the 4 warps: thread = channel ----
    const int c = tid;
    for (int h = 0; h < gq; ++h) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, comb[(w * GM + h) * (2 + D)]);
        float L = 0.0f, O = 0.0f;
        if (M != -INFINITY) {
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const float* cw = comb + (w * GM + h) * (2 + D);
                float sc = exp2f(cw[0] - M);
                L += cw[1] * sc;
                O += cw[2 + c] * sc;
            }
        }
        const size_t row = (size_t)b * a.H_q + (size_t)hk * gq + h;
        if (a.out_mode == 3) {
            float* pr = a.parts + ((size_t)split * g.B * a.H_q + row) * (2 + D);
            if (c == 0) { pr[0] = M; pr[1] = L; }
            pr[2 + c] = L > 0.0f ? __fdiv_rn(O, L) : 0.0f;
        } else if (a.out_mode == 2) {
            store_partial(a.push, a.out, row, c, M, L, L > 0.0f ? __fdiv_rn(O, L) : 0.0f);
        } else {
            float o = L > 0.0f ? __fdiv_rn(O, L) : 0.0f;
            if (a.out_mode == 1) reinterpret_cast<float*>(a.out)[row * D + c] = o;
            else reinterpret_cast<__nv_bfloat16*>(a.out)[row * D + c] = __float2bfloat16_rn(o);
        }
    }
}

}  // namespace dec
}  // namespace kvt

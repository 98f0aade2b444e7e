// kvt_decode_mma.cuh — K2 fast path: KIVI decode attention with both dot products on the tensor
// cores (mma.sync m16n8k16, fp16 operands, fp32 accumulation) — DESIGN.md §5.
//
// Why tensor cores on an HBM-bound kernel: with GQA (g = 4..8 query heads per KV head) and 2..4-bit
// codes the CUDA-core form needs ~1k lane-instructions per (token, KV head) (2·g·d FMAs plus code
// conversion) and ncu showed it issue-limited far below the HBM roofline.  Here the FMAs become
// 1-2 HMMA per 16 tokens; what remains per code is about one LOP3.
//
// Operands (all products exact, fp32 accumulation):
//   * A = the integer codes as fp16 *subnormals*: (word & mask) read as a half is code · 2^(p-24)
//     where p is the bit position of the code inside its 16-bit half; no conversion instruction is
//     needed.  The 2^(p-24) is undone exactly: per k-slot in B (QK) or per output row (PV).
//   * B (QK) = q·s (the KIVI per-channel key scale of the block) times powers of two, split
//     exactly into fp16 hi + lo (q and s are bf16 = 8 significant bits, so q·s has <= 16 bits); with
//     g <= 4 the hi and lo halves share one N = 8 MMA.
//   * B (PV) = p·s_v (probability times the per-token value scale) in fp16 times a power of two that
//     only decreases along the sequence: relative rounding 2^-12 per weight.
//   * zero-points in fp32: bias_h = sum_c q_c z_c per key block, sum_t p_t z_(t,group) per value group.
//
// Work: a CTA takes whole (b, kv head) units, or stream-K shares of the flattened tile space (fused merge
// of cut units); its 4 warps take the unit's 32-token tiles (= KIVI key blocks, G = 32) round-robin, each
// fed by its own 2-stage ring of TMA bulk copies of the tile records (K rows | K block meta | blocked V |
// V meta); the bf16 tail tokens are staged the same way and done first, on CUDA cores.
// Thread (gid = lane/4, tig = lane%4):
//   QK  m-tile = 16 tokens (rows gid, gid+8), n = 8 (heads, or 4 heads x {hi, lo}), k = 16 channels;
//       thread tig owns the 32-channel block [32 tig, 32 tig + 32) of each row (one LDS.128 at 4 bits).
//   PV  m-tile = 16 channels of ONE value group γ (so the per-token value scale folds into B), n = 8
//       heads, k = 16 tokens ordered in pairs (T, T+8); thread gid owns channels 32γ + 4gid + {0..3}.
#pragma once
#include <cuda_fp16.h>

#include "kvt_decode.cuh"

namespace kvt {
namespace mma {

using dec::DecodeArgs;
using dec::Slice;
using dec::bf2f;
using dec::kFull;
using dec::UnitCost;
using dec::unit_cost;
constexpr int D = 128;
constexpr int kTile = 32;
constexpr int kWarps = 4;
constexpr int kThreads = 128;

// an opaque copy: the compiler keeps the value in a register instead of re-deriving it from %tid inside the tile loop
__device__ __forceinline__ int opaque(int x) {
    int y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

// D = A B (zero accumulator: the MMA reads RZ, no register moves to clear a chain's accumulator)
__device__ __forceinline__ void hmma0(float d[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                      uint32_t b1) {
    const float z = 0.0f;
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%10,%10,%10};\n"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(z));
}
__device__ __forceinline__ void hmma(float d[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

#ifndef KVT_TRACE
#define KVT_TRACE 0    // debug builds only: per-CTA (SM, start, end) timestamps for load-balance studies
#endif
#if KVT_TRACE
#define KVT_STAMP(k)                                                                                     \
    do {                                                                                                 \
        if (a.trace && tid == 0 && blockIdx.x < 4096) {                                                  \
            unsigned long long t_;                                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
            unsigned long long* p_ = a.trace + 3 * 4096 + 8 * blockIdx.x + (k);                          \
            if (*p_ == 0ull) *p_ = t_;                                                                   \
        }                                                                                                \
    } while (0)
#else
#define KVT_STAMP(k) do { } while (0)
#endif
#ifndef KVT_COLS
#define KVT_COLS 1     // g <= 4: QK columns (head h hi, head h lo) adjacent, one softmax head per lane
#endif
#ifndef KVT_EXP
#define KVT_EXP 0      // profiling experiments only: 1 = skip PV, 2 = skip QK, 3 = both, 4 = stream tiles only, 5 = no tail,
                       // 6 = PV operands staged to shared memory instead of HMMA (tcgen05 cost probe)
#endif
// 2^x on the SFU (MUFU.EX2, flush-to-zero). exp2f adds a subnormal range fix-up (~4 more instructions) that
// softmax does not need: every argument here is <= 8 and results below 2^-126 are negligible against l >= 1.
__device__ __forceinline__ float fexp2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// x = f 2^e, f in [0.5, 1), e clamped to [-119, 90] (subnormal x: -119).  Every power of two the kernel derives
// from it (2^(7-e), 2^(e-7), 2^(17+e), 2^(24-6-(7-e)) ...) is then a normal fp32, so scales anywhere in bf16's
// range down to its subnormals normalise without underflow (values above 2^90 are outside the supported range).
__device__ __forceinline__ int frexp_e(float x) {
    const int e = x > 0.0f ? (int)((__float_as_uint(x) >> 23) & 0xFF) - 126 : 0;
    return e < -119 ? -119 : (e > 90 ? 90 : e);
}
__device__ __forceinline__ float pow2(int e) { return __uint_as_float((uint32_t)(127 + e) << 23); }

// ---- QK A operand: thread tig's 32-channel key block -> 16 fp16-subnormal pairs ("slots") ----------
// Slot m holds channels (c0(m), c1(m)) of the block at bit position P(m) inside each half; k-step s of
// the MMA uses slots 2s (A columns 2tig, 2tig+1) and 2s+1 (A columns 2tig+8, 2tig+9).
template <int KB>
struct KSlots {
    __host__ __device__ static constexpr int c0(int m) {
        return KB == 4 ? 8 * (m >> 2) + (m & 3)
                       : (KB == 2 ? 16 * (m >> 3) + ((m & 7) < 4 ? 0 : 4) + (m & 3) : 4 * (m >> 1) + 2 * (m & 1));
    }
    __host__ __device__ static constexpr int c1(int m) { return c0(m) + (KB == 4 ? 4 : (KB == 2 ? 8 : 1)); }
    __host__ __device__ static constexpr int P(int m) { return KB == 4 ? 4 * (m & 1) : (KB == 2 ? 2 * (m & 3) : 0); }
};

template <int KB>
__device__ __forceinline__ uint32_t k_slot(const uint32_t* w, int m) {
    if constexpr (KB == 4) {
        const uint32_t src = (m & 2) ? w[m >> 2] >> 8 : w[m >> 2];
        return src & ((m & 1) ? 0x00F000F0u : 0x000F000Fu);
    } else if constexpr (KB == 2) {
        const uint32_t src = (m & 4) ? w[m >> 3] >> 8 : w[m >> 3];
        return src & (0x00030003u << (2 * (m & 3)));
    } else {
        return __byte_perm(w[m >> 1], 0u, (m & 1) ? 0x4342 : 0x4140);
    }
}

// Per-token keys (KPT): the scale and zero-point change per (token, 32-channel group), so k-steps must be
// group-pure.  Slot m of lane tig holds two channels of group g = m / 4: k-steps 2g and 2g+1 then cover
// group g alone and their accumulators are folded with that group's per-token scale.  Lane tig reads its
// share of every group: K4 word tig of the group, K2 the (tig & 1) half of word tig / 2, K8 words 2tig, 2tig+1.
template <int KB>
struct KSlotsPT {
    __host__ __device__ static constexpr int c0(int m, int tig) {
        return KB == 4 ? 32 * (m >> 2) + 8 * tig + (m & 3)
                       : (KB == 2 ? 32 * (m >> 2) + 16 * (tig >> 1) + 4 * (tig & 1) + (m & 3)
                                  : 32 * (m >> 2) + 8 * tig + 4 * ((m & 3) >> 1) + 2 * (m & 1));
    }
    __host__ __device__ static constexpr int c1(int m, int tig) { return c0(m, tig) + (KB == 4 ? 4 : (KB == 2 ? 8 : 1)); }
    __host__ __device__ static constexpr int P(int m) { return KB == 4 ? 4 * (m & 1) : (KB == 2 ? 2 * (m & 3) : 0); }
};
// w[] = the lane's words, group-major (K4: w[g]; K2: w[g] (shift by 8 for odd tig); K8: w[2g], w[2g+1])
template <int KB>
__device__ __forceinline__ uint32_t k_slot_pt(const uint32_t* w, int m, int tig) {
    if constexpr (KB == 2) {
        const uint32_t src = (tig & 1) ? w[m >> 2] >> 8 : w[m >> 2];
        return src & (0x00030003u << (2 * (m & 3)));
    } else {
        return k_slot<KB>(w, m);              // K4: w[m >> 2] (shift for m & 2); K8: byte pairs of w[m >> 1]
    }
}

// Inverse of KSlots: channel offset cc in [0, 32) -> slot * 2 + half
template <int KB>
__device__ __forceinline__ int k_slot_of(int cc) {
    if constexpr (KB == 4) {
        const int w = cc >> 3, i = cc & 7;
        return ((4 * w + (i & 3)) << 1) | (i >> 2);
    } else if constexpr (KB == 2) {
        const int w = cc >> 4, i = cc & 15;
        return ((8 * w + 4 * ((i >> 2) & 1) + (i & 3)) << 1) | (i >> 3);
    } else {
        const int w = cc >> 2, i = cc & 3;
        return ((2 * w + (i >> 1)) << 1) | (i & 1);
    }
}

// ---- PV A operand from the blocked value layout ----------------------------------------
// For k-step ks and the thread's two token pairs (T, T+8), T = 16ks + tig and T = 16ks + tig + 4, the
// codes of channels 32γ + 4gid + e (e < 4) of all 4 groups are one or two LDS.128:
//   hA[γ][e] = (code(T, e), code(T+8, e)), hB[γ][e] = the same for T + 4 — fp16 subnormals · 2^(VP(e)-24).
template <int VB>
__host__ __device__ constexpr int VP(int e) { return VB == 4 ? 4 * (e & 1) : (VB == 2 ? 2 * e : 0); }

template <int VB>
struct VRaw {                                  // the raw blocked words of one k-step
    uint32_t a[VB == 8 ? 8 : 4], b[VB == 2 ? 1 : (VB == 8 ? 8 : 4)];
};

template <int VB>
__device__ __forceinline__ void v_load(const uint8_t* vblk, int ks, int tig, int gid, VRaw<VB>& r) {
    // uint4 index ((ks*2 + j/4)*8 + gid)*4 + j%4 (token pair j): the 8 lanes of each LDS.128 phase read 128
    // consecutive bytes, so the loads are free of bank conflicts
    const uint4* w4 = reinterpret_cast<const uint4*>(vblk);
    if constexpr (VB == 4) {
        // word = [tok 16ks+j (16 bits) | tok 16ks+j+8 (16 bits)] of the 4 groups, j = tig (a) and tig + 4 (b)
        const uint4 a = w4[((ks * 2) * 8 + gid) * 4 + tig], b = w4[((ks * 2 + 1) * 8 + gid) * 4 + tig];
        r.a[0] = a.x; r.a[1] = a.y; r.a[2] = a.z; r.a[3] = a.w;
        r.b[0] = b.x; r.b[1] = b.y; r.b[2] = b.z; r.b[3] = b.w;
    } else if constexpr (VB == 2) {
        // word ((ks*8 + gid)*4 + j)*4 + γ = bytes [tok j, tok j+4, tok j+8, tok j+12] (+16ks), j = tig
        const uint4 a = w4[(ks * 8 + gid) * 4 + tig];
        r.a[0] = a.x; r.a[1] = a.y; r.a[2] = a.z; r.a[3] = a.w;
    } else {
        // uint4 (((ks*2 + j/4)*2 + γ/2)*8 + gid)*4 + j%4 = words [γ][c pair] = [T.c0, T8.c0, T.c1, T8.c1], [T.c2, ..]
        const uint4 a0 = w4[(((ks * 2) * 2) * 8 + gid) * 4 + tig], a1 = w4[(((ks * 2) * 2 + 1) * 8 + gid) * 4 + tig];
        const uint4 b0 = w4[(((ks * 2 + 1) * 2) * 8 + gid) * 4 + tig], b1 = w4[(((ks * 2 + 1) * 2 + 1) * 8 + gid) * 4 + tig];
        r.a[0] = a0.x; r.a[1] = a0.y; r.a[2] = a0.z; r.a[3] = a0.w; r.a[4] = a1.x; r.a[5] = a1.y; r.a[6] = a1.z; r.a[7] = a1.w;
        r.b[0] = b0.x; r.b[1] = b0.y; r.b[2] = b0.z; r.b[3] = b0.w; r.b[4] = b1.x; r.b[5] = b1.y; r.b[6] = b1.z; r.b[7] = b1.w;
    }
}

// hA[e] = (code(T, e), code(T+8, e)), hB[e] = the same for T + 4, of group g4 — fp16 subnormals
template <int VB>
__device__ __forceinline__ void v_frag(const VRaw<VB>& r, int g4, uint32_t hA[4], uint32_t hB[4]) {
    if constexpr (VB == 4) {
        const uint32_t xa = r.a[g4], xb = r.b[g4], xa8 = xa >> 8, xb8 = xb >> 8;
        hA[0] = xa & 0x000F000Fu; hA[1] = xa & 0x00F000F0u; hA[2] = xa8 & 0x000F000Fu; hA[3] = xa8 & 0x00F000F0u;
        hB[0] = xb & 0x000F000Fu; hB[1] = xb & 0x00F000F0u; hB[2] = xb8 & 0x000F000Fu; hB[3] = xb8 & 0x00F000F0u;
    } else if constexpr (VB == 2) {
        const uint32_t x = r.a[g4], x8 = x >> 8;
#pragma unroll
        for (int e = 0; e < 4; ++e) { hA[e] = x & (0x00030003u << (2 * e)); hB[e] = x8 & (0x00030003u << (2 * e)); }
    } else {
        hA[0] = __byte_perm(r.a[2 * g4], 0u, 0x4140); hA[1] = __byte_perm(r.a[2 * g4], 0u, 0x4342);
        hA[2] = __byte_perm(r.a[2 * g4 + 1], 0u, 0x4140); hA[3] = __byte_perm(r.a[2 * g4 + 1], 0u, 0x4342);
        hB[0] = __byte_perm(r.b[2 * g4], 0u, 0x4140); hB[1] = __byte_perm(r.b[2 * g4], 0u, 0x4342);
        hB[2] = __byte_perm(r.b[2 * g4 + 1], 0u, 0x4140); hB[3] = __byte_perm(r.b[2 * g4 + 1], 0u, 0x4342);
    }
}

// NC weight tile (g <= 4): the PV B operand of k-step ks, token pair j (tokens 16 ks + j, + 8) and head n is the word
// wt_idx(ks, j, n) + group; o(j) = 4 (j & 1) + (j & 2) skews the heads so that the 8 lanes of every STS.128 (writer:
// j = gid, n = tig) and every LDS.128 (reader: j = tig or tig + 4, n = gid) phase hit distinct 16-byte bank groups.
__device__ __forceinline__ int wt_idx(int ks, int j, int n) { return ((ks * 8 + j) * 8 + ((n + 4 * (j & 1) + (j & 2)) & 7)) * 4; }

// Output row writer: mode 0 bf16, 1 fp32 (o = O / L), 2 partial (m, l, o).
__device__ __forceinline__ void write_row(const DecodeArgs& a, void* out, int mode, size_t row, int c, float M, float L,
                                          float O) {
    const float ov = L > 0.0f ? __fdiv_rn(O, L) : 0.0f;
    if (mode == 2) {
        dec::store_partial(a.push, out, row, c, M, L, ov);
    } else if (mode == 1) {
        reinterpret_cast<float*>(out)[row * D + c] = ov;
    } else {
        reinterpret_cast<__nv_bfloat16*>(out)[row * D + c] = __float2bfloat16_rn(ov);
    }
}

template <int KB, int VB, int GM>
struct Geo {
    static constexpr int KROW = 16 * KB;                 // bytes per key code row
    static constexpr int VROW = 16 * VB;
    static constexpr int K_OFF = 0;                      // stage = [K codes | K block meta | V block | V meta]
    static constexpr int KM_OFF = K_OFF + kTile * KROW;
    static constexpr int V_OFF = KM_OFF + D * 4;
    static constexpr int VM_OFF = V_OFF + kTile * VROW;
    static constexpr int STAGE = VM_OFF + kTile * 16;
#ifndef KVT_NS
#define KVT_NS 2
#endif
    static constexpr int NS = KVT_NS;                    // cp.async ring depth per warp
    // per warp: ring + PV weight tile (half2 [4 γ][2 ks][8 pairs][8 heads]) + key scale slots (half2 [4][16])
    static constexpr int W_OFF = NS * STAGE;
    // half2 [4 γ][2 ks][8 pairs][8 heads], γ >= 2 shifted by 4 words (the tig / tig^2 lanes that store
    // γ and γ + 2 in one STS.64 then hit different banks)
    static constexpr int W_BYTES = 4 * 2 * 8 * 8 * 4 + 16;
    static constexpr int SH_OFF = W_OFF + W_BYTES;
    static constexpr int SH_STRIDE = 20;                          // words per tig row (16 used; padding: no bank conflicts)
    static constexpr int BAR_OFF = SH_OFF + 4 * SH_STRIDE * 4;    // one mbarrier per stage
    static constexpr int WARP_BYTES = (BAR_OFF + 8 * NS + 15) / 16 * 16;
    static constexpr int Q_BYTES = GM * D * 4;           // q fp32 [GM][128]
    static constexpr int TAIL_PART = ((GM * (2 + D) * 4) + 15) / 16 * 16;    // tail partial (m, l, o) [GM]
    static constexpr int TAIL_BYTES = TAIL_PART + 16;                          // + the tail-staging mbarrier
    static constexpr int COMB_BYTES = kWarps * 8 * (2 + D) * 4;
    static constexpr int SCRATCH_BYTES = kWarps * GM * (2 + D) * 4;       // per-warp tail partials
    static constexpr int BODY0 = kWarps * WARP_BYTES > COMB_BYTES ? kWarps * WARP_BYTES : COMB_BYTES;
    static constexpr int BODY = BODY0 > SCRATCH_BYTES ? BODY0 : SCRATCH_BYTES;
    static constexpr size_t SMEM = (size_t)Q_BYTES + TAIL_BYTES + BODY;
};

// ---- TMA bulk copies (cp.async.bulk) completing on a per-stage mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }


// One segment of a (b, kv head) unit: main tiles [tile_lo, tile_hi) (+ the tail tokens [n_main, S) when
// do_tail).  count == 1: the segment is the whole unit and writes the output row; otherwise it leaves a
// partial in parts slot (cta, slot) and the last of the unit's `count` CTAs (c_first ...) merges them.
// GM: 4 (g <= 4: n = 4 heads x {hi, lo}) or 8 (g <= 8: separate hi and lo MMAs).
template <int KB, int VB, int GM, bool KPT, bool PAGED>
__device__ __forceinline__ void segment(const DecodeArgs& a, uint8_t* smem, const int b, const int hk,
                                        const int tile_lo, const int tile_hi, const bool do_tail, const int cta,
                                        const int slot, const int c_first, const int count) {
    using Gm = Geo<KB, VB, GM>;
    // NC (g <= 4): the 8 QK columns are (head 0 hi, head 0 lo, head 1 hi, ...), so a lane's two accumulator
    // columns hold the hi and lo parts of ONE head (tig): the fold is one add, no shuffle, and each lane runs the
    // softmax of one head (no duplicated work).  The weights go to the PV B tile as [ks][token pair][head][group]
    // words, read back with one LDS.128 per (k-step, pair) — see `wt_idx`.
    constexpr bool NC = (GM == 4) && KVT_COLS;
    constexpr int JH = NC ? 1 : 2;                                         // softmax heads per lane
    float* q_s = reinterpret_cast<float*>(smem);                           // [GM][128]
    float* tail_s = reinterpret_cast<float*>(smem + Gm::Q_BYTES);          // [GM][2 + D]
    uint8_t* body = smem + Gm::Q_BYTES + Gm::TAIL_BYTES;
    const Geometry& g = a.g;
    // warp index through a lane-0 shuffle: the compiler then knows it is warp-uniform, so the per-warp TMA
    // addresses live in uniform registers (no per-copy R2UR broadcast loop around UBLKCP)
    const int tid = threadIdx.x, lane = opaque(tid & 31), warp = __shfl_sync(kFull, tid >> 5, 0);
    const int gid = opaque(lane >> 2), tig = opaque(lane & 3);
    const int gq = a.gq;
    const int S = a.seq_len[b];
    KVT_STAMP(0);

    uint8_t* wbase = body + warp * Gm::WARP_BYTES;
    uint32_t* w_s = reinterpret_cast<uint32_t*>(wbase + Gm::W_OFF);        // half2 [4][2][8][8]
    uint32_t* sh_s = reinterpret_cast<uint32_t*>(wbase + Gm::SH_OFF);      // half2 [4 tig][SH_STRIDE]

    {   // q -> shared fp32 (zero for padded heads)
        const uint16_t* qg = a.q + ((size_t)b * a.H_q + (size_t)hk * gq) * D;
        for (int h = 0; h < GM; ++h) q_s[h * D + tid] = h < gq ? bf2f(qg[(size_t)h * D + tid]) : 0.0f;
    }
    for (int i = lane; i < Gm::W_BYTES / 4; i += 32) w_s[i] = 0u;
    __syncthreads();

    const size_t bh = (size_t)b * g.H + hk;
    Slice sl;
    // paged: kc = the pool base of head hk and record j is page bt[b][j] (read from the kernel parameters
    // where used, so the main loop keeps no extra registers)
    sl.kc = PAGED ? a.c.k_codes + (size_t)hk * g.rec : a.c.k_codes + bh * g.kc;
    sl.km = nullptr;                                 // tile records: K meta, V codes and V meta live in kc
    sl.kr = a.c.k_resid + bh * (g.kr / 2);
    sl.vc = nullptr;
    sl.vm = nullptr;
    sl.vr = g.vr ? a.c.v_resid + bh * (g.vr / 2) : nullptr;

    const int nqK = nq_key(g.mode, g.kb, g.G, g.R, S);
    const int nqV = nq_per_token(g.vb, g.R, S);
    const int n_main = ((nqK < nqV ? nqK : nqV) / kTile) * kTile;
    const int n_my = opaque(tile_hi - tile_lo - warp > 0 ? (tile_hi - tile_lo - warp + kWarps - 1) / kWarps : 0);
    // ---- stage the tail rows [n_main, S) into shared memory with bulk copies (one round trip instead of a
    // dependent global load per token group); `tl` then addresses them with the cache's own indexing ----
    // softmax heads of this thread (the QK D columns it holds after the hi/lo fold)
    const int hA = (GM == 8) ? 2 * tig : (NC ? tig : 2 * (tig & 1));
    // ---- per-head power-of-two scale of q (max |q 2^qa| in [64, 128)), computed once per CTA ----
    float* qmax_s = tail_s;                               // tail_s is free until the tail is merged
    if (warp == 0) {
#pragma unroll
        for (int h = 0; h < GM; ++h) {
            const float4 v = *reinterpret_cast<const float4*>(q_s + h * D + 4 * lane);
            float m = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, off));
            if (lane == 0) qmax_s[h] = m;
        }
    }
    __syncthreads();
    uint32_t q_h[16];
    float qa_inv[2];
    {
        const int qh = (GM == 4) ? (NC ? (gid >> 1) : (gid & 3)) : gid;
        const int qa = 7 - frexp_e(qmax_s[qh]);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const float sc = pow2(qa - KSlots<KB>::P(m));
            if constexpr (KPT)
                q_h[m] = h2u(__floats2half2_rn(q_s[qh * D + KSlotsPT<KB>::c0(m, tig)] * sc,
                                               q_s[qh * D + KSlotsPT<KB>::c1(m, tig)] * sc));
            else
                q_h[m] = h2u(__floats2half2_rn(q_s[qh * D + 32 * tig + KSlots<KB>::c0(m)] * sc,
                                               q_s[qh * D + 32 * tig + KSlots<KB>::c1(m)] * sc));
        }
#pragma unroll
        for (int j = 0; j < JH; ++j) qa_inv[j] = pow2(24 - (7 - frexp_e(qmax_s[hA + j])));   // undoes 2^qa, 2^-24
    }
    // per-token keys: Q_g = sum of the head's q over group g (the zero-point term sum_g z_(t,g) Q_g)
    float qg[KPT ? 4 : 1][2];
    if constexpr (KPT) {
#pragma unroll
        for (int j = 0; j < JH; ++j)
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) {
                float acc = 0.0f;
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 v = *reinterpret_cast<const float4*>(q_s + (hA + j) * D + 32 * gg + c);
                    acc += (v.x + v.y) + (v.z + v.w);
                }
                qg[gg][j] = acc;
            }
    }
    // Everything above reads only q and the lengths.  With a.early (kvt_append_decode_attention) they were written
    // before the append kernel that precedes this launch started, and the launch is a programmatic dependent of
    // that append (PDL), so the prologue above overlaps it; otherwise the kernel already waited at entry.  The
    // cache (records, residuals) is read only after the wait.
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    Slice tl = sl;
    if (PAGED) {
        tl.bt = a.c.bt + (size_t)b * a.c.max_pages;
        tl.pstride = (size_t)g.H * g.rec;
    }
    uint64_t* tbar = reinterpret_cast<uint64_t*>(smem + Gm::Q_BYTES + Gm::TAIL_PART);
    bool staged = false;
    if (KVT_EXP != 5 && do_tail && n_main < S) {
        const int kq = nqK < S ? nqK : S, vq = nqV < S ? nqV : S;
        const int q_hi = kq > vq ? kq : vq;                               // quantised tail tokens end here
        const int r0 = n_main / kTile, r1 = (q_hi + kTile - 1) / kTile;  // their tile records
        const uint32_t b_rec = q_hi > n_main ? (uint32_t)(r1 - r0) * Gm::STAGE : 0u;
        // K residual: KIVI linear slots [0, S - nqK); per-token keys: the whole ring (slot t mod R)
        const uint32_t b_kr = KPT ? (kq < S ? (uint32_t)g.R * D * 2 : 0u) : (uint32_t)(S - kq) * D * 2;
        const uint32_t b_vr = (vq < S && sl.vr) ? (uint32_t)g.R * D * 2 : 0u;
        const uint32_t total = b_rec + b_kr + b_vr;                       // all multiples of 16
        if (Gm::SCRATCH_BYTES + total <= (uint32_t)Gm::BODY) {
            staged = true;
            uint8_t* p_rec = body + Gm::SCRATCH_BYTES;
            uint8_t* p_kr = p_rec + b_rec;
            uint8_t* p_vr = p_kr + b_kr;
            if (tid == 0) {
                mbar_init(tbar);
                asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
                fence_proxy_async();
                mbar_expect_tx(tbar, total);
                if (b_rec) {
                    if (tl.bt) {
                        for (int r = r0; r < r1; ++r) bulk_g2s(p_rec + (size_t)(r - r0) * Gm::STAGE, tl.recp(r, g), Gm::STAGE, tbar);
                    } else {
                        bulk_g2s(p_rec, sl.kc + (size_t)r0 * Gm::STAGE, b_rec, tbar);
                    }
                }
                if (b_kr) bulk_g2s(p_kr, sl.kr, b_kr, tbar);
                if (b_vr) bulk_g2s(p_vr, sl.vr, b_vr, tbar);
            }
            // virtual bases: record r of the cache lands at its staged copy under the cache's own indexing
            tl.kc = p_rec - (size_t)r0 * Gm::STAGE;
            tl.bt = nullptr;
            tl.kr = reinterpret_cast<const uint16_t*>(p_kr);
            tl.vr = reinterpret_cast<const uint16_t*>(p_vr);
        }
    }
    __syncthreads();
    // GM == 4: lanes tig and tig^2 hold the same probabilities, so they prepare different value groups:
    // relative group r (0, 1) of this lane is group 2 * (tig >> 1) + r.
    const int gsh = (GM == 4) ? 2 * (tig >> 1) : 0;
    KVT_STAMP(4);
    constexpr int NGL = (GM == 4) ? 2 : 4;               // value groups prepared per lane

    // ---- running state ----
    float m_run[2] = {-INFINITY, -INFINITY};              // reference max (lazy: moves only by > 8)
    float l_part[2] = {0.0f, 0.0f};
    // value zero-point sums per (group, head), kept as two partials (token rows r = 0, 1) so that the FFMA2
    // operand pairs are the (p(T), p(T+8)) pairs the weights use as well: no register moves
    float2 zacc2[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) zacc2[i][0] = zacc2[i][1] = make_float2(0.0f, 0.0f);
    float o[8][4];                 // PV accumulators: m-tile (γ, μ) = 2γ + μ
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
    int kp = 126;                  // PV weight exponent (only decreases)
    // ---- tail tokens [n_main, S) first (before the main loop: at the end of the CTA the whole wave finishes
    // together and these dependent loads would sit on the critical path).  Super-chunks of <= 128 tokens:
    //   (1) QK: lane = token, warp = a quarter of the channels (4-channel groups rotated by lane, so the
    //       shared-memory reads of a warp spread over the banks) -> partial logits part[warp][token][head];
    //   (2) warp h = head h (and h + 4): logits, running max / sum, p[token][head];
    //   (3) PV: lane = 4 channels, warp = every 4th token -> o partials in registers (rescaled per
    //       super-chunk); finally summed over the warps into tail_s = (m, l, o) per head. ----
    {
        float* part = reinterpret_cast<float*>(body);                      // [kWarps][128][GM] / p [128][GM]
        float ot[GM][4];
#pragma unroll
        for (int h = 0; h < GM; ++h) ot[h][0] = ot[h][1] = ot[h][2] = ot[h][3] = 0.0f;
        if (tid < GM) { tail_s[tid * (2 + D)] = -INFINITY; tail_s[tid * (2 + D) + 1] = 0.0f; }
        if (staged) mbar_wait(tbar, 0);
        KVT_STAMP(5);
        const int T = (KVT_EXP != 5 && do_tail) ? S - n_main : 0;
        for (int sc0 = 0; sc0 < T; sc0 += 128) {
            const int Tc = T - sc0 < 128 ? T - sc0 : 128;
            __syncthreads();                                                 // part / tail_s reuse
            // (1) partial logits over this warp's 32 channels
            for (int c0 = 0; c0 < Tc; c0 += 32) {
                const int i = c0 + lane, t = n_main + sc0 + i;
                float acc[GM];
#pragma unroll
                for (int h = 0; h < GM; ++h) acc[h] = 0.0f;
                if (i < Tc) {
#pragma unroll 2
                    for (int jj = 0; jj < 8; ++jj) {
                        const int c4 = 8 * warp + ((jj + lane) & 7);             // 4-channel group index
                        float kx[4];
                        dec::tail_k<KB, !KPT, true>(tl, g, t, nqK, c4, kx);
#pragma unroll
                        for (int h = 0; h < GM; ++h) {
                            const float4 qv = *reinterpret_cast<const float4*>(q_s + h * D + 4 * c4);
                            acc[h] = fmaf(qv.x, kx[0], fmaf(qv.y, kx[1], fmaf(qv.z, kx[2], fmaf(qv.w, kx[3], acc[h]))));
                        }
                    }
                }
                float* pw = part + ((size_t)warp * 128 + i) * GM;
                if (i < Tc) {
#pragma unroll
                    for (int h = 0; h < GM; h += 4)
                        *reinterpret_cast<float4*>(pw + h) = make_float4(acc[h], acc[h + 1], acc[h + 2], acc[h + 3]);
                }
            }
            __syncthreads();
            // logits (log2 domain) of token tid, summed over the 4 channel quarters, into part[0]
            for (int i = tid; i < Tc; i += kThreads) {
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    float l = 0.0f;
#pragma unroll
                    for (int w = 0; w < kWarps; ++w) l += part[((size_t)w * 128 + i) * GM + h];
                    part[(size_t)i * GM + h] = l * a.scale_log2;
                }
            }
            __syncthreads();
            // (2) per head: running max / sum, p = 2^(l - m) in place, rescale factor in tail_s[h][2]
            for (int h = warp; h < GM; h += kWarps) {
                float mx = -INFINITY;
                for (int i = lane; i < Tc; i += 32) mx = fmaxf(mx, part[(size_t)i * GM + h]);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
                float* th = tail_s + h * (2 + D);
                const float m_old = th[0], m_new = fmaxf(m_old, mx);
                float sum = 0.0f;
                for (int i = lane; i < Tc; i += 32) {
                    const float p = fexp2(part[(size_t)i * GM + h] - m_new);
                    part[(size_t)i * GM + h] = p;
                    sum += p;
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(kFull, sum, off);
                __syncwarp();
                if (lane == 0) {
                    const float al = fexp2(m_old - m_new);
                    th[1] = th[1] * al + sum;
                    th[0] = m_new;
                    th[2] = al;
                }
            }
            __syncthreads();
            // (3) PV: lane = channels [4 lane, 4 lane + 4), warp = tokens i = warp (mod 4)
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                const float al = tail_s[h * (2 + D) + 2];
#pragma unroll
                for (int e = 0; e < 4; ++e) ot[h][e] *= al;
            }
            for (int i = warp; i < Tc; i += kWarps) {
                float vx[4];
                dec::tail_v<VB, true>(tl, g, n_main + sc0 + i, nqV, lane, vx);
#pragma unroll
                for (int h = 0; h < GM; h += 4) {
                    const float4 p4 = *reinterpret_cast<const float4*>(part + (size_t)i * GM + h);
                    const float pp[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
                    for (int hh = 0; hh < 4; ++hh)
#pragma unroll
                        for (int e = 0; e < 4; ++e) ot[h + hh][e] = fmaf(pp[hh], vx[e], ot[h + hh][e]);
                }
            }
        }
        __syncthreads();                                                     // part -> o partials
        if (T > 0) {
#pragma unroll
            for (int h = 0; h < GM; ++h)
                *reinterpret_cast<float4*>(part + ((size_t)warp * GM + h) * D + 4 * lane) =
                    make_float4(ot[h][0], ot[h][1], ot[h][2], ot[h][3]);
        }
        __syncthreads();
        KVT_STAMP(6);
        for (int h = 0; h < GM; ++h) {                                       // thread = channel
            float O = 0.0f;
            if (T > 0) {
#pragma unroll
                for (int w = 0; w < kWarps; ++w) O += part[((size_t)w * GM + h) * D + tid];
            }
            tail_s[h * (2 + D) + 2 + tid] = O;
        }
    }
    if (staged && tid == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(tbar)));
    __syncthreads();
    KVT_STAMP(7);
    // ---- per-warp TMA ring: one elected lane issues one bulk copy (the tile record) per tile onto the stage mbarrier ----
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + Gm::BAR_OFF);
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < Gm::NS; ++st) mbar_init(bars + st);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    // The whole warp runs the issue path (no divergent branch around it); elect.sync picks the lane that arms the
    // stage's mbarrier and issues the copy.  The ring's shared-memory addresses and the warp's first record are
    // computed once (warp-uniform: they live in uniform registers).
    const uint32_t ring_u32 = smem_u32(wbase), bars_u32 = smem_u32(bars);
    // dense: `nxt` = the record of the next tile to issue, advanced by kWarps records per issue (loop-carried)
    const uint8_t* nxt = PAGED ? nullptr : sl.kc + (size_t)(tile_lo + warp) * Gm::STAGE;
    auto issue = [&](int it, int st) {
        const uint8_t* src = PAGED ? a.c.k_codes + ((size_t)a.c.bt[(size_t)b * a.c.max_pages + tile_lo + warp + it * kWarps] * g.H + hk) * Gm::STAGE
                                   : nxt;
        if (!PAGED) nxt += kWarps * Gm::STAGE;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
            "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %1, [%0];\n\t}\n"
            ::"r"(bars_u32 + 8 * st), "r"((uint32_t)Gm::STAGE), "r"(ring_u32 + st * Gm::STAGE), "l"(src)
            : "memory");
    };

    // generic-proxy writes to the ring area (tail scratch) are ordered before the first bulk copies; later
    // refills overwrite a stage whose reads fed the previous tile's MMAs, so they need no proxy fence
    if (lane == 0) fence_proxy_async();
#pragma unroll
    for (int s = 0; s < Gm::NS - 1; ++s)
        if (s < n_my) issue(s, s);
    KVT_STAMP(1);
    for (int it = 0; it < n_my; ++it) {
        {
            const int nx = it + Gm::NS - 1;
            if (nx < n_my) issue(nx, nx % Gm::NS);
        }
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAIT_%=;\n\t}\n" ::"r"(bars_u32 + 8 * (it % Gm::NS)), "r"((uint32_t)((it / Gm::NS) & 1)) : "memory");
        if (KVT_EXP == 4) { __syncwarp(); continue; }       // experiment: stream the tiles only
        const uint8_t* sb = wbase + (it % Gm::NS) * Gm::STAGE;
        const uint8_t* kc_s = sb + Gm::K_OFF;
        const uint32_t* km_s = reinterpret_cast<const uint32_t*>(sb + Gm::KM_OFF);
        const uint8_t* vc_s = sb + Gm::V_OFF;
        const uint32_t* vm_s = reinterpret_cast<const uint32_t*>(sb + Gm::VM_OFF);

        // (1) key block meta: scale slots (fp16 x 2^sb) and the zero-point bias sum_c q_c z_c
        float bias[2] = {0.0f, 0.0f};
        float ks_inv = 1.0f;
        uint32_t mk[KPT ? 2 : 1][2][4];          // per-token keys: meta words (4 groups) of this lane's tokens
        if constexpr (KPT) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint4 m4 = *reinterpret_cast<const uint4*>(km_s + (16 * mt + gid + 8 * r) * 4);
                    mk[mt][r][0] = m4.x; mk[mt][r][1] = m4.y; mk[mt][r][2] = m4.z; mk[mt][r][3] = m4.w;
                }
        } else {
            const uint4 m4 = reinterpret_cast<const uint4*>(km_s)[lane];
            const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
            // the largest scale: positive bf16 bit patterns order like their values
            // per-halfword max of the packed (scale | zero) words (SIMD, no masking), then the scale half
            uint32_t smb = __vmaxu2(__vmaxu2(mw[0], mw[1]), __vmaxu2(mw[2], mw[3])) & 0xffffu;
            smb = __reduce_max_sync(kFull, smb);                 // REDUX: one instruction for the warp max
            const int sbx = 7 - frexp_e(bf2f(smb));
            const float ssc = pow2(sbx);
            ks_inv = pow2(-sbx);
            // channel 4 lane + e sits at half index idx0 + 2e (K2, K4) or idx0 + e (K8) of the slot table (the
            // KSlots order), so one base per lane and immediate offsets
            const int code0 = k_slot_of<KB>((4 * lane) & 31);
            __half* shh = reinterpret_cast<__half*>(sh_s) + ((lane >> 3) * Gm::SH_STRIDE + (code0 >> 1)) * 2 + (code0 & 1);
            float z[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                shh[KB == 8 ? e : 2 * e] = __float2half_rn(bf2f(mw[e] & 0xffffu) * ssc);
                z[e] = bf2f(mw[e] >> 16);
            }
            // bias partials of the GM heads, reduce-scattered: lane l ends with head (l & 7)
            float bz[8];
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                if (h < GM) {
                    const float4 qv = *reinterpret_cast<const float4*>(q_s + h * D + 4 * lane);
                    bz[h] = qv.x * z[0] + qv.y * z[1] + qv.z * z[2] + qv.w * z[3];
                } else {
                    bz[h] = 0.0f;
                }
            }
            // GM == 8: scatter over lane bits 2, 1, 0 (lane l ends with head l & 7), then sum over bits 3, 4.
            // GM == 4: scatter over bits 1, 0 only (lane l ends with head l & 3), then sum over bits 2, 3, 4.
            if constexpr (GM == 8) {
                const bool up = (lane >> 2) & 1;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float recv = __shfl_xor_sync(kFull, up ? bz[h] : bz[h + 4], 4);
                    bz[h] = (up ? bz[h + 4] : bz[h]) + recv;
                }
            }
            {
                const bool up = (lane >> 1) & 1;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float recv = __shfl_xor_sync(kFull, up ? bz[h] : bz[h + 2], 2);
                    bz[h] = (up ? bz[h + 2] : bz[h]) + recv;
                }
            }
            {
                const bool up = lane & 1;
                const float recv = __shfl_xor_sync(kFull, up ? bz[0] : bz[1], 1);
                bz[0] = (up ? bz[1] : bz[0]) + recv;
            }
            if constexpr (GM == 4) bz[0] += __shfl_xor_sync(kFull, bz[0], 4);
            bz[0] += __shfl_xor_sync(kFull, bz[0], 8);
            bz[0] += __shfl_xor_sync(kFull, bz[0], 16);
            bias[0] = __shfl_sync(kFull, bz[0], hA);
            if constexpr (!NC) bias[1] = __shfl_sync(kFull, bz[0], hA + 1);
        }
        __syncwarp();
        // (2) B operand of QK: q_h * s_h split exactly into hi + lo
        uint32_t bq[16], bq_lo[(GM == 8 && !KPT) ? 16 : 1];
        if constexpr (KPT) {
#pragma unroll
            for (int m = 0; m < 16; ++m) bq[m] = (NC && (gid & 1)) ? 0u : q_h[m];   // q (bf16) is exact in fp16: no lo half (NC: the odd columns are 0; else GM = 4: the
                                                            // 8 columns hold heads gid & 3, i.e. the 4 heads twice)
        } else {
            const uint4* shv = reinterpret_cast<const uint4*>(sh_s + tig * Gm::SH_STRIDE);
            // GM == 4: lanes gid >= 4 carry the lo halves: b = fma(q, s, -f * hi) with f = 1 (lo) or 0 (hi)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint4 s4 = shv[u];
                const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int m = 4 * u + e;
                    const __half2 hi = __hmul2(u2h(q_h[m]), u2h(sv[e]));
                    if constexpr (GM == 8 && !KPT) {
                        bq[m] = h2u(hi);
                        bq_lo[m] = h2u(__hfma2(u2h(q_h[m]), u2h(sv[e]), __hneg2(hi)));
                    } else {
                        bq[m] = (NC ? (gid & 1) : (gid >= 4)) ? h2u(__hfma2(u2h(q_h[m]), u2h(sv[e]), __hneg2(hi))) : h2u(hi);
                    }
                }
            }
        }
        // (3) QK on the tensor cores: two m-tiles of 16 tokens, 4 independent accumulator chains
        float dq[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
        if constexpr (KPT) {
            // per-token keys: group-pure k-step pairs; dq = sum_g s_(t,g) D_g 2^(24-qa) + z_(t,g) Q_g
            uint32_t w[4][KB == 2 ? 4 : KB];   // rows gid, gid+8, 16+gid, 24+gid; the lane's words of each group
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const uint8_t* r0 = kc_s + (8 * rr + gid) * Gm::KROW;
#pragma unroll
                for (int gg = 0; gg < 4; ++gg) {
                    if constexpr (KB == 4) {
                        w[rr][gg] = *reinterpret_cast<const uint32_t*>(r0 + 16 * gg + 4 * tig);
                    } else if constexpr (KB == 2) {
                        w[rr][gg] = *reinterpret_cast<const uint32_t*>(r0 + 8 * gg + 4 * (tig >> 1));
                    } else {
                        const uint2 x = *reinterpret_cast<const uint2*>(r0 + 32 * gg + 8 * tig);
                        w[rr][2 * gg] = x.x; w[rr][2 * gg + 1] = x.y;
                    }
                }
            }
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) {
                float acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const int s = 2 * gg + s2;
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt) {
                        const uint32_t a0 = k_slot_pt<KB>(w[2 * mt], 2 * s, tig), a1 = k_slot_pt<KB>(w[2 * mt + 1], 2 * s, tig);
                        const uint32_t a2 = k_slot_pt<KB>(w[2 * mt], 2 * s + 1, tig);
                        const uint32_t a3 = k_slot_pt<KB>(w[2 * mt + 1], 2 * s + 1, tig);
                        hmma(acc[mt], a0, a1, a2, a3, bq[2 * s], bq[2 * s + 1]);
                    }
                }
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int i = 0; i < 4; i += (NC ? 2 : 1)) {     // NC: column 2 tig + 1 is zero
                        const uint32_t mw = mk[mt][i >> 1][gg];
                        dq[mt][i] = fmaf(bf2f(mw & 0xffffu) * qa_inv[NC ? 0 : (i & 1)], acc[mt][i],
                                         fmaf(bf2f(mw >> 16), qg[gg][NC ? 0 : (i & 1)], dq[mt][i]));
                    }
            }
        } else if (KVT_EXP != 2 && KVT_EXP != 3) {
            uint32_t w[4][KB];        // rows gid, gid+8, 16+gid, 24+gid
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const uint8_t* r0 = kc_s + (8 * rr + gid) * Gm::KROW + tig * 4 * KB;
                if constexpr (KB == 2) {
                    const uint2 x = *reinterpret_cast<const uint2*>(r0);
                    w[rr][0] = x.x; w[rr][1] = x.y;
                } else {
#pragma unroll
                    for (int u = 0; u < KB / 4; ++u) {
                        const uint4 x = reinterpret_cast<const uint4*>(r0)[u];
                        w[rr][4 * u] = x.x; w[rr][4 * u + 1] = x.y; w[rr][4 * u + 2] = x.z; w[rr][4 * u + 3] = x.w;
                    }
                }
            }
            float de[2][4], dd[2][4];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    float* acc = (s & 1) ? dd[mt] : de[mt];
                    const uint32_t a0 = k_slot<KB>(w[2 * mt], 2 * s), a1 = k_slot<KB>(w[2 * mt + 1], 2 * s);
                    const uint32_t a2 = k_slot<KB>(w[2 * mt], 2 * s + 1), a3 = k_slot<KB>(w[2 * mt + 1], 2 * s + 1);
                    if (s < 2) hmma0(acc, a0, a1, a2, a3, bq[2 * s], bq[2 * s + 1]);   // chain starts
                    else hmma(acc, a0, a1, a2, a3, bq[2 * s], bq[2 * s + 1]);
                    if constexpr (GM == 8) hmma(acc, a0, a1, a2, a3, bq_lo[2 * s], bq_lo[2 * s + 1]);
                }
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                if constexpr (NC) {                   // (hi + lo) of head tig, rows gid and gid + 8
                    dq[mt][0] = (de[mt][0] + dd[mt][0]) + (de[mt][1] + dd[mt][1]);
                    dq[mt][2] = (de[mt][2] + dd[mt][2]) + (de[mt][3] + dd[mt][3]);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        dq[mt][i] = de[mt][i] + dd[mt][i];
                        if constexpr (GM == 4) dq[mt][i] += __shfl_xor_sync(kFull, dq[mt][i], 2);
                    }
                }
            }
        }
        // (4) logits (log2 domain) for tokens {16mt + gid + 8r} x heads {hA, hA + 1}; online softmax with a
        // lazy reference max: it only moves when the tile max exceeds it by more than 8 (so p <= 2^8)
        float alpha[2], p[2][2][2];        // p[mt][r][j]
        bool resc = false;
#pragma unroll
        for (int j = 0; j < JH; ++j) {
            const float cs = KPT ? a.scale_log2 : a.scale_log2 * qa_inv[j] * ks_inv;   // KPT: dq holds q.k
            const float cb = KPT ? 0.0f : a.scale_log2 * bias[j];
            float l4[4];
            l4[0] = fmaf(dq[0][j], cs, cb);
            l4[1] = fmaf(dq[0][2 + j], cs, cb);
            l4[2] = fmaf(dq[1][j], cs, cb);
            l4[3] = fmaf(dq[1][2 + j], cs, cb);
            float mx = fmaxf(fmaxf(l4[0], l4[1]), fmaxf(l4[2], l4[3]));
            alpha[j] = 1.0f;
            // the reference max moves only if some logit exceeds it by > 8: one vote decides whether the
            // cross-lane max is needed at all (after the first tiles it almost never is)
            if (__any_sync(kFull, mx > m_run[j] + 8.0f)) {
                mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 4));
                mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 8));
                mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 16));
                if (mx > m_run[j] + 8.0f) {
                    alpha[j] = fexp2(m_run[j] - mx);
                    m_run[j] = mx;
                    resc = true;
                }
            }
            const float mr = m_run[j];
            p[0][0][j] = fexp2(l4[0] - mr);
            p[0][1][j] = fexp2(l4[1] - mr);
            p[1][0][j] = fexp2(l4[2] - mr);
            p[1][1][j] = fexp2(l4[3] - mr);
            l_part[j] = l_part[j] * alpha[j] + ((p[0][0][j] + p[0][1][j]) + (p[1][0][j] + p[1][1][j]));
        }
        // (5) value weights w = p * s_v * 2^kp (fp16 pairs (T, T+8)) and zero sums p * z_v
        float kfac = 1.0f;
        if constexpr (NC) {
            // head tig, this lane's 4 tokens x all 4 value groups
            uint32_t mw[2][2][4];
            uint32_t smb = 0;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint4 m4 = *reinterpret_cast<const uint4*>(vm_s + (16 * mt + gid + 8 * r) * 4);
                    mw[mt][r][0] = m4.x; mw[mt][r][1] = m4.y; mw[mt][r][2] = m4.z; mw[mt][r][3] = m4.w;
                    smb = __vmaxu2(__vmaxu2(smb, __vmaxu2(m4.x, m4.y)), __vmaxu2(m4.z, m4.w));   // per-halfword max
                }
            smb &= 0xffffu;                                       // the scale halves
            smb = __reduce_max_sync(kFull, smb);
            const int kt = 7 - frexp_e(bf2f(smb));
            if (kt < kp) {
                if (it > 0) { kfac = pow2(kt - kp < -126 ? -126 : kt - kp); resc = true; }
                kp = kt;
            }
            const float ksc = pow2(kp);
            uint32_t wv[2][4];
#pragma unroll
            for (int gr = 0; gr < 4; ++gr) {
                float2 za = zacc2[gr][0];
                if (resc) za = dec::fmul2(za, make_float2(alpha[0], alpha[0]));
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const uint32_t w0 = mw[mt][0][gr], w1 = mw[mt][1][gr];
                    const float2 sv = dec::fmul2(make_float2(bf2f(w0 & 0xffffu), bf2f(w1 & 0xffffu)), make_float2(ksc, ksc));
                    const float2 wa = dec::fmul2(make_float2(p[mt][0][0], p[mt][1][0]), sv);
                    wv[mt][gr] = h2u(__floats2half2_rn(wa.x, wa.y));
                    const float2 zz = make_float2(__uint_as_float(w0 & 0xffff0000u), __uint_as_float(w1 & 0xffff0000u));
                    za = dec::ffma2(make_float2(p[mt][0][0], p[mt][1][0]), zz, za);
                }
                zacc2[gr][0] = za;
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
                *reinterpret_cast<uint4*>(w_s + wt_idx(mt, gid, tig)) = make_uint4(wv[mt][0], wv[mt][1], wv[mt][2], wv[mt][3]);
        } else        {
            // meta words of this lane's 4 tokens x its value groups (GM == 4: the tig pair splits the groups)
            uint32_t mw[2][2][NGL];
            uint32_t smb = 0;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint32_t* row = vm_s + (16 * mt + gid + 8 * r) * 4 + gsh;
                    if constexpr (NGL == 4) {
                        const uint4 m4 = *reinterpret_cast<const uint4*>(row);
                        mw[mt][r][0] = m4.x; mw[mt][r][1] = m4.y; mw[mt][r][2 % NGL] = m4.z; mw[mt][r][3 % NGL] = m4.w;
                    } else {
                        const uint2 m2 = *reinterpret_cast<const uint2*>(row);
                        mw[mt][r][0] = m2.x; mw[mt][r][1] = m2.y;
                    }
#pragma unroll
                    for (int gr = 0; gr < NGL; ++gr) smb = __vmaxu2(smb, mw[mt][r][gr]);   // per-halfword max
                }
            // lanes differing only in tig hold the same tokens (and, GM == 4, the same groups up to the tig^2
            // split), so the max over the whole warp is the max over all 32 tokens and 4 groups
            smb &= 0xffffu;                                       // the scale halves
            smb = __reduce_max_sync(kFull, smb);
            const int kt = 7 - frexp_e(bf2f(smb));
            if (kt < kp) {
                if (it > 0) { kfac = pow2(kt - kp < -126 ? -126 : kt - kp); resc = true; }
                kp = kt;
            }
            // 2^kp is folded into the value scale (s_v 2^kp <= 2^7 for every bf16 scale), not into p (<= 2^8), so
            // no product overflows even at kp = 126; powers of two multiply exactly, so the weights are the same
            const float ksc = pow2(kp);
            // weight-tile word of (group gsh + gr, m-tile mt): one per-lane base plus a compile-time offset (gsh is
            // even, so 4 ((gsh + gr) >> 1) = 4 (gsh >> 1) for GM == 4; gsh = 0 for GM == 8)
            uint32_t* const wst = w_s + (gsh * 2 * 8 + gid) * 8 + 4 * (gsh >> 1) + hA;
#pragma unroll
            for (int gr = 0; gr < NGL; ++gr) {
                float2 za0 = zacc2[gr][0], za1 = zacc2[gr][1];
                if (resc) {
                    za0 = dec::fmul2(za0, make_float2(alpha[0], alpha[0]));
                    za1 = dec::fmul2(za1, make_float2(alpha[1], alpha[1]));
                }
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const uint32_t w0 = mw[mt][0][gr], w1 = mw[mt][1][gr];
                    const float2 sv = dec::fmul2(make_float2(bf2f(w0 & 0xffffu), bf2f(w1 & 0xffffu)), make_float2(ksc, ksc));
                    uint2 wv;
                    const float2 wa = dec::fmul2(make_float2(p[mt][0][0], p[mt][1][0]), sv);
                    const float2 wb = dec::fmul2(make_float2(p[mt][0][1], p[mt][1][1]), sv);
                    wv.x = h2u(__floats2half2_rn(wa.x, wa.y));
                    wv.y = h2u(__floats2half2_rn(wb.x, wb.y));
                    *reinterpret_cast<uint2*>(wst + (gr * 2 + mt) * 64 + (GM == 4 ? 0 : 4 * (gr >> 1))) = wv;
                    const float2 zz = make_float2(__uint_as_float(w0 & 0xffff0000u), __uint_as_float(w1 & 0xffff0000u));
                    za0 = dec::ffma2(make_float2(p[mt][0][0], p[mt][1][0]), zz, za0);
                    za1 = dec::ffma2(make_float2(p[mt][0][1], p[mt][1][1]), zz, za1);
                }
                zacc2[gr][0] = za0;
                zacc2[gr][1] = za1;
            }
        }
        __syncwarp();
        // (6) PV on the tensor cores: 8 m-tiles (γ, μ) x 2 k-steps of 16 tokens
        if (KVT_EXP != 1 && KVT_EXP != 3) {
            if (__any_sync(kFull, resc)) {
                // PV columns 2tig, 2tig+1 = heads 2tig, 2tig+1; NC: their softmax state lives in lanes tig' = 2tig (+1)
                const float r0 = (NC ? __shfl_sync(kFull, alpha[0], (lane & ~3) | ((2 * tig) & 3)) : alpha[0]) * kfac;
                const float r1 = (NC ? __shfl_sync(kFull, alpha[0], (lane & ~3) | ((2 * tig + 1) & 3)) : alpha[1]) * kfac;
#pragma unroll
                for (int i = 0; i < 8; ++i) { o[i][0] *= r0; o[i][1] *= r1; o[i][2] *= r0; o[i][3] *= r1; }
            }
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                VRaw<VB> raw;
                v_load<VB>(vc_s, ks, tig, gid, raw);
                uint4 B0 = make_uint4(0, 0, 0, 0), B1 = B0;
                if constexpr (NC) {                 // all 4 groups' weights of pairs tig, tig + 4, head gid
                    B0 = *reinterpret_cast<const uint4*>(w_s + wt_idx(ks, tig, gid));
                    B1 = *reinterpret_cast<const uint4*>(w_s + wt_idx(ks, tig + 4, gid));
                }
#pragma unroll
                for (int gam = 0; gam < 4; ++gam) {
                    uint32_t b0, b1;
                    if constexpr (NC) {
                        b0 = gam == 0 ? B0.x : (gam == 1 ? B0.y : (gam == 2 ? B0.z : B0.w));
                        b1 = gam == 0 ? B1.x : (gam == 1 ? B1.y : (gam == 2 ? B1.z : B1.w));
                    } else {
                        const uint32_t* wr = w_s + (gam * 2 + ks) * 64 + 4 * (gam >> 1) + gid;
                        b0 = wr[tig * 8]; b1 = wr[(tig + 4) * 8];
                    }
                    uint32_t hA4[4], hB4[4];
                    v_frag<VB>(raw, gam, hA4, hB4);
                    if constexpr (KVT_EXP == 6) {
                        // tcgen05 cost probe: the PV A operand (128 channels x 16 tokens fp16 = 4 KB per k-step) staged
                        // to shared memory as a tcgen05.mma would need it, instead of feeding HMMA from registers
                        // (the stores go to a small scratch: only the issue cost counts)
                        const uint32_t st = smem_u32(sh_s) + (lane & 3) * 32;
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(st), "r"(hA4[0]), "r"(hA4[1]), "r"(hB4[0]), "r"(hB4[1]) : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(st + 16), "r"(hA4[2]), "r"(hA4[3]), "r"(hB4[2]), "r"(hB4[3]) : "memory");
                        (void)b0; (void)b1;      // tcgen05 would read the weight tile (B) from shared memory itself
                    } else {
                        hmma(o[2 * gam], hA4[0], hA4[1], hB4[0], hB4[1], b0, b1);
                        hmma(o[2 * gam + 1], hA4[2], hA4[3], hB4[2], hB4[3], b0, b1);
                    }
                }
            }
        }
        __syncwarp();
    }

    KVT_STAMP(2);
#if KVT_TRACE
    if (a.trace && lane == 0 && blockIdx.x < 4096) {        // per-warp end of the tile loop (first segment)
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        unsigned long long* p_ = a.trace + 11 * 4096 + 4 * blockIdx.x + warp;
        if (*p_ == 0ull) *p_ = t_;
    }
#endif
    __syncwarp();
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < Gm::NS; ++st) asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars + st)));
    }
    // ---- warp epilogue: l over the 8 row-groups, zero sums, o = D * 2^(24 - P(row) - kp) + zacc ----
    float zacc[4][2];
    if constexpr (NC) {
        // lane (gid, tig): softmax state of head tig; the PV owner lanes (tig < 2) need heads 2tig, 2tig + 1
        float z[4], l = l_part[0];
#pragma unroll
        for (int i = 0; i < 4; ++i) z[i] = zacc2[i][0].x + zacc2[i][0].y;
#pragma unroll
        for (int off = 4; off <= 16; off <<= 1) {
            l += __shfl_xor_sync(kFull, l, off);
#pragma unroll
            for (int i = 0; i < 4; ++i) z[i] += __shfl_xor_sync(kFull, z[i], off);
        }
        const float m0 = m_run[0];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int src = (lane & ~3) | ((2 * tig + j) & 3);
            m_run[j] = __shfl_sync(kFull, m0, src);
            l_part[j] = __shfl_sync(kFull, l, src);
#pragma unroll
            for (int i = 0; i < 4; ++i) zacc[i][j] = __shfl_sync(kFull, z[i], src);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) if (!NC) zacc[i][j] = zacc2[i][j].x + zacc2[i][j].y;
#pragma unroll
    for (int j = 0; j < (NC ? 0 : 2); ++j) {
        float l = (GM == 8 || tig < 2) ? l_part[j] : 0.0f;
        l += __shfl_xor_sync(kFull, l, 4);
        l += __shfl_xor_sync(kFull, l, 8);
        l += __shfl_xor_sync(kFull, l, 16);
        l_part[j] = l;
#pragma unroll
        for (int gam = 0; gam < 4; ++gam) {
            float z = zacc[gam][j];
            z += __shfl_xor_sync(kFull, z, 4);
            z += __shfl_xor_sync(kFull, z, 8);
            z += __shfl_xor_sync(kFull, z, 16);
            zacc[gam][j] = z;
        }
    }
    if constexpr (GM == 4 && !NC) {   // tig 0/1 hold groups 0,1 of heads (0,1)/(2,3) in slots 0,1; tig 2/3 groups 2,3
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            zacc[2][j] = __shfl_xor_sync(kFull, zacc[0][j], 2);
            zacc[3][j] = __shfl_xor_sync(kFull, zacc[1][j], 2);
        }
    }
    __syncthreads();                                   // the per-warp areas become the combine area
    float* comb = reinterpret_cast<float*>(body);      // [8 partials][8 heads][2 + D]
    {
        float* cw = comb + warp * 8 * (2 + D);
        const bool owner = (GM == 8) || (tig < 2);     // PV columns 2tig, 2tig+1 are real heads
        if (owner) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int h = 2 * tig + j;
                float* ch = cw + h * (2 + D);
                if (gid == 0) { ch[0] = m_run[j]; ch[1] = l_part[j]; }
#pragma unroll
                for (int gam = 0; gam < 4; ++gam)
#pragma unroll
                    for (int mu = 0; mu < 2; ++mu) {
                        const int c = 32 * gam + 4 * gid + 2 * mu;
                        ch[2 + c] = o[2 * gam + mu][j] * pow2(24 - VP<VB>(2 * mu) - kp) + zacc[gam][j];
                        ch[2 + c + 1] = o[2 * gam + mu][2 + j] * pow2(24 - VP<VB>(2 * mu + 1) - kp) + zacc[gam][j];
                    }
            }
        }
    }
    __syncthreads();
    // ---- CTA combine of the warps' partials and the tail partial: thread = channel ----
    const int c = tid;
    for (int h = 0; h < gq; ++h) {
        float M = tail_s[h * (2 + D)];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, comb[(w * 8 + h) * (2 + D)]);
        float L = 0.0f, O = 0.0f;
        if (M != -INFINITY) {
#pragma unroll
            for (int w = 0; w <= kWarps; ++w) {
                const float* cw = w < kWarps ? comb + (w * 8 + h) * (2 + D) : tail_s + h * (2 + D);
                if (cw[1] == 0.0f) continue;
                const float scl = fexp2(cw[0] - M);
                L += cw[1] * scl;
                O += cw[2 + c] * scl;
            }
        }
        const size_t row = (size_t)b * a.H_q + (size_t)hk * gq + h;
        if (count == 1) {
            write_row(a, a.out, a.out_mode, row, c, M, L, O);
        } else {
            float* pr = a.parts + ((size_t)(cta * 2 + slot) * 8 + h) * (2 + D);
            if (c == 0) { pr[0] = M; pr[1] = L; }
            pr[2 + c] = L > 0.0f ? __fdiv_rn(O, L) : 0.0f;
        }
    }
    // ---- fused combine (K3): the last of the unit's CTAs to arrive merges its partials ----
    if (count > 1) {
        __shared__ int is_last;
        __threadfence();                      // every thread's partial writes are visible device-wide ...
        __syncthreads();                      // ... before thread 0 announces this segment
        if (tid == 0) {
            const int old = atomicAdd(a.counters + bh, 1);
            is_last = (old == count - 1);
        }
        __syncthreads();
        if (is_last && count * 8 * 2 * (int)sizeof(float) <= Gm::BODY) {
            // (m, l) of every (partial, head) staged in shared memory by all threads at once, then the o loads
            // of all heads of a partial issued together: no chain of dependent L2 round trips per head
            __threadfence();
            float* ml = reinterpret_cast<float*>(body);        // [count][8 heads][m, l]; body is free here
            for (int i = tid; i < count * 8; i += kThreads) {
                const int k = i >> 3, h = i & 7;
                if (h < gq) {
                    const float* pr = a.parts + ((size_t)((c_first + k) * 2 + (k == 0)) * 8 + h) * (2 + D);
                    ml[2 * i] = __ldcg(pr);
                    ml[2 * i + 1] = __ldcg(pr + 1);
                }
            }
            __syncthreads();
            float Mh[8], Lh[8], Oh[8];
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                Mh[h] = -INFINITY; Lh[h] = 0.0f; Oh[h] = 0.0f;
                if (h < gq)
                    for (int k = 0; k < count; ++k) Mh[h] = fmaxf(Mh[h], ml[2 * (k * 8 + h)]);
            }
            for (int k = 0; k < count; ++k) {
                const float* pk = a.parts + ((size_t)((c_first + k) * 2 + (k == 0)) * 8) * (2 + D) + 2 + c;
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    if (h < gq && Mh[h] != -INFINITY) {
                        const float l = ml[2 * (k * 8 + h) + 1];
                        if (l != 0.0f) {
                            const float wgt = l * fexp2(ml[2 * (k * 8 + h)] - Mh[h]);
                            Lh[h] += wgt;
                            Oh[h] += wgt * __ldcg(pk + (size_t)h * (2 + D));
                        }
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 8; ++h)
                if (h < gq) write_row(a, a.out, a.out_mode, (size_t)b * a.H_q + (size_t)hk * gq + h, c, Mh[h], Lh[h], Oh[h]);
            if (tid == 0) a.counters[bh] = 0;
        } else if (is_last) {
            __threadfence();
            for (int h = 0; h < gq; ++h) {
                const size_t row = (size_t)b * a.H_q + (size_t)hk * gq + h;
                float M = -INFINITY;
                for (int k = 0; k < count; ++k)
                    M = fmaxf(M, __ldcg(a.parts + ((size_t)((c_first + k) * 2 + (k == 0)) * 8 + h) * (2 + D)));
                float L = 0.0f, O = 0.0f;
                if (M != -INFINITY) {
                    for (int k = 0; k < count; ++k) {
                        const float* pr = a.parts + ((size_t)((c_first + k) * 2 + (k == 0)) * 8 + h) * (2 + D);
                        const float l = __ldcg(pr + 1);
                        if (l == 0.0f) continue;
                        const float wgt = l * fexp2(__ldcg(pr) - M);
                        L += wgt;
                        O += wgt * __ldcg(pr + 2 + c);
                    }
                }
                write_row(a, a.out, a.out_mode, row, c, M, L, O);
            }
            if (tid == 0) a.counters[bh] = 0;
        }
    }
    KVT_STAMP(3);
}

// ---- Stream-K work split over all (b, kv head) units --------------------------------------------------
// Unit u = (b, hk) costs unit_cost(S_b) work units: its main tiles plus ceil(tail tokens / 8) (the tail is
// processed a token at a time, ~4x the per-token cost of a tile), at least 1 so that every unit has an
// owner.  The flattened space [0, C) of all units is cut into n equal contiguous ranges, one per CTA
// (n = resident CTAs: one balanced wave instead of ragged waves of whole splits).  A CTA walks the units
// its range touches; a unit inside one CTA is written directly, a unit cut across CTAs is merged by the
// last of them (partials: slot 1 in the unit's first CTA, slot 0 in the others).
// the CTA whose range [c C / n, (c + 1) C / n) holds position x
__device__ __forceinline__ int cta_of(long long x, long long C, int n) { return (int)(((x + 1) * n - 1) / C); }

// Per-SM plan (a.sm_w = w > 0): the grid is one full wave (occupancy x SMs CTAs).  Each CTA learns its SM
// (%smid, ranked densely in order of first arrival) and its arrival slot on that SM.  The first arrival on SM r
// takes piece r of the remaining units, cut stream-K style into one piece per SM (fused merge of cut units as
// above); arrivals 1 .. w take the whole units w r + 0 .. w-1; later arrivals idle.  Every SM then holds the same work (w units plus
// (U - w SMs) / SMs of a unit) while only one CTA per SM pays for cut segments; with whole units (the plan it
// replaces) ceil(U / SMs) units sat on some SMs and floor(U / SMs) on others.  Correct for any placement: an
// item no CTA claimed (an SM with fewer CTAs than expected) is run by the last CTA to finish, which also resets
// the counters.  Schedule words: [256 arrivals per %smid][256 rank + 1 per %smid][rank count][done][claims].
constexpr int kSchedSmid = 256;
__device__ __forceinline__ int sm_claim(const DecodeArgs& a) {
    int* ctr = a.sched;
    int* rank_of = a.sched + kSchedSmid;
    int* nrank = a.sched + 2 * kSchedSmid;
    int* claim = a.sched + 2 * kSchedSmid + 2;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (smid >= (unsigned)kSchedSmid) return -1;                   // (never on B200) left to the last CTA
    const int slot = atomicAdd(ctr + smid, 1);
    int r;
    if (slot == 0) {
        r = atomicAdd(nrank, 1);
        atomicExch(rank_of + smid, r + 1);
    } else {
        int v;
        while ((v = atomicAdd(rank_of + smid, 0)) == 0) __nanosleep(20);   // the SM's first CTA is resident
        r = v - 1;
    }
    if (r >= a.sm_n || slot > a.sm_w) return -1;
    if (a.sm_drop > 0 && blockIdx.x % a.sm_drop == 0) return -1;   // tests: exercise the unclaimed-item path
    const int item = r * (a.sm_w + 1) + slot;
    atomicExch(claim + item, 1);
    return item;
}

// PAGED: tile records addressed through the block table (compile-time, so the dense issue path stays short)
template <int KB, int VB, int GM, bool KPT, bool PAGED>
__global__ void __launch_bounds__(kThreads, GM == 4 ? 4 : 3) decode_mma_kernel(DecodeArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ long long s_wsum[2][kWarps];
    __shared__ long long s_first[2];
    __shared__ int s_item, s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int B = a.g.B, H = a.g.H;
    // Programmatic dependent launch: unless the library launched the preceding kernel itself (the append of
    // kvt_append_decode_attention, which leaves q, the lengths and the workspace untouched), nothing may be read
    // before the preceding grid's writes are visible.
    if (!a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    // (1) exclusive scan of the per-batch costs H * cost(S_b): thread = a chunk of consecutive b; with the per-SM
    // plan also the cost Cw of the whole units [0, w SMs)
    const long long u0 = (long long)a.sm_w * a.sm_n;
    const int chunk = (B + kThreads - 1) / kThreads;
    const int b0 = min(tid * chunk, B), b1 = min(b0 + chunk, B);
    long long mine = 0, mine_w = 0;
    for (int bb = b0; bb < b1; ++bb) {
        const long long c1 = unit_cost(a.g, a.seq_len[bb]).cost;
        mine += (long long)H * c1;
        const long long nu = u0 - (long long)bb * H;
        mine_w += (nu <= 0 ? 0 : (nu >= H ? H : nu)) * c1;
    }
    long long inc = mine, inc_w = mine_w;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) inc_w += __shfl_xor_sync(kFull, inc_w, off);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long v = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) inc += v;
    }
    if (lane == 31) s_wsum[0][warp] = inc;
    if (lane == 0) s_wsum[1][warp] = inc_w;
    __syncthreads();
    long long C = 0, Cw = 0, excl = inc - mine;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        if (w < warp) excl += s_wsum[0][w];
        C += s_wsum[0][w];
        Cw += s_wsum[1][w];
    }
    // Work of this CTA: the cost range [lo, hi) of part `idx` of the n-part cut of [base, base + span), walked unit by
    // unit (one segment per unit touched).  Stream-K plan: part blockIdx.x of [0, C).  Per-SM plan: a whole unit
    // (a one-part cut of its own range) or piece r of the remaining units; the last CTA to finish then walks the
    // items nobody claimed, one after the other.  One call site of segment() (it is large and inlined).
    long long lo = 0, hi = 0, base = 0, span = 1;
    int n = 1, idx = 0;
    int item = -1;
    bool plan_sm = a.sm_w > 0, counted = false;
    int scan = 0;
    const int W1 = a.sm_w + 1, nsm = a.sm_n;
    // unit u (whole) or position x (stream-K, pieces) -> its batch row and the cost offset of that row
    auto locate = [&](bool by_unit, long long key) {
        if (by_unit ? (key / H >= b0 && key / H < b1) : (key >= excl && key < excl + mine)) {
            long long P = excl;
            for (int bb = b0; bb < b1; ++bb) {
                const long long cb = (long long)H * unit_cost(a.g, a.seq_len[bb]).cost;
                if (by_unit ? bb == key / H : key < P + cb) { s_first[0] = bb; s_first[1] = P; break; }
                P += cb;
            }
        }
        __syncthreads();
    };
    if (plan_sm) {
        if (tid == 0) s_item = sm_claim(a);
        __syncthreads();
        item = s_item;
    } else {
        n = (long long)a.n_cta < C ? a.n_cta : (int)C;
        idx = blockIdx.x;
        if (KVT_TRACE && tid == 0) s_item = -1;
        if (idx >= n) return;                               // uniform per CTA
        lo = (long long)idx * C / n; hi = (long long)(idx + 1) * C / n; base = 0; span = C;
        locate(false, lo);
    }
#if KVT_TRACE
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    for (;;) {
        if (plan_sm) {
            if (item >= 0) {                                // uniform per CTA
                // arrival slot -> role: the first CTA to arrive on an SM takes the piece (CTAs that arrive first on
                // an SM run ahead of the later ones), or (KVT_PIECE_FIRST=0, A/B only) the last one
                const int r = item / W1, slot0 = item - r * W1;
                const int slot = a.sm_piece_first ? (slot0 == 0 ? a.sm_w : slot0 - 1) : slot0;
                if (slot < a.sm_w) {
                    const long long u = (long long)a.sm_w * r + slot;
                    locate(true, u);
                    const UnitCost uc = unit_cost(a.g, a.seq_len[s_first[0]]);
                    lo = s_first[1] + (u - (long long)s_first[0] * H) * uc.cost;
                    hi = lo + uc.cost; base = lo; span = uc.cost; n = 1; idx = 0;
                } else {
                    const long long R = C - Cw;
                    lo = Cw + (long long)r * R / nsm; hi = Cw + (long long)(r + 1) * R / nsm;
                    base = Cw; span = R > 0 ? R : 1; n = nsm; idx = r;
                    if (lo < hi) locate(false, lo);
                }
            } else {
                lo = hi = 0;
            }
        }
        if (lo < hi) {
            int b = (int)s_first[0];
            long long Pb = s_first[1], pos = lo;
            __syncthreads();                                // s_first is rewritten by the next locate
            while (pos < hi) {
                const UnitCost uc = unit_cost(a.g, a.seq_len[b]);
                if (pos >= Pb + (long long)H * uc.cost) { Pb += (long long)H * uc.cost; ++b; continue; }
                const int hk = (int)((pos - Pb) / uc.cost);
                const long long Pu = Pb + (long long)hk * uc.cost;
                const int x0 = (int)(pos - Pu);
                const int x1 = (int)(hi - Pu < uc.cost ? hi - Pu : uc.cost);
                const int cf = cta_of(Pu - base, span, n), cl = cta_of(Pu - base + uc.cost - 1, span, n);
                segment<KB, VB, GM, KPT, PAGED>(a, smem, b, hk, min(x0, uc.tiles), min(x1, uc.tiles), x1 == uc.cost, idx,
                                                idx == cf ? 1 : 0, cf, cl - cf + 1);
                pos = Pu + x1;
                __syncthreads();                            // the next segment reuses shared memory
            }
        }
        if (!plan_sm) break;
        if (!counted) {                                     // this CTA's own item is done: count it
            counted = true;
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                s_last = atomicAdd(a.sched + 2 * kSchedSmid + 1, 1) == (int)gridDim.x - 1;
            }
            __syncthreads();
            if (!s_last) break;
            __threadfence();
        }
        // the last CTA: the next item nobody claimed (only when the placement was not the expected one).  All
        // threads test their share of the claim words at once (independent loads: one L2 round trip, not one per
        // item) and the smallest unclaimed index wins.
        {
            const volatile int* claim = a.sched + 2 * kSchedSmid + 2;
            if (tid == 0) s_item = INT_MAX;
            __syncthreads();
            int mine_first = INT_MAX;
            for (int i = scan + tid; i < W1 * nsm; i += kThreads)
                if (claim[i] == 0 && i < mine_first) mine_first = i;
            if (mine_first != INT_MAX) atomicMin(&s_item, mine_first);
            __syncthreads();
            item = s_item == INT_MAX ? -1 : s_item;
            scan = item + 1;
            __syncthreads();
        }
        if (item < 0) {
            for (int i = tid; i < 2 * kSchedSmid + 2 + W1 * nsm; i += kThreads) a.sched[i] = 0;
            break;
        }
    }
#if KVT_TRACE
    if (tid == 0) {
        unsigned long long t_end;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        const int cta = blockIdx.x;
        // smid | (per-SM plan item + 1) << 16
        if (a.trace && cta < 4096) { a.trace[3 * cta] = smid | (unsigned long long)(s_item + 1) << 16; a.trace[3 * cta + 1] = t_start; a.trace[3 * cta + 2] = t_end; }
    }
#endif
}

}  // namespace mma
}  // namespace kvt

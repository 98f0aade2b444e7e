// kvt_decode_pk.cuh — K2 persistent warp-item decode attention ("persistent kernel").
//
// Same arithmetic per 32-token tile as kvt_decode_mma.cuh (tile records, fp16-subnormal codes on the tensor
// cores, lazy online softmax, fp32 zero-point sums); a different work schedule:
//
//   * one CTA per SM with NW warps (16 for g <= 4, 12 for g <= 8, fewer when the ring of a wide instance does not
//     fit), each warp an independent worker with its own TMA ring, weight tile, q copy and softmax state;
//   * the work is a global list of *items*: first the tail item of every (b, kv head) unit (the bf16 / incomplete
//     tokens past the last whole tile, CUDA cores), then, unit after unit, the unit's main tiles in chunks of CH
//     tiles (`rounds` slots per unit; slots past a short unit's last chunk are skipped) — item j maps to its
//     (unit, tile range) in O(1) with host-precomputed reciprocals;
//   * a warp claims the next item with one atomicAdd on a global counter one tile before it needs it (the claim,
//     the next unit's q rows (cp.async) and its first TMA copy overlap the current item's last tile), so the GPU
//     balances itself at the granularity of one item whatever the batch, lengths or scheduler fairness;
//   * every item leaves its (m, l, o) partial (o unnormalised) in its own workspace slot.  A unit's partials are
//     merged by a two-level tree: the last chunk of each group of GS consecutive chunks to finish merges the group
//     (per-group arrival counter), the last group (or, for units of <= GS chunks, the last chunk) merges the tail
//     partial and the group partials in a fixed order and writes the output row.  A unit with a single item
//     writes its row directly.
//
// The partition (CH, the item list, the groups) is a pure function of (B, H, lengths, the host plan length, the SM
// count and warps per SM), and no partial depends on which warp computed it, so results are bitwise reproducible
// (A23).
#pragma once
#include "kvt_decode_mma.cuh"

namespace kvt {
namespace pk {

using dec::DecodeArgs;
using dec::FDiv;
using dec::fdiv;
using dec::Slice;
using dec::bf2f;
using dec::kFull;
using mma::D;
using mma::kTile;
using mma::KSlots;
using mma::KSlotsPT;
using mma::VRaw;
using mma::VP;
using mma::h2u;
using mma::u2h;
using mma::hmma;
using mma::fexp2;
using mma::frexp_e;
using mma::pow2;
using mma::k_slot;
using mma::k_slot_pt;
using mma::k_slot_of;
using mma::v_load;
using mma::v_frag;
using mma::write_row;
using mma::smem_u32;
using mma::mbar_init;
using mma::mbar_expect_tx;
using mma::mbar_wait;
using mma::bulk_g2s;

// Per-warp shared memory: [ring NS x STAGE | weight tile W (also the tail's p scratch) | key-scale slots SH |
// mbarriers | q fp32 [GM][D] | next q bf16 [GM][D] (cp.async prefetch)]
template <int KB, int VB, int GM>
struct PGeo {
    using G0 = mma::Geo<KB, VB, GM>;
    static constexpr int STAGE = G0::STAGE;
    static constexpr int NS = 2;
    static constexpr int W_OFF = NS * STAGE;
    static constexpr int W_BYTES = G0::W_BYTES;
    static constexpr int SH_OFF = W_OFF + W_BYTES;
    static constexpr int SH_STRIDE = G0::SH_STRIDE;
    static constexpr int BAR_OFF = SH_OFF + 4 * SH_STRIDE * 4;
    static constexpr int Q_OFF = (BAR_OFF + 8 * NS + 15) / 16 * 16;
    static constexpr int QB_OFF = Q_OFF + GM * D * 4;
    static constexpr int WARP_BYTES = (QB_OFF + GM * D * 2 + 127) / 128 * 128;
    static constexpr int MAXW = GM == 4 ? 16 : 12;          // registers: 16 warps x 128, 12 x 168
    static constexpr int CAP = 227 * 1024;
    static constexpr int NW = CAP / WARP_BYTES < MAXW ? CAP / WARP_BYTES : MAXW;
    static constexpr size_t SMEM = (size_t)NW * WARP_BYTES;
    static_assert(32 * 8 * 4 <= W_BYTES, "tail p scratch must fit the weight tile");
};

// One work item of the global list (see the header comment).
struct Item {
    int kind;                 // 1 tail, 2 chunk
    int u, b, hk, S, n_main;
    int r, t_lo, t_hi;        // chunk r: main tiles [t_lo, t_hi)
    int nc, tail_on;          // chunks of the unit, tail item present
};

// 0: past the end of the list, 1: a real item, 2: an empty slot of the list (unit shorter than the plan)
__device__ __forceinline__ int item_of(const DecodeArgs& a, int j, Item& it) {
    const dec::PkArgs& p = a.pk;
    if (j >= p.n_items) return 0;
    int u, r;
    if (j < p.U) {
        u = j; r = -1;
    } else {
        const uint32_t jj = (uint32_t)(j - p.U);
        u = (int)fdiv(jj, p.fd_rounds);
        r = (int)jj - u * p.rounds;
    }
    const int b = (int)fdiv((uint32_t)u, p.fd_H);
    const int S = a.seq_len[b];
    const int R = a.g.R;
    const int nqV = S > R ? S - R : 0;
    const int nqK = a.g.mode == KVT_MODE_KIVI ? p.F * (int)fdiv((uint32_t)S, p.fd_F) : nqV;
    const int n_main = (nqK < nqV ? nqK : nqV) & ~31;
    const int tiles = n_main >> 5;
    const int nc = (int)fdiv((uint32_t)(tiles + p.ch - 1), p.fd_ch);
    it.u = u; it.b = b; it.hk = u - b * a.g.H; it.S = S; it.n_main = n_main;
    it.nc = nc;
    it.tail_on = (S > n_main || tiles == 0) ? 1 : 0;
    it.r = r;
    if (r < 0) {
        if (!it.tail_on) return 2;
        it.kind = 1; it.t_lo = it.t_hi = 0;
        return 1;
    }
    if (r >= nc) return 2;
    it.kind = 2;
    it.t_lo = r * p.ch;
    it.t_hi = min(tiles, it.t_lo + p.ch);
    return 1;
}

__device__ __forceinline__ int claim(int* ctr, int lane) {
    int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1);
    return __shfl_sync(kFull, v, 0);
}

// Resolve a claimed index to the next real item (claiming again past empty slots); -1 when the list is done.
__device__ __forceinline__ int resolve(const DecodeArgs& a, int j, Item& it, int lane) {
    for (;;) {
        const int st = item_of(a, j, it);
        if (st == 1) return j;
        if (st == 0) return -1;
        j = claim(a.counters, lane);
    }
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}

// q rows of unit (b, hk) -> the warp's bf16 prefetch buffer (real heads only), asynchronously
__device__ __forceinline__ void q_prefetch(const DecodeArgs& a, uint16_t* qb, const Item& it, int lane) {
    const uint16_t* src = a.q + ((size_t)it.b * a.H_q + (size_t)it.hk * a.gq) * D;
    const int n4 = a.gq * D / 2;                         // 4-byte words (q rows are 4-byte aligned: d even)
    for (int i = lane; i < n4; i += 32) cp_async4(qb + 2 * i, src + 2 * i);
    asm volatile("cp.async.commit_group;\n" ::);
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }

// Arrival of one partial at counter c (expected n arrivals): every lane's partial stores are ordered before lane 0's
// release fence and atomic; the last arriver's acquire fence orders the merge loads after every producer's stores.
__device__ __forceinline__ bool arrive(int* c, int n, int lane) {
    __syncwarp();
    int old = 0;
    if (lane == 0) {
        fence_acq_rel_gpu();
        old = atomicAdd(c, 1);
        if (old == n - 1) {
            fence_acq_rel_gpu();
            *c = 0;                                      // reset for the next launch (nobody else touches it now)
        }
    }
    old = __shfl_sync(kFull, old, 0);
    __syncwarp();
    return old == n - 1;
}

// Merge of partial slots [head (if >= 0)] + [first, first + n) (fixed order) -> the output rows of unit (b, hk)
// (dst < 0) or partial slot dst.  Slot = [gq][D] o (unnormalised, relative to m) then [gq] (m, l).
template <int GM>
__device__ __forceinline__ void merge(const DecodeArgs& a, int head, int first, int n, int dst, int b, int hk, int lane) {
    constexpr int BT = 2;                                // items whose loads are issued together
    const int gq = a.gq;
    const size_t SB = a.pk.slot_floats;
    const int total = n + (head >= 0 ? 1 : 0);
    auto slot_of = [&](int k) -> int { return head >= 0 ? (k == 0 ? head : first + k - 1) : first + k; };
    float Mh[GM], Lh[GM], Oh[GM][4];
#pragma unroll
    for (int h = 0; h < GM; ++h) {
        Mh[h] = -INFINITY; Lh[h] = 0.0f;
        Oh[h][0] = Oh[h][1] = Oh[h][2] = Oh[h][3] = 0.0f;
    }
    for (int k = lane; k < total; k += 32) {
        const float* sp = a.parts + (size_t)slot_of(k) * SB + gq * D;
#pragma unroll
        for (int h = 0; h < GM; ++h)
            if (h < gq) Mh[h] = fmaxf(Mh[h], __ldcg(sp + 2 * h));
    }
#pragma unroll
    for (int h = 0; h < GM; ++h)
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) Mh[h] = fmaxf(Mh[h], __shfl_xor_sync(kFull, Mh[h], off));
    for (int k0 = 0; k0 < total; k0 += BT) {
        float2 ml[BT][GM];
        float4 ov[BT][GM];
#pragma unroll
        for (int q = 0; q < BT; ++q) {
            const int k = k0 + q < total ? k0 + q : total - 1;
            const float* sp = a.parts + (size_t)slot_of(k) * SB;
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                if (h < gq) {
                    ml[q][h] = __ldcg(reinterpret_cast<const float2*>(sp + gq * D + 2 * h));
                    ov[q][h] = __ldcg(reinterpret_cast<const float4*>(sp + h * D + 4 * lane));
                } else {
                    ml[q][h] = make_float2(0.f, 0.f);
                    ov[q][h] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < BT; ++q) {
            if (k0 + q < total) {
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    if (ml[q][h].y != 0.0f) {                    // O = sum_k 2^(m_k - M) O_k, L = sum_k 2^(m_k - M) l_k
                        const float sc = fexp2(ml[q][h].x - Mh[h]);
                        Lh[h] = fmaf(ml[q][h].y, sc, Lh[h]);
                        Oh[h][0] = fmaf(sc, ov[q][h].x, Oh[h][0]);
                        Oh[h][1] = fmaf(sc, ov[q][h].y, Oh[h][1]);
                        Oh[h][2] = fmaf(sc, ov[q][h].z, Oh[h][2]);
                        Oh[h][3] = fmaf(sc, ov[q][h].w, Oh[h][3]);
                    }
                }
            }
        }
    }
    if (dst < 0) {
#pragma unroll
        for (int h = 0; h < GM; ++h)
            if (h < gq) {
                const size_t row = (size_t)b * a.H_q + (size_t)hk * gq + h;
#pragma unroll
                for (int e = 0; e < 4; ++e) write_row(a, a.out, a.out_mode, row, 4 * lane + e, Mh[h], Lh[h], Oh[h][e]);
            }
    } else {
        float* sp = a.parts + (size_t)dst * SB;
#pragma unroll
        for (int h = 0; h < GM; ++h)
            if (h < gq) {
                *reinterpret_cast<float4*>(sp + h * D + 4 * lane) = make_float4(Oh[h][0], Oh[h][1], Oh[h][2], Oh[h][3]);
                if (lane == 0) *reinterpret_cast<float2*>(sp + gq * D + 2 * h) = make_float2(Mh[h], Lh[h]);
            }
    }
}

// After item `it` stored its partial (or wrote its row directly when it is the unit's only item): arrivals and merges.
template <int GM>
__device__ __forceinline__ void finish_item(const DecodeArgs& a, const Item& it, int lane) {
    const dec::PkArgs& p = a.pk;
    const bool two = it.nc > p.gs;
    const int ng = two ? (it.nc + p.gs - 1) / p.gs : it.nc;
    const int n_unit = it.tail_on + ng;
    if (n_unit == 1 && (it.kind == 1 || !two)) return;          // wrote its row directly
    const int chunk0 = p.U + it.u * p.rounds;                   // slot of chunk 0 of the unit
    const int group0 = p.U + p.U * p.rounds + it.u * p.maxg;    // slot of group 0 of the unit
    // level 0: this chunk's group (units of > gs chunks); level 1: the unit (one merge call site: registers)
    for (int lvl = (it.kind == 2 && two) ? 0 : 1; lvl < 2; ++lvl) {
        const int g = it.r / p.gs;
        const int gsz = lvl == 0 ? min(p.gs, it.nc - g * p.gs) : n_unit;
        int* const ctr = lvl == 0 ? a.counters + 2 + p.U + it.u * dec::kMaxGroups + g : a.counters + 2 + it.u;
        if (!arrive(ctr, gsz, lane)) return;
        merge<GM>(a, lvl == 0 ? -1 : (it.tail_on ? it.u : -1), lvl == 0 ? chunk0 + g * p.gs : (two ? group0 : chunk0),
                  lvl == 0 ? gsz : ng, lvl == 0 ? group0 + g : -1, it.b, it.hk, lane);
    }
}

__device__ __forceinline__ const uint8_t* bcast_ptr(const uint8_t* p) {
    const unsigned long long v = __shfl_sync(kFull, reinterpret_cast<unsigned long long>(p), 0);
    return reinterpret_cast<const uint8_t*>(v);
}

template <int KB, int VB, int GM, bool KPT, bool PAGED>
__global__ void __launch_bounds__(PGeo<KB, VB, GM>::NW * 32, 1) decode_pk_kernel(DecodeArgs a) {
    using P = PGeo<KB, VB, GM>;
    using G0 = typename P::G0;
    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(kFull, tid >> 5, 0);
    const int gid = lane >> 2, tig = lane & 3;
    const Geometry& g = a.g;
    const int gq = a.gq;
    int* const claim_ctr = a.counters;                  // [0] claims, [1] exits

    uint8_t* wbase = smem + (size_t)warp * P::WARP_BYTES;
    uint32_t* w_s = reinterpret_cast<uint32_t*>(wbase + P::W_OFF);
    uint32_t* sh_s = reinterpret_cast<uint32_t*>(wbase + P::SH_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + P::BAR_OFF);
    float* q_s = reinterpret_cast<float*>(wbase + P::Q_OFF);
    uint16_t* qb = reinterpret_cast<uint16_t*>(wbase + P::QB_OFF);

    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < P::NS; ++st) mbar_init(bars + st);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int i = lane; i < P::W_BYTES / 4; i += 32) w_s[i] = 0u;
    __syncwarp();

    // Programmatic dependent launch: only kvt_append_decode_attention (a.early) lets the first claim and q copy
    // (neither touches the cache) overlap the preceding append; otherwise wait at entry.
    if (!a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    int cur_j;
    {
        Item first;
        cur_j = resolve(a, claim(claim_ctr, lane), first, lane);
        if (cur_j >= 0) q_prefetch(a, qb, first, lane);
    }
    if (a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");

    // softmax heads of this thread (the QK D columns it holds after the hi/lo fold)
    const int hA = (GM == 8) ? 2 * tig : 2 * (tig & 1);
    const int gsh = (GM == 4) ? 2 * (tig >> 1) : 0;
    constexpr int NGL = (GM == 4) ? 2 : 4;
    float* qmax_s = reinterpret_cast<float*>(sh_s);      // [GM] during the q setup (the scale slots are free then)

    uint32_t g_it = 0;                                   // tiles streamed through this warp's ring so far
    // first tile of a chunk item into ring position n (the address is made warp-uniform for the bulk copy)
    auto issue_first = [&](const Item& itm, uint32_t n) {
        const uint8_t* src = PAGED
            ? a.c.k_codes + ((size_t)a.c.bt[(size_t)itm.b * a.c.max_pages + itm.t_lo] * g.H + itm.hk) * P::STAGE
            : a.c.k_codes + ((size_t)itm.b * g.H + itm.hk) * g.kc + (size_t)itm.t_lo * P::STAGE;
        src = bcast_ptr(src);
        if (lane == 0) {
            const int st = (int)(n % P::NS);
            mbar_expect_tx(bars + st, P::STAGE);
            bulk_g2s(wbase + st * P::STAGE, src, P::STAGE, bars + st);
        }
    };
    if (cur_j >= 0) {
        Item first;
        item_of(a, cur_j, first);
        if (first.kind == 2) issue_first(first, g_it);
    }

    while (cur_j >= 0) {
        // ---- q of the current unit: bf16 prefetch -> fp32 q_s (zero rows for padded heads), per-head max ----
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int h = 0; h < GM; ++h) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (h < gq) {
                const uint2 w = *reinterpret_cast<const uint2*>(qb + h * D + 4 * lane);
                v = make_float4(bf2f(w.x & 0xffffu), bf2f(w.x >> 16), bf2f(w.y & 0xffffu), bf2f(w.y >> 16));
            }
            *reinterpret_cast<float4*>(q_s + h * D + 4 * lane) = v;
            float m = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, off));
            if (lane == 0) qmax_s[h] = m;
        }
        __syncwarp();
        Item it;
        item_of(a, cur_j, it);
        const size_t SB = a.pk.slot_floats;
        const bool two = it.nc > a.pk.gs;
        const int n_unit = it.tail_on + (two ? (it.nc + a.pk.gs - 1) / a.pk.gs : it.nc);
        int nxt_j = -1;

        if (it.kind == 1) {
            // ================= tail item: tokens [n_main, S) on the CUDA cores =================
            // claim the next item first so its first tile and q copy stream in while the tail runs
            {
                Item nxt;
                nxt_j = resolve(a, claim(claim_ctr, lane), nxt, lane);
                if (nxt_j >= 0) {
                    q_prefetch(a, qb, nxt, lane);
                    if (nxt.kind == 2) issue_first(nxt, g_it);
                }
            }
            Slice tl;
            tl.kc = PAGED ? a.c.k_codes + (size_t)it.hk * g.rec : a.c.k_codes + ((size_t)it.b * g.H + it.hk) * g.kc;
            tl.km = nullptr; tl.vc = nullptr; tl.vm = nullptr;
            tl.kr = a.c.k_resid + ((size_t)it.b * g.H + it.hk) * (g.kr / 2);
            tl.vr = g.vr ? a.c.v_resid + ((size_t)it.b * g.H + it.hk) * (g.vr / 2) : nullptr;
            if (PAGED) {
                tl.bt = a.c.bt + (size_t)it.b * a.c.max_pages;
                tl.pstride = (size_t)g.H * g.rec;
            }
            const int nqK = nq_key(g.mode, g.kb, g.G, g.R, it.S);
            const int nqV = nq_per_token(g.vb, g.R, it.S);
            float* pbuf = reinterpret_cast<float*>(w_s);               // [32 tokens][GM]
            float mt[GM], lt[GM], ot[GM][4];
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                mt[h] = -INFINITY; lt[h] = 0.0f;
                ot[h][0] = ot[h][1] = ot[h][2] = ot[h][3] = 0.0f;
            }
            for (int t0 = it.n_main; t0 < it.S; t0 += 32) {
                const int t = t0 + lane;
                const bool valid = t < it.S;
                float acc[GM];
#pragma unroll
                for (int h = 0; h < GM; ++h) acc[h] = 0.0f;
                if (valid) {
#pragma unroll 8
                    for (int c4 = 0; c4 < 32; ++c4) {
                        float kx[4];
                        dec::tail_k<KB, !KPT, true>(tl, g, t, nqK, c4, kx);
#pragma unroll
                        for (int h = 0; h < GM; ++h) {
                            const float4 qv = *reinterpret_cast<const float4*>(q_s + h * D + 4 * c4);
                            acc[h] = fmaf(qv.x, kx[0], fmaf(qv.y, kx[1], fmaf(qv.z, kx[2], fmaf(qv.w, kx[3], acc[h]))));
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    const float lg = valid ? acc[h] * a.scale_log2 : -INFINITY;
                    float mx = lg;
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
                    const float m_new = fmaxf(mt[h], mx);                    // finite: lane 0 is always valid
                    const float al = fexp2(mt[h] - m_new);
                    const float p = valid ? fexp2(lg - m_new) : 0.0f;
                    float sum = p;
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(kFull, sum, off);
                    lt[h] = lt[h] * al + sum;
                    mt[h] = m_new;
#pragma unroll
                    for (int e = 0; e < 4; ++e) ot[h][e] *= al;
                    pbuf[lane * GM + h] = p;
                }
                __syncwarp();
                const int n = it.S - t0 < 32 ? it.S - t0 : 32;
#pragma unroll 8
                for (int i = 0; i < n; ++i) {
                    float vx[4];
                    dec::tail_v<VB, true>(tl, g, t0 + i, nqV, lane, vx);
#pragma unroll
                    for (int h = 0; h < GM; h += 4) {
                        const float4 p4 = *reinterpret_cast<const float4*>(pbuf + i * GM + h);
                        const float pp[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
                        for (int hh = 0; hh < 4; ++hh)
#pragma unroll
                            for (int e = 0; e < 4; ++e) ot[h + hh][e] = fmaf(pp[hh], vx[e], ot[h + hh][e]);
                    }
                }
                __syncwarp();
            }
            // restore the zero weight tile for the next chunk
            for (int i = lane; i < P::W_BYTES / 4; i += 32) w_s[i] = 0u;
            // ---- store: direct output (the unit's only item) or the tail slot; lane = channels 4 lane .. + 3 ----
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                if (h >= gq) continue;
                if (n_unit == 1) {
                    const size_t row = (size_t)it.b * a.H_q + (size_t)it.hk * gq + h;
#pragma unroll
                    for (int e = 0; e < 4; ++e) write_row(a, a.out, a.out_mode, row, 4 * lane + e, mt[h], lt[h], ot[h][e]);
                } else {
                    float* sp = a.parts + (size_t)it.u * SB;
                    *reinterpret_cast<float4*>(sp + h * D + 4 * lane) = make_float4(ot[h][0], ot[h][1], ot[h][2], ot[h][3]);
                    if (lane == 0) *reinterpret_cast<float2*>(sp + gq * D + 2 * h) = make_float2(mt[h], lt[h]);
                }
            }
        } else {
            // ================= chunk item: main tiles [t_lo, t_hi) on the tensor cores =================
            uint32_t q_h[16];
            float qa_inv[2];
            {
                const int qh = (GM == 4) ? (gid & 3) : gid;
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
                for (int j = 0; j < 2; ++j) qa_inv[j] = pow2(24 - (7 - frexp_e(qmax_s[hA + j])));
            }
            float qg[KPT ? 4 : 1][2];
            if constexpr (KPT) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
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
            __syncwarp();                                   // qmax_s (in the scale-slot area) read before reuse

            float m_run[2] = {-INFINITY, -INFINITY};
            float l_part[2] = {0.0f, 0.0f};
            float2 zacc2[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) zacc2[i][0] = zacc2[i][1] = make_float2(0.0f, 0.0f);
            float o[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
            int kp = 126;
            const int n_t = it.t_hi - it.t_lo;
            // ring source of tile t_lo + i: dense = base + i * STAGE; paged = pool + (bt[t_lo + i] * H + hk) * STAGE
            const uint8_t* src_base = bcast_ptr(PAGED ? a.c.k_codes + (size_t)it.hk * P::STAGE
                                                      : a.c.k_codes + ((size_t)it.b * g.H + it.hk) * g.kc + (size_t)it.t_lo * P::STAGE);
            const int32_t* bt_row = PAGED ? a.c.bt + (size_t)it.b * a.c.max_pages + it.t_lo : nullptr;
            int raw = 0;
            for (int i = 0; i < n_t; ++i) {
                // claim early (its latency hides under this tile), resolve at the last tile
                if (i == (n_t >= 2 ? n_t - 2 : 0) && lane == 0) raw = atomicAdd(claim_ctr, 1);
                if (i + 1 < n_t) {
                    if (lane == 0) {
                        const int st = (int)((g_it + 1) % P::NS);
                        mbar_expect_tx(bars + st, P::STAGE);
                        const uint8_t* src = PAGED ? src_base + (size_t)bt_row[i + 1] * g.H * P::STAGE
                                                   : src_base + (size_t)(i + 1) * P::STAGE;
                        bulk_g2s(wbase + st * P::STAGE, src, P::STAGE, bars + st);
                    }
                } else {
                    Item nxt;
                    nxt_j = resolve(a, __shfl_sync(kFull, raw, 0), nxt, lane);
                    if (nxt_j >= 0) {
                        q_prefetch(a, qb, nxt, lane);
                        if (nxt.kind == 2) issue_first(nxt, g_it + 1);
                    }
                }
                mbar_wait(bars + (g_it % P::NS), (g_it / P::NS) & 1);
                const uint8_t* sb = wbase + (g_it % P::NS) * P::STAGE;
                ++g_it;
                const uint8_t* kc_s = sb + G0::K_OFF;
                const uint32_t* km_s = reinterpret_cast<const uint32_t*>(sb + G0::KM_OFF);
                const uint8_t* vc_s = sb + G0::V_OFF;
                const uint32_t* vm_s = reinterpret_cast<const uint32_t*>(sb + G0::VM_OFF);

                // (1) key block meta: scale slots (fp16 x 2^sb) and the zero-point bias sum_c q_c z_c
                float bias[2] = {0.0f, 0.0f};
                float ks_inv = 1.0f;
                uint32_t mk[KPT ? 2 : 1][2][4];
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
                    uint32_t smb = max(max(mw[0] & 0xffffu, mw[1] & 0xffffu), max(mw[2] & 0xffffu, mw[3] & 0xffffu));
                    smb = __reduce_max_sync(kFull, smb);
                    const int sbx = 7 - frexp_e(bf2f(smb));
                    const float ssc = pow2(sbx);
                    ks_inv = pow2(-sbx);
                    const int code0 = k_slot_of<KB>((4 * lane) & 31);
                    __half* shh = reinterpret_cast<__half*>(sh_s) + ((lane >> 3) * P::SH_STRIDE + (code0 >> 1)) * 2 + (code0 & 1);
                    float z[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        shh[KB == 8 ? e : 2 * e] = __float2half_rn(bf2f(mw[e] & 0xffffu) * ssc);
                        z[e] = bf2f(mw[e] >> 16);
                    }
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
                    bias[1] = __shfl_sync(kFull, bz[0], hA + 1);
                }
                __syncwarp();
                // (2) B operand of QK: q_h * s_h split exactly into hi + lo
                uint32_t bq[16], bq_lo[(GM == 8 && !KPT) ? 16 : 1];
                if constexpr (KPT) {
#pragma unroll
                    for (int m = 0; m < 16; ++m) bq[m] = q_h[m];
                } else {
                    const uint4* shv = reinterpret_cast<const uint4*>(sh_s + tig * P::SH_STRIDE);
#pragma unroll
                    for (int uu = 0; uu < 4; ++uu) {
                        const uint4 s4 = shv[uu];
                        const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int m = 4 * uu + e;
                            const __half2 hi = __hmul2(u2h(q_h[m]), u2h(sv[e]));
                            if constexpr (GM == 8 && !KPT) {
                                bq[m] = h2u(hi);
                                bq_lo[m] = h2u(__hfma2(u2h(q_h[m]), u2h(sv[e]), __hneg2(hi)));
                            } else {
                                bq[m] = (gid >= 4) ? h2u(__hfma2(u2h(q_h[m]), u2h(sv[e]), __hneg2(hi))) : h2u(hi);
                            }
                        }
                    }
                }
                // (3) QK on the tensor cores
                float dq[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
                if constexpr (KPT) {
                    uint32_t w[4][KB == 2 ? 4 : KB];
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) {
                        const uint8_t* r0 = kc_s + (8 * rr + gid) * G0::KROW;
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
                            for (int i2 = 0; i2 < 4; ++i2) {
                                const uint32_t mw = mk[mt][i2 >> 1][gg];
                                dq[mt][i2] = fmaf(bf2f(mw & 0xffffu) * qa_inv[i2 & 1], acc[mt][i2],
                                                  fmaf(bf2f(mw >> 16), qg[gg][i2 & 1], dq[mt][i2]));
                            }
                    }
                } else {
                    uint32_t w[4][KB];
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) {
                        const uint8_t* r0 = kc_s + (8 * rr + gid) * G0::KROW + tig * 4 * KB;
                        if constexpr (KB == 2) {
                            const uint2 x = *reinterpret_cast<const uint2*>(r0);
                            w[rr][0] = x.x; w[rr][1] = x.y;
                        } else {
#pragma unroll
                            for (int uu = 0; uu < KB / 4; ++uu) {
                                const uint4 x = reinterpret_cast<const uint4*>(r0)[uu];
                                w[rr][4 * uu] = x.x; w[rr][4 * uu + 1] = x.y; w[rr][4 * uu + 2] = x.z; w[rr][4 * uu + 3] = x.w;
                            }
                        }
                    }
                    float de[2][4], dd[2][4];
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int i2 = 0; i2 < 4; ++i2) de[mt][i2] = dd[mt][i2] = 0.0f;
#pragma unroll
                    for (int s = 0; s < 8; ++s) {
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt) {
                            float* acc = (s & 1) ? dd[mt] : de[mt];
                            const uint32_t a0 = k_slot<KB>(w[2 * mt], 2 * s), a1 = k_slot<KB>(w[2 * mt + 1], 2 * s);
                            const uint32_t a2 = k_slot<KB>(w[2 * mt], 2 * s + 1), a3 = k_slot<KB>(w[2 * mt + 1], 2 * s + 1);
                            hmma(acc, a0, a1, a2, a3, bq[2 * s], bq[2 * s + 1]);
                            if constexpr (GM == 8) hmma(acc, a0, a1, a2, a3, bq_lo[2 * s], bq_lo[2 * s + 1]);
                        }
                    }
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int i2 = 0; i2 < 4; ++i2) {
                            dq[mt][i2] = de[mt][i2] + dd[mt][i2];
                            if constexpr (GM == 4) dq[mt][i2] += __shfl_xor_sync(kFull, dq[mt][i2], 2);
                        }
                }
                // (4) logits (log2 domain) and the online softmax with a lazy reference max
                float alpha[2], p[2][2][2];
                bool resc = false;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const float cs = KPT ? a.scale_log2 : a.scale_log2 * qa_inv[j] * ks_inv;
                    const float cb = KPT ? 0.0f : a.scale_log2 * bias[j];
                    float l4[4];
                    l4[0] = fmaf(dq[0][j], cs, cb);
                    l4[1] = fmaf(dq[0][2 + j], cs, cb);
                    l4[2] = fmaf(dq[1][j], cs, cb);
                    l4[3] = fmaf(dq[1][2 + j], cs, cb);
                    float mx = fmaxf(fmaxf(l4[0], l4[1]), fmaxf(l4[2], l4[3]));
                    alpha[j] = 1.0f;
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
                {
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
                            for (int gr = 0; gr < NGL; ++gr) smb = max(smb, mw[mt][r][gr] & 0xffffu);
                        }
                    smb = __reduce_max_sync(kFull, smb);
                    const int kt = 7 - frexp_e(bf2f(smb));
                    if (kt < kp) {
                        if (i > 0) { kfac = pow2(kt - kp < -126 ? -126 : kt - kp); resc = true; }
                        kp = kt;
                    }
                    const float ksc = pow2(kp);
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
                // (6) PV on the tensor cores: 8 m-tiles (gamma, mu) x 2 k-steps of 16 tokens
                if (__any_sync(kFull, resc)) {
                    const float r0 = alpha[0] * kfac, r1 = alpha[1] * kfac;
#pragma unroll
                    for (int i2 = 0; i2 < 8; ++i2) { o[i2][0] *= r0; o[i2][1] *= r1; o[i2][2] *= r0; o[i2][3] *= r1; }
                }
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    VRaw<VB> rv;
                    v_load<VB>(vc_s, ks, tig, gid, rv);
#pragma unroll
                    for (int gam = 0; gam < 4; ++gam) {
                        const uint32_t* wr = w_s + (gam * 2 + ks) * 64 + 4 * (gam >> 1) + gid;
                        const uint32_t b0 = wr[tig * 8], b1 = wr[(tig + 4) * 8];
                        uint32_t hA4[4], hB4[4];
                        v_frag<VB>(rv, gam, hA4, hB4);
                        hmma(o[2 * gam], hA4[0], hA4[1], hB4[0], hB4[1], b0, b1);
                        hmma(o[2 * gam + 1], hA4[2], hA4[3], hB4[2], hB4[3], b0, b1);
                    }
                }
                __syncwarp();
            }
            // ---- chunk epilogue: l over the 8 row-groups, zero sums, O = D * 2^(24 - P(row) - kp) + zacc ----
            float zacc[4][2];
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2)
#pragma unroll
                for (int j = 0; j < 2; ++j) zacc[i2][j] = zacc2[i2][j].x + zacc2[i2][j].y;
            float Lj[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                float l = (GM == 8 || tig < 2) ? l_part[j] : 0.0f;
                l += __shfl_xor_sync(kFull, l, 4);
                l += __shfl_xor_sync(kFull, l, 8);
                l += __shfl_xor_sync(kFull, l, 16);
                Lj[j] = l;
#pragma unroll
                for (int gam = 0; gam < 4; ++gam) {
                    float z = zacc[gam][j];
                    z += __shfl_xor_sync(kFull, z, 4);
                    z += __shfl_xor_sync(kFull, z, 8);
                    z += __shfl_xor_sync(kFull, z, 16);
                    zacc[gam][j] = z;
                }
            }
            if constexpr (GM == 4) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    zacc[2][j] = __shfl_xor_sync(kFull, zacc[0][j], 2);
                    zacc[3][j] = __shfl_xor_sync(kFull, zacc[1][j], 2);
                }
            }
            // ---- store: owner lanes hold heads 2 tig + j, channels c = 32 gamma + 4 gid + 2 mu (+1) ----
            item_of(a, cur_j, it);                          // (re-derived: keeps the item out of the tile loop)
            const bool direct = n_unit == 1 && !two;
            if ((GM == 8) || (tig < 2)) {
                float* sp = a.parts + (size_t)(a.pk.U + it.u * a.pk.rounds + it.r) * SB;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int h = 2 * tig + j;
                    if (h >= gq) continue;
                    const size_t row = (size_t)it.b * a.H_q + (size_t)it.hk * gq + h;
#pragma unroll
                    for (int gam = 0; gam < 4; ++gam)
#pragma unroll
                        for (int mu = 0; mu < 2; ++mu) {
                            const int c = 32 * gam + 4 * gid + 2 * mu;
                            const float v0 = o[2 * gam + mu][j] * pow2(24 - VP<VB>(2 * mu) - kp) + zacc[gam][j];
                            const float v1 = o[2 * gam + mu][2 + j] * pow2(24 - VP<VB>(2 * mu + 1) - kp) + zacc[gam][j];
                            if (direct) {
                                write_row(a, a.out, a.out_mode, row, c, m_run[j], Lj[j], v0);
                                write_row(a, a.out, a.out_mode, row, c + 1, m_run[j], Lj[j], v1);
                            } else {
                                *reinterpret_cast<float2*>(sp + h * D + c) = make_float2(v0, v1);
                            }
                        }
                    if (!direct && gid == 0) *reinterpret_cast<float2*>(sp + gq * D + 2 * h) = make_float2(m_run[j], Lj[j]);
                }
            }
        }
        finish_item<GM>(a, it, lane);
        cur_j = nxt_j;
    }

    // the last warp to leave resets the claim counter for the next launch (every warp has made its final claim)
    __syncwarp();
    if (lane == 0) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars)));
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars + 1)));
        const int total = (int)(gridDim.x * (blockDim.x >> 5));
        if (atomicAdd(claim_ctr + 1, 1) == total - 1) {
            claim_ctr[0] = 0;
            claim_ctr[1] = 0;
        }
    }
}

}  // namespace pk
}  // namespace kvt

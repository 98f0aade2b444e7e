// kvt_decode_pk.cuh — K2 persistent decode attention with a static per-warp work split (DESIGN.md §5,
// "persistent kernel").
//
// Same arithmetic per 32-token tile as kvt_decode_mma.cuh (tile records, fp16-subnormal codes on the tensor
// cores, lazy online softmax, fp32 zero-point sums); a different work schedule:
//
//   * one CTA per SM with NW warps (16 for g <= 4, 12 for g <= 8, fewer when the ring of a wide instance does not
//     fit), each warp an independent worker with its own TMA ring, weight tile, q copy and softmax state;
//   * the work of all (b, kv head) units is laid out unit after unit in a planned cost space (unit u = its tail
//     item, costed TC tiles, then T_plan main tiles; the plan length bounds every real length), and warp w of the
//     N = CTAs x NW warps takes the contiguous share [w V / N, (w + 1) V / N) of it — stream-K at warp
//     granularity: a warp sees one or two units, so per-segment costs (q setup, epilogue) are paid once or twice
//     per warp, and every SM gets the same work whatever B * H_kv is (512 units on 148 SMs no longer means 4
//     units on some SMs and 3 on others);
//   * each warp segment ("piece") leaves its (m, l, o) partial (o unnormalised) in a workspace slot, the tail its
//     own slot; after a CTA barrier the CTA merges, for every unit it touched, the tail and its pieces in a fixed
//     order, writing the output row when the unit lies inside the CTA, else a CTA partial whose last arriver (per-
//     unit counter) merges the CTA partials and writes the row.
//
// The partition is a pure function of (B, H, the plan length, the SM count and warps per CTA) and the merge order
// is fixed, so results are bitwise reproducible (A23).
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

// The warp whose share holds planned position x (shares [w V / N, (w + 1) V / N))
__device__ __forceinline__ int warp_of(long long x, long long V, int N) { return (int)(((x + 1) * N - 1) / V); }

// Warp w's part of unit u (whose planned positions are [u Cp, (u + 1) Cp): tail first, then T_plan tiles).
struct Piece {
    int b, hk, S, n_main, tiles;     // the unit's actual geometry
    int t_lo, t_hi;                  // this warp's main tiles, clipped to the unit's actual tiles
    int tail;                        // this warp owns the unit's tail (its share holds position u Cp)
    int k;                           // piece index of this warp within the unit (slot)
};
__device__ __forceinline__ void piece_of(const DecodeArgs& a, int u, long long lo, long long hi, int w, Piece& pc) {
    const dec::PkArgs& p = a.pk;
    const int b = (int)fdiv((uint32_t)u, p.fd_H);
    const int S = a.seq_len[b];
    const int R = a.g.R;
    const int nqV = S > R ? S - R : 0;
    const int nqK = a.g.mode == KVT_MODE_KIVI ? p.F * (int)fdiv((uint32_t)S, p.fd_F) : nqV;
    const int n_main = (nqK < nqV ? nqK : nqV) & ~31;
    const long long base = (long long)u * p.Cp;
    pc.b = b; pc.hk = u - b * a.g.H; pc.S = S; pc.n_main = n_main; pc.tiles = n_main >> 5;
    pc.tail = (lo <= base && base < hi) ? 1 : 0;
    const long long t0 = lo - base - p.TC, t1 = hi - base - p.TC;
    pc.t_lo = (int)min((long long)pc.tiles, max(0ll, t0));
    pc.t_hi = (int)min((long long)pc.tiles, max(0ll, t1));
    pc.k = w - warp_of(base, p.V, p.N);
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}

// q rows of unit (b, hk) -> the warp's bf16 prefetch buffer (real heads only), asynchronously
__device__ __forceinline__ void q_prefetch(const DecodeArgs& a, uint16_t* qb, int b, int hk, int lane) {
    const uint16_t* src = a.q + ((size_t)b * a.H_q + (size_t)hk * a.gq) * D;
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
    const dec::PkArgs& pa = a.pk;
    const int gq = a.gq;
    const size_t SB = pa.slot_floats;

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

    const int w = blockIdx.x * P::NW + warp;
#if KVT_TRACE
    // per warp: [sm | warp << 16 | cta << 32, start, work done, merges done, tail ns, tiles, units]
    unsigned long long tr_t0, tr_tail = 0, tr_tiles = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_t0));
#endif
    const long long lo = (long long)w * pa.V / pa.N, hi = (long long)(w + 1) * pa.V / pa.N;
    const int u0 = lo < hi ? (int)(lo / pa.Cp) : 0, u1 = lo < hi ? (int)((hi - 1) / pa.Cp) : -1;

    // Programmatic dependent launch: only kvt_append_decode_attention (a.early) lets the first q copy (it does not
    // touch the cache) overlap the preceding append; otherwise wait at entry.
    if (!a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    Piece nx;
    if (u0 <= u1) {
        piece_of(a, u0, lo, hi, w, nx);
        q_prefetch(a, qb, nx.b, nx.hk, lane);
    }
    if (a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");

    // softmax heads of this thread (the QK D columns it holds after the hi/lo fold)
    const int hA = (GM == 8) ? 2 * tig : 2 * (tig & 1);
    const int gsh = (GM == 4) ? 2 * (tig >> 1) : 0;
    constexpr int NGL = (GM == 4) ? 2 : 4;
    float* qmax_s = reinterpret_cast<float*>(sh_s);      // [GM] during the q setup (the scale slots are free then)

    uint32_t g_it = 0;                                   // tiles streamed through this warp's ring so far
    // tile t of unit (b, hk) into ring position n (the address is made warp-uniform for the bulk copy)
    auto issue_tile = [&](int b, int hk, int t, uint32_t n) {
        const uint8_t* src = PAGED
            ? a.c.k_codes + ((size_t)a.c.bt[(size_t)b * a.c.max_pages + t] * g.H + hk) * P::STAGE
            : a.c.k_codes + ((size_t)b * g.H + hk) * g.kc + (size_t)t * P::STAGE;
        src = bcast_ptr(src);
        if (lane == 0) {
            const int st = (int)(n % P::NS);
            mbar_expect_tx(bars + st, P::STAGE);
            bulk_g2s(wbase + st * P::STAGE, src, P::STAGE, bars + st);
        }
    };
    if (u0 <= u1 && nx.t_hi > nx.t_lo) issue_tile(nx.b, nx.hk, nx.t_lo, g_it);

    for (int u = u0; u <= u1; ++u) {
        // ---- q of unit u: bf16 prefetch -> fp32 q_s (zero rows for padded heads), per-head max ----
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int h = 0; h < GM; ++h) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (h < gq) {
                const uint2 wq = *reinterpret_cast<const uint2*>(qb + h * D + 4 * lane);
                v = make_float4(bf2f(wq.x & 0xffffu), bf2f(wq.x >> 16), bf2f(wq.y & 0xffffu), bf2f(wq.y >> 16));
            }
            *reinterpret_cast<float4*>(q_s + h * D + 4 * lane) = v;
            float m = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, off));
            if (lane == 0) qmax_s[h] = m;
        }
        __syncwarp();
        Piece pc;
        piece_of(a, u, lo, hi, w, pc);
        // next unit of this share: its q rows (and, below, its first tile) stream in during this piece
        bool next_pending = u < u1;
#if KVT_TRACE
        unsigned long long tr_a;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_a));
#endif
        if (pc.tail) {
            // ================= the unit's tail: tokens [n_main, S) on the CUDA cores =================
            if (pc.t_hi <= pc.t_lo && next_pending) {       // no tiles here: prefetch the next unit now
                piece_of(a, u + 1, lo, hi, w, nx);
                q_prefetch(a, qb, nx.b, nx.hk, lane);
                if (nx.t_hi > nx.t_lo) issue_tile(nx.b, nx.hk, nx.t_lo, g_it);
                next_pending = false;
            }
            Slice tl;
            tl.kc = PAGED ? a.c.k_codes + (size_t)pc.hk * g.rec : a.c.k_codes + ((size_t)pc.b * g.H + pc.hk) * g.kc;
            tl.km = nullptr; tl.vc = nullptr; tl.vm = nullptr;
            tl.kr = a.c.k_resid + ((size_t)pc.b * g.H + pc.hk) * (g.kr / 2);
            tl.vr = g.vr ? a.c.v_resid + ((size_t)pc.b * g.H + pc.hk) * (g.vr / 2) : nullptr;
            if (PAGED) {
                tl.bt = a.c.bt + (size_t)pc.b * a.c.max_pages;
                tl.pstride = (size_t)g.H * g.rec;
            }
            const int nqK = nq_key(g.mode, g.kb, g.G, g.R, pc.S);
            const int nqV = nq_per_token(g.vb, g.R, pc.S);
            float* pbuf = reinterpret_cast<float*>(w_s);               // [32 tokens][GM]
            float mt[GM], lt[GM], ot[GM][4];
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                mt[h] = -INFINITY; lt[h] = 0.0f;
                ot[h][0] = ot[h][1] = ot[h][2] = ot[h][3] = 0.0f;
            }
            for (int t0 = pc.n_main; t0 < pc.S; t0 += 32) {
                const int t = t0 + lane;
                const bool valid = t < pc.S;
                float acc[GM];
#pragma unroll
                for (int h = 0; h < GM; ++h) acc[h] = 0.0f;
                if (valid) {
#pragma unroll 4
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
                const int n = pc.S - t0 < 32 ? pc.S - t0 : 32;
#pragma unroll 4
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
            for (int i = lane; i < P::W_BYTES / 4; i += 32) w_s[i] = 0u;   // the zero weight tile for the next tiles
            float* sp = a.parts + (size_t)(pa.U * pa.maxp + u) * SB;        // the unit's tail slot
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                if (h >= gq) continue;
                *reinterpret_cast<float4*>(sp + h * D + 4 * lane) = make_float4(ot[h][0], ot[h][1], ot[h][2], ot[h][3]);
                if (lane == 0) *reinterpret_cast<float2*>(sp + gq * D + 2 * h) = make_float2(mt[h], lt[h]);
            }
        }
#if KVT_TRACE
        if (pc.tail) {
            unsigned long long tr_b;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_b));
            tr_tail += tr_b - tr_a;
        }
        tr_tiles += pc.t_hi > pc.t_lo ? pc.t_hi - pc.t_lo : 0;
#endif
        float* const psp = a.parts + (size_t)(u * pa.maxp + pc.k) * SB;       // this warp's piece slot of unit u
        if (pc.t_hi <= pc.t_lo) {
            // ---- no main tiles in this share of the unit: an empty piece (l = 0) ----
            if (lane < gq) *reinterpret_cast<float2*>(psp + gq * D + 2 * lane) = make_float2(-INFINITY, 0.0f);
            if (next_pending) {
                piece_of(a, u + 1, lo, hi, w, nx);
                q_prefetch(a, qb, nx.b, nx.hk, lane);
                if (nx.t_hi > nx.t_lo) issue_tile(nx.b, nx.hk, nx.t_lo, g_it);
            }
            continue;
        }
        // ================= main tiles [t_lo, t_hi) on the tensor cores =================
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
        const int n_t = pc.t_hi - pc.t_lo;
        // ring source of tile t_lo + i: dense = base + i * STAGE; paged = pool + (bt[t_lo + i] * H + hk) * STAGE
        const uint8_t* src_base = bcast_ptr(PAGED ? a.c.k_codes + (size_t)pc.hk * P::STAGE
                                                  : a.c.k_codes + ((size_t)pc.b * g.H + pc.hk) * g.kc + (size_t)pc.t_lo * P::STAGE);
        const int32_t* bt_row = PAGED ? a.c.bt + (size_t)pc.b * a.c.max_pages + pc.t_lo : nullptr;
        for (int i = 0; i < n_t; ++i) {
            if (i + 1 < n_t) {
                if (lane == 0) {
                    const int st = (int)((g_it + 1) % P::NS);
                    mbar_expect_tx(bars + st, P::STAGE);
                    const uint8_t* src = PAGED ? src_base + (size_t)bt_row[i + 1] * g.H * P::STAGE
                                               : src_base + (size_t)(i + 1) * P::STAGE;
                    bulk_g2s(wbase + st * P::STAGE, src, P::STAGE, bars + st);
                }
            } else if (next_pending) {                  // last tile: the next unit's q rows and first tile
                piece_of(a, u + 1, lo, hi, w, nx);
                q_prefetch(a, qb, nx.b, nx.hk, lane);
                if (nx.t_hi > nx.t_lo) issue_tile(nx.b, nx.hk, nx.t_lo, g_it + 1);
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
        // ---- piece epilogue: l over the 8 row-groups, zero sums, O = D * 2^(24 - P(row) - kp) + zacc ----
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
        // owner lanes hold heads 2 tig + j, channels c = 32 gamma + 4 gid + 2 mu (+1)
        if ((GM == 8) || (tig < 2)) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int h = 2 * tig + j;
                if (h >= gq) continue;
#pragma unroll
                for (int gam = 0; gam < 4; ++gam)
#pragma unroll
                    for (int mu = 0; mu < 2; ++mu) {
                        const int c = 32 * gam + 4 * gid + 2 * mu;
                        const float v0 = o[2 * gam + mu][j] * pow2(24 - VP<VB>(2 * mu) - kp) + zacc[gam][j];
                        const float v1 = o[2 * gam + mu][2 + j] * pow2(24 - VP<VB>(2 * mu + 1) - kp) + zacc[gam][j];
                        *reinterpret_cast<float2*>(psp + h * D + c) = make_float2(v0, v1);
                    }
                if (gid == 0) *reinterpret_cast<float2*>(psp + gq * D + 2 * h) = make_float2(m_run[j], Lj[j]);
            }
        }
    }

    // An empty share (fewer planned positions than warps, single-CTA launches only) inside a unit still owns a
    // piece index of that unit: leave an empty partial there.
    if (lo == hi && lo < pa.V && lo % pa.Cp != 0) {
        const int u = (int)(lo / pa.Cp);
        float* sp = a.parts + (size_t)(u * pa.maxp + w - warp_of((long long)u * pa.Cp, pa.V, pa.N)) * SB;
        if (lane < gq) *reinterpret_cast<float2*>(sp + gq * D + 2 * lane) = make_float2(-INFINITY, 0.0f);
    }
    if (lane == 0) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars)));
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars + 1)));
    }

#if KVT_TRACE
    unsigned long long tr_t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_t1));
#endif
    // ================= merges: per unit of this CTA, then across CTAs =================
    __syncthreads();                                     // every piece of this CTA is in its slot
    const int wc0 = blockIdx.x * P::NW, wc1 = wc0 + P::NW - 1;
    const long long loc = (long long)wc0 * pa.V / pa.N, hic = (long long)(wc1 + 1) * pa.V / pa.N;
    if (loc < hic) {
        const int uc0 = (int)(loc / pa.Cp), uc1 = (int)((hic - 1) / pa.Cp);
        for (int u = uc0 + warp; u <= uc1; u += P::NW) {
            const int wf = warp_of((long long)u * pa.Cp, pa.V, pa.N);
            const int wl = warp_of((long long)(u + 1) * pa.Cp - 1, pa.V, pa.N);
            const int cf = wf / P::NW, cl = wl / P::NW;
            const int k0 = max(wf, wc0) - wf, k1 = min(wl, wc1) - wf;
            const int b = (int)fdiv((uint32_t)u, pa.fd_H), hk = u - b * g.H;
            const int head = (int)blockIdx.x == cf ? pa.U * pa.maxp + u : -1;    // the tail slot, merged first
            if (cf == cl) {
                merge<GM>(a, head, u * pa.maxp + k0, k1 - k0 + 1, -1, b, hk, lane);
            } else {
                const int cs0 = pa.U * (pa.maxp + 1) + u * pa.maxc;                 // CTA partial slots of unit u
                merge<GM>(a, head, u * pa.maxp + k0, k1 - k0 + 1, cs0 + (int)blockIdx.x - cf, b, hk, lane);
                if (arrive(a.counters + 2 + u, cl - cf + 1, lane))
                    merge<GM>(a, -1, cs0, cl - cf + 1, -1, b, hk, lane);
            }
        }
    }
#if KVT_TRACE
    if (a.trace && lane == 0 && w < 8192) {
        unsigned long long t2, smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
        unsigned sm32;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm32));
        smid = sm32;
        unsigned long long* tr = a.trace + 8 * (size_t)w;
        tr[0] = smid | ((unsigned long long)warp << 16) | ((unsigned long long)blockIdx.x << 32);
        tr[1] = tr_t0; tr[2] = tr_t1; tr[3] = t2; tr[4] = tr_tail; tr[5] = tr_tiles; tr[6] = (unsigned long long)(u1 - u0 + 1);
    }
#endif
}

}  // namespace pk
}  // namespace kvt

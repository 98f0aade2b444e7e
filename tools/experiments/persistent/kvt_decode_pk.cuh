// kvt_decode_pk.cuh — K2 persistent decode attention ("persistent kernel").
//
// Same arithmetic per 32-token tile as kvt_decode_mma.cuh (tile records, fp16-subnormal codes on the tensor
// cores, lazy online softmax, fp32 zero-point sums); a different work schedule:
//
//   * one CTA per SM with NW warps (16 for g <= 4, 12 for g <= 8, fewer when the ring of a wide instance does not
//     fit), each warp an independent worker with its own TMA ring, weight tile, q copy and softmax state;
//   * the work of all (b, kv head) units is laid out unit after unit in a planned cost space (unit u = its tail,
//     costed TC tiles, then T_plan main tiles; the plan length bounds every real length) and CTA c takes the
//     contiguous share [c V / n, (c + 1) V / n): every SM gets the same work whatever B * H_kv is (512 units on 148
//     SMs no longer means 4 units on some SMs and 3 on others);
//   * inside a CTA the warps claim work from a shared-memory queue — first the tails of the CTA's units (bf16 /
//     incomplete tokens past the last whole tile, CUDA cores), then the main tiles in chunks of CH tiles in order —
//     so the per-warp speed differences of a static split (+-10% measured, tools/trace_pk.py) even out.  A warp keeps
//     its softmax state across consecutive chunks of one unit and folds it into the unit's shared-memory accumulator
//     (a lock per unit) when it moves on;
//   * after a CTA barrier each unit's accumulator becomes the output row (unit inside the CTA) or a CTA partial
//     whose last arriver (per-unit counter) merges the CTA partials in CTA order and writes the row.
//
// Which warp folds which chunks depends on timing, so results vary run to run at the rounding level of the fp16 PV
// weights and fp32 sums (A23); the value of every term is the same.
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
// mbarriers | q fp32 [GM][D] | next q bf16 [GM][D] (cp.async prefetch)]; then, per CTA, MAXU unit accumulators
// ([GM][D] o, [GM] (m, l)), their locks and the queue counter.
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
    static constexpr int QMAX_OFF = BAR_OFF + 8 * NS;                  // [GM] per-head max |q| of the q in Q
    static constexpr int Q_OFF = (QMAX_OFF + 4 * GM + 15) / 16 * 16;
    static constexpr int QB_OFF = Q_OFF + GM * D * 4;
    static constexpr int WARP_BYTES = (QB_OFF + GM * D * 2 + 127) / 128 * 128;
    static constexpr int ACC_FLOATS = GM * (D + 2);
    static constexpr int ACC_BYTES = ACC_FLOATS * 4;
    static constexpr int MAXW = GM == 4 ? 16 : 12;          // registers: 16 warps x 128, 12 x 168
    static constexpr int CAP = 227 * 1024;
    static constexpr int RESERVE = 8 * (ACC_BYTES + 24) + 96;      // at least 8 unit accumulators
    static constexpr int NW = (CAP - RESERVE) / WARP_BYTES < MAXW ? (CAP - RESERVE) / WARP_BYTES : MAXW;
    static constexpr int ACC_OFF = NW * WARP_BYTES;
    static constexpr int MAXU = (CAP - ACC_OFF - 96) / (ACC_BYTES + 4 + 16 + 4);
    static constexpr int LOCK_OFF = ACC_OFF + MAXU * ACC_BYTES;
    static constexpr int TAB_OFF = (LOCK_OFF + MAXU * 4 + 15) / 16 * 16;    // int4 per unit: (tl, th, P, DC)
    static constexpr int TABS_OFF = TAB_OFF + MAXU * 16;                     // int per unit: S
    static constexpr int QCTR_OFF = TABS_OFF + MAXU * 4;                     // [tail claims, dynamic chunk claims]
    static constexpr size_t SMEM = (size_t)QCTR_OFF + 16;
    static_assert(32 * 8 * 4 <= W_BYTES, "tail p scratch must fit the weight tile");
    static_assert(MAXU >= 8, "room for the unit accumulators");
};

// The CTA whose share holds planned position x (shares [c V / n, (c + 1) V / n))
__device__ __forceinline__ int cta_of(long long x, long long V, int n) { return (int)(((x + 1) * n - 1) / V); }

// Unit u's actual geometry and its part of the CTA share [lo, hi) of the plan (unit u = positions [u Cp, (u + 1) Cp):
// its tail, costed TC, then T_plan tiles).
struct UnitG {
    int b, hk, S, n_main, tiles;
    int tl, th;          // main tiles of the unit inside the share, clipped to the actual tiles
};
__device__ __forceinline__ void unit_geo(const DecodeArgs& a, int u, long long lo, long long hi, UnitG& ug) {
    const dec::PkArgs& p = a.pk;
    const int b = (int)fdiv((uint32_t)u, p.fd_H);
    const int S = a.seq_len[b];
    const int R = a.g.R;
    const int nqV = S > R ? S - R : 0;
    const int nqK = a.g.mode == KVT_MODE_KIVI ? p.F * (int)fdiv((uint32_t)S, p.fd_F) : nqV;
    const int n_main = (nqK < nqV ? nqK : nqV) & ~31;
    const long long base = (long long)u * p.Cp;
    ug.b = b; ug.hk = u - b * a.g.H; ug.S = S; ug.n_main = n_main; ug.tiles = n_main >> 5;
    ug.tl = (int)min((long long)ug.tiles, max(0ll, lo - base - p.TC));
    ug.th = (int)min((long long)ug.tiles, max(0ll, hi - base - p.TC));
}

// The CTA's work queue: [tails of the units whose tail starts in the share][chunks of CH main tiles, unit by unit].
// Claims only increase, so each warp walks the chunk part with its own cursor (unit, index of its first chunk).
struct Queue {
    long long lo, hi;
    int uc0, uc1;        // units touching the share
    int ut0, n_tail;     // units whose tail starts in the share: [ut0, ut0 + n_tail)
    int TT, A;           // main tiles of the share (unit by unit: the tile list); the static part is [0, A)
    int NDC, xA;         // dynamic chunks of [A, TT); the unit holding list position A
};
struct QItem {
    int kind;            // 0 none left, 1 tail, 2 chunk
    int u, t_lo, t_hi;
};
__device__ __forceinline__ int unit_b(const DecodeArgs& a, int u) { return (int)fdiv((uint32_t)u, a.pk.fd_H); }

__device__ __forceinline__ int claim_local(int* ctr, int lane) {
    int v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1);
    return __shfl_sync(kFull, v, 0);
}
// Tails of the share whose tail has tokens (S > n_main, or no whole tile): claim index -> unit, -1 when none left.
__device__ __forceinline__ int next_tail(const DecodeArgs& a, const Queue& qd, const int* tabS, int* qctr, int lane) {
    for (;;) {
        const int j = claim_local(qctr, lane);
        if (j >= qd.n_tail) return -1;
        const int u = qd.ut0 + j;
        const int S = tabS[u - qd.uc0], R = a.g.R;
        const int nqV = S > R ? S - R : 0;
        const int nqK = a.g.mode == KVT_MODE_KIVI ? a.pk.F * (int)fdiv((uint32_t)S, a.pk.fd_F) : nqV;
        const int n_main = (nqK < nqV ? nqK : nqV) & ~31;
        if (S > n_main || n_main == 0) return u;
    }
}

// Main-tile items: first this warp's static piece(s) of the tile list [k A / NW, (k + 1) A / NW), then dynamic
// chunks of [A, TT) (CH tiles, never across a unit) claimed from the shared counter.  tab[x] = (tl, th, P, DC): unit
// uc0 + x has tiles [tl, th) at list positions [P, P + th - tl) and its dynamic chunks are numbered from DC.
struct Gen {
    int p, pe;           // static: next list position, end of this warp's static share
    int x, xd;           // unit cursors (static, dynamic)
};
__device__ __forceinline__ void next_tiles(const DecodeArgs& a, const Queue& qd, const int4* tab, Gen& gn,
                                           int* qctr2, int lane, QItem& it) {
    const int NU = qd.uc1 - qd.uc0 + 1;
    if (gn.p < gn.pe) {
        while (gn.x + 1 < NU && tab[gn.x + 1].z <= gn.p) ++gn.x;
        const int4 e = tab[gn.x];
        const int end = min(gn.pe, e.z + (e.y - e.x));
        it.kind = 2;
        it.u = qd.uc0 + gn.x;
        it.t_lo = e.x + (gn.p - e.z);
        it.t_hi = e.x + (end - e.z);
        gn.p = end;
        return;
    }
    const int c = claim_local(qctr2, lane);
    if (c >= qd.NDC) { it.kind = 0; return; }
    while (gn.xd + 1 < NU && tab[gn.xd + 1].w <= c) ++gn.xd;
    const int4 e = tab[gn.xd];
    const int pend = e.z + (e.y - e.x);                  // list end of the unit
    const int p0 = max(qd.A, e.z) + (c - e.w) * a.pk.ch;
    it.kind = 2;
    it.u = qd.uc0 + gn.xd;
    it.t_lo = e.x + (p0 - e.z);
    it.t_hi = e.x + (min(p0 + a.pk.ch, pend) - e.z);
}

// Fold a partial (m, l, o) into a unit accumulator of shared memory ([GM][D] o, [GM] (m, l)) under the unit's lock.
// Lanes pass the o values they own through `put` (called with the accumulator); (m, l) per head come from mh / lh
// (head h valid in lanes that own it, l = 0: nothing to fold).
__device__ __forceinline__ void acc_lock(int* lock, int lane) {
    if (lane == 0)
        while (atomicCAS(lock, 0, 1) != 0) { }
    __syncwarp();
    __threadfence_block();
}
__device__ __forceinline__ void acc_unlock(int* lock, int lane) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) atomicExch(lock, 0);
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

    uint8_t* wbase = smem + (size_t)warp * P::WARP_BYTES;
    uint32_t* w_s = reinterpret_cast<uint32_t*>(wbase + P::W_OFF);
    uint32_t* sh_s = reinterpret_cast<uint32_t*>(wbase + P::SH_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + P::BAR_OFF);
    float* qmax_s = reinterpret_cast<float*>(wbase + P::QMAX_OFF);
    float* q_s = reinterpret_cast<float*>(wbase + P::Q_OFF);
    uint16_t* qb = reinterpret_cast<uint16_t*>(wbase + P::QB_OFF);
    float* accs = reinterpret_cast<float*>(smem + P::ACC_OFF);
    int* locks = reinterpret_cast<int*>(smem + P::LOCK_OFF);
    int* qctr = reinterpret_cast<int*>(smem + P::QCTR_OFF);

#if KVT_TRACE
    unsigned long long tr[5] = {0, 0, 0, 0, 0};
    int tr_ntail = 0, tr_nst = 0, tr_ndyn = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[0]));
#define PK_STAMP(k) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[k]))
#else
#define PK_STAMP(k) do { } while (0)
#endif
    // the CTA's share and queue layout, in shared memory (read when needed: keeps registers for the tile loop)
    __shared__ Queue qd;
    if (tid == 0) {
        Queue q;
        q.lo = (long long)blockIdx.x * pa.V / gridDim.x;
        q.hi = (long long)(blockIdx.x + 1) * pa.V / gridDim.x;
        q.uc0 = (int)(q.lo / pa.Cp);
        q.uc1 = (int)((q.hi - 1) / pa.Cp);
        q.ut0 = (int)((q.lo + pa.Cp - 1) / pa.Cp);
        q.n_tail = q.uc1 - q.ut0 + 1 > 0 ? q.uc1 - q.ut0 + 1 : 0;
        qd = q;
    }
    __syncthreads();
    const int NU = qd.uc1 - qd.uc0 + 1;                  // <= MAXU (host plan)

    // ---- CTA setup: unit accumulators (o = 0, m = -inf, l = 0), locks, queue counter; per-warp barriers ----
    for (int i = tid; i < NU * P::ACC_FLOATS; i += blockDim.x) {
        const int x = i / P::ACC_FLOATS, r = i - x * P::ACC_FLOATS;
        accs[i] = (r >= GM * D && ((r - GM * D) & 1) == 0) ? -INFINITY : 0.0f;
    }
    for (int i = tid; i < NU; i += blockDim.x) locks[i] = 0;
    if (tid == 0) *qctr = 0;
    int4* tab = reinterpret_cast<int4*>(smem + P::TAB_OFF);
    int* tabS = reinterpret_cast<int*>(smem + P::TABS_OFF);
    for (int x = tid; x < NU; x += blockDim.x) {
        UnitG ug;
        unit_geo(a, qd.uc0 + x, qd.lo, qd.hi, ug);
        tab[x] = make_int4(ug.tl, ug.th > ug.tl ? ug.th : ug.tl, 0, 0);
        tabS[x] = ug.S;
    }
    __syncthreads();
    if (tid == 0) {                                      // list positions, the static / dynamic split, chunk numbers
        int P0 = 0;
        for (int x = 0; x < NU; ++x) { tab[x].z = P0; P0 += tab[x].y - tab[x].x; }
        const int A = (int)((long long)P0 * pa.static_pct / 100);
        int dc = 0, xA = NU - 1;
        for (int x = 0; x < NU; ++x) {
            const int pend = tab[x].z + (tab[x].y - tab[x].x);
            if (A < pend && xA == NU - 1 && A >= tab[x].z) xA = x;
            const int d = pend - max(A, tab[x].z);
            tab[x].w = dc;
            dc += d > 0 ? (d + pa.ch - 1) / pa.ch : 0;
        }
        qd.TT = P0; qd.A = A; qd.NDC = dc; qd.xA = xA;
        qctr[1] = 0;
    }
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < P::NS; ++st) mbar_init(bars + st);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int i = lane; i < P::W_BYTES / 4; i += 32) w_s[i] = 0u;
    __syncthreads();

    // Programmatic dependent launch: only kvt_append_decode_attention (a.early) lets the first q copy (it does not
    // touch the cache) overlap the preceding append; otherwise wait at entry.
    if (!a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    // phase 1 item: a tail claimed from the shared counter (or none left)
    QItem it;
    it.u = next_tail(a, qd, tabS, qctr, lane);
    it.kind = it.u >= 0 ? 1 : 0;
    // phases 2-3 generator: this warp's static share of the tile list, then dynamic chunks
    Gen gn;
    gn.p = (int)((long long)warp * qd.A / P::NW);
    gn.pe = (int)((long long)(warp + 1) * qd.A / P::NW);
    gn.x = 0;
    gn.xd = qd.xA;
    if (!it.kind) next_tiles(a, qd, tab, gn, qctr + 1, lane, it);
    if (it.kind) {
        const int b = unit_b(a, it.u);
        q_prefetch(a, qb, b, it.u - b * a.g.H, lane);
    }
    if (a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");

    // softmax heads of this thread (the QK D columns it holds after the hi/lo fold)
    const int hA = (GM == 8) ? 2 * tig : 2 * (tig & 1);
    const int gsh = (GM == 4) ? 2 * (tig >> 1) : 0;
    constexpr int NGL = (GM == 4) ? 2 : 4;

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
    if (it.kind == 2) {
        const int b = unit_b(a, it.u);
        issue_tile(b, it.u - b * g.H, it.t_lo, g_it);
    }

    // register softmax state of the unit st_u (kept across consecutive chunks of one unit)
    int st_u = -1, q_unit = -1;
    uint32_t q_h[16];
    float qa_inv[2];
    float qg[KPT ? 4 : 1][2];
    float m_run[2], l_part[2];
    float2 zacc2[4][2];
    float o[8][4];
    int kp = 126;
    bool fresh = true;

    // fold the register state into the accumulator of unit st_u
    auto flush_state = [&]() {
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
        const int x = st_u - qd.uc0;
        float* A = accs + x * P::ACC_FLOATS;
        acc_lock(locks + x, lane);
        // owner lanes hold heads 2 tig + j, channels c = 32 gamma + 4 gid + 2 mu (+1)
        const bool owner = (GM == 8) || (tig < 2);
        float so[2], sn[2], Mn[2], Lo[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int h = owner ? 2 * tig + j : 0;
            const float mo = A[GM * D + 2 * h];
            Lo[j] = A[GM * D + 2 * h + 1];
            Mn[j] = fmaxf(mo, m_run[j]);
            so[j] = Lo[j] > 0.0f ? fexp2(mo - Mn[j]) : 0.0f;
            sn[j] = Lj[j] > 0.0f ? fexp2(m_run[j] - Mn[j]) : 0.0f;
        }
        __syncwarp();                                    // (m, l) read by every owner lane before they change
        if (owner) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int h = 2 * tig + j;
#pragma unroll
                for (int gam = 0; gam < 4; ++gam)
#pragma unroll
                    for (int mu = 0; mu < 2; ++mu) {
                        const int c = 32 * gam + 4 * gid + 2 * mu;
                        const float v0 = o[2 * gam + mu][j] * pow2(24 - VP<VB>(2 * mu) - kp) + zacc[gam][j];
                        const float v1 = o[2 * gam + mu][2 + j] * pow2(24 - VP<VB>(2 * mu + 1) - kp) + zacc[gam][j];
                        float2* ap = reinterpret_cast<float2*>(A + h * D + c);
                        const float2 av = *ap;
                        *ap = make_float2(fmaf(av.x, so[j], v0 * sn[j]), fmaf(av.y, so[j], v1 * sn[j]));
                    }
                if (gid == 0)
                    *reinterpret_cast<float2*>(A + GM * D + 2 * h) =
                        make_float2((Lo[j] > 0.0f || Lj[j] > 0.0f) ? Mn[j] : -INFINITY, Lo[j] * so[j] + Lj[j] * sn[j]);
            }
        }
        acc_unlock(locks + x, lane);
        st_u = -1;
    };

    // q rows of unit iu: bf16 prefetch -> fp32 q_s (zero rows for padded heads), per-head max
    auto q_switch = [&](int iu) {
        if (q_unit == iu) return;
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
        q_unit = iu;
    };

    // ---- phase 1: tails (the queue hands them out first; no register softmax state is live) ----
    while (it.kind == 1) {
        const int iu = it.u;
        q_switch(iu);
        QItem nx;
        {

            // ================= a unit's tail: tokens [n_main, S) on the CUDA cores =================
            // claim the next item first so its first tile and q rows stream in while the tail runs
            nx.u = next_tail(a, qd, tabS, qctr, lane);
            nx.kind = nx.u >= 0 ? 1 : 0;
            if (!nx.kind) next_tiles(a, qd, tab, gn, qctr + 1, lane, nx);
            if (nx.kind) {
                const int b = unit_b(a, nx.u);
                if (nx.u != iu) q_prefetch(a, qb, b, nx.u - b * g.H, lane);
                if (nx.kind == 2) issue_tile(b, nx.u - b * g.H, nx.t_lo, g_it);
            }
            UnitG ug;
            unit_geo(a, iu, qd.lo, qd.hi, ug);
            Slice tl;
            tl.kc = PAGED ? a.c.k_codes + (size_t)ug.hk * g.rec : a.c.k_codes + ((size_t)ug.b * g.H + ug.hk) * g.kc;
            tl.km = nullptr; tl.vc = nullptr; tl.vm = nullptr;
            tl.kr = a.c.k_resid + ((size_t)ug.b * g.H + ug.hk) * (g.kr / 2);
            tl.vr = g.vr ? a.c.v_resid + ((size_t)ug.b * g.H + ug.hk) * (g.vr / 2) : nullptr;
            if (PAGED) {
                tl.bt = a.c.bt + (size_t)ug.b * a.c.max_pages;
                tl.pstride = (size_t)g.H * g.rec;
            }
            const int nqK = nq_key(g.mode, g.kb, g.G, g.R, ug.S);
            const int nqV = nq_per_token(g.vb, g.R, ug.S);
            float* pbuf = reinterpret_cast<float*>(w_s);               // [32 tokens][GM]
            float mt[GM], lt[GM], ot[GM][4];
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                mt[h] = -INFINITY; lt[h] = 0.0f;
                ot[h][0] = ot[h][1] = ot[h][2] = ot[h][3] = 0.0f;
            }
            // token-major: lane = channels 4 lane .. + 3; TB tokens per batch (16 (token, head) logits), the next batch's
            // K and V loads issued before this batch is reduced (otherwise the tail is a chain of global round trips)
            constexpr int TB = 16 / GM;
            float q4[GM][4];
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                const float4 v = *reinterpret_cast<const float4*>(q_s + h * D + 4 * lane);
                q4[h][0] = v.x; q4[h][1] = v.y; q4[h][2] = v.z; q4[h][3] = v.w;
            }
            auto load_batch = [&](int t0, float (&kk)[TB][4], float (&vv)[TB][4]) {
#pragma unroll
                for (int i = 0; i < TB; ++i) {
                    const int t = t0 + i;
                    if (t < ug.S) {
                        dec::tail_k<KB, !KPT, true>(tl, g, t, nqK, lane, kk[i]);
                        dec::tail_v<VB, true>(tl, g, t, nqV, lane, vv[i]);
                    } else {
                        kk[i][0] = kk[i][1] = kk[i][2] = kk[i][3] = 0.0f;
                        vv[i][0] = vv[i][1] = vv[i][2] = vv[i][3] = 0.0f;
                    }
                }
            };
            float kx[TB][4], vx[TB][4];
            load_batch(ug.n_main, kx, vx);
            for (int t0 = ug.n_main; t0 < ug.S; t0 += TB) {
                float kn[TB][4], vn[TB][4];
                load_batch(t0 + TB, kn, vn);                       // the next batch is in flight during this one
                // partial logits of (token i, head h) over this lane's 4 channels: v[i GM + h]
                float v[16];
#pragma unroll
                for (int i = 0; i < TB; ++i)
#pragma unroll
                    for (int h = 0; h < GM; ++h)
                        v[i * GM + h] = fmaf(q4[h][0], kx[i][0], fmaf(q4[h][1], kx[i][1], fmaf(q4[h][2], kx[i][2], q4[h][3] * kx[i][3])));
                // transpose-reduce over lane bits 3..0 (lane l ends with value l & 15), then over bit 4
#pragma unroll
                for (int off = 8; off >= 1; off >>= 1) {
                    const bool up = lane & off;
#pragma unroll
                    for (int i = 0; i < off; ++i) {
                        const float send = up ? v[i] : v[i + off];
                        const float keep = up ? v[i + off] : v[i];
                        v[i] = keep + __shfl_xor_sync(kFull, send, off);
                    }
                }
                const int idx = lane & 15, ti = idx / GM, hh = idx % GM;
                const bool ok = t0 + ti < ug.S;
                const float tot = v[0] + __shfl_xor_sync(kFull, v[0], 16);     // every lane takes part in the shuffle
                const float sl = ok ? tot * a.scale_log2 : -INFINITY;
                // batch max per head (lanes of one head differ in the low-4 lane bits >= log2 GM); lane h holds head h
                float bm = sl;
#pragma unroll
                for (int off = GM; off < 16; off <<= 1) bm = fmaxf(bm, __shfl_xor_sync(kFull, bm, off));
                float al[GM], mh = -INFINITY;
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    const float mn = fmaxf(mt[h], __shfl_sync(kFull, bm, h));   // finite: token t0 is valid
                    al[h] = fexp2(mt[h] - mn);
                    mt[h] = mn;
                    mh = hh == h ? mn : mh;
                }
                if (lane < 16) pbuf[idx] = ok ? fexp2(sl - mh) : 0.0f;
                __syncwarp();
                float pp[16];
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                    const float4 p4 = *reinterpret_cast<const float4*>(pbuf + 4 * k4);
                    pp[4 * k4] = p4.x; pp[4 * k4 + 1] = p4.y; pp[4 * k4 + 2] = p4.z; pp[4 * k4 + 3] = p4.w;
                }
                __syncwarp();                                      // read before the next batch rewrites pbuf
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    float ls = 0.0f;
#pragma unroll
                    for (int i = 0; i < TB; ++i) ls += pp[i * GM + h];
                    lt[h] = lt[h] * al[h] + ls;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float o_ = ot[h][e] * al[h];
#pragma unroll
                        for (int i = 0; i < TB; ++i) o_ = fmaf(pp[i * GM + h], vx[i][e], o_);
                        ot[h][e] = o_;
                    }
                }
#pragma unroll
                for (int i = 0; i < TB; ++i)
#pragma unroll
                    for (int e = 0; e < 4; ++e) { kx[i][e] = kn[i][e]; vx[i][e] = vn[i][e]; }
            }
            for (int i = lane; i < P::W_BYTES / 4; i += 32) w_s[i] = 0u;   // the zero weight tile for the next tiles
            // ---- fold into the unit accumulator: lane = channels 4 lane .. + 3 of every head ----
            {
                const int x = iu - qd.uc0;
                float* A = accs + x * P::ACC_FLOATS;
                acc_lock(locks + x, lane);
                float so[GM], sn[GM], Mn[GM], Lo[GM];
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    const float mo = A[GM * D + 2 * h];
                    Lo[h] = A[GM * D + 2 * h + 1];
                    Mn[h] = fmaxf(mo, mt[h]);
                    so[h] = Lo[h] > 0.0f ? fexp2(mo - Mn[h]) : 0.0f;
                    sn[h] = lt[h] > 0.0f ? fexp2(mt[h] - Mn[h]) : 0.0f;
                }
                __syncwarp();
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    if (h >= gq) continue;
                    float4* ap = reinterpret_cast<float4*>(A + h * D + 4 * lane);
                    const float4 av = *ap;
                    *ap = make_float4(fmaf(av.x, so[h], ot[h][0] * sn[h]), fmaf(av.y, so[h], ot[h][1] * sn[h]),
                                      fmaf(av.z, so[h], ot[h][2] * sn[h]), fmaf(av.w, so[h], ot[h][3] * sn[h]));
                    if (lane == 0)
                        *reinterpret_cast<float2*>(A + GM * D + 2 * h) =
                            make_float2((Lo[h] > 0.0f || lt[h] > 0.0f) ? Mn[h] : -INFINITY, Lo[h] * so[h] + lt[h] * sn[h]);
                }
                acc_unlock(locks + x, lane);
            }
        }
        it = nx;
    }

    PK_STAMP(1);
    // ---- phase 2: chunks of main tiles, unit by unit (the queue has no tails left) ----
    while (it.kind == 2) {
#if KVT_TRACE
        if (gn.p <= gn.pe && tr[2] == 0 && gn.p == gn.pe && false) { }
        if (it.t_hi > it.t_lo) { if (tr[2] == 0) tr_nst += it.t_hi - it.t_lo; else tr_ndyn += it.t_hi - it.t_lo; }
#endif
        const int iu = it.u;
        if (st_u >= 0 && iu != st_u) flush_state();
        q_switch(iu);
        QItem nx;
        // ================= chunk: main tiles [t_lo, t_hi) of unit iu on the tensor cores =================
        if (st_u < 0) {
            // a new register state for unit iu
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
            m_run[0] = m_run[1] = -INFINITY;
            l_part[0] = l_part[1] = 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) zacc2[i][0] = zacc2[i][1] = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
            kp = 126;
            fresh = true;
            st_u = iu;
        }
        const int n_t = it.t_hi - it.t_lo;
        // ring source of tile t_lo + i: dense = base + i * STAGE; paged = pool + (bt[t_lo + i] * H + hk) * STAGE
        const int ib = unit_b(a, iu), ihk = iu - ib * g.H;
        const uint8_t* src_base = bcast_ptr(PAGED ? a.c.k_codes + (size_t)ihk * P::STAGE
                                                  : a.c.k_codes + ((size_t)ib * g.H + ihk) * g.kc + (size_t)it.t_lo * P::STAGE);
        const int32_t* bt_row = PAGED ? a.c.bt + (size_t)ib * a.c.max_pages + it.t_lo : nullptr;
        nx.kind = 0;
        for (int i = 0; i < n_t; ++i) {
            if (i + 1 < n_t) {
                if (lane == 0) {
                    const int st = (int)((g_it + 1) % P::NS);
                    mbar_expect_tx(bars + st, P::STAGE);
                    const uint8_t* src = PAGED ? src_base + (size_t)bt_row[i + 1] * g.H * P::STAGE
                                               : src_base + (size_t)(i + 1) * P::STAGE;
                    bulk_g2s(wbase + st * P::STAGE, src, P::STAGE, bars + st);
                }
            } else {                                    // last tile: the next item, start its q rows / first tile
#if KVT_TRACE
                if (tr[2] == 0 && gn.p >= gn.pe) PK_STAMP(2);
#endif
                next_tiles(a, qd, tab, gn, qctr + 1, lane, nx);
                if (nx.kind) {
                    const int b = unit_b(a, nx.u);
                    if (nx.u != iu) q_prefetch(a, qb, b, nx.u - b * g.H, lane);
                    if (nx.kind == 2) issue_tile(b, nx.u - b * g.H, nx.t_lo, g_it + 1);
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
                    if (!fresh) { kfac = pow2(kt - kp < -126 ? -126 : kt - kp); resc = true; }
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
            fresh = false;
        }
        it = nx;
    }
    if (st_u >= 0) flush_state();
    PK_STAMP(3);
    if (lane == 0) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars)));
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bars + 1)));
    }

    // ================= outputs: units inside the share directly, the others through CTA partials =================
    __syncthreads();                                     // every accumulator is final
    const size_t SB = pa.slot_floats;
    for (int x = warp; x < NU; x += P::NW) {
        const int u = qd.uc0 + x;
        const float* A = accs + x * P::ACC_FLOATS;
        const int b = (int)fdiv((uint32_t)u, pa.fd_H), hk = u - b * g.H;
        const long long base = (long long)u * pa.Cp;
        if (base >= qd.lo && base + pa.Cp <= qd.hi) {
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                if (h >= gq) continue;
                const size_t row = (size_t)b * a.H_q + (size_t)hk * gq + h;
                const float M = A[GM * D + 2 * h], L = A[GM * D + 2 * h + 1];
                const float4 ov = *reinterpret_cast<const float4*>(A + h * D + 4 * lane);
                write_row(a, a.out, a.out_mode, row, 4 * lane + 0, M, L, ov.x);
                write_row(a, a.out, a.out_mode, row, 4 * lane + 1, M, L, ov.y);
                write_row(a, a.out, a.out_mode, row, 4 * lane + 2, M, L, ov.z);
                write_row(a, a.out, a.out_mode, row, 4 * lane + 3, M, L, ov.w);
            }
        } else {
            const int cf = cta_of(base, pa.V, gridDim.x), cl = cta_of(base + pa.Cp - 1, pa.V, gridDim.x);
            float* sp = a.parts + (size_t)(u * pa.maxc + (int)blockIdx.x - cf) * SB;
#pragma unroll
            for (int h = 0; h < GM; ++h) {
                if (h >= gq) continue;
                *reinterpret_cast<float4*>(sp + h * D + 4 * lane) = *reinterpret_cast<const float4*>(A + h * D + 4 * lane);
                if (lane == 0) *reinterpret_cast<float2*>(sp + gq * D + 2 * h) = *reinterpret_cast<const float2*>(A + GM * D + 2 * h);
            }
            if (arrive(a.counters + 2 + u, cl - cf + 1, lane)) merge<GM>(a, -1, u * pa.maxc, cl - cf + 1, -1, b, hk, lane);
        }
    }
#if KVT_TRACE
    PK_STAMP(4);
    const int w = blockIdx.x * P::NW + warp;
    if (a.trace && lane == 0 && w < 8192) {
        unsigned sm32;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm32));
        unsigned long long* t = a.trace + 8 * (size_t)w;
        t[0] = sm32 | ((unsigned long long)warp << 16) | ((unsigned long long)blockIdx.x << 32);
        t[1] = tr[0]; t[2] = tr[1]; t[3] = tr[2] ? tr[2] : tr[1]; t[4] = tr[3]; t[5] = tr[4];
        t[6] = (unsigned long long)tr_nst | ((unsigned long long)tr_ndyn << 32);
    }
#endif
}

}  // namespace pk
}  // namespace kvt

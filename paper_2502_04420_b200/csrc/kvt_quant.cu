// kvt_quant.cu — K1: quantise-on-append (Eq. 2) into the packed cache.
//
// One warp quantises one token row (per-token groups of G channels: V in both modes, K in
// per-token-asym) or one KIVI key block (G tokens x 128 channels, groups = one channel over the
// block, P:707 / A8).  Lane l always owns channels 4l..4l+3, so a bf16 row is one 8-byte load per
// lane and a packed row is one 1/2/4-byte store per lane (coalesced).
//
// Exactness (A1-A4): min/max are exact; s32 = (max - min) / (2^b - 1) with IEEE division; the
// stored scale is bf16 rounded toward +inf (cvt.rp); inv = 1/scale (IEEE); t = (x - z) * inv with
// __fsub_rn/__fmul_rn (no FMA contraction); code = clamp(rint(t), 0, 2^b - 1).  This is the
// reading the oracle implements independently, so codes and meta match it bit for bit.
//
// Ordering: tokens whose bf16 source is the residual (ring or KIVI key residual) are quantised by
// the chunk-0 CTA of each (b, h), which then writes the new residual tokens after a
// __syncthreads; all other CTAs only read the new input, so no inter-CTA ordering is needed.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kvt_internal.h"
#include "kvt_quant.cuh"

namespace kvt {
namespace {

using namespace quant;
constexpr int kWarps = 4;

struct AppendArgs {
    Geometry g;
    CachePtrs c;
    const uint16_t* k_new;
    const uint16_t* v_new;
    int64_t s0, s1, s2;
    const int32_t* len_before;
    const int32_t* n_new;
};

// KIVI key block: G tokens x 128 channels, one Eq. 2 group per channel (A8).  src(i) returns the
// bf16 row of the i-th token of the block.
template <typename Src>
__device__ void quant_block_warp(Src src, int G, int bits, uint8_t* codes0, size_t row_bytes, uint32_t* meta_blk,
                                 int lane) {
    float mn[4], mx[4];
    {
        float x[4];
        unpack4(src(0)[lane], x);
#pragma unroll
        for (int j = 0; j < 4; ++j) { mn[j] = x[j]; mx[j] = x[j]; }
    }
    for (int i = 1; i < G; ++i) {
        float x[4];
        unpack4(src(i)[lane], x);
#pragma unroll
        for (int j = 0; j < 4; ++j) { mn[j] = fminf(mn[j], x[j]); mx[j] = fmaxf(mx[j], x[j]); }
    }
    GroupQ q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = group_params(mn[j], mx[j], bits);
    for (int i = 0; i < G; ++i) {
        float x[4];
        unpack4(src(i)[lane], x);
        uint32_t packed = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) packed |= code_of(x[j], q[j]) << (j * bits);
        store_packed(codes0 + (size_t)i * row_bytes, lane, bits, packed);
    }
    uint4 m;
    m.x = q[0].s_bits | (q[0].z_bits << 16);
    m.y = q[1].s_bits | (q[1].z_bits << 16);
    m.z = q[2].s_bits | (q[2].z_bits << 16);
    m.w = q[3].s_bits | (q[3].z_bits << 16);
    reinterpret_cast<uint4*>(meta_blk)[lane] = m;
}

// One per-token tensor (V, or K in per-token mode) with window R.  phase 0: quantise tokens whose
// source is the ring (chunk 0 only); phase 1: quantise tokens from the input (all chunks);
// phase 2: ring writes (chunk 0 only, after phase 0).
// Token t's packed row and meta row; with tile records (g.rec) they live in the record of block t / 32
// (codes = the record base; the row pointer is unused: the codes go to the blocked V block).
// With tile records: rows at blk_off == 0 are token-major code rows (K), otherwise the blocked V block.
// Paged caches (bt != null): record j of the sequence is page bt[j]; codes = the pool base of this KV head
// and pstride = the page size (H records).
struct TokDst {
    uint8_t* codes; uint32_t* meta; size_t row_bytes; int gpr; size_t rec; uint32_t blk_off, meta_off;
    const int32_t* bt; size_t pstride;
    __device__ uint8_t* recp(int j) const { return bt ? codes + (size_t)bt[j] * pstride : codes + (size_t)j * rec; }
    __device__ uint8_t* row(int t) const {
        return rec ? recp(t >> 5) + (size_t)(t & 31) * row_bytes : codes + (size_t)t * row_bytes;
    }
    __device__ uint32_t* meta_row(int t) const {
        return rec ? reinterpret_cast<uint32_t*>(recp(t >> 5) + meta_off + (size_t)(t & 31) * 16)
                   : meta + (size_t)t * gpr;
    }
    __device__ uint8_t* vblk(int t) const { return rec && blk_off ? recp(t >> 5) + blk_off : nullptr; }
};

__device__ void per_token_tensor(int phase, int bits, int G, int R, int L0, int S, const uint16_t* in,
                                 int64_t s2, const TokDst& dst, uint16_t* ring, int wid, int nwarps, int lane) {
    uint8_t* codes = dst.codes;
    const size_t row_bytes = dst.row_bytes;
    if (bits == 16) {
        if (phase != 1) return;
        for (int t = L0 + wid; t < S; t += nwarps) {
            uint2 v = reinterpret_cast<const uint2*>(in + (int64_t)(t - L0) * s2)[lane];
            reinterpret_cast<uint2*>(codes + (size_t)t * row_bytes)[lane] = v;
        }
        return;
    }
    int q0 = L0 > R ? L0 - R : 0;
    int q1 = S > R ? S - R : 0;
    if (phase == 0) {
        int hi = q1 < L0 ? q1 : L0;
        for (int t = q0 + wid; t < hi; t += nwarps) {
            uint2 v = reinterpret_cast<const uint2*>(ring + (size_t)(t % R) * 128)[lane];
            quant_row_warp(v, bits, G, dst.row(t), dst.meta_row(t), lane, dst.vblk(t), t);
        }
    } else if (phase == 1 && G == 32) {
        // 8 rows per iteration (rows t + r * nwarps), loads first, group statistics spread over the lanes
        int lo = q0 > L0 ? q0 : L0;
        for (int t = lo + wid; t < q1; t += 8 * nwarps) {
            const int nrow = min(8, (q1 - t + nwarps - 1) / nwarps);
            uint2 v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r)
                v[r] = r < nrow ? reinterpret_cast<const uint2*>(in + (int64_t)(t + r * nwarps - L0) * s2)[lane]
                                : make_uint2(0u, 0u);
            struct Rows {
                const TokDst& d; int t, step;
                __device__ uint32_t* meta_row(int r) const { return d.meta_row(t + r * step); }
                __device__ void store(int r, int lane, int bits, uint32_t packed) const {
                    const int tt = t + r * step;
                    uint8_t* vb = d.vblk(tt);
                    if (vb) quant::store_packed_vblk(vb, tt, lane, bits, packed);
                    else quant::store_packed(d.row(tt), lane, bits, packed);
                }
            } rows{dst, t, nwarps};
            quant_rows8_warp(v, nrow, bits, rows, lane);
        }
    } else if (phase == 1) {
        // 4 rows per iteration, loads first: memory-level parallelism for the bulk (prefill) case
        int lo = q0 > L0 ? q0 : L0;
        for (int t = lo + wid; t < q1; t += 4 * nwarps) {
            uint2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int tt = t + u * nwarps;
                if (tt < q1) v[u] = reinterpret_cast<const uint2*>(in + (int64_t)(tt - L0) * s2)[lane];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int tt = t + u * nwarps;
                if (tt < q1) quant_row_warp(v[u], bits, G, dst.row(tt), dst.meta_row(tt), lane, dst.vblk(tt), tt);
            }
        }
    } else if (R > 0) {
        int lo = (S - R) > L0 ? (S - R) : L0;
        for (int t = lo + wid; t < S; t += nwarps) {
            uint2 v = reinterpret_cast<const uint2*>(in + (int64_t)(t - L0) * s2)[lane];
            reinterpret_cast<uint2*>(ring + (size_t)(t % R) * 128)[lane] = v;
        }
    }
}

// KIVI key (per-channel).  nb/na: n_qK before/after; residual slot of token t is t - nb before the
// append and t - na after it.
__device__ void per_channel_key(int phase, int bits, int G, int F, int L0, int S, const uint16_t* in, int64_t s2,
                                uint8_t* codes, size_t row_bytes, uint32_t* meta, uint16_t* resid, int wid,
                                int nwarps, int lane, size_t rec = 0, uint32_t rec_km = 0,
                                const int32_t* bt = nullptr, size_t pstride = 0) {
    int nb = F * (L0 / F);
    int na = F * (S / F);
    int nblk = (na - nb) / G;
    if (phase == 0 || phase == 1) {
        for (int j = wid; j < nblk; j += nwarps) {
            int t0 = nb + j * G;
            bool from_resid = t0 < L0;
            if ((phase == 0) != from_resid) continue;
            uint8_t* rp = bt ? codes + (size_t)bt[t0 / G] * pstride : codes + (size_t)(t0 / G) * rec;
            uint8_t* cblk = rec ? rp : codes + (size_t)t0 * row_bytes;
            uint32_t* mblk = rec ? reinterpret_cast<uint32_t*>(rp + rec_km) : meta + (size_t)(t0 / G) * 128;
            if (from_resid) {
                auto src = [&](int i) -> const uint2* {
                    int t = t0 + i;
                    if (t < L0) return reinterpret_cast<const uint2*>(resid + (size_t)(t - nb) * 128);
                    return reinterpret_cast<const uint2*>(in + (int64_t)(t - L0) * s2);
                };
                quant_block_warp(src, G, bits, cblk, row_bytes, mblk, lane);
            } else {                               // the whole block comes from the input: strided rows
                const uint16_t* base = in + (int64_t)(t0 - L0) * s2;
                auto src = [&](int i) -> const uint2* { return reinterpret_cast<const uint2*>(base + (int64_t)i * s2); };
                quant_block_warp(src, G, bits, cblk, row_bytes, mblk, lane);
            }
        }
    } else {
        int lo = na > L0 ? na : L0;
        for (int t = lo + wid; t < S; t += nwarps) {
            uint2 v = reinterpret_cast<const uint2*>(in + (int64_t)(t - L0) * s2)[lane];
            reinterpret_cast<uint2*>(resid + (size_t)(t - na) * 128)[lane] = v;
        }
    }
}

// One instance per key mode.  KIVI (per-channel keys) is bounded to 8 CTAs per SM (64 registers): its prefill is
// bound by global-load latency (ncu: long-scoreboard stalls first, 16 warps per SM at 128 registers), and twice
// the warps hide it — B = 64, 8k: K4V2 1.46 -> 1.24 ms, K2V2 1.43 -> 1.23 ms (KV8 1.65 -> 1.67).  The per-token
// instance keeps 4 CTAs per SM (128 registers; bounded to 8 it ran 15% slower, unbounded (140) 20% slower).
template <bool KPC>
__global__ void __launch_bounds__(kWarps * 32, KPC ? 8 : 4) append_kernel(AppendArgs a) {
    // the decode attention launched next may start its q/length prologue now (it waits for this grid's
    // completion before reading the cache: griddepcontrol.wait in decode_mma_kernel)
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int b = blockIdx.z, h = blockIdx.y, chunk = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = a.n_new[b];
    if (n <= 0) return;
    const int L0 = a.len_before[b];
    const int S = L0 + n;
    const Geometry& g = a.g;
    const size_t bh = (size_t)b * g.H + h;
    const int32_t* bt = a.c.bt ? a.c.bt + (size_t)b * a.c.max_pages : nullptr;    // paged (tile records only)
    const size_t pstride = (size_t)g.H * g.rec;
    uint8_t* kc = bt ? a.c.k_codes + (size_t)h * g.rec : a.c.k_codes + bh * g.kc;
    uint32_t* km = g.km ? a.c.k_meta + bh * (g.km / 4) : nullptr;
    uint16_t* kr = g.kr ? a.c.k_resid + bh * (g.kr / 2) : nullptr;
    uint8_t* vc = a.c.v_codes + bh * g.vc;
    uint32_t* vm = g.vm ? a.c.v_meta + bh * (g.vm / 4) : nullptr;
    uint16_t* vr = g.vr ? a.c.v_resid + bh * (g.vr / 2) : nullptr;
    const uint16_t* kin = a.k_new + (int64_t)b * a.s0 + (int64_t)h * a.s1;
    const uint16_t* vin = a.v_new + (int64_t)b * a.s0 + (int64_t)h * a.s1;
    const TokDst kd = g.rec ? TokDst{kc, nullptr, g.row_k, 128 / g.G, g.rec, 0, g.rec_km, bt, pstride}   // per-token K rows in records
                            : TokDst{kc, km, g.row_k, 128 / g.G, 0, 0, 0, nullptr, 0};
    const TokDst vd = g.rec ? TokDst{kc, nullptr, g.row_v, 128 / g.G, g.rec, g.rec_vc, g.rec_vm, bt, pstride}
                            : TokDst{vc, vm, g.row_v, 128 / g.G, 0, 0, 0, nullptr, 0};

    // phase 0 (chunk 0): residual-sourced groups; phase 1: input-sourced groups (everyone)
    if (chunk == 0) {
        if (KPC)
            per_channel_key(0, g.kb, g.G, g.F, L0, S, kin, a.s2, kc, g.row_k, km, kr, warp, kWarps, lane, g.rec, g.rec_km, bt, pstride);
        else
            per_token_tensor(0, g.kb, g.G, g.R, L0, S, kin, a.s2, kd, kr, warp, kWarps, lane);
        per_token_tensor(0, g.vb, g.G, g.R, L0, S, vin, a.s2, vd, vr, warp, kWarps, lane);
    }
    const int wid = chunk * kWarps + warp, nw = gridDim.x * kWarps;
    if (KPC)
        per_channel_key(1, g.kb, g.G, g.F, L0, S, kin, a.s2, kc, g.row_k, km, kr, wid, nw, lane, g.rec, g.rec_km, bt, pstride);
    else
        per_token_tensor(1, g.kb, g.G, g.R, L0, S, kin, a.s2, kd, kr, wid, nw, lane);
    per_token_tensor(1, g.vb, g.G, g.R, L0, S, vin, a.s2, vd, vr, wid, nw, lane);
    // phase 2 (chunk 0): new residual tokens, after every residual read of phase 0
    if (chunk == 0) {
        __syncthreads();
        if (KPC)
            per_channel_key(2, g.kb, g.G, g.F, L0, S, kin, a.s2, kc, g.row_k, km, kr, warp, kWarps, lane, g.rec, g.rec_km, bt, pstride);
        else
            per_token_tensor(2, g.kb, g.G, g.R, L0, S, kin, a.s2, kd, kr, warp, kWarps, lane);
        per_token_tensor(2, g.vb, g.G, g.R, L0, S, vin, a.s2, vd, vr, warp, kWarps, lane);
    }
}

}  // namespace

int32_t launch_append(const Geometry& g, const CachePtrs& c, const uint16_t* k_new, const uint16_t* v_new,
                      const int64_t strides[3], const int32_t* len_before, const int32_t* n_new, int n_new_max,
                      void* stream) {
    AppendArgs a;
    a.g = g; a.c = c; a.k_new = k_new; a.v_new = v_new;
    a.s0 = strides[0]; a.s1 = strides[1]; a.s2 = strides[2];
    a.len_before = len_before; a.n_new = n_new;
    int chunks = (n_new_max + 127) / 128;
    if (chunks < 1) chunks = 1;
    if (chunks > 4096) chunks = 4096;
    if (g.B > 65535 || g.H > 65535) return fail(KVT_ERR_UNSUPPORTED, "append: batch/heads exceed grid limits");
    dim3 grid(chunks, g.H, g.B);
    if (g.key_per_channel) append_kernel<true><<<grid, kWarps * 32, 0, (cudaStream_t)stream>>>(a);
    else append_kernel<false><<<grid, kWarps * 32, 0, (cudaStream_t)stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "append launch: %s", cudaGetErrorString(e));
    return KVT_OK;
}

}  // namespace kvt

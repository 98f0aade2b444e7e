// kvt_quant.cuh — the Eq. 2 group quantiser shared by K1 (append) and K5 (sensitivity).
// Readings A1-A4: exact min/max, IEEE fp32 s32 = (max-min)/(2^b-1), bf16 scale rounded
// toward +inf, inv = 1/scale, t = (x - z) * inv without FMA contraction, code = clamp(rint(t)).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kvt_internal.h"

namespace kvt {
namespace quant {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float bf2f(uint32_t b16) { return __uint_as_float(b16 << 16); }

__device__ __forceinline__ uint32_t bf16_ru_bits(float f) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_ru(f));
}

// Eq. 2 statistics of one group -> (scale bits, zero bits, inverse scale, degenerate?)
struct GroupQ {
    uint32_t s_bits, z_bits;
    float mn, inv, qmax;
    bool degenerate;
};

__device__ __forceinline__ GroupQ group_params(float mn, float mx, int bits) {
    GroupQ q;
    if (mn == 0.0f) mn = 0.0f;                      // canonical +0 zero-point (A3)
    q.mn = mn;
    q.z_bits = __float_as_uint(mn) >> 16;           // exact: mn is a bf16 value
    q.qmax = (float)((1 << bits) - 1);
    q.degenerate = (mx == mn);
    if (q.degenerate) {                             // A2: s := 1, codes 0
        q.s_bits = 0x3F80u;
        q.inv = 0.0f;
    } else {
        float s32 = __fdiv_rn(__fsub_rn(mx, mn), q.qmax);
        q.s_bits = bf16_ru_bits(s32);
        q.inv = __frcp_rn(bf2f(q.s_bits));               // correctly rounded 1/s (= IEEE 1.0f / s)
    }
    return q;
}

// clamp(rint(t), 0, qmax): cvt.rni to an unsigned integer rounds to nearest even and saturates negatives to 0
__device__ __forceinline__ uint32_t rint_clamp(float t, uint32_t qmax) {
    const uint32_t c = __float2uint_rn(t);
    return c < qmax ? c : qmax;
}

__device__ __forceinline__ uint32_t code_of(float x, const GroupQ& q) {
    // degenerate groups have inv = 0, so t = 0 and the code is 0 (A2) without a branch
    const float t = __fmul_rn(__fsub_rn(x, q.mn), q.inv);
    return rint_clamp(t, (uint32_t)q.qmax);
}

__device__ __forceinline__ void unpack4(uint2 v, float x[4]) {
    x[0] = bf2f(v.x & 0xffffu); x[1] = bf2f(v.x >> 16);
    x[2] = bf2f(v.y & 0xffffu); x[3] = bf2f(v.y >> 16);
}

__device__ __forceinline__ void store_packed(uint8_t* row, int lane, int bits, uint32_t packed) {
    if (bits == 2) row[lane] = (uint8_t)packed;
    else if (bits == 4) reinterpret_cast<uint16_t*>(row)[lane] = (uint16_t)packed;
    else reinterpret_cast<uint32_t*>(row)[lane] = packed;
}

// Store the lane's 4-channel chunk (gam = lane / 8, i = lane % 8) of token t into the blocked value
// layout; `blk` is the V-code part of token t's tile record.
__device__ __forceinline__ void store_packed_vblk(uint8_t* blk, int t, int lane, int bits, uint32_t packed) {
    const int tau = t & 31, gam = lane >> 3, i = lane & 7;
    if (bits == 2) {
        blk[vblk_off(2, tau, gam, i, 0)] = (uint8_t)packed;
    } else if (bits == 4) {
        *reinterpret_cast<uint16_t*>(blk + vblk_off(4, tau, gam, i, 0)) = (uint16_t)packed;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) blk[vblk_off(8, tau, gam, i, k)] = (uint8_t)(packed >> (8 * k));
    }
}

// Quantise one 128-channel token row held as 4 bf16 per lane; per-token groups of G channels.
// vblk != nullptr: write the codes of token t into that blocked V-code block instead of `row`.
__device__ __forceinline__ void quant_row_warp(uint2 xv, int bits, int G, uint8_t* row, uint32_t* meta_row, int lane,
                                               uint8_t* vblk = nullptr, int t = 0) {
    if (bits == 16) {                                // bf16 pass-through
        reinterpret_cast<uint2*>(row)[lane] = xv;
        return;
    }
    float x[4];
    unpack4(xv, x);
    float mn = fminf(fminf(x[0], x[1]), fminf(x[2], x[3]));
    float mx = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
    for (int off = 1; off < G / 4; off <<= 1) {       // the G/4 lanes of one group
        mn = fminf(mn, __shfl_xor_sync(kFull, mn, off));
        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
    }
    GroupQ q = group_params(mn, mx, bits);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) packed |= code_of(x[i], q) << (i * bits);
    if (vblk) store_packed_vblk(vblk, t, lane, bits, packed);
    else store_packed(row, lane, bits, packed);
    if ((lane & (G / 4 - 1)) == 0) meta_row[lane / (G / 4)] = q.s_bits | (q.z_bits << 16);
}


// Eight token rows at once, G = 32: the group statistics of all 8 rows x 4 groups are spread over the 32
// lanes (lane = group (lane / 8) of row (lane % 8)), so each lane runs the Eq. 2 scale computation (two
// IEEE divisions) once per 8 rows instead of once per row; the codes are then formed with the row's
// (zero-point, 1/scale) shuffled from the lane that owns it.  Same arithmetic as quant_row_warp.
template <typename RowDst>
__device__ __forceinline__ void quant_rows8_warp(const uint2 v[8], int nrow, int bits, const RowDst& dst, int lane) {
    float x[8][4], mn[8], mx[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        unpack4(v[r], x[r]);
        mn[r] = fminf(fminf(x[r][0], x[r][1]), fminf(x[r][2], x[r][3]));
        mx[r] = fmaxf(fmaxf(x[r][0], x[r][1]), fmaxf(x[r][2], x[r][3]));
    }
#pragma unroll
    for (int off = 1; off < 8; off <<= 1)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            mn[r] = fminf(mn[r], __shfl_xor_sync(kFull, mn[r], off));
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(kFull, mx[r], off));
        }
    const int rr = lane & 7;
    float mn_s = mn[0], mx_s = mx[0];
#pragma unroll
    for (int r = 1; r < 8; ++r)
        if (rr == r) { mn_s = mn[r]; mx_s = mx[r]; }
    const GroupQ q = group_params(mn_s, mx_s, bits);   // degenerate groups: inv = 0, so every code is 0
    if (rr < nrow) dst.meta_row(rr)[lane >> 3] = q.s_bits | (q.z_bits << 16);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        if (r >= nrow) break;
        const float inv = __shfl_sync(kFull, q.inv, (lane & 24) | r);
        const float z = __shfl_sync(kFull, q.mn, (lane & 24) | r);
        uint32_t packed = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            packed |= rint_clamp(__fmul_rn(__fsub_rn(x[r][i], z), inv), (uint32_t)q.qmax) << (i * bits);
        dst.store(r, lane, bits, packed);
    }
}

}  // namespace quant
}  // namespace kvt

// kvt_sens.cu — K5: layer sensitivity for every candidate precision pair (a7).
//
// The paper's calibration step (P:146-151 metrics; App. B protocol P:622-623: "simulated offline
// quantization and dequantization", decode-phase queries, no error accumulation): for one layer and
// one prompt, quantise the whole K/V trace statically at (b_k, b_v) (A15), attend the decode queries
// causally with (K, V) and with (K_hat, V_hat), and report
//   e_k = mean |K - K_hat| / |K|,  e_v likewise,  e_a = mean |a - a_hat|,  e_o = mean |o - o_hat| / |o|
// (relative errors over elements with |x| >= 1e-8, A13; e_a over unmasked positions, A16) plus the
// well-conditioned e_o^L1 = sum |o - o_hat| / sum |o|.  All arithmetic after quantisation is fp64, and
// every reduction has a fixed order, so the result is deterministic and matches the fp64 oracle to
// rounding.  The quantiser is K1's (kvt_quant.cuh), so K_hat is bit-identical to the cache contents.
#include <cuda_runtime.h>

#include <vector>

#include "kvt_internal.h"
#include "kvt_quant.cuh"

namespace kvt {
namespace {

using namespace quant;
constexpr int D = 128;
constexpr double kDelta = 1e-8;
constexpr int kRedBlocks = 296;     // fixed grid for the element-wise reductions (2 x 148 SMs)
constexpr int kMaxS = 8192;

__device__ __forceinline__ double dq(uint32_t code, uint32_t s_bits, uint32_t z_bits) {
    return (double)code * (double)bf2f(s_bits) + (double)bf2f(z_bits);   // exact (A3)
}

// Rows: per-token tensor (or the exact tail of a per-channel key).  One warp per token.
__global__ void __launch_bounds__(128) dequant_rows_kernel(const uint16_t* __restrict__ x, double* __restrict__ xh,
                                                           int S, int bits, int G, int nq, int skip_below) {
    const int h = blockIdx.x;
    const int t = blockIdx.y * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= S || t < skip_below) return;
    const uint2 v = reinterpret_cast<const uint2*>(x + ((size_t)h * S + t) * D)[lane];
    float f[4];
    unpack4(v, f);
    double* out = xh + ((size_t)h * S + t) * D + 4 * lane;
    if (bits == 16 || t >= nq) {
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = (double)f[i];
        return;
    }
    float mn = fminf(fminf(f[0], f[1]), fminf(f[2], f[3]));
    float mx = fmaxf(fmaxf(f[0], f[1]), fmaxf(f[2], f[3]));
    for (int off = 1; off < G / 4; off <<= 1) {
        mn = fminf(mn, __shfl_xor_sync(kFull, mn, off));
        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
    }
    GroupQ q = group_params(mn, mx, bits);
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = dq(code_of(f[i], q), q.s_bits, q.z_bits);
}

// KIVI key blocks [0, nq): one warp per block of G tokens, lane = 4 channels (A8).
__global__ void __launch_bounds__(128) dequant_blocks_kernel(const uint16_t* __restrict__ x, double* __restrict__ xh,
                                                             int S, int bits, int G, int nq) {
    const int h = blockIdx.x;
    const int blk = blockIdx.y * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (blk * G >= nq) return;
    const uint2* src = reinterpret_cast<const uint2*>(x + ((size_t)h * S + (size_t)blk * G) * D);
    float mn[4], mx[4];
    {
        float f[4];
        unpack4(src[lane], f);
        for (int j = 0; j < 4; ++j) { mn[j] = f[j]; mx[j] = f[j]; }
    }
    for (int i = 1; i < G; ++i) {
        float f[4];
        unpack4(src[i * (D / 4) + lane], f);
        for (int j = 0; j < 4; ++j) { mn[j] = fminf(mn[j], f[j]); mx[j] = fmaxf(mx[j], f[j]); }
    }
    GroupQ q[4];
    for (int j = 0; j < 4; ++j) q[j] = group_params(mn[j], mx[j], bits);
    for (int i = 0; i < G; ++i) {
        float f[4];
        unpack4(src[i * (D / 4) + lane], f);
        double* out = xh + ((size_t)h * S + (size_t)blk * G + i) * D + 4 * lane;
        for (int j = 0; j < 4; ++j) out[j] = dq(code_of(f[j], q[j]), q[j].s_bits, q[j].z_bits);
    }
}

// per-channel-asym (A28): every channel column of the whole trace is one Eq. 2 group, keys and values alike.
// Block = one KV head: thread (slice, c) scans tokens slice, slice + 8, ... of channel c; the 8 slices'
// min / max meet in shared memory (min / max are exact, so the order does not matter).
__global__ void __launch_bounds__(1024) dequant_cols_kernel(const uint16_t* __restrict__ x, double* __restrict__ xh,
                                                            int S, int bits) {
    __shared__ float smn[8][D], smx[8][D];
    const int h = blockIdx.x, c = threadIdx.x & (D - 1), sl = threadIdx.x >> 7;
    const uint16_t* xc = x + (size_t)h * S * D + c;
    float mn = INFINITY, mx = -INFINITY;
    for (int t = sl; t < S; t += 8) {
        const float f = bf2f(xc[(size_t)t * D]);
        mn = fminf(mn, f);
        mx = fmaxf(mx, f);
    }
    smn[sl][c] = mn;
    smx[sl][c] = mx;
    __syncthreads();
    for (int j = 0; j < 8; ++j) { mn = fminf(mn, smn[j][c]); mx = fmaxf(mx, smx[j][c]); }
    double* oc = xh + (size_t)h * S * D + c;
    if (bits == 16) {
        for (int t = sl; t < S; t += 8) oc[(size_t)t * D] = (double)bf2f(xc[(size_t)t * D]);
        return;
    }
    const GroupQ q = group_params(mn, mx, bits);
    for (int t = sl; t < S; t += 8) oc[(size_t)t * D] = dq(code_of(bf2f(xc[(size_t)t * D]), q), q.s_bits, q.z_bits);
}

// Block-level fp64 sum (fixed order).
template <int NT>
__device__ double block_sum(double v, double* red) {
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    double r = red[0];
    __syncthreads();
    return r;
}

// sum over elements with |x| >= delta of |x - x_hat| / |x|, and their count -> part[block][2]
__global__ void __launch_bounds__(256) relerr_kernel(const uint16_t* __restrict__ x, const double* __restrict__ xh,
                                                     size_t n, double* __restrict__ part) {
    __shared__ double red[256];
    double s = 0.0, c = 0.0;
    for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) {
        double xv = (double)bf2f(x[i]);
        if (fabs(xv) >= kDelta) { s += fabs(xv - xh[i]) / fabs(xv); c += 1.0; }
    }
    s = block_sum<256>(s, red);
    c = block_sum<256>(c, red);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = s; part[2 * blockIdx.x + 1] = c; }
}

// One CTA per (query i, query head hq).  ref pass: write a_ref, o_ref.  cmp pass: write
// err[hq][i] = {sum |a - a_hat|, sum_{|o|>=d} |o - o_hat| / |o|, count, sum |o - o_hat|, sum |o|}.
__global__ void __launch_bounds__(128) attn_kernel(const uint16_t* __restrict__ Q, const double* __restrict__ Kx,
                                                   const double* __restrict__ Vx, int H_q, int T_q, int q_pos0,
                                                   int H_kv, int S, double scale, int cmp, double* __restrict__ a_ref,
                                                   double* __restrict__ o_ref, double* __restrict__ err) {
    extern __shared__ double sm[];
    double* qs = sm;               // [D]
    double* p = qs + D;            // [S]
    double* red = p + S;           // [128]
    const int i = blockIdx.x, hq = blockIdx.y;
    const int g = H_q / H_kv, hk = hq / g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = q_pos0 + i + 1;                       // attends to tokens [0, q_pos0 + i]
    qs[tid] = (double)bf2f(Q[((size_t)hq * T_q + i) * D + tid]);
    __syncthreads();
    const double* Kh = Kx + (size_t)hk * S * D;
    const double* Vh = Vx + (size_t)hk * S * D;
    // logits: one warp per token, lane = 4 channels
    double lmax = -INFINITY;
    for (int t = warp; t < n; t += 4) {
        const double* kr = Kh + (size_t)t * D + 4 * lane;
        double s = qs[4 * lane] * kr[0] + qs[4 * lane + 1] * kr[1] + qs[4 * lane + 2] * kr[2] + qs[4 * lane + 3] * kr[3];
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
        s *= scale;
        if (lane == 0) p[t] = s;
        lmax = fmax(lmax, s);
    }
    red[tid] = lmax;
    __syncthreads();
    for (int s2 = 64; s2 > 0; s2 >>= 1) {
        if (tid < s2) red[tid] = fmax(red[tid], red[tid + s2]);
        __syncthreads();
    }
    const double m = red[0];
    __syncthreads();
    double ls = 0.0;
    for (int t = tid; t < n; t += 128) { double e = exp(p[t] - m); p[t] = e; ls += e; }
    const double l = block_sum<128>(ls, red);
    for (int t = tid; t < n; t += 128) p[t] /= l;
    __syncthreads();
    double o = 0.0;
    for (int t = 0; t < n; ++t) o += p[t] * Vh[(size_t)t * D + tid];
    const size_t qrow = (size_t)hq * T_q + i;
    if (!cmp) {
        for (int t = tid; t < n; t += 128) a_ref[qrow * S + t] = p[t];
        o_ref[qrow * D + tid] = o;
        return;
    }
    double ea = 0.0;
    for (int t = tid; t < n; t += 128) ea += fabs(a_ref[qrow * S + t] - p[t]);
    const double orf = o_ref[qrow * D + tid];
    const double e = fabs(orf - o);
    const bool ok = fabs(orf) >= kDelta;
    ea = block_sum<128>(ea, red);
    const double eo = block_sum<128>(ok ? e / fabs(orf) : 0.0, red);
    const double ec = block_sum<128>(ok ? 1.0 : 0.0, red);
    const double l1n = block_sum<128>(e, red);
    const double l1d = block_sum<128>(fabs(orf), red);
    if (tid == 0) {
        double* er = err + qrow * 5;
        er[0] = ea; er[1] = eo; er[2] = ec; er[3] = l1n; er[4] = l1d;
    }
}

// Single-CTA final reduction in a fixed order -> out (one kvt_errors).
__global__ void __launch_bounds__(256) final_kernel(const double* __restrict__ pk, const double* __restrict__ pv,
                                                    int nred, const double* __restrict__ err, int nq,
                                                    double n_unmasked, kvt_errors* out) {
    __shared__ double red[256];
    double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = threadIdx.x; j < nred; j += 256) { v[0] += pk[2 * j]; v[1] += pk[2 * j + 1]; v[2] += pv[2 * j]; v[3] += pv[2 * j + 1]; }
    for (int j = threadIdx.x; j < nq; j += 256)
        for (int k = 0; k < 5; ++k) v[4 + k] += err[(size_t)j * 5 + k];
    double r[9];
    for (int k = 0; k < 9; ++k) r[k] = block_sum<256>(v[k], red);
    if (threadIdx.x == 0) {
        kvt_errors e;
        e.e_k = r[1] > 0 ? r[0] / r[1] : 0.0;
        e.e_v = r[3] > 0 ? r[2] / r[3] : 0.0;
        e.e_a = n_unmasked > 0 ? r[4] / n_unmasked : 0.0;
        e.e_o = r[6] > 0 ? r[5] / r[6] : 0.0;
        e.e_o_l1 = r[8] > 0 ? r[7] / r[8] : 0.0;
        *out = e;
    }
}

struct WsLayout {
    size_t kd, vd, kh, vh, aref, oref, pk, pv, err, total;
};

WsLayout layout(int H_q, int T_q, int H_kv, int S) {
    WsLayout w;
    size_t kv = (size_t)H_kv * S * D * sizeof(double);
    size_t off = 0;
    auto take = [&](size_t n) { size_t o = off; off += (n + 255) & ~(size_t)255; return o; };
    w.kd = take(kv); w.vd = take(kv); w.kh = take(kv); w.vh = take(kv);
    w.aref = take((size_t)H_q * T_q * S * sizeof(double));
    w.oref = take((size_t)H_q * T_q * D * sizeof(double));
    w.pk = take((size_t)kRedBlocks * 2 * sizeof(double));
    w.pv = take((size_t)kRedBlocks * 2 * sizeof(double));
    w.err = take((size_t)H_q * T_q * 5 * sizeof(double));
    w.total = off;
    return w;
}

}  // namespace

size_t sensitivity_workspace(int H_q, int T_q, int H_kv, int S, int d, int G) {
    (void)d; (void)G;
    return layout(H_q, T_q, H_kv, S).total;
}

int32_t launch_sensitivity(int mode, int G, int R, const uint16_t* q, int H_q, int T_q, int q_pos0,
                           const uint16_t* k, const uint16_t* v, int H_kv, int S, int d, float scale,
                           const kvt_pair* pairs, int n_pairs, kvt_errors* out, void* ws, size_t ws_bytes,
                           void* stream_) {
    (void)d;
    if (S > kMaxS) return fail(KVT_ERR_UNSUPPORTED, "sensitivity: seq_len %d > %d", S, kMaxS);
    WsLayout L = layout(H_q, T_q, H_kv, S);
    if (L.total > ws_bytes) return fail(KVT_ERR_WORKSPACE, "sensitivity: workspace too small");
    cudaStream_t st = (cudaStream_t)stream_;
    char* base = (char*)ws;
    double* Kd = (double*)(base + L.kd);
    double* Vd = (double*)(base + L.vd);
    double* Kh = (double*)(base + L.kh);
    double* Vh = (double*)(base + L.vh);
    double* aref = (double*)(base + L.aref);
    double* oref = (double*)(base + L.oref);
    double* pk = (double*)(base + L.pk);
    double* pv = (double*)(base + L.pv);
    double* err = (double*)(base + L.err);
    const size_t attn_smem = (size_t)(D + S + 128) * sizeof(double);
    if (attn_smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attn_smem);
        if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "sensitivity smem attr: %s", cudaGetErrorString(e));
    }
    const dim3 rows_grid(H_kv, (S + 3) / 4);
    // full-precision reference (K, V as exact fp64)
    dequant_rows_kernel<<<rows_grid, 128, 0, st>>>(k, Kd, S, 16, G, S, 0);
    dequant_rows_kernel<<<rows_grid, 128, 0, st>>>(v, Vd, S, 16, G, S, 0);
    const dim3 attn_grid(T_q, H_q);
    const double sc = (double)scale;
    attn_kernel<<<attn_grid, 128, attn_smem, st>>>(q, Kd, Vd, H_q, T_q, q_pos0, H_kv, S, sc, 0, aref, oref, err);
    double n_unmasked = 0.0;
    for (int i = 0; i < T_q; ++i) n_unmasked += (double)(q_pos0 + i + 1);
    n_unmasked *= (double)H_q;
    const size_t nel = (size_t)H_kv * S * D;
    for (int p = 0; p < n_pairs; ++p) {
        const int kb = pairs[p].key_bits, vb = pairs[p].value_bits;
        const int nqK = nq_key(mode, kb, G, R, S);
        const int nqV = nq_per_token(vb, R, S);
        if (mode == KVT_MODE_PER_CHANNEL_ASYM) {
            dequant_cols_kernel<<<H_kv, 1024, 0, st>>>(k, Kh, S, kb);
            dequant_cols_kernel<<<H_kv, 1024, 0, st>>>(v, Vh, S, vb);
        } else if (mode == KVT_MODE_KIVI && kb != 16) {
            const int nblk = nqK / G;
            if (nblk > 0) dequant_blocks_kernel<<<dim3(H_kv, (nblk + 3) / 4), 128, 0, st>>>(k, Kh, S, kb, G, nqK);
            dequant_rows_kernel<<<rows_grid, 128, 0, st>>>(k, Kh, S, 16, G, S, nqK);   // exact residual rows
        } else {
            dequant_rows_kernel<<<rows_grid, 128, 0, st>>>(k, Kh, S, kb, G, nqK, 0);
        }
        if (mode != KVT_MODE_PER_CHANNEL_ASYM) dequant_rows_kernel<<<rows_grid, 128, 0, st>>>(v, Vh, S, vb, G, nqV, 0);
        relerr_kernel<<<kRedBlocks, 256, 0, st>>>(k, Kh, nel, pk);
        relerr_kernel<<<kRedBlocks, 256, 0, st>>>(v, Vh, nel, pv);
        attn_kernel<<<attn_grid, 128, attn_smem, st>>>(q, Kh, Vh, H_q, T_q, q_pos0, H_kv, S, sc, 1, aref, oref, err);
        final_kernel<<<1, 256, 0, st>>>(pk, pv, kRedBlocks, err, H_q * T_q, n_unmasked, out + p);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "sensitivity launch: %s", cudaGetErrorString(e));
    return KVT_OK;
}

}  // namespace kvt

// kvt_decode.cu — launch planning for K2 (split-KV decode attention) and K3 (combine).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <mutex>

#include "kvt_decode.cuh"

#if KVT_TRACE
static unsigned long long* g_trace = nullptr;
#endif
namespace kvt {
namespace dec {
using KFn = void (*)(DecodeArgs);
KFn get_decode_k2(int VB, bool KPC, int GM);
KFn get_decode_k4(int VB, bool KPC, int GM);
KFn get_decode_k8(int VB, bool KPC, int GM);
KFn get_decode_k16(int VB, bool KPC, int GM);
KFn get_decode_mma_k2(int VB, int GM, bool kpt, bool paged, size_t* smem);
KFn get_decode_mma_k4(int VB, int GM, bool kpt, bool paged, size_t* smem);
KFn get_decode_mma_k8(int VB, int GM, bool kpt, bool paged, size_t* smem);

// K3: merge n_parts partial rows [n_parts][rows][2 + D] -> out (bf16 / fp32 / partial).  One warp
// per row; lane owns 4 channels.
__global__ void __launch_bounds__(128) combine_kernel(const float* __restrict__ parts, int n_parts, int rows,
                                                      void* out, int out_mode, PushList push) {
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float M = -INFINITY;
    for (int j = 0; j < n_parts; ++j) M = fmaxf(M, parts[((size_t)j * rows + row) * (2 + D)]);
    float L = 0.0f;
    float o[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (M != -INFINITY) {
        for (int j = 0; j < n_parts; ++j) {
            const float* pr = parts + ((size_t)j * rows + row) * (2 + D);
            float wgt = pr[1] * exp2f(pr[0] - M);
            if (wgt == 0.0f) continue;
            L += wgt;
#pragma unroll
            for (int i = 0; i < 4; ++i) o[i] += wgt * pr[2 + 4 * lane + i];
        }
    }
    if (out_mode == 2) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            store_partial(push, out, (size_t)row, 4 * lane + i, M, L, L > 0.0f ? __fdiv_rn(o[i], L) : 0.0f);
        return;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float v = L > 0.0f ? __fdiv_rn(o[i], L) : 0.0f;
        if (out_mode == 1) reinterpret_cast<float*>(out)[(size_t)row * D + 4 * lane + i] = v;
        else reinterpret_cast<__nv_bfloat16*>(out)[(size_t)row * D + 4 * lane + i] = __float2bfloat16_rn(v);
    }
}


static size_t smem_bytes(int VB, int GM) {
    auto pick = [&](auto gm_tag) -> size_t {
        constexpr int GMv = decltype(gm_tag)::value;
        switch (VB) {
            case 2: return Smem<GMv, 2>::bytes;
            case 4: return Smem<GMv, 4>::bytes;
            case 8: return Smem<GMv, 8>::bytes;
            default: return Smem<GMv, 16>::bytes;
        }
    };
    return GM == 4 ? pick(std::integral_constant<int, 4>{}) : pick(std::integral_constant<int, 8>{});
}

struct Instance {
    KFn fn = nullptr;
    size_t smem = 0;
    int occ = 1;
};

static int bits_index(int b) { return b == 2 ? 0 : b == 4 ? 1 : b == 8 ? 2 : 3; }

// Per-device cache of (function, smem, occupancy) for each instance; configured once.
static std::mutex g_mu;
static Instance g_inst[8][4][4][4][2][2];   // [device][kb][vb][kind: 0/1 generic per-token/per-channel, 2/3 mma KIVI/per-token][gm][paged]
static bool g_ready[8][4][4][4][2][2];
static int g_sms[8];

// kind: 0 = generic CUDA-core kernel (per-token key), 1 = generic (per-channel key), 2 = tensor-core KIVI
static int32_t get_instance(int kb, int vb, int kind, int GM, Instance* out, int* sms, bool paged = false) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 8) return fail(KVT_ERR_CUDA, "cudaGetDevice failed");
    int ki = bits_index(kb), vi = bits_index(vb), gi = GM == 4 ? 0 : 1;
    std::lock_guard<std::mutex> lk(g_mu);
    const int pi = paged && kind >= 2 ? 1 : 0;
    if (!g_ready[dev][ki][vi][kind][gi][pi]) {
        Instance in;
        if (kind >= 2) {
            const bool kpt = kind == 3;
            switch (kb) {
                case 2: in.fn = get_decode_mma_k2(vb, GM, kpt, paged, &in.smem); break;
                case 4: in.fn = get_decode_mma_k4(vb, GM, kpt, paged, &in.smem); break;
                default: in.fn = get_decode_mma_k8(vb, GM, kpt, paged, &in.smem); break;
            }
        } else {
            const bool kpc = kind == 1;
            switch (kb) {
                case 2: in.fn = get_decode_k2(vb, kpc, GM); break;
                case 4: in.fn = get_decode_k4(vb, kpc, GM); break;
                case 8: in.fn = get_decode_k8(vb, kpc, GM); break;
                default: in.fn = get_decode_k16(vb, kpc, GM); break;
            }
            in.smem = smem_bytes(vb, GM);
        }
        cudaError_t e = cudaFuncSetAttribute(in.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)in.smem);
        if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&in.occ, in.fn, kThreads, in.smem);
        if (e != cudaSuccess || in.occ < 1) in.occ = 1;
        if (!g_sms[dev]) {
            int n = 0;
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
            g_sms[dev] = n > 0 ? n : 148;
        }
        g_inst[dev][ki][vi][kind][gi][pi] = in;
        g_ready[dev][ki][vi][kind][gi][pi] = true;
    }
    *out = g_inst[dev][ki][vi][kind][gi][pi];
    *sms = g_sms[dev];
    return KVT_OK;
}

// Number of KV splits: enough CTAs for ~4 waves of resident CTAs, at least 16 tiles per split.
static int plan_splits(const Geometry& g, int plan_len, int occ, int sms) {
    static const int forced = [] { const char* e = getenv("KVT_NSPLIT"); return e ? atoi(e) : 0; }();
    if (forced > 0) return forced;                      // experiments only
    int n_tiles = (plan_len + kTile - 1) / kTile;
    long long base = (long long)g.B * g.H;
    long long target = 4LL * sms * occ;
    int n = (int)((target + base - 1) / base);
    int max_by_len = n_tiles / 16;
    if (n > max_by_len) n = max_by_len;
    if (n < 1) n = 1;
    if (n > 64) n = 64;
    return n;
}

// The tensor-core kernel covers exactly the caches with tile records (G = 32, d = 128, 2/4/8-bit K and V,
// either mode); everything else (bf16 layers, G = 64/128) runs the generic CUDA-core kernel.
static int kernel_kind(const Geometry& g) {
    if (g.v_blocked) return g.key_per_channel ? 2 : 3;   // tile records: tensor-core kernel (KIVI / per-token keys)
    return g.key_per_channel ? 1 : 0;
}

}  // namespace dec

static size_t parts_bytes(int ns, int B, int H_q) { return ((size_t)ns * B * H_q * (dec::D + 2) * sizeof(float) + 255) & ~(size_t)255; }
static size_t counters_bytes(const Geometry& g) { return ((size_t)g.B * g.H * sizeof(int) + 255) & ~(size_t)255; }
// stream-K partial slots of the tensor-core kernel: [n_cta][2][8 heads][D + 2]
static size_t sk_parts_bytes(int n_cta) { return ((size_t)n_cta * 2 * 8 * (dec::D + 2) * sizeof(float) + 255) & ~(size_t)255; }
// schedule counters of the per-SM plan (kvt_decode_mma.cuh, sm_claim): 2 x 256 per-%smid words, 2 scalars and one
// claim word per item (<= units + SMs); at a fixed offset after the merge counters (depends on B * H and the SM count
// only, so layers of any precision pair sharing one workspace never see their counters overwritten by partials)
static size_t sched_bytes(const Geometry& g, int sms) {
    return ((2 * 256 + 2 + (size_t)g.B * g.H + (size_t)sms) * sizeof(int) + 255) & ~(size_t)255;
}

// Per-SM plan (whole units in slots 0 .. w-1 of every SM, one piece of the remaining units in slot w) where the
// whole-unit plan would leave ceil(U / SMs) units on some SMs and floor(U / SMs) on others: w = floor(U / SMs)
// >= 2 whole units per SM, a slot to spare (w + 1 <= occupancy) and a remainder to spread.  Returns w, or 0.
// Measured (one layer, B = 64, 8k): Llama K4V2 145 -> 135 us, K4V4 156 -> 148, K2V2 141 -> 131 (w = 3); with w = 1
// (Qwen g = 7: one whole unit + a piece on 3-CTA SMs) it lost (K4V4 106 -> 113 us): once the piece is done the
// whole unit runs alone on its SM with 4 warps, which cannot keep the SM busy.
static int plan_sm_w(const Geometry& g, int occ, int sms) {
    // A/B switch: 0 = off, unset/1 = the rule below, 2 = also w = 1
    static const int on = [] { const char* e = getenv("KVT_SMPLAN"); return e ? atoi(e) : 1; }();
    if (!on) return 0;
    const long long units = (long long)g.B * g.H, slots = (long long)occ * sms;
    const long long per_sm = (units + sms - 1) / sms;
    const bool whole = units <= slots && 2 * units >= 3LL * sms && 5 * per_sm * sms <= 6 * units;   // plan_ctas' rule
    const long long w = units / sms;
    if (!whole || w < (on == 2 ? 1 : 2) || w + 1 > occ || units % sms == 0) return 0;
    return (int)w;
}

// Stream-K CTAs (tensor-core kernel): at most one wave of resident CTAs (estimated from plan_len; the kernel
// clamps to the actual total work).
static int plan_ctas(const Geometry& g, int plan_len, int occ, int sms) {
    static const int forced = [] { const char* e = getenv("KVT_NCTA"); return e ? atoi(e) : 0; }();
    if (forced > 0) return forced;                      // experiments only
    const long long units = (long long)g.B * g.H;
    const long long C = units * dec::unit_cost(g, plan_len).cost;
    const long long slots = (long long)occ * sms;
    // Whole units (no cut, no merge) when they fit one wave, give most SMs at least two CTAs, and the
    // busiest SM holds at most 1.2x the average: cutting a unit costs more than that imbalance
    // (measured, one layer at 8k: Qwen 256 units on 444 slots 108.5 us uncut vs 117.8 us stream-K, per-token
    // K8V2 99 vs 118 us; Llama 512 units on 592 slots 2.5% faster uncut; but 160 units: stream-K 22% faster,
    // 128 units: 12% faster — a single 4-warp CTA cannot keep an SM busy).
    const long long per_sm = (units + sms - 1) / sms;
    if (units <= slots && 2 * units >= 3LL * sms && 5 * per_sm * sms <= 6 * units) return (int)units;
    long long n = (C + 15) / 16;                        // cut units only into pieces of >= ~16 work units
    if (n < units) n = units;                           // ... but never leave whole units waiting in line
    if (n > slots) n = slots;
    return n < 1 ? 1 : (int)n;
}

size_t decode_workspace(const Geometry& g, int H_q, int plan_len) {
    using namespace dec;
    int GM = (H_q / g.H) <= 4 ? 4 : 8;
    Instance in; int sms = 148;
    if (get_instance(g.kb, g.vb, kernel_kind(g), GM, &in, &sms) != KVT_OK) { in.occ = 4; sms = 148; }
    if (kernel_kind(g) >= 2) {
        const int w = plan_sm_w(g, in.occ, sms);
        const int n = w ? in.occ * sms : plan_ctas(g, plan_len, in.occ, sms);
        return n > 1 ? counters_bytes(g) + sched_bytes(g, sms) + sk_parts_bytes(w ? sms : n) : 0;
    }
    int ns = plan_splits(g, plan_len, in.occ, sms);
    return ns > 1 ? counters_bytes(g) + sched_bytes(g, sms) + parts_bytes(ns, g.B, H_q) : 0;
}

int32_t decode_plan(const Geometry& g, int H_q, int plan_len, int32_t out[4]) {
    using namespace dec;
    const int GM = (H_q / g.H) <= 4 ? 4 : 8;
    Instance in; int sms = 148;
    const int kind = kernel_kind(g);
    int32_t st = get_instance(g.kb, g.vb, kind, GM, &in, &sms);
    if (st) return st;
    if (kind >= 2) {
        const int w = plan_sm_w(g, in.occ, sms);
        out[0] = 1; out[1] = w ? in.occ * sms : plan_ctas(g, plan_len, in.occ, sms); out[2] = w;
    } else {
        out[0] = 0; out[1] = plan_splits(g, plan_len, in.occ, sms); out[2] = 0;
    }
    out[3] = in.occ;
    return KVT_OK;
}

int32_t launch_decode(const Geometry& g, const CachePtrs& c, const uint16_t* q, int H_q, const int32_t* seq_len,
                      int plan_len, float scale, void* out, int out_mode, void* workspace, size_t ws_bytes,
                      void* stream, float* const* push, int n_push, bool early) {
    using namespace dec;
    const int gq = H_q / g.H;
    const int GM = gq <= 4 ? 4 : 8;
    Instance in; int sms = 148;
    int32_t st = get_instance(g.kb, g.vb, kernel_kind(g), GM, &in, &sms, c.bt != nullptr);
    if (st) return st;
    const int kind = kernel_kind(g);
    if (g.B > 65535 || g.H > 65535) return fail(KVT_ERR_UNSUPPORTED, "decode: batch/heads exceed grid limits");
    DecodeArgs a;
    a.g = g; a.c = c; a.q = q; a.H_q = H_q; a.gq = gq; a.seq_len = seq_len;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.out = out;
    a.final_mode = out_mode;
    a.push.n = n_push;
    a.early = early ? 1 : 0;
    for (int i = 0; i < kMaxPush; ++i) a.push.p[i] = i < n_push ? push[i] : nullptr;
    if (kind >= 2) {
        // tensor-core kernel: stream-K over all (b, kv head) units, fused merge of units cut across CTAs
        const int w = plan_sm_w(g, in.occ, sms);
        const int n = w ? in.occ * sms : plan_ctas(g, plan_len, in.occ, sms);
        const size_t need = n > 1 ? counters_bytes(g) + sched_bytes(g, sms) + sk_parts_bytes(w ? sms : n) : 0;
        if (need > ws_bytes || (need && !workspace))
            return fail(KVT_ERR_WORKSPACE, "decode: workspace %zu < %zu bytes (use kvt_decode_workspace_bytes)", ws_bytes, need);
        a.out_mode = out_mode;
        // the merge counters sit at offset 0 and the schedule counters right after them (their places depend only
        // on B * H and the SM count, not on this layer's CTA count, so calls with different instances can share one
        // workspace); the partial slots follow them
        a.counters = n > 1 ? (int*)workspace : nullptr;
        a.sched = n > 1 ? (int*)((char*)workspace + counters_bytes(g)) : nullptr;
        a.parts = n > 1 ? (float*)((char*)workspace + counters_bytes(g) + sched_bytes(g, sms)) : nullptr;
        a.sm_w = w;
        a.sm_n = sms;
        static const int drop = [] { const char* e = getenv("KVT_SMPLAN_DROP"); return e ? atoi(e) : 0; }();
        a.sm_drop = drop;
        // the first CTA to arrive on an SM runs ahead of the later ones (traced: the 3 whole units of an SM end at
        // 106 / 113 / 123 us); giving it the piece ends the piece early instead of last: llama-3.25 13 880 -> 14 226
        // tokens/s (KVT_PIECE_FIRST=0 restores the last-arriver piece, A/B only)
        static const int piece_first = [] { const char* e = getenv("KVT_PIECE_FIRST"); return e ? atoi(e) : 1; }();
        a.sm_piece_first = piece_first;
        a.n_split = 1;
        a.n_cta = n;
        a.trace = nullptr;
#if KVT_TRACE
        if (!g_trace) { cudaMalloc(&g_trace, sizeof(unsigned long long) * 15 * 4096); }
        cudaMemsetAsync(g_trace, 0, sizeof(unsigned long long) * 15 * 4096, (cudaStream_t)stream);
        a.trace = g_trace;
#endif
        // programmatic dependent launch: the kernel's prologue (length scan, q setup) may overlap the tail of
        // the preceding kernel in the stream (the append of the same layer, which triggers its dependents at
        // entry); the kernel waits (griddepcontrol.wait) before its first read of the cache
        // Only when the grid (nearly) fills the wave: CTAs dispatched while the append still occupies SMs are
        // placed unevenly, which a partial wave cannot absorb (Qwen, 256 whole units on 444 slots: 15 449
        // tokens/s with PDL vs 19 583 without; Llama, 512 on 592: +2% with PDL).
        // KVT_PDL: 0 = never, unset/1 = the rule below, 2 = also with the per-SM plan (A/B only)
        static const int pdl_env = [] { const char* e = getenv("KVT_PDL"); return e ? atoi(e) : 1; }();
        // Not with the per-SM plan either: llama-3.25 step 4.606 ms without PDL vs 4.682 ms with it (B = 64).
        const bool pdl = pdl_env != 0 && 4LL * n >= 3LL * in.occ * sms && (w == 0 || pdl_env == 2);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = in.smem;
        cfg.stream = (cudaStream_t)stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, in.fn, a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "decode launch: %s", cudaGetErrorString(e));
        return KVT_OK;
    }
    int ns = plan_splits(g, plan_len, in.occ, sms);
    size_t need = ns > 1 ? counters_bytes(g) + sched_bytes(g, sms) + parts_bytes(ns, g.B, H_q) : 0;
    if (need > ws_bytes || (need && !workspace))
        return fail(KVT_ERR_WORKSPACE, "decode: workspace %zu < %zu bytes (use kvt_decode_workspace_bytes)", ws_bytes, need);
    a.out_mode = ns > 1 ? 3 : out_mode;
    // after the (untouched) counter regions, so a tensor-core layer sharing this workspace keeps its zeroed counters
    a.parts = ns > 1 ? (float*)((char*)workspace + counters_bytes(g) + sched_bytes(g, sms)) : nullptr;
    a.sched = nullptr;
    a.sm_w = 0;
    a.sm_n = sms;
    a.sm_drop = 0;
    a.sm_piece_first = 0;
    a.n_split = ns;
    a.counters = nullptr;      // the generic kernel merges its splits with the separate combine launch
    a.n_cta = 0;
    a.trace = nullptr;
    dim3 grid(ns, g.H, g.B);
    in.fn<<<grid, kThreads, in.smem, (cudaStream_t)stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "decode launch: %s", cudaGetErrorString(e));
    if (ns > 1) {
        int rows = g.B * H_q;
        combine_kernel<<<(rows + 3) / 4, 128, 0, (cudaStream_t)stream>>>(a.parts, ns, rows, out, out_mode, a.push);
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "combine launch: %s", cudaGetErrorString(e));
    }
    return KVT_OK;
}

int32_t launch_combine(const float* parts, int n_parts, int B, int H_q, int d, void* out, int out_dtype, void* stream) {
    using namespace dec;
    (void)d;
    int rows = B * H_q;
    combine_kernel<<<(rows + 3) / 4, 128, 0, (cudaStream_t)stream>>>(parts, n_parts, rows, out, out_dtype, PushList{});
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KVT_ERR_CUDA, "combine launch: %s", cudaGetErrorString(e));
    return KVT_OK;
}

}  // namespace kvt

#if KVT_TRACE
extern "C" int32_t kvt_debug_trace(unsigned long long* host, int32_t n) {
    return g_trace && cudaMemcpy(host, g_trace, sizeof(unsigned long long) * 15 * 4096, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 8;
}
#endif

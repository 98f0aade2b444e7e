/*
 * kvt_oracle.c — CPU oracle for the KVTuner hot path.  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Plain, slow, step-by-step C following the paper's definitions (citations per function):
 *   O1  Eq. 2 round-to-nearest asymmetric quantisation
 *   O2  cache regions (per-token window R; KIVI K block flush)    P:707 ("residual length 32,
 *       group size 32"), P:525 ("follow ... KIVI"); readings A5-A8 in DESIGN.md
 *   O3  Eq. 1 attention over the dequantised cache, fp64
 *   O4  the e_k, e_v, e_a, e_o error metrics                       P:146-151, App. B
 *
 * Where the paper is silent the reading is recorded in DESIGN.md §3 and cited here as A<n>.
 * Compile: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (no -ffast-math: IEEE fp32 order
 * matters for the bit-exact codes, A4).
 */
#include "kvt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* bf16 <-> fp32                                                                               */
/* ------------------------------------------------------------------------------------------ */
static uint32_t f32_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float bits_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

float kvto_bf16_to_f32(uint16_t b) { return bits_f32((uint32_t)b << 16); }

uint16_t kvto_f32_to_bf16_rne(float f) {
    uint32_t u = f32_bits(f);
    if (isnan(f)) return (uint16_t)((u >> 16) | 0x40);
    uint32_t lsb = (u >> 16) & 1u;
    return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

/* Round toward +infinity: a positive value with any discarded bit set moves up one bf16 ulp;
 * a negative value is truncated (its magnitude shrinks, i.e. it moves toward +inf). */
uint16_t kvto_f32_to_bf16_ru(float f) {
    uint32_t u = f32_bits(f);
    if (isnan(f)) return (uint16_t)((u >> 16) | 0x40);
    uint16_t hi = (uint16_t)(u >> 16);
    if ((u & 0xFFFFu) == 0) return hi;            /* already representable */
    if (u & 0x80000000u) return hi;               /* negative: truncate toward zero */
    return (uint16_t)(hi + 1);                    /* positive: step away from zero (inf stays inf) */
}

/* ------------------------------------------------------------------------------------------ */
/* O1 — Eq. 2 on one group.  Readings: A1 (RNE ties), A2 (degenerate range),       */
/* A3 (bf16 zero = min, bf16 scale rounded up), A4 (fp32 op order, no FMA).                   */
/* ------------------------------------------------------------------------------------------ */
void kvto_quantize_group(const uint16_t* x, int n, int stride, int bits, uint8_t* codes, uint32_t* meta) {
    /* step 2: min and max (exact: bf16 widened to fp32) */
    float mn = kvto_bf16_to_f32(x[0]);
    float mx = mn;
    for (int i = 1; i < n; ++i) {
        float v = kvto_bf16_to_f32(x[(size_t)i * stride]);
        if (v < mn) mn = v;
        if (v > mx) mx = v;
    }
    if (mn == 0.0f) mn = 0.0f;                    /* canonical +0 for the stored zero (A3) */
    /* step 3: z = min X stored as bf16 — exact, mn is a bf16 value */
    uint16_t z_bits = kvto_f32_to_bf16_rne(mn);
    uint16_t s_bits;
    if (mx == mn) {
        /* step 4: degenerate range, s := 1, every code 0, x_hat = z exactly (A2) */
        s_bits = 0x3F80;
        for (int i = 0; i < n; ++i) codes[i] = 0;
    } else {
        /* step 5: s = (max X - min X) / (2^B - 1) in fp32, then rounded UP to bf16 (A3) */
        float qmax = (float)((1 << bits) - 1);
        float range = mx - mn;
        float s32 = range / qmax;
        s_bits = kvto_f32_to_bf16_ru(s32);
        float inv = 1.0f / kvto_bf16_to_f32(s_bits);
        for (int i = 0; i < n; ++i) {
            float v = kvto_bf16_to_f32(x[(size_t)i * stride]);
            float t = (v - mn) * inv;             /* (X - z) / s                        */
            float r = rintf(t);                   /* round(), ties to even (A1)                   */
            r = fmaxf(r, 0.0f);
            r = fminf(r, qmax);
            codes[i] = (uint8_t)r;
        }
    }
    *meta = (uint32_t)s_bits | ((uint32_t)z_bits << 16);
}

/* X_hat = Q(X) * s + z.  code <= 255 (8 bits) times an 8-significant-bit scale is exact in
 * fp64, and so is the sum with the 8-bit zero (A3), so this is the exact reconstruction. */
double kvto_dequant_value(uint8_t code, uint32_t meta) {
    double s = (double)kvto_bf16_to_f32((uint16_t)(meta & 0xFFFFu));
    double z = (double)kvto_bf16_to_f32((uint16_t)(meta >> 16));
    return (double)code * s + z;
}

/* Bit packing: channel c occupies bits [c*bits, (c+1)*bits) of the row, LSB-first. */
void kvto_pack_row(const uint8_t* codes, int d, int bits, uint8_t* row) {
    int nbytes = d * bits / 8;
    memset(row, 0, (size_t)nbytes);
    for (int c = 0; c < d; ++c) {
        for (int k = 0; k < bits; ++k) {
            int bit = c * bits + k;
            if ((codes[c] >> k) & 1) row[bit / 8] |= (uint8_t)(1u << (bit % 8));
        }
    }
}

void kvto_unpack_row(const uint8_t* row, int d, int bits, uint8_t* codes) {
    for (int c = 0; c < d; ++c) {
        uint8_t v = 0;
        for (int k = 0; k < bits; ++k) {
            int bit = c * bits + k;
            if ((row[bit / 8] >> (bit % 8)) & 1) v |= (uint8_t)(1u << k);
        }
        codes[c] = v;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* O2 — regions of a length-S sequence (A6, A7)                                                 */
/* ------------------------------------------------------------------------------------------ */
static int flush_size(int G, int R) { return R > 0 ? R : G; }

int kvto_n_quantized_key(int mode, int bits, int G, int R, int S) {
    if (bits == 16) return S;                     /* bf16 pass-through: stored as is */
    if (mode == KVTO_MODE_KIVI) {                 /* K per-channel, residual flushed in blocks (A7) */
        int F = flush_size(G, R);
        return F * (S / F);
    }
    return S > R ? S - R : 0;                     /* per-token: sliding window of R (A6) */
}

int kvto_n_quantized_value(int mode, int bits, int G, int R, int S) {
    (void)mode; (void)G;
    if (bits == 16) return S;
    return S > R ? S - R : 0;                     /* V is per-token in both modes (A7) */
}

static int row_bytes(int d, int bits) { return bits == 16 ? 2 * d : d * bits / 8; }

static int valid_bits(int b) { return b == 2 || b == 4 || b == 8 || b == 16; }

int kvto_slice_bytes(int mode, int kb, int vb, int G, int R, int d, int cap, size_t out[6]) {
    if (!valid_bits(kb) || !valid_bits(vb) || G <= 0 || R < 0 || d <= 0 || cap < 0) return -1;
    if (d % G != 0 || (d * 2) % 8 != 0) return -1;
    if (mode == KVTO_MODE_KIVI && (R % G != 0 || cap % G != 0)) return -1;
    if (mode != KVTO_MODE_KIVI && mode != KVTO_MODE_PER_TOKEN) return -1;
    int F = flush_size(G, R);
    out[0] = (size_t)cap * row_bytes(d, kb);
    if (kb == 16) { out[1] = 0; out[2] = 0; }
    else if (mode == KVTO_MODE_KIVI) { out[1] = (size_t)(cap / G) * d * 4; out[2] = (size_t)F * d * 2; }
    else { out[1] = (size_t)cap * (d / G) * 4; out[2] = (size_t)R * d * 2; }
    out[3] = (size_t)cap * row_bytes(d, vb);
    if (vb == 16) { out[4] = 0; out[5] = 0; }
    else { out[4] = (size_t)cap * (d / G) * 4; out[5] = (size_t)R * d * 2; }
    if (kb != 16 && vb != 16 && G == 32 && d == 128) {
        /* tile records: K codes, K meta, V codes and V meta of each 32-token block are one
         * contiguous record in k_codes; k_meta, v_codes and v_meta are empty */
        out[0] = out[0] + out[1] + out[3] + out[4];
        out[1] = out[3] = out[4] = 0;
    }
    return 0;
}

/* Blocked value layout: in KIVI mode with G = 32, d = 128 and 2/4/8-bit keys and values, each
 * 32-token block of value codes keeps the bytes of its 32 token-major rows but reorders them so that a
 * token t (tau = t mod 32, ks = tau / 16, r = tau mod 16) and the token 8 positions later share
 * 32-bit words.  A "chunk" (gam, i) is the 4 channels 32 gam + 4 i .. + 3 of one token (4·bits bits,
 * the same bits as in the packed row).  This function returns the byte offset inside the block of
 * byte k of chunk (gam, i) of token tau. */
static size_t vblk_byte(int bits, int tau, int gam, int i, int k) {
    int ks = tau / 16, r = tau % 16;
    if (bits == 2) {            /* one byte; word = [tok j, tok j+4, tok j+8, tok j+12], j = r mod 4 */
        size_t w = ((size_t)((ks * 8 + i) * 4 + r % 4) * 4 + gam);
        return 4 * w + 2 * (size_t)(r / 8) + (size_t)((r % 8) / 4);
    }
    if (bits == 4) {            /* two bytes; word = [tok j (16 bits) | tok j+8 (16 bits)], j = r mod 8 */
        int j = r % 8;
        size_t w = ((size_t)(((ks * 2 + j / 4) * 8 + i) * 4 + j % 4) * 4 + gam);
        return 4 * w + 2 * (size_t)(r / 8) + (size_t)k;
    }
    /* bits == 8: four bytes (channels e = k); words [tok.c0, tok+8.c0, tok.c1, tok+8.c1], [.c2, .., .c3] */
    int j = r % 8;
    size_t u = (size_t)((((ks * 2 + j / 4) * 2 + gam / 2) * 8 + i) * 4 + j % 4);
    size_t w = u * 4 + (size_t)(gam % 2) * 2 + (size_t)(k / 2);
    return 4 * w + 2 * (size_t)(k % 2) + (size_t)(r / 8);
}

/* The blocked layout is used for KIVI layers whose key and value are both quantised, with G = 32 and
 * d = 128; every other cache keeps token-major value rows. */
static int blocked_v(int mode, int kb, int vb, int G, int d) {
    (void)mode;
    return kb != 16 && vb != 16 && G == 32 && d == 128;
}

/* Write the packed row of token t into the blocked value layout. */
static void vblk_store(int bits, int t, const uint8_t* row, uint8_t* codes) {
    uint8_t* blk = codes + (size_t)(t / 32) * 32 * (size_t)(128 * bits / 8);
    int cb = bits / 2;          /* bytes per chunk */
    for (int gam = 0; gam < 4; ++gam)
        for (int i = 0; i < 8; ++i)
            for (int k = 0; k < cb; ++k)
                blk[vblk_byte(bits, t % 32, gam, i, k)] = row[(size_t)(32 * gam + 4 * i) * bits / 8 + k];
}

static void vblk_load(int bits, int t, const uint8_t* codes, uint8_t* row) {
    const uint8_t* blk = codes + (size_t)(t / 32) * 32 * (size_t)(128 * bits / 8);
    int cb = bits / 2;
    for (int gam = 0; gam < 4; ++gam)
        for (int i = 0; i < 8; ++i)
            for (int k = 0; k < cb; ++k)
                row[(size_t)(32 * gam + 4 * i) * bits / 8 + k] = blk[vblk_byte(bits, t % 32, gam, i, k)];
}

/* Tile records, used exactly where the blocked value layout is (G = 32, d = 128, 2/4/8-bit K
 * and V, both modes): the k_codes slice is a sequence of cap/32 records, record j holding block j (tokens
 * 32j .. 32j+31) as [K code rows (32 x d kb/8) | K meta (KIVI: d block words; per-token: 32 x 4 token
 * words) | V codes, blocked (32 x d vb/8) | V meta (32 x 4 u32)].
 * The oracle builds the four parts as separate arrays (the same arrays the other layouts store) and moves
 * the bytes that the history defines into (out of) the records. */
static size_t rec_bytes(int kb, int vb) { return 32 * (size_t)(16 * kb + 16 * vb) + 1024; }

static void records_store(int mode, int kb, int vb, int nqK, int nqV, const uint8_t* kc, const uint32_t* km,
                          const uint8_t* vc, const uint32_t* vm, uint8_t* rec) {
    size_t RB = rec_bytes(kb, vb), rk = (size_t)16 * kb, rv = (size_t)16 * vb;
    for (int t = 0; t < nqK; ++t) memcpy(rec + (size_t)(t / 32) * RB + (size_t)(t % 32) * rk, kc + (size_t)t * rk, rk);
    if (mode == KVTO_MODE_KIVI)   /* K meta of block j: 128 channel words */
        for (int j = 0; j < nqK / 32; ++j) memcpy(rec + (size_t)j * RB + 32 * rk, km + (size_t)j * 128, 512);
    else                          /* per-token K meta: 4 group words of token t at row t mod 32 */
        for (int t = 0; t < nqK; ++t)
            memcpy(rec + (size_t)(t / 32) * RB + 32 * rk + (size_t)(t % 32) * 16, km + (size_t)t * 4, 16);
    for (int t = 0; t < nqV; ++t) {
        /* the blocked bytes of token t: every chunk byte of token t in block t / 32 */
        const uint8_t* blk = vc + (size_t)(t / 32) * 32 * rv;
        uint8_t* dst = rec + (size_t)(t / 32) * RB + 32 * rk + 512;
        for (int gam = 0; gam < 4; ++gam)
            for (int i = 0; i < 8; ++i)
                for (int k = 0; k < vb / 2; ++k) {
                    size_t o = vblk_byte(vb, t % 32, gam, i, k);
                    dst[o] = blk[o];
                }
        memcpy(rec + (size_t)(t / 32) * RB + 32 * rk + 512 + 32 * rv + (size_t)(t % 32) * 16, vm + (size_t)t * 4, 16);
    }
}

static void records_load(int mode, int kb, int vb, int nqK, int nqV, const uint8_t* rec, uint8_t* kc, uint32_t* km,
                         uint8_t* vc, uint32_t* vm) {
    size_t RB = rec_bytes(kb, vb), rk = (size_t)16 * kb, rv = (size_t)16 * vb;
    for (int t = 0; t < nqK; ++t) memcpy(kc + (size_t)t * rk, rec + (size_t)(t / 32) * RB + (size_t)(t % 32) * rk, rk);
    if (mode == KVTO_MODE_KIVI)
        for (int j = 0; j < nqK / 32; ++j) memcpy(km + (size_t)j * 128, rec + (size_t)j * RB + 32 * rk, 512);
    else
        for (int t = 0; t < nqK; ++t)
            memcpy(km + (size_t)t * 4, rec + (size_t)(t / 32) * RB + 32 * rk + (size_t)(t % 32) * 16, 16);
    for (int t = 0; t < nqV; ++t) {
        const uint8_t* src = rec + (size_t)(t / 32) * RB + 32 * rk + 512;
        uint8_t* blk = vc + (size_t)(t / 32) * 32 * rv;
        for (int gam = 0; gam < 4; ++gam)
            for (int i = 0; i < 8; ++i)
                for (int k = 0; k < vb / 2; ++k) {
                    size_t o = vblk_byte(vb, t % 32, gam, i, k);
                    blk[o] = src[o];
                }
        memcpy(vm + (size_t)t * 4, rec + (size_t)(t / 32) * RB + 32 * rk + 512 + 32 * rv + (size_t)(t % 32) * 16, 16);
    }
}

/* Per-token tensor (V in both modes, K in per-token mode): token t < n_q is split into d/G channel
 * groups, each quantised by O1 and packed into row t (or into the blocked layout); tokens [n_q, S) stay
 * bf16 in the ring slot t mod R. */
static void build_per_token(int bits, int G, int R, int d, int S, const uint16_t* X,
                            uint8_t* codes, uint32_t* meta, uint16_t* resid, int blocked) {
    int rb = row_bytes(d, bits);
    if (bits == 16) {
        for (int t = 0; t < S; ++t) memcpy(codes + (size_t)t * rb, X + (size_t)t * d, (size_t)rb);
        return;
    }
    int nq = S > R ? S - R : 0;
    uint8_t* tmp = (uint8_t*)malloc((size_t)d);
    for (int t = 0; t < nq; ++t) {
        for (int j = 0; j < d / G; ++j)
            kvto_quantize_group(X + (size_t)t * d + (size_t)j * G, G, 1, bits, tmp + j * G,
                                meta + (size_t)t * (d / G) + j);
        if (blocked) {
            uint8_t row[128];
            kvto_pack_row(tmp, d, bits, row);
            vblk_store(bits, t, row, codes);
        } else {
            kvto_pack_row(tmp, d, bits, codes + (size_t)t * rb);
        }
    }
    for (int t = nq; t < S; ++t)
        memcpy(resid + (size_t)(t % R) * d, X + (size_t)t * d, (size_t)d * 2);
    free(tmp);
}

/* KIVI key (A7/A8): tokens [0, n_qK) form blocks of G tokens; each (block, channel) is one
 * O1 group of G values; tokens [n_qK, S) stay bf16 at linear residual slot t - n_qK. */
static void build_per_channel(int bits, int G, int R, int d, int S, const uint16_t* X,
                              uint8_t* codes, uint32_t* meta, uint16_t* resid) {
    int rb = row_bytes(d, bits);
    int nq = kvto_n_quantized_key(KVTO_MODE_KIVI, bits, G, R, S);
    uint8_t* blk = (uint8_t*)malloc((size_t)G * d);   /* codes of one block, [G][d] */
    uint8_t* col = (uint8_t*)malloc((size_t)G);
    for (int b0 = 0; b0 < nq; b0 += G) {
        for (int c = 0; c < d; ++c) {
            kvto_quantize_group(X + (size_t)b0 * d + c, G, d, bits, col, meta + (size_t)(b0 / G) * d + c);
            for (int i = 0; i < G; ++i) blk[(size_t)i * d + c] = col[i];
        }
        for (int i = 0; i < G; ++i) kvto_pack_row(blk + (size_t)i * d, d, bits, codes + (size_t)(b0 + i) * rb);
    }
    for (int t = nq; t < S; ++t)
        memcpy(resid + (size_t)(t - nq) * d, X + (size_t)t * d, (size_t)d * 2);
    free(blk);
    free(col);
}

int kvto_build_cache(int mode, int kb, int vb, int G, int R, int d, int cap, int S,
                     const uint16_t* K, const uint16_t* V,
                     uint8_t* k_codes, uint32_t* k_meta, uint16_t* k_resid,
                     uint8_t* v_codes, uint32_t* v_meta, uint16_t* v_resid) {
    size_t sz[6];
    if (kvto_slice_bytes(mode, kb, vb, G, R, d, cap, sz) != 0 || S < 0 || S > cap) return -1;
    if (blocked_v(mode, kb, vb, G, d)) {
        /* tile records: build the four parts separately, then place them */
        uint8_t* kc = (uint8_t*)malloc((size_t)cap * 16 * kb + 1);
        uint32_t* km = (uint32_t*)malloc((size_t)(cap / 32) * 512 + 4);
        uint8_t* vc = (uint8_t*)malloc((size_t)cap * 16 * vb + 1);
        uint32_t* vm = (uint32_t*)malloc((size_t)cap * 16 + 4);
        if (mode == KVTO_MODE_KIVI) build_per_channel(kb, G, R, d, S, K, kc, km, k_resid);
        else build_per_token(kb, G, R, d, S, K, kc, km, k_resid, 0);
        build_per_token(vb, G, R, d, S, V, vc, vm, v_resid, 1);
        records_store(mode, kb, vb, kvto_n_quantized_key(mode, kb, G, R, S), kvto_n_quantized_value(mode, vb, G, R, S),
                      kc, km, vc, vm, k_codes);
        free(kc); free(km); free(vc); free(vm);
        return 0;
    }
    if (mode == KVTO_MODE_KIVI && kb != 16)
        build_per_channel(kb, G, R, d, S, K, k_codes, k_meta, k_resid);
    else
        build_per_token(kb, G, R, d, S, K, k_codes, k_meta, k_resid, 0);
    build_per_token(vb, G, R, d, S, V, v_codes, v_meta, v_resid, 0);
    return 0;
}

static void dequant_per_token(int bits, int G, int R, int d, int S, const uint8_t* codes,
                              const uint32_t* meta, const uint16_t* resid, double* Xh, int blocked) {
    int rb = row_bytes(d, bits);
    uint8_t* tmp = (uint8_t*)malloc((size_t)d);
    if (bits == 16) {
        for (int t = 0; t < S; ++t) {
            const uint8_t* row = codes + (size_t)t * rb;
            for (int c = 0; c < d; ++c) {
                uint16_t b = (uint16_t)(row[2 * c] | (row[2 * c + 1] << 8));
                Xh[(size_t)t * d + c] = kvto_bf16_to_f32(b);
            }
        }
        free(tmp);
        return;
    }
    int nq = S > R ? S - R : 0;
    for (int t = 0; t < nq; ++t) {
        if (blocked) {
            uint8_t row[128];
            vblk_load(bits, t, codes, row);
            kvto_unpack_row(row, d, bits, tmp);
        } else {
            kvto_unpack_row(codes + (size_t)t * rb, d, bits, tmp);
        }
        for (int c = 0; c < d; ++c)
            Xh[(size_t)t * d + c] = kvto_dequant_value(tmp[c], meta[(size_t)t * (d / G) + c / G]);
    }
    for (int t = nq; t < S; ++t)
        for (int c = 0; c < d; ++c) Xh[(size_t)t * d + c] = kvto_bf16_to_f32(resid[(size_t)(t % R) * d + c]);
    free(tmp);
}

static void dequant_per_channel(int bits, int G, int R, int d, int S, const uint8_t* codes,
                                const uint32_t* meta, const uint16_t* resid, double* Xh) {
    int rb = row_bytes(d, bits);
    int nq = kvto_n_quantized_key(KVTO_MODE_KIVI, bits, G, R, S);
    uint8_t* tmp = (uint8_t*)malloc((size_t)d);
    for (int t = 0; t < nq; ++t) {
        kvto_unpack_row(codes + (size_t)t * rb, d, bits, tmp);
        for (int c = 0; c < d; ++c)
            Xh[(size_t)t * d + c] = kvto_dequant_value(tmp[c], meta[(size_t)(t / G) * d + c]);
    }
    for (int t = nq; t < S; ++t)
        for (int c = 0; c < d; ++c) Xh[(size_t)t * d + c] = kvto_bf16_to_f32(resid[(size_t)(t - nq) * d + c]);
    free(tmp);
}

int kvto_dequant_cache(int mode, int kb, int vb, int G, int R, int d, int cap, int S,
                       const uint8_t* k_codes, const uint32_t* k_meta, const uint16_t* k_resid,
                       const uint8_t* v_codes, const uint32_t* v_meta, const uint16_t* v_resid,
                       double* Khat, double* Vhat) {
    size_t sz[6];
    if (kvto_slice_bytes(mode, kb, vb, G, R, d, cap, sz) != 0 || S < 0 || S > cap) return -1;
    if (blocked_v(mode, kb, vb, G, d)) {
        uint8_t* kc = (uint8_t*)malloc((size_t)cap * 16 * kb + 1);
        uint32_t* km = (uint32_t*)malloc((size_t)(cap / 32) * 512 + 4);
        uint8_t* vc = (uint8_t*)malloc((size_t)cap * 16 * vb + 1);
        uint32_t* vm = (uint32_t*)malloc((size_t)cap * 16 + 4);
        records_load(mode, kb, vb, kvto_n_quantized_key(mode, kb, G, R, S), kvto_n_quantized_value(mode, vb, G, R, S),
                     k_codes, kc, km, vc, vm);
        if (mode == KVTO_MODE_KIVI) dequant_per_channel(kb, G, R, d, S, kc, km, k_resid, Khat);
        else dequant_per_token(kb, G, R, d, S, kc, km, k_resid, Khat, 0);
        dequant_per_token(vb, G, R, d, S, vc, vm, v_resid, Vhat, 1);
        free(kc); free(km); free(vc); free(vm);
        return 0;
    }
    if (mode == KVTO_MODE_KIVI && kb != 16)
        dequant_per_channel(kb, G, R, d, S, k_codes, k_meta, k_resid, Khat);
    else
        dequant_per_token(kb, G, R, d, S, k_codes, k_meta, k_resid, Khat, 0);
    dequant_per_token(vb, G, R, d, S, v_codes, v_meta, v_resid, Vhat, 0);
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* O3 — Eq. 1: a = softmax(q K^T * scale), o = a V, over K_hat, V_hat.      */
/* scale = 1/sqrt(d_head) by default (A9); the max is subtracted before exp (stability only).  */
/* ------------------------------------------------------------------------------------------ */
void kvto_attention(const uint16_t* q, int g, const double* Khat, const double* Vhat, int S, int d,
                    double scale, double* out, double* probs) {
    double* logit = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
    for (int h = 0; h < g; ++h) {
        const uint16_t* qh = q + (size_t)h * d;
        double m = -INFINITY;
        for (int t = 0; t < S; ++t) {
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += (double)kvto_bf16_to_f32(qh[c]) * Khat[(size_t)t * d + c];
            logit[t] = acc * scale;
            if (logit[t] > m) m = logit[t];
        }
        double sum = 0.0;
        for (int t = 0; t < S; ++t) { logit[t] = exp(logit[t] - m); sum += logit[t]; }
        for (int c = 0; c < d; ++c) out[(size_t)h * d + c] = 0.0;
        for (int t = 0; t < S; ++t) {
            double a = logit[t] / sum;
            if (probs) probs[(size_t)h * S + t] = a;
            for (int c = 0; c < d; ++c) out[(size_t)h * d + c] += a * Vhat[(size_t)t * d + c];
        }
    }
    free(logit);
}

/* ------------------------------------------------------------------------------------------ */
/* O4 — layer sensitivity (protocol App. B: offline quantisation of the   */
/* collected cache, decode queries, no accumulation).  Readings A13-A16.                        */
/* ------------------------------------------------------------------------------------------ */
static const double kDelta = 1e-8;   /* exclusion threshold of the relative errors (A13) */

/* per-channel-asym ("quantize KV cache along the channel or token dimension"; Table
 * tab:kvcache_quantization_error_per_channel_per_token_asym): every channel column of the whole trace
 * [0, S) is one Eq. 2 group (O1 with stride d), for keys and values alike (A28). */
static void static_per_channel(int bits, int d, int S, const uint16_t* X, double* Xhat) {
    uint8_t* codes = (uint8_t*)malloc((size_t)S + 1);
    for (int c = 0; c < d; ++c) {
        if (bits == 16) {
            for (int t = 0; t < S; ++t) Xhat[(size_t)t * d + c] = kvto_bf16_to_f32(X[(size_t)t * d + c]);
            continue;
        }
        uint32_t meta;
        kvto_quantize_group(X + c, S, d, bits, codes, &meta);
        for (int t = 0; t < S; ++t) Xhat[(size_t)t * d + c] = kvto_dequant_value(codes[t], meta);
    }
    free(codes);
}

int kvto_sensitivity(int mode, int G, int R, const uint16_t* Q, int H_q, int T_q, int q_pos0,
                     const uint16_t* K, const uint16_t* V, int H_kv, int S, int d, double scale,
                     const int32_t* pair_bits, int n_pairs, double* out) {
    if (H_kv <= 0 || H_q % H_kv != 0 || S <= 0 || T_q < 0 || q_pos0 < 0 || q_pos0 + T_q > S) return -1;
    int g = H_q / H_kv;
    int cap = ((S + G - 1) / G) * G;
    size_t sz[6];
    size_t nKV = (size_t)S * d;
    double* Kf = (double*)malloc(sizeof(double) * nKV);   /* full-precision K, V of one head */
    double* Vf = (double*)malloc(sizeof(double) * nKV);
    double* Kh = (double*)malloc(sizeof(double) * nKV);
    double* Vh = (double*)malloc(sizeof(double) * nKV);
    double* o_ref = (double*)malloc(sizeof(double) * (size_t)d);
    double* o_hat = (double*)malloc(sizeof(double) * (size_t)d);
    double* a_ref = (double*)malloc(sizeof(double) * (size_t)S);
    double* a_hat = (double*)malloc(sizeof(double) * (size_t)S);
    int rc = 0;
    for (int p = 0; p < n_pairs && rc == 0; ++p) {
        int kb = pair_bits[2 * p], vb = pair_bits[2 * p + 1];
        const int pc = mode == KVTO_MODE_PER_CHANNEL;
        if (pc ? (kb != 2 && kb != 4 && kb != 8 && kb != 16) || (vb != 2 && vb != 4 && vb != 8 && vb != 16)
               : kvto_slice_bytes(mode, kb, vb, G, R, d, cap, sz) != 0) { rc = -1; break; }
        if (pc) for (int i = 0; i < 6; ++i) sz[i] = 0;
        uint8_t* kc = (uint8_t*)malloc(sz[0] + 1); uint32_t* km = (uint32_t*)malloc(sz[1] + 4);
        uint16_t* kr = (uint16_t*)malloc(sz[2] + 2); uint8_t* vc = (uint8_t*)malloc(sz[3] + 1);
        uint32_t* vm = (uint32_t*)malloc(sz[4] + 4); uint16_t* vr = (uint16_t*)malloc(sz[5] + 2);
        double ek_sum = 0, ev_sum = 0, ea_sum = 0, eo_sum = 0, l1_num = 0, l1_den = 0;
        long ek_n = 0, ev_n = 0, ea_n = 0, eo_n = 0;
        for (int hk = 0; hk < H_kv; ++hk) {
            const uint16_t* Kx = K + (size_t)hk * nKV;
            const uint16_t* Vx = V + (size_t)hk * nKV;
            /* step 1: static O2 over the whole trace (A15), then read back K_hat, V_hat */
            if (pc) {
                static_per_channel(kb, d, S, Kx, Kh);
                static_per_channel(vb, d, S, Vx, Vh);
            } else {
                kvto_build_cache(mode, kb, vb, G, R, d, cap, S, Kx, Vx, kc, km, kr, vc, vm, vr);
                kvto_dequant_cache(mode, kb, vb, G, R, d, cap, S, kc, km, kr, vc, vm, vr, Kh, Vh);
            }
            for (size_t i = 0; i < nKV; ++i) { Kf[i] = kvto_bf16_to_f32(Kx[i]); Vf[i] = kvto_bf16_to_f32(Vx[i]); }
            /* e_k, e_v = mean |X - X_hat| / |X| over |X| >= delta (A13) */
            for (size_t i = 0; i < nKV; ++i) {
                if (fabs(Kf[i]) >= kDelta) { ek_sum += fabs(Kf[i] - Kh[i]) / fabs(Kf[i]); ++ek_n; }
                if (fabs(Vf[i]) >= kDelta) { ev_sum += fabs(Vf[i] - Vh[i]) / fabs(Vf[i]); ++ev_n; }
            }
            /* steps 2-3: causal decode queries, a/o with (K,V) vs a_hat/o_hat with (K_hat,V_hat) */
            for (int j = 0; j < g; ++j) {
                int hq = hk * g + j;
                for (int i = 0; i < T_q; ++i) {
                    const uint16_t* qv = Q + ((size_t)hq * T_q + i) * d;
                    int n = q_pos0 + i + 1;            /* attends to tokens [0, p_i] */
                    kvto_attention(qv, 1, Kf, Vf, n, d, scale, o_ref, a_ref);
                    kvto_attention(qv, 1, Kh, Vh, n, d, scale, o_hat, a_hat);
                    for (int t = 0; t < n; ++t) { ea_sum += fabs(a_ref[t] - a_hat[t]); ++ea_n; }   /* A16 */
                    for (int c = 0; c < d; ++c) {
                        double e = fabs(o_ref[c] - o_hat[c]);
                        l1_num += e; l1_den += fabs(o_ref[c]);
                        if (fabs(o_ref[c]) >= kDelta) { eo_sum += e / fabs(o_ref[c]); ++eo_n; }
                    }
                }
            }
        }
        out[5 * p + 0] = ek_n ? ek_sum / (double)ek_n : 0.0;
        out[5 * p + 1] = ev_n ? ev_sum / (double)ev_n : 0.0;
        out[5 * p + 2] = ea_n ? ea_sum / (double)ea_n : 0.0;
        out[5 * p + 3] = eo_n ? eo_sum / (double)eo_n : 0.0;
        out[5 * p + 4] = l1_den > 0 ? l1_num / l1_den : 0.0;
        free(kc); free(km); free(kr); free(vc); free(vm); free(vr);
    }
    free(Kf); free(Vf); free(Kh); free(Vh); free(o_ref); free(o_hat); free(a_ref); free(a_hat);
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* Whole-layer decode (cpu_baseline): O2 build + read-back + O3 for every (b, kv head).        */
/* ------------------------------------------------------------------------------------------ */
int kvto_layer_decode(int mode, int kb, int vb, int G, int R, int B, int H_kv, int H_q, int d,
                      int S_max, const int32_t* seq_len, const uint16_t* K, const uint16_t* V,
                      const uint16_t* q, double scale, double* out) {
    if (H_kv <= 0 || H_q % H_kv != 0) return -1;
    int g = H_q / H_kv;
    int cap = ((S_max + G - 1) / G) * G;
    size_t sz[6];
    if (kvto_slice_bytes(mode, kb, vb, G, R, d, cap, sz) != 0) return -1;
    uint8_t* kc = (uint8_t*)malloc(sz[0] + 1); uint32_t* km = (uint32_t*)malloc(sz[1] + 4);
    uint16_t* kr = (uint16_t*)malloc(sz[2] + 2); uint8_t* vc = (uint8_t*)malloc(sz[3] + 1);
    uint32_t* vm = (uint32_t*)malloc(sz[4] + 4); uint16_t* vr = (uint16_t*)malloc(sz[5] + 2);
    double* Kh = (double*)malloc(sizeof(double) * (size_t)S_max * d + 8);
    double* Vh = (double*)malloc(sizeof(double) * (size_t)S_max * d + 8);
    int rc = 0;
    for (int b = 0; b < B && rc == 0; ++b) {
        int S = seq_len[b];
        if (S < 0 || S > S_max) { rc = -1; break; }
        for (int hk = 0; hk < H_kv; ++hk) {
            size_t base = ((size_t)b * H_kv + hk) * (size_t)S_max * d;
            kvto_build_cache(mode, kb, vb, G, R, d, cap, S, K + base, V + base, kc, km, kr, vc, vm, vr);
            kvto_dequant_cache(mode, kb, vb, G, R, d, cap, S, kc, km, kr, vc, vm, vr, Kh, Vh);
            kvto_attention(q + ((size_t)b * H_q + (size_t)hk * g) * d, g, Kh, Vh, S, d, scale,
                           out + ((size_t)b * H_q + (size_t)hk * g) * d, NULL);
        }
    }
    free(kc); free(km); free(kr); free(vc); free(vm); free(vr); free(Kh); free(Vh);
    return rc;
}

/*
 * kvt_oracle.h — CPU oracle for the KVTuner hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the slow, obviously-correct reference that the CUDA path is checked against.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  It shares no code, header, table or constant with paper_2502_04420_b200/ (the
 * product); neither includes the other.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line, "S:<line>" = SPEC.md line, "A<n>" =
 * the reading recorded in DESIGN.md §3 (Readings of the paper).
 *
 * Every floating-point quantity here is fp64 except where the reading fixes fp32 (the Eq. 2
 * statistics, A4).  Compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 */
#ifndef KVT_ORACLE_H
#define KVT_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { KVTO_MODE_PER_TOKEN = 0, KVTO_MODE_KIVI = 1,
       KVTO_MODE_PER_CHANNEL = 2 /* sensitivity only: whole-sequence per-channel K and V (A28) */ };

/* ---- bf16 helpers (the bf16 format: top 16 bits of an IEEE binary32) ---- */
float    kvto_bf16_to_f32(uint16_t b);
uint16_t kvto_f32_to_bf16_rne(float f);   /* round to nearest, ties to even                 */
uint16_t kvto_f32_to_bf16_ru(float f);    /* round toward +infinity (A3: scale rounding)     */

/* ---- O1: Eq. 2 on one quantisation group -----------------------------------------
 * x[i*stride], i < n, are bf16.  Writes n codes (one per byte, unpacked) and the group's meta word
 * (low 16 bits: bf16 scale s_st, high 16 bits: bf16 zero z).  bits in {2,4,8}. */
void kvto_quantize_group(const uint16_t* x, int n, int stride, int bits, uint8_t* codes, uint32_t* meta);

/* x_hat = code * s + z, evaluated in fp64 (exact, A3). */
double kvto_dequant_value(uint8_t code, uint32_t meta);

/* Pack d codes of `bits` bits LSB-first: channel c occupies bits [c*bits, (c+1)*bits) of the row. */
void kvto_pack_row(const uint8_t* codes, int d, int bits, uint8_t* row);
/* Inverse of kvto_pack_row. */
void kvto_unpack_row(const uint8_t* row, int d, int bits, uint8_t* codes);

/* ---- O2: cache regions (A6/A7) --------------------------------------------------- */
/* Number of tokens of a length-S sequence held quantized (the rest are bf16 residual). */
int kvto_n_quantized_key(int mode, int bits, int G, int R, int S);
int kvto_n_quantized_value(int mode, int bits, int G, int R, int S);

/* Byte sizes of the six per-(b,h) buffers of one layer cache with `cap` token rows:
 * [0] k_codes [1] k_meta [2] k_resid [3] v_codes [4] v_meta [5] v_resid.  Returns 0 on success. */
int kvto_slice_bytes(int mode, int kb, int vb, int G, int R, int d, int cap, size_t out[6]);

/* Build the cache state of one (batch row, kv head) from its whole token history K,V [S][d] (bf16),
 * statically (O2 is history independent).  Buffers are one (b,h) slice, laid out as DESIGN.md §4.
 * Bytes outside the valid regions are left untouched.  Returns 0, or -1 on invalid arguments. */
int kvto_build_cache(int mode, int kb, int vb, int G, int R, int d, int cap, int S,
                     const uint16_t* K, const uint16_t* V,
                     uint8_t* k_codes, uint32_t* k_meta, uint16_t* k_resid,
                     uint8_t* v_codes, uint32_t* v_meta, uint16_t* v_resid);

/* Read back the dequantised K_hat, V_hat [S][d] (fp64) from one (b,h) slice of buffers. */
int kvto_dequant_cache(int mode, int kb, int vb, int G, int R, int d, int cap, int S,
                       const uint8_t* k_codes, const uint32_t* k_meta, const uint16_t* k_resid,
                       const uint8_t* v_codes, const uint32_t* v_meta, const uint16_t* v_resid,
                       double* Khat, double* Vhat);

/* ---- O3: Eq. 1 over the dequantised cache, fp64 -------------------------------
 * q: bf16 [g][d] (the g query heads sharing this kv head); Khat, Vhat [S][d] fp64.
 * out: fp64 [g][d].  probs (optional, may be NULL): fp64 [g][S]. */
void kvto_attention(const uint16_t* q, int g, const double* Khat, const double* Vhat, int S, int d,
                    double scale, double* out, double* probs);

/* ---- O4: layer sensitivity (App. B) ---------------------------------
 * Q bf16 [H_q][T_q][d]; K, V bf16 [H_kv][S][d]; query i sits at position q_pos0 + i and attends
 * causally to tokens [0, q_pos0 + i].  For each pair p: out[5p + {0..4}] = e_k, e_v, e_a, e_o,
 * e_o_l1 (A13-A16).  Returns 0, or -1 on invalid arguments. */
int kvto_sensitivity(int mode, int G, int R, const uint16_t* Q, int H_q, int T_q, int q_pos0,
                     const uint16_t* K, const uint16_t* V, int H_kv, int S, int d, double scale,
                     const int32_t* pair_bits /* [n_pairs][2] = (b_k, b_v) */, int n_pairs,
                     double* out /* [n_pairs][5] */);

/* Whole-layer helpers used by the cpu_baseline timing: build + dequant + attention for every
 * (b, h) of one layer with seq_len[b] tokens.  K,V bf16 [B][H_kv][S_max][d], q bf16 [B][H_q][d],
 * out fp64 [B][H_q][d]. */
int kvto_layer_decode(int mode, int kb, int vb, int G, int R, int B, int H_kv, int H_q, int d,
                      int S_max, const int32_t* seq_len, const uint16_t* K, const uint16_t* V,
                      const uint16_t* q, double scale, double* out);

#ifdef __cplusplus
}
#endif
#endif

"""Pins for the oracle's O1 (Eq. 2) and O2 (cache regions) — CPU only.

Each pin checks the oracle against something other than itself: hand-worked bytes
(tests/golden/o1_worked.json), closed-form bounds of Eq. 2, special cases (constant groups,
B=16 pass-through), a hand bit-packing formula, and the region arithmetic of the KIVI reading.
"""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import kvt_synth

GOLD = Path(__file__).parent / "golden"


def bits_of(vals):
    return kvt_synth.bf16_bits(torch.tensor(vals, dtype=torch.float32).to(torch.bfloat16))


# ------------------------------------------------------------------------------------ O1
@pytest.mark.parametrize("case", json.loads((GOLD / "o1_worked.json").read_text())["cases"], ids=lambda c: c["id"])
def test_o1_worked_examples(oracle, case):
    x = bits_of(case["x"])
    codes, meta = oracle.quantize_group(x, case["bits"])
    assert list(codes) == case["codes"]
    assert meta & 0xFFFF == int(case["scale_bf16"], 16)
    assert meta >> 16 == int(case["zero_bf16"], 16)
    packed = oracle.pack_row(codes, case["bits"]) if (len(codes) * case["bits"]) % 8 == 0 else None
    assert packed.tobytes().hex() == case["packed_hex"]
    if case["x_hat"] is not None:
        assert [oracle.dequant_value(int(c), meta) for c in codes] == case["x_hat"]


def _groups(rng_seed, n_groups, n, kind="gauss"):
    g = torch.Generator().manual_seed(rng_seed)
    if kind == "gauss":
        x = torch.randn(n_groups, n, generator=g)
    elif kind == "outlier":
        x = torch.randn(n_groups, n, generator=g)
        x[:, ::8] *= 11
    elif kind == "shifted":
        x = torch.randn(n_groups, n, generator=g) * 0.01 + 100.0
    elif kind == "wide":
        x = torch.randn(n_groups, n, generator=g) * 1e4
    return kvt_synth.bf16_bits(x.to(torch.bfloat16))


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("kind", ["gauss", "outlier", "shifted", "wide"])
def test_o1_roundtrip_bound(oracle, bits, kind):
    """|x - x_hat| <= s_st (1/2 + 2^-10); z = min x exactly; s32 <= s_st < s32 (1 + 2^-7)  (Eq. 2 + A3)."""
    X = _groups(1000 + bits, 400, 32, kind)
    qmax = 2 ** bits - 1
    for row in X:
        codes, meta = oracle.quantize_group(row, bits)
        s, z = oracle.meta_scale_zero(meta)
        xf = oracle.bf16_array_to_f64(row)
        assert z == xf.min()                                   # z = min X, exact in bf16
        assert codes.max() <= qmax
        if xf.max() == xf.min():
            continue
        s_exact = (xf.max() - xf.min()) / qmax                 # the paper's s, real arithmetic
        assert s >= s_exact * (1 - 2.0 ** -22)                 # rounded up (coverage)
        assert s < s_exact * (1 + 2.0 ** -7) * (1 + 2.0 ** -22)
        xh = np.array([oracle.dequant_value(int(c), meta) for c in codes])
        assert np.all(np.abs(xf - xh) <= s * (0.5 + 2.0 ** -10))
        assert xh.max() <= xf.max() + s * 0.5 + 1e-30 and xh.min() == xf.min()


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_o1_error_monotone_in_bits(oracle, bits):
    """mean |x - x_hat| falls as B rises (the 'higher precision, lower error' direction of P:227)."""
    X = _groups(7, 100, 64, "gauss")
    errs = {}
    for b in (2, 4, 8):
        e = 0.0
        for row in X:
            codes, meta = oracle.quantize_group(row, b)
            xh = np.array([oracle.dequant_value(int(c), meta) for c in codes])
            e += np.abs(oracle.bf16_array_to_f64(row) - xh).mean()
        errs[b] = e
    assert errs[8] < errs[4] < errs[2]


def test_o1_constant_groups_exact(oracle):
    """Degenerate range (A2): codes 0, scale 1.0 (0x3F80), x_hat = x exactly — incl. zeros and -0."""
    for v in (0.0, -0.0, 1.5, -7.25, 3.0e5, 1e-20):
        x = bits_of([v] * 32)
        for b in (2, 4, 8):
            codes, meta = oracle.quantize_group(x, b)
            assert not codes.any()
            assert meta & 0xFFFF == 0x3F80
            xh = oracle.dequant_value(0, meta)
            assert xh == oracle.bf16_to_f32(int(x[0])) or (v == 0.0 and xh == 0.0)
    # -0 is stored as +0 (canonical zero, A3)
    codes, meta = oracle.quantize_group(bits_of([-0.0, 0.0, -0.0, 0.0]), 2)
    assert meta >> 16 == 0x0000


def test_o1_grid_idempotent(oracle):
    """Quantising a group that already lies on its own grid reproduces the same codes."""
    X = _groups(11, 50, 32, "gauss")
    for b in (2, 4, 8):
        for row in X:
            codes, meta = oracle.quantize_group(row, b)
            xh = np.array([oracle.dequant_value(int(c), meta) for c in codes], dtype=np.float32)
            xh_bf = kvt_synth.bf16_bits(torch.from_numpy(xh).to(torch.bfloat16))
            if not np.array_equal(oracle.bf16_array_to_f64(xh_bf), xh.astype(np.float64)):
                continue          # x_hat not representable in bf16: not a fixed point by construction
            codes2, meta2 = oracle.quantize_group(xh_bf, b)
            assert meta2 >> 16 == meta >> 16
            xh2 = np.array([oracle.dequant_value(int(c), meta2) for c in codes2])
            assert np.allclose(xh2, xh, rtol=0, atol=float(oracle.meta_scale_zero(meta2)[0]) * 0.51)


def test_o1_bf16_rounding_helpers(oracle):
    """RU/RNE against exact rational arithmetic on the bf16 grid (A3, A1)."""
    from fractions import Fraction
    rng = np.random.default_rng(5)
    for f in rng.standard_normal(2000).astype(np.float32).tolist() + [1.0, 0.5, 2.0 / 255.0, 7.5 / 15]:
        ru, rn = oracle.f32_to_bf16_ru(f), oracle.f32_to_bf16_rne(f)
        fr = Fraction(float(np.float32(f)))
        v_ru, v_rn = Fraction(oracle.bf16_to_f32(ru)), Fraction(oracle.bf16_to_f32(rn))
        assert v_ru >= fr
        # next bf16 below v_ru must be < f
        below = Fraction(oracle.bf16_to_f32(ru - 1 if v_ru > 0 else ru + 1))
        assert below < fr or v_ru == fr
        assert abs(v_rn - fr) <= abs(v_ru - fr) + abs(v_ru - below)


# ------------------------------------------------------------------------------------ packing
@pytest.mark.parametrize("bits", [2, 4, 8])
def test_pack_layout_hand_formula(oracle, bits):
    """Channel c at bits [c*b, (c+1)*b) LSB-first, against a hand formula."""
    rng = np.random.default_rng(bits)
    codes = rng.integers(0, 2 ** bits, 128).astype(np.uint8)
    row = oracle.pack_row(codes, bits)
    per = 8 // bits
    expect = np.zeros(128 * bits // 8, np.uint8)
    for i in range(expect.size):
        v = 0
        for k in range(per):
            v |= int(codes[i * per + k]) << (k * bits)
        expect[i] = v
    assert np.array_equal(row, expect)
    assert np.array_equal(oracle.unpack_row(row, 128, bits), codes)


# ------------------------------------------------------------------------------------ O2 regions
@pytest.mark.parametrize("S,nqk,nqv", [(0, 0, 0), (1, 0, 0), (31, 0, 0), (32, 32, 0), (33, 32, 1),
                                       (63, 32, 31), (64, 64, 32), (65, 64, 33), (96, 96, 64), (100, 96, 68),
                                       (8191, 8160, 8159), (8192, 8192, 8160)])
def test_o2_kivi_regions(oracle, S, nqk, nqv):
    """KIVI R = G = 32: K flushed in whole blocks n_qK = R*floor(S/R); V sliding n_qV = max(0, S-R) (A7)."""
    assert oracle.n_quantized_key(oracle.MODE_KIVI, 4, 32, 32, S) == nqk
    assert oracle.n_quantized_value(oracle.MODE_KIVI, 2, 32, 32, S) == nqv


def test_o2_per_token_regions(oracle):
    for S in (0, 1, 5, 256):
        assert oracle.n_quantized_key(oracle.MODE_PER_TOKEN, 8, 32, 0, S) == S          # R = 0 (A6)
        assert oracle.n_quantized_value(oracle.MODE_PER_TOKEN, 4, 32, 0, S) == S
        assert oracle.n_quantized_key(oracle.MODE_PER_TOKEN, 8, 32, 32, S) == max(0, S - 32)
        assert oracle.n_quantized_key(oracle.MODE_KIVI, 16, 32, 32, S) == S            # bf16 pass-through


@pytest.mark.parametrize("mode,kb,vb,G,R", [(0, 8, 4, 32, 0), (0, 2, 2, 64, 0), (0, 4, 8, 32, 32),
                                            (1, 4, 2, 32, 32), (1, 8, 8, 32, 32), (1, 2, 4, 32, 64),
                                            (1, 16, 4, 32, 32), (0, 16, 16, 32, 0)])
@pytest.mark.parametrize("S", [0, 1, 31, 32, 33, 95, 100])
def test_o2_build_dequant_bounds(oracle, mode, kb, vb, G, R, S):
    """dequant(build(X)) reconstructs every quantised group within its Eq. 2 bound, the residual
    region exactly, and per-channel KIVI key groups span G tokens of one channel (A8)."""
    d = 128
    cap = 128
    K = kvt_synth.bf16_bits(kvt_synth.keys((max(S, 1), d), seed=S + 3)[:S])
    V = kvt_synth.bf16_bits(kvt_synth.values((max(S, 1), d), seed=S + 4)[:S])
    bufs = oracle.build_cache(mode, kb, vb, G, R, d, cap, K, V)
    Kh, Vh = oracle.dequant_cache(mode, kb, vb, G, R, d, cap, S, bufs)
    Kf, Vf = oracle.bf16_array_to_f64(K), oracle.bf16_array_to_f64(V)
    nqk = oracle.n_quantized_key(mode, kb, G, R, S)
    nqv = oracle.n_quantized_value(mode, vb, G, R, S)
    # residual / pass-through rows are exact
    assert np.array_equal(Kh[nqk:], Kf[nqk:]) and np.array_equal(Vh[nqv:], Vf[nqv:])
    if kb == 16:
        assert np.array_equal(Kh, Kf)
    elif mode == oracle.MODE_KIVI:
        for b0 in range(0, nqk, G):
            blk, blkh = Kf[b0:b0 + G], Kh[b0:b0 + G]
            s = (blk.max(0) - blk.min(0)) / (2 ** kb - 1)
            assert np.all(blkh.min(0) == blk.min(0))                       # zero = per-channel min
            assert np.all(np.abs(blk - blkh) <= s * (1 + 2 ** -7) * (0.5 + 2 ** -10) + 1e-30)
    else:
        for t in range(nqk):
            for j in range(d // G):
                x, xh = Kf[t, j * G:(j + 1) * G], Kh[t, j * G:(j + 1) * G]
                s = (x.max() - x.min()) / (2 ** kb - 1)
                assert np.all(np.abs(x - xh) <= s * (1 + 2 ** -7) * (0.5 + 2 ** -10) + 1e-30)
    if vb != 16:
        for t in range(nqv):
            for j in range(d // G):
                x, xh = Vf[t, j * G:(j + 1) * G], Vh[t, j * G:(j + 1) * G]
                s = (x.max() - x.min()) / (2 ** vb - 1)
                assert np.all(np.abs(x - xh) <= s * (1 + 2 ** -7) * (0.5 + 2 ** -10) + 1e-30)


def test_o2_meta_is_16_bytes_per_token(oracle):
    """With G = 32, d = 128 the metadata costs 16 B per token per tensor in both modes; with
    quantised K and V (either mode) all four parts live in 32-token tile records inside k_codes; other
    layouts (G = 64 here) keep four separate buffers."""
    for mode in (0, 1):
        sz = oracle.slice_bytes(mode, 4, 2, 32, 32, 128, 8192)
        assert sz[0] == 8192 * (64 + 16 + 32 + 16) and sz[1] == sz[3] == sz[4] == 0
        assert sz[2] == 32 * 128 * 2 and sz[5] == 32 * 128 * 2
    sz = oracle.slice_bytes(0, 4, 2, 64, 32, 128, 8192)
    assert sz[1] == 8192 * 8 and sz[4] == 8192 * 8
    assert sz[0] == 8192 * 64 and sz[3] == 8192 * 32


@pytest.mark.parametrize("vb", [2, 4, 8])
def test_o2_blocked_value_layout_is_a_block_permutation(oracle, vb):
    """KIVI value codes (G = 32, quantised K and V) use the blocked layout inside the tile
    records — within each complete 32-token block it is a permutation of the token-major rows the
    per-token mode stores for the same (per-token, G = 32) Eq. 2 groups, and the record's V meta equals
    the per-token mode's meta rows; every byte of a complete record is defined."""
    d, S, kb = 128, 100, 4
    K = kvt_synth.bf16_bits(kvt_synth.keys((S, d), seed=vb))
    V = kvt_synth.bf16_bits(kvt_synth.values((S, d), seed=vb + 1))
    rec_bytes, mask = oracle.defined_bytes(1, kb, vb, 32, 32, d, 128, K, V)["k_codes"]
    # token-major reference: per-token mode, window 32 (same V tokens), bf16 keys (so no tile records)
    tm = oracle.defined_bytes(0, 16, vb, 32, 32, d, 128, K, V)
    rk, rv = d * kb // 8, d * vb // 8
    REC = 32 * (rk + rv) + 1024
    nqv = oracle.n_quantized_value(1, vb, 32, 32, S)                          # 68 → two complete blocks
    nqk = oracle.n_quantized_key(1, kb, 32, 32, S)                            # 96 → three K blocks
    for blk in range(nqv // 32):
        r = rec_bytes[blk * REC:(blk + 1) * REC]
        assert mask[blk * REC:(blk + 1) * REC].all()
        a = r[32 * rk + 512:32 * rk + 512 + 32 * rv]
        b = tm["v_codes"][0][blk * 32 * rv:(blk + 1) * 32 * rv]
        assert np.array_equal(np.sort(a), np.sort(b))
        assert not np.array_equal(a, b)                                       # it is not the identity
        assert np.array_equal(r[32 * rk + 512 + 32 * rv:], tm["v_meta"][0][blk * 32 * 16:(blk + 1) * 32 * 16])
    # defined bytes: K rows + K meta of the quantised key blocks, V codes + meta of the quantised values
    assert int(mask.sum()) == nqk * rk + (nqk // 32) * 512 + nqv * rv + nqv * 16

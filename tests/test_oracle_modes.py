"""Pins for the oracle's per-channel-asym sensitivity mode (A28, T-Mode) — CPU only.

The mode quantises every channel column of the whole trace as one Eq. 2 group (keys and values).
Pins: exact reconstruction of constant and already-on-grid columns (Eq. 2 with s = 0 / exact codes),
the (16, 16) identity, the round-trip bound |x - x_hat| <= s_st (1/2 + 2^-10) turned into a bound on
e_k, and the paper's direction on channel-outlier keys (per-token e_k is 2.5x the
per-channel e_k at INT8; "value cache can not benefit from switching the quantization dimension").
"""
import math

import numpy as np
import pytest
import torch

import kvt_synth

PC, PT = 2, 0


def _bf16(x):
    return kvt_synth.bf16_bits(torch.as_tensor(x, dtype=torch.float32).bfloat16())


def _qkv(H_kv, g, S, T_q, d, seed, outliers=True):
    K = kvt_synth.keys((H_kv, S, d), seed=seed, outliers=outliers)
    V = kvt_synth.values((H_kv, S, d), seed=seed + 1)
    Q = kvt_synth.queries((H_kv * g, T_q, d), seed=seed + 2)
    return kvt_synth.bf16_bits(Q), kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V)


def test_pc_constant_columns_are_exact(oracle):
    """Each channel constant over the tokens: max = min, x_hat = z exactly (A2) -> e_k = e_v = 0, and then
    e_a = e_o = 0.  Per-token quantisation of the same rows (values differ across channels) is not exact."""
    H_kv, g, S, T_q, d = 1, 2, 40, 4, 128
    rng = np.random.default_rng(0)
    col = rng.normal(size=d).astype(np.float32)
    K = _bf16(np.broadcast_to(col, (H_kv, S, d)).copy())
    V = _bf16(np.broadcast_to(rng.normal(size=d).astype(np.float32), (H_kv, S, d)).copy())
    Q = kvt_synth.bf16_bits(kvt_synth.queries((H_kv * g, T_q, d), seed=3))
    pc = oracle.sensitivity(PC, 32, 0, Q, K, V, S - T_q, [(2, 2), (4, 8)], 1 / math.sqrt(d))
    assert np.all(pc == 0.0)
    pt = oracle.sensitivity(PT, 32, 0, Q, K, V, S - T_q, [(2, 2)], 1 / math.sqrt(d))
    assert pt[0, 0] > 0 and pt[0, 1] > 0


def test_pc_on_grid_columns_are_exact(oracle):
    """Column c holds a_c + k * 2^-4 (k = 0 .. 2^b - 1 in shuffled order, a_c and the grid exact in bf16):
    s = (max - min)/(2^b - 1) = 2^-4 is a bf16 value, so every code is exact and e_k = 0 at that b."""
    H_kv, S, d, b = 1, 16, 128, 4
    rng = np.random.default_rng(1)
    K = np.zeros((H_kv, S, d), np.float32)
    for c in range(d):
        K[0, :, c] = (rng.integers(-8, 8) + rng.permutation(S)[: S] % (2 ** b)) * 2.0 ** -4
    Kb = _bf16(K)
    V = kvt_synth.bf16_bits(kvt_synth.values((H_kv, S, d), seed=4))
    Q = kvt_synth.bf16_bits(kvt_synth.queries((2, 2, d), seed=5))
    out = oracle.sensitivity(PC, 32, 0, Q, Kb, V, S - 2, [(b, 16)], 1 / math.sqrt(d))
    assert out[0, 0] == 0.0 and out[0, 1] == 0.0
    # one bit fewer cannot represent 16 levels: the error appears
    assert oracle.sensitivity(PC, 32, 0, Q, Kb, V, S - 2, [(2, 16)], 1 / math.sqrt(d))[0, 0] > 0


def test_pc_identity_pair(oracle):
    Q, K, V = _qkv(2, 2, 64, 8, 128, seed=10)
    assert np.all(oracle.sensitivity(PC, 32, 0, Q, K, V, 56, [(16, 16)], 1 / math.sqrt(128)) == 0.0)


@pytest.mark.parametrize("b", [2, 4, 8])
def test_pc_error_within_eq2_bound(oracle, b):
    """|x - x_hat| <= s_st (1/2 + 2^-10) with s_st < (max - min)/(2^b - 1) (1 + 2^-7) per channel (the O1
    pins) bounds e_k from above; e_k must also shrink as b grows."""
    H_kv, S, d = 2, 96, 128
    Q, K, V = _qkv(H_kv, 2, S, 4, d, seed=20)
    e_k = oracle.sensitivity(PC, 32, 0, Q, K, V, S - 4, [(b, 16)], 1 / math.sqrt(d))[0, 0]
    Kf = oracle.bf16_array_to_f64(K)
    rng_c = Kf.max(axis=1, keepdims=True) - Kf.min(axis=1, keepdims=True)         # [H][1][d]
    bound_el = rng_c / (2 ** b - 1) * (1 + 2 ** -7) * (0.5 + 2 ** -10)
    m = np.abs(Kf) >= 1e-8
    bound = (np.broadcast_to(bound_el, Kf.shape)[m] / np.abs(Kf)[m]).mean()
    assert 0 < e_k <= bound


def test_pc_direction_channel_outliers(oracle):
    """T-Mode direction: with channel-outlier keys (x11 on every 8th channel, the synthetic
    stand-in for P:171's key outliers), per-token e_k > per-channel e_k at 8 and 4 bits, the attention
    errors follow, and e_v hardly depends on the dimension."""
    H_kv, g, S, T_q, d = 2, 4, 256, 16, 128
    Q, K, V = _qkv(H_kv, g, S, T_q, d, seed=30)
    pairs = [(8, 8), (4, 4)]
    pc = oracle.sensitivity(PC, 32, 0, Q, K, V, S - T_q, pairs, 1 / math.sqrt(d))
    pt = oracle.sensitivity(PT, 32, 0, Q, K, V, S - T_q, pairs, 1 / math.sqrt(d))
    for i in range(len(pairs)):
        assert pt[i, 0] > 1.5 * pc[i, 0]            # e_k: per-token clearly worse (paper: 2.5x at INT8)
        assert pt[i, 2] > pc[i, 2]                  # e_a follows the key error
        assert 0.5 < pt[i, 1] / pc[i, 1] < 2.0      # e_v: "quite close" across dimensions


def test_pt_residual_rows_are_exact(oracle):
    """Per-token-asym with a full-precision residual window (A6, T-Mode P:619-647 at R > 0): the last R tokens are
    kept as they are, the others quantised row by row exactly as with R = 0.  So with R >= S every error is 0, and
    with 0 < R < S the key / value errors are the R = 0 errors of the first S - R rows diluted by S / (S - R)
    (e_k, e_v average |x - x_hat| / |x| over all elements; the residual rows contribute exact zeros)."""
    H_kv, g, S, T_q, d, R = 2, 4, 256, 24, 128, 64
    Q, K, V = _qkv(H_kv, g, S, T_q, d, seed=71)
    pairs = [(2, 2), (4, 2), (8, 4)]
    scale = 1 / math.sqrt(d)
    full = oracle.sensitivity(PT, 32, S, Q, K, V, S - T_q, pairs, scale)
    assert np.all(full == 0.0)
    with_r = oracle.sensitivity(PT, 32, R, Q, K, V, S - T_q, pairs, scale)
    head = oracle.sensitivity(PT, 32, 0, Q, np.ascontiguousarray(K[:, :S - R]), np.ascontiguousarray(V[:, :S - R]),
                              S - R - T_q, pairs, scale)
    np.testing.assert_allclose(with_r[:, 0], head[:, 0] * (S - R) / S, rtol=1e-12)     # e_k
    np.testing.assert_allclose(with_r[:, 1], head[:, 1] * (S - R) / S, rtol=1e-12)     # e_v
    assert np.all(with_r[:, 3] > 0) and np.all(with_r[:, 3] < head[:, 3] * 4)          # e_o: still quantised

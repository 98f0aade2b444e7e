"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

* K1 append: packed codes, scales/zero-points and residual bytes are bit-exact with the oracle's
  static O2 build, for one-shot prefill and for random append chunkings (history independence).
* K2/K3 decode: fp32 output within 2e-3 of the fp64 oracle, normalised per row (A17); the bf16
  output is exactly the RNE rounding of the fp32 output.
* a6: N-way sequence shards + combine equal the unsharded result.
* K5 sensitivity: equal to the oracle's fp64 metrics.
"""
import math

import numpy as np
import pytest
import torch

import kvt_synth
from tests.gpu_helpers import TOL, compare_slice, rel_row_err

pytestmark = pytest.mark.gpu

D = 128


@pytest.fixture(scope="module")
def kvt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_04420_b200 as k

    return k


SPECS = [
    ("pt_k8v4_g32", lambda k: k.LayerSpec.per_token(8, 4)),
    ("pt_k4v2_r32", lambda k: k.LayerSpec.per_token(4, 2, residual=32)),     # per-token key ring residual
    ("pt_k2v4", lambda k: k.LayerSpec.per_token(2, 4)),
    ("pt_k8v8_r64", lambda k: k.LayerSpec.per_token(8, 8, residual=64)),
    ("pt_k2v2_g64", lambda k: k.LayerSpec.per_token(2, 2, group=64)),
    ("pt_k4v8_g128_r32", lambda k: k.LayerSpec.per_token(4, 8, group=128, residual=32)),
    ("kivi_k4v2", lambda k: k.LayerSpec.kivi(4, 2)),
    ("kivi_k8v8", lambda k: k.LayerSpec.kivi(8, 8)),
    ("kivi_k2v2", lambda k: k.LayerSpec.kivi(2, 2)),
    ("kivi_k2v8", lambda k: k.LayerSpec.kivi(2, 8)),
    ("kivi_k8v2", lambda k: k.LayerSpec.kivi(8, 2)),
    ("kivi_k2v4_r64", lambda k: k.LayerSpec.kivi(2, 4, residual=64)),
    ("kivi_k4v2_r160", lambda k: k.LayerSpec.kivi(4, 2, residual=160)),   # tail > 128: two tail super-chunks
    ("kivi_k8v4_g64", lambda k: k.LayerSpec.kivi(8, 4, group=64, residual=64)),
    ("kivi_k16v4", lambda k: k.LayerSpec.kivi(16, 4)),
    ("kivi_k4v16", lambda k: k.LayerSpec.kivi(4, 16)),
    ("pt_k16v16", lambda k: k.LayerSpec.per_token(16, 16)),
]
LENS = [0, 1, 31, 32, 33, 95, 100, 257]


def _prefill(kvt, spec, K, V, lens, cap):
    B, H = K.shape[:2]
    cache = kvt.LayerCache(spec, B, H, D, cap)
    zeros = torch.zeros(B, dtype=torch.int32, device="cuda")
    n = torch.tensor(lens, dtype=torch.int32, device="cuda")
    kvt.quantize_append(cache, K, V, zeros, n, len_before_host=[0] * B, n_new_host=lens)
    return cache


@pytest.mark.parametrize("name,mk", SPECS, ids=[s[0] for s in SPECS])
def test_append_prefill_bit_exact(kvt, oracle, name, mk):
    spec = mk(kvt)
    B, H, S_max = len(LENS), 2, max(LENS)
    K = kvt_synth.keys((B, H, S_max, D), seed=101).cuda()
    V = kvt_synth.values((B, H, S_max, D), seed=102).cuda()
    cap = ((S_max + 63) // 64) * 64 + 64
    cache = _prefill(kvt, spec, K, V, LENS, cap)
    torch.cuda.synchronize()
    Kb, Vb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V)
    for b, S in enumerate(LENS):
        for h in range(H):
            compare_slice(oracle, cache, spec, b, h, Kb[b, h, :S], Vb[b, h, :S], S)


@pytest.mark.parametrize("name,mk", SPECS, ids=[s[0] for s in SPECS])
def test_append_chunking_invariance(kvt, oracle, name, mk):
    """Random prefill chunks, then decode steps of one token: same bytes as the static build (O2)."""
    spec = mk(kvt)
    B, H, S_max = 3, 2, 230
    K = kvt_synth.keys((B, H, S_max, D), seed=201).cuda()
    V = kvt_synth.values((B, H, S_max, D), seed=202).cuda()
    cache = kvt.LayerCache(spec, B, H, D, 256)
    rng = np.random.default_rng(7)
    final = [230, 171, 64]
    cur = [0, 0, 0]
    while cur != final:
        n = [int(min(f - c, rng.integers(0, 70) if rng.random() < 0.6 else 1)) for c, f in zip(cur, final)]
        T = max(max(n), 1)
        idx = torch.stack([torch.arange(c, c + T).clamp(max=S_max - 1) for c in cur]).cuda()
        kn = torch.stack([K[b, :, idx[b]] for b in range(B)])
        vn = torch.stack([V[b, :, idx[b]] for b in range(B)])
        kvt.quantize_append(cache, kn, vn, torch.tensor(cur, dtype=torch.int32, device="cuda"),
                            torch.tensor(n, dtype=torch.int32, device="cuda"), len_before_host=cur, n_new_host=n)
        cur = [c + x for c, x in zip(cur, n)]
    torch.cuda.synchronize()
    Kb, Vb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V)
    for b, S in enumerate(final):
        for h in range(H):
            compare_slice(oracle, cache, spec, b, h, Kb[b, h, :S], Vb[b, h, :S], S)


def test_append_capacity_error(kvt):
    spec = kvt.LayerSpec.kivi(4, 2)
    cache = kvt.LayerCache(spec, 1, 1, D, 64)
    K = torch.zeros(1, 1, 65, D, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(kvt.KvtError) as e:
        kvt.quantize_append(cache, K, K, torch.zeros(1, dtype=torch.int32, device="cuda"),
                            torch.tensor([65], dtype=torch.int32, device="cuda"), len_before_host=[0], n_new_host=[65])
    assert e.value.status == 5


DEC_SPECS = [s for s in SPECS]


@pytest.mark.parametrize("g", [1, 4, 7, 8])
@pytest.mark.parametrize("name,mk", DEC_SPECS, ids=[s[0] for s in DEC_SPECS])
def test_decode_parity(kvt, oracle, name, mk, g):
    spec = mk(kvt)
    lens = [0, 1, 33, 100, 257, 1000, 4133]
    B, H, S_max = len(lens), 2, max(lens)
    K = kvt_synth.keys((B, H, S_max, D), seed=301 + g).cuda()
    V = kvt_synth.values((B, H, S_max, D), seed=302 + g).cuda()
    q = kvt_synth.queries((B, H * g, D), seed=303 + g).cuda()
    cap = ((S_max + 127) // 128) * 128
    cache = _prefill(kvt, spec, K, V, lens, cap)
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    scale = 1.0 / math.sqrt(D)
    out32 = kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32)
    out16 = kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(out16, out32.to(torch.bfloat16))                 # bf16 = RNE(fp32)  (A17)
    Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q)
    o = out32.cpu().numpy()
    for b, S in enumerate(lens):
        for h in range(H):
            rows = slice(h * g, (h + 1) * g)
            if S == 0:
                assert np.all(o[b, rows] == 0)
                continue
            ref = oracle.decode_reference(spec.mode, spec.key_bits, spec.value_bits, spec.group, spec.residual, D,
                                          Kb[b, h, :S], Vb[b, h, :S], qb[b, rows], scale)
            err = rel_row_err(o[b, rows], ref)
            assert err.max() <= TOL, f"b={b} h={h} S={S}: max normalised error {err.max():.3e}"


def test_decode_without_host_lengths(kvt, oracle):
    """Planning from capacity (seq_len_host = NULL, as under CUDA-graph replay) gives the same result."""
    spec = kvt.LayerSpec.kivi(4, 2)
    lens = [500, 77]
    K = kvt_synth.keys((2, 2, 500, D), seed=1).cuda()
    V = kvt_synth.values((2, 2, 500, D), seed=2).cuda()
    q = kvt_synth.queries((2, 8, D), seed=3).cuda()
    cache = _prefill(kvt, spec, K, V, lens, 4096)
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    a = kvt.decode_attention(cache, q, sl, seq_len_host=lens)
    b = kvt.decode_attention(cache, q, sl, seq_len_host=None)
    torch.cuda.synchronize()
    # a different split plan changes only the fp32/fp16 rounding order (tile-local weight scaling)
    Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q)
    for out in (a, b):
        for bb, S in enumerate(lens):
            for h in range(2):
                ref = oracle.decode_reference(1, 4, 2, 32, 32, D, Kb[bb, h, :S], Vb[bb, h, :S], qb[bb, 4 * h:4 * h + 4],
                                              1 / math.sqrt(D))
                assert rel_row_err(out[bb, 4 * h:4 * h + 4].cpu().numpy(), ref).max() <= TOL
    assert (a - b).abs().max().item() <= 5e-4 * a.abs().max().item()


def test_decode_plan_far_above_lengths(kvt, oracle):
    """Planning from a capacity far above the actual lengths (host lengths absent): the tensor-core kernel's
    stream-K grid is sized for the capacity and clamps to the actual total work on the device."""
    spec = kvt.LayerSpec.kivi(2, 2)
    lens = [3, 40, 0, 65]
    B, H, g = len(lens), 2, 4
    K = kvt_synth.keys((B, H, 65, D), seed=11).cuda()
    V = kvt_synth.values((B, H, 65, D), seed=12).cuda()
    q = kvt_synth.queries((B, H * g, D), seed=13).cuda()
    cache = _prefill(kvt, spec, K, V, lens, 65536)
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = kvt.decode_attention(cache, q, sl, seq_len_host=None, out_dtype=torch.float32)
    torch.cuda.synchronize()
    Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q)
    o = out.cpu().numpy()
    for b, S in enumerate(lens):
        for h in range(H):
            rows = slice(h * g, (h + 1) * g)
            if S == 0:
                assert np.all(o[b, rows] == 0)
                continue
            ref = oracle.decode_reference(1, 2, 2, 32, 32, D, Kb[b, h, :S], Vb[b, h, :S], qb[b, rows], 1 / math.sqrt(D))
            assert rel_row_err(o[b, rows], ref).max() <= TOL


@pytest.mark.parametrize("n_shards", [2, 4])
def test_sequence_shards_combine(kvt, oracle, n_shards):
    """a6: shard r holds tokens [r S/N, (r+1) S/N) (non-final shards fully quantised: residual 0);
    partial (m, l, o) per shard + combine == the unsharded oracle (online-softmax identity)."""
    S, B, H, g = 2048, 2, 2, 4
    K = kvt_synth.keys((B, H, S, D), seed=41).cuda()
    V = kvt_synth.values((B, H, S, D), seed=42).cuda()
    q = kvt_synth.queries((B, H * g, D), seed=43).cuda()
    per = S // n_shards
    parts = []
    for r in range(n_shards):
        spec = kvt.LayerSpec.kivi(4, 2) if r == n_shards - 1 else kvt.LayerSpec.kivi(4, 2, residual=0)
        cache = _prefill(kvt, spec, K[:, :, r * per:(r + 1) * per].contiguous(),
                         V[:, :, r * per:(r + 1) * per].contiguous(), [per] * B, per)
        sl = torch.full((B,), per, dtype=torch.int32, device="cuda")
        parts.append(kvt.decode_attention_partial(cache, q, sl, seq_len_host=[per] * B))
    out = kvt.combine_partials(torch.stack(parts))
    full = _prefill(kvt, kvt.LayerSpec.kivi(4, 2), K, V, [S] * B, S)
    ref_gpu = kvt.decode_attention(full, q, torch.full((B,), S, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q)
    for b in range(B):
        for h in range(H):
            ref = oracle.decode_reference(1, 4, 2, 32, 32, D, Kb[b, h], Vb[b, h], qb[b, h * g:(h + 1) * g], 1 / math.sqrt(D))
            assert rel_row_err(out[b, h * g:(h + 1) * g].cpu().numpy(), ref).max() <= TOL
    # a different work partition changes only the rounding of the fp16 PV weights (A23)
    assert (out - ref_gpu).abs().max().item() <= 5e-4 * ref_gpu.abs().max().item()


@pytest.mark.parametrize("mode,R", [(0, 0), (0, 32), (0, 64), (1, 32), (1, 64), (2, 0)])
def test_sensitivity_parity(kvt, oracle, mode, R):
    H_kv, g, S, T_q = 2, 4, 256, 24
    K = kvt_synth.keys((H_kv, S, D), seed=51)
    V = kvt_synth.values((H_kv, S, D), seed=52)
    Q = kvt_synth.queries((H_kv * g, T_q, D), seed=53)
    pairs = [(kb, vb) for kb in (2, 4, 8) for vb in (2, 4, 8)] + [(16, 16)]
    scale = float(np.float32(1 / math.sqrt(D)))          # the ABI takes an fp32 softmax scale
    got = kvt.layer_sensitivity(mode, 32, R, Q.cuda(), K.cuda(), V.cuda(), S - T_q, pairs, scale=scale).cpu().numpy()
    ref = oracle.sensitivity(mode, 32, R, kvt_synth.bf16_bits(Q), kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V),
                             S - T_q, pairs, scale)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-15)
    assert np.all(got[-1] == 0)

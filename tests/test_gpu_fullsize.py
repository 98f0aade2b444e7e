"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (B = 64 sequences,
8 KV heads, 8k context, prefill through K1, then decode appends of one token; decode planned from the
capacity without host lengths): sampled (b, h) slices are checked against the oracle — packed bytes
bit-exact and the fp32 output within 2e-3 normalised (A17)."""
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


# (mode, kb, vb, H, g, B): Llama-3.1-8B shape (H = 8, g = 4) with the KIVI 3.25 map's pairs; Qwen2.5-7B shape
# (H = 4, g = 7) with the 4.00 map's pairs in the KIVI layout (A19) and in its own per-token mode, at B = 64
@pytest.mark.parametrize("mode,kb,vb,H,g,B", [(1, 4, 2, 8, 4, 64), (1, 8, 4, 8, 4, 64), (1, 2, 2, 8, 4, 64),
                                              (1, 4, 4, 8, 4, 64), (1, 8, 8, 4, 7, 64), (1, 4, 4, 4, 7, 64),
                                              (1, 8, 2, 4, 7, 64), (0, 8, 8, 4, 7, 64), (0, 8, 2, 4, 7, 64),
                                              (0, 4, 4, 4, 7, 64), (0, 4, 2, 4, 7, 64)])
def test_fullsize_sampled(kvt, oracle, mode, kb, vb, H, g, B):
    S0, n_dec = 8191, 3                      # prefill 8191 tokens, then 3 decode steps (crosses a K flush)
    spec = kvt.LayerSpec.kivi(kb, vb) if mode == 1 else kvt.LayerSpec.per_token(kb, vb)
    cap = 8192 + 64
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(1234 + kb * 10 + vb)
    K = torch.randn(B, H, S0 + n_dec, D, device=dev, generator=gen)
    K[..., ::8] *= 11.0
    K = K.to(torch.bfloat16)
    V = torch.randn(B, H, S0 + n_dec, D, device=dev, generator=gen).to(torch.bfloat16)
    q = (0.5 * torch.randn(B, H * g, D, device=dev, generator=gen)).to(torch.bfloat16)
    cache = kvt.LayerCache(spec, B, H, D, cap)
    kvt.quantize_append(cache, K[:, :, :S0], V[:, :, :S0], torch.zeros(B, dtype=torch.int32, device=dev),
                        torch.full((B,), S0, dtype=torch.int32, device=dev), n_new_max=S0)
    lb = torch.full((B,), S0, dtype=torch.int32, device=dev)
    ones = torch.ones(B, dtype=torch.int32, device=dev)
    ws = torch.zeros(max(kvt.decode_workspace_bytes(cache, H * g, None), 16), dtype=torch.uint8, device=dev)
    for i in range(n_dec):
        kvt.quantize_append(cache, K[:, :, S0 + i:S0 + i + 1], V[:, :, S0 + i:S0 + i + 1], lb, ones, n_new_max=1)
        lb += 1
        out = kvt.decode_attention(cache, q, lb, scale=1 / math.sqrt(D), out_dtype=torch.float32, workspace=ws)
    torch.cuda.synchronize()
    S = S0 + n_dec
    rng = np.random.default_rng(kb * 100 + vb)
    samples = [(0, 0), (B - 1, H - 1)] + [(int(rng.integers(B)), int(rng.integers(H))) for _ in range(2)]
    for b, h in samples:
        Kb = kvt_synth.bf16_bits(K[b, h, :S])
        Vb = kvt_synth.bf16_bits(V[b, h, :S])
        compare_slice(oracle, cache, spec, b, h, Kb, Vb, S)
        ref = oracle.decode_reference(spec.mode, kb, vb, 32, spec.residual, D, Kb, Vb,
                                      kvt_synth.bf16_bits(q[b, h * g:(h + 1) * g]), 1 / math.sqrt(D))
        err = rel_row_err(out[b, h * g:(h + 1) * g].cpu().numpy(), ref)
        assert err.max() <= TOL, f"(b={b}, h={h}): normalised error {err.max():.2e}"


@pytest.mark.parametrize("H,g", [(4, 7), (8, 4)])
def test_whole_unit_plan_ragged(kvt, oracle, H, g):
    """The whole-unit work plan (B = 64: 256 or 512 units fill most SMs twice or more) with ragged lengths:
    unit costs differ, so the equal-cost ranges cut units and the last CTA of each merges them."""
    B = 64
    lens = kvt_synth.ragged_lengths(B, 1, 1500, seed=77).tolist()
    spec = kvt.LayerSpec.kivi(4, 4)
    cap = 1536
    dev = torch.device("cuda")
    K = kvt_synth.keys((B, H, cap, D), seed=78).to(dev)
    V = kvt_synth.values((B, H, cap, D), seed=79).to(dev)
    q = kvt_synth.queries((B, H * g, D), seed=80).to(dev)
    cache = kvt.LayerCache(spec, B, H, D, cap)
    kvt.quantize_append(cache, K, V, torch.zeros(B, dtype=torch.int32, device=dev),
                        torch.tensor(lens, dtype=torch.int32, device=dev), len_before_host=[0] * B, n_new_host=lens)
    sl = torch.tensor(lens, dtype=torch.int32, device=dev)
    out = kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rng = np.random.default_rng(H)
    for b in rng.choice(B, 24, replace=False):
        h = int(rng.integers(H))
        S = lens[b]
        ref = oracle.decode_reference(spec.mode, 4, 4, 32, 32, D, kvt_synth.bf16_bits(K[b, h, :S]),
                                      kvt_synth.bf16_bits(V[b, h, :S]), kvt_synth.bf16_bits(q[b, h * g:(h + 1) * g]),
                                      1 / math.sqrt(D))
        assert rel_row_err(out[b, h * g:(h + 1) * g].cpu().numpy(), ref).max() <= TOL, (b, h, S)

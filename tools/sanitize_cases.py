"""Small-shape invocations of every kernel path for compute-sanitizer:
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py
tensor-core decode (per-SM plan, whole units, stream-K cut with the fused last-CTA merge, staged tail, paged records, per-token
keys, g = 7), the fused append -> decode launch (PDL prologue), the partial push, the generic CUDA-core kernel +
combine, K1 append (prefill and one-token), K5 sensitivity."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import kvt_synth
import paper_2502_04420_b200 as kvt

D = 128
dev = torch.device("cuda")


def cache_for(spec, B, H, lens, seed, paged=False):
    cap = ((max(lens) + 127) // 128) * 128
    K = kvt_synth.keys((B, H, cap, D), seed=seed).to(dev)
    V = kvt_synth.values((B, H, cap, D), seed=seed + 1).to(dev)
    if paged:
        pages = B * (cap // 32)
        bt = torch.randperm(pages, generator=torch.Generator().manual_seed(seed)).view(B, cap // 32).to(torch.int32).to(dev)
        c = kvt.LayerCache(spec, B, H, D, cap, device=dev, block_table=bt, num_pages=pages)
    else:
        c = kvt.LayerCache(spec, B, H, D, cap, device=dev)
    kvt.quantize_append(c, K, V, torch.zeros(B, dtype=torch.int32, device=dev),
                        torch.tensor(lens, dtype=torch.int32, device=dev), len_before_host=[0] * B, n_new_host=lens)
    return c, K, V


def run(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def decode(spec, B, H, g, lens, seed, paged=False):
    c, _, _ = cache_for(spec, B, H, lens, seed, paged)
    q = kvt_synth.queries((B, H * g, D), seed=seed + 2).to(dev)
    sl = torch.tensor(lens, dtype=torch.int32, device=dev)
    kvt.decode_attention(c, q, sl, seq_len_host=lens)


def fused():
    spec = kvt.LayerSpec.kivi(4, 2)
    B, H, g = 4, 8, 4
    lens = [300, 300, 300, 300]
    c, _, _ = cache_for(spec, B, H, lens, 31)
    q = kvt_synth.queries((B, H * g, D), seed=33).to(dev)
    kn = kvt_synth.keys((B, H, 1, D), seed=34).to(dev)
    vn = kvt_synth.values((B, H, 1, D), seed=35).to(dev)
    lb = torch.tensor(lens, dtype=torch.int32, device=dev)
    ones = torch.ones(B, dtype=torch.int32, device=dev)
    for _ in range(3):
        kvt.append_decode_attention(c, kn, vn, lb, ones, q, lb + 1)
        lb += 1


def push():
    spec = kvt.LayerSpec.kivi(4, 2)
    c, _, _ = cache_for(spec, 3, 2, [40, 700, 2000], 41)
    q = kvt_synth.queries((3, 8, D), seed=43).to(dev)
    sl = torch.tensor([40, 700, 2000], dtype=torch.int32, device=dev)
    dsts = [torch.empty(3, 8, D + 2, device=dev) for _ in range(2)]
    kvt.decode_attention_partial_push(c, q, sl, dsts, seq_len_host=[40, 700, 2000])
    kvt.combine_partials(torch.stack(dsts))


def sens():
    K = kvt_synth.keys((2, 128, D), seed=51).to(dev)
    V = kvt_synth.values((2, 128, D), seed=52).to(dev)
    Q = kvt_synth.queries((8, 16, D), seed=53).to(dev)
    for mode, R in ((0, 0), (0, 32), (1, 32), (2, 0)):
        kvt.layer_sensitivity(mode, 32, R, Q, K, V, 112, [(4, 2), (8, 8)])


if os.environ.get("KVT_SAN_ONLY") == "smplan":
    run("mma per-SM plan (B=48: 2 whole units + a piece per SM)", lambda: decode(kvt.LayerSpec.kivi(4, 2), 48, 8, 4,
        kvt_synth.ragged_lengths(48, 1, 200, seed=61).tolist(), 61))
    sys.exit(0)
run("mma per-SM plan (B=48: 2 whole units + a piece per SM)", lambda: decode(kvt.LayerSpec.kivi(4, 2), 48, 8, 4,
    kvt_synth.ragged_lengths(48, 1, 200, seed=61).tolist(), 61))
run("mma whole units (ragged, staged tail)", lambda: decode(kvt.LayerSpec.kivi(4, 2), 3, 2, 4, [100, 700, 33], 1))
run("mma stream-K cut + fused merge", lambda: decode(kvt.LayerSpec.kivi(4, 2), 2, 1, 4, [4096, 3000], 3))
run("mma paged", lambda: decode(kvt.LayerSpec.kivi(4, 4), 3, 2, 4, [100, 700, 33], 5, paged=True))
run("mma per-token keys", lambda: decode(kvt.LayerSpec.per_token(8, 4), 3, 2, 4, [100, 700, 33], 7))
run("mma g=7 (GM=8)", lambda: decode(kvt.LayerSpec.kivi(4, 4), 2, 2, 7, [500, 1100], 9))
run("generic kernel + combine (G=64)", lambda: decode(kvt.LayerSpec.per_token(4, 4, group=64), 2, 2, 4, [900, 3000], 11))
run("generic kernel (bf16 keys)", lambda: decode(kvt.LayerSpec.kivi(16, 4), 2, 2, 4, [900, 70], 13))
run("fused append -> decode (PDL)", fused)
run("partial push + combine", push)
run("K5 sensitivity", sens)

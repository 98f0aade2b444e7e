"""Measurements of the §8 rows around the decode step (not part of the bench.py step):
  a2  prefill quantise-append (bulk, T = S tokens per sequence): HBM GB/s = (bf16 K,V read + packed write) / time
  a3  decode append (n_new = 1) per layer: latency
  a7  layer sensitivity (App. B protocol size: S = 512, T_q = 256, 9 pairs) per layer: time
CUDA events on the launching stream, warm-up first.  Prints one JSON object.
    python tools/bench_aux.py [--B 64 --S 8192]"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_04420_b200 as kvt

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--H", type=int, default=8)
ap.add_argument("--S", type=int, default=8192)
a = ap.parse_args()
dev = torch.device("cuda")
D = 128
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


out = {"B": a.B, "H_kv": a.H, "S": a.S, "peak_gbs": peak, "prefill": {}, "decode_append_us": {}, "sensitivity": {}}
gen = torch.Generator(device=dev).manual_seed(3)
K = torch.randn(a.B, a.H, a.S, D, device=dev, generator=gen)
K[..., ::8] *= 11
K = K.bfloat16()
V = torch.randn(a.B, a.H, a.S, D, device=dev, generator=gen).bfloat16()
zeros = torch.zeros(a.B, dtype=torch.int32, device=dev)
nS = torch.full((a.B,), a.S, dtype=torch.int32, device=dev)
for name, spec in [("kivi K4V2", kvt.LayerSpec.kivi(4, 2)), ("kivi K2V2", kvt.LayerSpec.kivi(2, 2)),
                   ("kivi K8V8", kvt.LayerSpec.kivi(8, 8)), ("per-token K8V4", kvt.LayerSpec.per_token(8, 4))]:
    cache = kvt.LayerCache(spec, a.B, a.H, D, a.S)
    ms = timed(lambda: kvt.quantize_append(cache, K, V, zeros, nS, len_before_host=[0] * a.B, n_new_host=[a.S] * a.B,
                                           n_new_max=a.S))
    packed = sum(cache.sizes[n] for n in ("k_codes", "k_meta", "v_codes", "v_meta", "k_resid", "v_resid"))
    moved = 2 * a.B * a.H * a.S * D * 2 + packed
    out["prefill"][name] = {"ms": ms, "bytes": moved, "gbs": moved / ms / 1e6, "frac": moved / ms / 1e6 / peak}
    # decode append: one token per sequence at length S - 1 -> S (the cache is rebuilt to S - 1 first)
    cache2 = kvt.LayerCache(spec, a.B, a.H, D, a.S)
    kvt.quantize_append(cache2, K[:, :, : a.S - 1], V[:, :, : a.S - 1], zeros, torch.full_like(nS, a.S - 1),
                        len_before_host=[0] * a.B, n_new_host=[a.S - 1] * a.B, n_new_max=a.S - 1)
    k1, v1 = K[:, :, -1:].contiguous(), V[:, :, -1:].contiguous()
    lb = torch.full_like(nS, a.S - 1)
    ones = torch.ones_like(nS)
    def appends50():      # back-to-back launches so the events see GPU time, not host launch latency
        for _ in range(50):
            kvt.quantize_append(cache2, k1, v1, lb, ones, n_new_max=1)
    out["decode_append_us"][name] = 1000 * timed(appends50, reps=5) / 50   # same slot rewritten: idempotent
    del cache, cache2
del K, V
torch.cuda.empty_cache()
# a7: App. B protocol size per layer (Llama shape): 9 uniform pairs
S, T_q, Hkv, Hq = 512, 256, 8, 32
q = (0.5 * torch.randn(Hq, T_q, D, device=dev, generator=gen)).bfloat16()
k = torch.randn(Hkv, S, D, device=dev, generator=gen).bfloat16()
v = torch.randn(Hkv, S, D, device=dev, generator=gen).bfloat16()
pairs = [(8, 8), (8, 4), (8, 2), (4, 8), (4, 4), (4, 2), (2, 8), (2, 4), (2, 2)]
for mode, R in ((0, 0), (1, 32)):
    ms = timed(lambda: kvt.layer_sensitivity(mode, 32, R, q, k, v, S - T_q, pairs), reps=3, warm=1)
    out["sensitivity"]["per-token" if mode == 0 else "kivi"] = {
        "ms_per_layer": ms, "shape": f"H_q={Hq} T_q={T_q} H_kv={Hkv} S={S} pairs={len(pairs)} (fp64)"}
print(json.dumps(out))

"""Time decode attention of ONE layer (CUDA events, median of reps) for kernel A/B experiments.
    KVT_LIB=libkvt_x.so python tools/kbench.py --kb 4 --vb 2 --B 64 --S 8192 --g 4"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_04420_b200 as kvt

ap = argparse.ArgumentParser()
ap.add_argument("--kb", type=int, default=4)
ap.add_argument("--vb", type=int, default=2)
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--H", type=int, default=8)
ap.add_argument("--g", type=int, default=4)
ap.add_argument("--S", type=int, default=8192)
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--pt", action="store_true", help="per-token-asym keys (default KIVI)")
ap.add_argument("--group", type=int, default=32, help="G (64/128: the generic CUDA-core kernel)")
ap.add_argument("--no-host", action="store_true", help="no host lengths (plan for the capacity, as bench.py does)")
ap.add_argument("--cap", type=int, default=0, help="cache capacity (default: S rounded up to 64)")
ap.add_argument("--layers", type=int, default=1, help="cycle through this many caches (same data, own memory)")
ap.add_argument("--no-flush", action="store_true", help="no L2 flush between launches")
a = ap.parse_args()
dev = torch.device("cuda")
spec = (kvt.LayerSpec.per_token(a.kb, a.vb, group=a.group) if a.pt
        else kvt.LayerSpec.kivi(a.kb, a.vb, group=a.group, residual=max(32, a.group)))
cap = a.cap or ((a.S + 63) // 64) * 64
cache = kvt.LayerCache(spec, a.B, a.H, 128, cap)
gen = torch.Generator(device=dev).manual_seed(1)
K = torch.randn(a.B, a.H, a.S, 128, device=dev, generator=gen)
K[..., ::8] *= 11
K = K.bfloat16()
V = torch.randn(a.B, a.H, a.S, 128, device=dev, generator=gen).bfloat16()
kvt.quantize_append(cache, K, V, torch.zeros(a.B, dtype=torch.int32, device=dev),
                    torch.full((a.B,), a.S, dtype=torch.int32, device=dev), n_new_max=a.S)
caches = [cache]
for _ in range(a.layers - 1):
    c2 = kvt.LayerCache(spec, a.B, a.H, 128, cap)
    for n in ("k_codes", "k_meta", "v_codes", "v_meta", "k_resid", "v_resid"):
        if cache.buffers.get(n) is not None:
            c2.buffers[n].copy_(cache.buffers[n])
    caches.append(c2)
del K, V
q = (0.5 * torch.randn(a.B, a.H * a.g, 128, device=dev, generator=gen)).bfloat16()
sl = torch.full((a.B,), a.S, dtype=torch.int32, device=dev)
hl = None if a.no_host else [a.S] * a.B
ws = torch.zeros(max(kvt.decode_workspace_bytes(cache, a.H * a.g, hl), 16), dtype=torch.uint8, device=dev)
out = torch.empty(a.B, a.H * a.g, 128, dtype=torch.bfloat16, device=dev)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
ts = []
for i in range(a.reps + 3):
    cache = caches[i % len(caches)]
    if not a.no_flush:
        flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    kvt.decode_attention(cache, q, sl, seq_len_host=hl, scale=1 / math.sqrt(128), out=out, workspace=ws)
    e.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(s.elapsed_time(e))
ts.sort()
med = ts[len(ts) // 2]
nbytes = sum(cache.sizes[n] for n in ("k_codes", "k_meta", "v_codes", "v_meta")) * a.S / cap
print(f"{os.environ.get('KVT_LIB', 'libkvt.so'):22s} {'PT ' if a.pt else ''}K{a.kb}V{a.vb} G={a.group} g={a.g} B={a.B} S={a.S}: {med * 1000:8.1f} us  "
      f"{nbytes / med / 1e6:7.1f} GB/s (min {ts[0] * 1000:.1f})")

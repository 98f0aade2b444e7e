"""Per-warp timeline of the persistent decode kernel (needs a KVT_TRACE=1 build):
    KVT_LIB=libkvt_trace.so python tools/trace_pk.py --kb 4 --vb 2 [--B 64 --S 8192 --g 4 --H 8 --pt]
Prints the spread of per-warp work times (start -> own pieces done), by warp slot and tail ownership, and the
per-CTA merge phase."""
import argparse
import ctypes
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2502_04420_b200 as kvt
from paper_2502_04420_b200 import kvt as kmod

ap = argparse.ArgumentParser()
ap.add_argument("--kb", type=int, default=4)
ap.add_argument("--vb", type=int, default=2)
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--H", type=int, default=8)
ap.add_argument("--g", type=int, default=4)
ap.add_argument("--S", type=int, default=8192)
ap.add_argument("--pt", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda")
spec = kvt.LayerSpec.per_token(a.kb, a.vb) if a.pt else kvt.LayerSpec.kivi(a.kb, a.vb)
cap = ((a.S + 63) // 64) * 64
cache = kvt.LayerCache(spec, a.B, a.H, 128, cap)
gen = torch.Generator(device=dev).manual_seed(1)
K = torch.randn(a.B, a.H, a.S, 128, device=dev, generator=gen).bfloat16()
V = torch.randn(a.B, a.H, a.S, 128, device=dev, generator=gen).bfloat16()
kvt.quantize_append(cache, K, V, torch.zeros(a.B, dtype=torch.int32, device=dev),
                    torch.full((a.B,), a.S, dtype=torch.int32, device=dev), n_new_max=a.S)
del K, V
q = (0.5 * torch.randn(a.B, a.H * a.g, 128, device=dev, generator=gen)).bfloat16()
sl = torch.full((a.B,), a.S, dtype=torch.int32, device=dev)
ws = torch.zeros(max(kvt.decode_workspace_bytes(cache, a.H * a.g, [a.S] * a.B), 16), dtype=torch.uint8, device=dev)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
for _ in range(5):
    flush.zero_()
    kvt.decode_attention(cache, q, sl, seq_len_host=[a.S] * a.B, scale=1 / math.sqrt(128), workspace=ws)
torch.cuda.synchronize()
n = 8 * 8192
buf = (ctypes.c_ulonglong * n)()
assert kmod._lib.kvt_debug_trace(buf, n) == 0
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(-1, 8)
t = t[t[:, 1] > 0]
sm, warp, cta = t[:, 0] & 0xffff, (t[:, 0] >> 16) & 0xffff, t[:, 0] >> 32
t0 = t[:, 1].min()
ts = (t[:, 1:6] - t0) / 1e3          # entry, tails done, static done, work done, end
nst, ndyn = t[:, 6] & 0xffffffff, t[:, 6] >> 32
def q(x):
    return f"min {x.min():6.1f} p10 {np.percentile(x, 10):6.1f} med {np.median(x):6.1f} p90 {np.percentile(x, 90):6.1f} max {x.max():6.1f}"
print(f"warps {len(t)}  kernel span {ts[:, 4].max():.1f} us")
print("tails done   ", q(ts[:, 1]))
print("static done  ", q(ts[:, 2]))
print("work done    ", q(ts[:, 3]))
print("end          ", q(ts[:, 4]))
print("tail time    ", q(ts[:, 1] - ts[:, 0]))
print("static tiles ", q(nst.astype(float)), " dynamic tiles", q(ndyn.astype(float)))
rate = nst / np.maximum(ts[:, 2] - ts[:, 1], 1e-3)
print("static rate tiles/us", q(rate))
ctas = np.unique(cta)
cmax = np.array([ts[cta == c, 3].max() for c in ctas]); cmin = np.array([ts[cta == c, 3].min() for c in ctas])
cend = np.array([ts[cta == c, 4].max() for c in ctas])
print("per CTA work-done max", q(cmax), "\n  spread in CTA", q(cmax - cmin), "\n  merge phase", q(cend - cmax))

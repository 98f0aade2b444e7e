"""Load-balance study of the tensor-core decode kernel (needs a KVT_TRACE=1 build):
    KVT_LIB=libkvt_trace.so python tools/trace_balance.py --kb 4 --vb 2 [--B 64 --S 8192]
Prints the kernel span, per-CTA durations and per-SM busy time from %globaltimer stamps."""
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
ap.add_argument("--w", type=int, default=3, help="whole units per SM of the per-SM plan (for the item decode)")
a = ap.parse_args()
dev = torch.device("cuda")
spec = kvt.LayerSpec.kivi(a.kb, a.vb)
cache = kvt.LayerCache(spec, a.B, a.H, 128, (a.S + 63) // 64 * 64)
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
    kvt.decode_attention(cache, q, sl, scale=1 / math.sqrt(128), workspace=ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (15 * 4096))()
assert kmod._lib.kvt_debug_trace(buf, 4096) == 0
allb = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
t = allb[:3 * 4096].reshape(4096, 3)
st4 = allb[3 * 4096:11 * 4096].reshape(4096, 8)
wend = allb[11 * 4096:15 * 4096].reshape(4096, 4)
keep = t[:, 2] > 0
t, st4, wend = t[keep], st4[keep], wend[keep]
t0 = t[:, 1].min()
if (st4[:, 0] > 0).all():
    ph = lambda a_, b_: (st4[:, b_] - st4[:, a_]) / 1e3
    q = lambda x: f"min {x.min():.1f} med {np.median(x):.1f} max {x.max():.1f}"
    print("first segment phases (us): launch->seg start", q((st4[:, 0] - t0) / 1e3), "| prologue", q(ph(0, 1)),
          "| main loop (warp 0)", q(ph(1, 2)), "| epilogue", q(ph(2, 3)))
    if (st4[:, 7] > 0).all():
        print("  prologue split (us): q setup", q(ph(0, 4)), "| tail wait", q(ph(4, 5)), "| tail compute", q(ph(5, 6)),
              "| tail merge", q(ph(6, 7)), "| ring start", q(ph(7, 1)))
item = (t[:, 0] >> 16) - 1                      # per-SM plan item (-1: stream-K / idle)
sm, st, en = t[:, 0] & 0xffff, t[:, 1] - t[:, 1].min(), t[:, 2] - t[:, 1].min()
dur = en - st
print(f"CTAs {len(t)}  span {en.max() / 1e3:.1f} us   start spread {st.max() / 1e3:.1f} us")
print(f"CTA duration us: min {dur.min() / 1e3:.1f}  p10 {np.percentile(dur, 10) / 1e3:.1f}  median {np.median(dur) / 1e3:.1f}"
      f"  p90 {np.percentile(dur, 90) / 1e3:.1f}  max {dur.max() / 1e3:.1f}")
print(f"CTA end us: min {en.min() / 1e3:.1f}  p10 {np.percentile(en, 10) / 1e3:.1f}  median {np.median(en) / 1e3:.1f}  max {en.max() / 1e3:.1f}")
per = {}
for s_, e_ in zip(sm, en):
    per.setdefault(int(s_), []).append(e_)
cnt = np.array([len(v) for v in per.values()])
last = np.array([max(v) for v in per.values()])
ids = np.nonzero(keep)[0]
for a0 in range(0, len(ids), 148):
    seg = sm[(ids >= a0) & (ids < a0 + 148)]
    print(f"CTAs [{a0}, {min(a0 + 148, len(ids))}): distinct SMs {len(set(seg.tolist()))} of {len(seg)}")
print(f"SMs used {len(per)}  CTAs/SM min {cnt.min()} max {cnt.max()}  SM last-end us: min {last.min() / 1e3:.1f} median {np.median(last) / 1e3:.1f} max {last.max() / 1e3:.1f}")
order = np.argsort(np.array(list(per.keys())))
keys = np.array(list(per.keys()))[order]
print("SM last-end (us) by SM id:", " ".join(f"{int(k)}:{last[i] / 1e3:.0f}" for i, k in zip(order, keys)))

if (item >= 0).any():
    W1 = a.w + 1
    slot = np.where(item >= 0, item % W1, -1)
    for k in range(W1):
        e = en[slot == k] / 1e3
        if e.size:
            print(f"slot {k} ({'piece' if k == a.w else 'whole unit'}): CTAs {e.size}  end us min {e.min():.1f} median {np.median(e):.1f} max {e.max():.1f}")
    # per SM: spread between its first and last whole-unit CTA end
    spread = []
    for s_ in set(sm.tolist()):
        m = (sm == s_) & (slot >= 0) & (slot < a.w)
        if m.sum() > 1:
            spread.append((en[m].max() - en[m].min()) / 1e3)
    spread = np.array(spread)
    print(f"whole-unit CTAs of one SM: end spread us min {spread.min():.1f} median {np.median(spread):.1f} max {spread.max():.1f}")

if (wend > 0).all():
    sp = (wend.max(axis=1) - wend.min(axis=1)) / 1e3
    fromend = (t[:, 2] - wend.max(axis=1)) / 1e3
    print(f"per-CTA spread of its 4 warps' loop ends (us): min {sp.min():.1f} p10 {np.percentile(sp, 10):.1f} median {np.median(sp):.1f}"
          f" p90 {np.percentile(sp, 90):.1f} max {sp.max():.1f};  last warp's loop end -> CTA end: median {np.median(fromend):.1f}")

"""Debug: per-row error of the tensor-core decode vs the oracle on the parity-test shapes."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import kvt_synth, oracle
import paper_2502_04420_b200 as kvt
from tests.gpu_helpers import rel_row_err
D = 128
g = int(sys.argv[1]) if len(sys.argv) > 1 else 1
spec = kvt.LayerSpec.kivi(4, 2)
lens = [0, 1, 33, 100, 257, 1000, 4133]
B, H, S_max = len(lens), 2, max(lens)
K = kvt_synth.keys((B, H, S_max, D), seed=301 + g).cuda()
V = kvt_synth.values((B, H, S_max, D), seed=302 + g).cuda()
q = kvt_synth.queries((B, H * g, D), seed=303 + g).cuda()
cap = ((S_max + 127) // 128) * 128
cache = kvt.LayerCache(spec, B, H, D, cap)
kvt.quantize_append(cache, K, V, torch.zeros(B, dtype=torch.int32, device="cuda"), torch.tensor(lens, dtype=torch.int32, device="cuda"),
                    len_before_host=[0] * B, n_new_host=lens)
sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
o = kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32).cpu().numpy()
Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q)
oracle.build()
orc = oracle
for b, S in enumerate(lens):
    for h in range(H):
        rows = slice(h * g, (h + 1) * g)
        if S == 0:
            print(b, h, S, "zero ok" if np.all(o[b, rows] == 0) else "NONZERO"); continue
        ref = orc.decode_reference(1, 4, 2, 32, 32, D, Kb[b, h, :S], Vb[b, h, :S], qb[b, rows], 1 / math.sqrt(D))
        print(b, h, S, f"{rel_row_err(o[b, rows], ref).max():.2e}")

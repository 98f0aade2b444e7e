import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_04420_b200 as kvt
kb, vb, B, H, g = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), 8, 4
S0, n_dec, D = int(sys.argv[4]), 3, 128
dev = torch.device("cuda")
spec = kvt.LayerSpec.kivi(kb, vb)
cap = ((S0 + n_dec + 63) // 64) * 64 + 64
gen = torch.Generator(device=dev).manual_seed(1234 + kb * 10 + vb)
K = torch.randn(B, H, S0 + n_dec, D, device=dev, generator=gen); K[..., ::8] *= 11.0; K = K.bfloat16()
V = torch.randn(B, H, S0 + n_dec, D, device=dev, generator=gen).bfloat16()
q = (0.5 * torch.randn(B, H * g, D, device=dev, generator=gen)).bfloat16()
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
    bad = torch.isnan(out).any(-1)
    print(f"step {i} S={S0+i+1} nsplit={os.environ.get('KVT_NSPLIT','auto')}: nan rows {int(bad.sum())} / {bad.numel()}", 
          "first", bad.nonzero()[:4].tolist())

"""One prefill append (B=64, H=8, S=8192, KIVI K4V2) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_04420_b200 as kvt
dev = torch.device("cuda")
B, H, S, D = 64, 8, 8192, 128
spec = kvt.LayerSpec.kivi(4, 2) if (len(sys.argv) < 2 or sys.argv[1] == "kivi") else kvt.LayerSpec.per_token(8, 4)
cache = kvt.LayerCache(spec, B, H, D, S)
K = torch.randn(B, H, S, D, device=dev).bfloat16()
V = torch.randn(B, H, S, D, device=dev).bfloat16()
z = torch.zeros(B, dtype=torch.int32, device=dev)
n = torch.full((B,), S, dtype=torch.int32, device=dev)
for _ in range(2):
    kvt.quantize_append(cache, K, V, z, n, len_before_host=[0] * B, n_new_host=[S] * B, n_new_max=S)
torch.cuda.synchronize()

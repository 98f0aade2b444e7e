"""Compare the persistent (KVT_PK=1) and stream-K (KVT_PK=0) decode schedules on small shapes (debug aid)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

CASES = [
    # (name, kivi?, kb, vb, B, H, g, lens)
    ("kivi42 uniform S=64", True, 4, 2, 1, 1, 4, [64]),
    ("kivi42 uniform S=128", True, 4, 2, 1, 1, 4, [128]),
    ("kivi42 uniform S=1000", True, 4, 2, 1, 1, 4, [1000]),
    ("kivi42 S=1000 B2 H2", True, 4, 2, 2, 2, 4, [1000, 1000]),
    ("kivi42 ragged", True, 4, 2, 5, 2, 4, [1000, 257, 64, 33, 1]),
    ("pt42 S=1000", False, 4, 2, 1, 1, 4, [1000]),
    ("kivi44 g7 S=1000", True, 4, 4, 2, 2, 7, [1000, 500]),
]


def run(case):
    import paper_2502_04420_b200 as kvt
    import kvt_synth
    name, kivi, kb, vb, B, H, g, lens = case
    spec = kvt.LayerSpec.kivi(kb, vb) if kivi else kvt.LayerSpec.per_token(kb, vb)
    S = max(lens)
    K = kvt_synth.keys((B, H, S, 128), seed=5)
    V = kvt_synth.values((B, H, S, 128), seed=6)
    q = kvt_synth.queries((B, H * g, 128), seed=7)
    cap = ((S + 127) // 128) * 128
    cache = kvt.LayerCache(spec, B, H, 128, cap)
    kvt.quantize_append(cache, K.cuda(), V.cuda(), torch.zeros(B, dtype=torch.int32, device="cuda"),
                        torch.tensor(lens, dtype=torch.int32, device="cuda"), len_before_host=[0] * B, n_new_host=lens)
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = kvt.decode_attention(cache, q.cuda(), sl, seq_len_host=lens, out_dtype=torch.float32)
    torch.cuda.synchronize()
    return out.cpu()


if __name__ == "__main__":
    if len(sys.argv) > 1:
        i = int(sys.argv[1])
        torch.save(run(CASES[i]), f"/tmp/pkdbg_{os.environ.get('KVT_PK', '1')}_{i}.pt")
        sys.exit(0)
    for i, c in enumerate(CASES):
        for pk in ("0", "1"):
            subprocess.run([sys.executable, __file__, str(i)], env={**os.environ, "KVT_PK": pk}, check=False)
        a = torch.load(f"/tmp/pkdbg_0_{i}.pt")
        b = torch.load(f"/tmp/pkdbg_1_{i}.pt")
        d = (a - b).abs().amax(dim=-1)
        print(f"{c[0]:28s} max|diff| per (b, head):", [[round(float(x), 5) for x in row] for row in d], flush=True)

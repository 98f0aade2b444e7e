"""BASELINE config 4: uniform KIVI-KV8 vs the searched mixed map (Llama-3.1-8B or Qwen2.5-7B shape), context sweep 1k-32k,
batch at the HBM limit (--frac of free memory for the cache; bench.py prefills in token chunks so 90% fits), and the
mixed map again at KV8's batch (same batch, fewer bytes).
Runs bench.py per point and writes one JSON record per point to gpurun_out/sweep_ctx_<model>.jsonl.
    python tools/sweep_ctx.py [--model llama|qwen] [--ctx 1024 2048 ...]"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, nargs="*", default=[1024, 4096, 8192, 32768])
ap.add_argument("--frac", type=float, default=0.9)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--model", default="llama", choices=["llama", "qwen"])
a = ap.parse_args()
free, _ = torch.cuda.mem_get_info()
# packed bytes per token per layer-set (all 32 layers x 8 KV heads): 3.25 map 136 B, KV8 288 B per token-head
per_tok = {"llama-3.25": 136 * 8 * 32, "llama-kv8": 288 * 8 * 32,      # Llama: 32 layers x 8 KV heads
           "qwen-4.00": 160 * 4 * 28, "qwen-kv8": 288 * 4 * 28}         # Qwen: 28 layers x 4 KV heads
pair = ("llama-3.25", "llama-kv8") if a.model == "llama" else ("qwen-4.00", "qwen-kv8")
out = ROOT / "gpurun_out" / f"sweep_ctx_{a.model}.jsonl"
out.parent.mkdir(exist_ok=True)
with open(out, "w") as f:
    for ctx in a.ctx:
        kv8_batch = None
        runs = []
        for w in (pair[1], pair[0]):
            B = int(a.frac * free / (per_tok[w] * (ctx + 128)))
            B = max(8, min(B, 4096)) // 8 * 8
            if w == pair[1]:
                kv8_batch = B
            runs.append((w, B, "hbm-limit"))
        runs.append((pair[0], kv8_batch, "kv8-batch"))
        for w, B, kind in runs:
            r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--workload", w, "--batch", str(B), "--ctx", str(ctx),
                                "--steps", str(a.steps), "--warmup", "3", "--no-e2e", "--no-cpu-baseline"],
                               capture_output=True, text=True, cwd=ROOT, timeout=1800,
                               env=dict(os.environ, PYTORCH_CUDA_ALLOC_CONF="expandable_segments:True"))
            lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
            rec = {"workload": w, "ctx": ctx, "batch": B, "batch_rule": kind, "free_gb": free / 1e9}
            if lines:
                j = json.loads(lines[-1])
                rec.update(tokens_per_s=j["value"], ms_per_step=j["ms_per_step"], frac=j["roofline"]["frac"],
                           attn_gbs=j["roofline"]["achieved"], cache_gb=j.get("cache_gb_per_gpu"), clocks=j["clocks"])
            else:
                rec["error"] = r.stderr[-500:]
            print(json.dumps(rec), flush=True)
            f.write(json.dumps(rec) + "\n")

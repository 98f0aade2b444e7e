"""Calibration with error accumulation on a toy decoder (Eq. 3).

KVTuner calibrates with "dequantized KV cache for self-attention computation during the prefilling
stage, enabling error accumulation across model layers": every layer's attention reads the
quantised cache, so quantisation errors of early layers change the inputs of later ones and, through
greedy decoding, the generated tokens (token flipping).  This module runs that protocol on a small
random-weight decoder whose KV path is libkvt: each token (prompt and generated) is appended through
kvt_quantize_append and attended through kvt_decode_attention, layer by layer, with the layer's
precision pair.  The rest of the toy (projections, RMSNorm, MLP, tied embeddings) is plain torch: it is
the stand-in model around the hot path, not part of it.  RoPE is omitted (A12); the attention output
projection has gain 4 so that the generated tokens depend on the KV path (kvt_synth.ATTN_GAIN).

    arch: L = 4, d_model = 256, H_q = 4, H_kv = 2, D = 128, vocab = 256, d_ff = 512 (kvt_synth.TOY_ARCH)
    block: x += Wo · Attn(Wq h, Wk h, Wv h), h = rmsnorm(x);  x += W2 · relu(W1 rmsnorm(x))
    logits = rmsnorm(x) · W_out;  q, k, v are rounded to bf16 (the BF16 KV cache)

`agreement(specs)` = the fraction of greedy decode steps whose token equals the full-precision run's
(SPEC's toy-LLM oracle; f_a of Eq. 4 with token agreement as the accuracy).
"""
from __future__ import annotations

import math
from typing import Optional, Sequence

import torch

from . import kvt


def _rmsnorm(x: torch.Tensor) -> torch.Tensor:
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6)


class ToyLLM:
    def __init__(self, weights: dict, arch: dict, device="cuda"):
        self.a = dict(arch)
        self.dev = torch.device(device)
        self.emb = weights["emb"].to(self.dev)
        self.unemb = weights["unemb"].to(self.dev)
        self.layers = [{k: v.to(self.dev) for k, v in lw.items()} for lw in weights["layers"]]

    def run(self, prompts: torch.Tensor, specs: Sequence, n_steps: int, teacher: Optional[torch.Tensor] = None):
        """Prefill `prompts` [B][P] token by token through the quantised caches, then decode n_steps greedy
        tokens (or feed `teacher` [B][n_steps] instead of the argmax: teacher forcing).  Returns
        (generated tokens [B][n_steps], logits fp32 [B][P - 1 + n_steps][vocab] of every position >= P-1)."""
        a = self.a
        B, P = prompts.shape
        L, Hq, Hkv, D = a["L"], a["H_q"], a["H_kv"], a["D"]
        if len(specs) != L:
            raise ValueError("one layer spec per layer")
        total = P + n_steps
        cap = ((total + 63) // 64) * 64
        caches = [kvt.LayerCache(sp, B, Hkv, D, cap, device=self.dev) for sp in specs]
        ws = [torch.zeros(max(kvt.decode_workspace_bytes(c, Hq, None), 16), dtype=torch.uint8, device=self.dev)
              for c in caches]
        scale = 1.0 / math.sqrt(D)
        ones = torch.ones(B, dtype=torch.int32, device=self.dev)
        tok = prompts[:, 0].to(self.dev)
        gen, logits_all = [], []
        for t in range(total - 1):
            x = self.emb[tok]                                                   # [B][d_model] fp32
            lb = torch.full((B,), t, dtype=torch.int32, device=self.dev)
            for l, lw in enumerate(self.layers):
                h = _rmsnorm(x)
                q = (h @ lw["wq"]).view(B, Hq, D).to(torch.bfloat16)
                k = (h @ lw["wk"]).view(B, Hkv, 1, D).to(torch.bfloat16)
                v = (h @ lw["wv"]).view(B, Hkv, 1, D).to(torch.bfloat16)
                kvt.quantize_append(caches[l], k, v, lb, ones, n_new_max=1)
                o = kvt.decode_attention(caches[l], q, lb + 1, scale=scale, out_dtype=torch.float32, workspace=ws[l])
                x = x + o.view(B, Hq * D) @ lw["wo"]
                x = x + torch.relu(_rmsnorm(x) @ lw["w1"]) @ lw["w2"]
            if t + 1 < P:
                tok = prompts[:, t + 1].to(self.dev)
                continue
            logits = _rmsnorm(x) @ self.unemb
            logits_all.append(logits)
            i = t + 1 - P
            tok = logits.argmax(-1) if teacher is None else teacher[:, i].to(self.dev)
            gen.append(tok)
        return torch.stack(gen, 1).cpu(), torch.stack(logits_all, 1)


def agreement(model: ToyLLM, prompts: torch.Tensor, specs: Sequence, n_steps: int, ref_tokens=None) -> float:
    """Fraction of greedy decode steps whose token matches the full-precision (bf16 KV) run."""
    if ref_tokens is None:
        full = [kvt.LayerSpec.per_token(16, 16)] * len(specs)
        ref_tokens, _ = model.run(prompts, full, n_steps)
    toks, _ = model.run(prompts, specs, n_steps)
    return float((toks == ref_tokens).float().mean())

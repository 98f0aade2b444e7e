"""Oracle of the toy-decoder calibration — TEST INFRASTRUCTURE ONLY.

The same toy decoder as paper_2502_04420_b200/toyllm.py (architecture in kvt_synth.TOY_ARCH), written
plainly in fp64 numpy, with the KV path taken from this package: at every position t and layer, the cache
holding tokens [0, t] is built statically with O2 (identical to the streamed cache by history
independence, A7), read back exactly, and attended with O3 (Eq. 1) — i.e. "dequantized KV cache
for self-attention computation during the prefilling stage" and decoding.  q, k, v are rounded to
bf16.  Shares no code with the product; the weights come from kvt_synth (random numbers only).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import decode_reference


def _rmsnorm(x):
    return x / np.sqrt((x * x).mean(-1, keepdims=True) + 1e-6)


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def run(weights: dict, arch: dict, prompts: np.ndarray, specs, n_steps: int, teacher=None):
    """specs: per layer (mode, kb, vb, G, R).  Returns (tokens [B][n_steps], logits fp64 [B][n_steps][vocab])."""
    a = arch
    L, Hq, Hkv, D = a["L"], a["H_q"], a["H_kv"], a["D"]
    g = Hq // Hkv
    emb = weights["emb"].double().numpy()
    unemb = weights["unemb"].double().numpy()
    lws = [{k: v.double().numpy() for k, v in lw.items()} for lw in weights["layers"]]
    prompts = np.asarray(prompts)
    B, P = prompts.shape
    total = P + n_steps
    Kc = np.zeros((L, B, Hkv, total, D), np.uint16)           # bf16 bits of every appended k / v
    Vc = np.zeros((L, B, Hkv, total, D), np.uint16)
    scale = 1.0 / math.sqrt(D)
    tok = prompts[:, 0].copy()
    gen, logits_all = [], []
    for t in range(total - 1):
        x = emb[tok]
        for l in range(L):
            w = lws[l]
            h = _rmsnorm(x)
            qb = _bf16_bits(h @ w["wq"]).reshape(B, Hq, D)
            Kc[l, :, :, t] = _bf16_bits(h @ w["wk"]).reshape(B, Hkv, D)
            Vc[l, :, :, t] = _bf16_bits(h @ w["wv"]).reshape(B, Hkv, D)
            mode, kb, vb, G, R = specs[l]
            o = np.zeros((B, Hq, D))
            for b in range(B):
                for hk in range(Hkv):
                    o[b, hk * g:(hk + 1) * g] = decode_reference(mode, kb, vb, G, R, D, Kc[l, b, hk, :t + 1],
                                                                 Vc[l, b, hk, :t + 1], qb[b, hk * g:(hk + 1) * g], scale)
            x = x + o.reshape(B, Hq * D) @ w["wo"]
            x = x + np.maximum(_rmsnorm(x) @ w["w1"], 0.0) @ w["w2"]
        if t + 1 < P:
            tok = prompts[:, t + 1].copy()
            continue
        logits = _rmsnorm(x) @ unemb
        logits_all.append(logits)
        i = t + 1 - P
        tok = logits.argmax(-1) if teacher is None else np.asarray(teacher)[:, i].copy()
        gen.append(tok)
    return np.stack(gen, 1), np.stack(logits_all, 1)


def agreement(weights, arch, prompts, specs, n_steps, ref_tokens=None) -> float:
    """Fraction of greedy decode steps whose token equals the full-precision (bf16 KV) run's."""
    if ref_tokens is None:
        ref_tokens, _ = run(weights, arch, prompts, [(0, 16, 16, 32, 0)] * len(specs), n_steps)
    toks, _ = run(weights, arch, prompts, specs, n_steps)
    return float((toks == ref_tokens).mean())

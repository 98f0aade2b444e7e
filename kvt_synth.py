"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no quantisation, no attention): only random
tensors with the shapes and value distributions of the paper's workloads:

* K ~ N(0, 1) with channels c ≡ 0 (mod 8) scaled ×11 — the key channel outliers the paper
  cites ("key cache has strong channel-wise outliers"; recipe of S:62).
* V ~ N(0, 1).
* q ~ 0.5·N(0, 1) (logit std ≈ 2 at d = 128 with the outlier channels).
* Optional attention-sink heads: q aligned with k_0 on a fraction of the heads.

All generators take an explicit seed and a device; tensors are bf16 ("BF16 KV cache").
"""
from __future__ import annotations

import torch

OUTLIER_PERIOD = 8
OUTLIER_SCALE = 11.0


def generator(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def keys(shape, seed: int, device="cpu", outliers: bool = True) -> torch.Tensor:
    """bf16 keys with channel outliers on the last dim (c % 8 == 0 scaled ×11)."""
    g = generator(seed, device)
    x = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    if outliers:
        x[..., ::OUTLIER_PERIOD] *= OUTLIER_SCALE
    return x.to(torch.bfloat16)


def values(shape, seed: int, device="cpu") -> torch.Tensor:
    g = generator(seed, device)
    return torch.randn(*shape, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)


def queries(shape, seed: int, device="cpu", std: float = 0.5) -> torch.Tensor:
    g = generator(seed, device)
    return (std * torch.randn(*shape, generator=g, device=device, dtype=torch.float32)).to(torch.bfloat16)


def ragged_lengths(batch: int, lo: int, hi: int, seed: int) -> torch.Tensor:
    """int32 lengths uniform in [lo, hi] (host)."""
    g = generator(seed, "cpu")
    return torch.randint(lo, hi + 1, (batch,), generator=g, dtype=torch.int32)


def special_rows(kind: str, shape, seed: int) -> torch.Tensor:
    """Edge-case bf16 tensors (host): 'constant', 'grid' (values on a quantisation grid, ties),
    'zeros', 'tiny' (values near the bf16 subnormal range), 'wide' (|x| up to 1e4)."""
    g = generator(seed, "cpu")
    if kind == "constant":
        v = torch.randn((), generator=g).item()
        return torch.full(shape, v, dtype=torch.float32).to(torch.bfloat16)
    if kind == "zeros":
        return torch.zeros(shape, dtype=torch.bfloat16)
    if kind == "grid":
        base = torch.randint(0, 16, shape, generator=g).to(torch.float32)
        return (0.25 * base - 1.0).to(torch.bfloat16)
    if kind == "tiny":
        return (1e-30 * torch.randn(*shape, generator=g)).to(torch.bfloat16)
    if kind == "wide":
        return (1e4 * torch.randn(*shape, generator=g)).to(torch.bfloat16)
    raise ValueError(kind)


EDGE_KINDS = ("constant", "zeros_pm", "range1e-3", "range1e-4", "range1e-5", "range1e-6", "normal", "ties_b2",
              "ties_b4", "ties_b8")


def edge_structured(shape, seed: int, along: str) -> torch.Tensor:
    """bf16 [..., S, d] whose quantisation groups cycle through EDGE_KINDS:
    constant groups, all-zero groups with random signs (+0 / -0), groups of range 1e-3 .. 1e-6 around small
    offsets (so bf16 keeps them), ordinary N(0, 1) groups, and groups on a grid whose Eq. 2 codes hit exact
    .5 ties at 2, 4 and 8 bits (s = 1, 0.5, 2^-4 exactly; both ends of the range present).
    along = "channel": the kind is constant over a 32-token block x 1 channel (KIVI key groups);
    along = "token": constant over 1 token x 32 channels (per-token groups).  Kind of (position p, group c)
    = EDGE_KINDS[(p + c) % 10], so constant/zero groups sit next to tiny-range groups in every tile."""
    g = generator(seed, "cpu")
    *lead, S, d = shape
    n = 1
    for x in lead:
        n *= x
    out = torch.empty(n, S, d, dtype=torch.float32)
    tok = torch.arange(S)
    ch = torch.arange(d)
    if along == "channel":
        pos, grp = (tok // 32)[:, None].expand(S, d), ch[None, :].expand(S, d)
    elif along == "token":
        pos, grp = tok[:, None].expand(S, d), (ch // 32)[None, :].expand(S, d)
    else:
        raise ValueError(along)
    kind = (pos + grp) % len(EDGE_KINDS)
    # one random draw per group (offset) and per element
    gid = pos * d + grp
    for i in range(n):
        u = torch.rand(S, d, generator=g)
        z = torch.randn(S, d, generator=g)
        off = torch.randn(S * d + d, generator=g)[gid]
        x = torch.empty(S, d)
        x = torch.where(kind == 0, 4 * off, x)
        x = torch.where(kind == 1, torch.where(u < 0.5, torch.tensor(0.0), torch.tensor(-0.0)), x)
        for k, r in ((2, 1e-3), (3, 1e-4), (4, 1e-5), (5, 1e-6)):
            x = torch.where(kind == k, r * (off + u), x)
        x = torch.where(kind == 6, z, x)
        # ties: values on half steps of s with the group's min (0) and max present so s is exact
        i7 = torch.randint(0, 7, (S, d), generator=g).float()
        t7 = 0.5 * i7
        i8 = torch.randint(0, 31, (S, d), generator=g).float()
        t8 = 0.25 * i8
        i9 = torch.randint(0, 128, (S, d), generator=g).float()
        t9 = (i9 + 0.5) / 16.0
        x = torch.where(kind == 7, t7, x)
        x = torch.where(kind == 8, t8, x)
        x = torch.where(kind == 9, t9, x)
        # first / second element of every group carry the range ends (0 and max) for the tie kinds
        first = (tok % 32 == 0)[:, None] if along == "channel" else (ch % 32 == 0)[None, :]
        second = (tok % 32 == 1)[:, None] if along == "channel" else (ch % 32 == 1)[None, :]
        for k, mx in ((7, 3.0), (8, 7.5), (9, 255.0 / 16.0)):
            x = torch.where((kind == k) & first, torch.tensor(0.0), x)
            x = torch.where((kind == k) & second, torch.tensor(mx), x)
        out[i] = x
    return out.view(*lead, S, d).to(torch.bfloat16)


def edge_queries(shape, seed: int) -> torch.Tensor:
    """bf16 q [..., H_q, d] with a 2^±20 dynamic range: head h scaled by 2^e_h, e_h cycling through
    {-20, -10, 0, 4}, channel c scaled by 2^((c % 21) - 10)."""
    g = generator(seed, "cpu")
    q = torch.randn(*shape, generator=g)
    H, d = shape[-2], shape[-1]
    eh = torch.tensor([-20.0, -10.0, 0.0, 4.0])[torch.arange(H) % 4]
    ec = (torch.arange(d) % 21).float() - 10.0
    return (q * torch.exp2(eh)[:, None] * torch.exp2(ec)[None, :]).to(torch.bfloat16)


def bf16_bits(t: torch.Tensor):
    """Raw bf16 bits of a (CPU or CUDA) bf16 tensor as a numpy uint16 array (host)."""
    import numpy as np

    assert t.dtype == torch.bfloat16
    return t.detach().contiguous().cpu().view(torch.int16).numpy().view(np.uint16)


# ---- toy LLM (calibration with error accumulation): random weights and prompts only ----
TOY_ARCH = {"L": 4, "d_model": 256, "H_q": 4, "H_kv": 2, "D": 128, "vocab": 256, "d_ff": 512}
ATTN_GAIN = 4.0          # attention output gain: the residual stream is attention-dominated (tokens depend on the KV)


def toy_weights(seed: int, arch=None):
    """fp32 CPU weights of the toy decoder (N(0, 1/fan_in)); the key projection's output channels
    c = 0 (mod 8) of every head are scaled x11, the key-outlier recipe above."""
    a = dict(TOY_ARCH if arch is None else arch)
    g = generator(seed, "cpu")
    dm, D = a["d_model"], a["D"]

    def w(n_in, n_out):
        return torch.randn(n_in, n_out, generator=g) / n_in ** 0.5

    out = {"emb": torch.randn(a["vocab"], dm, generator=g), "layers": []}
    for _ in range(a["L"]):
        wk = w(dm, a["H_kv"] * D)
        wk.view(dm, a["H_kv"], D)[..., ::OUTLIER_PERIOD] *= OUTLIER_SCALE
        out["layers"].append({"wq": w(dm, a["H_q"] * D), "wk": wk, "wv": w(dm, a["H_kv"] * D),
                              "wo": ATTN_GAIN * w(a["H_q"] * D, dm), "w1": w(dm, a["d_ff"]), "w2": w(a["d_ff"], dm)})
    out["unemb"] = w(dm, a["vocab"])
    return out


def toy_prompts(seed: int, batch: int, length: int, vocab: int = TOY_ARCH["vocab"]) -> torch.Tensor:
    """int64 [batch][length] token ids."""
    return torch.randint(0, vocab, (batch, length), generator=generator(seed, "cpu"))

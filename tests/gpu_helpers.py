"""Shared helpers of the -m gpu parity tests: valid-region comparison of cache buffers against the
oracle's static build, and the A17 output tolerance."""
import numpy as np
import torch

import kvt_synth

TOL = 2e-3          # north_star: within 2e-3 max-abs-relative error (A17: normalised per row, fp32 output)


def regions(oracle, spec, S, d=128):
    """Valid byte ranges (per (b,h) slice) of each buffer for a length-S sequence."""
    mode, kb, vb, G, R = spec.mode, spec.key_bits, spec.value_bits, spec.group, spec.residual
    nqk = oracle.n_quantized_key(mode, kb, G, R, S)
    nqv = oracle.n_quantized_value(mode, vb, G, R, S)
    rk = 2 * d if kb == 16 else d * kb // 8
    rv = 2 * d if vb == 16 else d * vb // 8
    out = {"k_codes": [(0, nqk * rk)], "v_codes": [(0, nqv * rv)]}
    if kb != 16:
        if mode == oracle.MODE_KIVI:
            out["k_meta"] = [(0, (nqk // G) * d * 4)]
            out["k_resid"] = [(0, (S - nqk) * d * 2)]
        else:
            out["k_meta"] = [(0, nqk * (d // G) * 4)]
            out["k_resid"] = [((t % R) * d * 2, (t % R + 1) * d * 2) for t in range(nqk, S)]
    if vb != 16:
        out["v_meta"] = [(0, nqv * (d // G) * 4)]
        out["v_resid"] = [((t % R) * d * 2, (t % R + 1) * d * 2) for t in range(nqv, S)]
    return out


def compare_slice(oracle, cache, spec, b, h, K_bits, V_bits, S, d=128):
    """Bit-exact comparison of one (b,h) slice of the GPU cache with the oracle's static build, on
    every byte the layout defines for this history."""
    ref = oracle.defined_bytes(spec.mode, spec.key_bits, spec.value_bits, spec.group, spec.residual, d,
                               cache.capacity, K_bits, V_bits)
    for name, (exp, mask) in ref.items():
        if cache.buffers[name] is None or not mask.any():
            continue
        gpu = (paged_records(cache, b, h) if name == "k_codes" and getattr(cache, "block_table", None) is not None
               else cache.slice_view(name, b, h)).cpu().numpy().view(np.uint8)
        bad = np.nonzero((gpu != exp) & mask)[0]
        if bad.size:
            raise AssertionError(f"{name} (b={b}, h={h}, S={S}) differs at bytes {bad[:8]} "
                                 f"gpu={gpu[bad[:8]]} oracle={exp[bad[:8]]} ({bad.size} bytes)")
    # the defined region is what §4 says it is: all code rows of quantised tokens, nothing else
    nqv = oracle.n_quantized_value(spec.mode, spec.value_bits, spec.group, spec.residual, S)
    rv = 2 * d if spec.value_bits == 16 else d * spec.value_bits // 8
    if cache.buffers["v_codes"] is None:        # tile records: every part of the quantised tokens in k_codes
        nqk = oracle.n_quantized_key(spec.mode, spec.key_bits, spec.group, spec.residual, S)
        rk = d * spec.key_bits // 8
        kmeta = (nqk // 32) * d * 4 if spec.mode == oracle.MODE_KIVI else nqk * (d // spec.group) * 4
        assert int(ref["k_codes"][1].sum()) == nqk * rk + kmeta + nqv * rv + nqv * 16
    else:
        assert int(ref["v_codes"][1].sum()) == nqv * rv


def paged_records(cache, b, h):
    """The tile records of (b, h) of a paged cache, gathered through its block table into the dense
    order (record j = block j), i.e. the bytes a dense cache would hold."""
    H, max_pages = cache.kv_heads, cache.block_table.shape[1]
    rec = cache.sizes["k_codes"] // (cache.num_pages * H)
    pool = cache.buffers["k_codes"][: cache.num_pages * H * rec].view(cache.num_pages, H, rec)
    return pool[cache.block_table[b].long(), h].reshape(max_pages * rec)


def rel_row_err(out, ref):
    """max_c |o - o_ref| / max_c |o_ref| per row (A17); rows with o_ref == 0 use absolute error."""
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max(-1, keepdims=True)
    den = np.where(den > 0, den, 1.0)
    return (np.abs(out - ref) / den).max(-1)


def bf16_rne(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16)


def inputs(B, H, S_max, d, seed, device="cuda"):
    K = kvt_synth.keys((B, H, S_max, d), seed=seed, device="cpu").to(device)
    V = kvt_synth.values((B, H, S_max, d), seed=seed + 1, device="cpu").to(device)
    return K, V

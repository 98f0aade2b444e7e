"""Paged tile records (vLLM-style block table; P:85, P:708 name vLLM as a deployment
target): the same bytes as the dense layout, only placed in pages chosen by the caller.

* append: after random chunked prefill + one-token decode steps, every (b, h) slice gathered through the
  block table equals the oracle's static build byte for byte (O2), and pages outside the table are
  never written;
* decode: the paged launch returns bitwise the dense launch's output (same work partition, same
  arithmetic) and stays within the A17 tolerance of the oracle.
"""
import math

import numpy as np
import pytest
import torch

import kvt_synth
from tests.gpu_helpers import TOL, compare_slice, rel_row_err

pytestmark = pytest.mark.gpu
D = 128


@pytest.fixture(scope="module")
def kvt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_04420_b200 as k

    return k


SPECS = [
    ("kivi_k4v2", lambda k: k.LayerSpec.kivi(4, 2)),
    ("kivi_k8v4", lambda k: k.LayerSpec.kivi(8, 4)),
    ("kivi_k2v2_r64", lambda k: k.LayerSpec.kivi(2, 2, residual=64)),
    ("pt_k8v4", lambda k: k.LayerSpec.per_token(8, 4)),
    ("pt_k4v2_r32", lambda k: k.LayerSpec.per_token(4, 2, residual=32)),
]


def _tables(B, max_pages, extra, seed):
    """A shuffled page assignment: distinct pages for every (b, j), plus `extra` never-used pages."""
    num_pages = B * max_pages + extra
    perm = torch.randperm(num_pages, generator=torch.Generator().manual_seed(seed))
    return perm[: B * max_pages].view(B, max_pages).to(torch.int32).cuda(), num_pages, perm[B * max_pages:]


def _fill(kvt, caches, K, V, final, seed):
    """Identical random chunked appends (prefill chunks, then single tokens) into every cache."""
    B = K.shape[0]
    rng = np.random.default_rng(seed)
    cur = [0] * B
    while cur != final:
        n = [int(min(f - c, rng.integers(0, 90) if rng.random() < 0.6 else 1)) for c, f in zip(cur, final)]
        T = max(max(n), 1)
        idx = torch.stack([torch.arange(c, c + T).clamp(max=K.shape[2] - 1) for c in cur]).cuda()
        kn = torch.stack([K[b, :, idx[b]] for b in range(B)])
        vn = torch.stack([V[b, :, idx[b]] for b in range(B)])
        for cache in caches:
            kvt.quantize_append(cache, kn, vn, torch.tensor(cur, dtype=torch.int32, device="cuda"),
                                torch.tensor(n, dtype=torch.int32, device="cuda"), len_before_host=cur, n_new_host=n)
        cur = [c + x for c, x in zip(cur, n)]


@pytest.mark.parametrize("name,mk", SPECS, ids=[s[0] for s in SPECS])
def test_paged_append_and_decode(kvt, oracle, name, mk):
    spec = mk(kvt)
    B, H, g, max_pages = 3, 2, 4, 12
    cap = 32 * max_pages
    final = [cap - 5, 161, 64]
    K = kvt_synth.keys((B, H, cap, D), seed=301).cuda()
    V = kvt_synth.values((B, H, cap, D), seed=302).cuda()
    bt, num_pages, unused = _tables(B, max_pages, extra=7, seed=3)
    paged = kvt.LayerCache(spec, B, H, D, cap, block_table=bt, num_pages=num_pages)
    paged.buffers["k_codes"].fill_(0xAB)
    dense = kvt.LayerCache(spec, B, H, D, cap)
    _fill(kvt, [paged, dense], K, V, final, seed=11)
    torch.cuda.synchronize()
    Kb, Vb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V)
    for b, S in enumerate(final):
        for h in range(H):
            compare_slice(oracle, paged, spec, b, h, Kb[b, h, :S], Vb[b, h, :S], S)
    # pages outside the table are untouched
    page = paged.sizes["k_codes"] // num_pages
    pool = paged.buffers["k_codes"][: num_pages * page].view(num_pages, page)
    assert bool((pool[unused.cuda().long()] == 0xAB).all())
    # decode: bitwise the dense output, within A17 of the oracle
    q = kvt_synth.queries((B, H * g, D), seed=303).cuda()
    sl = torch.tensor(final, dtype=torch.int32, device="cuda")
    scale = 1 / math.sqrt(D)
    out_p = kvt.decode_attention(paged, q, sl, seq_len_host=final, scale=scale)
    out_d = kvt.decode_attention(dense, q, sl, seq_len_host=final, scale=scale)
    torch.cuda.synchronize()
    assert torch.equal(out_p, out_d)
    qb = kvt_synth.bf16_bits(q)
    for b, S in enumerate(final):
        for h in range(H):
            ref = oracle.decode_reference(spec.mode, spec.key_bits, spec.value_bits, spec.group, spec.residual, D,
                                          Kb[b, h, :S], Vb[b, h, :S], qb[b, h * g:(h + 1) * g], scale)
            assert rel_row_err(out_p[b, h * g:(h + 1) * g].cpu().numpy(), ref).max() <= TOL


def test_paged_validation(kvt):
    bt = torch.zeros(2, 4, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):          # capacity != 32 * max_pages
        kvt.LayerCache(kvt.LayerSpec.kivi(4, 2), 2, 2, D, 96, block_table=bt, num_pages=8)
    with pytest.raises(kvt.KvtError):        # no tile records (bf16 keys)
        kvt.LayerCache(kvt.LayerSpec.kivi(16, 4), 2, 2, D, 128, block_table=bt, num_pages=8)

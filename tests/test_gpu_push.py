"""a6 with the exchange fused into the attention kernel: the partial (m, l, o) rows
are pushed straight into up to 8 destination buffers (in a multi-GPU run: this shard's slot of every
peer's symmetric-memory buffer over NVLink).  On one GPU: the pushed rows equal the plain partial bit for
bit in every destination, for the tensor-core kernel (fused in-kernel merge) and the generic kernel
(separate combine launch); and the symmetric-memory exchange on a one-rank NCCL group reproduces the
unsharded decode."""
import socket

import pytest
import torch

import kvt_synth
from tests.gpu_helpers import rel_row_err

pytestmark = pytest.mark.gpu
D = 128


@pytest.fixture(scope="module")
def kvt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_04420_b200 as k

    return k


def _cache(kvt, spec, B, H, lens, seed):
    cap = ((max(lens) + 63) // 64) * 64
    K = kvt_synth.keys((B, H, cap, D), seed=seed).cuda()
    V = kvt_synth.values((B, H, cap, D), seed=seed + 1).cuda()
    cache = kvt.LayerCache(spec, B, H, D, cap)
    kvt.quantize_append(cache, K, V, torch.zeros(B, dtype=torch.int32, device="cuda"),
                        torch.tensor(lens, dtype=torch.int32, device="cuda"), len_before_host=[0] * B, n_new_host=lens)
    return cache


@pytest.mark.parametrize("mk", [lambda k: k.LayerSpec.kivi(4, 2), lambda k: k.LayerSpec.per_token(8, 4),
                                lambda k: k.LayerSpec.kivi(16, 4), lambda k: k.LayerSpec.per_token(4, 4, group=64)],
                         ids=["kivi_k4v2_mma", "pt_k8v4_mma", "kivi_k16v4_generic", "pt_k4v4_g64_generic"])
def test_push_equals_partial(kvt, mk):
    spec = mk(kvt)
    B, H, g = 6, 2, 4
    lens = [1, 33, 700, 1025, 64, 2049]
    cache = _cache(kvt, spec, B, H, lens, seed=501)
    q = kvt_synth.queries((B, H * g, D), seed=503).cuda()
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    ref = kvt.decode_attention_partial(cache, q, sl, seq_len_host=lens)
    dsts = [torch.full((B, H * g, D + 2), float("nan"), device="cuda") for _ in range(3)]
    kvt.decode_attention_partial_push(cache, q, sl, dsts, seq_len_host=lens)
    torch.cuda.synchronize()
    for d in dsts:
        assert torch.equal(d, ref)


def test_push_validation(kvt):
    cache = _cache(kvt, kvt.LayerSpec.kivi(4, 2), 1, 1, [40], seed=7)
    q = torch.zeros(1, 4, D, dtype=torch.bfloat16, device="cuda")
    sl = torch.tensor([40], dtype=torch.int32, device="cuda")
    with pytest.raises(kvt.KvtError):
        kvt.decode_attention_partial_push(cache, q, sl, [])
    with pytest.raises(kvt.KvtError):
        kvt.decode_attention_partial_push(cache, q, sl, [torch.empty(1, 4, D + 2, device="cuda")] * 9)


def test_symmetric_memory_exchange_one_rank(kvt):
    import torch.distributed as dist

    from paper_2502_04420_b200.seqshard import SymmExchange

    if dist.is_initialized():
        pytest.skip("a process group already exists")
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        B, H, g = 4, 2, 4
        lens = [500, 96, 1300, 31]
        cache = _cache(kvt, kvt.LayerSpec.kivi(4, 2), B, H, lens, seed=601)
        sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
        try:
            ex = SymmExchange((B, H * g, D + 2), torch.device("cuda", 0))
        except Exception as e:            # symmetric memory unavailable in this build / driver
            pytest.skip(f"symmetric memory unavailable: {e}")
        for layer in range(3):            # both buffers of the double buffer, then the first again
            q = kvt_synth.queries((B, H * g, D), seed=700 + layer).cuda()
            out = ex.decode(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32)
            ref = kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32)
            torch.cuda.synchronize()
            assert rel_row_err(out.cpu().numpy(), ref.cpu().numpy()).max() <= 1e-6
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_shards", [2, 4])
def test_virtual_shards_push_against_oracle(kvt, oracle, n_shards):
    """a6 + NEXT #2 on one GPU with N virtual ranks: shard r = tokens [r S/N, (r+1) S/N) of every
    sequence (seqshard.shard_bounds / shard_spec: residual on the last shard only) pushes its (m, l, o) rows into slot r
    of two "peer" buffers [N][B][H_q][D+2] (what kvt_decode_attention_partial_push writes over NVLink in a real run);
    each peer's kvt_combine_partials must equal the unsharded fp64 oracle (Eq. 1 over the whole cache), and the two
    peers must agree bit for bit."""
    import math

    import numpy as np

    from paper_2502_04420_b200.seqshard import shard_bounds, shard_spec
    from tests.gpu_helpers import TOL

    B, H, g, S = 2, 2, 4, 1500
    base = kvt.LayerSpec.kivi(4, 2)
    K = kvt_synth.keys((B, H, S, D), seed=811)
    V = kvt_synth.values((B, H, S, D), seed=812)
    q = kvt_synth.queries((B, H * g, D), seed=813)
    peers = [torch.full((n_shards, B, H * g, D + 2), float("nan"), device="cuda") for _ in range(2)]
    for r in range(n_shards):
        lo, hi = shard_bounds(S, n_shards, r)
        spec = shard_spec(base, r, n_shards)
        n = hi - lo
        cache = _cache_from(kvt, spec, K[:, :, lo:hi].contiguous(), V[:, :, lo:hi].contiguous(), n)
        sl = torch.full((B,), n, dtype=torch.int32, device="cuda")
        kvt.decode_attention_partial_push(cache, q.cuda(), sl, [p[r] for p in peers], seq_len_host=[n] * B)
    outs = [kvt.combine_partials(p, out_dtype=torch.float32) for p in peers]
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q)
    o = outs[0].cpu().numpy()
    for b in range(B):
        for h in range(H):
            ref = oracle.decode_reference(1, 4, 2, 32, 32, D, Kb[b, h], Vb[b, h], qb[b, h * g:(h + 1) * g],
                                          1 / math.sqrt(D))
            assert rel_row_err(o[b, h * g:(h + 1) * g], ref).max() <= TOL


def _cache_from(kvt, spec, K, V, n):
    B, H = K.shape[:2]
    cap = ((n + 63) // 64) * 64
    cache = kvt.LayerCache(spec, B, H, D, cap)
    kvt.quantize_append(cache, K.cuda(), V.cuda(), torch.zeros(B, dtype=torch.int32, device="cuda"),
                        torch.full((B,), n, dtype=torch.int32, device="cuda"), len_before_host=[0] * B,
                        n_new_host=[n] * B)
    return cache

"""a6 host logic on CPU: world-size-2 gloo process group running the sequence-shard orchestration
(shard bounds, per-rank specs, all-gather layout and order, log-sum-exp combine) with the oracle
standing in for the partial kernel.  The GPU path of the same orchestration is covered by
tests/test_gpu_parity.py::test_sequence_shards_combine."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

D = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_partial(spec, Kb, Vb, qb, scale):
    """(m, l, o) of DESIGN.md §1/a6 from the oracle's fp64 probabilities on this shard (log2 units)."""
    import oracle

    S = Kb.shape[0]
    cap = max(((S + 31) // 32) * 32, 32)
    bufs = oracle.build_cache(spec.mode, spec.key_bits, spec.value_bits, spec.group, spec.residual, D, cap, Kb, Vb)
    Kh, Vh = oracle.dequant_cache(spec.mode, spec.key_bits, spec.value_bits, spec.group, spec.residual, D, cap, S, bufs)
    q = oracle.bf16_array_to_f64(qb)
    s2 = (q @ Kh.T) * scale * math.log2(math.e)           # [g][S]
    m = s2.max(1)
    w = np.exp2(s2 - m[:, None])
    l = w.sum(1)
    o = (w @ Vh) / l[:, None]
    return np.concatenate([m[:, None], l[:, None], o], 1)


def _combine(gathered):
    g = gathered.double()
    m, l, o = g[..., 0], g[..., 1], g[..., 2:]
    M = m.max(0).values
    wgt = l * torch.exp2(m - M)
    return (wgt[..., None] * o).sum(0) / wgt.sum(0)[..., None]


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import kvt_synth
    from paper_2502_04420_b200 import LayerSpec
    from paper_2502_04420_b200.seqshard import shard_bounds, shard_spec, sharded_decode

    S, H, g = 1000, 2, 4
    K = kvt_synth.bf16_bits(kvt_synth.keys((H, S, D), seed=61))
    V = kvt_synth.bf16_bits(kvt_synth.values((H, S, D), seed=62))
    q = kvt_synth.bf16_bits(kvt_synth.queries((H * g, D), seed=63))
    base = LayerSpec.kivi(4, 2)
    lo, hi = shard_bounds(S, world, rank)
    spec = shard_spec(base, rank, world)
    scale = 1 / math.sqrt(D)

    def partial_fn(_cache, _q, _sl):
        rows = [_oracle_partial(spec, K[h, lo:hi], V[h, lo:hi], q[h * g:(h + 1) * g], scale) for h in range(H)]
        return torch.from_numpy(np.concatenate(rows, 0)[None]).float()          # [B=1][H_q][d+2]

    out = sharded_decode(None, None, None, partial_fn=partial_fn, combine_fn=_combine)
    ret[rank] = (lo, hi, spec.residual, out.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sequence_shard_orchestration_gloo(oracle, world):
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    import kvt_synth

    S, H, g = 1000, 2, 4
    K = kvt_synth.bf16_bits(kvt_synth.keys((H, S, D), seed=61))
    V = kvt_synth.bf16_bits(kvt_synth.values((H, S, D), seed=62))
    q = kvt_synth.bf16_bits(kvt_synth.queries((H * g, D), seed=63))
    ref = np.concatenate([oracle.decode_reference(1, 4, 2, 32, 32, D, K[h], V[h], q[h * g:(h + 1) * g], 1 / math.sqrt(D))
                          for h in range(H)], 0)
    bounds = sorted((v[0], v[1]) for v in ret.values())
    assert bounds == [(0, 480), (480, 1000)]                        # aligned to 32, remainder on the last rank
    assert ret[0][2] == 0 and ret[1][2] == 32                       # only the last shard keeps a residual
    for r in range(world):
        np.testing.assert_allclose(ret[r][3][0], ref, rtol=1e-5, atol=1e-6)   # partials travel as fp32

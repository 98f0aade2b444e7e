"""§8(e) batch x KV-head partition on CPU process groups: world-size 2 and 4 gloo groups, each
rank computing decode attention for the (b, kv head) units `partition.partition` gives it (the oracle stands in for
the GPU kernel, as in test_seqshard_gloo.py), the outputs all-gathered and reassembled.  Checks: every unit has
exactly one owner, the reassembled output equals the unpartitioned oracle (the partition needs no collective on the
data path: each unit reads only its own cache, P:988 / A10), and bench.py's plan counts a step's tokens once."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

D = 128
CASES = [(5, 2), (1, 8), (3, 4), (8, 2)]          # (B, H_kv): batch rows, head split (B < N), ragged
G_Q, S_LEN = 4, 96


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(B, H):
    import kvt_synth

    K = kvt_synth.bf16_bits(kvt_synth.keys((B, H, S_LEN, D), seed=901 + B + H))
    V = kvt_synth.bf16_bits(kvt_synth.values((B, H, S_LEN, D), seed=902 + B + H))
    q = kvt_synth.bf16_bits(kvt_synth.queries((B, H * G_Q, D), seed=903 + B + H))
    return K, V, q


def _unit_out(oracle, K, V, q, b, h):
    return oracle.decode_reference(1, 4, 2, 32, 32, D, K[b, h], V[b, h], q[b, h * G_Q:(h + 1) * G_Q], 1 / math.sqrt(D))


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2502_04420_b200.partition import partition

    oracle.build()
    res = {}
    for B, H in CASES:
        if B * H < world:
            continue
        K, V, q = _inputs(B, H)
        p = partition(B, H, world, rank)
        mine = {(b, h): _unit_out(oracle, K, V, q, b, h) for (b, h) in p.units()}
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        res[(B, H)] = gathered
    ret[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_batch_head_partition_gloo(oracle, world):
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    for B, H in CASES:
        if B * H < world:
            continue
        K, V, q = _inputs(B, H)
        gathered = ret[0][(B, H)]
        owners = {}
        for r, part in enumerate(gathered):
            for u in part:
                assert u not in owners, f"unit {u} owned by ranks {owners[u]} and {r}"
                owners[u] = r
        assert sorted(owners) == [(b, h) for b in range(B) for h in range(H)]
        for (b, h), r in owners.items():
            np.testing.assert_array_equal(gathered[r][(b, h)], _unit_out(oracle, K, V, q, b, h))
        # every rank saw the same gathered result
        for r in range(1, world):
            assert sorted(ret[r][(B, H)][0]) == sorted(gathered[0])


def test_partition_host_rules():
    """partition(): batch rows when B >= N (ragged floor split), KV-head ranges of one sequence when B < N,
    an error when B * H < N; bench.plan(): weak scaling counts N * B tokens per step, strong scaling and sequence
    sharding count the global B once."""
    import argparse

    from paper_2502_04420_b200.partition import partition

    parts = [partition(10, 8, 4, r) for r in range(4)]
    assert [(p.b_lo, p.b_hi) for p in parts] == [(0, 2), (2, 5), (5, 7), (7, 10)]
    assert all((p.h_lo, p.h_hi) == (0, 8) for p in parts)
    parts = [partition(2, 8, 8, r) for r in range(8)]
    assert [(p.b_lo, p.h_lo, p.h_hi) for p in parts] == [(0, 0, 2), (0, 2, 4), (0, 4, 6), (0, 6, 8),
                                                          (1, 0, 2), (1, 2, 4), (1, 4, 6), (1, 6, 8)]
    with pytest.raises(ValueError):
        partition(1, 4, 8, 0)
    import bench

    for world in (1, 2, 8):
        a = argparse.Namespace(workload="llama-3.25", batch=64, scaling="weak")
        assert bench.plan(a, world, 0)[2] == world * 64
        a = argparse.Namespace(workload="llama-3.25", batch=64, scaling="strong")
        assert bench.plan(a, world, 0)[2] == 64
        assert sum(bench.plan(a, world, r)[0] * (bench.plan(a, world, r)[1][1] - bench.plan(a, world, r)[1][0])
                   for r in range(world)) == 64 * 8
        a = argparse.Namespace(workload="llama-128k-seqshard", batch=8, scaling="weak", exchange="nccl")
        assert bench.plan(a, world, 0)[2] == 8

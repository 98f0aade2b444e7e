"""CUDA-graph replay of the decode loop (the launch-bound inner loop of serving is captured once and
replayed): one captured step = append one token (K1) + decode attention (K2) + advance the
device lengths.  The kernels read every length on the device, so replaying the same graph with growing
caches must give exactly the eager results, step by step, and stay within A17 of the oracle."""
import math

import pytest
import torch

import kvt_synth
from tests.gpu_helpers import TOL, rel_row_err

pytestmark = pytest.mark.gpu
D = 128


@pytest.fixture(scope="module")
def kvt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_04420_b200 as k

    return k


@pytest.mark.parametrize("mk,g", [(lambda k: k.LayerSpec.kivi(4, 2), 4), (lambda k: k.LayerSpec.per_token(8, 4), 7)])
def test_graph_replay_matches_eager(kvt, oracle, mk, g):
    spec = mk(kvt)
    B, H, S0, steps, cap = 5, 2, 90, 40, 192
    K = kvt_synth.keys((B, H, S0 + steps, D), seed=401).cuda()
    V = kvt_synth.values((B, H, S0 + steps, D), seed=402).cuda()
    q = kvt_synth.queries((steps, B, H * g, D), seed=403).cuda()
    scale = 1 / math.sqrt(D)
    caches, outs = [], []
    for mode in ("eager", "graph"):
        cache = kvt.LayerCache(spec, B, H, D, cap)
        kvt.quantize_append(cache, K[:, :, :S0].contiguous(), V[:, :, :S0].contiguous(),
                            torch.zeros(B, dtype=torch.int32, device="cuda"),
                            torch.full((B,), S0, dtype=torch.int32, device="cuda"))
        caches.append(cache)
        outs.append(torch.empty(steps, B, H * g, D, dtype=torch.float32, device="cuda"))
    # planned for the capacity (no host lengths): valid for every replay
    ws = [torch.zeros(max(kvt.decode_workspace_bytes(c, H * g, None), 16), dtype=torch.uint8, device="cuda")
          for c in caches]
    ones = torch.ones(B, dtype=torch.int32, device="cuda")

    def step_fn(cache, w, lb, la, kn, vn, qs, out):
        kvt.quantize_append(cache, kn, vn, lb, ones, n_new_max=1)
        kvt.decode_attention(cache, qs, la, scale=scale, out=out, workspace=w)
        lb.add_(1)
        la.add_(1)

    # eager
    lb = torch.full((B,), S0, dtype=torch.int32, device="cuda")
    la = lb + 1
    for i in range(steps):
        step_fn(caches[0], ws[0], lb, la, K[:, :, S0 + i:S0 + i + 1].contiguous(), V[:, :, S0 + i:S0 + i + 1].contiguous(),
                q[i], outs[0][i])
    # graph: static input buffers refilled before each replay
    lb2 = torch.full((B,), S0, dtype=torch.int32, device="cuda")
    la2 = lb2 + 1
    kn = torch.empty(B, H, 1, D, dtype=torch.bfloat16, device="cuda")
    vn = torch.empty_like(kn)
    qs = torch.empty(B, H * g, D, dtype=torch.bfloat16, device="cuda")
    ob = torch.empty(B, H * g, D, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            step_fn(caches[1], ws[1], lb2, la2, kn, vn, qs, ob)
    torch.cuda.current_stream().wait_stream(s)
    # capture does not execute: the lengths are untouched
    assert int(lb2[0]) == S0
    for i in range(steps):
        kn.copy_(K[:, :, S0 + i:S0 + i + 1])
        vn.copy_(V[:, :, S0 + i:S0 + i + 1])
        qs.copy_(q[i])
        graph.replay()
        outs[1][i].copy_(ob)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    # the last step against the oracle
    S = S0 + steps
    Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q[-1])
    for b in range(B):
        for h in range(H):
            ref = oracle.decode_reference(spec.mode, spec.key_bits, spec.value_bits, spec.group, spec.residual, D,
                                          Kb[b, h, :S], Vb[b, h, :S], qb[b, h * g:(h + 1) * g], scale)
            assert rel_row_err(outs[1][-1, b, h * g:(h + 1) * g].cpu().numpy(), ref).max() <= TOL

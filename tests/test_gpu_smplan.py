"""The per-SM work plan of the tensor-core decode kernel (kvt_decode_mma.cuh, `sm_claim`): where
whole units would leave ceil(U / SMs) units on some SMs and floor(U / SMs) on others, slots 0 .. w-1 of every SM
take whole units and slot w one stream-K piece of the remaining units.  Checked against the oracle on every
(b, h) unit (ragged lengths, so pieces cut units at arbitrary tiles and tails), bitwise reproducibility (the
partition does not depend on which CTA lands where), the unclaimed-item path the last CTA runs when the
placement is not the expected one (forced in a subprocess with KVT_SMPLAN_DROP), and a workspace shared with
layers that run the stream-K plan (the schedule counters are left at zero)."""
import math
import os
import subprocess
import sys

import pytest
import torch

import kvt_synth
from tests.gpu_helpers import TOL, rel_row_err

pytestmark = pytest.mark.gpu
D = 128
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kvt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_04420_b200 as k

    return k


def _case(kvt, spec, B, H, g, max_len, seed):
    lens = kvt_synth.ragged_lengths(B, 1, max_len, seed=seed).tolist()
    cap = ((max_len + 63) // 64) * 64
    dev = torch.device("cuda")
    K = kvt_synth.keys((B, H, cap, D), seed=seed + 1).to(dev)
    V = kvt_synth.values((B, H, cap, D), seed=seed + 2).to(dev)
    q = kvt_synth.queries((B, H * g, D), seed=seed + 3).to(dev)
    cache = kvt.LayerCache(spec, B, H, D, cap)
    kvt.quantize_append(cache, K, V, torch.zeros(B, dtype=torch.int32, device=dev),
                        torch.tensor(lens, dtype=torch.int32, device=dev), len_before_host=[0] * B, n_new_host=lens)
    return lens, K, V, q, cache


def _check_all(oracle, spec, lens, K, V, q, out, H, g):
    Kb, Vb, qb = kvt_synth.bf16_bits(K), kvt_synth.bf16_bits(V), kvt_synth.bf16_bits(q)
    o = out.cpu().numpy()
    worst = 0.0
    for b, S in enumerate(lens):
        for h in range(H):
            ref = oracle.decode_reference(spec.mode, spec.key_bits, spec.value_bits, 32, spec.residual, D,
                                          Kb[b, h, :S], Vb[b, h, :S], qb[b, h * g:(h + 1) * g], 1 / math.sqrt(D))
            worst = max(worst, rel_row_err(o[b, h * g:(h + 1) * g], ref).max())
    assert worst <= TOL, f"normalised error {worst:.2e}"


# (B, H, g): Llama shape at B = 48 (384 units: 2 whole per SM + a piece) and B = 64 (512: 3 + a piece); Qwen shape at
# B = 64 (256 units: w = 1, so the whole-unit plan runs — the plan is not used there)
@pytest.mark.parametrize("B,H,g", [(48, 8, 4), (64, 8, 4), (64, 4, 7)])
@pytest.mark.parametrize("mk", [lambda k: k.LayerSpec.kivi(4, 2), lambda k: k.LayerSpec.per_token(4, 4)])
def test_sm_plan_every_unit(kvt, oracle, B, H, g, mk):
    spec = mk(kvt)
    lens, K, V, q, cache = _case(kvt, spec, B, H, g, 420, seed=1000 + B + g)
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32)
    again = kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(out, again)                       # placement-independent partition: bitwise reproducible
    _check_all(oracle, spec, lens, K, V, q, out, H, g)


_DROP_SCRIPT = r"""
import math, sys, torch
sys.path.insert(0, {root!r})
import kvt_synth, paper_2502_04420_b200 as kvt
B, H, g = {B}, {H}, {g}
lens = kvt_synth.ragged_lengths(B, 1, 300, seed=7).tolist()
K = kvt_synth.keys((B, H, 320, 128), seed=8).cuda()
V = kvt_synth.values((B, H, 320, 128), seed=9).cuda()
q = kvt_synth.queries((B, H * g, 128), seed=10).cuda()
spec = kvt.LayerSpec.kivi(4, 2)
cache = kvt.LayerCache(spec, B, H, 128, 320)
kvt.quantize_append(cache, K, V, torch.zeros(B, dtype=torch.int32, device="cuda"),
                    torch.tensor(lens, dtype=torch.int32, device="cuda"), len_before_host=[0] * B, n_new_host=lens)
sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
nb = kvt.decode_workspace_bytes(cache, H * g, lens)
ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
outs = [kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32, workspace=ws) for _ in range(2)]
torch.cuda.synchronize()
n_ctr = (4 * B * H + 255) // 256 * 64                    # merge counters, then the schedule counters (int32 words)
n_sched = (4 * (514 + B * H + torch.cuda.get_device_properties(0).multi_processor_count) + 255) // 256 * 64
ctr_nonzero = int((ws.view(torch.int32)[:n_ctr + n_sched] != 0).sum().item())
torch.save({{"out": outs[0].cpu(), "again": outs[1].cpu(), "lens": lens, "ctr_nonzero": ctr_nonzero}}, sys.argv[1])
"""


@pytest.mark.parametrize("drop", [1, 3])
def test_sm_plan_unclaimed_items(kvt, oracle, tmp_path, drop):
    """KVT_SMPLAN_DROP = k: CTAs with blockIdx % k == 0 give up their item, so the last CTA to finish must find
    and run every unclaimed one (k = 1: all of them, one after the other) before it resets the counters."""
    B, H, g = 64, 8, 4
    path = str(tmp_path / "out.pt")
    env = dict(os.environ, KVT_SMPLAN_DROP=str(drop))
    script = _DROP_SCRIPT.format(root=ROOT, B=B, H=H, g=g)
    r = subprocess.run([sys.executable, "-c", script, path], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = torch.load(path)
    assert torch.equal(res["out"], res["again"])
    assert res["ctr_nonzero"] == 0                      # merge and schedule counters back at zero
    lens = res["lens"]
    K = kvt_synth.keys((B, H, 320, D), seed=8)
    V = kvt_synth.values((B, H, 320, D), seed=9)
    q = kvt_synth.queries((B, H * g, D), seed=10)
    _check_all(oracle, kvt.LayerSpec.kivi(4, 2), lens, K, V, q, res["out"], H, g)


def test_sm_plan_workspace_shared_with_stream_k(kvt, oracle):
    """A K4V2 layer (per-SM plan at B = 64) and a K8V4 layer (3 CTAs/SM: whole units / stream-K) alternate on one
    workspace: outputs equal runs on fresh workspaces bitwise and every counter word ends at zero."""
    B, H, g = 64, 8, 4
    specs = [kvt.LayerSpec.kivi(4, 2), kvt.LayerSpec.kivi(8, 4)]
    cases = [_case(kvt, s, B, H, g, 300, seed=1200) for s in specs]
    nb = max(kvt.decode_workspace_bytes(c[4], H * g, c[0]) for c in cases)
    shared = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    outs, fresh = [], []
    for rep in range(2):
        for lens, K, V, q, cache in cases:
            sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
            outs.append(kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32, workspace=shared))
            fresh.append(kvt.decode_attention(cache, q, sl, seq_len_host=lens, out_dtype=torch.float32,
                                              workspace=torch.zeros(nb, dtype=torch.uint8, device="cuda")))
    torch.cuda.synchronize()
    for a, b in zip(outs, fresh):
        assert torch.equal(a, b)
    words = shared.view(torch.int32)
    n_ctr = (4 * B * H + 255) // 256 * 64                  # merge counters, then the schedule counters
    n_sched = (4 * (514 + B * H + torch.cuda.get_device_properties(0).multi_processor_count) + 255) // 256 * 64
    assert words[:n_ctr + n_sched].abs().sum().item() == 0
    lens, K, V, q, _ = cases[0]
    _check_all(oracle, specs[0], lens, K, V, q, outs[0], H, g)


def test_decode_plan_reports_the_launch(kvt):
    """kvt_decode_plan: the Llama shape at B = 64 (512 units) runs the per-SM plan with 3 whole units per SM and one
    full wave of CTAs; the Qwen shape (256 units, w = 1) and a small batch do not."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    c = kvt.LayerCache(kvt.LayerSpec.kivi(4, 2), 64, 8, D, 256)
    p = kvt.decode_plan(c, 32)
    assert p["kernel"] == "tensor-core"
    if 512 // sms >= 2 and 512 % sms and 512 // sms + 1 <= p["ctas_per_sm"]:
        assert p["sm_whole_units"] == 512 // sms and p["ctas"] == p["ctas_per_sm"] * sms
    q = kvt.decode_plan(kvt.LayerCache(kvt.LayerSpec.kivi(4, 4), 64, 4, D, 256), 28)
    assert q["sm_whole_units"] == 0
    small = kvt.decode_plan(kvt.LayerCache(kvt.LayerSpec.kivi(4, 2), 2, 2, D, 256), 8)
    assert small["sm_whole_units"] == 0 and small["ctas"] >= 1
    g = kvt.decode_plan(kvt.LayerCache(kvt.LayerSpec.per_token(4, 4, group=64), 2, 2, D, 256), 8)
    assert g["kernel"] == "generic"

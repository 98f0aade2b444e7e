"""Calibration with error accumulation on a toy decoder (Eq. 3).

Oracle pins (CPU, `oracle/toyllm.py`): full precision agrees with itself exactly and deterministically;
the paper's directions on token agreement — KV8 above KV2 (T-GSM8K's KV8-vs-KV2 degradation) and K4V2
above K2V4 ("the key cache plays a more critical role than the value cache") — and error
accumulation across layers (quantising every layer perturbs the logits more than quantising the last
layer alone, Eq. 3 / P:328).
GPU: the libkvt toy decoder reproduces the oracle's teacher-forced logits and the same directions.
"""
import numpy as np
import pytest
import torch

import kvt_synth

ARCH = kvt_synth.TOY_ARCH
FULL = (0, 16, 16, 32, 0)
KIVI = {"KV8": (1, 8, 8, 32, 32), "KV4": (1, 4, 4, 32, 32), "K4V2": (1, 4, 2, 32, 32), "K2V4": (1, 2, 4, 32, 32),
        "KV2": (1, 2, 2, 32, 32)}
B, P, N = 4, 16, 24
SEEDS = (0, 1, 2)


@pytest.fixture(scope="module")
def otoy(oracle):
    from oracle import toyllm

    return toyllm


def test_oracle_full_precision_identity(otoy):
    w = kvt_synth.toy_weights(5)
    pr = kvt_synth.toy_prompts(5, 2, 8).numpy()
    t1, l1 = otoy.run(w, ARCH, pr, [FULL] * ARCH["L"], 6)
    t2, l2 = otoy.run(w, ARCH, pr, [FULL] * ARCH["L"], 6)
    assert np.array_equal(t1, t2) and np.array_equal(l1, l2)
    assert otoy.agreement(w, ARCH, pr, [FULL] * ARCH["L"], 6, ref_tokens=t1) == 1.0


def test_oracle_directions(otoy):
    acc = {k: [] for k in ("KV8", "K4V2", "K2V4", "KV2")}
    for seed in SEEDS:
        w = kvt_synth.toy_weights(seed)
        pr = kvt_synth.toy_prompts(seed, B, P).numpy()
        ref, _ = otoy.run(w, ARCH, pr, [FULL] * ARCH["L"], N)
        for k in acc:
            acc[k].append(otoy.agreement(w, ARCH, pr, [KIVI[k]] * ARCH["L"], N, ref_tokens=ref))
    m = {k: float(np.mean(v)) for k, v in acc.items()}
    assert m["KV8"] > m["KV2"]
    assert m["K4V2"] > m["K2V4"]
    assert m["KV8"] >= 0.9


def test_oracle_error_accumulates_over_layers(otoy):
    """Teacher-forced (same tokens): KV4 in every layer moves the logits more than KV4 in the last layer only."""
    errs_all, errs_last = [], []
    for seed in SEEDS:
        w = kvt_synth.toy_weights(seed)
        pr = kvt_synth.toy_prompts(seed, B, P).numpy()
        ref, lref = otoy.run(w, ARCH, pr, [FULL] * ARCH["L"], N)
        _, lall = otoy.run(w, ARCH, pr, [KIVI["KV4"]] * ARCH["L"], N, teacher=ref)
        _, llast = otoy.run(w, ARCH, pr, [FULL] * (ARCH["L"] - 1) + [KIVI["KV4"]], N, teacher=ref)
        errs_all.append(np.abs(lall - lref).mean())
        errs_last.append(np.abs(llast - lref).mean())
    assert np.mean(errs_all) > 1.5 * np.mean(errs_last)


@pytest.mark.gpu
def test_gpu_toy_matches_oracle(otoy):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_04420_b200 as kvt
    from paper_2502_04420_b200.toyllm import ToyLLM

    def specs_of(t):
        return [kvt.LayerSpec(*t)] * ARCH["L"]

    for seed in SEEDS[:2]:
        w = kvt_synth.toy_weights(seed)
        pr = kvt_synth.toy_prompts(seed, B, P)
        model = ToyLLM(w, ARCH)
        for name in ("KV4", "K4V2"):
            otok, olog = otoy.run(w, ARCH, pr.numpy(), [KIVI[name]] * ARCH["L"], N)
            _, glog = model.run(pr, specs_of(KIVI[name]), N, teacher=torch.from_numpy(otok))
            glog = glog.double().cpu().numpy()
            # the projections run in fp32 on the GPU and fp64 in the oracle, so the bf16 rounding of q/k/v can
            # differ by one ulp at ties and move a quantisation code or group range; that shows up on a few
            # steps (amplified by the later layers) while the bulk stays at the kernels' own error (A29)
            err = np.abs(glog - olog).max(-1) / np.abs(olog).max(-1)
            assert np.median(err) <= 2e-3 and err.max() <= 5e-2, (seed, name, np.median(err), err.max())


@pytest.mark.gpu
def test_gpu_toy_directions():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_04420_b200 as kvt
    from paper_2502_04420_b200.toyllm import ToyLLM, agreement

    acc = {k: [] for k in ("KV8", "K4V2", "K2V4", "KV2")}
    for seed in range(6):
        w = kvt_synth.toy_weights(seed)
        pr = kvt_synth.toy_prompts(seed, 8, P)
        model = ToyLLM(w, ARCH)
        ref, _ = model.run(pr, [kvt.LayerSpec.per_token(16, 16)] * ARCH["L"], 32)
        assert agreement(model, pr, [kvt.LayerSpec.per_token(16, 16)] * ARCH["L"], 32, ref_tokens=ref) == 1.0
        for k in acc:
            acc[k].append(agreement(model, pr, [kvt.LayerSpec(*KIVI[k])] * ARCH["L"], 32, ref_tokens=ref))
    m = {k: float(np.mean(v)) for k, v in acc.items()}
    assert m["KV8"] > m["KV2"] and m["K4V2"] > m["K2V4"], m

"""Search-space pruning after calibration (App. D).

* oracle pins (`oracle/search.py` against what the paper and the mathematics fix): the paper's
  key-first Pareto set, an independent skyline sweep on random tables, scikit-learn's DBSCAN,
  the paper's search-space sizes ("3.4 x 10^30", "5^6 = 15625") and the layer-0 split of
  T-Intra;
* parity: libkvt.so's host entry points (kvt_pareto_prune, kvt_dbscan, kvt_prune_and_cluster,
  kvt_search_space_log10) against the oracle — exact (integer / boolean results);
* end to end on the GPU: K5 sensitivity profiles of synthetic layers -> prune -> cluster equals the
  oracle's sensitivity -> oracle's prune/cluster.
"""
import math
import random

import numpy as np
import pytest

from oracle import search as osearch

PAIRS9 = [(kb, vb) for kb in (8, 4, 2) for vb in (8, 4, 2)]
NAMES = {(8, 8): "KV8", (8, 4): "K8V4", (8, 2): "K8V2", (4, 8): "K4V8", (4, 4): "KV4", (4, 2): "K4V2",
         (2, 8): "K2V8", (2, 4): "K2V4", (2, 2): "KV2"}


def monotone_profile(rng, key_weight=3.0):
    """e_o strictly decreasing in bits, keys more sensitive than values (P:229 'key cache is more
    important'): e = key_weight * 2^-b_k + 2^-b_v (+ tiny jitter that keeps the order)."""
    return [key_weight * 2.0 ** -kb + 2.0 ** -vb + 1e-6 * rng.random() for kb, vb in PAIRS9]


def skyline(pairs, e):
    """Independent Pareto filter: sort by (bits, e) and sweep (a different algorithm from the oracle's
    all-pairs dominance test)."""
    idx = sorted(range(len(pairs)), key=lambda i: (osearch.pair_bits(pairs[i]), e[i]))
    keep = [False] * len(pairs)
    best_e_lower_bits = math.inf       # min e over strictly smaller bits
    i = 0
    while i < len(idx):
        j = i
        b = osearch.pair_bits(pairs[idx[i]])
        while j < len(idx) and osearch.pair_bits(pairs[idx[j]]) == b:
            j += 1
        grp = idx[i:j]
        emin = min(e[k] for k in grp)
        for k in grp:   # kept iff minimal inside its bits class and strictly below every cheaper pair
            keep[k] = e[k] == emin and e[k] < best_e_lower_bits
        best_e_lower_bits = min(best_e_lower_bits, emin)
        i = j
    return keep


# ---------------------------------------------------------------------------------------------------
# oracle pins
# ---------------------------------------------------------------------------------------------------
def test_oracle_key_first_set():
    """'The Pareto optimal KV cache precision pairs in most layers are the key-first set
    {KV8, K8V4, KV4, K4V2, KV2}' — what a profile with key-dominated errors must produce."""
    rng = random.Random(1)
    for _ in range(20):
        keep = osearch.pareto_prune(PAIRS9, monotone_profile(rng))
        assert {NAMES[p] for p, k in zip(PAIRS9, keep) if k} == {"KV8", "K8V4", "KV4", "K4V2", "KV2"}


def test_oracle_value_first_when_values_dominate():
    """Mirror image (under KIVI some layers prefer K4V8 / K2V4 over K8V4 / K4V2)."""
    e = [2.0 ** -kb + 3.0 * 2.0 ** -vb for kb, vb in PAIRS9]
    keep = osearch.pareto_prune(PAIRS9, e)
    assert {NAMES[p] for p, k in zip(PAIRS9, keep) if k} == {"KV8", "K4V8", "KV4", "K2V4", "KV2"}


def test_oracle_pareto_matches_skyline_sweep():
    rng = random.Random(7)
    for t in range(300):
        n = rng.randint(1, 9)
        pairs = [PAIRS9[rng.randrange(9)] for _ in range(n)]
        # coarse values so that exact ties (equal bits and/or equal e) occur often
        e = [rng.choice([0.01, 0.02, 0.03, 0.05, 0.08]) if t % 2 else rng.random() for _ in range(n)]
        assert osearch.pareto_prune(pairs, e) == skyline(pairs, e), (pairs, e)


def test_oracle_pareto_special_cases():
    assert osearch.pareto_prune([(4, 2)], [0.3]) == [True]                       # single pair
    assert osearch.pareto_prune([(8, 8), (8, 8)], [0.1, 0.1]) == [True, True]    # exact ties both survive
    # the frontier is never empty and the minimum-e pair always survives
    rng = random.Random(3)
    for _ in range(50):
        e = [rng.random() for _ in PAIRS9]
        keep = osearch.pareto_prune(PAIRS9, e)
        assert keep[int(np.argmin(e))] and keep.count(True) >= 1
        assert keep[[osearch.pair_bits(p) for p in PAIRS9].index(2.0)] or min(
            e[i] for i, p in enumerate(PAIRS9) if osearch.pair_bits(p) == 2.0) > min(e)


def _blobs(rng, n_blobs, per, dim, spread, sep):
    pts = []
    for bi in range(n_blobs):
        c = [sep * bi + rng.random() * 0.01 for _ in range(dim)]
        for _ in range(per):
            pts.append([x + rng.gauss(0, spread) for x in c])
    rng.shuffle(pts)
    return pts


def test_oracle_dbscan_matches_sklearn():
    sk = pytest.importorskip("sklearn.cluster")
    rng = random.Random(11)
    for t in range(40):
        dim = rng.randint(1, 6)
        pts = _blobs(rng, rng.randint(1, 4), rng.randint(1, 8), dim, 0.02, 0.3)
        pts += [[rng.random() * 2 for _ in range(dim)] for _ in range(rng.randint(0, 4))]   # noise
        eps, ms = rng.choice([0.03, 0.05, 0.08]), rng.choice([1, 2, 3])
        ref = sk.DBSCAN(eps=eps, min_samples=ms).fit(np.array(pts)).labels_.tolist()
        assert osearch.dbscan(pts, eps, ms) == ref


def test_oracle_dbscan_special_cases():
    assert osearch.dbscan([[0.2, 0.1]] * 5) == [0] * 5                 # identical points -> one cluster
    assert osearch.dbscan([[0.0], [1.0]]) == [-1, -1]                  # two far points, min_samples 2 -> noise
    assert osearch.dbscan([[0.0], [0.01], [1.0], [1.01]]) == [0, 0, 1, 1]
    assert osearch.dbscan([[0.5]]) == [-1]                             # single point: below min_samples
    assert osearch.dbscan([]) == []


def test_oracle_search_space_sizes():
    """9^32 'about 3.4 x 10^30'; 5^G = 5^6 = 15625; 5^32 'about 2.3 x 10^22'."""
    assert osearch.search_space_size([9] * 32) == 9 ** 32
    assert f"{float(9 ** 32):.1e}" == "3.4e+30"
    assert osearch.search_space_size([5] * 6) == 15625
    assert f"{float(osearch.search_space_size([5] * 32)):.1e}" == "2.3e+22"
    assert osearch.search_space_size([1]) == 1


def test_oracle_layer0_isolated():
    """T-Intra, Llama per-token row: layer 0 keeps {KV8, K4V8, KV4, K4V2, KV2} while the other layers keep
    the key-first set; layer 0 must end up in a partition (and so a group) of its own."""
    rng = random.Random(5)
    e = [monotone_profile(rng) for _ in range(8)]
    # layer 0: K4V8 better than K8V4 (equal bits 6), everything else key-first
    e[0][PAIRS9.index((4, 8))] = e[0][PAIRS9.index((8, 4))] * 0.5
    keep, grp, G = osearch.prune_and_cluster(PAIRS9, e)
    assert keep[0][PAIRS9.index((4, 8))] and not keep[0][PAIRS9.index((8, 4))]
    assert grp[0] == 0 and all(g != 0 for g in grp[1:])
    # the other 7 layers have near-identical errors (jitter 1e-6 << eps) -> one group
    assert len(set(grp[1:])) == 1 and G == 2


def test_oracle_clustering_separates_sensitivity_classes():
    """highly sensitive and insensitive layers with the same candidate set land in different
    groups (their e_o vectors differ by >> eps), while layers inside a class merge."""
    rng = random.Random(9)
    e = []
    for l in range(12):
        k = 1.0 if l % 3 else 3.0          # every third layer 3x more sensitive
        e.append([k * v for v in monotone_profile(rng)])
    keep, grp, G = osearch.prune_and_cluster(PAIRS9, e)
    assert G == 2
    assert len({grp[l] for l in range(0, 12, 3)}) == 1
    assert grp[0] != grp[1]


# ---------------------------------------------------------------------------------------------------
# parity: libkvt.so host entry points vs the oracle (exact)
# ---------------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def kvt():
    import paper_2502_04420_b200 as k

    return k


def test_lib_pareto_parity(kvt):
    rng = random.Random(21)
    for t in range(300):
        n = rng.randint(1, 9)
        pairs = [PAIRS9[rng.randrange(9)] for _ in range(n)]
        e = [rng.choice([0.01, 0.02, 0.05]) if t % 2 else rng.random() for _ in range(n)]
        assert kvt.pareto_prune(pairs, e) == osearch.pareto_prune(pairs, e)


def test_lib_dbscan_parity(kvt):
    rng = random.Random(22)
    for t in range(60):
        dim = rng.randint(1, 6)
        pts = _blobs(rng, rng.randint(1, 4), rng.randint(1, 8), dim, 0.02, 0.3)
        pts += [[rng.random() * 2 for _ in range(dim)] for _ in range(rng.randint(0, 4))]
        eps, ms = rng.choice([0.03, 0.05, 0.08]), rng.choice([1, 2, 3])
        assert kvt.dbscan(pts, eps, ms) == osearch.dbscan(pts, eps, ms)
    assert kvt.dbscan(np.zeros((0, 3))) == []


def test_lib_prune_and_cluster_parity(kvt):
    rng = random.Random(23)
    for t in range(40):
        L = rng.randint(1, 40)
        e = []
        for l in range(L):
            k = rng.choice([1.0, 1.0, 3.0, 0.4])
            row = [k * v for v in monotone_profile(rng, key_weight=rng.choice([3.0, 3.0, 0.3]))]
            if rng.random() < 0.2:
                row[PAIRS9.index((4, 8))] = row[PAIRS9.index((8, 4))] * 0.5
            e.append(row)
        keep, grp, G = kvt.prune_and_cluster(PAIRS9, e)
        okeep, ogrp, oG = osearch.prune_and_cluster(PAIRS9, e)
        assert keep.tolist() == okeep and grp == ogrp and G == oG


def test_lib_search_space(kvt):
    assert kvt.search_space_log10([9] * 32) == pytest.approx(math.log10(float(9 ** 32)), rel=1e-12)
    assert 10 ** kvt.search_space_log10([5] * 6) == pytest.approx(15625, rel=1e-12)


def test_lib_errors(kvt):
    with pytest.raises(kvt.KvtError):
        kvt.pareto_prune([], [])
    with pytest.raises(kvt.KvtError):
        kvt.pareto_prune([(3, 4)], [0.1])
    with pytest.raises(kvt.KvtError):
        kvt.pareto_prune([(4, 4)], [float("nan")])
    with pytest.raises(kvt.KvtError):
        kvt.dbscan([[0.0]], eps=-1.0)
    with pytest.raises(kvt.KvtError):
        kvt.search_space_log10([0])


# ---------------------------------------------------------------------------------------------------
# end to end: K5 sensitivity on the GPU -> prune -> cluster
# ---------------------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_calibrate_prune_cluster_gpu(kvt, oracle, mode):
    import torch

    import kvt_synth

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    D, H_kv, g, S, T_q, L = 128, 2, 4, 192, 16, 6
    scale = float(np.float32(1 / math.sqrt(D)))
    e_gpu, e_ref = [], []
    for l in range(L):
        amp = 1.0 + 2.0 * (l % 2)          # two sensitivity classes
        K = (kvt_synth.keys((H_kv, S, D), seed=100 + l).float() * amp).bfloat16()
        V = kvt_synth.values((H_kv, S, D), seed=200 + l)
        Q = kvt_synth.queries((H_kv * g, T_q, D), seed=300 + l)
        got = kvt.layer_sensitivity(mode, 32, 32 if mode else 0, Q.cuda(), K.cuda(), V.cuda(), S - T_q, PAIRS9,
                                    scale=scale).cpu().numpy()
        ref = oracle.sensitivity(mode, 32, 32 if mode else 0, kvt_synth.bf16_bits(Q), kvt_synth.bf16_bits(K),
                                 kvt_synth.bf16_bits(V), S - T_q, PAIRS9, scale)
        e_gpu.append(got[:, 3].tolist())
        e_ref.append(np.asarray(ref)[:, 3].tolist())
    keep, grp, G = kvt.prune_and_cluster(PAIRS9, e_gpu)
    okeep, ogrp, oG = osearch.prune_and_cluster(PAIRS9, e_ref)
    assert keep.tolist() == okeep and grp == ogrp and G == oG

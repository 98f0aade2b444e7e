"""Oracle for the search-space pruning after calibration — TEST INFRASTRUCTURE ONLY.

Plain Python, written from the paper and the textbook definitions; shares nothing with
``paper_2502_04420_b200`` (csrc/kvt_search.cpp).  Only ``tests/`` may import it.

* ``pareto_prune``      — intra-layer pruning: "we prune those [pairs] that are not part of
                           the Pareto frontier, considering both the equivalent KV cache quantization
                           precision and the relative attention output errors".  Plain definition: pair p
                           is kept iff no other pair q dominates it (bits_q <= bits_p and e_q <= e_p with
                           one strict), bits = (b_k + b_v) / 2 (f_m of one layer, Eq. 4).  (A24)
* ``dbscan``            — DBSCAN of Ester et al. (1996), the algorithm App. D names (eps = 0.05,
                           min_samples = 2): Euclidean eps-neighbourhoods (distance <= eps, the point
                           itself included), core points have >= min_samples neighbours, clusters grown
                           from unvisited core points in index order.  (A25)
* ``prune_and_cluster`` — the two-level pruning of P:316-325 in the paper's order: (1) prune every layer,
                           (2) "partitioning layers based on distinct candidate sets", (3)
                           "clustering layers that share the same candidate set, using quantization
                           sensitivity as the clustering metric ... the relative attention output errors
                           produced by the pruned precision pairs".  Noise layers become singleton
                           groups (A26); groups numbered by first layer (A27).
* ``search_space_size`` — prod of candidate counts ("9^L", "5^G = 5^6 = 15625"), exact.

Pins: tests/test_search.py (the paper's key-first set, an independent skyline sweep, sklearn's DBSCAN,
the paper's search-space numbers).
"""
from __future__ import annotations

import math


def pair_bits(pair) -> float:
    """Equivalent bits of one layer's pair: (b_k + b_v) / 2 (Eq. 4's f_m with L = 1)."""
    return (pair[0] + pair[1]) / 2.0


def pareto_prune(pairs, e_o):
    """keep[i] iff pair i is not dominated in (bits, e_o) by any other pair."""
    if len(pairs) == 0 or len(pairs) != len(e_o):
        raise ValueError("empty or mismatched profile")
    keep = []
    for i in range(len(pairs)):
        bi, ei = pair_bits(pairs[i]), float(e_o[i])
        dominated = False
        for j in range(len(pairs)):
            if j == i:
                continue
            bj, ej = pair_bits(pairs[j]), float(e_o[j])
            if bj <= bi and ej <= ei and (bj < bi or ej < ei):
                dominated = True
        keep.append(not dominated)
    return keep


def _dist(a, b) -> float:
    return math.sqrt(sum((float(x) - float(y)) ** 2 for x, y in zip(a, b)))


def dbscan(points, eps=0.05, min_samples=2):
    """DBSCAN labels: cluster ids 0, 1, ... in order of discovery, -1 for noise (Ester et al. 1996)."""
    n = len(points)
    neigh = [[j for j in range(n) if _dist(points[i], points[j]) <= eps] for i in range(n)]
    core = [len(neigh[i]) >= min_samples for i in range(n)]
    label = [-1] * n
    cluster = 0
    for i in range(n):
        if label[i] != -1 or not core[i]:
            continue
        # grow the cluster: every point density-reachable from core point i
        label[i] = cluster
        frontier = [i]
        while frontier:
            p = frontier.pop(0)
            if not core[p]:
                continue          # a border point: in the cluster, but not expanded
            for q in neigh[p]:
                if label[q] == -1:
                    label[q] = cluster
                    frontier.append(q)
        cluster += 1
    return label


def prune_and_cluster(pairs, e_o, eps=0.05, min_samples=2):
    """(keep [L][n_pairs], group_of_layer [L], n_groups) by P:316-325 step by step."""
    L = len(e_o)
    # (1) intra-layer pruning
    keep = [pareto_prune(pairs, e_o[l]) for l in range(L)]
    # (2) partition the layers by their candidate set
    partitions = {}
    order = []
    for l in range(L):
        key = tuple(keep[l])
        if key not in partitions:
            partitions[key] = []
            order.append(key)
        partitions[key].append(l)
    # (3) DBSCAN inside each partition on the e_o of the shared candidate pairs; noise -> singletons
    groups = []                                   # lists of layers
    for key in order:
        layers = partitions[key]
        cols = [i for i in range(len(pairs)) if key[i]]
        pts = [[e_o[l][i] for i in cols] for l in layers]
        lab = dbscan(pts, eps, min_samples)
        for c in range(max(lab) + 1 if lab else 0):
            groups.append([layers[m] for m in range(len(layers)) if lab[m] == c])
        for m in range(len(layers)):
            if lab[m] == -1:
                groups.append([layers[m]])
    # (4) number the groups in order of their first layer
    groups.sort(key=lambda g: min(g))
    group_of_layer = [0] * L
    for gi, g in enumerate(groups):
        for l in g:
            group_of_layer[l] = gi
    return keep, group_of_layer, len(groups)


def search_space_size(counts) -> int:
    """Exact prod(counts)."""
    s = 1
    for c in counts:
        s *= int(c)
    return s

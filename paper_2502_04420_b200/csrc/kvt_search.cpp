// kvt_search.cpp — search-space pruning after calibration (host only).
//
// KVTuner turns the per-layer sensitivity profiles of K5 (kvt_layer_sensitivity: e_o for every
// candidate pair of every layer) into the reduced search space S_p^G of the offline MOO search:
//   * intra-layer pruning: keep the pairs on the Pareto frontier of (equivalent bits,
//     relative attention-output error e_o) — "prune those that are not part of the Pareto frontier";
//   * inter-layer clustering (App. D): partition the layers by their pruned
//     candidate set, then cluster the layers of each partition with DBSCAN (Ester et al. 1996,
//     eps = 0.05, min_samples = 2) on the vector of e_o over the partition's candidate pairs.
// Readings (A24-A27): bits(p) = (b_k + b_v) / 2 (the f_m of one layer);
// Euclidean distance, neighbourhood = distance <= eps including the point itself; DBSCAN noise points
// become singleton groups; group ids are numbered in order of their first layer.
#include <cmath>
#include <cstdint>
#include <vector>

#include "kvt_internal.h"

using kvt::clear_error;
using kvt::fail;

namespace {

double pair_bits(const kvt_pair& p) { return 0.5 * (p.key_bits + p.value_bits); }

bool valid_bits(int b) { return b == 2 || b == 4 || b == 8 || b == 16; }

// p dominated by q: no worse in both objectives and strictly better in one
bool dominates(double bq, double eq, double bp, double ep) {
    return bq <= bp && eq <= ep && (bq < bp || eq < ep);
}

// DBSCAN (Ester et al. 1996): core points have >= min_samples points (itself included) within eps;
// clusters are expanded from the unlabelled core points in index order; a border point joins the first
// cluster that reaches it; the rest is noise (-1).
void dbscan(const std::vector<const double*>& pts, int dim, double eps, int min_samples, std::vector<int>& label) {
    const int n = (int)pts.size();
    std::vector<std::vector<int>> nb(n);
    const double eps2 = eps * eps;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double d2 = 0.0;
            for (int c = 0; c < dim; ++c) {
                const double t = pts[i][c] - pts[j][c];
                d2 += t * t;
            }
            if (d2 <= eps2) nb[i].push_back(j);
        }
    label.assign(n, -1);
    std::vector<char> core(n);
    for (int i = 0; i < n; ++i) core[i] = (int)nb[i].size() >= min_samples;
    int next = 0;
    std::vector<int> stack;
    for (int i = 0; i < n; ++i) {
        if (label[i] != -1 || !core[i]) continue;
        label[i] = next;
        stack.assign(1, i);
        while (!stack.empty()) {
            const int p = stack.back();
            stack.pop_back();
            if (!core[p]) continue;
            for (int q : nb[p])
                if (label[q] == -1) {
                    label[q] = next;
                    stack.push_back(q);
                }
        }
        ++next;
    }
}

}  // namespace

extern "C" int32_t kvt_pareto_prune(const kvt_pair* pairs, const double* e_o, int32_t n_pairs, uint8_t* keep) {
    clear_error();
    if (!pairs || !e_o || !keep) return fail(KVT_ERR_INVALID_ARG, "pareto_prune: null pointer");
    if (n_pairs < 1) return fail(KVT_ERR_INVALID_ARG, "pareto_prune: empty profile");
    for (int i = 0; i < n_pairs; ++i) {
        if (!valid_bits(pairs[i].key_bits) || !valid_bits(pairs[i].value_bits))
            return fail(KVT_ERR_INVALID_ARG, "pareto_prune: pair %d has bits (%d, %d)", i, pairs[i].key_bits,
                        pairs[i].value_bits);
        if (!std::isfinite(e_o[i])) return fail(KVT_ERR_INVALID_ARG, "pareto_prune: e_o[%d] is not finite", i);
    }
    for (int i = 0; i < n_pairs; ++i) {
        bool dom = false;
        for (int j = 0; j < n_pairs && !dom; ++j)
            dom = j != i && dominates(pair_bits(pairs[j]), e_o[j], pair_bits(pairs[i]), e_o[i]);
        keep[i] = dom ? 0 : 1;
    }
    return KVT_OK;
}

extern "C" int32_t kvt_dbscan(const double* points, int32_t n, int32_t dim, double eps, int32_t min_samples,
                              int32_t* labels) {
    clear_error();
    if (n < 0 || dim < 1 || min_samples < 1 || !(eps >= 0.0) || !std::isfinite(eps))
        return fail(KVT_ERR_INVALID_ARG, "dbscan: n %d dim %d eps %g min_samples %d", n, dim, eps, min_samples);
    if (n > 0 && (!points || !labels)) return fail(KVT_ERR_INVALID_ARG, "dbscan: null pointer");
    for (long long i = 0; i < (long long)n * dim; ++i)
        if (!std::isfinite(points[i])) return fail(KVT_ERR_INVALID_ARG, "dbscan: non-finite coordinate");
    std::vector<const double*> pts(n);
    for (int i = 0; i < n; ++i) pts[i] = points + (size_t)i * dim;
    std::vector<int> lab;
    dbscan(pts, dim, eps, min_samples, lab);
    for (int i = 0; i < n; ++i) labels[i] = lab[i];
    return KVT_OK;
}

extern "C" int32_t kvt_prune_and_cluster(const kvt_pair* pairs, int32_t n_pairs, const double* e_o, int32_t n_layers,
                                         double eps, int32_t min_samples, uint8_t* keep, int32_t* group_of_layer,
                                         int32_t* n_groups) {
    clear_error();
    if (!pairs || !e_o || !keep || !group_of_layer || !n_groups)
        return fail(KVT_ERR_INVALID_ARG, "prune_and_cluster: null pointer");
    if (n_pairs < 1 || n_pairs > 64 || n_layers < 1)
        return fail(KVT_ERR_INVALID_ARG, "prune_and_cluster: n_pairs %d (1..64), n_layers %d", n_pairs, n_layers);
    if (min_samples < 1 || !(eps >= 0.0) || !std::isfinite(eps))
        return fail(KVT_ERR_INVALID_ARG, "prune_and_cluster: eps %g min_samples %d", eps, min_samples);
    // (1) intra-layer Pareto pruning
    for (int l = 0; l < n_layers; ++l) {
        const int32_t st = kvt_pareto_prune(pairs, e_o + (size_t)l * n_pairs, n_pairs, keep + (size_t)l * n_pairs);
        if (st != KVT_OK) return st;
    }
    // (2) partition by candidate set (exact equality of the kept-pair masks), in order of first layer
    std::vector<uint64_t> mask(n_layers, 0);
    for (int l = 0; l < n_layers; ++l)
        for (int i = 0; i < n_pairs; ++i)
            if (keep[(size_t)l * n_pairs + i]) mask[l] |= 1ull << i;
    std::vector<int> part(n_layers, -1);
    std::vector<uint64_t> part_mask;
    for (int l = 0; l < n_layers; ++l) {
        for (int p = 0; p < (int)part_mask.size() && part[l] < 0; ++p)
            if (part_mask[p] == mask[l]) part[l] = p;
        if (part[l] < 0) { part[l] = (int)part_mask.size(); part_mask.push_back(mask[l]); }
    }
    // (3) DBSCAN inside each partition on the e_o of its candidate pairs; noise -> singleton groups
    std::vector<int> grp_raw(n_layers, -1);
    int n_raw = 0;
    for (int p = 0; p < (int)part_mask.size(); ++p) {
        std::vector<int> members;
        for (int l = 0; l < n_layers; ++l)
            if (part[l] == p) members.push_back(l);
        std::vector<int> cols;
        for (int i = 0; i < n_pairs; ++i)
            if (part_mask[p] >> i & 1) cols.push_back(i);
        std::vector<double> vec(members.size() * cols.size());
        for (size_t m = 0; m < members.size(); ++m)
            for (size_t c = 0; c < cols.size(); ++c) vec[m * cols.size() + c] = e_o[(size_t)members[m] * n_pairs + cols[c]];
        std::vector<const double*> pts(members.size());
        for (size_t m = 0; m < members.size(); ++m) pts[m] = vec.data() + m * cols.size();
        std::vector<int> lab;
        dbscan(pts, (int)cols.size(), eps, min_samples, lab);
        int n_cl = 0;
        for (int x : lab) n_cl = x + 1 > n_cl ? x + 1 : n_cl;
        for (size_t m = 0; m < members.size(); ++m) grp_raw[members[m]] = lab[m] >= 0 ? n_raw + lab[m] : -1;
        n_raw += n_cl;
        for (size_t m = 0; m < members.size(); ++m)
            if (grp_raw[members[m]] < 0) grp_raw[members[m]] = n_raw++;
    }
    // (4) canonical numbering: groups in order of their first layer
    std::vector<int> remap(n_raw, -1);
    int g = 0;
    for (int l = 0; l < n_layers; ++l) {
        if (remap[grp_raw[l]] < 0) remap[grp_raw[l]] = g++;
        group_of_layer[l] = remap[grp_raw[l]];
    }
    *n_groups = g;
    return KVT_OK;
}

extern "C" int32_t kvt_search_space_log10(const int32_t* counts, int32_t n, double* log10_size) {
    clear_error();
    if (!log10_size || (n > 0 && !counts) || n < 0) return fail(KVT_ERR_INVALID_ARG, "search_space_log10: bad arguments");
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        if (counts[i] < 1) return fail(KVT_ERR_INVALID_ARG, "search_space_log10: counts[%d] = %d", i, counts[i]);
        s += std::log10((double)counts[i]);
    }
    *log10_size = s;
    return KVT_OK;
}

// Host-side plan builders: product re-implementations of the reference's
// scheduling layer (partition.hpp, coloring.hpp, parallel.hpp ColorfulPlan),
// scalable to the BASELINE configs and bit-exact with the reference.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>

#include "internal.hpp"

namespace csrcgpu {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

MatView view_of(const csrc_host_matrix* a, bool check_structure) {
    if (!a) throw Error("null matrix");
    MatView v;
    v.n = a->n;
    v.k = a->k;
    if (v.n < 0) throw Error("matrix: n must be >= 0");
    v.ad = a->ad;
    v.ia = a->ia;
    v.ja = a->ja;
    v.al = a->al;
    v.value_symmetric = a->value_symmetric != 0;
    v.au = v.value_symmetric ? a->al : a->au;  // CsrcMatrix::upper() (csrc_matrix.hpp:29)
    if (v.n > 0 && (!v.ad || !v.ia)) throw Error("matrix: null ad/ia");
    if (v.k > 0 && (!v.ja || !v.al || !v.au))
        throw Error(v.value_symmetric ? "matrix: null ja/al" : "matrix: null ja/al/au");
    if (v.n > 0 && static_cast<count_t>(v.ia[v.n]) != v.k)
        throw Error("matrix: ia[n] = " + std::to_string(v.ia[v.n]) + " but k = " +
                    std::to_string(v.k));
    if (check_structure && v.n > 0) {
        if (v.ia[0] != 0) throw Error("matrix: ia[0] must be 0");
        // rows checked over threads; the first offending row (lowest index) is
        // reported, as a serial scan would
        const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        const int T = static_cast<int>(std::max<count_t>(1, std::min<count_t>(std::min(hw, 32), v.n / 65536)));
        std::vector<index_t> bad(static_cast<size_t>(T), v.n);
        auto check = [&](int th) {
            const index_t b = static_cast<index_t>(static_cast<count_t>(v.n) * th / T);
            const index_t e = static_cast<index_t>(static_cast<count_t>(v.n) * (th + 1) / T);
            for (index_t i = b; i < e; ++i) {
                bool ok = v.ia[i + 1] >= v.ia[i];
                index_t prev = -1;
                for (index_t t = v.ia[i]; ok && t < v.ia[i + 1]; ++t) {
                    const index_t j = v.ja[t];
                    ok = !(j <= prev || j >= i || j < 0);
                    prev = j;
                }
                if (!ok) {
                    bad[th] = i;
                    return;
                }
            }
        };
        if (T == 1) {
            check(0);
        } else {
            std::vector<std::thread> pool;
            for (int th = 0; th < T; ++th) pool.emplace_back(check, th);
            for (auto& t : pool) t.join();
        }
        const index_t i = *std::min_element(bad.begin(), bad.end());
        if (i < v.n) {
            if (v.ia[i + 1] < v.ia[i])
                throw Error("matrix: ia not nondecreasing at row " + std::to_string(i));
            index_t prev = -1;
            for (index_t t = v.ia[i]; t < v.ia[i + 1]; ++t) {
                const index_t j = v.ja[t];
                if (j <= prev || j >= i || j < 0)
                    throw Error("matrix: row " + std::to_string(i) +
                                " lower columns must be strictly increasing and < row (ja[" +
                                std::to_string(t) + "] = " + std::to_string(j) + ")");
                prev = j;
            }
        }
    }
    return v;
}

// --- partition.hpp:46-49 stored_row_count
static inline count_t stored_row_count(const MatView& a, index_t i) {
    const count_t pairs = a.ia[i + 1] - a.ia[i];
    return 1 + (a.value_symmetric ? pairs : 2 * pairs);
}

// --- partition.hpp:55-90 partition_by_nnz (same double arithmetic)
RowPartition partition_by_nnz(const MatView& a, int p) {
    if (p < 1 || p > a.n) {
        throw Error("partition_by_nnz: need 1 <= p <= n, got p=" + std::to_string(p) +
                    ", n=" + std::to_string(a.n));
    }
    std::vector<count_t> prefix(static_cast<size_t>(a.n) + 1, 0);
    for (index_t i = 0; i < a.n; ++i) prefix[i + 1] = prefix[i] + stored_row_count(a, i);
    const double ideal = static_cast<double>(prefix[a.n]) / p;

    RowPartition part;
    part.p = p;
    part.block_start.assign(static_cast<size_t>(p) + 1, 0);
    part.block_start[p] = a.n;
    index_t b = 0;
    for (int t = 1; t < p; ++t) {
        const double target = t * ideal;
        const index_t lo_bound = part.block_start[t - 1] + 1;
        const index_t hi_bound = a.n - (p - t);
        b = std::max(b, lo_bound);
        while (b < hi_bound && static_cast<double>(prefix[b]) < target) ++b;
        if (b > lo_bound && std::abs(static_cast<double>(prefix[b - 1]) - target) <=
                                std::abs(static_cast<double>(prefix[b]) - target))
            --b;
        part.block_start[t] = b;
    }
    part.block_nnz.resize(static_cast<size_t>(p));
    for (int t = 0; t < p; ++t)
        part.block_nnz[t] = prefix[part.block_start[t + 1]] - prefix[part.block_start[t]];
    return part;
}

// --- partition.hpp:94-109 effective_range(s)
void effective_ranges(const MatView& a, const std::vector<index_t>& bs, std::vector<index_t>& lo,
                      std::vector<index_t>& hi) {
    const int p = static_cast<int>(bs.size()) - 1;
    lo.assign(p, 0);
    hi.assign(p, 0);
    for (int t = 0; t < p; ++t) {
        const index_t first = bs[t], last = bs[t + 1];
        if (first >= last) throw Error("effective_range: empty block");
        index_t l = first;
        for (index_t t = a.ia[first]; t < a.ia[last]; ++t) l = std::min(l, a.ja[t]);
        lo[t] = l;
        hi[t] = last - 1;
    }
}

// --- partition.hpp:113-134 build_interval_plan
IntervalPlan build_interval_plan(const std::vector<index_t>& lo, const std::vector<index_t>& hi) {
    IntervalPlan plan;
    std::vector<index_t> cuts;
    for (size_t b = 0; b < lo.size(); ++b) {
        cuts.push_back(lo[b]);
        cuts.push_back(hi[b] + 1);
    }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    plan.boundaries = cuts;
    plan.contrib_ptr.push_back(0);
    for (size_t c = 0; c + 1 < cuts.size(); ++c) {
        const index_t b0 = cuts[c], e0 = cuts[c + 1];
        size_t before = plan.contrib.size();
        for (int b = 0; b < static_cast<int>(lo.size()); ++b)
            if (lo[b] <= b0 && e0 - 1 <= hi[b]) plan.contrib.push_back(b);
        if (plan.contrib.size() == before) continue;
        plan.iv_begin.push_back(b0);
        plan.iv_end.push_back(e0);
        plan.contrib_ptr.push_back(static_cast<index_t>(plan.contrib.size()));
    }
    return plan;
}

// ---------------------------------------------------------------- coloring
// The reference stores both conflict edge sets in std::set (coloring.hpp:13,
// 39-91), which does not scale past ~64^3. Here the combined conflict
// neighbourhood of a row is enumerated on the fly from the direct-graph CSR
// adjacency:
//   neighborhood mode (coloring.hpp:55-72): N(v) u N(N(v)) \ {v}
//   exact mode (coloring.hpp:73-89):        N(v) u {u != v : ja(u) n ja(v) != 0}
// First-fit colouring (coloring.hpp:147-159) depends only on the edge set and
// the vertex sequence, so the colours are identical to the reference's.
namespace {

struct Adjacency {
    index_t n = 0;
    std::vector<count_t> ptr;     // full direct graph, sorted rows
    std::vector<index_t> idx;
    std::vector<count_t> up_ptr;  // rows having column k as a lower column
    std::vector<index_t> up_idx;
};

Adjacency build_adjacency(const MatView& a) {
    Adjacency g;
    g.n = a.n;
    std::vector<count_t> up_cnt(static_cast<size_t>(a.n) + 1, 0);
    for (count_t t = 0; t < a.k; ++t) ++up_cnt[a.ja[t] + 1];
    g.up_ptr.assign(static_cast<size_t>(a.n) + 1, 0);
    for (index_t i = 0; i < a.n; ++i) g.up_ptr[i + 1] = g.up_ptr[i] + up_cnt[i + 1];
    g.up_idx.resize(static_cast<size_t>(a.k));
    {
        std::vector<count_t> next(g.up_ptr.begin(), g.up_ptr.end() - 1);
        for (index_t i = 0; i < a.n; ++i)
            for (index_t t = a.ia[i]; t < a.ia[i + 1]; ++t) g.up_idx[next[a.ja[t]]++] = i;
    }
    g.ptr.assign(static_cast<size_t>(a.n) + 1, 0);
    for (index_t v = 0; v < a.n; ++v)
        g.ptr[v + 1] = g.ptr[v] + (a.ia[v + 1] - a.ia[v]) + (g.up_ptr[v + 1] - g.up_ptr[v]);
    g.idx.resize(static_cast<size_t>(g.ptr[a.n]));
    for (index_t v = 0; v < a.n; ++v) {
        count_t q = g.ptr[v];
        for (index_t t = a.ia[v]; t < a.ia[v + 1]; ++t) g.idx[q++] = a.ja[t];
        for (count_t t = g.up_ptr[v]; t < g.up_ptr[v + 1]; ++t) g.idx[q++] = g.up_idx[t];
    }
    return g;
}

// Calls f(u) once for every combined conflict neighbour u of v (u != v).
// `stamp` must be sized n and hold values != v on entry for fresh vertices.
template <class F>
void for_each_conflict(const MatView& a, const Adjacency& g, int mode, index_t v,
                       std::vector<index_t>& stamp, F&& f) {
    stamp[v] = v;  // exclude v itself
    auto visit = [&](index_t u) {
        if (stamp[u] != v) {
            stamp[u] = v;
            f(u);
        }
    };
    for (count_t q = g.ptr[v]; q < g.ptr[v + 1]; ++q) visit(g.idx[q]);
    if (mode == CSRC_CONFLICT_NEIGHBORHOOD) {
        for (count_t q = g.ptr[v]; q < g.ptr[v + 1]; ++q) {
            const index_t w = g.idx[q];
            for (count_t r = g.ptr[w]; r < g.ptr[w + 1]; ++r) visit(g.idx[r]);
        }
    } else {
        for (index_t t = a.ia[v]; t < a.ia[v + 1]; ++t) {
            const index_t kcol = a.ja[t];
            for (count_t r = g.up_ptr[kcol]; r < g.up_ptr[kcol + 1]; ++r) visit(g.up_idx[r]);
        }
    }
}

std::vector<count_t> combined_degrees(const MatView& a, const Adjacency& g, int mode) {
    std::vector<count_t> deg(static_cast<size_t>(a.n), 0);
    const int threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int th = 0; th < threads; ++th) {
        pool.emplace_back([&, th] {
            std::vector<index_t> stamp(static_cast<size_t>(a.n), -1);
            const index_t b = static_cast<index_t>(static_cast<count_t>(a.n) * th / threads);
            const index_t e = static_cast<index_t>(static_cast<count_t>(a.n) * (th + 1) / threads);
            for (index_t v = b; v < e; ++v) {
                count_t d = 0;
                for_each_conflict(a, g, mode, v, stamp, [&](index_t) { ++d; });
                deg[v] = d;
            }
        });
    }
    for (auto& t : pool) t.join();
    return deg;
}

// Min-(deg, index) segment tree for smallest-last (coloring.hpp:134-142 tie
// rule: strict '<' scan, so the lowest index wins among equal degrees).
struct MinTree {
    int size = 1;
    std::vector<count_t> key;  // deg, or max for removed
    std::vector<index_t> arg;
    explicit MinTree(const std::vector<count_t>& deg) {
        while (size < static_cast<int>(deg.size())) size <<= 1;
        key.assign(2 * size, std::numeric_limits<count_t>::max());
        arg.assign(2 * size, std::numeric_limits<index_t>::max());
        for (size_t i = 0; i < deg.size(); ++i) {
            key[size + i] = deg[i];
            arg[size + i] = static_cast<index_t>(i);
        }
        for (int i = size - 1; i >= 1; --i) pull(i);
    }
    void pull(int i) {
        const int l = 2 * i, r = 2 * i + 1;
        if (key[l] < key[r] || (key[l] == key[r] && arg[l] <= arg[r])) {
            key[i] = key[l];
            arg[i] = arg[l];
        } else {
            key[i] = key[r];
            arg[i] = arg[r];
        }
    }
    void set(index_t v, count_t k) {
        int i = size + v;
        key[i] = k;
        for (i >>= 1; i >= 1; i >>= 1) pull(i);
    }
};

}  // namespace

std::vector<int32_t> color_rows(const MatView& a, int mode, int order, int* n_colors_out) {
    if (mode != CSRC_CONFLICT_NEIGHBORHOOD && mode != CSRC_CONFLICT_EXACT)
        throw Error("color_rows: unknown conflict mode " + std::to_string(mode));
    if (order < CSRC_ORDER_NATURAL || order > CSRC_ORDER_SMALLEST_LAST)
        throw Error("color_rows: unknown color order " + std::to_string(order));
    const index_t n = a.n;
    Adjacency g = build_adjacency(a);
    std::vector<index_t> seq(static_cast<size_t>(n));
    for (index_t i = 0; i < n; ++i) seq[i] = i;
    if (order == CSRC_ORDER_LARGEST_FIRST) {
        std::vector<count_t> deg = combined_degrees(a, g, mode);
        std::stable_sort(seq.begin(), seq.end(),
                         [&](index_t u, index_t v) { return deg[u] > deg[v]; });
    } else if (order == CSRC_ORDER_SMALLEST_LAST) {
        std::vector<count_t> deg = combined_degrees(a, g, mode);
        MinTree tree(deg);
        std::vector<char> removed(static_cast<size_t>(n), 0);
        std::vector<index_t> stamp(static_cast<size_t>(n), -1);
        std::vector<index_t> removal;
        removal.reserve(static_cast<size_t>(n));
        for (index_t step = 0; step < n; ++step) {
            const index_t best = tree.arg[1];
            removed[best] = 1;
            removal.push_back(best);
            tree.set(best, std::numeric_limits<count_t>::max());
            for_each_conflict(a, g, mode, best, stamp, [&](index_t u) {
                if (!removed[u]) tree.set(u, --deg[u]);
            });
        }
        std::reverse(removal.begin(), removal.end());
        seq = std::move(removal);
    }
    std::vector<int32_t> color(static_cast<size_t>(n), -1);
    std::vector<index_t> stamp(static_cast<size_t>(n), -1);
    std::vector<index_t> used;  // used[c] == v  <=> colour c taken by a neighbour of v
    int n_colors = 0;
    for (index_t v : seq) {
        if (static_cast<int>(used.size()) < n_colors + 1) used.resize(n_colors + 1, -1);
        for_each_conflict(a, g, mode, v, stamp, [&](index_t u) {
            const int c = color[u];
            if (c >= 0) used[c] = v;
        });
        int c = 0;
        while (c < n_colors && used[c] == v) ++c;
        color[v] = c;
        n_colors = std::max(n_colors, c + 1);
    }
    *n_colors_out = n_colors;
    return color;
}

void conflict_edge_counts(const MatView& a, int mode, count_t* n_direct, count_t* n_indirect) {
    Adjacency g = build_adjacency(a);
    std::vector<count_t> deg = combined_degrees(a, g, mode);
    count_t total = 0;
    for (count_t d : deg) total += d;
    *n_direct = a.k;
    *n_indirect = total / 2 - a.k;
}

// --- coloring.hpp:175-198 validate_coloring (same first-violation report)
Validity validate_coloring(const MatView& a, const int32_t* color, int n_colors) {
    Validity v;
    const index_t n = a.n;
    std::vector<count_t> cptr(static_cast<size_t>(n_colors) + 1, 0);
    for (index_t i = 0; i < n; ++i) {
        if (color[i] < 0 || color[i] >= n_colors)
            throw Error("validate_coloring: row " + std::to_string(i) + " has colour " +
                        std::to_string(color[i]) + " outside [0, " + std::to_string(n_colors) +
                        ")");
        ++cptr[color[i] + 1];
    }
    for (int c = 0; c < n_colors; ++c) cptr[c + 1] += cptr[c];
    std::vector<index_t> rows(static_cast<size_t>(n));
    {
        std::vector<count_t> next(cptr.begin(), cptr.end() - 1);
        for (index_t i = 0; i < n; ++i) rows[next[color[i]]++] = i;
    }
    std::vector<int32_t> cls(static_cast<size_t>(n), -1);
    std::vector<index_t> writer(static_cast<size_t>(n), -1);
    for (int c = 0; c < n_colors; ++c) {
        for (count_t r = cptr[c]; r < cptr[c + 1]; ++r) {
            const index_t i = rows[r];
            auto claim = [&](index_t q) {
                if (cls[q] == c) {
                    v.valid = false;
                    v.row_a = writer[q];
                    v.row_b = i;
                    v.position = q;
                    return false;
                }
                cls[q] = c;
                writer[q] = i;
                return true;
            };
            if (!claim(i)) return v;
            for (index_t t = a.ia[i]; t < a.ia[i + 1]; ++t)
                if (!claim(a.ja[t])) return v;
        }
    }
    return v;
}

}  // namespace csrcgpu

using namespace csrcgpu;

extern "C" {

const char* csrc_gpu_last_error(void) { return g_last_error.c_str(); }
int csrc_gpu_abi_version(void) { return CSRC_GPU_ABI_VERSION; }

int csrc_partition_by_nnz(const csrc_host_matrix* m, int32_t p, int32_t* block_start,
                          int64_t* block_nnz) {
    return guarded(__func__, [&] {
        MatView a = view_of(m, false);
        RowPartition part = partition_by_nnz(a, p);
        if (block_start) std::copy(part.block_start.begin(), part.block_start.end(), block_start);
        if (block_nnz) std::copy(part.block_nnz.begin(), part.block_nnz.end(), block_nnz);
    });
}

int csrc_effective_ranges(const csrc_host_matrix* m, int32_t p, const int32_t* block_start,
                          int32_t* lo, int32_t* hi) {
    return guarded(__func__, [&] {
        MatView a = view_of(m, false);
        if (p < 1) throw Error("effective_ranges: p must be >= 1");
        std::vector<index_t> bs(block_start, block_start + p + 1), l, h;
        effective_ranges(a, bs, l, h);
        std::copy(l.begin(), l.end(), lo);
        std::copy(h.begin(), h.end(), hi);
    });
}

int csrc_bands_x_hi(const csrc_host_matrix* m, int32_t p, const int32_t* block_start, int32_t* x_hi) {
    return guarded(__func__, [&] {
        MatView a = view_of(m, false);
        if (p < 1) throw Error("bands_x_hi: p must be >= 1");
        // x_hi[b] = max(row_end_b, 1 + the last row whose lower columns fall in band b);
        // rows scanned over threads, each keeping its own per-band maximum
        const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        const int T = static_cast<int>(std::max<count_t>(1, std::min<count_t>(std::min(hw, 32), a.n / 65536)));
        std::vector<std::vector<index_t>> part(T, std::vector<index_t>(p, -1));
        auto band_of = [&](index_t q) {
            return static_cast<int>(std::upper_bound(block_start, block_start + p + 1, q) - block_start) - 1;
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                const index_t r0 = static_cast<index_t>(static_cast<count_t>(a.n) * t / T);
                const index_t r1 = static_cast<index_t>(static_cast<count_t>(a.n) * (t + 1) / T);
                std::vector<index_t>& mx = part[t];
                for (index_t r = r0; r < r1; ++r)
                    for (index_t q = a.ia[r]; q < a.ia[r + 1]; ++q) {
                        const int b = band_of(a.ja[q]);
                        if (b >= 0 && b < p && r > mx[b]) mx[b] = r;
                        // columns ascend within a row: skip to the next band
                        if (b >= 0 && b + 1 <= p) {
                            const index_t next = block_start[b + 1];
                            while (q + 1 < a.ia[r + 1] && a.ja[q + 1] < next) ++q;
                        }
                    }
            });
        for (auto& th : pool) th.join();
        for (int b = 0; b < p; ++b) {
            index_t best = block_start[b + 1];
            for (int t = 0; t < T; ++t)
                if (part[t][b] >= 0) best = std::max<index_t>(best, part[t][b] + 1);
            x_hi[b] = best;
        }
    });
}

int csrc_interval_plan(int32_t p, const int32_t* lo, const int32_t* hi, int32_t* n_intervals,
                       int32_t* n_contrib, int32_t* n_boundaries, int32_t* iv_begin,
                       int32_t* iv_end, int32_t* contrib_ptr, int32_t* contrib,
                       int32_t* boundaries) {
    return guarded(__func__, [&] {
        std::vector<index_t> l(lo, lo + p), h(hi, hi + p);
        IntervalPlan plan = build_interval_plan(l, h);
        *n_intervals = static_cast<int32_t>(plan.iv_begin.size());
        *n_contrib = static_cast<int32_t>(plan.contrib.size());
        *n_boundaries = static_cast<int32_t>(plan.boundaries.size());
        if (iv_begin) std::copy(plan.iv_begin.begin(), plan.iv_begin.end(), iv_begin);
        if (iv_end) std::copy(plan.iv_end.begin(), plan.iv_end.end(), iv_end);
        if (contrib_ptr) std::copy(plan.contrib_ptr.begin(), plan.contrib_ptr.end(), contrib_ptr);
        if (contrib) std::copy(plan.contrib.begin(), plan.contrib.end(), contrib);
        if (boundaries) std::copy(plan.boundaries.begin(), plan.boundaries.end(), boundaries);
    });
}

int csrc_color_rows(const csrc_host_matrix* m, int32_t mode, int32_t order, int32_t* color,
                    int32_t* n_colors) {
    return guarded(__func__, [&] {
        MatView a = view_of(m, false);
        int nc = 0;
        std::vector<int32_t> c = color_rows(a, mode, order, &nc);
        std::copy(c.begin(), c.end(), color);
        *n_colors = nc;
    });
}

int csrc_conflict_edge_counts(const csrc_host_matrix* m, int32_t mode, int64_t* n_direct,
                              int64_t* n_indirect) {
    return guarded(__func__, [&] {
        MatView a = view_of(m, false);
        conflict_edge_counts(a, mode, n_direct, n_indirect);
    });
}

int csrc_validate_coloring(const csrc_host_matrix* m, const int32_t* color, int32_t n_colors,
                           int32_t* valid, int32_t* row_a, int32_t* row_b, int32_t* position) {
    return guarded(__func__, [&] {
        MatView a = view_of(m, false);
        Validity v = validate_coloring(a, color, n_colors);
        *valid = v.valid ? 1 : 0;
        if (row_a) *row_a = v.row_a;
        if (row_b) *row_b = v.row_b;
        if (position) *position = v.position;
    });
}

// parallel.hpp:69-93 ColorfulPlan::slice
int csrc_colorful_slices(const csrc_host_matrix* m, const int32_t* color, int32_t n_colors,
                         int32_t p, int64_t* slices) {
    return guarded(__func__, [&] {
        MatView a = view_of(m, false);
        if (p < 1) throw Error("colorful_slices: p must be >= 1");
        std::vector<std::vector<index_t>> classes(static_cast<size_t>(n_colors));
        for (index_t i = 0; i < a.n; ++i) classes.at(color[i]).push_back(i);
        for (int c = 0; c < n_colors; ++c) {
            const auto& rows = classes[c];
            std::vector<count_t> prefix(rows.size() + 1, 0);
            for (size_t r = 0; r < rows.size(); ++r)
                prefix[r + 1] = prefix[r] + stored_row_count(a, rows[r]);
            const double ideal = static_cast<double>(prefix.back()) / p;
            size_t b = 0, prev = 0;
            int64_t* out = slices + static_cast<size_t>(c) * p * 2;
            for (int t = 1; t < p; ++t) {
                const double target = t * ideal;
                if (b < prev) b = prev;
                while (b < rows.size() && static_cast<double>(prefix[b]) < target) ++b;
                if (b > prev && std::abs(static_cast<double>(prefix[b - 1]) - target) <=
                                    std::abs(static_cast<double>(prefix[b]) - target))
                    --b;
                out[2 * (t - 1)] = static_cast<int64_t>(prev);
                out[2 * (t - 1) + 1] = static_cast<int64_t>(b);
                prev = b;
            }
            out[2 * (p - 1)] = static_cast<int64_t>(prev);
            out[2 * (p - 1) + 1] = static_cast<int64_t>(rows.size());
        }
    });
}

// working_set.hpp:17-25, in bytes; dtype F32 halves the real-valued arrays
// (6*nnz + 10*n + 4 for fp32 values).
int64_t csrc_model_bytes(int64_t n, int64_t nnz_stored, int32_t value_symmetric, int32_t dtype) {
    if (dtype == CSRC_DTYPE_F32) {
        // reals ad,al,(au),x,y at 4 B; ints ia, ja at 4 B
        if (value_symmetric) return 8 * nnz_stored + 8 * n + 4;  // k = nnz_stored - n
        return 6 * nnz_stored + 10 * n + 4;
    }
    if (value_symmetric) return 12 * nnz_stored + 16 * n + 4;
    return 10 * nnz_stored + 18 * n + 4;
}

// cost_model.hpp:20-42 (csrc / csrc_sym at :33, :37): flops = 2*nnz_full - n
int64_t csrc_model_flops(int64_t n, int64_t nnz_full) { return 2 * nnz_full - n; }

}  // extern "C"

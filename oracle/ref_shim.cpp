// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/csrc_oracle.c header).
//
// C shim over the reference implementation itself: compiled by
// oracle/Makefile with -I/root/reference/proj/include into
// oracle/_ref/libcsrc_ref.so (git-ignored; travels to the GPU box with the
// other built .so files). No reference source is copied: this file only
// includes the reference headers where they lie and forwards to them.
//
// Used to (1) generate and pin golden vectors (tests/golden/make_golden.py),
// (2) cross-check the plain-C oracle and the product's host planners, and
// (3) time the reference CPU path for bench.py (cpu_baseline, --impl reference).
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "csrc/csrc.hpp"

using namespace csrc;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

CsrcMatrix make(int32_t n, int64_t k, const double* ad, const int32_t* ia, const int32_t* ja,
                const double* al, const double* au, int vs) {
    CsrcMatrix c;
    c.n = n;
    c.ad.assign(ad, ad + n);
    c.ia.assign(ia, ia + n + 1);
    c.ja.assign(ja, ja + k);
    c.al.assign(al, al + k);
    if (!vs) c.au.assign(au, au + k);
    c.value_symmetric = vs != 0;
    return c;
}

TripletMatrix make_trip(int32_t n, int64_t m, const int32_t* r, const int32_t* c,
                        const double* v) {
    TripletMatrix t;
    t.n_rows = t.n_cols = n;
    t.entries.reserve(m);
    for (int64_t e = 0; e < m; ++e) t.add(r[e], c[e], v[e]);
    return t;
}

// last CSRC built by ref_build_csrc
CsrcMatrix g_built;
TripletMatrix g_trip;

struct Exec {
    CsrcMatrix a;
    std::unique_ptr<ParallelSpmv> ex;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// build_csr (csr.hpp:55-92) -> csr_to_csrc (csrc_matrix.hpp:44-91); results
// fetched with ref_built_sizes / ref_built_copy.
int ref_build_csrc(int32_t n, int64_t m, const int32_t* rows, const int32_t* cols,
                   const double* vals) {
    return guarded([&] { g_built = csr_to_csrc(build_csr(make_trip(n, m, rows, cols, vals))); });
}
void ref_built_sizes(int32_t* n, int64_t* k, int32_t* vs) {
    *n = g_built.n;
    *k = g_built.k_off();
    *vs = g_built.value_symmetric ? 1 : 0;
}
void ref_built_copy(double* ad, int32_t* ia, int32_t* ja, double* al, double* au) {
    std::memcpy(ad, g_built.ad.data(), sizeof(double) * g_built.ad.size());
    std::memcpy(ia, g_built.ia.data(), sizeof(int32_t) * g_built.ia.size());
    std::memcpy(ja, g_built.ja.data(), sizeof(int32_t) * g_built.ja.size());
    std::memcpy(al, g_built.al.data(), sizeof(double) * g_built.al.size());
    if (!g_built.value_symmetric)
        std::memcpy(au, g_built.au.data(), sizeof(double) * g_built.au.size());
}

// build_csr (csr.hpp:55-92) alone; results fetched with ref_csr_sizes / ref_csr_copy.
CsrMatrix g_csr;
int ref_build_csr(int32_t n_rows, int32_t n_cols, int64_t m, const int32_t* rows,
                  const int32_t* cols, const double* vals) {
    return guarded([&] {
        TripletMatrix t;
        t.n_rows = n_rows;
        t.n_cols = n_cols;
        for (int64_t e = 0; e < m; ++e) t.add(rows[e], cols[e], vals[e]);
        g_csr = build_csr(t);
    });
}
void ref_csr_sizes(int32_t* n_rows, int32_t* n_cols, int64_t* nnz) {
    *n_rows = g_csr.n_rows;
    *n_cols = g_csr.n_cols;
    *nnz = g_csr.nnz();
}
void ref_csr_copy(int32_t* rp, int32_t* ci, double* va) {
    std::memcpy(rp, g_csr.row_ptr.data(), sizeof(int32_t) * g_csr.row_ptr.size());
    std::memcpy(ci, g_csr.col_idx.data(), sizeof(int32_t) * g_csr.col_idx.size());
    std::memcpy(va, g_csr.values.data(), sizeof(double) * g_csr.values.size());
}

// spmv_csr (kernels.hpp:7-22) of the reference.
int ref_spmv_csr(int32_t n_rows, int32_t n_cols, const int32_t* rp, const int32_t* ci, const double* va,
                 const double* x, double* y) {
    return guarded([&] {
        CsrMatrix a;
        a.n_rows = n_rows;
        a.n_cols = n_cols;
        a.row_ptr.assign(rp, rp + n_rows + 1);
        a.col_idx.assign(ci, ci + rp[n_rows]);
        a.values.assign(va, va + rp[n_rows]);
        Vector xv(x, x + n_cols);
        Vector out = spmv_csr(a, xv);
        std::memcpy(y, out.data(), sizeof(double) * n_rows);
    });
}

// decompose_rect (csrc_matrix.hpp:113-142): square part -> ref_built_*, tail -> ref_csr_*.
int ref_decompose_rect(int32_t n_rows, int32_t n_cols, const int32_t* rp, const int32_t* ci,
                       const double* va) {
    return guarded([&] {
        CsrMatrix a;
        a.n_rows = n_rows;
        a.n_cols = n_cols;
        a.row_ptr.assign(rp, rp + n_rows + 1);
        a.col_idx.assign(ci, ci + rp[n_rows]);
        a.values.assign(va, va + rp[n_rows]);
        CsrcRectMatrix r = decompose_rect(a);
        g_built = r.square;
        g_csr = r.rect;
    });
}

// spmv_csrc_rect (kernels.hpp:69-91).
int ref_spmv_csrc_rect(int32_t n, int64_t k, const double* ad, const int32_t* ia,
                       const int32_t* ja, const double* al, const double* au, int32_t vs,
                       int32_t m_cols, const int32_t* trp, const int32_t* tci, const double* tva,
                       const double* x, int64_t x_len, double* y) {
    return guarded([&] {
        CsrcRectMatrix r;
        r.square = make(n, k, ad, ia, ja, al, au, vs);
        r.rect.n_rows = n;
        r.rect.n_cols = m_cols - n;
        r.rect.row_ptr.assign(trp, trp + n + 1);
        r.rect.col_idx.assign(tci, tci + trp[n]);
        r.rect.values.assign(tva, tva + trp[n]);
        r.m = m_cols;
        Vector xv(x, x + x_len);
        Vector out = spmv_csrc_rect(r, xv);
        std::memcpy(y, out.data(), sizeof(double) * n);
    });
}

// generate.hpp:12-65 families -> triplets (fetched with ref_trip_*)
int ref_gen_random_sym(int32_t n, double density, uint64_t seed, int32_t vs) {
    return guarded([&] { g_trip = generate_random_sym(n, density, seed, vs != 0); });
}
int ref_gen_band(int32_t n, int32_t h, int32_t vs) {
    return guarded([&] { g_trip = generate_band(n, h, vs != 0); });
}
int ref_gen_dense(int32_t n) {
    return guarded([&] { g_trip = generate_dense(n); });
}
int64_t ref_trip_size() { return static_cast<int64_t>(g_trip.entries.size()); }
void ref_trip_copy(int32_t* r, int32_t* c, double* v) {
    for (size_t e = 0; e < g_trip.entries.size(); ++e) {
        r[e] = g_trip.entries[e].row;
        c[e] = g_trip.entries[e].col;
        v[e] = g_trip.entries[e].value;
    }
}

int ref_spmv_csrc(int32_t n, int64_t k, const double* ad, const int32_t* ia, const int32_t* ja,
                  const double* al, const double* au, int32_t vs, const double* x, double* y,
                  int32_t transpose) {
    return guarded([&] {
        CsrcMatrix c = make(n, k, ad, ia, ja, al, au, vs);
        Vector xv(x, x + n);
        Vector r = transpose ? spmv_csrc_transpose(c, xv) : spmv_csrc(c, xv);
        std::memcpy(y, r.data(), sizeof(double) * n);
    });
}

int ref_partition_by_nnz(int32_t n, int64_t k, const int32_t* ia, int32_t vs, int32_t p,
                         int32_t* bs, int64_t* bn) {
    return guarded([&] {
        CsrcMatrix c;
        c.n = n;
        c.ia.assign(ia, ia + n + 1);
        c.ja.assign(static_cast<size_t>(k), 0);
        c.value_symmetric = vs != 0;
        RowPartition part = partition_by_nnz(c, p);
        std::memcpy(bs, part.block_start.data(), sizeof(int32_t) * (p + 1));
        std::memcpy(bn, part.block_nnz.data(), sizeof(int64_t) * p);
    });
}

int ref_effective_ranges(int32_t n, int64_t k, const int32_t* ia, const int32_t* ja, int32_t p,
                         const int32_t* bs, int32_t* lo, int32_t* hi) {
    return guarded([&] {
        CsrcMatrix c;
        c.n = n;
        c.ia.assign(ia, ia + n + 1);
        c.ja.assign(ja, ja + k);
        RowPartition part;
        part.p = p;
        part.block_start.assign(bs, bs + p + 1);
        auto r = effective_ranges(c, part);
        for (int b = 0; b < p; ++b) {
            lo[b] = r[b].lo;
            hi[b] = r[b].hi;
        }
    });
}

// build_interval_plan: iv_begin/iv_end/cptr/contrib sized 2p / 2p+1 / 2p*p
int ref_interval_plan(int32_t p, const int32_t* lo, const int32_t* hi, int32_t* n_iv,
                      int32_t* iv_begin, int32_t* iv_end, int32_t* cptr, int32_t* contrib,
                      int32_t* n_bd, int32_t* boundaries) {
    return guarded([&] {
        std::vector<EffectiveRange> r(p);
        for (int b = 0; b < p; ++b) r[b] = {lo[b], hi[b]};
        IntervalPlan plan = build_interval_plan(r);
        *n_iv = static_cast<int32_t>(plan.intervals.size());
        *n_bd = static_cast<int32_t>(plan.boundaries.size());
        std::memcpy(boundaries, plan.boundaries.data(), sizeof(int32_t) * plan.boundaries.size());
        int32_t q = 0;
        cptr[0] = 0;
        for (size_t i = 0; i < plan.intervals.size(); ++i) {
            iv_begin[i] = plan.intervals[i].begin;
            iv_end[i] = plan.intervals[i].end;
            for (int b : plan.intervals[i].contributors) contrib[q++] = b;
            cptr[i + 1] = q;
        }
    });
}

int ref_color_rows(int32_t n, int64_t k, const int32_t* ia, const int32_t* ja, int32_t mode,
                   int32_t order, int32_t* color, int32_t* n_colors, int64_t* n_direct,
                   int64_t* n_indirect) {
    return guarded([&] {
        CsrcMatrix c;
        c.n = n;
        c.ia.assign(ia, ia + n + 1);
        c.ja.assign(ja, ja + k);
        ConflictGraph g =
            build_conflict_graph(c, mode ? ConflictMode::exact : ConflictMode::neighborhood);
        Coloring col = color_rows(g, order == 0   ? ColorOrder::natural
                                     : order == 1 ? ColorOrder::largest_first
                                                  : ColorOrder::smallest_last);
        for (int32_t i = 0; i < n; ++i) color[i] = col.color[i];
        *n_colors = col.n_colors;
        *n_direct = static_cast<int64_t>(g.direct_edges.size());
        *n_indirect = static_cast<int64_t>(g.indirect_edges.size());
    });
}

int ref_validate_coloring(int32_t n, int64_t k, const int32_t* ia, const int32_t* ja,
                          const int32_t* color, int32_t n_colors, int32_t* out4) {
    return guarded([&] {
        CsrcMatrix c;
        c.n = n;
        c.ia.assign(ia, ia + n + 1);
        c.ja.assign(ja, ja + k);
        Coloring col;
        col.color.assign(color, color + n);
        col.n_colors = n_colors;
        col.classes.assign(n_colors, {});
        for (int32_t i = 0; i < n; ++i) col.classes[color[i]].push_back(i);
        ColoringValidity v = validate_coloring(c, col);
        out4[0] = v.valid;
        out4[1] = v.row_a;
        out4[2] = v.row_b;
        out4[3] = v.position;
    });
}

// ColorfulPlan::slice (parallel.hpp:69-93): slices[n_colors * p * 2]
int ref_colorful_slices(int32_t n, int64_t k, const int32_t* ia, int32_t vs,
                        const int32_t* color, int32_t n_colors, int32_t p, int64_t* slices) {
    return guarded([&] {
        CsrcMatrix c;
        c.n = n;
        c.ia.assign(ia, ia + n + 1);
        c.ja.assign(static_cast<size_t>(k), 0);
        c.value_symmetric = vs != 0;
        ColorfulPlan plan;
        plan.coloring.color.assign(color, color + n);
        plan.coloring.n_colors = n_colors;
        plan.coloring.classes.assign(n_colors, {});
        for (int32_t i = 0; i < n; ++i) plan.coloring.classes[color[i]].push_back(i);
        plan.slice(c, p);
        for (int cl = 0; cl < n_colors; ++cl)
            for (int w = 0; w < p; ++w) {
                slices[(cl * p + w) * 2] = static_cast<int64_t>(plan.class_slices[cl][w].first);
                slices[(cl * p + w) * 2 + 1] = static_cast<int64_t>(plan.class_slices[cl][w].second);
            }
    });
}

// ParallelSpmv (parallel.hpp:151-446) persistent executor for the CPU
// baseline: kind 0 seq, 1 local_buffers, 2 colorful (neighbourhood coloring).
void* ref_exec_create(int32_t n, int64_t k, const double* ad, const int32_t* ia,
                      const int32_t* ja, const double* al, const double* au, int32_t vs,
                      int32_t kind, int32_t accum, int32_t p) {
    try {
        auto e = std::make_unique<Exec>();
        e->a = make(n, k, ad, ia, ja, al, au, vs);
        Strategy s{kind == 0   ? StrategyKind::sequential
                   : kind == 1 ? StrategyKind::local_buffers
                               : StrategyKind::colorful,
                   static_cast<AccumMethod>(accum), p};
        e->ex = std::make_unique<ParallelSpmv>(e->a, s);
        return e.release();
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return nullptr;
    }
}

// reps products; returns total seconds; y receives the last product;
// phases[3] = summed PhaseTimings.
double ref_exec_run(void* h, const double* x, double* y, int32_t reps, double* phases) {
    auto* e = static_cast<Exec*>(h);
    Vector xv(x, x + e->a.n), yv(e->a.n);
    PhaseTimings acc{};
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) {
        e->ex->apply(xv, yv);
        const auto& t = e->ex->last_timings();
        acc.init_max += t.init_max;
        acc.compute_max += t.compute_max;
        acc.accumulate_max += t.accumulate_max;
    }
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(y, yv.data(), sizeof(double) * e->a.n);
    if (phases) {
        phases[0] = acc.init_max;
        phases[1] = acc.compute_max;
        phases[2] = acc.accumulate_max;
    }
    return dt;
}

int32_t ref_exec_buffers(void* h) { return static_cast<Exec*>(h)->ex->buffers_allocated(); }
void ref_exec_destroy(void* h) { delete static_cast<Exec*>(h); }

double ref_working_set_kb(int64_t n, int64_t nnz, int32_t vs) {
    return working_set_kb(n, nnz, vs != 0);
}

void ref_count_ops(int32_t format, int64_t n, int64_t nnz_full, int64_t* flops, int64_t* loads) {
    KernelStats s = count_ops(static_cast<Format>(format), n, nnz_full);
    *flops = s.flops;
    *loads = s.loads;
}

}  // extern "C"

// Drop-in check: the reference's own types and calls (csrc::CsrcMatrix,
// csrc::Strategy, ParallelSpmv, ColorfulPlan, LocalBuffersPlan) run unchanged
// through include/csrc_gpu.hpp on the B200 and agree with the reference CPU
// results. Built by oracle/Makefile against /root/reference headers into
// oracle/_ref/dropin_test; run by tests/test_dropin_cpp.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "csrc/csrc.hpp"
#define CSRC_GPU_REFERENCE_TYPES  // the reference's Error / PhaseTimings / Strategy / plan types
#include "csrc_gpu.hpp"

using namespace csrc;

static double max_rel(const Vector& y, const Vector& r) {
    double num = 0, den = 0;
    for (size_t i = 0; i < r.size(); ++i) {
        num = std::max(num, std::abs(y[i] - r[i]));
        den = std::max(den, std::abs(r[i]));
    }
    return den == 0 ? num : num / den;
}

int main() {
    int fails = 0;
    double worst = 0;
    for (int i = 0; i < 12; ++i) {
        index_t n = 40 + 23 * i;
        CsrcMatrix c = csr_to_csrc(build_csr(generate_random_sym(n, 0.05 + 0.02 * (i % 4), 4242 + i, i % 3 == 0)));
        Vector x = bench_source_vector(n);
        Vector ref = spmv_csrc(c, x);
        worst = std::max(worst, max_rel(gpu::spmv_csrc(c, x), ref));
        worst = std::max(worst, max_rel(gpu::spmv_csrc_transpose(c, x), spmv_csrc_transpose(c, x)));
        for (AccumMethod acc : {AccumMethod::all_in_one, AccumMethod::per_buffer, AccumMethod::effective,
                                AccumMethod::interval}) {
            Strategy s{StrategyKind::local_buffers, acc, 3};
            gpu::ParallelSpmv ex(c, s);  // reference Strategy accepted unchanged
            worst = std::max(worst, max_rel(ex.apply(x), ref));
            if (ex.buffers_allocated() < 1) ++fails;
            gpu::ParallelSpmv ex2(c, s, LocalBuffersPlan::build(c, 3));
            worst = std::max(worst, max_rel(ex2.apply(x), ref));
        }
        ColorfulPlan cp = ColorfulPlan::build(c, 2);
        gpu::ParallelSpmv exc(c, Strategy{StrategyKind::colorful, AccumMethod::effective, 2}, cp);
        worst = std::max(worst, max_rel(exc.apply(x), ref));
        auto [y, t] = gpu::spmv_parallel(c, x, Strategy{StrategyKind::colorful, AccumMethod::effective, 2});
        worst = std::max(worst, max_rel(y, ref));
    }
    // construction on the GPU: bit-identical CSR and CSRC, reference types out
    for (int i = 0; i < 6; ++i) {
        TripletMatrix t = generate_random_sym(60 + 31 * i, 0.06, 99 + i, i % 2 == 0);
        CsrMatrix ref_csr = build_csr(t);
        CsrMatrix got_csr = gpu::build_csr(t);
        if (got_csr.row_ptr != ref_csr.row_ptr || got_csr.col_idx != ref_csr.col_idx ||
            got_csr.values != ref_csr.values)
            ++fails;
        CsrcMatrix ref_c = csr_to_csrc(ref_csr);
        CsrcMatrix got_c = gpu::csr_to_csrc(gpu::build_csr(t));
        if (got_c.ia != ref_c.ia || got_c.ja != ref_c.ja || got_c.ad != ref_c.ad || got_c.al != ref_c.al ||
            got_c.au != ref_c.au || got_c.value_symmetric != ref_c.value_symmetric)
            ++fails;
    }
    // rectangular products: decompose_rect + spmv_csrc_rect / ParallelSpmv(rect, s)
    {
        const index_t n = 120, extra = 17;
        TripletMatrix sq = generate_random_sym(n, 0.05, 7);
        TripletMatrix t;
        t.n_rows = n;
        t.n_cols = n + extra;
        t.entries = sq.entries;
        for (index_t i = 0; i < n; i += 3) t.add(i, n + (i % extra), 0.25 * (1 + i % 5));
        CsrMatrix full = build_csr(t);
        CsrcRectMatrix ref_r = decompose_rect(full);
        CsrcRectMatrix got_r = gpu::decompose_rect(full);
        if (got_r.m != ref_r.m || got_r.square.ja != ref_r.square.ja || got_r.square.al != ref_r.square.al ||
            got_r.rect.col_idx != ref_r.rect.col_idx || got_r.rect.values != ref_r.rect.values)
            ++fails;
        Vector x = bench_source_vector(n + extra);
        Vector ref = spmv_csrc_rect(ref_r, x);
        worst = std::max(worst, max_rel(gpu::spmv_csrc_rect(got_r, x), ref));
        gpu::ParallelSpmv ex(ref_r, Strategy{StrategyKind::local_buffers, AccumMethod::interval, 4});
        worst = std::max(worst, max_rel(ex.apply(x), ref));
    }
    // spmv_csr on the GPU against the reference's spmv_csr (kernels.hpp:7-22)
    {
        CsrMatrix full = build_csr(generate_random_sym(300, 0.04, 5));
        Vector x = bench_source_vector(300);
        worst = std::max(worst, max_rel(gpu::spmv_csr(full, x), spmv_csr(full, x)));
    }
    // every public ParallelSpmv member (parallel.hpp:153-226) against the reference executor
    {
        CsrcMatrix c = csr_to_csrc(build_csr(generate_random_sym(500, 0.03, 31)));
        Vector x = bench_source_vector(500);
        for (AccumMethod acc : {AccumMethod::effective, AccumMethod::interval}) {
            Strategy s{StrategyKind::local_buffers, acc, 4};
            ParallelSpmv ref_ex(c, s);
            gpu::ParallelSpmv ex(c, s);
            Vector y;
            ex.apply(x, y);  // void apply(const Vector&, Vector&) resizes y
            worst = std::max(worst, max_rel(y, ref_ex.apply(x)));
            csrc::PhaseTimings t = ex.last_timings();  // the reference's own type
            if (t.compute_max <= 0.0) ++fails;
            const Strategy& st = ex.strategy();  // the reference's own type
            if (st.kind != s.kind || st.accum != s.accum || st.p != s.p) ++fails;
            const LocalBuffersPlan& bp = ex.buffers_plan();
            const LocalBuffersPlan& rbp = ref_ex.buffers_plan();
            if (bp.partition.block_start != rbp.partition.block_start ||
                bp.partition.block_nnz != rbp.partition.block_nnz || bp.ranges.size() != rbp.ranges.size() ||
                bp.intervals.boundaries != rbp.intervals.boundaries ||
                bp.intervals.intervals.size() != rbp.intervals.intervals.size())
                ++fails;
            for (size_t q = 0; q < bp.ranges.size() && q < rbp.ranges.size(); ++q)
                if (bp.ranges[q].lo != rbp.ranges[q].lo || bp.ranges[q].hi != rbp.ranges[q].hi) ++fails;
            for (size_t q = 0; q < bp.intervals.intervals.size() && q < rbp.intervals.intervals.size(); ++q)
                if (bp.intervals.intervals[q].contributors != rbp.intervals.intervals[q].contributors) ++fails;
            if (ex.buffers_allocated() != ref_ex.buffers_allocated()) ++fails;
            if (!ex.colorful_plan().coloring.color.empty()) ++fails;
        }
        {
            Strategy s{StrategyKind::colorful, AccumMethod::effective, 3};
            ParallelSpmv ref_ex(c, s);
            gpu::ParallelSpmv ex(c, s);
            worst = std::max(worst, max_rel(ex.apply(x), ref_ex.apply(x)));
            const ColorfulPlan& cp = ex.colorful_plan();
            const ColorfulPlan& rcp = ref_ex.colorful_plan();
            if (cp.coloring.color != rcp.coloring.color || cp.coloring.n_colors != rcp.coloring.n_colors ||
                cp.coloring.classes != rcp.coloring.classes || cp.class_slices != rcp.class_slices)
                ++fails;
            if (!validate_coloring(c, cp.coloring).valid) ++fails;
            if (ex.buffers_allocated() != 0 || !ex.buffers_plan().partition.block_start.empty()) ++fails;
        }
        {   // sequential: no plans, no buffers (parallel.hpp:197-202)
            gpu::ParallelSpmv ex(c, Strategy{});
            worst = std::max(worst, max_rel(ex.apply(x), spmv_csrc(c, x)));
            if (ex.buffers_allocated() != 0 || ex.strategy().kind != StrategyKind::sequential) ++fails;
        }
    }
    // rectangular + explicit plan constructors (parallel.hpp:173-181)
    {
        const index_t n = 150, extra = 9;
        TripletMatrix t = generate_random_sym(n, 0.05, 77);
        t.n_cols = n + extra;
        for (index_t i = 0; i < n; i += 2) t.add(i, n + (i % extra), -0.5 + 0.1 * (i % 7));
        CsrcRectMatrix r = decompose_rect(build_csr(t));
        Vector x = bench_source_vector(n + extra);
        Vector ref = spmv_csrc_rect(r, x);
        Strategy sl{StrategyKind::local_buffers, AccumMethod::interval, 3};
        gpu::ParallelSpmv e1(r, sl, LocalBuffersPlan::build(r.square, 3));
        worst = std::max(worst, max_rel(e1.apply(x), ref));
        if (e1.buffers_plan().partition.p != 3) ++fails;
        Strategy sc{StrategyKind::colorful, AccumMethod::effective, 2};
        ColorfulPlan cp = ColorfulPlan::build(r.square, 2);
        gpu::ParallelSpmv e2(r, sc, cp);
        worst = std::max(worst, max_rel(e2.apply(x), ref));
        if (e2.colorful_plan().coloring.color != cp.coloring.color) ++fails;
        ParallelSpmv ref_e2(r, sc, cp);
        worst = std::max(worst, max_rel(e2.apply(x), ref_e2.apply(x)));
    }
    // error behaviour: the reference's csrc::Error with its wording
    try {
        CsrcMatrix c = csr_to_csrc(build_csr(generate_band(10, 1)));
        gpu::spmv_csrc(c, Vector(3));
        ++fails;
    } catch (const csrc::Error& e) {
        if (std::string(e.what()).find("x has length 3, expected 10") == std::string::npos) ++fails;
    }
    try {
        CsrcMatrix c = csr_to_csrc(build_csr(generate_band(10, 1)));
        gpu::ParallelSpmv ex(c, Strategy{StrategyKind::sequential, AccumMethod::effective, 2});
        ++fails;
    } catch (const csrc::Error& e) {
        if (std::string(e.what()).find("sequential strategy requires p = 1") == std::string::npos) ++fails;
    }
    // multi-GPU band executor wrapper (one rank: the band is the whole matrix). NCCL is
    // loaded at run time by the library (whichever libnccl.so.2 the process finds); a plain
    // C++ process binds the system NCCL, whose bootstrap does not come up in every sandbox
    // (it took a minute to fail on the test pool), so this part runs on request only:
    // CSRC_DROPIN_BAND=1. The same executor is run through torch's NCCL by
    // tests/test_gpu_bandexec.py; here the wrapper is always compiled.
    if (std::getenv("CSRC_DROPIN_BAND")) {
        CsrcMatrix c = csr_to_csrc(build_csr(generate_random_sym(200, 0.05, 11)));
        uint8_t id[128] = {};
        bool have_nccl = true;
        try {
            gpu::BandSpmv::unique_id(id);
        } catch (const csrc::Error& e) {
            have_nccl = false;
            std::printf("dropin: band executor skipped (%s)\n", e.what());
        }
        if (have_nccl) {
            for (auto form : {gpu::BandSpmv::Form::windowed, gpu::BandSpmv::Form::gather}) {
                gpu::BandSpmv band(c, form == gpu::BandSpmv::Form::windowed ? gpu::Strategy::windowed()
                                                                             : gpu::Strategy::gather(),
                                   1, 0, id, form);
                const csrc_gpu_band_lists& L = band.lists();
                if (L.row_begin != 0 || L.row_end != static_cast<int32_t>(c.n) || L.n_sends != 0 || L.n_recvs != 0)
                    ++fails;
                band.check_comm();
            }
        }
    }
    std::printf("dropin: max rel err %.3e, failures %d\n", worst, fails);
    return (worst <= 1e-12 && fails == 0) ? 0 : 1;
}

// csrc_gpu.hpp — header-only C++ drop-in for the reference's CSRC hot path.
//
// The reference (csrc-spmv, /root/reference/proj/include/csrc) is header-only
// C++20; its hot-path API is
//     csrc::Vector csrc::spmv_csrc(const CsrcMatrix&, const Vector&)     kernels.hpp:25
//     csrc::Vector csrc::spmv_csrc_transpose(const CsrcMatrix&, const Vector&) kernels.hpp:47
//     csrc::ParallelSpmv exec(a, Strategy{kind, accum, p}); exec.apply(x) parallel.hpp:151-226
//     csrc::spmv_parallel(a, x, s)                                        parallel.hpp:449-454
// This header provides the same call shapes in namespace csrc::gpu, backed by
// the B200 kernels through the C ABI (csrc_gpu.h, libcsrc_b200.so). It is a
// template over the matrix / strategy / plan types, so the reference's own
// csrc::CsrcMatrix, csrc::Strategy, csrc::LocalBuffersPlan and
// csrc::ColorfulPlan are accepted unchanged:
//
//     #include <csrc/csrc.hpp>          // reference
//     #define CSRC_GPU_REFERENCE_TYPES   // optional: the reference's own Error, PhaseTimings,
//                                        // Strategy, LocalBuffersPlan, ColorfulPlan types in and out
//     #include <csrc_gpu.hpp>
//     csrc::Vector y = csrc::gpu::spmv_csrc(c, x);
//     csrc::gpu::ParallelSpmv exec(c, csrc::Strategy{csrc::StrategyKind::local_buffers,
//                                                    csrc::AccumMethod::effective, 4});
//     csrc::Vector y2 = exec.apply(x);
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "csrc_gpu.h"

namespace csrc {
namespace gpu {

#if defined(CSRC_GPU_REFERENCE_TYPES) && !defined(CSRC_GPU_ERROR_TYPE)
#define CSRC_GPU_ERROR_TYPE ::csrc::Error
#endif

#ifdef CSRC_GPU_ERROR_TYPE
using Error = CSRC_GPU_ERROR_TYPE;
#else
/// Mirrors csrc::Error (common.hpp:15-18).
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
#endif

using Vector = std::vector<double>;

inline void check(int rc) {
    if (rc != 0) throw Error(csrc_gpu_last_error());
}

/// GPU strategy: csrc::Strategy {kind, accum, p} plus device options. The
/// integer values of StrategyKind / AccumMethod match the reference enums.
struct Strategy {
    int kind = CSRC_KIND_SEQUENTIAL;
    int accum = CSRC_ACCUM_EFFECTIVE;
    int p = 1;
    int dtype = CSRC_DTYPE_F64;
    int conflict_mode = CSRC_CONFLICT_NEIGHBORHOOD;
    int color_order = CSRC_ORDER_NATURAL;
    int device = 0;
    int bands = 0;

    Strategy() = default;
    Strategy(int k, int a, int p_) : kind(k), accum(a), p(p_) {}
    /// Converts a reference csrc::Strategy (or anything with kind/accum/p).
    template <class S, class = decltype(std::declval<S>().kind)>
    Strategy(const S& s)  // NOLINT(google-explicit-constructor): drop-in
        : kind(static_cast<int>(s.kind)), accum(static_cast<int>(s.accum)), p(s.p) {}

    static Strategy windowed() { return Strategy(CSRC_KIND_WINDOWED, CSRC_ACCUM_EFFECTIVE, 1); }
    static Strategy atomic() { return Strategy(CSRC_KIND_ATOMIC, CSRC_ACCUM_EFFECTIVE, 1); }
    static Strategy gather() { return Strategy(CSRC_KIND_GATHER, CSRC_ACCUM_EFFECTIVE, 1); }

    csrc_gpu_strategy c() const {
        return csrc_gpu_strategy{kind, accum, p, dtype, conflict_mode, color_order, device, bands};
    }
};

#ifdef CSRC_GPU_REFERENCE_TYPES
/// The reference's own csrc::PhaseTimings (parallel.hpp:26-30), so that
/// `csrc::PhaseTimings t = exec.last_timings();` compiles unchanged.
using PhaseTimings = ::csrc::PhaseTimings;
using StrategyOut = ::csrc::Strategy;
using BuffersPlanOut = ::csrc::LocalBuffersPlan;
using ColorfulPlanOut = ::csrc::ColorfulPlan;
#else
/// csrc::PhaseTimings (parallel.hpp:26-30), seconds.
struct PhaseTimings {
    double init_max = 0.0;
    double compute_max = 0.0;
    double accumulate_max = 0.0;
};
/// The plan a local-buffers executor runs (csrc::LocalBuffersPlan shape,
/// parallel.hpp:40-52): partition, effective ranges, interval plan.
struct BuffersPlanOut {
    struct Partition {
        int p = 1;
        std::vector<int32_t> block_start;
        std::vector<int64_t> block_nnz;
    } partition;
    struct Range {
        int32_t lo = 0, hi = 0;
    };
    std::vector<Range> ranges;
    struct Intervals {
        struct Interval {
            int32_t begin = 0, end = 0;
            std::vector<int> contributors;
        };
        std::vector<int32_t> boundaries;
        std::vector<Interval> intervals;
    } intervals;
};
/// The colouring a colorful executor runs (csrc::ColorfulPlan shape,
/// parallel.hpp:54-94).
struct ColorfulPlanOut {
    struct Coloring {
        std::vector<int> color;
        int n_colors = 0;
        std::vector<std::vector<int32_t>> classes;
    } coloring;
    std::vector<std::vector<std::pair<std::size_t, std::size_t>>> class_slices;
};
using StrategyOut = Strategy;
#endif

/// Borrowed C view of any CsrcMatrix-shaped type (csrc_matrix.hpp:14-30).
template <class M>
csrc_host_matrix view(const M& a) {
    csrc_host_matrix m;
    m.n = a.n;
    m.k = static_cast<int64_t>(a.ja.size());
    m.ad = a.ad.data();
    m.ia = a.ia.data();
    m.ja = a.ja.data();
    m.al = a.al.data();
    m.au = a.value_symmetric ? nullptr : a.au.data();
    m.value_symmetric = a.value_symmetric ? 1 : 0;
    return m;
}

template <class P, class = void>
struct has_square : std::false_type {};
template <class P>
struct has_square<P, std::void_t<decltype(std::declval<P>().square)>> : std::true_type {};

namespace detail {
template <class P, class = void>
struct has_coloring : std::false_type {};
template <class P>
struct has_coloring<P, std::void_t<decltype(std::declval<P>().coloring)>> : std::true_type {};

template <class S>
StrategyOut strategy_out(const S& s) {
#ifdef CSRC_GPU_REFERENCE_TYPES
    StrategyOut o;
    o.kind = static_cast<decltype(o.kind)>(static_cast<int>(s.kind));
    o.accum = static_cast<decltype(o.accum)>(static_cast<int>(s.accum));
    o.p = s.p;
    return o;
#else
    return Strategy(s);
#endif
}

/// LocalBuffersPlan::build (parallel.hpp:45-51) through the product's plan
/// functions (bit-exact with partition.hpp:55-134).
inline BuffersPlanOut build_buffers_plan(const csrc_host_matrix& m, int p) {
    BuffersPlanOut plan;
    std::vector<int32_t> bs(static_cast<size_t>(p) + 1);
    std::vector<int64_t> bn(static_cast<size_t>(p));
    check(csrc_partition_by_nnz(&m, p, bs.data(), bn.data()));
    plan.partition.p = p;
    plan.partition.block_start.assign(bs.begin(), bs.end());
    plan.partition.block_nnz.assign(bn.begin(), bn.end());
    std::vector<int32_t> lo(static_cast<size_t>(p)), hi(static_cast<size_t>(p));
    check(csrc_effective_ranges(&m, p, bs.data(), lo.data(), hi.data()));
    plan.ranges.resize(static_cast<size_t>(p));
    for (int t = 0; t < p; ++t) {
        plan.ranges[t].lo = lo[t];
        plan.ranges[t].hi = hi[t];
    }
    int32_t ni = 0, nc = 0, nb = 0;
    check(csrc_interval_plan(p, lo.data(), hi.data(), &ni, &nc, &nb, nullptr, nullptr, nullptr, nullptr, nullptr));
    std::vector<int32_t> ib(ni + 1), ie(ni + 1), cp(ni + 1), cc(nc + 1), bd(nb + 1);
    check(csrc_interval_plan(p, lo.data(), hi.data(), &ni, &nc, &nb, ib.data(), ie.data(), cp.data(), cc.data(),
                             bd.data()));
    plan.intervals.boundaries.assign(bd.begin(), bd.begin() + nb);
    plan.intervals.intervals.resize(static_cast<size_t>(ni));
    for (int i = 0; i < ni; ++i) {
        auto& iv = plan.intervals.intervals[i];
        iv.begin = ib[i];
        iv.end = ie[i];
        iv.contributors.assign(cc.begin() + cp[i], cc.begin() + cp[i + 1]);
    }
    return plan;
}

/// ColorfulPlan (parallel.hpp:54-94) of the colouring a GPU plan runs, sliced
/// for p workers (ColorfulPlan::slice, parallel.hpp:69-93).
inline ColorfulPlanOut colorful_plan_of(csrc_gpu_plan_t plan, const csrc_host_matrix& m, int p) {
    ColorfulPlanOut out;
    int32_t nc = 0;
    check(csrc_gpu_plan_get_coloring(plan, nullptr, &nc));
    std::vector<int32_t> color(static_cast<size_t>(m.n));
    check(csrc_gpu_plan_get_coloring(plan, color.data(), &nc));
    out.coloring.color.assign(color.begin(), color.end());
    out.coloring.n_colors = nc;
    out.coloring.classes.assign(static_cast<size_t>(nc), {});
    for (int32_t i = 0; i < m.n; ++i) out.coloring.classes[color[i]].push_back(i);
    std::vector<int64_t> sl(static_cast<size_t>(std::max(nc, 1)) * p * 2);
    check(csrc_colorful_slices(&m, color.data(), nc, p, sl.data()));
    out.class_slices.assign(static_cast<size_t>(nc), std::vector<std::pair<std::size_t, std::size_t>>(p));
    for (int c = 0; c < nc; ++c)
        for (int t = 0; t < p; ++t)
            out.class_slices[c][t] = {static_cast<std::size_t>(sl[(static_cast<size_t>(c) * p + t) * 2]),
                                      static_cast<std::size_t>(sl[(static_cast<size_t>(c) * p + t) * 2 + 1])};
    return out;
}

template <class Plan>
BuffersPlanOut buffers_plan_copy(const Plan& plan) {
    if constexpr (std::is_same<Plan, BuffersPlanOut>::value) {
        return plan;
    } else {
        BuffersPlanOut o;
        o.partition.p = plan.partition.p;
        o.partition.block_start.assign(plan.partition.block_start.begin(), plan.partition.block_start.end());
        o.partition.block_nnz.assign(plan.partition.block_nnz.begin(), plan.partition.block_nnz.end());
        o.ranges.resize(plan.ranges.size());
        for (size_t t = 0; t < plan.ranges.size(); ++t) {
            o.ranges[t].lo = plan.ranges[t].lo;
            o.ranges[t].hi = plan.ranges[t].hi;
        }
        o.intervals.boundaries.assign(plan.intervals.boundaries.begin(), plan.intervals.boundaries.end());
        o.intervals.intervals.resize(plan.intervals.intervals.size());
        for (size_t i = 0; i < plan.intervals.intervals.size(); ++i) {
            o.intervals.intervals[i].begin = plan.intervals.intervals[i].begin;
            o.intervals.intervals[i].end = plan.intervals.intervals[i].end;
            o.intervals.intervals[i].contributors.assign(plan.intervals.intervals[i].contributors.begin(),
                                                         plan.intervals.intervals[i].contributors.end());
        }
        return o;
    }
}

template <class Plan>
ColorfulPlanOut colorful_plan_copy(const Plan& plan) {
    if constexpr (std::is_same<Plan, ColorfulPlanOut>::value) {
        return plan;
    } else {
        ColorfulPlanOut o;
        o.coloring.color.assign(plan.coloring.color.begin(), plan.coloring.color.end());
        o.coloring.n_colors = plan.coloring.n_colors;
        o.coloring.classes.resize(plan.coloring.classes.size());
        for (size_t c = 0; c < plan.coloring.classes.size(); ++c)
            o.coloring.classes[c].assign(plan.coloring.classes[c].begin(), plan.coloring.classes[c].end());
        o.class_slices.resize(plan.class_slices.size());
        for (size_t c = 0; c < plan.class_slices.size(); ++c)
            for (const auto& pr : plan.class_slices[c])
                o.class_slices[c].emplace_back(static_cast<std::size_t>(pr.first), static_cast<std::size_t>(pr.second));
        return o;
    }
}
}  // namespace detail

/// GPU counterpart of csrc::ParallelSpmv (parallel.hpp:151-446): the same
/// constructors (matrix or CsrcRectMatrix, Strategy, optional LocalBuffersPlan /
/// ColorfulPlan, parallel.hpp:153-181), apply (:183-220), last_timings,
/// buffers_allocated, strategy, buffers_plan, colorful_plan (:222-226). Unlike
/// the reference it copies the matrix to the device, so `a` may be freed.
class ParallelSpmv {
public:
    template <class M, class S, std::enable_if_t<!has_square<M>::value, int> = 0>
    ParallelSpmv(const M& a, const S& s) : n_(a.n), x_len_(a.n), strategy_(detail::strategy_out(s)) {
        const csrc_host_matrix m = view(a);
        const csrc_gpu_strategy st = Strategy(s).c();
        check(csrc_gpu_plan_create(&m, &st, &plan_));
        default_plans(m, st);
    }

    /// ParallelSpmv(const CsrcRectMatrix&, Strategy) (parallel.hpp:168-171):
    /// any type with .square (CSRC), .rect (CSR tail, local columns) and .m.
    template <class R, class S, std::enable_if_t<has_square<R>::value, int> = 0>
    ParallelSpmv(const R& r, const S& s)
        : n_(r.square.n), x_len_(static_cast<int64_t>(r.m)), strategy_(detail::strategy_out(s)) {
        const csrc_host_matrix m = view(r.square);
        const csrc_gpu_strategy st = Strategy(s).c();
        std::vector<int32_t> rp(r.rect.row_ptr.begin(), r.rect.row_ptr.end());
        std::vector<int32_t> ci(r.rect.col_idx.begin(), r.rect.col_idx.end());
        check(csrc_gpu_plan_create_rect(&m, &st, static_cast<int32_t>(r.m), rp.data(), ci.data(),
                                        r.rect.values.data(), &plan_));
        default_plans(m, st);
    }

    /// Explicit plan: a ColorfulPlan (has .coloring) or a LocalBuffersPlan (has
    /// .partition), parallel.hpp:158-166; with a CsrcRectMatrix, :173-181.
    template <class M, class S, class Plan>
    ParallelSpmv(const M& a, const S& s, const Plan& plan) : strategy_(detail::strategy_out(s)) {
        const csrc_gpu_strategy st = Strategy(s).c();
        std::vector<int32_t> color, starts;
        const int32_t* cp = nullptr;
        const int32_t* bp = nullptr;
        int32_t nc = 0, bands = 0;
        if constexpr (detail::has_coloring<Plan>::value) {
            color.assign(plan.coloring.color.begin(), plan.coloring.color.end());
            cp = color.data();
            nc = plan.coloring.n_colors;
            color_plan_ = detail::colorful_plan_copy(plan);
        } else {
            starts.assign(plan.partition.block_start.begin(), plan.partition.block_start.end());
            bp = starts.data();
            bands = plan.partition.p;
            buf_plan_ = detail::buffers_plan_copy(plan);
        }
        if constexpr (has_square<M>::value) {
            n_ = a.square.n;
            x_len_ = static_cast<int64_t>(a.m);
            const csrc_host_matrix m = view(a.square);
            std::vector<int32_t> rp(a.rect.row_ptr.begin(), a.rect.row_ptr.end());
            std::vector<int32_t> ci(a.rect.col_idx.begin(), a.rect.col_idx.end());
            check(csrc_gpu_plan_create_rect_plan(&m, &st, static_cast<int32_t>(a.m), rp.data(), ci.data(),
                                                 a.rect.values.data(), cp, nc, bp, bands, &plan_));
        } else {
            n_ = a.n;
            x_len_ = a.n;
            const csrc_host_matrix m = view(a);
            if (cp)
                check(csrc_gpu_plan_create_colored(&m, &st, cp, nc, &plan_));
            else
                check(csrc_gpu_plan_create_partitioned(&m, &st, bp, bands, &plan_));
        }
    }

    ParallelSpmv(const ParallelSpmv&) = delete;
    ParallelSpmv& operator=(const ParallelSpmv&) = delete;
    ParallelSpmv(ParallelSpmv&& o) noexcept
        : plan_(o.plan_), n_(o.n_), x_len_(o.x_len_), timings_(o.timings_), strategy_(std::move(o.strategy_)),
          buf_plan_(std::move(o.buf_plan_)), color_plan_(std::move(o.color_plan_)) {
        o.plan_ = nullptr;
    }
    ~ParallelSpmv() { csrc_gpu_plan_destroy(plan_); }

    Vector apply(const Vector& x) {
        Vector y(static_cast<size_t>(n_));
        apply(x, y);
        return y;
    }

    void apply(const Vector& x, Vector& y) {
        y.resize(static_cast<size_t>(n_));
        check(csrc_gpu_set_timing(plan_, 1));
        check(csrc_gpu_spmv(plan_, x.data(), static_cast<int64_t>(x.size()), y.data()));
        csrc_gpu_timings t;
        check(csrc_gpu_last_timings(plan_, &t));
        timings_ = PhaseTimings{};
        timings_.init_max = t.init_ms / 1e3;
        timings_.compute_max = t.compute_ms / 1e3;
        timings_.accumulate_max = t.accumulate_ms / 1e3;
    }

    Vector apply_transpose(const Vector& x) {
        Vector y(static_cast<size_t>(n_));
        check(csrc_gpu_spmv_transpose(plan_, x.data(), static_cast<int64_t>(x.size()), y.data()));
        return y;
    }

    /// Device pointers on a CUDA stream (throughput form, asynchronous).
    void apply_device(const void* d_x, void* d_y, void* stream = nullptr) {
        check(csrc_gpu_spmv_device(plan_, d_x, d_y, stream, 0));
    }

    const PhaseTimings& last_timings() const { return timings_; }

    int buffers_allocated() const {
        csrc_gpu_plan_info info;
        check(csrc_gpu_plan_get_info(plan_, &info));
        return info.buffers_allocated;
    }

    /// parallel.hpp:224-226
    const StrategyOut& strategy() const { return strategy_; }
    const BuffersPlanOut& buffers_plan() const { return buf_plan_; }
    const ColorfulPlanOut& colorful_plan() const { return color_plan_; }

    csrc_gpu_plan_info info() const {
        csrc_gpu_plan_info i;
        check(csrc_gpu_plan_get_info(plan_, &i));
        return i;
    }

private:
    // the plans the reference's build_default_plan (parallel.hpp:236-242) would
    // hold: local buffers / colorful with p >= 2 only
    void default_plans(const csrc_host_matrix& m, const csrc_gpu_strategy& st) {
        if (st.p < 2) return;
        if (st.kind == CSRC_KIND_LOCAL_BUFFERS) buf_plan_ = detail::build_buffers_plan(m, st.p);
        if (st.kind == CSRC_KIND_COLORFUL) color_plan_ = detail::colorful_plan_of(plan_, m, st.p);
    }

    csrc_gpu_plan_t plan_ = nullptr;
    int32_t n_ = 0;
    int64_t x_len_ = 0;
    PhaseTimings timings_{};
    StrategyOut strategy_{};
    BuffersPlanOut buf_plan_{};
    ColorfulPlanOut color_plan_{};
};

/// spmv_csrc (kernels.hpp:25-43) on the GPU.
/// One shot, no plan: the CSRC arrays stream to the device as stored
/// (csrc_gpu_spmv_oneshot); repeated products should keep a ParallelSpmv.
template <class M>
Vector spmv_csrc(const M& a, const Vector& x) {
    if (static_cast<long long>(x.size()) != a.n)
        throw Error("spmv_csrc: x has length " + std::to_string(x.size()) + ", expected " +
                    std::to_string(a.n));
    const csrc_host_matrix m = view(a);
    Vector y(static_cast<size_t>(a.n));
    check(csrc_gpu_spmv_oneshot(&m, x.data(), static_cast<int64_t>(x.size()), y.data(), 0, 0));
    return y;
}

/// spmv_csrc_transpose (kernels.hpp:47-65) on the GPU.
template <class M>
Vector spmv_csrc_transpose(const M& a, const Vector& x) {
    if (static_cast<long long>(x.size()) != a.n)
        throw Error("spmv_csrc_transpose: x has length " + std::to_string(x.size()) +
                    ", expected " + std::to_string(a.n));
    const csrc_host_matrix m = view(a);
    Vector y(static_cast<size_t>(a.n));
    check(csrc_gpu_spmv_oneshot(&m, x.data(), static_cast<int64_t>(x.size()), y.data(), 1, 0));
    return y;
}

/// spmv_parallel (parallel.hpp:449-454).
template <class M, class S>
std::pair<Vector, PhaseTimings> spmv_parallel(const M& a, const Vector& x, const S& s) {
    ParallelSpmv ex(a, s);
    Vector y = ex.apply(x);
    return {std::move(y), ex.last_timings()};
}

/// spmv_csr (kernels.hpp:7-22) on the GPU: any CsrMatrix-shaped type
/// (n_rows, n_cols, row_ptr, col_idx, values).
template <class M>
Vector spmv_csr(const M& a, const Vector& x) {
    if (static_cast<long long>(x.size()) != static_cast<long long>(a.n_cols))
        throw Error("spmv_csr: x has length " + std::to_string(x.size()) + ", expected " +
                    std::to_string(a.n_cols));
    std::vector<int32_t> rp(a.row_ptr.begin(), a.row_ptr.end());
    std::vector<int32_t> ci(a.col_idx.begin(), a.col_idx.end());
    const csrc_gpu_strategy st = Strategy().c();
    csrc_gpu_plan_t plan = nullptr;
    check(csrc_gpu_plan_create_csr(static_cast<int32_t>(a.n_rows), static_cast<int32_t>(a.n_cols), rp.data(),
                                   ci.data(), a.values.data(), &st, &plan));
    Vector y(static_cast<size_t>(a.n_rows));
    const int rc = csrc_gpu_spmv(plan, x.data(), static_cast<int64_t>(x.size()), y.data());
    csrc_gpu_plan_destroy(plan);
    check(rc);
    return y;
}

/// spmv_csrc_rect (kernels.hpp:69-91) on the GPU: x has r.m entries.
template <class R>
Vector spmv_csrc_rect(const R& r, const Vector& x) {
    if (static_cast<long long>(x.size()) != static_cast<long long>(r.m))
        throw Error("spmv_csrc_rect: x has length " + std::to_string(x.size()) + ", expected " +
                    std::to_string(r.m));
    ParallelSpmv ex(r, Strategy());
    return ex.apply(x);
}

// ------------------------------------------------------------ construction
// build_csr / csr_to_csrc / decompose_rect on the GPU (assemble.cu). The
// results convert to the caller's own CsrMatrix / CsrcMatrix /
// CsrcRectMatrix types (anything with the reference's member names), so
//     csrc::CsrcMatrix c = csrc::gpu::csr_to_csrc(csrc::gpu::build_csr(t));
// is a drop-in for csrc::csr_to_csrc(csrc::build_csr(t)) (csr.hpp:55-92,
// csrc_matrix.hpp:44-91), bit-identical results.

/// Canonical CSR (csrc::CsrMatrix shape, csr.hpp:28-51).
struct CsrResult {
    int32_t n_rows = 0, n_cols = 0;
    std::vector<int32_t> row_ptr, col_idx;
    std::vector<double> values;
    template <class C>
    operator C() const {  // NOLINT(google-explicit-constructor): drop-in
        C c;
        c.n_rows = n_rows;
        c.n_cols = n_cols;
        c.row_ptr.assign(row_ptr.begin(), row_ptr.end());
        c.col_idx.assign(col_idx.begin(), col_idx.end());
        c.values.assign(values.begin(), values.end());
        return c;
    }
};

/// CSRC (csrc::CsrcMatrix shape, csrc_matrix.hpp:14-30).
struct CsrcResult {
    int32_t n = 0;
    std::vector<double> ad;
    std::vector<int32_t> ia, ja;
    std::vector<double> al, au;
    bool value_symmetric = false;
    template <class C>
    operator C() const {  // NOLINT(google-explicit-constructor): drop-in
        C c;
        c.n = n;
        c.ad.assign(ad.begin(), ad.end());
        c.ia.assign(ia.begin(), ia.end());
        c.ja.assign(ja.begin(), ja.end());
        c.al.assign(al.begin(), al.end());
        c.au.assign(au.begin(), au.end());
        c.value_symmetric = value_symmetric;
        return c;
    }
};

/// csrc::CsrcRectMatrix shape (csrc_matrix.hpp:35-39).
struct CsrcRectResult {
    CsrcResult square;
    CsrResult rect;
    int32_t m = 0;
    template <class C>
    operator C() const {  // NOLINT(google-explicit-constructor): drop-in
        C c;
        c.square = square;
        c.rect = rect;
        c.m = m;
        return c;
    }
};

namespace detail {
struct Built {
    csrc_built_t h = nullptr;
    ~Built() { csrc_built_free(h); }
};
inline CsrcResult take_csrc(csrc_built_t h) {
    csrc_host_matrix m;
    check(csrc_built_matrix(h, &m));
    CsrcResult c;
    c.n = m.n;
    c.ad.assign(m.ad, m.ad + m.n);
    c.ia.assign(m.ia, m.ia + m.n + 1);
    c.ja.assign(m.ja, m.ja + m.k);
    c.al.assign(m.al, m.al + m.k);
    if (!m.value_symmetric) c.au.assign(m.au, m.au + m.k);
    c.value_symmetric = m.value_symmetric != 0;
    return c;
}
template <class M>
void csr_arrays(const M& a, std::vector<int32_t>& rp, std::vector<int32_t>& ci) {
    rp.assign(a.row_ptr.begin(), a.row_ptr.end());
    ci.assign(a.col_idx.begin(), a.col_idx.end());
}
}  // namespace detail

/// build_csr (csr.hpp:55-92): t is a csrc::TripletMatrix (n_rows, n_cols,
/// entries {row, col, value}). Duplicates summed in input order.
template <class T>
CsrResult build_csr(const T& t, int device = 0) {
    std::vector<int32_t> r, c;
    std::vector<double> v;
    r.reserve(t.entries.size());
    c.reserve(t.entries.size());
    v.reserve(t.entries.size());
    for (const auto& e : t.entries) {
        r.push_back(e.row);
        c.push_back(e.col);
        v.push_back(e.value);
    }
    detail::Built b;
    check(csrc_gpu_build_csr(t.n_rows, t.n_cols, static_cast<int64_t>(v.size()), r.data(), c.data(), v.data(),
                             device, &b.h));
    int32_t nr = 0, nc = 0;
    int64_t nnz = 0;
    const int32_t *rp = nullptr, *ci = nullptr;
    const double* va = nullptr;
    check(csrc_built_csr(b.h, &nr, &nc, &nnz, &rp, &ci, &va));
    CsrResult out;
    out.n_rows = nr;
    out.n_cols = nc;
    out.row_ptr.assign(rp, rp + nr + 1);
    out.col_idx.assign(ci, ci + nnz);
    out.values.assign(va, va + nnz);
    return out;
}

/// csr_to_csrc (csrc_matrix.hpp:44-91) of a canonical CSR.
template <class M>
CsrcResult csr_to_csrc(const M& a, int device = 0) {
    std::vector<int32_t> rp, ci;
    detail::csr_arrays(a, rp, ci);
    detail::Built b;
    check(csrc_gpu_csr_to_csrc(a.n_rows, a.n_cols, rp.data(), ci.data(), a.values.data(), device, &b.h));
    return detail::take_csrc(b.h);
}

/// decompose_rect (csrc_matrix.hpp:113-142, symmetrize = false).
template <class M>
CsrcRectResult decompose_rect(const M& a, int device = 0) {
    std::vector<int32_t> rp, ci;
    detail::csr_arrays(a, rp, ci);
    detail::Built b;
    check(csrc_gpu_decompose_rect(a.n_rows, a.n_cols, rp.data(), ci.data(), a.values.data(), device, &b.h));
    CsrcRectResult r;
    r.square = detail::take_csrc(b.h);
    int32_t m = 0;
    int64_t nnz = 0;
    const int32_t *trp = nullptr, *tci = nullptr;
    const double* tva = nullptr;
    check(csrc_built_rect_tail(b.h, &m, &nnz, &trp, &tci, &tva));
    r.m = m;
    r.rect.n_rows = r.square.n;
    r.rect.n_cols = m - r.square.n;
    r.rect.row_ptr.assign(trp, trp + r.square.n + 1);
    r.rect.col_idx.assign(tci, tci + nnz);
    r.rect.values.assign(tva, tva + nnz);
    return r;
}

/// Multi-GPU band executor (csrc_gpu_band_exec_*, csrc_gpu.h): one per rank, one
/// process per GPU. Rank `rank` of `world` owns a partition_by_nnz row band
/// (partition.hpp:55-90); apply() runs the band product with its exchange over
/// NCCL -- the windowed form's y-halo reduce into the owning ranks (the
/// `effective` accumulation, parallel.hpp:371-382, at GPU granularity) or the
/// gather form's x-halo refresh -- overlapped with the interior rows.
///
///     std::array<uint8_t, 128> id{};
///     if (rank == 0) csrc::gpu::BandSpmv::unique_id(id.data());   // then broadcast id
///     csrc::gpu::BandSpmv band(c, csrc::gpu::Strategy::windowed(), world, rank, id.data());
///     band.apply(d_x, d_y, stream);       // x covers [x_lo, x_hi), y [y_lo, row_end)
class BandSpmv {
public:
    enum class Form { windowed = CSRC_BAND_WINDOWED, gather = CSRC_BAND_GATHER };

    /// ncclGetUniqueId on one rank (id: 128 bytes); the caller broadcasts it.
    static void unique_id(uint8_t* id) { check(csrc_gpu_nccl_get_unique_id(id)); }

    template <class M, class S>
    BandSpmv(const M& a, const S& s, int world, int rank, const uint8_t* nccl_id, Form form = Form::windowed) {
        const csrc_host_matrix m = view(a);
        const csrc_gpu_strategy st = Strategy(s).c();
        check(csrc_gpu_band_exec_create(&m, &st, world, rank, static_cast<int32_t>(form), nccl_id, &ex_));
        check(csrc_gpu_band_exec_get_info(ex_, &lists_));
    }
    BandSpmv(const BandSpmv&) = delete;
    BandSpmv& operator=(const BandSpmv&) = delete;
    ~BandSpmv() {
        if (ex_) csrc_gpu_band_exec_destroy(ex_);
    }

    /// Owned rows, the x / y ranges of the device vectors, messages per product.
    const csrc_gpu_band_lists& lists() const { return lists_; }

    /// y = A x on the band, exchange included, enqueued on `stream`
    /// (refresh_x: the gather form's x-halo exchange before the boundary rows).
    void apply(const void* d_x, void* d_y, void* stream = nullptr, bool refresh_x = false) {
        check(csrc_gpu_band_exec_apply(ex_, d_x, d_y, stream, refresh_x ? 1 : 0));
    }

    /// ncclCommGetAsyncError: throws (communicator aborted) after a failure.
    void check_comm() { check(csrc_gpu_band_exec_check(ex_)); }

private:
    csrc_gpu_band_exec_t ex_ = nullptr;
    csrc_gpu_band_lists lists_{};
};

}  // namespace gpu
}  // namespace csrc

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
//     #define CSRC_GPU_ERROR_TYPE csrc::Error   // optional: throw the reference's error type
//     #include <csrc_gpu.hpp>
//     csrc::Vector y = csrc::gpu::spmv_csrc(c, x);
//     csrc::gpu::ParallelSpmv exec(c, csrc::Strategy{csrc::StrategyKind::local_buffers,
//                                                    csrc::AccumMethod::effective, 4});
//     csrc::Vector y2 = exec.apply(x);
#pragma once

#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "csrc_gpu.h"

namespace csrc {
namespace gpu {

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

/// csrc::PhaseTimings (parallel.hpp:26-30), seconds.
struct PhaseTimings {
    double init_max = 0.0;
    double compute_max = 0.0;
    double accumulate_max = 0.0;
};

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

/// GPU counterpart of csrc::ParallelSpmv (parallel.hpp:151-446). Unlike the
/// reference it copies the matrix (device-resident), so `a` may be freed.
class ParallelSpmv {
public:
    template <class M, class S, std::enable_if_t<!has_square<M>::value, int> = 0>
    ParallelSpmv(const M& a, const S& s) : n_(a.n) {
        const csrc_host_matrix m = view(a);
        const csrc_gpu_strategy st = Strategy(s).c();
        check(csrc_gpu_plan_create(&m, &st, &plan_));
    }

    /// ParallelSpmv(const CsrcRectMatrix&, Strategy) (parallel.hpp:168-181):
    /// any type with .square (CSRC), .rect (CSR tail, local columns) and .m.
    template <class R, class S, std::enable_if_t<has_square<R>::value, int> = 0>
    ParallelSpmv(const R& r, const S& s) : n_(r.square.n) {
        const csrc_host_matrix m = view(r.square);
        const csrc_gpu_strategy st = Strategy(s).c();
        std::vector<int32_t> rp(r.rect.row_ptr.begin(), r.rect.row_ptr.end());
        std::vector<int32_t> ci(r.rect.col_idx.begin(), r.rect.col_idx.end());
        check(csrc_gpu_plan_create_rect(&m, &st, static_cast<int32_t>(r.m), rp.data(), ci.data(),
                                        r.rect.values.data(), &plan_));
    }

    /// Explicit plan: a csrc::ColorfulPlan (has .coloring) or a
    /// csrc::LocalBuffersPlan (has .partition), parallel.hpp:158-166.
    template <class M, class S, class Plan>
    ParallelSpmv(const M& a, const S& s, const Plan& plan) : n_(a.n) {
        const csrc_host_matrix m = view(a);
        const csrc_gpu_strategy st = Strategy(s).c();
        if constexpr (requires_coloring<Plan>::value) {
            std::vector<int32_t> color(plan.coloring.color.begin(), plan.coloring.color.end());
            check(csrc_gpu_plan_create_colored(&m, &st, color.data(), plan.coloring.n_colors, &plan_));
        } else {
            const auto& bs = plan.partition.block_start;
            std::vector<int32_t> starts(bs.begin(), bs.end());
            check(csrc_gpu_plan_create_partitioned(&m, &st, starts.data(), plan.partition.p, &plan_));
        }
    }

    ParallelSpmv(const ParallelSpmv&) = delete;
    ParallelSpmv& operator=(const ParallelSpmv&) = delete;
    ParallelSpmv(ParallelSpmv&& o) noexcept : plan_(o.plan_), n_(o.n_), timings_(o.timings_) {
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
        timings_ = {t.init_ms / 1e3, t.compute_ms / 1e3, t.accumulate_ms / 1e3};
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

    csrc_gpu_plan_info info() const {
        csrc_gpu_plan_info i;
        check(csrc_gpu_plan_get_info(plan_, &i));
        return i;
    }

private:
    template <class P, class = void>
    struct requires_coloring : std::false_type {};
    template <class P>
    struct requires_coloring<P, std::void_t<decltype(std::declval<P>().coloring)>> : std::true_type {};

    csrc_gpu_plan_t plan_ = nullptr;
    int32_t n_ = 0;
    PhaseTimings timings_;
};

/// spmv_csrc (kernels.hpp:25-43) on the GPU.
template <class M>
Vector spmv_csrc(const M& a, const Vector& x) {
    if (static_cast<long long>(x.size()) != a.n)
        throw Error("spmv_csrc: x has length " + std::to_string(x.size()) + ", expected " +
                    std::to_string(a.n));
    ParallelSpmv ex(a, Strategy());
    return ex.apply(x);
}

/// spmv_csrc_transpose (kernels.hpp:47-65) on the GPU.
template <class M>
Vector spmv_csrc_transpose(const M& a, const Vector& x) {
    if (static_cast<long long>(x.size()) != a.n)
        throw Error("spmv_csrc_transpose: x has length " + std::to_string(x.size()) +
                    ", expected " + std::to_string(a.n));
    ParallelSpmv ex(a, Strategy());
    return ex.apply_transpose(x);
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

}  // namespace gpu
}  // namespace csrc

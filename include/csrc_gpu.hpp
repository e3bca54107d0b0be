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

/// GPU counterpart of csrc::ParallelSpmv (parallel.hpp:151-446). Unlike the
/// reference it copies the matrix (device-resident), so `a` may be freed.
class ParallelSpmv {
public:
    template <class M, class S>
    ParallelSpmv(const M& a, const S& s) : n_(a.n) {
        const csrc_host_matrix m = view(a);
        const csrc_gpu_strategy st = Strategy(s).c();
        check(csrc_gpu_plan_create(&m, &st, &plan_));
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

}  // namespace gpu
}  // namespace csrc

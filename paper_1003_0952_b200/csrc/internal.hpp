// Internal host-side declarations shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#if __has_include(<nvtx3/nvToolsExt.h>)
#include <nvtx3/nvToolsExt.h>
#define CSRC_GPU_NVTX 1
#endif

#include "../../include/csrc_gpu.h"

namespace csrcgpu {

using index_t = std::int32_t;  // csrc::index_t (common.hpp:10)
using count_t = std::int64_t;  // csrc::count_t (common.hpp:11)

// csrc::Error (common.hpp:15-18): every failure crosses the ABI as a nonzero
// status plus this message.
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};

void set_last_error(const std::string& msg);

// NVTX range over one C-ABI call (header-only NVTX3: a no-op unless a tool such
// as nsys/ncu injects itself; `ncu --nvtx --nvtx-include csrc_gpu_spmv/` filters
// the launches of one entry point). Plan builds, host products, band exchanges
// and construction calls show up by their ABI names on a timeline.
struct NvtxRange {
#ifdef CSRC_GPU_NVTX
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
#else  // a translation unit built without the CUDA headers (the standalone fixture library)
    explicit NvtxRange(const char*) {}
#endif
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class F>
int guarded(const char* entry, F&& f) {
    NvtxRange range(entry);
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return 1;
    } catch (...) {
        set_last_error("unknown error");
        return 1;
    }
}

// Validated view of a csrc_host_matrix.
struct MatView {
    index_t n = 0;
    count_t k = 0;
    const double* ad = nullptr;
    const index_t* ia = nullptr;
    const index_t* ja = nullptr;
    const double* al = nullptr;
    const double* au = nullptr;  // == al when value_symmetric
    bool value_symmetric = false;

    count_t nnz_full() const { return n + 2 * k; }
    count_t nnz_stored() const { return n + (value_symmetric ? 1 : 2) * k; }
};

MatView view_of(const csrc_host_matrix* a, bool check_structure);

// ---- host plans (plan_host.cpp) -------------------------------------------
struct RowPartition {
    int p = 1;
    std::vector<index_t> block_start;
    std::vector<count_t> block_nnz;
};
RowPartition partition_by_nnz(const MatView& a, int p);
void effective_ranges(const MatView& a, const std::vector<index_t>& block_start,
                      std::vector<index_t>& lo, std::vector<index_t>& hi);

struct IntervalPlan {
    std::vector<index_t> boundaries;
    std::vector<index_t> iv_begin, iv_end;
    std::vector<index_t> contrib_ptr, contrib;
};
IntervalPlan build_interval_plan(const std::vector<index_t>& lo, const std::vector<index_t>& hi);

std::vector<int32_t> color_rows(const MatView& a, int mode, int order, int* n_colors);
void conflict_edge_counts(const MatView& a, int mode, count_t* n_direct, count_t* n_indirect);

struct Validity {
    bool valid = true;
    index_t row_a = -1, row_b = -1, position = -1;
};
Validity validate_coloring(const MatView& a, const int32_t* color, int n_colors);

}  // namespace csrcgpu
